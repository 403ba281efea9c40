set -x
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 python tools/kbench.py c4 > gpurun_out/kbench_c4.log 2>&1; echo kb=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-scale > gpurun_out/ncu_list.log 2>&1; echo list=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cgs_fused|syev_update|ritz_wide|csr_tile_pipe|gram1_vec" -s 200 -c 6 -o gpurun_out/r01d_c2_top python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-scale > gpurun_out/ncu_full.log 2>&1; echo full=$?
