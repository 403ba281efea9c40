# JDQMR inner-stopping sweep (development helper)
for k in c1 c2 c3L; do
  JD=1 timeout 300 python tools/time_config.py $k full 1 | grep rep
  JD=1 LFAC=1.0 timeout 300 python tools/time_config.py $k full 1 | grep rep
  JD=1 ETOL=0.1 timeout 300 python tools/time_config.py $k full 1 | grep rep
done
JD=1 timeout 300 python tools/time_config.py c3S full 1 60000 | grep rep
JD=1 timeout 300 python tools/time_config.py c5 full 1 20000 | grep rep
JD=1 timeout 300 python tools/jd_diag.py c2 > gpurun_out/jdd.log 2>&1
JD=1 timeout 300 python tools/jd_diag.py c3S full 30000 > gpurun_out/jdd3.log 2>&1
