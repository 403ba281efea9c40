# A/B of a kernel-variant knob on the bench workload (development helper):
#   bash tools/ab_bench.sh KEY=VALUE [rounds]
for i in $(seq 1 ${2:-2}); do
  for t in "" "--tune $1"; do
    python bench.py --no-cpu --no-scale $t 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tune=[$t]', 'value %.5f' % d['value'], 'e2e %.5f' % d['e2e']['value'])"
  done
done
