# A/B of an environment switch on the bench workload (development helper):
#   bash tools/ab_env.sh NAME=VALUE [rounds]
for i in $(seq 1 ${2:-2}); do
  for e in "" "$1"; do
    env $e python bench.py --no-cpu --no-scale 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('env=[$e]', 'value %.5f' % d['value'], 'e2e %.5f' % d['e2e']['value'], 'mv', d['result']['stage1_matvecs'], 'conv', d['result']['converged'])"
  done
done
