#!/bin/bash
# A/B of an environment switch on the step (1 GPU): bash tools/ab_env.sh "TFS_PDL=0" "TFS_PDL=1"
cd "$(dirname "$0")/.."
for rep in $(seq 1 ${AB_REPS:-2}); do
 for w in X Z; do
  for e in "$@"; do
   steps=100; [ $w = Z ] && steps=20
   env $e timeout 300 python bench.py --workload $w --steps $steps --warmup 5 --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err || tail -3 /tmp/ab.err
   python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$e $w', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value']/1e6,2), 'ssm', round(r['sampled_softmax_call']['ms']*1e3,1), {k: round(v['ms']*1e3,1) for k, v in r['kernels'].items()})"
  done
 done
done
