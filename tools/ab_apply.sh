#!/bin/bash
# A/B of the sparse apply: per-call apply / plan times and HBM fractions at X and Z (1 GPU).
cd "$(dirname "$0")/.."
export TFS_ALLOW_VARIANT_LIB=1
for rep in 1 2; do
 for w in X Z; do
  for v in "$@"; do
   if [ "$v" = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/$v; fi
   steps=100; [ $w = Z ] && steps=20
   timeout 300 python bench.py --workload $w --steps $steps --warmup 5 --no-cpu-baseline > /tmp/ab.json 2>/dev/null
   python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); c=d['hbm']['calls']
print('$v $w', round(d['ms_per_step']*1e3,1), {k: (round(v['us'],1), round(v['frac'],2)) for k, v in c.items() if k.startswith('apply')}, round(d['hbm']['scatter_frac'],3))"
  done
 done
done
