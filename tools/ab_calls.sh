#!/bin/bash
# A/B of libtfs builds on the HBM-bound calls: step time and per-call gather / apply times and
# HBM fractions at X and Z (1 GPU).  Usage: bash tools/ab_calls.sh base variants/NAME.so ...
cd "$(dirname "$0")/.."
export TFS_ALLOW_VARIANT_LIB=1
for rep in $(seq 1 ${AB_REPS:-2}); do
 for w in X Z; do
  for v in "$@"; do
   if [ "$v" = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/$v; fi
   steps=100; [ $w = Z ] && steps=20
   timeout 300 python bench.py --workload $w --steps $steps --warmup 5 --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err || tail -3 /tmp/ab.err
   python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); c=d['hbm']['calls']
print('$v $w', round(d['ms_per_step']*1e3,1), {k: (round(v['us'],1), round(v['frac'],2)) for k, v in c.items()}, 'plan', {k: round(v,1) for k, v in d['hbm']['scatter_plan_us'].items()})"
  done
 done
done
