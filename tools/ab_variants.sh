#!/bin/bash
# A/B of libtfs build variants on the GPU: for every .so given (or "base" = the product build),
# bench.py on workloads X and Z; prints "variant workload ms_per_step gemm_stats gemm_grad|- grad_pass|-
# gemm_store (us)".  Build variants first:
#   python tools/build_variant.py variants/NAME.so -DSWITCH=VALUE
# then:  gpurun -- bash tools/ab_variants.sh base variants/NAME.so ...
cd "$(dirname "$0")/.."
export TFS_ALLOW_VARIANT_LIB=1
for rep in ${AB_REPS:-1 2}; do
 for w in X Z; do
  for v in "$@"; do
   if [ "$v" = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/$v; fi
   steps=100; [ $w = Z ] && steps=20
   r=$(timeout 300 python bench.py --workload $w --no-cpu-baseline --steps $steps --warmup 5 --phase-steps 10 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['roofline']['kernels']
print(round(d['ms_per_step']*1e3,1), *(round(k[n]['ms']*1e3,1) if n in k else '-' for n in ('gemm_stats','gemm_grad','grad_pass','gemm_store')), d['library']['path'])")
   echo "$v $w $rep $r"
  done
 done
done
