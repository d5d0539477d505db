#!/bin/bash
# A/B of sparse-apply build variants (profiles/r1_ab_seg_chunk_variants.log).
# Build here first:  python tools/build_variant.py variants/minb2.so -DTFS_SEG_MINB=2
#                    python tools/build_variant.py variants/c4m4.so -DTFS_SEG_CHUNK=4 -DTFS_SEG_MINB=4
# then on the GPU:   gpurun -- bash tools/ab_seg_variants.sh
# Prints "variant workload rep ms_per_step phases_ms" per run.
cd "$(dirname "$0")/.."
export TFS_ALLOW_VARIANT_LIB=1   # _lib.py honours TFS_LIB only with this set
for rep in 1 2 3; do
 for w in X Z; do
  for v in base minb2 c4m4; do
   if [ $v = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/variants/$v.so; fi
   r=$(timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 200 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('phases_ms',''))")
   echo "$v $w $rep $r"
  done
 done
done
