#!/bin/bash
# A/B of libtfs variants on whole steps: "N variant..." -> ms/step and words/s per variant
# (N = 1: bench.py; N > 1: torchrun).  gpurun [--gpus N] -- bash tools/ab_step.sh N base v.so ...
cd "$(dirname "$0")/.."
export TFS_ALLOW_VARIANT_LIB=1
N=$1; shift
for rep in 1 2; do
 for v in "$@"; do
  if [ "$v" = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/$v; fi
  if [ "$N" = 1 ]; then
    timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > /tmp/ab.json 2>/dev/null
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 200 --warmup 10 > /tmp/ab.json 2>/dev/null
  fi
  python -c "import json;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]);print('$v N=$N rep $rep', round(d['ms_per_step']*1e3,1), round(d['value']/1e6,2))"
 done
done
