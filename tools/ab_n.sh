#!/bin/bash
# A/B of libtfs builds at N GPUs (the bench X step): bash tools/ab_n.sh N base variants/X.so ...
cd "$(dirname "$0")/.."
export TFS_ALLOW_VARIANT_LIB=1
N=$1; shift
for rep in 1 2; do
 for v in "$@"; do
  if [ "$v" = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/$v; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 100 --warmup 10 --no-cpu-baseline > /tmp/abn.json 2>/tmp/abn.err || tail -3 /tmp/abn.err
  python -c "
import json; d=json.loads(open('/tmp/abn.json').read().strip().splitlines()[-1])
print('$v N=$N rep $rep', round(d['ms_per_step']*1e3,1), round(d['value']/1e6,2))"
 done
done
