#!/bin/bash
# The round's measurement runs on an N-GPU box (N = 1, 2 or 4): GPU tests, bench lines for
# X / Z / F (and L, X-fp32, the optimizers, the oracle arm at N = 1), the null step, and NVLink
# counters around the N > 1 runs.  Output: gpurun_out/final/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/final
run() {  # name, then the bench arguments
  local name=$1; shift
  if [ "$N" -gt 1 ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $N "$@" > $O/$name.json 2> $O/$name.err
  else
    timeout 600 python bench.py "$@" > $O/$name.json 2> $O/$name.err
  fi
  echo "$name rc=$?"
}
nvidia-smi topo -m > $O/topo_n$N.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf > $O/pytest_gpu_n$N.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu_n$N.log
nvidia-smi nvlink -gt d > $O/nvlink_before_n$N.txt 2>&1
run bench_X_n$N --steps 200 --warmup 10
nvidia-smi nvlink -gt d > $O/nvlink_after_X_n$N.txt 2>&1
run bench_F_n$N --workload F --steps 50 --warmup 5
run bench_Z_n$N --workload Z --steps 20 --warmup 3
run null_n$N --null-step --steps 100 --warmup 10
if [ "$N" -eq 1 ]; then
  run bench_L_n1 --workload L --steps 200 --warmup 10
  run bench_X_f32_n1 --dtype f32 --steps 20 --warmup 3 --no-cpu-baseline
  run bench_X_momentum_n1 --optimizer momentum --steps 100 --warmup 5 --no-cpu-baseline
  run bench_X_adagrad_n1 --optimizer adagrad --steps 100 --warmup 5 --no-cpu-baseline
  run ref_X_n1 --impl reference --steps 3 --warmup 1
fi
ls -la $O
