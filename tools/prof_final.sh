#!/bin/bash
# The round's ncu evidence on one GPU: launch lists (device time + DRAM bytes per launch) of
# bench X and Z, and full-section captures of the apply and GEMM kernels.  -> gpurun_out/prof_final/
cd "$(dirname "$0")/.."
O=gpurun_out/prof_final; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -c 400 --csv --log-file $O/launches_X.csv python bench.py --workload X --steps 3 --warmup 3 --no-cpu-baseline > $O/ncuX.log 2>&1; echo launchesX=$?
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file $O/launches_Z.csv python bench.py --workload Z --steps 3 --warmup 3 --no-cpu-baseline > $O/ncuZ.log 2>&1; echo launchesZ=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_window|gemm_kernel|gather_vec4" --launch-skip 12 -c 9 -o $O/x_full python bench.py --workload X --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_x_full.log 2>&1; echo fullX=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_window|gather_vec4" --launch-skip 8 -c 4 -o $O/z_sparse python bench.py --workload Z --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_z.log 2>&1; echo fullZ=$?
ls -la $O
