mkdir -p gpurun_out/prof3
O=gpurun_out/prof3
timeout 300 python bench.py --workload X --steps 20 --warmup 5 --no-cpu-baseline > $O/plainX.json 2> $O/plainX.err; echo plainX=$?
timeout 300 python bench.py --workload Z --steps 10 --warmup 3 --no-cpu-baseline > $O/plainZ.json 2> $O/plainZ.err; echo plainZ=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_X.csv python bench.py --workload X --steps 3 --warmup 3 --no-cpu-baseline > $O/ncuX.log 2>&1; echo ncuX=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_Z.csv python bench.py --workload Z --steps 3 --warmup 3 --no-cpu-baseline > $O/ncuZ.log 2>&1; echo ncuZ=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_window|gather_vec4|sort_segment|digit_scatter|make_keys|heads" --launch-skip 40 -c 12 -o $O/z_sparse python bench.py --workload Z --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_sparse.log 2>&1; echo ncusparse=$?
ls -la $O
