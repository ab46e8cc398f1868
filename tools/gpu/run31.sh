mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs > gpurun_out/plain5.json 2> gpurun_out/plain5.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -s 43 -c 43 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs > gpurun_out/ncu5.log 2>&1
python tools/ncu_traffic.py gpurun_out/launches_cfg5.csv gpurun_out/plain5.json 5 profiles/traffic.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 23 --launch-count 1 -f -o gpurun_out/full_op24 python tools/ncu_one.py 5 16384 > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/full_op24.ncu-rep --page raw --csv > gpurun_out/full_op24_raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_full.log
