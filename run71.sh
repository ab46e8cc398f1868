export SC_SKIP_BUILD=1
mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
bash tools/bench_all.sh; cp gpurun_out/bench_all.jsonl $O/bench_all.jsonl
python tools/summarize_bench.py $O/bench_all.jsonl > $O/bench_all.md 2>&1
timeout 900 python tools/parity_table.py > $O/parity_table.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -c 160 --csv --log-file $O/ncu_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-graphs --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 23 --launch-count 1 -f -o $O/op24 python tools/ncu_one.py 5 > $O/ncu_op24.log 2>&1
ncu -i $O/op24.ncu-rep --page raw --csv > $O/op24_raw.csv 2>/dev/null
ncu -i $O/op24.ncu-rep --page source --csv --print-source sass > $O/op24_sass.csv 2>/dev/null
rm -f $O/op24.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 28 --launch-count 1 -f -o $O/op29 python tools/ncu_one.py 5 > $O/ncu_op29.log 2>&1
ncu -i $O/op29.ncu-rep --page source --csv --print-source sass > $O/op29_sass.csv 2>/dev/null
ncu -i $O/op29.ncu-rep --page raw --csv > $O/op29_raw.csv 2>/dev/null
rm -f $O/op29.ncu-rep
ls -la $O
