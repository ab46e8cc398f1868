mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs > gpurun_out/plain5.json 2> gpurun_out/plain5.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -s 41 -c 41 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs > gpurun_out/ncu5.log 2>&1
python tools/ncu_traffic.py gpurun_out/launches_cfg5.csv gpurun_out/plain5.json 5 profiles/traffic.json
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "import json; a=json.load(open('gpurun_out/bench_default.json')); print(a['value'], a['ms_per_step'], a['e2e']['value'], a['roofline']['frac_of_path_ceiling'], a['step_roofline']['layerwise'], a['roofline']['traffic'])"
