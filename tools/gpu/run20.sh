mkdir -p gpurun_out
SC_SKIP_BUILD=1 timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
tail -4 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg5.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac_of_path_ceiling'], d['clocks'])"
