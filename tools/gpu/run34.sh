SC_SKIP_BUILD=1 timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>gpurun_out/b.err
tail -2 gpurun_out/b.err
python -c "import json; a=json.load(open('gpurun_out/b.json')); print('cfg5', round(a['ms_per_step'],3), a['e2e']['value']/1e9, a['gpu_launches'], [ (k,v) for k,v in a['profile_ms'].items() if 'pqmf' in k or 'gress' in k])"
