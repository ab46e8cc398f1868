SC_SKIP_BUILD=1 timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --streams 2048 > gpurun_out/bench_2048.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_16k.json 2>/dev/null
python -c "
import json; a=json.load(open('gpurun_out/bench_16k.json')); b=json.load(open('gpurun_out/bench_2048.json'))
print('16384', a['ms_per_step'], '2048', b['ms_per_step'], 'proj 1->8', a['ms_per_step']/b['ms_per_step'])
print('op18', a['profile_ms']['op18 conv 1024->256 K3 d1 [tc]'], b['profile_ms']['op18 conv 1024->256 K3 d1 [tc]'])"
