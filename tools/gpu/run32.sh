SC_SKIP_BUILD=1 timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
python -c "import json; a=json.load(open('gpurun_out/b.json')); print('cfg5', round(a['ms_per_step'],3), a['clocks']['sm_mhz'], a['step_roofline']['layerwise'])"
done
python tools/prof_table.py gpurun_out/b.json > gpurun_out/prof.txt; grep -E "64->64|64->32|step" gpurun_out/prof.txt
