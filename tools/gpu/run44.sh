SC_SKIP_BUILD=1 timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
python -c "import json; a=json.load(open('gpurun_out/b.json')); print('cfg5', round(a['ms_per_step'],3), a['clocks']['sm_mhz'], (a['step_roofline']['layerwise'] or {}).get('frac'))"
done
python tools/prof_table.py gpurun_out/b.json 2>/dev/null | head -24
