SC_SKIP_BUILD=1 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f16split.py -q -rf -x -k "fp32 or bit_identity or repeat" > gpurun_out/pytest_hf.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_hf.log
timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
echo "bench rc=$?"
python -c "import json; a=json.load(open('gpurun_out/b.json')); print('cfg5', round(a['ms_per_step'],3), a['clocks']['sm_mhz'])"
python tools/prof_table.py gpurun_out/b.json 2>/dev/null | head -12
