SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f16split.py -q -rf -x -k "fp32 or bit_identity or repeat" > gpurun_out/pytest_hf.log 2>&1
tail -2 gpurun_out/pytest_hf.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
python -c "import json; a=json.load(open('gpurun_out/b.json')); print('cfg5', round(a['ms_per_step'],3), a['clocks']['sm_mhz'], (a['step_roofline']['layerwise'] or {}).get('frac'))"
done
python tools/prof_table.py gpurun_out/b.json 2>/dev/null | head -14
export SC_LIB_PATH=exp/libstreamconv_b200.so
SC_TC_TRACE_OP=29 python tools/trace_tc.py 5 fp32 > gpurun_out/trace_a.txt 2>&1
