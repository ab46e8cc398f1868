SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f16split.py -q -rf -x > gpurun_out/pytest_hf.log 2>&1
tail -2 gpurun_out/pytest_hf.log
for pdl in 1 0 1 0; do
for S in 2048 16384; do
SC_PDL=$pdl timeout 600 python bench.py --no-cpu-baseline --streams $S > gpurun_out/b.json 2>/dev/null
python -c "import json; a=json.load(open('gpurun_out/b.json')); print('pdl $pdl streams $S', round(a['ms_per_step'],3))"
done; done
