set -x
mkdir -p gpurun_out
python tools/tf32_peak.py --out gpurun_out/tf32_peak.json > gpurun_out/tf32_peak.log 2>&1
SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf > gpurun_out/pytest_parity.log 2>&1
tail -5 gpurun_out/pytest_parity.log
(python tools/bf16_err.py; SC_BF16_SKIP=bf16 python tools/bf16_err.py; SC_BF16_STORE=0 python tools/bf16_err.py) > gpurun_out/bf16_err.log 2>&1
python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/b5bf.json 2>&1
SC_BF16_SKIP=bf16 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/b5bf_skipbf.json 2>&1
python bench.py --config 4 --precision bf16 --no-cpu-baseline > gpurun_out/b4bf.json 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs > gpurun_out/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -s 41 -c 41 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs > gpurun_out/ncu5.log 2>&1
cat gpurun_out/tf32_peak.log gpurun_out/bf16_err.log
