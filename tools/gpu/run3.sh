set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
SC_SKIP_BUILD=1 timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config 5 --streams 2048 --no-cpu-baseline > gpurun_out/bench_cfg5_2048.json 2> gpurun_out/bench_cfg5_2048.err
cat gpurun_out/bench_cfg5.json gpurun_out/bench_ref.json gpurun_out/bench_cfg5_2048.json
