mkdir -p gpurun_out
SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_f16split.py -q -rf > gpurun_out/pytest_f16.log 2>&1
tail -8 gpurun_out/pytest_f16.log
