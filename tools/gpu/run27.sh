SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_redzone.py -q -rf > gpurun_out/pytest_rz.log 2>&1
tail -15 gpurun_out/pytest_rz.log
