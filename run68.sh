export SC_SKIP_BUILD=1
timeout 600 python -m pytest "tests/test_gpu_f16split.py::test_f16_and_tf32_splits_agree" -x -q -m gpu 2>&1 | tail -30
