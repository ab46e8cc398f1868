python tools/diag_x2.py 2>&1 | tail -5
SC_FP32_SPLIT=tf32 python tools/diag_x2.py 2>&1 | tail -3
