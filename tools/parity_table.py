"""Max |gpu - oracle| / RMS(oracle) per config for the fp32-accurate splits (3xFP16 default,
3xTF32) and the bf16 variant — the numbers DESIGN.md §5 quotes.  GPU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import oracle_model
from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from test_gpu_parity import run_gpu, rel_err

CASES = [(1, 1, [2048] * 64), (2, 4, [2048, 2048]), (3, 3, [4096, 4096]), (4, 4, [1] * 8),
         (5, 2, [2048] * 20), (5, 2, [8192] * 5)]  # (B = 512 < ratio runs in phase state: tests/test_gpu_parity.py)
for cfg, S, parts in CASES:
    m = configs.build(cfg, seed=cfg)
    x = configs.batch_input(cfg, range(S), m.in_channels, sum(parts), seed=cfg)
    y_or = po.run(oracle_model(cfg, seed=cfg), x, parts, "stream")
    row = []
    for tag, env, prec in [("3xFP16", None, "fp32"), ("3xTF32", "tf32", "fp32"), ("bf16", None, "bf16")]:
        if env:
            os.environ["SC_FP32_SPLIT"] = env
        y, _, _ = run_gpu(m, x, parts, precision=prec)
        os.environ.pop("SC_FP32_SPLIT", None)
        err, rms = rel_err(y, y_or)
        row.append(f"{tag} {err:.2e}")
    print(f"cfg{cfg} streams={S} parts={len(parts)}x{parts[0]}: " + "  ".join(row), flush=True)
