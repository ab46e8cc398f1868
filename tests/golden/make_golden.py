"""Generate golden vectors from the REFERENCE's own compiled code (oracle/_ref, built from the
unmodified /root/reference/proj/src/kernels.cpp by oracle/Makefile).  Run in the builder
container (where the reference tree exists); the .npz fixtures are committed and travel.

  python tests/golden/make_golden.py
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import pyoracle as po  # noqa: E402
from paper_2204_07064_b200 import configs  # noqa: E402
from paper_2204_07064_b200.graph import Model  # noqa: E402

assert po.ref_available(), "oracle/_ref/libref_streamconv.so missing: run `make -C oracle`"
rng = np.random.default_rng(2204_07064)

# 1) conv1d (kernels.cpp:73-104) on random shapes, serial path (conv1d_serial)
cases = []
for (M, N, K, S, d, L) in [(1, 1, 3, 1, 1, 8), (2, 3, 4, 1, 2, 17), (3, 2, 5, 2, 1, 23), (4, 4, 3, 3, 3, 40),
                           (8, 8, 16, 1, 1, 64), (5, 7, 9, 4, 1, 130), (16, 16, 7, 1, 5, 100)]:
    x = rng.uniform(-1, 1, (M, L)).astype(np.float32)
    w = rng.uniform(-1, 1, (N, M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, N).astype(np.float32)
    y = po.conv1d(x, w, b, S, d, use_ref=True)
    cases.append(dict(x=x, w=w, b=b, S=S, d=d, y=y))
np.savez_compressed(ROOT / "tests/golden/ref_conv1d.npz",
                    **{f"{k}{i}": v for i, c in enumerate(cases) for k, v in c.items()}, n=len(cases))

# 2) zero_upsample / pad_zeros / activation through the reference
x = rng.uniform(-2, 2, (3, 11)).astype(np.float32)
np.savez_compressed(ROOT / "tests/golden/ref_ops.npz", x=x,
                    zup3=po.zero_upsample(x, 3, use_ref=True),
                    pad21=po.pad_zeros(x, 2, 1, use_ref=True),
                    lrelu02=po.activation(x, 2, 0.2, use_ref=True).reshape(x.shape),
                    tanh=po.activation(x, 1, 0.0, use_ref=True).reshape(x.shape))

# 3) streaming outputs of small graphs with the REFERENCE conv1d inside the SPEC
#    process_buffer restatement (these pin the executor + causalize on reference arithmetic)
sys.path.insert(0, str(ROOT / "tests" / "golden"))
from models import small_models  # noqa: E402

out = {}
for name, m in small_models().items():
    r = po.graph_info(m)["ratio"]
    T = 16 * r
    x = rng.standard_normal((2, m.in_channels, T)).astype(np.float32)
    parts = [r, 2 * r, 7 * r, 6 * r]
    out[f"{name}_x"] = x
    out[f"{name}_parts"] = np.array(parts)
    out[f"{name}_y"] = po.run(m, x, parts, "stream", use_ref=True)
np.savez_compressed(ROOT / "tests/golden/ref_stream.npz", **out)
print("golden vectors written")
