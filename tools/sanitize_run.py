#!/usr/bin/env python
"""compute-sanitizer workload: the streaming path through the C-ABI at small stream counts,
covering the state machinery the kernels share:
  * cfg2 (chained k3 + 1x1 tensor-core conv), cfg3 (strided / ConvT polyphase), cfg5 (PQMF,
    window-mode tiles, densified head) — fp32, and cfg2 / cfg5 bf16;
  * strip wrap-around (carry_kernel): run with SC_STRIP_K=3 so a few calls force a carry;
  * subset reset between calls; cfg5 phase state (B = 512 < compression ratio 2048);
  * CUDA-graph replay and eager launches.
Checks the outputs are finite; parity itself is tests/test_gpu_parity.py.  Usage:
  SC_STRIP_K=3 compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2204_07064_b200 import configs  # noqa: E402
from paper_2204_07064_b200.runtime import Plan, StreamState  # noqa: E402

CASES = [  # cfg, precision, streams, parts, reset-after-call
    (2, "fp32", 3, [512, 256, 512, 768], 1),
    (3, "fp32", 2, [1024, 1024, 2048], 1),
    (5, "fp32", 2, [2048, 2048, 2048], 1),
    (5, "fp32", 2, [512] * 8, 3),        # phase state; reset at a period boundary (4 x 512)
    (2, "bf16", 2, [512, 512, 1024], 1),
    (5, "bf16", 2, [2048, 2048], 0),
]
only = os.environ.get("SAN_ONLY")
for i, (cfg, prec, S, parts, rst) in enumerate(CASES):
    if only is not None and str(i) not in only.split(","):
        continue
    m = configs.build(cfg, seed=cfg)
    x = configs.batch_input(cfg, range(S), m.in_channels, sum(parts), seed=cfg)
    plan = Plan(m, precision=prec, device=0)
    num, den, cout = plan.sink
    st = StreamState(plan, S, max(parts))
    st.set_graphs(i % 2 == 0)
    xd = torch.from_numpy(x).cuda()
    t0 = 0
    for j, p in enumerate(parts):
        y = torch.empty((S, cout, p * num // den), device="cuda")
        st.process_buffer(xd[:, :, t0:t0 + p].contiguous(), y, p)
        torch.cuda.synchronize()
        assert torch.isfinite(y).all(), (cfg, prec, j)
        t0 += p
        if j == rst:
            st.reset([S - 1])
    print(f"case {i}: cfg{cfg} {prec} streams={S} parts={parts} ok", flush=True)
print("sanitize_run: done")
