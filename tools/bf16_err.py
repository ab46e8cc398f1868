"""Diagnostic: bf16-variant error vs the fp32 oracle (NRMSE, max/RMS, correlation) per config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.runtime import Plan, StreamState

for cfg, S, parts in [(2, 2, [2048, 2048]), (3, 2, [4096, 4096]), (4, 4, [1] * 8), (5, 2, [2048] * 8)]:
    m = configs.build(cfg, seed=cfg)
    x = configs.batch_input(cfg, range(S), m.in_channels, sum(parts), seed=cfg)
    yo = po.run(m, x, parts, "stream")
    plan = Plan(m, precision="bf16")
    num, den, cout = plan.sink
    st = StreamState(plan, S, max(parts))
    xd = torch.from_numpy(x).cuda()
    outs, t0 = [], 0
    for p in parts:
        y = torch.empty((S, cout, p * num // den), device="cuda")
        st.process_buffer(xd[:, :, t0:t0 + p].contiguous(), y, p)
        outs.append(y); t0 += p
    torch.cuda.synchronize()
    yg = torch.cat(outs, 2).cpu().numpy()
    rms = np.sqrt(np.mean(yo.astype(np.float64) ** 2))
    nrmse = np.sqrt(np.mean((yg.astype(np.float64) - yo) ** 2)) / rms
    print(f"cfg{cfg} nrmse={nrmse:.3e} max/rms={np.abs(yg - yo).max() / rms:.3e} corr={np.corrcoef(yg.ravel(), yo.ravel())[0, 1]:.6f}", flush=True)
