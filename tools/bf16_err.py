"""Diagnostic: bf16-variant error vs the fp32 oracle (NRMSE, max/RMS, correlation) per config.
Run under different SC_BF16_SKIP / SC_BF16_STORE settings to separate operand rounding from
activation-storage rounding.  cfg5 runs past its 32848-sample latency."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pqmf_design
from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.runtime import Plan, StreamState

tag = " ".join(f"{k}={os.environ[k]}" for k in ("SC_BF16_SKIP", "SC_BF16_STORE") if k in os.environ) or "default"
for cfg, S, parts, rs in [(2, 2, [2048, 2048], None), (3, 2, [4096, 4096], None), (4, 4, [1] * 8, None),
                          (4, 4, [1] * 8, 0.5), (5, 2, [2048] * 20, None)]:
    m = configs.build(cfg, seed=cfg, res_scale=rs)
    x = configs.batch_input(cfg, range(S), m.in_channels, sum(parts), seed=cfg)
    yo = po.run(pqmf_design.twin(m), x, parts, "stream")
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
    print(f"[{tag}] cfg{cfg}{'' if rs is None else f' res_scale={rs}'} nrmse={nrmse:.3e} "
          f"max/rms={np.abs(yg - yo).max() / rms:.3e} corr={np.corrcoef(yg.ravel(), yo.ravel())[0, 1]:.6f}", flush=True)
