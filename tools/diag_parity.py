"""Diagnostic: per-config / per-prefix max|gpu-oracle|/RMS for the TC and SIMT paths."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.graph import Model
from paper_2204_07064_b200.runtime import Plan, StreamState


PREC = os.environ.get("SC_PREC", "fp32")


def run(m, x, parts):
    plan = Plan(m, precision=PREC)
    num, den, cout = plan.sink
    S = x.shape[0]
    st = StreamState(plan, S, max(parts))
    xd = torch.from_numpy(x).cuda()
    outs, t0 = [], 0
    for p in parts:
        y = torch.empty((S, cout, p * num // den), device="cuda")
        st.process_buffer(xd[:, :, t0:t0 + p].contiguous(), y, p)
        outs.append(y)
        t0 += p
    torch.cuda.synchronize()
    return torch.cat(outs, 2).cpu().numpy(), plan


def err(m, x, parts):
    yo = po.run(m, x, parts, "stream")
    yg, plan = run(m, x, parts)
    rms = np.sqrt(np.mean(yo.astype(np.float64) ** 2))
    return np.abs(yg - yo).max() / rms, rms, plan


def prefixes3():
    chans = [16, 64, 128, 256, 512]
    strides = [4, 4, 4, 2]
    out = []
    for n in range(1, 9):
        m = Model(16, 3)
        k = 0
        for i, s in enumerate(strides):
            if k == n: break
            if i: m.leaky_relu(0.2)
            m.conv(chans[i], chans[i + 1], 2 * s + 1, stride=s, padding=(s, s)); k += 1
        dec = strides[::-1]; rc = chans[::-1]
        for i, r in enumerate(dec):
            if k == n: break
            m.leaky_relu(0.2)
            m.conv_transpose(rc[i], rc[i + 1], 2 * r, r, padding=(r, r - 1)); k += 1
        out.append((f"cfg3[:{n}]", m))
    return out


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, m in prefixes3():
        x = configs.batch_input(3, range(3), 16, 8192, seed=3)
        e, rms, plan = err(m, x, [4096, 4096])
        print(f"{name:12s} err/rms={e:.3e} rms={rms:.3e}", flush=True)
    for cfg, S, parts in [(1, 1, [2048] * 8), (2, 4, [2048, 2048]), (3, 3, [4096, 4096]), (4, 4, [1, 1, 1]), (5, 2, [2048, 2048])]:
        m = configs.build(cfg, seed=cfg)
        x = configs.batch_input(cfg, range(S), m.in_channels, sum(parts), seed=cfg)
        e, rms, plan = err(m, x, parts)
        print(f"cfg{cfg} err/rms={e:.3e} rms={rms:.3e}", flush=True)
        if cfg == 3:
            print(plan.describe())
