"""Diagnostic: determinism and mode-equivalence of the 3xFP16 X2 kernels (awin on/off, stream
subsets) for cfg4 / cfg5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.runtime import Plan, StreamState


def run(cfg, S, calls, env=None, pick=None, seed=0):
    if env:
        os.environ.update(env)
    m = configs.build(cfg, seed=cfg)
    plan = Plan(m)
    num, den, cout = plan.sink
    F = configs.CONFIGS[cfg]["frames"]
    g = torch.Generator(device="cuda").manual_seed(seed)
    xs = [torch.randn((S, m.in_channels, F), device="cuda", generator=g) for _ in range(calls)]
    if pick is not None:
        xs = [x[pick].contiguous() for x in xs]
    st = StreamState(plan, xs[0].shape[0], F)
    ys = []
    for x in xs:
        y = torch.empty((x.shape[0], cout, F * num // den), device="cuda")
        st.process_buffer(x, y, F)
        ys.append(y)
    torch.cuda.synchronize()
    if env:
        for k in env:
            del os.environ[k]
    return torch.cat(ys, 2).cpu().numpy()


for cfg, S, calls in [(4, 256, 4), (5, 256, 3)]:
    a = run(cfg, S, calls)
    b = run(cfg, S, calls)
    c = run(cfg, S, calls, env={"SC_AWIN": "0"})
    pick = [0, S // 2 + 1, S - 1]
    d = run(cfg, S, calls, pick=pick)
    print(f"cfg{cfg}: det {np.array_equal(a, b)} ({np.abs(a-b).max():.3e})  awin0 {np.array_equal(a, c)} ({np.abs(a-c).max():.3e})"
          f"  subset {np.array_equal(a[pick], d)} ({np.abs(a[pick]-d).max():.3e})", flush=True)
