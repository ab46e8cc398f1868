"""Soak / determinism run on the GPU: many streaming calls per configuration at (near) full
stream counts, twice with the same seeded inputs — output hashes must match and every value stay
finite.  python tools/soak.py  (about a minute on a B200)."""
import sys, os, hashlib
sys.path.insert(0, os.getcwd())
import torch
from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.runtime import Plan, StreamState

def run(cfg, S, F, calls, seed):
    m = configs.build(cfg, seed=cfg)
    plan = Plan(m)
    num, den, cout = plan.sink
    st = StreamState(plan, S, F)
    g = torch.Generator(device="cuda").manual_seed(seed)
    h = hashlib.sha256()
    y = torch.empty((S, cout, F * num // den), device="cuda")
    acc = torch.zeros((), device="cuda", dtype=torch.float64)
    for c in range(calls):
        x = torch.randn((S, m.in_channels, F), device="cuda", generator=g)
        st.process_buffer(x, y, F)
        if c % 16 == 15 or c == calls - 1:
            h.update(y.cpu().numpy().tobytes())
        acc += y.double().abs().sum()
    torch.cuda.synchronize()
    assert torch.isfinite(acc).item()
    return h.hexdigest()

for cfg, S, F, calls in [(5, 16384, 2048, 96), (5, 4096, 512, 128), (5, 3000, 8192, 12), (4, 4096, 1, 160), (3, 1024, 4096, 64), (5, 333, 2048, 64)]:
    a = run(cfg, S, F, calls, 1)
    b = run(cfg, S, F, calls, 1)
    print(cfg, S, F, calls, "identical" if a == b else "DIFFERENT", a[:12], flush=True)
    assert a == b
print("soak ok")
