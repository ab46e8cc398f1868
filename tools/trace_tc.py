"""Experiment: per-K-block timeline of CTA 0 of the LAST launched TC conv (SC_TC_DEBUG=32).
Needs a library built with -DSC_TC_EXPERIMENTS=1 (the trace hooks are compiled out otherwise)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2204_07064_b200 import configs, lib
from paper_2204_07064_b200.runtime import Plan, StreamState
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
op = int(sys.argv[3]) if len(sys.argv) > 3 else 0
m = configs.build(cfg)
plan = Plan(m, precision=prec)
F = configs.CONFIGS[cfg]["frames"]
S = configs.CONFIGS[cfg]["streams"]
st = StreamState(plan, S, F)
st.set_graphs(False)
num, den, cout = plan.sink
x = torch.randn(S, m.in_channels, F, device="cuda")
y = torch.empty(S, cout, F * num // den, device="cuda")
# run ops up to `op` only: run full step; trace holds the last TC launch -> use op index via env
st.process_buffer(x, y, F)
torch.cuda.synchronize()
buf = (C.c_longlong * (32 * 256))()
lib().sc_debug_tc_trace.argtypes = [C.POINTER(C.c_longlong)]
lib().sc_debug_tc_trace(buf)
a = np.array(buf, dtype=np.int64).reshape(32, 256)
t0 = a[0, 0]
print("(units: kilo-cycles of CTA 0 SM clock)")
names = ["tma_issue", "full(xf start)", "xform done", "mma start", "empty/xf comp", "tfull(drain)", "drain end", "mma issued", "q3 ready", "q0 ready", "q1 ready", "q2 ready"]
print("g   " + " ".join(f"{n:>14s}" for n in names))
st_, en_, sm_ = a[7, :148], a[8, :148], a[9, :148]
t00 = st_.min()
print("CTA start (us) min/max", (st_.min() - t00) / 1e3, (st_.max() - t00) / 1e3,
      " end min/max", (en_.min() - t00) / 1e3, (en_.max() - t00) / 1e3, " distinct SMs", len(set(sm_.tolist())))
order = np.argsort(st_)
print("latest-starting CTAs:", [(int(i), round((st_[i] - t00) / 1e3, 1), int(sm_[i])) for i in order[-6:]])
print("epilogue per tile: [start, after wait, after compute, after arrive]")
for k in range(6):
    e = a[6, 4 * k:4 * k + 4]
    print(k, [round((v - t0) / 1000, 2) for v in e])
for g in range(0, 40):
    print(f"{g:3d} " + " ".join(f"{(a[k, g] - t0) / 1000:14.2f}" if a[k, g] else f"{'-':>14s}" for k in (0, 1, 2, 3, 4, 5, 10, 11, 12, 13, 14, 15)))

print("X2 transform per lane quarter: [landed, math done, A slot free, arrived] (kilo-cycles)")
for g in range(16, 40):
    print(f"{g:3d} " + "  ".join("[" + " ".join(f"{(a[16 + 4 * qq + k, g] - t0) / 1000:6.2f}" if a[16 + 4 * qq + k, g] else "   -  " for k in range(4)) + "]" for qq in range(4)),
          f" mma {(a[3, g] - t0) / 1000:6.2f}")
