import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_07064_b200 import configs
from tools.diag_parity import err
for S, parts in [(4, [8192] * 4), (8, [2048] * 16)]:
    m = configs.build(5, seed=5)
    x = configs.batch_input(5, range(S), 1, sum(parts), seed=5)
    t = time.time()
    e, rms, _ = err(m, x, parts)
    print(f"cfg5 S={S} T={sum(parts)} err/rms={e:.3e} rms={rms:.3e} ({time.time()-t:.1f}s)", flush=True)
