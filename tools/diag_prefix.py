"""Diagnostic: error growth along a config's node list (prefix models), TC vs oracle."""
import copy
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from tools.diag_parity import err

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 2
m = configs.build(cfg, seed=cfg)
parts = [2048] * nb if cfg != 4 else [1] * nb
x = configs.batch_input(cfg, range(S), m.in_channels, sum(parts), seed=cfg)
depth = 0
cuts = []
for k, nd in enumerate(m.nodes):
    if nd["kind"] == 3:
        depth += 1
    elif nd["kind"] == 4:
        depth -= 1
    if depth == 0 and nd["kind"] in (0, 1, 4):
        cuts.append(k + 1)
for k in cuts:
    mm = copy.copy(m)
    mm.nodes = m.nodes[:k]
    # output must be frame-aligned: prefixes ending at rate != 1 still work (sink rate)
    e, rms, plan = err(mm, x, parts)
    last = m.nodes[k - 1]
    print(f"nodes[:{k:3d}] kind={last['kind']} {last['in_channels']}->{last['out_channels']} K{last['taps']} "
          f"S{last['stride']}  err/rms={e:.3e} rms={rms:.3e}", flush=True)
