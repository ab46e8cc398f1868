#!/usr/bin/env python
"""Per-launch table from a bench.py JSON line: ms, algorithmic TFLOP/s (or GB/s for non-GEMM
launches is not computed here), and the share of the step.   python tools/prof_table.py bench.json"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2204_07064_b200 import configs  # noqa: E402
from paper_2204_07064_b200.runtime import Plan  # noqa: E402

d = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])
cfg = int(d["config"]["workload"].split(":")[0][3:])
streams, frames = d["config"]["streams_per_gpu"], d["config"]["frames_per_call"]
plan = Plan(configs.build(cfg, seed=0), precision=d["config"]["precision"], device=-1)
macs = plan.op_macs()
prof = d["profile_ms"]
tot = sum(prof.values())
print(f"cfg{cfg} {d['config']['precision']}: step (profiled, un-graphed) {tot:.3f} ms, timed {d['ms_per_step']:.3f} ms")
for name, ms in sorted(prof.items(), key=lambda kv: -kv[1]):
    tf = ""
    if name.startswith("op"):
        ois = [int(k) for k in name.split()[0][2:].split("+")]
        fl = 2.0 * sum(macs[i] for i in ois) * frames * streams
        tf = f"{fl / (ms / 1e3) / 1e12:7.1f} TF/s"
    print(f"{ms:8.4f} ms {100 * ms / tot:5.1f}%  {tf:>14}  {name}")
