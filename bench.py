#!/usr/bin/env python
"""bench.py — aggregate streamed samples/s (x real-time @ 48 kHz) over concurrent streams.

Metric (BASELINE.json): streamed audio samples/s over concurrent independent streams and its
roofline fraction.  One step = one process_buffer call for every stream of
the rank's shard.  Default workload: BASELINE config 2 (configs[1]: 4 dilated residual
blocks, C=128, 256 streams x 2048 frames, fp32).  `--config N` selects another config.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

N>1: launched by torchrun, one rank per GPU; every rank runs its own shard of streams (weak
scaling: per-GPU streams fixed), no collective on the data path; barrier + CUDA events on
both sides; the max over ranks is the step time.

`value`  : device-resident I/O (inputs already in HBM), CUDA events on the launching stream.
`e2e`    : same metric through the public API with pinned HOST buffers, H2D of the step's
           input and D2H of its output inside the timed region.
`roofline`: dominant kernel (by device time in an un-graphed profiling pass with CUDA events
           between launches) — algorithmic FLOPs per launch / its mean duration, vs the
           measured peak in MEASURED_PEAKS.json.
`cpu_baseline`: the reference's own conv1d (oracle/_ref, kernels.cpp) driven by the SPEC
           process_buffer restatement (oracle/oracle.cpp), all host threads, bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SR = 48000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "bf16"])
    ap.add_argument("--streams", type=int, default=0, help="streams per rank (default: config)")
    ap.add_argument("--total-streams", type=int, default=0,
                    help="strong scaling: split this many streams over the ranks")
    ap.add_argument("--frames", type=int, default=0, help="input frames per call (default: config)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--io", default="fp32", choices=["fp32", "bf16"],
                    help="host buffer type of the e2e leg (bf16: sc_process_host_bf16, half the PCIe bytes)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sus=d.get("bf16_tflops_sustained", 1400.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(cfg, first_stream, streams, cin, frames, slot):
    from paper_2204_07064_b200 import configs
    # seeded per GLOBAL stream index and slot, so any sharding sees the same streams
    return np.stack([configs.stream_input(cfg, first_stream + s, cin, frames, seed=1000 + slot)
                     for s in range(streams)])


def cpu_reference_rate(model, cfg, frames, seconds, threads):
    """Streamed samples/s of the reference CPU path on a bounded sample (all `threads`)."""
    from oracle import pyoracle as po
    from paper_2204_07064_b200.runtime import Plan
    plan_h = Plan(model, device=-1)
    macs_call = plan_h.macs_per_sample * frames  # algorithmic; ConvT adds zero-stuffed MACs
    out_call = plan_h.out_frames(frames)
    use_ref = po.ref_available()
    # ~0.45 GMAC/s per core for the reference's scalar double-accumulate conv
    calls = max(threads, int(round(seconds * threads * 0.7e9 / max(macs_call, 1.0))))
    calls = max(threads, (calls // threads) * threads)
    x = make_inputs(cfg, 0, calls, model.in_channels, frames, slot=0)
    t0 = time.perf_counter()
    po.run(model, x, [frames], "stream", use_ref=use_ref, threads=threads)
    dt = time.perf_counter() - t0
    rate = calls * out_call / dt
    return dict(value=rate, unit="samples/s", cores=threads,
                kind="reference" if use_ref else "port",
                sample=f"{calls} stream-calls x {frames} frames (fresh state), {dt:.1f} s wall, "
                       f"reference conv1d (kernels.cpp) via SPEC process_buffer restatement, "
                       f"OpenMP across streams")


def main():
    args = parse()
    ws, rank, local = dist_setup()
    from paper_2204_07064_b200 import configs
    cfgd = configs.CONFIGS[args.config]
    frames = args.frames or cfgd["frames"]
    streams = args.streams or cfgd["streams"]
    metric = "streamed audio samples/s (x real-time @48kHz) over concurrent streams"
    model = configs.build(args.config, seed=0)

    if args.impl == "reference":
        if rank != 0:
            return 0
        threads = len(os.sched_getaffinity(0))
        vals = []
        last = None
        for _ in range(max(1, args.steps)):
            last = cpu_reference_rate(model, args.config, frames, max(2.0, 120.0 / max(1, args.steps)),
                                      threads)
            vals.append(last["value"])
        v = float(statistics.mean(vals))
        out_call = cfgd["out"]
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "samples/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": streams * out_call / v * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 accumulate)",
                "data": "synthetic (seeded)", "x_realtime": v / SR,
                "config": {"workload": f"cfg{args.config}:{cfgd['name']}", "streams": streams,
                           "frames_per_call": frames, "out_samples_per_call": out_call},
                "cpu_baseline": dict(last, value=v),
                "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    from paper_2204_07064_b200.runtime import Plan, StreamState

    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2204_07064_b200.shard import max_over_ranks, strong_range, weak_range
    if args.total_streams:
        my = strong_range(args.total_streams, ws, rank)
        scaling = "strong"
    else:
        my = weak_range(streams, rank)
        scaling = "weak"
    streams = len(my)
    plan = Plan(model, precision=args.precision, device=local)
    num, den, cout = plan.sink
    out_call = frames * num // den
    st = StreamState(plan, streams, frames)
    st.set_graphs(not args.no_graphs)
    cin = model.in_channels
    first = my.start
    xs = [torch.from_numpy(make_inputs(args.config, first, streams, cin, frames, k)).to(dev)
          for k in range(2)]
    ys = [torch.empty((streams, cout, out_call), device=dev) for _ in range(2)]
    stream = torch.cuda.current_stream(dev)
    in_bytes = xs[0].numel() * 4
    out_bytes = ys[0].numel() * 4
    l2_bytes = 126 * 1024 * 1024
    flush = None
    step_bytes = in_bytes + out_bytes
    if step_bytes < l2_bytes:
        flush = torch.empty(2 * l2_bytes // 4, device=dev)

    def barrier():
        if ws > 1:
            dist.barrier()

    for k in range(args.warmup):
        st.process_buffer(xs[k % 2], ys[k % 2], frames, stream)
    torch.cuda.synchronize()

    # ---- timed region: device-resident I/O
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    launched0 = st.launch_total()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            if flush is not None:
                flush.zero_()
            evs[k][0].record(stream)
            st.process_buffer(xs[k % 2], ys[k % 2], frames, stream)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    gpu_launches = st.launch_total() - launched0  # exact: counted by the library per call
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs), dev)
    total_streams = args.total_streams or streams * ws
    value = total_streams * out_call * args.steps / (ms / 1e3)

    # ---- e2e through the public C-ABI host-buffer call (sc_process_host): every step's
    # input is copied H2D from pinned host memory and its output D2H inside the timed region;
    # the library overlaps call k's copies with call k-1/k+1's compute on separate streams
    io16 = args.io == "bf16"
    io_dt = torch.bfloat16 if io16 else torch.float32
    hx = [xs[k].to(io_dt).cpu().pin_memory() for k in range(2)]
    hy = [torch.empty((streams, cout, out_call), dtype=io_dt, pin_memory=True) for _ in range(2)]
    host_call = st.process_host_bf16 if io16 else st.process_host
    st.reset(stream=stream)
    for k in range(2):
        host_call(hx[k], hy[k], frames, stream)
    st.host_wait(stream)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        host_call(hx[k % 2], hy[k % 2], frames, stream)
    st.host_wait(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ems = max_over_ranks(e0.elapsed_time(e1), dev)
    e2e_value = total_streams * out_call * args.steps / (ems / 1e3)

    # ---- per-launch profile (un-graphed, CUDA events between launches) for the roofline
    prof = st.profile(xs[0], ys[0], frames, steps=max(3, min(args.steps, 10)), stream=stream)
    op_macs = plan.op_macs()
    pk = peaks()
    conv_idx = [i for i, (n, _) in enumerate(prof) if n.startswith("op")]
    dom = max(conv_idx, key=lambda i: prof[i][1]) if conv_idx else max(range(len(prof)), key=lambda i: prof[i][1])
    dom_name, dom_ms = prof[dom]
    step_ms_prof = sum(t for _, t in prof)
    roof = None
    if dom_name.startswith("op"):
        # "op6+7 ...": a conv with a chained 1x1 conv in the same launch (both GEMMs' FLOPs)
        ois = [int(k) for k in dom_name.split()[0][2:].split("+")]
        flops = 2.0 * sum(op_macs[oi] for oi in ois) * frames * streams
        achieved = flops / (dom_ms / 1e3) / 1e12
        # the fp32-accurate path issues 3 tf32 MMAs per product at half the bf16 rate:
        # its tensor-core ceiling is peak_bf16 / 6 (algorithmic FLOPs)
        ceil = pk["bf16"] / 6.0 if (args.precision == "fp32" and "[tc]" in dom_name) else pk["bf16"]
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16"], "traffic": None, "kernel": dom_name,
                "kernel_ms": dom_ms, "kernel_share_of_step": dom_ms / step_ms_prof,
                "peak_source": f"{pk['src']} bf16 dense (burst; MEASURED_PEAKS.json)",
                "path_ceiling": ceil, "frac_of_path_ceiling": achieved / ceil,
                "path_ceiling_note": "3xTF32 = 3 tf32 MMAs (half bf16 rate) per fp32 product"
                if ceil != pk["bf16"] else "bf16 kind::f16 MMA",
                "flops_per_launch": flops}
        tfile = ROOT / "profiles" / "traffic.json"
        if tfile.exists():
            try:
                roof["traffic"] = json.loads(tfile.read_text()).get(f"cfg{args.config}:{dom_name}")
            except Exception:
                pass
    total_flops = 2.0 * plan.macs_per_sample * frames * streams
    step_bytes_min = in_bytes + out_bytes + streams * (st.cache_bytes * 2)
    step_roof_ms = max(total_flops / (pk["bf16_sus"] * 1e12), step_bytes_min / (pk["hbm"] * 1e9)) * 1e3
    # the same bound with this precision's tensor ceiling: 3xTF32 issues 3 tf32 MMAs (half
    # the bf16 rate) per fp32 product, so its ceiling is bf16_sustained / 6
    path_tf = pk["bf16_sus"] / 6.0 if args.precision == "fp32" else pk["bf16_sus"]
    step_path_ms = max(total_flops / (path_tf * 1e12), step_bytes_min / (pk["hbm"] * 1e9)) * 1e3

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_rate(model, args.config, frames, args.cpu_seconds,
                                     len(os.sched_getaffinity(0)))
        except Exception as e:  # the oracle is a reported baseline, never the product
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": "samples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "bf16 operands / f32 accumulate",
            "data": "synthetic (seeded: N(0,1) frames; cfg5 pink noise + partials)",
            "x_realtime": value / SR,
            "config": {"workload": f"cfg{args.config}:{cfgd['name']}", "streams_per_gpu": streams,
                       "frames_per_call": frames, "out_samples_per_call": out_call,
                       "out_channels": cout, "precision": args.precision,
                       "parallelism": f"stream-sharded x{ws}",
                       "l2": "inputs larger than L2" if flush is None else "L2 flushed between steps",
                       "cuda_graphs": not args.no_graphs},
            "roofline": roof,
            "step_roofline": {"ms": step_roof_ms, "frac": step_roof_ms / (ms / args.steps),
                              "flops_per_step": total_flops,
                              "path_ms": step_path_ms, "frac_of_path_ceiling": step_path_ms / (ms / args.steps),
                              "note": "whole-step bound max(F/P_bf16_sustained, bytes/HBM); path_ms uses "
                                      "the precision's tensor ceiling (3xTF32: P_bf16_sustained / 6)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": hx[0].numel() * hx[0].element_size(),
                    "d2h_bytes_per_step": hy[0].numel() * hy[0].element_size(), "host_io": args.io},
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
            "profile_ms": {n: round(t, 4) for n, t in prof},
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
