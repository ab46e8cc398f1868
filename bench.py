#!/usr/bin/env python
"""bench.py — aggregate streamed samples/s (x real-time @ 48 kHz) over concurrent streams.

Metric (BASELINE.json): streamed audio samples/s over concurrent independent streams and its
roofline fraction.  One step = one process_buffer call for every stream of
the rank's shard.  Default workload: BASELINE config 5 (configs[4], the largest single-GPU
config and the north star's target: the RAVE-style encoder + decoder, 16384 streams x 2048
samples, fp32).  `--config N` selects another config (4: the RAVE-style decoder).

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
--impl reference: that CPU path as the reference arm (rank 0 only; never loads the product
           library — PQMF filters from oracle/pqmf_design.py, frame counts from the oracle).
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
    ap.add_argument("--config", type=int, default=5)
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
        pk = dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                  bf16_sus=d.get("bf16_tflops_sustained", 1400.0), src="measured")
    else:
        pk = dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")
    # P_TF32: measured on the box by tools/tf32_peak.cu (kind::tf32 tcgen05 MMAs, all SMs),
    # committed as profiles/tf32_peak.json; the fp32-accurate path issues 3 tf32 MMAs per
    # product (3xTF32), so its tensor ceiling is P_TF32 / 3 in algorithmic FLOPs.
    t = ROOT / "profiles" / "tf32_peak.json"
    pk["tf32"] = pk["tf32_sus"] = None
    if t.exists():
        d = json.loads(t.read_text())
        pk["tf32"] = d.get("tf32_tflops")
        pk["tf32_sus"] = d.get("tf32_tflops_sustained", pk["tf32"])
        pk["f16"] = d.get("f16_tflops")
        pk["f16_sus"] = d.get("f16_tflops_sustained", pk["f16"])
    return pk


def fp32_path_ceiling(pk, sustained=False, split="tf32"):
    """(TFLOP/s, source) of the fp32-accurate path's tensor ceiling in algorithmic FLOPs: three
    MMAs per fp32 product — kind::tf32 (3xTF32, "[tc]" launches) or kind::f16 (3xFP16,
    "[tc-3xf16]" launches, the default split)."""
    if split == "f16":
        f = pk.get("f16_sus") if sustained else pk.get("f16")
        if f:
            return f / 3.0, "measured f16 (profiles/tf32_peak.json: kind::f16 TS N128) / 3"
        bf = pk["bf16_sus"] if sustained else pk["bf16"]
        return bf / 3.0, "bf16 dense / 3 (f16 unmeasured)"
    tf = pk["tf32_sus"] if sustained else pk["tf32"]
    if tf:
        return tf / 3.0, "measured tf32 (profiles/tf32_peak.json) / 3"
    bf = pk["bf16_sus"] if sustained else pk["bf16"]
    return bf / 6.0, "assumed: bf16 / 6 (tf32 unmeasured)"


class ClockSampler:
    """SM clock + throttle reasons sampled every ~10 ms (NVML) from before the warm-up to the
    end of the e2e leg; falls back to nvidia-smi (one sample per ~0.2 s) without pynvml."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period: float = 0.01):
        self.index = index
        self.period = period
        self.rows = []       # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = None
        self.src = "nvml"

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), int(bits)))
                self._stop.wait(self.period)
            return
        except Exception:
            self.src = "nvidia-smi"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                r = [v.strip() for v in out.split(",")]
                bits = sum(self.REASONS[n] for n, v in zip(names, r[2:6]) if v.lower() == "active")
                self.rows.append((float(r[0]), float(r[1]), bits))
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
        sm = [r[0] for r in self.rows]
        reasons = sorted(n for n, b in self.REASONS.items() if any(r[2] & b for r in self.rows))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(self.rows),
                "span": "warm-up + timed region + e2e leg", "source": self.src}


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


def config_dict(cfg, name, streams, frames, out_call, cout, precision, ws, in_bytes, out_bytes):
    """The `config` object — identical keys and values in both arms (ours / reference)."""
    l2_bytes = 126 * 1024 * 1024
    return {"workload": f"cfg{cfg}:{name}", "streams_per_gpu": streams,
            "frames_per_call": frames, "out_samples_per_call": out_call, "out_channels": cout,
            "precision": precision, "parallelism": f"stream-sharded x{ws}",
            "l2": ("inputs larger than L2" if in_bytes + out_bytes >= l2_bytes
                   else "L2 flushed between steps")}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_rates(cfg, frames, steps, step_seconds, threads, mode_a_seconds=8.0):
    """The reference's own CPU path for this workload: its conv1d (oracle/_ref = the
    unmodified proj/src/kernels.cpp; the oracle's restatement when the reference could not be
    built) driven by the SPEC process_buffer restatement (oracle/oracle.cpp), on the host.

    mode (B), the timed arm: set_parallel_kernels(false) (kernels.cpp:33) with one stream per
      thread (SPEC.md:302,304 allow independent states to run concurrently), all `threads`;
    mode (A), reported beside it: the reference default — OpenMP inside conv1d
      (kernels.cpp:88), streams one after another.
    Each step is a bounded sample of stream-calls (fresh zero-initialised state)
    sized to ~step_seconds; the rate is samples actually produced / wall time actually spent.
    Never loads the product library: the model's PQMF filters come from the oracle's
    independent design (oracle/pqmf_design.py), frame counts from the oracle's graph_info."""
    from oracle import pqmf_design
    from oracle import pyoracle as po
    from paper_2204_07064_b200 import configs
    model = configs.build(cfg, seed=0, pqmf_design=pqmf_design.filters)
    info = po.graph_info(model)
    out_call = frames * info["sink_num"] // info["sink_den"]
    use_ref = po.ref_available()
    if use_ref:
        po.ref().ref_set_parallel_kernels(0)
    # calibration (= warm-up): one stream-call per thread
    x = make_inputs(cfg, 0, threads, model.in_channels, frames, slot=0)
    t0 = time.perf_counter()
    po.run(model, x, [frames], "stream", use_ref=use_ref, threads=threads)
    t_cal = time.perf_counter() - t0
    per_step = threads * max(1, int(round(step_seconds / max(t_cal, 1e-6))))
    xs = make_inputs(cfg, 0, per_step, model.in_channels, frames, slot=1)
    secs = []
    for _ in range(steps):
        t0 = time.perf_counter()
        po.run(model, xs, [frames], "stream", use_ref=use_ref, threads=threads)
        secs.append(time.perf_counter() - t0)
    rates = [per_step * out_call / s for s in secs]
    b = dict(value=per_step * out_call * steps / sum(secs), unit="samples/s", cores=threads,
             kind="reference" if use_ref else "port",
             cpu_model=cpu_model(), nproc=os.cpu_count(),
             mode="B: set_parallel_kernels(false), OpenMP across streams",
             rate_mean=statistics.mean(rates),
             rate_std=statistics.pstdev(rates) if len(rates) > 1 else 0.0,
             trials=steps, step_s_mean=statistics.mean(secs),
             sample=f"{steps} trials x {per_step} stream-calls x {frames} frames -> {out_call} "
                    f"samples each (fresh state), {sum(secs):.1f} s wall timed; "
                    f"{'reference conv1d (kernels.cpp, oracle/_ref)' if use_ref else 'oracle port of conv1d'}"
                    f" via the SPEC process_buffer restatement")
    # mode (A): the reference default, OpenMP inside conv1d, one stream after another
    a = None
    if use_ref and mode_a_seconds > 0:
        po.ref().ref_set_parallel_kernels(1)
        n_a = max(1, int(round(mode_a_seconds / max(t_cal, 1e-6))))  # ~t_cal per call at full width
        xa = xs[:min(n_a, per_step)]
        t0 = time.perf_counter()
        po.run(model, xa, [frames], "stream", use_ref=True, threads=1)
        dt = time.perf_counter() - t0
        po.ref().ref_set_parallel_kernels(0)
        a = dict(value=xa.shape[0] * out_call / dt, unit="samples/s", cores=threads,
                 mode="A: reference default, OpenMP inside conv1d (kernels.cpp:88), streams sequential",
                 sample=f"{xa.shape[0]} stream-calls x {frames} frames, {dt:.1f} s wall")
    b["mode_a"] = a
    return b, out_call, info["out_channels"], secs


METRIC = "streamed audio samples/s (x real-time @48kHz) over concurrent streams"


def main_reference(args, ws, rank):
    """--impl reference: the reference's CPU path on the host cores, rank 0 only."""
    if rank != 0:
        return 0
    from paper_2204_07064_b200 import configs
    cfgd = configs.CONFIGS[args.config]
    frames = args.frames or cfgd["frames"]
    streams = args.streams or cfgd["streams"]
    if args.total_streams:
        streams = -(-args.total_streams // ws)
    threads = len(os.sched_getaffinity(0))
    # whole run (warm-up/calibration + K trials + mode A sample) within ~2 minutes
    step_s = min(4.0, max(1.0, 90.0 / max(1, args.steps)))
    cpu, out_call, cout, secs = reference_rates(args.config, frames, max(1, args.steps), step_s,
                                                threads, mode_a_seconds=8.0)
    v = cpu["value"]
    in_bytes = streams * configs.CONFIGS[args.config]["in_channels"] * frames * 4
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(secs) * 1e3,
            "ms_per_step_note": "wall time of one timed trial (a bounded sample of stream-calls, "
                                "see cpu_baseline.sample), not of a full-config step",
            "higher_is_better": True, "scaling": "strong" if args.total_streams else "weak",
            "vs_baseline": None, "dtype": "f32 (f64 accumulate, kernels.cpp:96-100)",
            "data": "synthetic (seeded: N(0,1) frames; cfg5 pink noise + partials)",
            "x_realtime": v / SR,
            "config": config_dict(args.config, cfgd["name"], streams, frames, out_call, cout,
                                  "fp32", ws, in_bytes, streams * cout * out_call * 4),
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        return main_reference(args, ws, rank)

    from paper_2204_07064_b200 import configs
    cfgd = configs.CONFIGS[args.config]
    frames = args.frames or cfgd["frames"]
    streams = args.streams or cfgd["streams"]
    model = configs.build(args.config, seed=0)

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
    cfg_line = config_dict(args.config, cfgd["name"], streams, frames, out_call, cout,
                           args.precision, ws, in_bytes, out_bytes)
    flush = None
    if cfg_line["l2"] != "inputs larger than L2":
        flush = torch.empty(2 * 126 * 1024 * 1024 // 4, device=dev)

    def barrier():
        if ws > 1:
            dist.barrier()

    clk = ClockSampler(local)
    clk.__enter__()
    for k in range(args.warmup):
        st.process_buffer(xs[k % 2], ys[k % 2], frames, stream)
    torch.cuda.synchronize()

    # ---- timed region: device-resident I/O
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    launched0 = st.launch_total()
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()
        evs[k][0].record(stream)
        st.process_buffer(xs[k % 2], ys[k % 2], frames, stream)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    gpu_launches = st.launch_total() - launched0  # exact: counted by the library per call
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = max_over_ranks(sum(step_ms), dev)
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
    clk.__exit__()
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
        if args.precision == "fp32" and ("[tc]" in dom_name or "[tc-3xf16]" in dom_name):
            ceil, csrc = fp32_path_ceiling(pk, split="f16" if "[tc-3xf16]" in dom_name else "tf32")
        else:
            ceil, csrc = pk["bf16"], "bf16 dense (burst; MEASURED_PEAKS.json)"
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16"], "traffic": None, "kernel": dom_name,
                "kernel_ms": dom_ms, "kernel_share_of_step": dom_ms / step_ms_prof,
                "peak_source": f"{pk['src']} bf16 dense (burst; MEASURED_PEAKS.json)",
                "path_ceiling": ceil, "frac_of_path_ceiling": achieved / ceil,
                "path_ceiling_source": csrc,
                "path_ceiling_note": ("3xFP16 = 3 kind::f16 MMAs per fp32 product (per-row power-of-two block scaling)"
                                      if "[tc-3xf16]" in dom_name else "3xTF32 = 3 kind::tf32 MMAs per fp32 product")
                if args.precision == "fp32" else "bf16 kind::f16 MMA",
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
    # the same bound with this precision's tensor ceiling (3xTF32: P_TF32 / 3, sustained)
    if args.precision == "fp32":
        path_tf, path_src = fp32_path_ceiling(pk, sustained=True,
                                              split="tf32" if os.environ.get("SC_FP32_SPLIT") == "tf32" else "f16")
    else:
        path_tf, path_src = pk["bf16_sus"], "bf16 dense sustained (MEASURED_PEAKS.json)"
    step_path_ms = max(total_flops / (path_tf * 1e12), step_bytes_min / (pk["hbm"] * 1e9)) * 1e3
    # layer-wise bound: sum over the step's launches of max(FLOPs / tensor ceiling, DRAM bytes /
    # HBM), with each launch's DRAM bytes from the committed ncu launch list of this config
    # (profiles/traffic.json, tools/ncu_traffic.py) — activations between layers count here
    layerwise = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists() and not args.frames and not args.streams:
        try:
            tr = json.loads(tfile.read_text())
            lw_ms, covered = 0.0, 0
            for name, _ in prof:
                b = tr.get(f"cfg{args.config}:{name}")
                if b is None:
                    continue
                covered += 1
                fl = 0.0
                if name.startswith("op") and "[tc" in name:
                    ois = [int(k) for k in name.split()[0][2:].split("+")]
                    fl = 2.0 * sum(op_macs[oi] for oi in ois) * frames * streams
                lw_ms += max(fl / (path_tf * 1e12), b / (pk["hbm"] * 1e9)) * 1e3
            if covered >= len(prof) - 1:
                layerwise = {"ms": lw_ms, "frac": lw_ms / (ms / args.steps), "launches_covered": covered,
                             "bytes_source": "profiles/traffic.json (ncu dram__bytes read+write per launch)"}
        except Exception:
            layerwise = None

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            threads = len(os.sched_getaffinity(0))
            trials = 3
            cpu = reference_rates(args.config, frames, trials, args.cpu_seconds / trials, threads,
                                  mode_a_seconds=0)[0]
        except Exception as e:  # the oracle is a reported baseline, never the product
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "ms_per_step_std": statistics.pstdev(step_ms) if len(step_ms) > 1 else 0.0,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "bf16 operands / f32 accumulate",
            "data": "synthetic (seeded: N(0,1) frames; cfg5 pink noise + partials)",
            "x_realtime": value / SR,
            "config": cfg_line,
            "cuda_graphs": not args.no_graphs,
            "roofline": roof,
            "step_roofline": {"ms": step_roof_ms, "frac": step_roof_ms / (ms / args.steps),
                              "flops_per_step": total_flops, "bytes_min_per_step": step_bytes_min,
                              "path_ms": step_path_ms,
                              "frac_of_path_ceiling": step_path_ms / (ms / args.steps),
                              "path_ceiling_tflops": path_tf, "path_ceiling_source": path_src,
                              "layerwise": layerwise,
                              "note": "whole-step bound max(F/P, bytes/HBM) (SURVEY §8d); `ms` uses "
                                      "P = bf16 sustained, `path_ms` this precision's tensor ceiling"},
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
