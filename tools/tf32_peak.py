#!/usr/bin/env python
"""Measure P_TF32 (and the bf16 methodology check) with tools/tf32_peak.cu on this GPU.

  python tools/tf32_peak.py [--out profiles/tf32_peak.json]

burst     = best of 5 single launches of ~20 ms each (all SMs, one CTA per SM)
sustained = back-to-back launches for ~4 s, total FLOPs / total device time
FLOPs are the MMAs' own (2 x M x N x K per instruction).  SM clocks and throttle reasons are
sampled with NVML during every measurement.  bench.py reads tf32_tflops /
tf32_tflops_sustained (TS form, N = 128 — the conv_tc_kernel issue shape) for the 3xTF32
path ceiling (P_TF32 / 3).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "tools" / "bin" / "libtf32_peak.so"
SRC = ROOT / "tools" / "tf32_peak.cu"


def build():
    if SO.exists() and SO.stat().st_mtime >= SRC.stat().st_mtime:
        return
    SO.parent.mkdir(exist_ok=True)
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-o", str(SO), str(SRC)])


class Clocks:
    def __init__(self):
        self.rows = []
        self._stop = threading.Event()

    def _run(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(0)
        while not self._stop.is_set():
            self.rows.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),
                              N.nvmlDeviceGetCurrentClocksEventReasons(h),
                              N.nvmlDeviceGetPowerUsage(h) / 1000.0))
            self._stop.wait(0.01)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()

    def summary(self):
        if not self.rows:
            return {}
        names = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown"}
        return {"sm_mhz_median": statistics.median(r[0] for r in self.rows),
                "sm_mhz_min": min(r[0] for r in self.rows),
                "power_w_max": max(r[2] for r in self.rows),
                "reasons": sorted({n for r in self.rows for b, n in names.items() if r[1] & b}),
                "samples": len(self.rows)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "tf32_peak.json"))
    args = ap.parse_args()
    build()
    import torch
    L = C.CDLL(str(SO))
    L.tf32_peak_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
    L.tf32_peak_run.restype = C.c_float
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = {"gpu": torch.cuda.get_device_name(0), "sms": sms, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "tools/tf32_peak.cu: one CTA per SM, one elected lane issues M128xNxK tcgen05.mma "
                  "back to back into TMEM (4 MMAs per 128-byte K row), random operands resident "
                  "in shared memory / TMEM; CUDA events; FLOPs = 2*M*N*K per MMA",
           "cases": {}}
    cases = [("tf32_ts_n128", 1, 128, 8), ("tf32_ts_n256", 1, 256, 8), ("tf32_ss_n128", 0, 128, 8),
             ("tf32_ss_n256", 0, 256, 8), ("bf16_ss_n256", 2, 256, 16), ("tf32_ts_n64", 1, 64, 8),
             ("f16_ts_n128", 3, 128, 16), ("f16_ts_n64", 3, 64, 16), ("bf16_ss_n128", 2, 128, 16)]
    for name, mode, n, k in cases:
        flop_iter = 4 * 2.0 * 128 * n * k * sms
        # size a launch to ~20 ms at a guessed 1 PFLOP/s
        iters = max(1000, int(0.02 * 1e15 / flop_iter))
        with Clocks() as cb:
            bursts = []
            for _ in range(5):
                ms = L.tf32_peak_run(mode, n, iters, sms, 1)
                if ms < 0:
                    raise RuntimeError(f"{name}: CUDA error {-ms}")
                bursts.append(flop_iter * iters / (ms / 1e3) / 1e12)
        launches = max(1, int(4000.0 / max(1e-3, flop_iter * iters / (max(bursts) * 1e12) * 1e3)))
        with Clocks() as cs:
            ms = L.tf32_peak_run(mode, n, iters, sms, launches)
        sus = flop_iter * iters * launches / (ms / 1e3) / 1e12
        res["cases"][name] = {"burst_tflops": max(bursts), "burst_all": bursts,
                              "sustained_tflops": sus, "sustained_s": ms / 1e3, "iters": iters,
                              "clocks_burst": cb.summary(), "clocks_sustained": cs.summary()}
        print(name, f"burst {max(bursts):.1f} TF/s  sustained {sus:.1f} TF/s", cs.summary(), flush=True)
    c = res["cases"]["f16_ts_n128"]
    res["f16_tflops"] = c["burst_tflops"]
    res["f16_tflops_sustained"] = c["sustained_tflops"]
    res["f16_note"] = ("TS form, N = 128, fp16 operands (kind::f16): the 3xFP16 fp32 path's issue "
                       "shape; its ceiling in algorithmic FLOPs is this / 3")
    c = res["cases"]["tf32_ts_n128"]
    res["tf32_tflops"] = c["burst_tflops"]
    res["tf32_tflops_sustained"] = c["sustained_tflops"]
    res["tf32_note"] = ("TS form (A from TMEM), N = 128: the conv_tc_kernel issue shape; the 3xTF32 "
                        "fp32 path's ceiling in algorithmic FLOPs is this / 3")
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(json.dumps({k: v for k, v in res.items() if k != "cases"}))


if __name__ == "__main__":
    sys.exit(main())
