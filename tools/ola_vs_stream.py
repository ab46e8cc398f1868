"""Streaming vs overlap-add on the GPU — the paper's comparison (PAPER §4.1-4.2, Fig. 11-13;
SPEC baseline_ola / metrics_bench), at scale: many concurrent streams of the config-5 RAVE-style
encoder/decoder (non-causal centered pads) through

  * the cached-padding streaming engine (causalized graph, buffers of B samples), and
  * the overlap-add baseline at 0 / 25 / 50 % overlap with chunks of B samples,

each scored against the offline run of the ORIGINAL graph over the whole signal (computed on the
GPU by the same offline program with one chunk spanning the signal), after removing the
streaming latency.  Throughput is the device time of the whole signal per method.

Usage: python tools/ola_vs_stream.py [--streams 64] [--samples 393216] > profiles/r1_ola_vs_stream.md
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2204_07064_b200 import configs  # noqa: E402
from paper_2204_07064_b200.graph import model_to_graph  # noqa: E402
from paper_2204_07064_b200.runtime import Ola, Plan, StreamState, best_lag, fidelity  # noqa: E402


TRIALS = 10  # SPEC metrics_bench: >= 10 trials


def timed(fn, reps=TRIALS):
    """Device ms per run: (mean, std) over `reps` trials after one warm-up run."""
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.mean(ts)), float(np.std(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=64)
    ap.add_argument("--samples", type=int, default=6 * 65536)  # 8.2 s: a multiple of every hop
    ap.add_argument("--buffers", default="512,2048,8192,32768")
    a = ap.parse_args()
    S = a.streams
    g = model_to_graph(configs.build(5, seed=0))
    T = a.samples
    x = configs.batch_input(5, range(S), 1, T, seed=0)
    xd = torch.from_numpy(x).cuda()
    # offline original over the whole signal: one chunk, no overlap
    ref = torch.empty((S, 1, T), device="cuda")
    off = Ola(g, T, 0, S, T)
    off.process(xd, ref, T)
    plan = Plan(g)
    lat = plan.latency
    # score every method on the same interior [W, T - W): W covers the receptive field, so the
    # reference's own zero padding at the signal ends does not enter (SPEC.md:213 interior)
    past, fut = g.receptive_field()
    W = past + fut + plan.ratio
    sl = slice(W, T - W)
    rows = []
    for B in [int(b) for b in a.buffers.split(",")]:
        st = StreamState(plan, S, B)
        y = torch.empty((S, 1, T), device="cuda")
        xin = [xd[:, :, t0:t0 + B].contiguous() for t0 in range(0, T, B)]  # per-call input buffers
        yout = [torch.empty((S, 1, B), device="cuda") for _ in range(0, T, B)]

        def stream_all():
            st.reset()
            for xi, yo in zip(xin, yout):
                st.process_buffer(xi, yo, B)

        ms, sd = timed(stream_all)
        y = torch.cat(yout, dim=2)
        # buffers below the compression ratio add the phase-state lag: measure the total lag
        # (SPEC best_lag) and check it against the plan's latency
        lag = int(best_lag(ref[:1, 0].contiguous(), y[:1, 0].contiguous(), lat + plan.ratio)[0])
        f = fidelity(ref[:, 0, W - lag:T - W - lag].contiguous(), y[:, 0, sl].contiguous())
        rows.append(dict(method="stream", buffer=B, calls=T // B, ms=ms, ms_std=sd, samples_per_s=S * T / ms * 1e3,
                         latency=lag, plan_latency=lat, macs=g.mac_count(T), state_bytes=plan.state_bytes,
                         L_s=float(np.median(f["L_s"])), L_w=float(np.median(f["L_w"])),
                         L_c=float(np.median(f["L_c"])), redundancy=1.0))
        del st
        for ov in (0, 25, 50):
            try:
                o = Ola(g, B, ov, S, T)
            except Exception as e:  # noqa: BLE001
                rows.append(dict(method=f"ola{ov}", buffer=B, error=str(e)))
                continue
            z = torch.empty((S, 1, T), device="cuda")
            ms, sd = timed(lambda: o.process(xd, z, T))
            nc = (T - B) // (B * (100 - ov) // 100) + 1
            f = fidelity(ref[:, 0, sl].contiguous(), z[:, 0, sl].contiguous())
            rows.append(dict(method=f"ola{ov}", buffer=B, calls=1, ms=ms, ms_std=sd, samples_per_s=S * T / ms * 1e3,
                             latency=B, macs=nc * g.mac_count(B), state_bytes=0,
                             L_s=float(np.median(f["L_s"])), L_w=float(np.median(f["L_w"])),
                             L_c=float(np.median(f["L_c"])), redundancy=Ola.redundancy(ov)))
            del o
    rms = float(torch.sqrt(torch.mean(ref.double() ** 2)))
    print(f"# Streaming vs overlap-add (cfg5 RAVE-style enc/dec, {S} streams x {T} samples, one B200)\n")
    print("Streaming makes one call per buffer (T / B calls, real-time usable); the OLA baseline runs "
          "all chunks of the whole signal in ONE batched call (offline: it needs the future chunks), "
          "so its device time is not a real-time throughput — its redundancy column is the MAC cost.\n")
    print(f"Scored on samples [{W}, {T - W}) (the receptive field past + future + ratio away from both ends). "
          f"Reference: offline run of the original (non-causal) graph over the whole signal, RMS {rms:.3g}. "
          f"Streaming is compared after removing its lag (plan latency {lat} samples, plus ratio - B for "
          f"buffers below the compression ratio {plan.ratio}; measured by best_lag). Medians over streams.\n")
    print("| method | buffer | calls | lag | L_s (spectral) | L_w (euclid) | L_c (corr) | redundancy | device ms | samples/s |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        if "error" in r:
            print(f"| {r['method']} | {r['buffer']} | | | n/a: {r['error'][:70]} | | | | | |")
            continue
        print(f"| {r['method']} | {r['buffer']} | {r['calls']} | {r['latency']} | {r['L_s']:.3e} | {r['L_w']:.3e} | {r['L_c']:.6f} | "
              f"{r['redundancy']:.2f} | {r['ms']:.2f} | {r['samples_per_s']:.3e} |")
    # SPEC metrics_bench BenchReport: per stream; rtf = device time share per
    # stream / audio duration (all streams processed concurrently), over TRIALS trials
    dur = T / configs.SR
    print("\nSPEC BenchReport (per stream, MACs per second of audio; rtf over %d trials):\n" % TRIALS)
    print("```csv")
    print("method,buffer,macs_per_sec,rtf_mean,rtf_std,state_bytes,latency_samples")
    for r in rows:
        if "error" in r:
            continue
        print(f"{r['method']},{r['buffer']},{r['macs'] / dur:.6e},{r['ms'] / 1e3 / S / dur:.6e},"
              f"{r['ms_std'] / 1e3 / S / dur:.3e},{r['state_bytes']},{r['latency']}")
    print("```")
    print("\n```json")
    for r in rows:
        print(json.dumps(r))
    print("```")


if __name__ == "__main__":
    main()
