import json, sys
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_all.jsonl"):
    d = json.loads(line)
    if "failed" in d:
        print("FAILED", d["failed"]); continue
    c = d["config"]; r = d.get("roofline") or {}
    print(f'{c["workload"]:28s} {c["precision"]:5s} F={c["frames_per_call"]:5d} S={c["streams_per_gpu"]:6d} '
          f'{d["value"]/1e6:9.1f} Msps {d["x_realtime"]:9.0f}xRT {d["ms_per_step"]:8.3f} ms '
          f'e2e {d["e2e"]["value"]/1e6:8.1f}{"(bf16 io)" if d["e2e"].get("host_io") == "bf16" else ""} step_roof {d["step_roofline"]["frac"]:.3f} '
          f'dom {r.get("kernel","-")[:34]:34s} {r.get("achieved",0):6.1f} TF')
