"""DRAM bytes per launch (ncu read + write) of every step launch, keyed the way bench.py looks
them up (`profiles/traffic.json`: "cfg<N>:<launch name>").

  python tools/ncu_traffic.py <ncu launch-list csv> <bench json line> <cfg> [profiles/traffic.json]

The launch list is the `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` capture of `bench.py --config <cfg>`; the bench line supplies the
launch names in launch order (its `profile_ms` keys).  Every ingest ... egress run in the
capture is one step; the per-name average over the captured steps is merged into the JSON file.
"""
import collections
import csv
import json
import sys


def launches(path):
    # ncu's own csv quotes every field; the trimmed lists under profiles/ quote only where needed
    rows = [r for r in csv.reader(line for line in open(path) if line[:1] == '"' or line[:2] == "ID" or line[:1].isdigit())]
    hdr, data = rows[0], rows[1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    by = collections.OrderedDict()
    for r in data:
        by.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    return list(by.values())


def kernel_token(launch_name):
    """The ncu kernel-name substring of a launch name's kernel (step boundaries)."""
    if launch_name == "ingest":
        return "ingest"
    if launch_name == "egress":
        return "egress"
    if "pqmf-analysis" in launch_name:
        return "pqmf_analysis"
    if "pqmf-synthesis" in launch_name:
        return "pqmf_synthesis"
    return "conv"


def main():
    seq = launches(sys.argv[1])
    # a capture window that starts mid-step: rotate so it starts at an ingest (the launches of
    # one step are the same every step, so the tail + head form one complete step)
    names0 = [n for n in json.loads(open(sys.argv[2]).read())["profile_ms"] if n != "carry"]
    t0, t1 = kernel_token(names0[0]), kernel_token(names0[-1])
    first = next((i for i, k in enumerate(seq) if t0 in k["name"]), 0)
    if first > 0 and len(seq) - first < len(names0):
        need = len(names0) - (len(seq) - first)
        seq = seq[first:] + seq[first - need:first]
    names = [n for n in json.loads(open(sys.argv[2]).read())["profile_ms"] if n != "carry"]
    cfg = sys.argv[3]
    out = sys.argv[4] if len(sys.argv) > 4 else "profiles/traffic.json"
    acc = collections.defaultdict(list)
    i = 0
    while i < len(seq):
        if t0 not in seq[i]["name"]:
            i += 1
            continue
        step = seq[i:i + len(names)]
        if len(step) < len(names) or t1 not in step[-1]["name"]:
            break
        for n, k in zip(names, step):
            acc[n].append(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"])
        i += len(names)
    try:
        table = json.loads(open(out).read())
    except FileNotFoundError:
        table = {}
    table = {k: v for k, v in table.items() if not k.startswith(f"cfg{cfg}:")}
    for n, v in acc.items():
        table[f"cfg{cfg}:{n}"] = sum(v) / len(v)
    open(out, "w").write(json.dumps(table, indent=1) + "\n")
    print(f"{len(acc)} launch names, {min(len(v) for v in acc.values())} steps")


if __name__ == "__main__":
    main()
