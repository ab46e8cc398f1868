"""Group an ncu SASS source page (csv) into runs of equal execution count and print the
stall samples of each run (with its distinct opcodes) — a quick map of which warp role
(producer / transform / MMA / drain / epilogue) the samples fall in.
  python tools/ncu_sass_groups.py page.csv [min_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
sc = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
groups = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    e = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    src = r[ix["Source"]].split()
    op = src[1] if src and src[0].startswith("@") else (src[0] if src else "")
    st = {k[6:]: int(r[ix[k]] or 0) for k in sc}
    if groups and groups[-1]["e"] == e:
        g = groups[-1]
        g["s"] += s
        g["n"] += 1
        g["ops"].add(op)
        for k, v in st.items():
            g["st"][k] = g["st"].get(k, 0) + v
    else:
        groups.append({"a": r[ix["Address"]], "e": e, "s": s, "n": 1, "ops": {op}, "st": st})
tot = sum(g["s"] for g in groups) or 1
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
LM = ("UTCHMMA", "UTCQMMA", "UTMALDG.3D", "F2FP", "LDTM", "STTM", "UTMASTG.3D", "SHFL")
for g in groups:
    pct = 100 * g["s"] / tot
    if pct >= mn or any(k in g["ops"] for k in LM):
        top = sorted(g["st"].items(), key=lambda kv: -kv[1])[:3]
        print(f"{g['a'][-5:]} exe={g['e']:>8} n={g['n']:>4} {pct:5.1f}% {top} {' '.join(sorted(g['ops']))[:110]}")
