"""Top stalled SASS instructions of an ncu report's source page (--page source --csv
--print-source sass):  python tools/ncu_sass_top.py page.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    data.append((s, r))
tot = sum(s for s, _ in data)
print("total samples", tot)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, r in sorted(data, key=lambda t: -t[0])[:N]:
    top = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stall_cols), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}% {r[ix['Address']]:>6} exe={r[ix['Instructions Executed']]:>9} {r[ix['Source']][:60]:60s} {top}")
