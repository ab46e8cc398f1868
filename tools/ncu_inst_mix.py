"""Executed-instruction mix of one kernel from an ncu SASS source page
(ncu -i X.ncu-rep --page source --csv --print-source sass > page.csv):
total warp-level instructions, wait-loop share (mbarrier try_wait polls and their branches),
executed instructions per opcode, and — given the launch's K-slab count and SM count — warp
instructions per K-slab per SM sub-partition, the number to hold against the MMA cycles of a slab.
  python tools/ncu_inst_mix.py page.csv [slabs_total] [sms]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
slabs = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sms = int(sys.argv[3]) if len(sys.argv) > 3 else 148
ops = collections.Counter()
tot = spin = 0
prev_try = False
items = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    e = int(r[ix["Instructions Executed"]] or 0)
    src = r[ix["Source"]].split()
    op = src[1] if src and src[0].startswith("@") else (src[0] if src else "")
    items.append((e, op))
# a wait loop = [YIELD] TRYWAIT + its backward branch: count the poll, the branch after it and a
# YIELD right before it
for i, (e, op) in enumerate(items):
    tot += e
    ops[op.split(".")[0]] += e
    if "TRYWAIT" in op:
        spin += e
        if i + 1 < len(items) and items[i + 1][1].startswith("BRA"):
            spin += min(e, items[i + 1][0])
        if i > 0 and items[i - 1][1] == "YIELD" and items[i - 1][0] == e:
            spin += e
print(f"warp-level instructions executed: {tot:,}")
print(f"wait loops (try_wait polls + branches): {spin:,} = {100 * spin / tot:.1f}%")
if slabs:
    per = tot / slabs / 4
    print(f"per K-slab per SM sub-partition: {per:.0f} instructions ({(tot - spin) / slabs / 4:.0f} outside wait loops)"
          f"  [{slabs} slabs over {sms} SMs]")
print("executed by opcode:")
for k, v in ops.most_common(24):
    print(f"  {k:12s} {v:>12,} {100 * v / tot:5.1f}%" + (f"  {v / slabs / 4:6.1f} / slab / SMSP" if slabs else ""))
