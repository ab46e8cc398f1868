"""Copy one evidence run (the directory tools' commands in profiles/README.md write: bench lines,
parity table, ncu launch list, raw / source pages of the op24 and op29 captures) into profiles/
under the round-2 names: the launch list trimmed to its first two steps and seven columns, the
key counters of the full captures, the instruction accounting, and traffic.json.
  python tools/install_evidence.py gpurun_out/final"""
import collections
import csv
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
F = Path(sys.argv[1])
P = ROOT / "profiles"

for src, dst in (("bench_default.json", "r2_bench_default.json"), ("bench_all.jsonl", "r2_bench_all.jsonl"),
                 ("bench_all.md", "r2_bench_all.md"), ("parity_table.txt", "r2_parity_table.txt"),
                 ("bench_reference.json", "r2_bench_reference_arm.json")):
    if (F / src).exists():
        shutil.copy(F / src, P / dst)

rows = [r for r in csv.reader(l for l in open(F / "ncu_launches_cfg5.csv") if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
sel = [0, 4, 7, 8, 12, 13, 14]
by = collections.OrderedDict()
for r in data:
    by.setdefault(int(r[0]), {"name": r[4]})[r[12]] = float(r[14].replace(",", ""))
keep, n = [], 0
for i in sorted(by):
    keep.append(i)
    if "pqmf_synthesis" in by[i]["name"]:
        n += 1
        if n == 2:
            break
with open(P / "r2_ncu_launches_cfg5.csv", "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow([hdr[i] for i in sel])
    for r in data:
        if int(r[0]) in keep:
            w.writerow([r[i][:70] if i == 4 else r[i] for i in sel])
second = keep[len(keep) // 2:]
tot = sum(by[i]["gpu__time_duration.sum"] for i in second)
tc = sum(by[i]["gpu__time_duration.sum"] for i in second if "conv_tc" in by[i]["name"])
print(f"launch list: {len(keep)} launches kept; second step {tot / 1e6:.3f} ms, tensor-core convs {100 * tc / tot:.1f}%")
for i in second:
    b = by[i]
    print(f"  {i:3d} {b['name'][10:46]:36s} {b['gpu__time_duration.sum'] / 1e3:7.1f} us "
          f"{(b['dram__bytes_read.sum'] + b['dram__bytes_write.sum']) / 1e6:6.0f} MB "
          f"tensor {b['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']:4.1f}%")

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]
for name, out, slabs, title in (
        ("op24", "r2_ncu_full_op24_convT_3xf16.csv", 131072, "op24 (convT4 512->256 K8, X2 3xFP16 tile)"),
        ("op29", "r2_ncu_full_op29_conv128_3xf16.csv", 98304,
         "op29 (conv 128->128 K3 d1, X2 3xFP16 tile, per-block input windows)")):
    raw = F / f"{name}_raw.csv"
    if not raw.exists():
        continue
    rr = list(csv.reader(open(raw)))
    h, u, v = rr[0], rr[1], rr[2]
    idx = [h.index(x) for x in WANT if x in h]
    with open(P / out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow([h[i] for i in idx]), w.writerow([u[i] for i in idx]), w.writerow([v[i] for i in idx])
    g = lambda k: v[h.index(k)]
    head = (f"# {title} — this build: {float(g('gpu__time_duration.sum')):.1f} us under ncu, tensor pipe "
            f"{float(g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active')):.1f}%, issue active "
            f"{float(g('smsp__issue_active.avg.pct_of_peak_sustained_active')):.1f}%\n"
            f"# ncu --set full --import-source on --clock-control none, source page -> tools/ncu_inst_mix.py page.csv {slabs}"
            f"  (NANOSLEEP = the back-off waits)\n")
    mix = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_inst_mix.py"), str(F / f"{name}_sass.csv"), str(slabs)],
                         capture_output=True, text=True).stdout
    dst = "r2_ncu_op29_inst_mix_after.txt" if name == "op29" else "r2_ncu_op24_inst_mix.txt"
    (P / dst).write_text(head + mix)
    print(head.split("\n")[0])
subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_traffic.py"), str(P / "r2_ncu_launches_cfg5.csv"),
                str(P / "r2_bench_default.json"), "5", str(P / "traffic.json")], check=True)
