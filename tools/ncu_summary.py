"""Summarise an ncu --set full capture (raw + source CSV pages): key
throughput metrics, stall samples, and SASS opcode counts per unit of work."""
import collections
import csv
import re
import sys

name = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0  # e.g. warp-terms
rows = list(csv.reader(open(f"gpurun_out/{name}_raw.csv")))
hdr, unit, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:70s} {vals[i]:>16s} {unit[i]}")
print("stall samples:")
st = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            st.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in st)
for v, h in sorted(st, reverse=True)[:10]:
    print(f"  {h:28s} {100 * v / tot:5.1f} %")
rows = list(csv.reader(open(f"gpurun_out/{name}_source.csv")))
hdr, data = rows[1], rows[2:]
iS, iI = hdr.index("Source"), hdr.index("Instructions Executed")
op = collections.Counter()
for r in data:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS])
    op[m.group(2) if m else r[iS]] += float(r[iI] or 0)
print(f"SASS per unit ({units:.3g} units): total {sum(op.values()) / units:.1f}")
print("  " + ", ".join(f"{o} {n / units:.1f}" for o, n in op.most_common(24)))
