"""Writes a profiles/ JSON summary of one ncu --set full capture made by
tools/ncu_kernel.sh.  Usage: ncu_to_profile.py <capture-name> <out.json>
<work-units> <unit-name> "<what>" "<reading>" """
import collections
import csv
import json
import re
import sys

name, out, units, unit_name, what, reading = sys.argv[1:7]
units = float(units)
rows = list(csv.reader(open(f"gpurun_out/{name}_raw.csv")))
hdr, unit, vals = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct"]
metrics = {k: f"{vals[hdr.index(k)]} {unit[hdr.index(k)]}".strip() for k in keys if k in hdr}
st = {}
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
        except ValueError:
            pass
tot = sum(st.values()) or 1.0
stalls = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]}
rows = list(csv.reader(open(f"gpurun_out/{name}_source.csv")))
h2, data = rows[1], rows[2:]
iS, iI = h2.index("Source"), h2.index("Instructions Executed")
op = collections.Counter()
for r in data:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS])
    op[m.group(2) if m else r[iS]] += float(r[iI] or 0)
doc = {"what": what, "metrics": metrics, "stall_pct": stalls,
       f"sass_per_{unit_name}": round(sum(op.values()) / units, 1),
       f"top_opcodes_per_{unit_name}": {o: round(n / units, 1) for o, n in op.most_common(12)},
       "reading": reading}
open(out, "w").write(json.dumps(doc, indent=1) + "\n")
print(json.dumps(doc, indent=1))
