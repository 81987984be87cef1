"""Turns the outputs of tools/refresh_profiles.sh (gpurun_out/) into the
committed profile summaries under profiles/ (round tag as argv[1])."""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main():
    bench = json.loads((OUT / "bench_default.json").read_text().strip().splitlines()[-1])
    (PROF / f"{tag}_bench_config5_full.json").write_text(json.dumps(bench) + "\n")
    ref = (OUT / "bench_ref.json").read_text().strip().splitlines()
    if ref:
        (PROF / f"{tag}_bench_reference_arm.json").write_text(ref[-1] + "\n")
    for wl in ("euler", "jacobian"):
        f = OUT / f"bench_{wl}.json"
        if f.exists() and f.read_text().strip():
            (PROF / f"{tag}_bench_irbc_{wl}_N150.json").write_text(f.read_text().strip().splitlines()[-1] + "\n")
    launches = OUT / "launches.csv"
    if launches.exists():
        (PROF / f"{tag}_launches_config5.csv").write_text(launches.read_text())
    rep = OUT / "prof_final_config5.ncu-rep"
    if rep.exists():
        m, units = raw_metrics(rep)
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
                "launch__block_size", "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active"]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        dram = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            dram += float(m[k].replace(",", "")) * scale.get(units.get(k, "byte"), 1.0)
        points = 447392
        doc = {"kernel": "ddsg_b200::fast::fast_hdmr_kernel<1, 0> (EXACT)",
               "capture": "ncu --set full --import-source on --clock-control none, tools/profile_run.py 5 447392 1 "
                          "(config 5, one launch of the bench's chunk size: 447,392 points x 19 column blocks)",
               "metrics": {k: f"{m[k]} {units.get(k, '')}".strip() for k in keys if k in m},
               "points_per_launch": points, "dram_bytes_per_launch": dram, "dram_bytes_per_point": dram / points}
        (PROF / f"{tag}_ncu_fast_hdmr_config5.json").write_text(json.dumps(doc, indent=1) + "\n")
        print(json.dumps(doc["metrics"], indent=1))


if __name__ == "__main__":
    main()
