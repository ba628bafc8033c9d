"""Summarise an ncu report: per kernel duration, DRAM bytes, issue activity and top stall reasons.
python tools/ncu_stalls.py REPORT.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"][:70], "grid", d.get("launch__grid_size"), "block", d.get("launch__block_size"),
          "regs", d.get("launch__registers_per_thread"))
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
              "smsp__warps_eligible.avg.per_cycle_active", "lts__t_sector_hit_rate.pct",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
        print("   ", k, d.get(k))
    st = [(k, float(d[k] or 0)) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda kv: -kv[1])
    print("    stalls/issue:", ", ".join(f"{k[34:-23]} {v:.2f}" for k, v in st[:7]))
