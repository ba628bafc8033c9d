"""Summarise tools/profile.sh output into profiles/: per-pass launch list (cold and warm), DRAM
traffic per launch (profiles/ncu_traffic.json, read by bench.py's roofline "traffic") and the
full-set metrics of one CG iteration.   python tools/ncu_summary.py ROUND_TAG"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROW = {0: "row_setpoint", 1: "row_setpoint_fwd", 2: "row_rss", 3: "row_k2", 4: "row_k4"}
COL = {0: "col_ifft_w", 1: "col_ifft_w_cg", 2: "col_fwdp", 3: "col_psf", 4: "col_resadj", 5: "col_adj1",
       6: "col_fft_w_normal", 7: "col_rhs_k1", 8: "col_fft_w_adj"}


def pass_name(kname, k5count):
    base = kname.split("(")[0].replace("void ", "").strip()
    if base.startswith("nlv::"):
        base = base[5:]
    if base.startswith("row_kernel<") or base.startswith("col_kernel<"):
        mode = int(base.split(",")[1].split(">")[0])
        return (ROW if base.startswith("row") else COL)[mode]
    if base.startswith("k5cg_kernel"):
        return "col_k5_newton" if k5count % 10 == 9 else "col_k5_cg_k1"
    return base.split("<")[0]


def launches(fn):
    rows = list(csv.reader(open(fn)))
    h = None
    per = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h is None or len(r) != len(h):
            continue
        d = dict(zip(h, r))
        per.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = collections.OrderedDict()
    k5 = 0
    for _, m in per.items():
        nm = pass_name(m["name"], k5)
        if "k5cg" in m["name"]:
            k5 += 1
        a = agg.setdefault(nm, collections.defaultdict(float))
        a["n"] += 1
        for k, v in m.items():
            if k != "name":
                a[k] += v
    return agg


def table(agg, title, extra_hit=False):
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    lines = [f"total kernel time {tot / 1e3:.1f} us", "",
             "| pass | launches | total us | share | avg us | DRAM rd MB/launch | DRAM wr MB/launch | L2 MB/launch |"
             + (" L2 hit % |" if extra_hit else ""),
             "|---|---|---|---|---|---|---|---|" + ("---|" if extra_hit else "")]
    for nm, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        n = a["n"]
        t = a["gpu__time_duration.sum"] / 1e3
        row = (f"| `{nm}` | {int(n)} | {t:.1f} | {t / (tot / 1e3):.3f} | {t / n:.2f} | "
               f"{a['dram__bytes_read.sum'] / n / 1e6:.2f} | {a['dram__bytes_write.sum'] / n / 1e6:.2f} | "
               f"{a['lts__t_bytes.sum'] / n / 1e6:.1f} |")
        if extra_hit:
            row += f" {a['lts__t_sector_hit_rate.pct'] / n:.1f} |"
        lines.append(row)
    return "\n".join(lines)


cold = launches(os.path.join(OUT, "launches_cold.csv"))
warm = launches(os.path.join(OUT, "launches_warm.csv"))
md = [f"# {tag} ncu launch list — default path (C2, one frame)", "",
      "`tools/profile.sh` under gpurun on one B200 over `tools/prof_frame.py 1` (eager launches, no CUDA graph, "
      "serialised by ncu: compare shares, not absolutes; bench timings are the graph + PDL numbers). "
      "Launches mapped to pass names by kernel template mode.", "",
      "## Cold cache (ncu flushes L2 before every kernel)", "", table(cold, "cold"), "",
      "## Warm cache (`--cache-control none`: the L2 state a real frame sees)", "", table(warm, "warm", True), ""]
open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w").write("\n".join(md))
traffic = {nm: {"dram_bytes_per_launch": (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / a["n"],
                "dram_bytes_per_launch_warm": (warm[nm]["dram__bytes_read.sum"] + warm[nm]["dram__bytes_write.sum"]) / warm[nm]["n"] if nm in warm else None,
                "avg_us_ncu": a["gpu__time_duration.sum"] / a["n"] / 1e3,
                "avg_us_ncu_warm": (warm[nm]["gpu__time_duration.sum"] / warm[nm]["n"] / 1e3) if nm in warm else None,
                "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cold = L2 flushed per kernel; warm = --cache-control none), tools/profile.sh, {tag}"}
           for nm, a in cold.items()}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
rep = os.path.join(OUT, "prof_iter.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), rep], capture_output=True, text=True).stdout
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_iteration.txt"), "w").write(
        f"# {tag}: ncu --set full of one steady-state CG iteration (tools/profile.sh step 3; cold cache per kernel)\n"
        "# fields: duration (us), DRAM MB, instructions, issue-active %, warps active/eligible per scheduler, L2 hit %,\n"
        "# smem bank conflicts, top stall reasons (cycles per issued instruction)\n\n" + out)
print(open(os.path.join(ROOT, "profiles", f"{tag}_launches.md")).read())
