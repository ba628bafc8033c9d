"""Per-pass DRAM throughput from tools/c5_passes.sh's ncu launch list: python tools/c5_summary.py [csv]."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
fn = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "c5_pk_passes.csv")
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6452.8
rows = list(csv.reader(open(fn)))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
per = collections.OrderedDict()
for r in rows[i + 1:]:
    if len(r) != len(h):
        continue
    x = dict(zip(h, r))
    k = x["Kernel Name"].split("(")[0].replace("void nlv::", "")[:45]
    per.setdefault(k, collections.defaultdict(float))
    per[k][x["Metric Name"]] += float(x["Metric Value"].replace(",", ""))
    if x["Metric Name"] == "gpu__time_duration.sum":
        per[k]["n"] += 1
print("| kernel | launches | us per launch | DRAM MB per launch | frac of HBM |")
print("|---|---|---|---|---|")
for k, v in per.items():
    us = v["gpu__time_duration.sum"] / v["n"] / 1e3
    mb = (v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / v["n"] / 1e6
    print(f"| `{k}` | {int(v['n'])} | {us:.1f} | {mb:.1f} | {mb / us * 1e3 / peak:.2f} |")
