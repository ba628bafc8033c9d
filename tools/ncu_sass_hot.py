"""Where a kernel's warps stall: ncu source-page stall samples by opcode class and along the code.
python tools/ncu_sass_hot.py REPORT.ncu-rep KERNEL_REGEX [launch_skip]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre, "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
iS, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
iN = h.index("Warp Stall Sampling (Not-issued Samples)")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[iS]) for r in data) or 1.0
print(rows[0][1][:90], "| SASS instructions", len(data), "| samples", int(tot))
cls, cnt = defaultdict(float), defaultdict(int)
for r in data:
    toks = r[iSrc].split()
    op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")).split(".")[0]
    cls[op] += f(r[iS])
    cnt[op] += 1
print("by opcode (share of stall samples, static count):")
for k, v in sorted(cls.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {k:10s} {v / tot:.3f}  {cnt[k]}")
print("along the code (deciles of the instruction stream):")
n = len(data)
for d in range(10):
    seg = data[d * n // 10:(d + 1) * n // 10]
    print(f"  {d}: {sum(f(r[iS]) for r in seg) / tot:.3f}")
