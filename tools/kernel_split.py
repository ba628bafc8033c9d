"""Per-kernel time split of one warm frame (every kernel bracketed by CUDA events, no graph):
python tools/kernel_split.py [J] [ng]. Environment switches (NLINV_*) select the execution path."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1301_1215_b200 import Plan, radial_mask

J = int(sys.argv[1]) if len(sys.argv) > 1 else 12
NG = int(sys.argv[2]) if len(sys.argv) > 2 else 384
plan = Plan(NG, J, radial_mask(NG, 15, 5, 0))
_, _, y = synth.frame_inputs(J, NG)
yd = torch.from_numpy(y.astype(np.complex64)).cuda()
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
for f in range(3):
    plan.reconstruct(yd, None if f == 0 else x, 7, 10, x_out=x, image_out=img)
torch.cuda.synchronize()
plan.set_profiling(True)
plan.reconstruct(yd, x, 7, 10, x_out=x, image_out=img)
prof = plan.profile()
plan.set_profiling(False)
tot = sum(v["ms"] for v in prof.values())
out = {"J": J, "ng": NG, "env": {k: v for k, v in os.environ.items() if k.startswith("NLINV_")}, "frame_ms_eager": round(tot, 4),
       "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 4), "us_per_launch": round(1e3 * v["ms"] / v["launches"], 2)}
                   for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}
print(json.dumps(out))
