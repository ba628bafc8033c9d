"""Run C2 frames eagerly (no CUDA graph) for ncu: python tools/prof_frame.py [frames]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NLINV_NO_GRAPH", "1")

import numpy as np
import torch

import synth
from paper_1301_1215_b200 import Plan, radial_mask

NG, J = int(os.environ.get("NG", 384)), int(os.environ.get("J", 12))
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mask = radial_mask(NG, 15, 5, 0)
plan = Plan(NG, J, mask)
_, _, y = synth.frame_inputs(J, NG)
yd = torch.from_numpy(y.astype(np.complex64)).cuda()
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
for f in range(frames):
    plan.reconstruct(yd, None if f == 0 else x, 7, 10, x_out=x, image_out=img)
torch.cuda.synchronize()
print("ok", plan.launch_count)
