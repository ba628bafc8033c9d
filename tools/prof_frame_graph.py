"""Run C2 frames through the CUDA-graph path (as bench.py does) for ncu --graph-profiling graph:
python tools/prof_frame_graph.py [frames]. Frame 0 captures the graph of the cold start, frame 1 the
warm-start graph; later frames replay it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
from paper_1301_1215_b200 import Plan, radial_mask

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 3
NG, J = 384, 12
plan = Plan(NG, J, radial_mask(NG, 15, 5, 0))
_, _, y = synth.frame_inputs(J, NG)
yd = torch.from_numpy(y.astype(np.complex64)).cuda()
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
s = torch.cuda.Stream()
for f in range(frames):
    plan.reconstruct(yd, None if f == 0 else x, 7, 10, x_out=x, image_out=img, stream=s)
torch.cuda.synchronize()
print("ok", plan.launch_count)
