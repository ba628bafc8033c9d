"""Standalone normal operator calls for ncu launch lists (C5): python tools/normal_probe.py NG COILS CALLS."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1301_1215_b200 import Plan, radial_mask

ng, J, calls = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else ("1024", "32", "2")))
plan = Plan(ng, J, radial_mask(ng, 15, 5, 0))
u = lambda seed, shape: torch.from_numpy(synth.splitmix64_uniform(seed, 2 * int(np.prod(shape))).astype(np.float32)
                                         .view(np.complex64).reshape(shape)).cuda()
x, dx = u(1, plan.x_shape), u(2, plan.x_shape)
out = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
img = u(4, (J, ng, ng))
imo = torch.empty_like(img)
plan.set_point(x)
for _ in range(calls):
    plan.normal(0.37, dx, out)
    plan.fft2d(img, False, imo)
torch.cuda.synchronize()
print("ok")
