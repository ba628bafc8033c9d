"""Small frames for compute-sanitizer (tools/sanitize.sh): a C1 frame (8 coils, 32^2, 3 Newton x 3 CG)
and a warm second frame on a 64^2 grid with 5 coils, through the C ABI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1301_1215_b200 import Plan, radial_mask

for ng, J, S in ((32, 8, 8), (64, 5, 11)):
    _, _, y = synth.frame_inputs(J, ng)
    plan = Plan(ng, J, radial_mask(ng, S, 1, 0))
    yd = torch.from_numpy(y.astype(np.complex64)).cuda()
    x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
    img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
    for f in range(2):
        plan.reconstruct(yd, None if f == 0 else x, 3, 3, x_out=x, image_out=img)
    torch.cuda.synchronize()
    print("ok", ng, J, plan.launch_count, float(img.abs().sum()))
    plan.close()
