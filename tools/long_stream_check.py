"""Long warm-started C2 stream against the oracle's own fp64 chain: does the fp32 reconstruction drift from
the oracle over many frames (each frame's prior is the previous frame's x on both sides)?
python tools/long_stream_check.py [frames]  -> one JSON line per frame + a summary (image and rho relative L2)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import synth
from paper_1301_1215_b200 import Plan

F = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ng, J, S, T, K, L = 384, 12, 15, 5, 7, 10
O.set_workers(os.cpu_count() or 1)
plan = Plan(ng, J, O.radial_mask(ng, S, T, 0))
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
frame = torch.empty(plan.y_shape, dtype=torch.complex64, device="cuda")
xo = O.initial_x(J, ng)
errs = []
t0 = time.time()
for f in range(F):
    _, _, y = synth.frame_inputs(J, ng, t=f)
    y = np.ascontiguousarray(y.astype(np.complex64))
    mask = O.radial_mask(ng, S, T, f)
    frame.copy_(torch.from_numpy(y))
    plan.set_mask(torch.from_numpy(mask).cuda())
    plan.reconstruct(frame, None if f == 0 else x, K, L, x_out=x, image_out=img)
    xo, _ = O.irgnm(y.astype(np.complex128), mask, xo, xo, K, L)
    io = O.image_from_x(xo)
    ig = img.cpu().numpy().astype(np.complex128)
    e = float(np.linalg.norm(ig - io) / np.linalg.norm(io))
    q, n = ng // 4, ng // 2
    xr = x[0].cpu().numpy().astype(np.complex128)[q:q + n, q:q + n]
    er = float(np.linalg.norm(xr - xo[0, q:q + n, q:q + n]) / np.linalg.norm(xo[0, q:q + n, q:q + n]))
    errs.append(e)
    print(json.dumps({"frame": f, "image_rel_l2": e, "rho_rel_l2": er, "elapsed_s": round(time.time() - t0, 1)}), flush=True)
print(json.dumps({"frames": F, "image_rel_l2_max": max(errs), "image_rel_l2_last": errs[-1],
                  "image_rel_l2_first5_max": max(errs[:5])}))
plan.close()
