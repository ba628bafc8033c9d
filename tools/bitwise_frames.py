"""Run a short warm C2 stream (and a C4 Newton step, and the standalone operators at 1024^2) with the
in-tree libnlinv.so and save every output, so two library builds can be compared bit for bit:
python tools/bitwise_frames.py OUT.npz   (then: python tools/bitwise_frames.py --compare A.npz B.npz)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in sorted(a.files):
        same = np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8))
        d = float(np.max(np.abs(a[k] - b[k]))) if not same else 0.0
        print(f"{k}: {'bit-identical' if same else 'DIFFERS (max abs %.3e)' % d}")
    sys.exit(0)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1301_1215_b200 import Plan, radial_mask  # noqa: E402

out = {}
ng, J = 384, 12
plan = Plan(ng, J, radial_mask(ng, 15, 5, 0))
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
for f in range(3):
    _, _, y = synth.frame_inputs(J, ng, t=f)
    plan.set_mask(radial_mask(ng, 15, 5, f))
    xo, img = plan.reconstruct(torch.from_numpy(y.astype(np.complex64)).cuda(), None if f == 0 else x, 7, 10)
    x = xo.clone()
    out[f"c2_frame{f}_image"] = img.cpu().numpy()
    out[f"c2_frame{f}_x"] = xo.cpu().numpy()
plan.close()
for ng, J in ((1024, 8), (384, 32)):
    plan = Plan(ng, J, radial_mask(ng, 15, 5, 1))
    xs = torch.from_numpy(synth.random_complex(5, plan.x_shape).astype(np.complex64)).cuda()
    dx = torch.from_numpy(synth.random_complex(6, plan.x_shape).astype(np.complex64)).cuda()
    plan.set_point(xs)
    out[f"normal_{ng}_{J}"] = plan.normal(0.37, dx).cpu().numpy()
    out[f"fft2d_{ng}_{J}"] = plan.fft2d(dx[1:].contiguous(), inverse=False).cpu().numpy()
    plan.close()
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1], len(out))
