"""Per-phase breakdown of the persistent frame kernel (C2) from %globaltimer stamps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1301_1215_b200 import Plan, radial_mask
NG, J, K, L = 384, int(os.environ.get("J", 12)), 7, 10
mask = radial_mask(NG, 15, 5, 0)
plan = Plan(NG, J, mask)
_, _, y = synth.frame_inputs(J, NG)
yd = torch.from_numpy(y.astype(np.complex64)).cuda()
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
plan.reconstruct(yd, None, K, L, x_out=x, image_out=img)
plan.phase_times_enable()
plan.reconstruct(yd, x, K, L, x_out=x, image_out=img)
ts = np.array(plan.phase_times(), dtype=np.float64)
d = np.diff(ts) / 1e3  # us
labels = []
for n in range(K):
    labels += ["N1 col setpoint", "N2 row setpoint+fwd", "N3 col resadj", "N4 row K4", "N5 col rhs"]
    for it in range(L):
        labels += ["P1 col K1(+p)", "P2 row K2", "P3 col K3", "P4 row K4", "P5 col K5", "P6 update"]
labels += ["O1 col setpoint", "O2 row rss"]
agg = {}
for lab, v in zip(labels, d):
    agg.setdefault(lab, []).append(v)
tot = sum(d)
print(f"frame {tot:.1f} us over {len(d)} phases (labels {len(labels)})")
for k, v in agg.items():
    print(f"{k:24s} n={len(v):3d} mean {np.mean(v):7.2f} us  total {np.sum(v):8.1f} us  share {np.sum(v)/tot:.3f}")
