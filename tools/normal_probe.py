"""One standalone normal-operator application at a size above L2 (for ncu): NG J REPS."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
from paper_1301_1215_b200 import Plan, radial_mask  # noqa: E402
ng, J, reps = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 32, 2)))
plan = Plan(ng, J, radial_mask(ng, 15, 5, 0))
x = torch.from_numpy(synth.random_complex(1, plan.x_shape).astype("complex64")).cuda()
dx = torch.from_numpy(synth.random_complex(2, plan.x_shape).astype("complex64")).cuda()
out = torch.empty_like(dx)
plan.set_point(x)
for _ in range(reps):
    plan.normal(0.37, dx, out)
torch.cuda.synchronize()
print("ok")
