"""Split a C2 frame's device time into Newton-step heads and CG iterations (graph mode):
time frames with L = 1, 5, 10 CG iterations; per-iteration cost = slope, head = intercept / K."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import synth  # noqa: E402
from paper_1301_1215_b200 import Plan, radial_mask  # noqa: E402
NG, J, K = 384, 12, 7
_, _, y = synth.frame_inputs(J, NG)
plan = Plan(NG, J, radial_mask(NG, 15, 5, 0))
yd = torch.from_numpy(y.astype(np.complex64)).cuda()
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
img = torch.empty(plan.image_shape, dtype=torch.complex64, device="cuda")
st = torch.cuda.current_stream()
res = {}
plan.reconstruct(yd, None, K, 10, x_out=x, image_out=img)
for L in (1, 5, 10):
    for _ in range(3):
        plan.reconstruct(yd, x, K, L, x_out=x, image_out=img)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        plan.reconstruct(yd, x, K, L, x_out=x, image_out=img)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    res[L] = statistics.median(ts)
it = (res[10] - res[1]) / 9 / K
head = (res[1] - K * it) / K
print({"ms_L1": res[1], "ms_L5": res[5], "ms_L10": res[10], "us_per_cg_iteration": round(it * 1e3, 2),
       "us_per_newton_head_incl_last_update": round(head * 1e3, 2),
       "head_share_at_L10": round(K * head / res[10], 3)})
