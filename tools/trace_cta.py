"""CTA timelines of one column pass (needs a -DNLV_TRACE build): python tools/trace_cta.py MODE"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NLINV_NO_FRAME"] = "1"
os.environ["NLINV_NO_GRAPH"] = "1"
import numpy as np, torch
import synth
from paper_1301_1215_b200 import Plan, radial_mask
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 3
NG, J = 384, int(os.environ.get("J", 12))
plan = Plan(NG, J, radial_mask(NG, 15, 5, 0))
_, _, y = synth.frame_inputs(J, NG)
yd = torch.from_numpy(y.astype(np.complex64)).cuda()
x = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
plan.reconstruct(yd, None, 1, 2, x_out=x, want_image=False)
plan.trace_enable(mode)
plan.reconstruct(yd, x, 1, 3, x_out=x, want_image=False)   # the last launch of that mode is kept
tr = plan.trace_read().astype(np.float64)
rows = tr[(tr[:, 0] > 0)]
t0 = rows[:, 0].min()
rel = (rows - t0) / 1e3
names = ["start", "tw+loads issued", "fft1 done", "mid done", "fft2 done", "epilogue done", "reduce done"]
if mode == 9:  # k5cg_kernel (one barrier): 7 = epilogue + dots, 3 = barrier, 5 = totals, 6 = tile updates, 4 = rho updates
    order = [0, 1, 2, 7, 3, 5, 6, 4]
    names6 = ["start", "prologue + rho stripe", "K5 fft done", "Ap + dots done", "barrier passed",
              "partial totals read", "tile r/dx/p updates issued", "rho stripe updates"]
if mode == 6:  # fused K5 + CG + K1 (iteration 1): 7 = epilogue done, 3 = barrier 1 passed, 4 = barrier 2 passed
    order = [0, 1, 2, 7, 3, 4, 5, 6]
    names6 = ["start", "prologue loads issued", "K5 fft done", "Ap + <p,Ap> done", "barrier 1 passed",
              "r update + barrier 2", "p update + K1 fft + store", "end"]
    tr0 = plan.trace_read().astype(np.float64) if False else None
print(f"mode {mode}: {len(rows)} CTAs; kernel span {(rows[:, 6].max() - t0)/1e3:.2f} us")
if mode in (6, 9):
    rows = rows[:, order]
    rel = (rows - t0) / 1e3
    names = names6
for k in range(1, 8 if mode in (6, 9) else 7):
    ok = rows[:, k] > 0
    if ok.sum() == 0: continue
    d = (rows[ok, k] - rows[ok, k - 1 if rows[ok, k-1].min() > 0 else 0]) / 1e3
    print(f"  {names[k]:18s} stamp mean {rel[ok, k].mean():7.2f} us  max {rel[ok, k].max():7.2f}   step mean {d.mean():6.2f} us")
print("  start times: min %.2f  median %.2f  max %.2f us" % (rel[:, 0].min(), np.median(rel[:, 0]), rel[:, 0].max()))
