"""Probe: throughput of 1 vs 2 vs 3 concurrent C2 reconstructions (separate plans/streams)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1301_1215_b200 import Plan, radial_mask
NG, J = 384, 12
mask = radial_mask(NG, 15, 5, 0)
_, _, y = synth.frame_inputs(J, NG)
yd = torch.from_numpy(y.astype(np.complex64)).cuda()
for P in (1, 2, 3, 4):
    plans = [Plan(NG, J, mask) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    xs = [torch.empty(plans[0].x_shape, dtype=torch.complex64, device="cuda") for _ in range(P)]
    def run(first):
        for p, s, x in zip(plans, streams, xs):
            with torch.cuda.stream(s):
                p.reconstruct(yd, None if first else x, 7, 10, x_out=x, want_image=False)
    run(True); run(False); run(False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): run(False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{P} concurrent: {10*P/dt:.1f} frames/s total, {dt/10*1e3:.2f} ms per round")
    for p in plans: p.close()
