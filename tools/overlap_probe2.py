"""Probe: 1 x J=12 frame vs P concurrent frames of J=12/P coils (same total working set)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1301_1215_b200 import Plan, radial_mask
NG = 384
mask = radial_mask(NG, 15, 5, 0)
_, _, y = synth.frame_inputs(12, NG)
for P in (1, 2, 3, 4):
    Jp = 12 // P
    yd = torch.from_numpy(y[:Jp].astype(np.complex64)).cuda()
    plans = [Plan(NG, Jp, mask) for _ in range(P)]
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
    print(f"{P} x J={Jp}: {dt/10*1e3:.2f} ms per round (12 coils total)")
    # serial (same stream) for comparison
    t = time.perf_counter()
    for _ in range(10):
        for p, x in zip(plans, xs):
            p.reconstruct(yd, x, 7, 10, x_out=x, want_image=False)
    torch.cuda.synchronize()
    print(f"   serial: {(time.perf_counter()-t)/10*1e3:.2f} ms per round")
    for p in plans: p.close()
