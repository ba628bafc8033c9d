"""Batched 2D FFT through nlinv_debug_fft2d (for ncu): python tools/fft_probe.py NG BATCH REPS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1301_1215_b200 import Plan, radial_mask
ng, batch, reps = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 32, 3)))
plan = Plan(ng, 1, radial_mask(ng, 4, 1, 0))
x = torch.randn(batch, ng, ng, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
for _ in range(reps):
    plan.fft2d(x, False, y)
torch.cuda.synchronize()
print("ok")
