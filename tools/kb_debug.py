"""Debug helper: KB-gridded reconstruction vs the oracle at several (K, L) (prints only)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle as O  # noqa: E402
from oracle import gridding as G  # noqa: E402
import synth  # noqa: E402
import paper_1301_1215_b200 as B  # noqa: E402

ng, J, S, T = 32, 8, 8, 1
raw = synth.radial_frame_inputs(J, ng, S, T, 0).astype(np.complex64)
plan = B.Plan(ng, J, O.radial_mask(ng, S, T, 0))
plan.set_trajectory(S, T, kernel="kb", width=4.0)
y = plan.grid_radial(0, torch.from_numpy(raw).cuda())
yo, psf = G.grid_kb(raw.astype(np.complex128), ng, S, T, 0, width=4.0)
r = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
print("gridded y rel", r(y.cpu().numpy()[:, psf > 0], yo[:, psf > 0]))
for K, L in ((2, 10), (3, 10)):
    x0 = O.initial_x(J, ng)
    xo, hist = O.irgnm(yo.astype(np.complex64).astype(np.complex128), np.sqrt(psf), x0, x0, K, L)
    x, img = plan.reconstruct(y, None, K, L)
    print("KB", K, L, "img rel", r(img.cpu().numpy(), O.image_from_x(xo)), "x rel", r(x.cpu().numpy(), xo),
          plan.stats()["residual"], hist)
    xo2, hist2 = O.irgnm(y.cpu().numpy().astype(np.complex128), np.sqrt(psf), x0, x0, K, L)
    print("KB same y", K, L, "img rel", r(img.cpu().numpy(), O.image_from_x(xo2)))
plan.set_mask(O.radial_mask(ng, S, T, 0))
for K, L in ((2, 10), (3, 10)):
    x0 = O.initial_x(J, ng)
    x2, img2 = plan.reconstruct(y, None, K, L)
    xb, hb = O.irgnm(y.cpu().numpy().astype(np.complex128), O.radial_mask(ng, S, T, 0), x0, x0, K, L)
    print("binary", K, L, "img rel", r(img2.cpu().numpy(), O.image_from_x(xb)), plan.stats()["residual"], hb)
