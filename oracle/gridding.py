"""fp64 CPU oracle of gridding radial samples onto the Cartesian grid -- TEST INFRASTRUCTURE ONLY.

PAPER.md P:233: "After an initial interpolation of the data to the grid which is performed as a
pre-processing step on the CPU, all further operations can be performed on the grid"; P:346
radial acquisition. SURVEY.md §8(f) row f2 moves this step onto the GPU.

Reading R20: nearest-cell interpolation with the cell rule of R12 (the one that
defines P_k): sample (s, i) of frame f goes to cell (ng/2 + round(r sin theta), ng/2 +
round(r cos theta)) (snapped, half away from zero), out-of-grid samples are dropped, and the
gridded value of a cell is the mean of its samples taken in ascending (s, i) order -- the
least-squares value of one cell fitted to all measurements that fall into it. P_k is the set of
cells with at least one sample, i.e. ``radial_mask``. Off P_k the grid is zero (R16: only P_k y
enters the method).

Plain loops; shares nothing with the CUDA path. Pinned by tests/test_oracle_gridding.py.
"""
from __future__ import annotations

import math

import numpy as np

from .nlinv_oracle import _radial_coords, _round_snapped, radial_margin

__all__ = ["radial_cells", "grid_nearest", "kb_beta", "kb_window", "grid_kb"]


def radial_cells(ng: int, spokes: int, turns: int, frame: int) -> np.ndarray:
    """Linear cell index ky*ng + kx of every sample (int64 [spokes, ng]); -1 if off the grid."""
    if radial_margin(ng, spokes, turns, frame) <= 1e-6:
        raise ValueError("radial sample within 1e-6 of a snap midpoint (R12)")
    out = np.full(spokes * ng, -1, dtype=np.int64)
    for q, (vx, vy) in enumerate(_radial_coords(ng, spokes, turns, frame)):
        kx = ng // 2 + _round_snapped(vx)
        ky = ng // 2 + _round_snapped(vy)
        if 0 <= kx < ng and 0 <= ky < ng:
            out[q] = ky * ng + kx
    return out.reshape(spokes, ng)


def grid_nearest(samples: np.ndarray, ng: int, spokes: int, turns: int, frame: int):
    """Gridded frame y [J, ng, ng] (mean of the samples of each cell, zero elsewhere) and the
    per-cell sample count [ng, ng] from raw samples [J, spokes, ng]."""
    cells = radial_cells(ng, spokes, turns, frame)
    J = samples.shape[0]
    acc = np.zeros((J, ng * ng), dtype=np.complex128)
    cnt = np.zeros(ng * ng, dtype=np.int64)
    for s in range(spokes):
        for i in range(ng):
            cidx = cells[s, i]
            if cidx < 0:
                continue
            cnt[cidx] += 1
            for j in range(J):
                acc[j, cidx] += samples[j, s, i]
    y = np.zeros_like(acc)
    hit = cnt > 0
    y[:, hit] = acc[:, hit] / cnt[hit]
    return y.reshape(J, ng, ng), cnt.reshape(ng, ng)


# --------------------------------------------------------------------------------------
# Convolution (Kaiser-Bessel) gridding with a real-valued PSF (reading R22)
# --------------------------------------------------------------------------------------
# The paper interpolates the radial data onto the 2x oversampled grid before the iteration
# ("to achieve a high accuracy when initially interpolating the measured data onto
# the Cartesian grid") and then treats F^-1 P_k F as a convolution with the point-spread function
# (P:234-236). Reading R22: the gridded value of a cell is the kernel-weighted least-squares fit to
# the samples around it, y_g(k) = sum_s h(k - k_s) d_s / sum_s h(k - k_s), and its weight in the
# data term is the PSF(k) = sum_s h(k - k_s), i.e. the method runs with the real-valued
# P_k = sqrt(PSF) on the data and P_k^2 = PSF inside the normal operator. h is the separable
# Kaiser-Bessel window of width W grid cells (Beatty et al.'s beta for oversampling 2).

def kb_beta(width: float, osf: float = 2.0) -> float:
    """Beatty-Brau-Nishimura optimal beta for a Kaiser-Bessel window of `width` cells."""
    return math.pi * math.sqrt((width / osf) ** 2 * (osf - 0.5) ** 2 - 0.8)


def kb_window(d: float, width: float, beta: float) -> float:
    """h(d) = I0(beta sqrt(1 - (2d/W)^2)) / I0(beta) for |d| <= W/2, else 0 (h(0) = 1)."""
    u = 2.0 * d / width
    if abs(u) > 1.0:
        return 0.0
    return _i0(beta * math.sqrt(1.0 - u * u)) / _i0(beta)


def _i0(z: float) -> float:
    """Modified Bessel function I0 by its power series (converges for all z; |z| <= 20 here)."""
    term, s, k = 1.0, 1.0, 1
    q = 0.25 * z * z
    while term > 1e-17 * s:
        term *= q / (k * k)
        s += term
        k += 1
    return s


def grid_kb(samples: np.ndarray, ng: int, spokes: int, turns: int, frame: int, width: float = 4.0,
            beta: float | None = None):
    """KB-gridded frame y_g [J, ng, ng] (weighted mean, zero where the PSF is 0) and the PSF
    [ng, ng] from raw samples [J, spokes, ng] of the R12 trajectory (coordinates from the grid
    centre; cells outside the grid are dropped)."""
    if beta is None:
        beta = kb_beta(width)
    J = samples.shape[0]
    c = ng // 2
    num = np.zeros((J, ng, ng), dtype=np.complex128)
    psf = np.zeros((ng, ng), dtype=np.float64)
    half = width / 2.0
    for s in range(spokes):
        theta = math.pi * (s * turns + (frame % turns)) / (spokes * turns)
        ct, st = math.cos(theta), math.sin(theta)
        for i in range(ng):
            r = float(i - ng // 2)
            kx, ky = c + r * ct, c + r * st            # continuous grid position of the sample
            for gy in range(math.ceil(ky - half), math.floor(ky + half) + 1):
                hy = kb_window(gy - ky, width, beta)
                if hy == 0.0 or not 0 <= gy < ng:
                    continue
                for gx in range(math.ceil(kx - half), math.floor(kx + half) + 1):
                    hx = kb_window(gx - kx, width, beta)
                    if hx == 0.0 or not 0 <= gx < ng:
                        continue
                    h = hx * hy
                    psf[gy, gx] += h
                    num[:, gy, gx] += h * samples[:, s, i]
    y = np.zeros_like(num)
    on = psf > 0
    y[:, on] = num[:, on] / psf[on]
    return y, psf
