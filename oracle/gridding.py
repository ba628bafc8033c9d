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

import numpy as np

from .nlinv_oracle import _radial_coords, _round_snapped, radial_margin

__all__ = ["radial_cells", "grid_nearest"]


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
