"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module is the ONLY code both sides of a parity comparison receive data from.
It holds none of the reconstruction method's arithmetic (no weights W, no masks
P_k / M_Omega, no operators, no CG / IRGNM): it only draws the things a scanner
and a patient would hand the method.

* ``splitmix64_uniform`` -- counter-based U[-1, 1) numbers (SURVEY.md §8(d), C5 recipe).
* ``shepp_logan``        -- the modified Shepp-Logan phantom, the
                            stand-in for the paper's cardiac scans (Fig. 10).
* ``coil_maps``          -- smooth complex Gaussian receive sensitivities c_j on a ring
                            ("Each coil possesses a unique spatial sensitivity map c_j").
* ``acquire``            -- full-grid k-space data y_j of Eq. 1,
                            discretised on the doubled Cartesian grid. The
                            projection onto the measured positions (P_k of Eq. 2) is NOT
                            applied here: it is part of the method, and both the oracle
                            and the CUDA path apply their own P_k (R3).

All arrays are numpy; complex data are complex128 here and are rounded to complex64
by the caller that feeds the GPU.
"""
from __future__ import annotations

import numpy as np

_MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """``count`` consecutive splitmix64 outputs for state ``seed`` (uint64, wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        k = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def splitmix64_uniform(seed: int, count: int) -> np.ndarray:
    """U[-1, 1) doubles from the top 53 bits of splitmix64. Callers that feed the GPU round
    them to fp32 first and hand the same rounded values to the oracle."""
    z = splitmix64(seed, count)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def random_complex(seed: int, shape) -> np.ndarray:
    """Complex array with re/im interleaved draws from ``splitmix64_uniform`` (complex128)."""
    n = int(np.prod(shape))
    u = splitmix64_uniform(seed, 2 * n)
    return (u[0::2] + 1j * u[1::2]).reshape(shape)


# Modified Shepp-Logan (A, a, b, x0, y0, phi_deg), SURVEY.md A14.
SHEPP_LOGAN = (
    (1.0, 0.69, 0.92, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.874, 0.0, -0.0184, 0.0),
    (-0.2, 0.11, 0.31, 0.22, 0.0, -18.0),
    (-0.2, 0.16, 0.41, -0.22, 0.0, 18.0),
    (0.1, 0.21, 0.25, 0.0, 0.35, 0.0),
    (0.1, 0.046, 0.046, 0.0, 0.1, 0.0),
    (0.1, 0.046, 0.046, 0.0, -0.1, 0.0),
    (0.1, 0.046, 0.023, -0.08, -0.605, 0.0),
    (0.1, 0.023, 0.023, 0.0, -0.606, 0.0),
    (0.1, 0.023, 0.046, 0.06, -0.605, 0.0),
)


def shepp_logan(n: int, t: float | None = None) -> np.ndarray:
    """n x n modified Shepp-Logan phantom sampled at pixel centres of [-1,1]^2 (real, float64).

    Row index runs top to bottom (y = +1 at row 0), column index left to right.
    ``t`` (frame index) enables the C4 motion model: ellipses 3 and 4 (1-based) have
    their semi-axes scaled by 1 + 0.1 sin(2 pi t / 25).
    """
    c = -1.0 + (2.0 * np.arange(n) + 1.0) / n
    X = c[None, :]
    Y = -c[:, None]
    img = np.zeros((n, n))
    for idx, (A, a, b, x0, y0, phi) in enumerate(SHEPP_LOGAN):
        if t is not None and idx in (2, 3):
            s = 1.0 + 0.1 * np.sin(2.0 * np.pi * t / 25.0)
            a, b = a * s, b * s
        ph = np.deg2rad(phi)
        xr = (X - x0) * np.cos(ph) + (Y - y0) * np.sin(ph)
        yr = -(X - x0) * np.sin(ph) + (Y - y0) * np.cos(ph)
        img = img + A * (((xr / a) ** 2 + (yr / b) ** 2) <= 1.0)
    return img


def embed(img: np.ndarray, ng: int) -> np.ndarray:
    """Place an n x n image in the centre of an ng x ng zero grid (rows/cols ng/4 .. 3ng/4)."""
    n = img.shape[-1]
    q = (ng - n) // 2
    out = np.zeros(img.shape[:-2] + (ng, ng), dtype=np.result_type(img, np.complex128))
    out[..., q:q + n, q:q + n] = img
    return out


def coil_maps(ncoils: int, ng: int) -> np.ndarray:
    """J smooth complex sensitivities on the ng x ng grid (complex128, [J, ng, ng]).

    Coil j: Gaussian lobe of width 0.4 n centred 0.6 n from the grid centre at angle
    phi_j = 2 pi j / J, times the constant phase e^{i phi_j}; normalised so that the
    root-sum-of-squares over the centred n x n field of view peaks at 1.
    """
    n = ng // 2
    cgrid = ng / 2.0
    yy, xx = np.meshgrid(np.arange(ng, dtype=np.float64), np.arange(ng, dtype=np.float64), indexing="ij")
    maps = np.empty((ncoils, ng, ng), dtype=np.complex128)
    for j in range(ncoils):
        phi = 2.0 * np.pi * j / ncoils
        cx = cgrid + 0.6 * n * np.cos(phi)
        cy = cgrid + 0.6 * n * np.sin(phi)
        d2 = (xx - cx) ** 2 + (yy - cy) ** 2
        maps[j] = np.exp(-d2 / (2.0 * (0.4 * n) ** 2)) * np.exp(1j * phi)
    q = (ng - n) // 2
    rss = np.sqrt(np.sum(np.abs(maps[:, q:q + n, q:q + n]) ** 2, axis=0))
    return maps / rss.max()


def acquire(image_grid: np.ndarray, coils: np.ndarray, norm: float | None = 100.0) -> np.ndarray:
    """Fully sampled grid k-space y_j[k] of Eq. 1: the sum over the grid
    points x of rho(x) c_j(x) e^{-i k.x}, with k and x both measured from the grid centre,
    normalised by 1/ng (complex128, [J, ng, ng]).

    The image is assumed to already lie inside the field of view (see ``embed``). The
    result is scaled so that its l2 norm is ``norm`` (None = unscaled).
    """
    ng = image_grid.shape[-1]
    obj = image_grid[None] * coils
    # centred DFT: shift the grid centre to index 0, transform, shift back.
    y = np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(obj, axes=(-2, -1))), axes=(-2, -1)) / ng
    if norm is not None:
        y = y * (norm / np.linalg.norm(y))
    return y


def frame_inputs(ncoils: int, ng: int, t: float | None = None, norm: float | None = 100.0):
    """Phantom (n x n), coil maps and full-grid data for one frame."""
    n = ng // 2
    img = shepp_logan(n, t)
    coils = coil_maps(ncoils, ng)
    y = acquire(embed(img, ng), coils, norm)
    return img, coils, y


def radial_trajectory(ng: int, spokes: int, turns: int, frame: int) -> np.ndarray:
    """k-space coordinates (kx, ky) in grid units from the grid centre of the radial spokes of one
    frame (float64, [spokes, ng, 2]): spoke s at theta = pi (s T + (f mod T)) / (S T), samples at
    r = i - ng/2 (SURVEY.md A12 / DESIGN.md R12). Acquisition geometry only: the assignment of
    samples to grid cells (the gridding) is not done here."""
    out = np.empty((spokes, ng, 2), dtype=np.float64)
    for s in range(spokes):
        theta = np.pi * (s * turns + (frame % turns)) / (spokes * turns)
        r = np.arange(ng, dtype=np.float64) - ng // 2
        out[s, :, 0] = r * np.cos(theta)
        out[s, :, 1] = r * np.sin(theta)
    return out


def acquire_radial(image_grid: np.ndarray, coils: np.ndarray, traj: np.ndarray, scale: float = 1.0) -> np.ndarray:
    """Non-Cartesian samples of Eq. 1 at the trajectory points: the sum over grid
    points x of rho(x) c_j(x) e^{-2 pi i k.x / ng}, k and x from the grid centre, / ng, times
    ``scale`` (complex128, [J, spokes, ng]). At integer k this is ``acquire`` at that cell.
    Evaluated separably (x then y) over the rows/columns where the object is non-zero."""
    ng = image_grid.shape[-1]
    c = ng // 2
    obj = image_grid[None] * coils                       # [J, ng, ng]
    rows = np.flatnonzero(np.any(np.abs(image_grid) > 0, axis=1))
    cols = np.flatnonzero(np.any(np.abs(image_grid) > 0, axis=0))
    sub = obj[:, rows][:, :, cols]                       # [J, ry, rx]
    k = traj.reshape(-1, 2)
    ex = np.exp(-2j * np.pi * np.outer(k[:, 0], cols - c) / ng)    # [ns, rx]
    ey = np.exp(-2j * np.pi * np.outer(k[:, 1], rows - c) / ng)    # [ns, ry]
    out = np.empty((obj.shape[0], k.shape[0]), dtype=np.complex128)
    for j in range(obj.shape[0]):
        t = ex @ sub[j].T                                # [ns, ry]: x-transform of every row
        out[j] = np.sum(t * ey, axis=1) / ng
    return out.reshape(obj.shape[0], traj.shape[0], traj.shape[1]) * scale


def radial_frame_inputs(ncoils: int, ng: int, spokes: int, turns: int, frame: int, t: float | None = None):
    """Raw radial samples of one frame [J, spokes, ng], scaled like ``frame_inputs`` (so that the
    fully sampled grid data have l2 norm 100)."""
    n = ng // 2
    img = embed(shepp_logan(n, t), ng)
    coils = coil_maps(ncoils, ng)
    scale = 100.0 / np.linalg.norm(acquire(img, coils, None))
    return acquire_radial(img, coils, radial_trajectory(ng, spokes, turns, frame), scale)
