"""fp64 CPU oracle of the NLINV / IRGNM hot path (§3.1-3.2) -- TEST INFRASTRUCTURE.

Plain, slow, written to be checked against the paper by eye. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may use it. It shares no code with the CUDA path.

Notation follows the paper:
  * x = (rho, chat_1 .. chat_J): the image and the weighted-domain coil sensitivities,
    jointly estimated ("image and coil sensitivities are calculated at the same time").
    Stored as one complex128 array of shape [J+1, ng, ng]; block 0 is rho.
  * F = P_k DTFT M_Omega C W^{-1}   (Eq. 2)
  * IRGNM step (Eq. 3), solved with CG.
Readings of what the paper leaves open are the DESIGN.md "R" items / SURVEY.md A1-A16;
each function names the one it relies on.

Every function here is pinned by ``tests/test_oracle.py`` against something other than
itself (brute-force sums, closed forms, invariants, Table 1 of the paper). No function is
"parity unpinned" except ``reconstruct`` at C2/C4 sizes beyond those properties (see
DESIGN.md §Parity).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OpCounters", "fc", "fch", "dft_matrix_1d", "fov_mask", "radial_mask", "radial_margin",
    "weights_inv", "coils_from_chat", "forward", "derivative", "adjoint", "normal",
    "inner", "cg", "irgnm", "image_from_x", "initial_x", "coil_partition", "Params",
    "newton_step", "set_workers",
]


# --------------------------------------------------------------------------------------
# Table 1 instrumentation: FFTs, channel sums, all-reduce steps per operator
# --------------------------------------------------------------------------------------
@dataclass
class OpCounters:
    fft: int = 0          # Table 1 column "FFT" (one batched transform over all channels = 1)
    chan_sum: int = 0     # column "sum c_j"
    allreduce: int = 0    # column "sum rho_g"

    def reset(self):
        self.fft = self.chan_sum = self.allreduce = 0


COUNTERS = OpCounters()


# --------------------------------------------------------------------------------------
# Centred unitary DFT (reading A1: the paper only says "DTFT")
# --------------------------------------------------------------------------------------
# Coil-parallel timing mode (bench.py's all-core cpu_baseline, SURVEY §8(d) "coil-parallel mode over
# all host cores"): set_workers(n) makes fc / fch transform the channels of a batch on n host threads,
# one channel per task, each with the same library call as the serial path (numpy's FFT releases the
# GIL). The per-channel transforms are independent, so results are bit-identical to the serial mode
# (tests/test_oracle.py::test_workers_bit_identical); nothing else of the method changes.
_POOL = None


def set_workers(n: int) -> None:
    global _POOL
    from concurrent.futures import ThreadPoolExecutor
    if _POOL is not None:
        _POOL.shutdown()
    _POOL = ThreadPoolExecutor(max_workers=n) if n > 1 else None


def _per_channel(f, z: np.ndarray) -> np.ndarray:
    if _POOL is None or z.ndim < 3 or z.shape[0] < 2:
        return f(z)
    return np.stack(list(_POOL.map(f, [z[j] for j in range(z.shape[0])])))


def _fc1(z):
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(z, axes=(-2, -1)), norm="ortho"), axes=(-2, -1))


def _fch1(z):
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(z, axes=(-2, -1)), norm="ortho"), axes=(-2, -1))


def fc(z: np.ndarray) -> np.ndarray:
    """Centred unitary 2D DFT over the last two axes (batched over leading axes = channels).

    (F_c z)[ky,kx] = 1/ng * sum_{y,x} z[y,x] exp(-2 pi i [(ky-c)(y-c) + (kx-c)(x-c)] / ng),
    c = ng/2. Realised with the library FFT and index shifts (exact for even ng).
    """
    COUNTERS.fft += 1
    return _per_channel(_fc1, z)


def fch(z: np.ndarray) -> np.ndarray:
    """Inverse (= adjoint) of ``fc``."""
    COUNTERS.fft += 1
    return _per_channel(_fch1, z)


def dft_matrix_1d(L: int, inverse: bool = False) -> np.ndarray:
    """The centred unitary 1D DFT matrix written out from its definition (tests only)."""
    c = L // 2
    k = np.arange(L)[:, None] - c
    i = np.arange(L)[None, :] - c
    s = 1.0 if inverse else -1.0
    return np.exp(s * 2j * np.pi * k * i / L) / math.sqrt(L)


# --------------------------------------------------------------------------------------
# Masks and weights (Eq. 2 symbols M_Omega, P_k, W; readings A2, A3, A12)
# --------------------------------------------------------------------------------------
def fov_mask(ng: int, fov_full: bool = False) -> np.ndarray:
    """M_Omega: 1 on the centred n x n square, n = ng/2 (A3); all ones in fov_full test mode."""
    m = np.zeros((ng, ng))
    if fov_full:
        m[:] = 1.0
        return m
    q = ng // 4
    m[q:q + ng // 2, q:q + ng // 2] = 1.0
    return m


_SNAP = 1 << 20  # v is snapped to the 2^-20 grid before rounding (A12)


def _radial_coords(ng: int, spokes: int, turns: int, frame: int):
    vs = []
    for s in range(spokes):
        theta = math.pi * (s * turns + (frame % turns)) / (spokes * turns)
        ct, st = math.cos(theta), math.sin(theta)
        for i in range(ng):
            r = float(i - ng // 2)
            vs.append((r * ct, r * st))
    return vs


def _round_snapped(v: float) -> int:
    """Snap v to the 2^-20 grid, then round half away from zero -- in integers (A12)."""
    s = int(round(v * _SNAP))            # snap (v is never near a snap midpoint, see radial_margin)
    a = abs(s)
    q = (a + (_SNAP >> 1)) >> 20         # half away from zero on |s| / 2^20
    return q if s >= 0 else -q


def radial_margin(ng: int, spokes: int, turns: int, frame: int) -> float:
    """Smallest distance (in 2^-20 units) of any v*2^20 from a snap midpoint; must exceed 1e-6."""
    m = 1.0
    for vx, vy in _radial_coords(ng, spokes, turns, frame):
        for v in (vx, vy):
            f = v * _SNAP
            m = min(m, abs(abs(f - math.floor(f)) - 0.5))
    return m


def radial_mask(ng: int, spokes: int, turns: int = 1, frame: int = 0) -> np.ndarray:
    """P_k rasterised from a radial trajectory (P:346 radial; P:233 gridding; rule A12).

    Spoke s of frame f has angle theta = pi (s T + (f mod T)) / (S T); it carries ng samples
    at radii r = i - ng/2; sample (r cos theta, r sin theta) lands on grid cell
    (ky, kx) = (ng/2 + round(r sin theta), ng/2 + round(r cos theta)). Out-of-grid cells are
    dropped, duplicates OR together. Returns uint8 [ng, ng].
    """
    if radial_margin(ng, spokes, turns, frame) <= 1e-6:
        raise ValueError("radial sample within 1e-6 of a snap midpoint (A12)")
    m = np.zeros((ng, ng), dtype=np.uint8)
    for vx, vy in _radial_coords(ng, spokes, turns, frame):
        kx = ng // 2 + _round_snapped(vx)
        ky = ng // 2 + _round_snapped(vy)
        if 0 <= kx < ng and 0 <= ky < ng:
            m[ky, kx] = 1
    return m


def weights_inv(ng: int, a: float = 220.0, b: float = 32.0) -> np.ndarray:
    """w^{-1}(k) = (1 + a |k|^2)^(-b/2), k = (index - ng/2)/ng in [-1/2, 1/2)^2 (A2; P:221 W)."""
    k = (np.arange(ng) - ng // 2) / ng
    k2 = k[:, None] ** 2 + k[None, :] ** 2
    return (1.0 + a * k2) ** (-b / 2.0)


# --------------------------------------------------------------------------------------
# Operators (Eq. 2 / Eq. 3; Table 1)
# --------------------------------------------------------------------------------------
@dataclass
class Params:
    a: float = 220.0
    b: float = 32.0
    alpha0: float = 1.0
    q: float = 1.0 / 3.0
    fov_full: bool = False
    partition: list | None = field(default=None)   # coil counts per emulated GPU (A10)


def coils_from_chat(chat: np.ndarray, winv: np.ndarray) -> np.ndarray:
    """c_j = W^{-1} chat_j = F_c^H (w^{-1} . chat_j)   (one batched FFT)."""
    return fch(winv * chat)


def _channel_sum(terms: np.ndarray, partition) -> np.ndarray:
    """sum_j terms_j in ascending coil order; with a partition, per-GPU partials rho_g first,
    then sum_g rho_g in ascending rank order ("rho = sum^G rho_g")."""
    COUNTERS.chan_sum += 1
    COUNTERS.allreduce += 1
    if partition is None:
        acc = np.zeros_like(terms[0])
        for j in range(terms.shape[0]):
            acc = acc + terms[j]
        return acc
    parts, j0 = [], 0
    for cnt in partition:
        acc = np.zeros_like(terms[0])
        for j in range(j0, j0 + cnt):
            acc = acc + terms[j]
        parts.append(acc)
        j0 += cnt
    acc = np.zeros_like(terms[0])
    for p in parts:
        acc = acc + p
    return acc


def forward(x: np.ndarray, P: np.ndarray, winv: np.ndarray, M: np.ndarray) -> np.ndarray:
    """F(x)_j = P . F_c( M . rho . c_j ),  c_j = W^{-1} chat_j   (Eq. 2; Table 1 row F: 2 FFT)."""
    rho, chat = x[0], x[1:]
    c = coils_from_chat(chat, winv)
    return P * fc(M * rho * c)


def derivative(x: np.ndarray, dx: np.ndarray, P, winv, M) -> np.ndarray:
    """DF_x(drho, dchat)_j = P . F_c( M . (drho . c_j + rho . W^{-1} dchat_j) )
    (Eq. 3 symbol DF; C is bilinear; Table 1 row DF: 2 FFT). c_j is the linearisation point's
    sensitivity; it is evaluated here for self-containment (counted as set-point work)."""
    rho, chat = x[0], x[1:]
    drho, dchat = dx[0], dx[1:]
    saved = COUNTERS.fft
    c = coils_from_chat(chat, winv)
    COUNTERS.fft = saved
    dc = fch(winv * dchat)
    return P * fc(M * (drho * c + rho * dc))


def adjoint(x: np.ndarray, dy: np.ndarray, P, winv, M, partition=None) -> np.ndarray:
    """DF_x^H dy = ( sum_j conj(c_j) . u_j ,  { w^{-1} . F_c( conj(rho) . u_j ) }_j ),
    u_j = M . F_c^H( P . dy_j )   (Eq. 3 symbol DF^H; Table 1 row DF^H: 2 FFT, 1 sum c_j,
    1 sum rho_g -- the all-reduce of P:246)."""
    rho, chat = x[0], x[1:]
    saved = COUNTERS.fft
    c = coils_from_chat(chat, winv)
    COUNTERS.fft = saved
    u = M * fch(P * dy)
    out = np.empty((chat.shape[0] + 1,) + rho.shape, dtype=np.complex128)
    out[0] = M * _channel_sum(np.conj(c) * u, partition)
    out[1:] = winv * fc(np.conj(rho) * u)
    return out


def normal(x: np.ndarray, alpha: float, dx: np.ndarray, P, winv, M, partition=None) -> np.ndarray:
    """(DF^H DF + alpha I) dx   (Eq. 3 left-hand side)."""
    return adjoint(x, derivative(x, dx, P, winv, M), P, winv, M, partition) + alpha * dx


def inner(a: np.ndarray, b: np.ndarray) -> complex:
    """<a, b> = sum conj(a) b over the whole unknown vector (rho counted once; A9)."""
    return complex(np.vdot(a.ravel(), b.ravel()))


def cg(apply_A, b: np.ndarray, iters: int) -> np.ndarray:
    """Textbook conjugate gradients from dx = 0 for exactly ``iters`` iterations (A5, A9).
    If <r,r> becomes exactly 0 all later step sizes are 0 (breakdown flag, no NaNs)."""
    dx = np.zeros_like(b)
    r = b.copy()
    p = b.copy()
    rr = inner(r, r).real
    for _ in range(iters):
        Ap = apply_A(p)
        pAp = inner(p, Ap).real
        gamma = rr / pAp if rr != 0.0 else 0.0
        dx = dx + gamma * p
        r = r - gamma * Ap
        rr_new = inner(r, r).real
        beta = rr_new / rr if rr != 0.0 else 0.0
        p = r + beta * p
        rr = rr_new
    return dx


def initial_x(ncoils: int, ng: int) -> np.ndarray:
    """x_0 = x_ref of the first frame: rho = 1 on the whole grid, chat = 0 (A6)."""
    x = np.zeros((ncoils + 1, ng, ng), dtype=np.complex128)
    x[0] = 1.0
    return x


def newton_step(x, xref, y, P, winv, M, alpha, cg_iters, partition=None):
    """One IRGNM step, Eq. 3: (DF^H DF + alpha_n)(x_{n+1} - x_n) = DF^H (y - F x_n) - alpha_n (x_n - x_ref).
    The data y may be full-grid; only P . y is used (y "zero outside mask support").
    Returns (x_{n+1}, ||P.y - F(x_n)||_2)."""
    r = P * y - forward(x, P, winv, M)
    res = float(np.linalg.norm(r))
    b = adjoint(x, r, P, winv, M, partition) - alpha * (x - xref)
    dx = cg(lambda v: normal(x, alpha, v, P, winv, M, partition), b, cg_iters)
    return x + dx, res


def irgnm(y, P, x0, xref, newton_steps, cg_iters, prm: Params | None = None):
    """IRGNM for one frame (A4: alpha_n = alpha0 q^n restarted every frame).
    Returns (x_K, [residual norm per Newton step])."""
    prm = prm or Params()
    ng = y.shape[-1]
    winv = weights_inv(ng, prm.a, prm.b)
    M = fov_mask(ng, prm.fov_full)
    P = P.astype(np.float64)
    x = x0.astype(np.complex128).copy()
    xref = xref.astype(np.complex128)
    y = y.astype(np.complex128)
    hist = []
    for n in range(newton_steps):
        alpha = prm.alpha0 * prm.q ** n
        x, res = newton_step(x, xref, y, P, winv, M, alpha, cg_iters, prm.partition)
        hist.append(res)
    return x, hist


def image_from_x(x: np.ndarray, prm: Params | None = None) -> np.ndarray:
    """Frame output: crop_Omega( rho . sqrt(sum_j |c_j|^2) )  (A13). [n, n] complex."""
    prm = prm or Params()
    ng = x.shape[-1]
    winv = weights_inv(ng, prm.a, prm.b)
    c = coils_from_chat(x[1:], winv)
    rss = np.sqrt(np.sum(np.abs(c) ** 2, axis=0))
    img = x[0] * rss
    if prm.fov_full:
        return img
    q = ng // 4
    return img[q:q + ng // 2, q:q + ng // 2]


def coil_partition(ncoils: int, world: int):
    """Contiguous coil blocks, remainder to the low ranks (A10; P:317 uneven distribution).
    Returns [(first, count)] per rank."""
    base, rem = divmod(ncoils, world)
    out, first = [], 0
    for r in range(world):
        cnt = base + (1 if r < rem else 0)
        out.append((first, cnt))
        first += cnt
    return out
