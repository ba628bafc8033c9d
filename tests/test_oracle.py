"""Pins for the fp64 oracle (oracle/nlinv_oracle.py) against what the paper and mathematics fix.

Each test names the oracle function it pins and the plausible mistake it would catch.
No expected value here is produced by the oracle itself.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- F_c (reading A1)
def _brute_centred_dft2(z, inverse=False):
    """Definition of the centred unitary DFT, summed term by term (no FFT, no shifts)."""
    ng = z.shape[-1]
    c = ng // 2
    s = 1.0 if inverse else -1.0
    out = np.zeros_like(z, dtype=np.complex128)
    ys = np.arange(ng) - c
    for ky in range(ng):
        for kx in range(ng):
            ph = np.exp(s * 2j * np.pi * ((ky - c) * ys[:, None] + (kx - c) * ys[None, :]) / ng)
            out[..., ky, kx] = np.sum(z * ph, axis=(-2, -1)) / ng
    return out


@pytest.mark.parametrize("ng", [4, 6, 8, 12, 16, 24])
def test_fc_matches_bruteforce_definition(ng):
    # catches: wrong shift direction, wrong normalisation, conjugated kernel
    z = synth.random_complex(7 + ng, (2, ng, ng))
    assert rel(O.fc(z), _brute_centred_dft2(z)) < 1e-12
    assert rel(O.fch(z), _brute_centred_dft2(z, inverse=True)) < 1e-12


@pytest.mark.parametrize("ng", [32, 48, 96, 384])
def test_fc_unitary_and_special_cases(ng):
    z = synth.random_complex(3, (ng, ng))
    # Parseval (unitarity), round trip
    assert abs(np.linalg.norm(O.fc(z)) - np.linalg.norm(z)) / np.linalg.norm(z) < 1e-13
    assert rel(O.fch(O.fc(z)), z) < 1e-13
    # impulse at the grid centre -> constant 1/ng; constant -> centred impulse of height ng
    d = np.zeros((ng, ng), complex)
    d[ng // 2, ng // 2] = 1.0
    assert np.allclose(O.fc(d), 1.0 / ng, atol=1e-15)
    e = O.fc(np.ones((ng, ng), complex))
    assert abs(e[ng // 2, ng // 2] - ng) < 1e-10
    e[ng // 2, ng // 2] = 0
    assert np.abs(e).max() < 1e-10


def test_fc_shift_theorem():
    # a one-pixel shift in image space multiplies k-space by exp(-2 pi i k/ng), k centred
    ng = 16
    z = synth.random_complex(11, (ng, ng))
    zs = np.roll(z, 1, axis=1)
    k = np.arange(ng) - ng // 2
    assert rel(O.fc(zs), O.fc(z) * np.exp(-2j * np.pi * k[None, :] / ng)) < 1e-12


# ---------------------------------------------------------------- masks and weights
def test_fov_mask():
    for ng in (16, 32, 384):
        M = O.fov_mask(ng)
        assert M.sum() == (ng // 2) ** 2
        assert M[ng // 4, ng // 4] == 1 and M[ng // 4 - 1, ng // 4] == 0
        assert M[3 * ng // 4 - 1, 3 * ng // 4 - 1] == 1 and M[3 * ng // 4, ng // 2] == 0
        assert np.array_equal(M * M, M)
    assert O.fov_mask(16, fov_full=True).sum() == 256


def test_weights_closed_form():
    ng = 32
    w = O.weights_inv(ng, 220.0, 32.0)
    assert w[16, 16] == 1.0                                   # k = 0
    assert math.isclose(w[0, 0], (1 + 220 * 0.5) ** -16, rel_tol=1e-14)   # corner k=(-1/2,-1/2)
    assert math.isclose(w[16, 20], (1 + 220 * (4 / 32) ** 2) ** -16, rel_tol=1e-14)
    assert np.all(O.weights_inv(ng, 0.0, 32.0) == 1.0)       # a = 0 -> W^{-1} = plain F^H
    assert w.min() > 1e-34 and w.max() == 1.0


def test_coils_from_dc_chat_is_constant():
    # chat = delta at k = 0 -> c = constant 1/ng (w(0) = 1, unitary centred transform)
    ng = 16
    chat = np.zeros((1, ng, ng), complex)
    chat[0, ng // 2, ng // 2] = 1.0
    c = O.coils_from_chat(chat, O.weights_inv(ng))
    assert np.allclose(c, 1.0 / ng, atol=1e-15)


def test_round_snapped_tie_rule():
    # half away from zero after the 2^-20 snap (A12)
    assert O.nlinv_oracle._round_snapped(0.5) == 1
    assert O.nlinv_oracle._round_snapped(-0.5) == -1
    assert O.nlinv_oracle._round_snapped(2.5) == 3
    assert O.nlinv_oracle._round_snapped(-2.5) == -3
    assert O.nlinv_oracle._round_snapped(0.4999) == 0
    assert O.nlinv_oracle._round_snapped(3 * math.cos(math.pi / 3)) == 2   # 1.5000000000000004
    assert O.nlinv_oracle._round_snapped(-3 * math.cos(math.pi / 3)) == -2


def test_radial_mask_special_angles():
    ng = 32
    # one spoke at theta = 0: the full centre row
    m = O.radial_mask(ng, 1, 1, 0)
    exp = np.zeros((ng, ng), np.uint8)
    exp[ng // 2, :] = 1
    assert np.array_equal(m, exp)
    # two spokes at 0 and pi/2: centre row + centre column
    m = O.radial_mask(ng, 2, 1, 0)
    exp[:, ng // 2] = 1
    assert np.array_equal(m, exp)
    assert m.sum() == 2 * ng - 1
    # turns: frame f uses angles offset by f/T of the spoke spacing -> frame 1 of T=2 with S=1
    # is theta = pi/2, the centre column
    m = O.radial_mask(ng, 1, 2, 1)
    col = np.zeros((ng, ng), np.uint8)
    col[:, ng // 2] = 1
    assert np.array_equal(m, col)


def test_radial_mask_against_rational_geometry():
    # theta = pi/4: r cos = r sin = r/sqrt2; a sample is on cell (c + round(r/sqrt2)) for both axes
    ng = 32
    m = O.radial_mask(ng, 4, 1, 0)                 # 0, pi/4, pi/2, 3pi/4
    c = ng // 2
    for i in range(ng):
        r = i - c
        v = abs(r) / math.sqrt(2)
        k = int(math.floor(v + 0.5)) * (1 if r >= 0 else -1)
        assert m[c + k, c + k] == 1
        assert m[c + k, c - k] == 1 if 0 <= c - k < ng else True
    # every set cell lies on one of the 4 lines to within half a cell
    ky, kx = np.nonzero(m)
    dy, dx = ky - c, kx - c
    on = (np.abs(dy) == 0) | (np.abs(dx) == 0) | (np.abs(np.abs(dy) - np.abs(dx)) <= 1)
    assert on.all()


def test_radial_mask_paper_workload_density():
    # C1 and C2 shapes; radial sampling gives a few % of the grid at C2
    m1 = O.radial_mask(32, 8, 1, 0)
    assert 150 < m1.sum() < 300
    for f in range(5):
        m = O.radial_mask(384, 15, 5, f)
        assert 0.03 < m.mean() < 0.045
        assert m[192, 192] == 1
        assert O.radial_margin(384, 15, 5, f) > 1e-6


# ---------------------------------------------------------------- operators
def _problem(ng=16, J=3, seed=1, fov_full=False, mask_density=True):
    x = synth.random_complex(seed, (J + 1, ng, ng))
    dx = synth.random_complex(seed + 100, (J + 1, ng, ng))
    dy = synth.random_complex(seed + 200, (J, ng, ng))
    P = O.radial_mask(ng, 6, 1, 0).astype(float)
    winv = O.weights_inv(ng, 2.0, 4.0)   # mild weights so every term has weight in the checks
    M = O.fov_mask(ng, fov_full)
    return x, dx, P * dy, P, winv, M


def test_adjoint_identity():
    # <DF dx, dy> = <dx, DF^H dy> -- catches a missing conj, a wrong mask or weight placement
    for seed in range(4):
        x, dx, dy, P, winv, M = _problem(seed=seed)
        lhs = O.inner(O.derivative(x, dx, P, winv, M), dy)
        rhs = O.inner(dx, O.adjoint(x, dy, P, winv, M))
        assert abs(lhs - rhs) / (np.linalg.norm(dx) * np.linalg.norm(dy)) < 1e-13


def test_adjoint_dense_matrix():
    # build DF column by column at ng=8, J=2 and compare DF^H with the conjugate transpose
    ng, J = 8, 2
    x, _, _, P, winv, M = _problem(ng=ng, J=J, seed=5)
    n_in, n_out = (J + 1) * ng * ng, J * ng * ng
    A = np.zeros((n_out, n_in), complex)
    for i in range(n_in):
        e = np.zeros(n_in, complex)
        e[i] = 1.0
        A[:, i] = O.derivative(x, e.reshape(J + 1, ng, ng), P, winv, M).ravel()
    B = np.zeros((n_in, n_out), complex)
    for i in range(n_out):
        e = np.zeros(n_out, complex)
        e[i] = 1.0
        B[:, i] = O.adjoint(x, e.reshape(J, ng, ng), P, winv, M).ravel()
    assert np.abs(B - A.conj().T).max() < 1e-13


def test_forward_bilinear_expansion():
    # F(x + e dx) = F(x) + e DF dx + e^2 P F_c(M drho W^{-1} dchat) exactly (C is bilinear)
    x, dx, _, P, winv, M = _problem(seed=9)
    for eps in (1e-3, 0.5, 2.0):
        lhs = O.forward(x + eps * dx, P, winv, M)
        second = P * O.fc(M * dx[0] * O.coils_from_chat(dx[1:], winv))
        rhs = O.forward(x, P, winv, M) + eps * O.derivative(x, dx, P, winv, M) + eps ** 2 * second
        assert rel(lhs, rhs) < 1e-13


def test_forward_respects_masks():
    x, _, _, P, winv, M = _problem(seed=2)
    y = O.forward(x, P, winv, M)
    assert np.all(y[:, P == 0] == 0)                          # P_k projection
    x2 = x.copy()
    x2[0, M == 0] = 123.0                                     # change rho outside Omega
    assert np.array_equal(O.forward(x2, P, winv, M), y)       # M_Omega restriction
    assert np.all(O.forward(x * np.array([0, 1, 1, 1])[:, None, None], P, winv, M) == 0)  # rho=0 -> 0


def test_normal_hermitian_positive():
    x, dx, _, P, winv, M = _problem(seed=4)
    dx2 = synth.random_complex(77, dx.shape)
    alpha = 0.37
    a = O.inner(O.normal(x, alpha, dx, P, winv, M), dx2)
    b = O.inner(dx, O.normal(x, alpha, dx2, P, winv, M))
    assert abs(a - b) / (np.linalg.norm(dx) * np.linalg.norm(dx2)) < 1e-13
    q = O.inner(dx, O.normal(x, alpha, dx, P, winv, M))
    assert abs(q.imag) < 1e-12 * abs(q) and q.real >= alpha * np.linalg.norm(dx) ** 2 * (1 - 1e-13)


def test_table1_operator_counts():
    gold = json.load(open(os.path.join(GOLDEN, "table1_opcounts.json")))
    x, dx, dy, P, winv, M = _problem(seed=3)
    C = O.nlinv_oracle.COUNTERS
    for name, fn in (("F", lambda: O.forward(x, P, winv, M)),
                     ("DF", lambda: O.derivative(x, dx, P, winv, M)),
                     ("DFH", lambda: O.adjoint(x, dy, P, winv, M))):
        C.reset()
        fn()
        assert (C.fft, C.chan_sum, C.allreduce) == (gold[name]["fft"], gold[name]["chan_sum"],
                                                   gold[name]["allreduce"]), name


def test_partition_invariance():
    # channel decomposition rho = sum_g rho_g: same result for any contiguous split
    x, dx, dy, P, winv, M = _problem(ng=16, J=7, seed=8)
    ref = O.adjoint(x, dy, P, winv, M)
    for world in (2, 3, 4, 7):
        part = [c for _, c in O.coil_partition(7, world)]
        assert rel(O.adjoint(x, dy, P, winv, M, part), ref) < 1e-14


def test_coil_partition_rule():
    assert O.coil_partition(12, 8) == [(0, 2), (2, 2), (4, 2), (6, 2), (8, 1), (9, 1), (10, 1), (11, 1)]
    assert O.coil_partition(12, 1) == [(0, 12)]
    assert O.coil_partition(10, 4) == [(0, 3), (3, 3), (6, 2), (8, 2)]


# ---------------------------------------------------------------- CG
def _spd(n, seed, alpha=0.1):
    A = synth.random_complex(seed, (n, n))
    return A.conj().T @ A + alpha * np.eye(n)


def test_cg_is_krylov_a_norm_minimiser():
    # the L-th CG iterate minimises ||x - x*||_A over K_L(A, b): solve that projected problem
    n = 12
    A = _spd(n, 21)
    b = synth.random_complex(22, (n,))
    for L in (1, 3, 6):
        K = np.stack([np.linalg.matrix_power(A, i) @ b for i in range(L)], axis=1)
        V, _ = np.linalg.qr(K)
        xk = V @ np.linalg.solve(V.conj().T @ A @ V, V.conj().T @ b)
        xc = O.cg(lambda v: A @ v, b, L)
        assert rel(xc, xk) < 1e-10


def test_cg_dense_solve_and_special_cases():
    for seed in range(20):
        n = 4 + seed % 12
        A = _spd(n, 300 + seed, alpha=1.0)
        b = synth.random_complex(400 + seed, (n,))
        assert rel(O.cg(lambda v: A @ v, b, 3 * n), np.linalg.solve(A, b)) < 1e-9
    b = synth.random_complex(5, (9,))
    assert rel(O.cg(lambda v: 2.5 * v, b, 1), b / 2.5) < 1e-15         # alpha I in one iteration
    assert np.all(O.cg(lambda v: 2.5 * v, np.zeros(4, complex), 5) == 0)  # rhs 0 -> breakdown -> 0


# ---------------------------------------------------------------- IRGNM
def test_newton_closed_form_diagonal_case():
    # fov_full, P = 1, J = 1, x0 = x_ref = (1, 0): DF restricted to chat is diag(w^{-1}), the rho
    # block sees sum conj(c) u = 0, so the converged step is dchat = w^{-1} y / (w^{-2} + alpha),
    # drho = 0 (derived from Eq. 3 with these substitutions).
    ng = 8
    prm = O.Params(a=3.0, b=2.0, fov_full=True)
    winv = O.weights_inv(ng, prm.a, prm.b)
    y = synth.random_complex(31, (1, ng, ng))
    P = np.ones((ng, ng))
    x0 = O.initial_x(1, ng)
    x1, _ = O.irgnm(y, P, x0, x0, 1, 60, prm)
    exp = winv * y[0] / (winv ** 2 + prm.alpha0)
    assert rel(x1[1], exp) < 1e-10
    assert np.all(x1[0] == 1.0)


def test_newton_step0_keeps_rho_bitexact():
    ng, J = 16, 4
    _, coils, y = synth.frame_inputs(J, ng)
    P = O.radial_mask(ng, 6, 1, 0)
    x0 = O.initial_x(J, ng)
    x1, _ = O.irgnm(y, P, x0, x0, 1, 5)
    assert np.all(x1[0] == 1.0)
    assert np.linalg.norm(x1[1:]) > 0


def test_fixed_point():
    ng, J = 16, 3
    x, _, _, P, winv, M = _problem(ng=ng, J=J, seed=12)
    prm = O.Params(a=2.0, b=4.0)
    y = O.forward(x, P, winv, M)
    x1, hist = O.irgnm(y, P, x, x, 1, 5, prm)
    assert np.array_equal(x1, x) and hist[0] == 0.0


@pytest.mark.slow
def test_reconstruction_quality_c1():
    # C1: 8 coils, 32^2, 8 spokes. NLINV beats zero-filled RSS and the residual decreases
    ng, J = 32, 8
    img, coils, y = synth.frame_inputs(J, ng)
    P = O.radial_mask(ng, 8, 1, 0)
    x0 = O.initial_x(J, ng)
    x, hist = O.irgnm(y, P, x0, x0, 6, 20)
    assert all(hist[i + 1] <= hist[i] * (1 + 1e-12) for i in range(len(hist) - 1))
    rec = O.image_from_x(x)
    q = ng // 4
    zf = O.fch(P * y)[:, q:q + ng // 2, q:q + ng // 2]
    zf = np.sqrt(np.sum(np.abs(zf) ** 2, axis=0))

    def err(a):
        a = np.abs(a)
        s = np.vdot(a.ravel(), img.ravel()).real / np.vdot(a.ravel(), a.ravel()).real
        return np.linalg.norm(s * a - img) / np.linalg.norm(img)

    assert err(rec) < err(zf)


# ---------------------------------------------------------------- frame output image_from_x (A13 / R13)
# image = crop_Omega( rho . sqrt(sum_j |c_j|^2) ), c_j = F_c^H (w^-1 chat_j). Three pins that do not
# reuse the oracle's own formula: a closed form, a marker pixel (crop geometry) and a term-by-term sum.
def test_image_from_x_dc_closed_form():
    # chat_j = a_j delta_DC  =>  c_j == a_j w^-1(0) / ng = a_j / ng  (w^-1(DC) = 1, unitary F_c), so
    # image == crop(rho) * sqrt(sum_j |a_j|^2) / ng exactly. Catches: missing sqrt (sum |a|^2 / ng^2),
    # rho only (no RSS factor), sum |c_j| instead of RSS (sum |a_j| / ng), conj / |rho| instead of rho.
    ng, J = 16, 3
    a = np.array([3.0 + 4.0j, -1.0 + 2.0j, 0.5 - 2.5j])
    x = np.zeros((J + 1, ng, ng), complex)
    x[0] = synth.random_complex(41, (ng, ng))
    for j in range(J):
        x[1 + j, ng // 2, ng // 2] = a[j]
    q, n = ng // 4, ng // 2
    want = x[0, q:q + n, q:q + n] * math.sqrt(sum(abs(v) ** 2 for v in a)) / ng
    got = O.image_from_x(x)
    assert got.shape == (n, n)
    assert rel(got, want) < 1e-13


def test_image_from_x_crop_marker():
    # a single marker pixel of rho at (ng/4, ng/4) (the first Omega pixel) lands at image[0, 0];
    # catches an off-by-one / transposed crop. RSS is made constant by DC-only coils.
    ng, J = 16, 2
    x = np.zeros((J + 1, ng, ng), complex)
    x[0, ng // 4, ng // 4] = 2.0 - 1.0j
    x[0, ng // 4 + 1, ng // 4 + 3] = 0.25j    # second marker: row 1, column 3 of the image
    x[1, ng // 2, ng // 2] = 1.0
    x[2, ng // 2, ng // 2] = 1.0j
    got = O.image_from_x(x)
    want = np.zeros((ng // 2, ng // 2), complex)
    want[0, 0] = (2.0 - 1.0j) * math.sqrt(2.0) / ng
    want[1, 3] = 0.25j * math.sqrt(2.0) / ng
    assert np.allclose(got, want, rtol=0, atol=1e-15)


def test_image_from_x_term_by_term():
    # ng = 8, J = 2: c_j summed term by term from the centred DFT definition and the w^-1 closed form,
    # then rho * sqrt(|c_1|^2 + |c_2|^2) pixel by pixel over the Omega crop
    ng, J = 8, 2
    x = synth.random_complex(43, (J + 1, ng, ng))
    c0 = ng // 2
    a_s, b_s = 220.0, 32.0
    want = np.zeros((ng // 2, ng // 2), complex)
    for yy in range(ng // 4, 3 * ng // 4):
        for xx in range(ng // 4, 3 * ng // 4):
            ss = 0.0
            for j in range(J):
                cj = 0.0 + 0.0j
                for ky in range(ng):
                    for kx in range(ng):
                        kk = ((ky - c0) ** 2 + (kx - c0) ** 2) / ng ** 2
                        w = (1.0 + a_s * kk) ** (-b_s / 2.0)
                        cj += w * x[1 + j, ky, kx] * np.exp(2j * np.pi * ((ky - c0) * (yy - c0) + (kx - c0) * (xx - c0)) / ng)
                cj /= ng
                ss += abs(cj) ** 2
            want[yy - ng // 4, xx - ng // 4] = x[0, yy, xx] * math.sqrt(ss)
    assert rel(O.image_from_x(x), want) < 1e-12


@pytest.mark.parametrize("kind", ["no_sqrt", "rho_only", "sum_abs", "crop_off_by_one", "conj_rho"])
def test_image_pins_catch_mutations(kind, monkeypatch):
    # meta-check of the three pins above: each plausible mistake in image_from_x fails at least one
    import oracle.nlinv_oracle as ON

    def mutant(x, prm=None):
        ng = x.shape[-1]
        c = ON.coils_from_chat(x[1:], ON.weights_inv(ng))
        p2 = np.sum(np.abs(c) ** 2, axis=0)
        rss = {"no_sqrt": p2, "rho_only": 1.0, "sum_abs": np.sum(np.abs(c), axis=0)}.get(kind, np.sqrt(p2))
        img = (np.conj(x[0]) if kind == "conj_rho" else x[0]) * rss
        q = ng // 4 + (1 if kind == "crop_off_by_one" else 0)
        return img[q:q + ng // 2, q:q + ng // 2]

    monkeypatch.setattr(O, "image_from_x", mutant)
    caught = 0
    for pin in (test_image_from_x_dc_closed_form, test_image_from_x_crop_marker, test_image_from_x_term_by_term):
        try:
            pin()
        except AssertionError:
            caught += 1
    assert caught >= 1


def test_workers_bit_identical():
    # the coil-parallel timing mode (set_workers) runs the same per-channel library call on host
    # threads: a Newton step must be bit-identical to the serial oracle
    ng, J = 32, 4
    x, _, y, P, winv, M = _problem(ng=ng, J=J, seed=5)
    ref = O.newton_step(x, x, y, P, winv, M, 1.0, 4)
    O.set_workers(4)
    try:
        par = O.newton_step(x, x, y, P, winv, M, 1.0, 4)
    finally:
        O.set_workers(1)
    assert np.array_equal(ref[0], par[0]) and ref[1] == par[1]
