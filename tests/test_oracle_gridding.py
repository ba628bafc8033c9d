"""Pins for the gridding oracle (oracle/gridding.py, reading R20) and for the
radial acquisition it consumes (synth.acquire_radial).

No expected value is produced by the oracle: spokes at theta = 0 and pi/2 sample integer k, where
the non-Cartesian samples must equal the Cartesian centred DFT (an independent FFT route) and
gridding must reproduce it exactly; supports are checked against the R12 mask and hand counts.
"""
import numpy as np

import oracle as O
from oracle import gridding as G
import synth


def test_integer_spokes_grid_to_cartesian_dft():
    # S = 2, T = 1: theta = 0 (row through the centre) and pi/2 (column): every sample sits on an
    # integer cell; the centre cell receives one sample from each spoke (equal values).
    # catches: wrong cell rule (x/y swapped), wrong mean, wrong NUDFT sign/centre
    ng, J = 16, 3
    img = synth.embed(synth.shepp_logan(ng // 2), ng)
    coils = synth.coil_maps(J, ng)
    y_cart = synth.acquire(img, coils, None)
    traj = synth.radial_trajectory(ng, 2, 1, 0)
    raw = synth.acquire_radial(img, coils, traj)
    y, cnt = G.grid_nearest(raw, ng, 2, 1, 0)
    mask = O.radial_mask(ng, 2, 1, 0)
    assert np.array_equal(cnt > 0, mask > 0)
    c = ng // 2
    assert cnt[c, c] == 2 and cnt.sum() == 2 * ng
    assert np.allclose(y[:, mask > 0], y_cart[:, mask > 0], atol=1e-12)
    assert np.all(y[:, mask == 0] == 0)
    # theta = 0 spoke: sample i is cell (c, i); theta = pi/2: cell (i, c)
    assert np.allclose(raw[:, 0, :], y_cart[:, c, :], atol=1e-12)
    assert np.allclose(raw[:, 1, :], y_cart[:, :, c], atol=1e-12)


def test_support_and_counts_match_mask():
    ng, S, T = 32, 8, 1
    cells = G.radial_cells(ng, S, T, 0)
    mask = O.radial_mask(ng, S, T, 0)
    hit = np.zeros(ng * ng, dtype=bool)
    hit[cells[cells >= 0]] = True
    assert np.array_equal(hit.reshape(ng, ng), mask > 0)
    # every spoke passes through the centre: its centre sample (i = ng/2, r = 0) is cell (c, c)
    c = ng // 2
    assert np.all(cells[:, ng // 2] == c * ng + c)


def test_constant_samples_give_constant_grid():
    ng, S, T = 24, 5, 2
    raw = np.full((2, S, ng), 1.5 - 0.25j)
    y, cnt = G.grid_nearest(raw, ng, S, T, 1)
    on = cnt > 0
    assert np.allclose(y[:, on], 1.5 - 0.25j, atol=1e-15)
    assert np.all(y[:, ~on] == 0)


def test_mean_of_duplicates_by_hand():
    # ng = 8, S = 2, T = 1: the centre cell gets sample i = 4 of both spokes -> their mean
    ng = 8
    raw = np.zeros((1, 2, ng), dtype=np.complex128)
    raw[0, 0, 4] = 2.0
    raw[0, 1, 4] = 4.0 + 2.0j
    y, cnt = G.grid_nearest(raw, ng, 2, 1, 0)
    assert cnt[4, 4] == 2 and y[0, 4, 4] == 3.0 + 1.0j


def test_acquire_radial_is_eq1_termwise():
    # tiny case, the definition summed term by term
    ng, J = 8, 1
    rng = np.random.default_rng(0)
    img = np.zeros((ng, ng), dtype=np.complex128)
    img[2:6, 2:6] = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    coils = np.ones((1, ng, ng), dtype=np.complex128)
    traj = synth.radial_trajectory(ng, 3, 1, 0)
    raw = synth.acquire_radial(img, coils, traj)
    c = ng // 2
    for s in range(3):
        for i in range(ng):
            kx, ky = traj[s, i]
            v = 0j
            for yy in range(ng):
                for xx in range(ng):
                    v += img[yy, xx] * np.exp(-2j * np.pi * (kx * (xx - c) + ky * (yy - c)) / ng)
            assert abs(raw[0, s, i] - v / ng) < 1e-12


def test_kb_window_closed_forms():
    # h(0) = 1, symmetric, 0 outside W/2; I0 series against scipy's I0 (an independent routine)
    import scipy.special as sp
    W = 4.0
    b = G.kb_beta(W)
    assert abs(b - np.pi * np.sqrt((W / 2) ** 2 * 1.5 ** 2 - 0.8)) < 1e-15
    for z in (0.0, 0.5, 3.0, 8.99, 15.0):
        assert abs(G._i0(z) - sp.i0(z)) < 1e-12 * sp.i0(z)
    assert G.kb_window(0.0, W, b) == 1.0
    for d in (0.3, 1.1, 1.99):
        assert abs(G.kb_window(d, W, b) - G.kb_window(-d, W, b)) < 1e-15
        assert abs(G.kb_window(d, W, b) - sp.i0(b * np.sqrt(1 - (2 * d / W) ** 2)) / sp.i0(b)) < 1e-12
    assert G.kb_window(2.0001, W, b) == 0.0


def test_grid_kb_constant_samples_and_psf_footprint():
    # constant samples -> weighted mean equals the constant wherever the PSF is positive
    ng, S, T = 24, 3, 1
    raw = np.full((2, S, ng), 0.75 + 0.5j)
    y, psf = G.grid_kb(raw, ng, S, T, 0, width=4.0)
    on = psf > 0
    assert np.allclose(y[:, on], 0.75 + 0.5j, atol=1e-13) and np.all(y[:, ~on] == 0)
    # the theta = 0 spoke's centre sample sits exactly on cell (c, c): with S = 1 the PSF there is
    # the kernel at 0 times itself (1) plus the neighbours' tails along the row
    y1, psf1 = G.grid_kb(np.ones((1, 1, ng)), ng, 1, 1, 0, width=4.0)
    c = ng // 2
    b = G.kb_beta(4.0)
    h1, h2 = G.kb_window(1.0, 4.0, b), G.kb_window(2.0, 4.0, b)   # h(W/2) = 1 / I0(beta), not 0
    row = 1.0 + 2 * h1 + 2 * h2                                       # samples at x = c-2 .. c+2
    assert abs(psf1[c, c] - row) < 1e-13
    assert abs(psf1[c + 1, c] - h1 * row) < 1e-13                     # one row up: h(1) in y
    assert abs(psf1[c + 3, c]) == 0.0                                 # beyond W/2


def test_grid_kb_is_weighted_least_squares_fit():
    # y_g(k) minimises sum_s h(k - k_s) |y - d_s|^2 : check the normal equation at a few cells
    rng = np.random.default_rng(4)
    ng, S, T = 16, 4, 1
    raw = rng.standard_normal((1, S, ng)) + 1j * rng.standard_normal((1, S, ng))
    y, psf = G.grid_kb(raw, ng, S, T, 0, width=3.0)
    b = G.kb_beta(3.0)
    traj = synth.radial_trajectory(ng, S, T, 0)
    c = ng // 2
    for (gy, gx) in ((c, c), (c + 2, c - 1), (c - 3, c + 3)):
        w = np.array([[G.kb_window(gx - (c + traj[s, i, 0]), 3.0, b) * G.kb_window(gy - (c + traj[s, i, 1]), 3.0, b)
                       for i in range(ng)] for s in range(S)])
        if w.sum() == 0:
            continue
        assert abs(w.sum() - psf[gy, gx]) < 1e-12
        assert abs(np.sum(w * (y[0, gy, gx] - raw[0])) ) < 1e-12 * w.sum() * np.abs(raw).max()
