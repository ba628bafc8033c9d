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
