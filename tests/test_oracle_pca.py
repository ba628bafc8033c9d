"""Pins for the PCA channel-compression oracle (oracle/pca.py).

No expected value is produced by the oracle itself: spectra are fixed by construction
(Y = U diag(s) W^H with orthonormal U, W), the covariance by a term-by-term double loop, the
duplicated-channel case by a rank argument.
"""
import numpy as np
import pytest

from oracle import pca as P


def _unitary(rng, n, m=None):
    m = n if m is None else m
    z = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))[None, :]


def test_covariance_matches_termwise_sum():
    # catches: transposed/conjugated operand (C = Y^T conj(Y) or Y^H Y)
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((4, 7)) + 1j * rng.standard_normal((4, 7))
    C = P.pca_covariance(Y)
    for a in range(4):
        for b in range(4):
            s = 0j
            for n in range(7):
                s += Y[a, n] * np.conj(Y[b, n])
            assert abs(C[a, b] - s) < 1e-12
    assert np.allclose(C, C.conj().T)


@pytest.mark.parametrize("J,Jc", [(8, 3), (12, 12), (32, 12)])
def test_fit_recovers_constructed_spectrum(J, Jc):
    # Y = U diag(s) W^H: C = U diag(s^2) U^H exactly, so the eigenvalues are s^2 (descending) and
    # the eigenvectors are U's columns up to a phase (fixed by the sign convention)
    # catches: ascending order, eigenvectors as rows, missing square, wrong phase rule
    rng = np.random.default_rng(J)
    nsamp = 3 * J
    U = _unitary(rng, J)
    W = _unitary(rng, nsamp, J)
    s = np.sort(rng.uniform(0.5, 3.0, J))[::-1] + np.arange(J)[::-1] * 0.3   # distinct, descending
    Y = U @ np.diag(s) @ W.conj().T
    V, w = P.pca_fit(Y, Jc)
    assert np.allclose(w, s ** 2, rtol=1e-12, atol=1e-12)
    for k in range(Jc):
        u = U[:, k]
        m = int(np.argmax(np.abs(u)))
        u = u * np.conj(u[m]) / abs(u[m])
        assert np.allclose(V[:, k], u, atol=1e-10)
        assert abs(V[m, k].imag) < 1e-14 and V[m, k].real > 0
    assert np.allclose(V.conj().T @ V, np.eye(Jc), atol=1e-12)
    assert abs(P.pca_energy(w, Jc) - (s[:Jc] ** 2).sum() / (s ** 2).sum()) < 1e-14


def test_full_rank_keeps_all_energy_and_is_invertible():
    # S:533 "J' = J -> captured energy fraction = 1"; V unitary so V V^H y = y
    rng = np.random.default_rng(1)
    Y = rng.standard_normal((6, 50)) + 1j * rng.standard_normal((6, 50))
    V, w = P.pca_fit(Y, 6)
    Yc = P.pca_apply(V, Y)
    assert abs(P.pca_energy(w, 6) - 1.0) < 1e-15
    assert np.allclose(V @ Yc, Y, atol=1e-12)
    assert abs(np.linalg.norm(Yc) ** 2 / np.linalg.norm(Y) ** 2 - 1.0) < 1e-12


def test_duplicated_channels_compress_to_half():
    # J = 4, two distinct signals duplicated -> J' = 2 captures all energy (rank 2)
    rng = np.random.default_rng(2)
    s1 = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    s2 = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    Y = np.stack([s1, s2, s1, s2])
    V, w = P.pca_fit(Y, 2)
    assert P.pca_energy(w, 2) >= 1 - 1e-12
    Yc = P.pca_apply(V, Y)
    assert abs(np.linalg.norm(Yc) ** 2 / np.linalg.norm(Y) ** 2 - 1.0) < 1e-12
    assert np.allclose(V @ Yc, Y, atol=1e-10)   # the rank-2 data are recovered exactly


def test_energy_monotone_and_matches_projection():
    # S:535 energy non-decreasing in J'; energy(J') = ||V^H y||^2 / ||y||^2
    rng = np.random.default_rng(5)
    Y = rng.standard_normal((8, 40)) + 1j * rng.standard_normal((8, 40))
    prev = 0.0
    for Jc in range(1, 9):
        V, w = P.pca_fit(Y, Jc)
        e = P.pca_energy(w, Jc)
        assert e >= prev - 1e-15
        prev = e
        Yc = P.pca_apply(V, Y)
        assert abs(np.linalg.norm(Yc) ** 2 / np.linalg.norm(Y) ** 2 - e) < 1e-12


def test_sign_convention_tie_takes_first_index():
    V = np.array([[1j], [-1j]]) / np.sqrt(2)    # equal magnitudes: index 0 is made real-positive
    out = P.pca_sign_convention(V)
    assert abs(out[0, 0] - 1 / np.sqrt(2)) < 1e-15 and abs(out[1, 0] + 1 / np.sqrt(2)) < 1e-15


def test_rejects_bad_target_count():
    with pytest.raises(ValueError):
        P.pca_fit(np.ones((3, 4)), 0)
    with pytest.raises(ValueError):
        P.pca_fit(np.ones((3, 4)), 4)
