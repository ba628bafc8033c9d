"""fp64 CPU oracle of PCA channel compression -- TEST INFRASTRUCTURE ONLY.

PAPER.md P:241 (§3.2): "A principal component analysis preprocessing step is applied before
reconstruction to compress the 32 channels to 8-12" [Huang 2007]. SPEC.md S:528-535
(compress_channels): form the J x J channel covariance from the data samples, eigendecompose,
project onto the top-J' eigenvectors in descending eigenvalue order, with the deterministic sign
convention "largest-magnitude component real-positive". SURVEY.md §8(f) row f3.

Definitions (samples y_j[n], j = 1..J channels, n over the sampled k-space points):
  C[a, b]   = sum_n y_a[n] conj(y_b[n])                 (Hermitian, positive semidefinite)
  C v_k     = lambda_k v_k,  lambda_1 >= ... >= lambda_J (orthonormal v_k)
  v_k       <- v_k * conj(v_k[m]) / |v_k[m]|, m = argmax_j |v_k[j]| (first index on ties)
  y'_k[n]   = sum_j conj(v_k[j]) y_j[n],  k = 1..J'      (y' = V^H y, V = [v_1 .. v_J'])
  energy(J') = sum_{k <= J'} lambda_k / sum_k lambda_k  (= ||y'||^2 / ||y||^2)

Plain numpy; ``numpy.linalg.eigh`` is the eigensolver step (a library primitive). Pinned by
``tests/test_oracle_pca.py`` (closed-form spectra, brute-force covariance, rank arguments).
Shares nothing with the CUDA path.
"""
from __future__ import annotations

import numpy as np

__all__ = ["pca_covariance", "pca_fit", "pca_apply", "pca_energy", "pca_sign_convention"]


def pca_covariance(Y: np.ndarray) -> np.ndarray:
    """C = Y Y^H over all samples (Y: [J, nsamp] complex). S:531 "J x J channel covariance"."""
    Y = np.asarray(Y, dtype=np.complex128).reshape(Y.shape[0], -1)
    return Y @ Y.conj().T


def pca_sign_convention(V: np.ndarray) -> np.ndarray:
    """Each column scaled by a unit phase so that its largest-magnitude component (first index
    on ties) is real and positive."""
    V = np.array(V, dtype=np.complex128, copy=True)
    for k in range(V.shape[1]):
        m = int(np.argmax(np.abs(V[:, k])))
        a = V[m, k]
        if a != 0:
            V[:, k] *= np.conj(a) / abs(a)
    return V


def pca_fit(Y: np.ndarray, Jc: int):
    """Compression matrix V [J, Jc] (top-Jc eigenvectors of C, descending) and all eigenvalues
    (descending). S:529-531."""
    J = Y.shape[0]
    if not 1 <= Jc <= J:
        raise ValueError("need 1 <= J' <= J (S:530)")
    C = pca_covariance(Y)
    w, U = np.linalg.eigh(C)          # ascending
    order = np.argsort(-w, kind="stable")
    w, U = w[order], U[:, order]
    return pca_sign_convention(U[:, :Jc]), w


def pca_apply(V: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """y' = V^H y, channel by channel over every sample (any trailing shape)."""
    Y = np.asarray(Y, dtype=np.complex128)
    flat = Y.reshape(Y.shape[0], -1)
    out = V.conj().T @ flat
    return out.reshape((V.shape[1],) + Y.shape[1:])


def pca_energy(w: np.ndarray, Jc: int) -> float:
    """Captured energy fraction of the top Jc components."""
    w = np.clip(np.asarray(w, dtype=np.float64), 0.0, None)
    tot = w.sum()
    return float(w[:Jc].sum() / tot) if tot > 0 else 1.0
