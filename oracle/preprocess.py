"""Oracle data preprocessing of PAPER.md Methods (test infrastructure only; see
oracle/__init__.py): sensitivity / coil-image normalisation with support masking
 and SVD coil compression (after Huang et al. 2008).
SURVEY.md 8(f) NEXT-3 and NEXT-4.

Coil stacks are [C, *image] complex128; `support` is a 0/1 array over the image.
"""
from __future__ import annotations

import numpy as np

__all__ = ["normalize_sens", "normalize_coil_images", "compression_matrix", "compress"]


def normalize_sens(sens, support=None):
    """S_hat_i = [sum_j S_j^H S_j]^{-1/2} S_i  (pixelwise: the S_j are
    diagonal), "given zero intensity outside the subject": S_hat = 0 where
    support == 0 or sum_j |S_j|^2 == 0."""
    s = np.asarray(sens, dtype=np.complex128)
    rss2 = np.sum(np.abs(s) ** 2, axis=0)
    keep = rss2 > 0
    if support is not None:
        keep = keep & (np.asarray(support) != 0)
    scale = np.where(keep, 1.0 / np.sqrt(np.where(rss2 > 0, rss2, 1.0)), 0.0)
    return s * scale[None]


def normalize_coil_images(m, sens_hat):
    """m_i <- S_hat_i sum_j S_hat_j^H m_j: the coil images are projected on
    the span of the normalised maps, so that the data model m_i = S_hat_i x is consistent."""
    m = np.asarray(m, dtype=np.complex128)
    x = np.sum(np.conj(sens_hat) * m, axis=0)
    return sens_hat * x[None]


def compression_matrix(data, c_out):
    """Huang et al. 2008: eigen-decomposition of the coil covariance
    G = sum_n d(n) d(n)^H over all samples n of the coil data d (images or k-space: the two
    give the same G under the unitary F), eigenvalues in decreasing order; the compression
    matrix keeps the c_out dominant eigenvectors: A = U[:, :c_out]^H (c_out x C).
    Returns (A, eigenvalues descending)."""
    d = np.asarray(data, dtype=np.complex128).reshape(data.shape[0], -1)
    G = d @ d.conj().T
    w, U = np.linalg.eigh(G)            # library primitive (ascending)
    order = np.argsort(w)[::-1]
    w, U = w[order], U[:, order]
    return U[:, :c_out].conj().T, w


def compress(stack, A):
    """Virtual coils: out_k = sum_c A[k, c] stack_c (pixelwise; "multiplied by the
    ... coil images and the coil sensitivity maps")."""
    s = np.asarray(stack, dtype=np.complex128)
    return np.tensordot(A, s, axes=(1, 0))
