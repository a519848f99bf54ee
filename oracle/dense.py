"""Dense brute-force matrices built from the DEFINITIONS (test infrastructure only; pins).

Independent of oracle.fft / oracle.ops: the DFT matrix is built from explicit exponentials,
D_x / D_y from the difference definition, the Haar matrix from the
two-tap analysis rows, S and R as diagonal matrices.  Vectors are image arrays raveled in
C order (d0 slowest).  Sizes are kept at N <= 4096.
"""
from __future__ import annotations

import numpy as np

__all__ = ["dft_unitary", "diff_matrix", "haar_matrix", "system_matrix", "dense_from_op"]


def _dft1(n):
    k = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(k, k) / n) / np.sqrt(n)


def dft_unitary(shape):
    """Dense unitary F = F_{d0} kron F_{d1} [kron F_{d2}] (C-order raveling)."""
    F = np.ones((1, 1), dtype=np.complex128)
    for n in shape:
        F = np.kron(F, _dft1(n))
    return F


def _eye_kron(mats):
    out = np.ones((1, 1))
    for m in mats:
        out = np.kron(out, m)
    return out


def diff_matrix(shape, axis):
    """D_axis with (D x)_i = x_i - x_{i-1 mod n} along `axis`."""
    n = shape[axis]
    d1 = np.eye(n)
    for i in range(n):
        d1[i, (i - 1) % n] -= 1.0
    return _eye_kron([d1 if a == axis else np.eye(s) for a, s in enumerate(shape)])


def _haar1(n):
    """1D orthonormal Haar analysis matrix: rows 0..n/2-1 (e_{2k} + e_{2k+1})/sqrt2, rows
    n/2.. (e_{2k} - e_{2k+1})/sqrt2."""
    h = np.zeros((n, n))
    for k in range(n // 2):
        h[k, 2 * k] = h[k, 2 * k + 1] = 1 / np.sqrt(2)
        h[n // 2 + k, 2 * k] = 1 / np.sqrt(2)
        h[n // 2 + k, 2 * k + 1] = -1 / np.sqrt(2)
    return h


def haar_matrix(shape, levels):
    """Dense Mallat-pyramid Haar W: level l applies kron(haar1) on the leading
    (shape >> l) block and identity elsewhere."""
    N = int(np.prod(shape))
    W = np.eye(N)
    for lvl in range(levels):
        sub = [s >> lvl for s in shape]
        Hs = _eye_kron([_haar1(s) for s in sub])
        # embed: indices of the leading block within the full C-order raveling
        idx = np.ravel_multi_index(np.meshgrid(*[np.arange(s) for s in sub], indexing="ij"),
                                   shape).ravel()
        L = np.eye(N)
        L[np.ix_(idx, idx)] = Hs
        W = L @ W
    return W


def system_matrix(sens, mask, mu, lam, gamma):
    """A = mu sum_c (R F S_c)^H R F S_c + lam sum_d D_d^H D_d + gamma I (PAPER.md:127-129,
    W^H W = I), assembled from dense factors."""
    shape = mask.shape
    N = mask.size
    F = dft_unitary(shape)
    R = np.diag(mask.ravel().astype(np.float64))
    A = np.zeros((N, N), dtype=np.complex128)
    for s in sens:
        E = R @ F @ np.diag(s.ravel())
        A += mu * (E.conj().T @ E)
    for ax in range(len(shape)):
        D = diff_matrix(shape, ax)
        A += lam * (D.T @ D)
    A += gamma * np.eye(N)
    return A


def dense_from_op(op, shape):
    """Column j = op(e_j)."""
    N = int(np.prod(shape))
    M = np.zeros((N, N), dtype=np.complex128)
    for j in range(N):
        e = np.zeros(N, dtype=np.complex128)
        e[j] = 1.0
        M[:, j] = np.asarray(op(e.reshape(shape))).ravel()
    return M
