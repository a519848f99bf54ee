"""Oracle circulant preconditioner (test infrastructure only; see oracle/__init__.py).

M^{-1} = F^H diag{k}^{-1} F  (Eq. precon), k = diag(K) with
k = mu k_c + lam k_d + gamma k_w  (Eq. Kdiag).

Notation: D = unnormalised DFT over the image axes (oracle.fft.fft), D^{-1} its exact
inverse (1/N included); F = D / sqrt(N) is the unitary DFT of reading A1.
"""
from __future__ import annotations

import numpy as np

from .fft import fft, fftn_u, ifftn_u

__all__ = ["dft_n", "idft_n", "k_c_paper", "k_c_direct", "k_d_closed", "k_d_fft",
           "build_k", "apply_Minv", "jacobi_diag"]


def dft_n(x, nd):
    """Unnormalised D over the last nd axes."""
    y = np.asarray(x, dtype=np.complex128)
    for ax in range(-nd, 0):
        y = fft(y, ax)
    return y


def idft_n(x, nd):
    """Exact inverse D^{-1} (with 1/N) over the last nd axes."""
    y = np.asarray(x, dtype=np.complex128)
    n = 1
    for ax in range(-nd, 0):
        y = fft(y, ax, inverse=True)
        n *= y.shape[ax]
    return y / n


def _reverse(x, nd):
    """Index reversal kappa -> -kappa (mod n) on every image axis: the paper's (.)^T on the
    first row of a BCCB matrix (reading A2)."""
    out = x
    for ax in range(-nd, 0):
        n = out.shape[ax]
        out = np.take(out, (-np.arange(n)) % n, axis=ax)
    return out


def k_c_paper(sens, mask):
    """k_c following PAPER.md:199-229 (Eq. d, Eq. diagonalelements, multi-coil form) in the
    paper's order, read per A2:

      1. c_{1;i}: the first row of C_i = F S_i F^H is, as a function of the index offset,
         hat s_i / N with hat s_i = D s_i  (C_i[q, nu] = hat s_i(q - nu) / N; PAPER.md:226,
         Table 1 row 1);
      2. the Hadamard products c^H o c^T summed over coils: g = sum_i |hat s_i|^2 / N^2
         (Eq. d; Table 1 row 2);
      3. the outer transpose (.)^T reverses the index: w(kappa) = g(-kappa);
      4. circular convolution theorem: k_c = D^{-1}{ D{w} o D{r} } (Eq. diagonalelements;
         Table 1 row 3).

    Pinned against diag(F A_dense F^H) (tests/test_oracle_precond.py)."""
    nd = mask.ndim
    n = mask.size
    hat_s = dft_n(sens, nd)                                  # step 1 (per coil)
    g = np.sum(np.abs(hat_s) ** 2, axis=0) / float(n) ** 2   # step 2
    w = _reverse(g, nd)                                      # step 3
    kc = idft_n(dft_n(w, nd) * dft_n(mask.astype(np.float64), nd), nd)  # step 4
    return kc


def k_c_direct(sens, mask):
    """O(N^2) direct evaluation k_c(nu) = sum_q g(q) r(q + nu) with g = sum_c |F s_c|^2 / N
    (the correlation form of reading A2; pins only)."""
    nd = mask.ndim
    n = mask.size
    g = np.sum(np.abs(fftn_u(sens, nd)) ** 2, axis=0) / n
    r = mask.astype(np.float64)
    out = np.zeros(mask.shape)
    for q in np.ndindex(*mask.shape):
        if g[q] == 0.0:
            continue
        out += g[q] * np.roll(r, shift=tuple(-qi for qi in q), axis=tuple(range(nd)))
    return out


def k_d_closed(shape):
    """Eigenvalues of sum_d D_d^H D_d: sum_d 4 sin^2(pi nu_d / n_d) (reading A3; PAPER.md:231
    k_d = F{t_1} evaluated in closed form)."""
    out = np.zeros(shape)
    for d, n in enumerate(shape):
        nu = np.arange(n).reshape([-1 if i == d else 1 for i in range(len(shape))])
        out = out + 4.0 * np.sin(np.pi * nu / n) ** 2
    return out


def k_d_fft(shape):
    """k_d = D{t_1}, t_1 the first row of sum_d D_d^H D_d: 2*nd at the origin,
    -1 at +-1 along each axis (periodic wrap adds up for n = 2)."""
    nd = len(shape)
    t1 = np.zeros(shape)
    t1[(0,) * nd] += 2.0 * nd
    for d, n in enumerate(shape):
        for s in (1, -1):
            idx = [0] * nd
            idx[d] = s % n
            t1[tuple(idx)] -= 1.0
    return dft_n(t1, nd)


def build_k(sens, mask, mu, lam, gamma):
    """k = mu k_c + lam k_d + gamma k_w, k_w = 1.  Returns real k.
    Raises on a singular k."""
    kc = k_c_paper(sens, mask)
    k = mu * kc.real + lam * k_d_closed(mask.shape) + gamma
    if not np.all(np.isfinite(k)) or np.min(np.abs(k)) <= 1e-14:
        raise ZeroDivisionError("singular k")
    return k


def apply_Minv(v, k):
    """M^{-1} v = F^H diag{k}^{-1} F v."""
    nd = k.ndim
    return ifftn_u(fftn_u(v, nd) / k, nd)


def jacobi_diag(sens, mask, mu, lam, gamma):
    """diag(A) = mu f sum_c |s_c|^2 + 2 nd lam + gamma, f = sampled fraction (
    the diagonal of F^H R F is mean(r)).  NEXT-1 comparison preconditioner."""
    nd = mask.ndim
    f = float(np.mean(mask))
    return mu * f * np.sum(np.abs(sens) ** 2, axis=0) + 2.0 * nd * lam + gamma
