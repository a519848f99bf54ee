"""Oracle operators (test infrastructure only; see oracle/__init__.py).

All images are complex128 arrays whose LAST `nd` axes are the image axes (nd = 2 or 3,
d0 first).  Coil stacks are [C, *image].  The mask r is a 0/1 array over the k-space grid.
"""
from __future__ import annotations

import numpy as np

from .fft import fftn_u, ifftn_u

__all__ = ["encode", "encode_adj", "data_normal", "diff", "diff_adj", "tv_normal",
           "haar_fwd", "haar_inv", "d4_fwd", "d4_inv", "wavelet_fwd", "wavelet_inv", "D4_H",
           "apply_A", "shrink", "rss_init"]


def encode(x, sens, mask):
    """E_c x = R F S_c x for every coil (Eq. ill0). Returns [C, *image]."""
    nd = x.ndim
    return mask * fftn_u(sens * x[None], nd)


def encode_adj(y, sens, mask):
    """sum_c S_c^H F^H R^H y_c (Alg. 1 step 4 first term; R^H = R)."""
    nd = y.ndim - 1
    return np.sum(np.conj(sens) * ifftn_u(mask * y, nd), axis=0)


def data_normal(x, sens, mask):
    """sum_c (R F S_c)^H R F S_c x  (first term of A)."""
    return encode_adj(encode(x, sens, mask), sens, mask)


def diff(x, axis, nd=None):
    """Periodic first difference (D_d x)_i = x_i - x_{i-1}, wrap at i = 0.
    `axis` counts image axes (0 = d0, the paper's i index); image axes are the last `nd`."""
    nd = x.ndim if nd is None else nd
    return x - np.roll(x, 1, axis=x.ndim - nd + axis)


def diff_adj(v, axis, nd=None):
    """Exact adjoint of `diff`: (D_d^H v)_i = v_i - v_{i+1} (transpose of the circulant)."""
    nd = v.ndim if nd is None else nd
    return v - np.roll(v, -1, axis=v.ndim - nd + axis)


def tv_normal(x, nd=None):
    """sum_d D_d^H D_d x (PAPER.md:128 second term; 2D: D_x^H D_x + D_y^H D_y)."""
    nd = x.ndim if nd is None else nd
    return sum(diff_adj(diff(x, d, nd), d, nd) for d in range(nd))


def _haar_axis_fwd(block, ax):
    """One orthonormal Haar analysis step along axis `ax` of `block`:
    a_k = (x_{2k} + x_{2k+1})/sqrt2 (stored first), d_k = (x_{2k} - x_{2k+1})/sqrt2."""
    ev = np.take(block, np.arange(0, block.shape[ax], 2), axis=ax)
    od = np.take(block, np.arange(1, block.shape[ax], 2), axis=ax)
    return np.concatenate(((ev + od) / np.sqrt(2.0), (ev - od) / np.sqrt(2.0)), axis=ax)


def _haar_axis_inv(block, ax):
    h = block.shape[ax] // 2
    a = np.take(block, np.arange(0, h), axis=ax)
    d = np.take(block, np.arange(h, 2 * h), axis=ax)
    ev = (a + d) / np.sqrt(2.0)
    od = (a - d) / np.sqrt(2.0)
    out = np.empty_like(block)
    idx_e = [slice(None)] * block.ndim
    idx_o = [slice(None)] * block.ndim
    idx_e[ax] = slice(0, 2 * h, 2)
    idx_o[ax] = slice(1, 2 * h, 2)
    out[tuple(idx_e)] = ev
    out[tuple(idx_o)] = od
    return out


def haar_fwd(x, levels, nd=None):
    """L-level orthonormal Haar W, Mallat pyramid (reading A6; the unitary W of PAPER.md:117).
    Each level transforms the current approximation block (leading 1/2^l corner) along every
    image axis in order d0, d1[, d2]."""
    nd = x.ndim if nd is None else nd
    shape = x.shape[-nd:]
    for s in shape:
        if s % (1 << levels):
            raise ValueError("image size not divisible by 2^levels")
    out = np.array(x, dtype=np.complex128, copy=True)
    lead = out.ndim - nd
    for lvl in range(levels):
        sl = tuple([slice(None)] * lead + [slice(0, s >> lvl) for s in shape])
        blk = out[sl]
        for d in range(nd):
            blk = _haar_axis_fwd(blk, lead + d)
        out[sl] = blk
    return out


def haar_inv(c, levels, nd=None):
    """W^H = W^{-1}: undo the levels from coarsest to finest (W^H W = I)."""
    nd = c.ndim if nd is None else nd
    shape = c.shape[-nd:]
    out = np.array(c, dtype=np.complex128, copy=True)
    lead = out.ndim - nd
    for lvl in reversed(range(levels)):
        sl = tuple([slice(None)] * lead + [slice(0, s >> lvl) for s in shape])
        blk = out[sl]
        for d in reversed(range(nd)):
            blk = _haar_axis_inv(blk, lead + d)
        out[sl] = blk
    return out


# Daubechies 4-tap scaling filter ("Daubechies 4"; reading A32: the 4-coefficient
# orthonormal wavelet D4), h = [1+r3, 3+r3, 3-r3, 1-r3] / (4 sqrt2); wavelet g_m = (-1)^m h_{3-m}.
_R3 = np.sqrt(3.0)
D4_H = np.array([1 + _R3, 3 + _R3, 3 - _R3, 1 - _R3]) / (4 * np.sqrt(2.0))
D4_G = np.array([D4_H[3], -D4_H[2], D4_H[1], -D4_H[0]])


def _d4_axis_fwd(block, ax):
    """One periodized D4 analysis step along axis `ax`: a_k = sum_m h_m x_{(2k+m) mod n},
    d_k = sum_m g_m x_{(2k+m) mod n}; approximation first (Mallat)."""
    n = block.shape[ax]
    k = np.arange(n // 2)
    a = sum(D4_H[m] * np.take(block, (2 * k + m) % n, axis=ax) for m in range(4))
    d = sum(D4_G[m] * np.take(block, (2 * k + m) % n, axis=ax) for m in range(4))
    return np.concatenate((a, d), axis=ax)


def _d4_axis_inv(block, ax):
    """Synthesis = transpose of the analysis (orthonormal): x_j = sum_k h_{(j-2k) mod n} a_k +
    g_{(j-2k) mod n} d_k, accumulated tap by tap."""
    n = block.shape[ax]
    h = n // 2
    a = np.take(block, np.arange(h), axis=ax)
    d = np.take(block, np.arange(h, n), axis=ax)
    out = np.zeros_like(block)
    k = np.arange(h)
    for m in range(4):  # scatter-add tap m (indices repeat when n < 4)
        np.add.at(np.moveaxis(out, ax, 0), (2 * k + m) % n, np.moveaxis(D4_H[m] * a + D4_G[m] * d, ax, 0))
    return out


def d4_fwd(x, levels, nd=None):
    """L-level periodized D4 DWT in the Mallat layout of haar_fwd (per level along d0, d1[, d2]
    on the current approximation block).  Orthonormal: the unitary W of PAPER.md:117."""
    nd = x.ndim if nd is None else nd
    shape = x.shape[-nd:]
    for s_ in shape:
        if s_ % (1 << levels):
            raise ValueError("image size not divisible by 2^levels")
    out = np.array(x, dtype=np.complex128, copy=True)
    lead = out.ndim - nd
    for lvl in range(levels):
        sl = tuple([slice(None)] * lead + [slice(0, s_ >> lvl) for s_ in shape])
        blk = out[sl]
        for d in range(nd):
            blk = _d4_axis_fwd(blk, lead + d)
        out[sl] = blk
    return out


def d4_inv(c, levels, nd=None):
    """W^H = W^{-1} for the D4 DWT (coarsest level first, axes in reverse order)."""
    nd = c.ndim if nd is None else nd
    shape = c.shape[-nd:]
    out = np.array(c, dtype=np.complex128, copy=True)
    lead = out.ndim - nd
    for lvl in reversed(range(levels)):
        sl = tuple([slice(None)] * lead + [slice(0, s_ >> lvl) for s_ in shape])
        blk = out[sl]
        for d in reversed(range(nd)):
            blk = _d4_axis_inv(blk, lead + d)
        out[sl] = blk
    return out


def wavelet_fwd(x, levels, nd=None, family="haar"):
    return d4_fwd(x, levels, nd) if family == "d4" else haar_fwd(x, levels, nd)


def wavelet_inv(c, levels, nd=None, family="haar"):
    return d4_inv(c, levels, nd) if family == "d4" else haar_inv(c, levels, nd)


def apply_A(x, sens, mask, mu, lam, gamma):
    """A x = mu sum_c (RFS_c)^H RFS_c x + lam sum_d D_d^H D_d x + gamma W^H W x
    (PAPER.md:127-129), with W^H W = I exactly (reading A7)."""
    return mu * data_normal(x, sens, mask) + lam * tv_normal(x) + gamma * x


def shrink(z, t):
    """Complex soft threshold z * max(|z| - t, 0) / |z|, 0 -> 0 (reading A9)."""
    a = np.abs(z)
    scale = np.where(a > t, (a - t) / np.where(a > 0, a, 1.0), 0.0)
    return z * scale


def rss_init(y):
    """x^[1] = Sum of Squares(y_i) read as sqrt(sum_c |F^H y_c|^2), real (reading A12;
    PAPER.md:139)."""
    nd = y.ndim - 1
    return np.sqrt(np.sum(np.abs(ifftn_u(y, nd)) ** 2, axis=0)).astype(np.complex128)
