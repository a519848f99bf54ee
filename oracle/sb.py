"""Oracle Split Bregman, Algorithm 1 of PAPER.md:136-157, literally (test infrastructure
only; see oracle/__init__.py).

W is the orthonormal Haar (reading A6) or, with wavelet="d4", the paper's Daubechies-4
(reading A32).  Readings: A8 literal thresholds 1/lambda and 1/gamma; A9 complex soft
threshold; A10 anisotropic TV (separate d_x, d_y[, d_z]); A11 all wavelet coefficients
shrunk; A12 RSS init; A13 nInner = 1 unless given; A14 auxiliaries persist across outer
iterations; lambda = 0 or gamma = 0 skips that branch.

Data feedback (steps 13-15) is done literally per coil in k-space:
    y_c^[j+1] = y_c^[j] + y_c^[1] - R F S_c x.
``feedback="image"`` instead carries u_j = sum_c E_c^H y_c^[j] and updates
u_{j+1} = u_j + u_1 - E^H E x (linearity of E^H); tests pin the two equal.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

from . import ops
from .pcg import pcg
from .precond import apply_Minv, build_k, jacobi_diag

__all__ = ["SbLog", "sb_recon"]


@dataclasses.dataclass
class SbLog:
    pcg_iters: List[int]
    final_relres: List[float]
    relres_hist: List[List[float]]
    k: Optional[np.ndarray]


def sb_recon(y, sens, mask, mu, lam, gamma, n_outer, n_inner=1, levels=1, eps=1e-3,
             max_iters=50, precond="circulant", feedback="literal", x_init=None,
             return_state=False, wavelet="haar"):
    """Algorithm 1.  y: [C, *image] zero-filled k-space, sens: [C, *image],
    mask: 0/1 over the k-space grid.  Returns (x, SbLog[, state])."""
    nd = mask.ndim
    # step 1
    x = ops.rss_init(y) if x_init is None else np.array(x_init, dtype=np.complex128)
    y1 = np.array(y, dtype=np.complex128, copy=True)
    yj = y1.copy()
    zero = np.zeros(mask.shape, dtype=np.complex128)
    d = [zero.copy() for _ in range(nd)]
    bd = [zero.copy() for _ in range(nd)]
    dw = zero.copy()
    bw = zero.copy()

    def A(v):
        return ops.apply_A(v, sens, mask, mu, lam, gamma)

    k = None
    Minv = None
    if precond == "circulant":
        k = build_k(sens, mask, mu, lam, gamma)          # built once
        Minv = lambda v: apply_Minv(v, k)                # noqa: E731
    elif precond == "jacobi":
        dj = jacobi_diag(sens, mask, mu, lam, gamma)
        Minv = lambda v: v / dj                          # noqa: E731
    elif precond != "none":
        raise ValueError(precond)

    u1 = ops.encode_adj(y1, sens, mask) if feedback == "image" else None
    uj = u1.copy() if feedback == "image" else None
    log = SbLog([], [], [], k)
    for _j in range(n_outer):                                           # step 2
        for _k in range(n_inner):                                       # step 3
            data = ops.encode_adj(yj, sens, mask) if feedback == "literal" else uj
            rhs = mu * data                                             # step 4
            if lam != 0:
                rhs = rhs + lam * sum(ops.diff_adj(d[a] - bd[a], a, nd) for a in range(nd))
            if gamma != 0:
                rhs = rhs + gamma * ops.wavelet_inv(dw - bw, levels, nd, wavelet)
            res = pcg(A, rhs, x, Minv, eps, max_iters)                   # step 5
            x = res.x
            log.pcg_iters.append(res.iters)
            log.final_relres.append(res.relres[-1])
            log.relres_hist.append(res.relres)
            if lam != 0:
                for a in range(nd):                                     # steps 6-7, 9-10
                    z = ops.diff(x, a, nd) + bd[a]
                    d[a] = ops.shrink(z, 1.0 / lam)
                    bd[a] = z - d[a]
            if gamma != 0:                                              # steps 8, 11
                z = ops.wavelet_fwd(x, levels, nd, wavelet) + bw
                dw = ops.shrink(z, 1.0 / gamma)
                bw = z - dw
        if feedback == "literal":                                       # steps 13-15
            yj = yj + y1 - ops.encode(x, sens, mask)
        else:
            uj = uj + u1 - ops.data_normal(x, sens, mask)
    if return_state:
        return x, log, dict(d=d, bd=bd, dw=dw, bw=bw, yj=yj, uj=uj)
    return x, log
