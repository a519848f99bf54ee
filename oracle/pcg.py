"""Oracle preconditioned conjugate gradient (test infrastructure only; see oracle/__init__.py).

A is Hermitian positive definite, "which motivates the choice for the conjugate gradient
(CG) method"; the circulant M^{-1} is applied once per iteration to the
residual.  Reading A15: this is standard PCG (mathematically the
paper's left-preconditioned form; the residual sign is immaterial), monitoring the
recurrence residual ||r_k|| / ||b||.  Reading A16: the iteration count is the number of
A p products inside the loop.  Reading A17: <u, v> = sum conj(u) v and only real parts
enter alpha, beta, rho.  Reading A18: eps = 0 runs exactly max_iters iterations (early
stop only when rho' == 0).
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional

import numpy as np

__all__ = ["PcgResult", "PcgError", "pcg", "vdot_re"]


class PcgError(ArithmeticError):
    def __init__(self, kind: str):
        super().__init__(kind)
        self.kind = kind  # "indefinite" | "nonfinite"


@dataclasses.dataclass
class PcgResult:
    x: np.ndarray
    iters: int
    converged: bool
    relres: List[float]          # [||r_0||/||b||, ||r_1||/||b||, ...]
    true_relres: float           # ||b - A x|| / ||b|| recomputed at exit


def vdot_re(u, v) -> float:
    """Re <u, v> = Re sum conj(u) v."""
    return float(np.real(np.vdot(u.ravel(), v.ravel())))


def pcg(apply_A: Callable, b: np.ndarray, x0: np.ndarray, apply_Minv: Optional[Callable],
        eps: float, max_iters: int) -> PcgResult:
    Minv = apply_Minv if apply_Minv is not None else (lambda v: v.copy())
    x = np.array(x0, dtype=np.complex128, copy=True)
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return PcgResult(np.zeros_like(x), 0, True, [0.0], 0.0)
    r = b - apply_A(x)
    rel = float(np.linalg.norm(r)) / nb
    hist = [rel]
    if eps > 0 and rel <= eps:
        return PcgResult(x, 0, True, hist, rel)
    z = Minv(r)
    p = z.copy()
    rho = vdot_re(r, z)
    converged = False
    it = 0
    for k in range(1, max_iters + 1):
        q = apply_A(p)
        sigma = vdot_re(p, q)
        if not np.isfinite(sigma):
            raise PcgError("nonfinite")
        if not sigma > 0:
            raise PcgError("indefinite")
        alpha = rho / sigma
        x = x + alpha * p
        r = r - alpha * q
        it = k
        rel = float(np.linalg.norm(r)) / nb
        hist.append(rel)
        if eps > 0 and rel <= eps:
            converged = True
            break
        z = Minv(r)
        rho_new = vdot_re(r, z)
        if rho_new == 0.0:
            converged = True
            break
        beta = rho_new / rho
        rho = rho_new
        p = z + beta * p
    else:
        converged = eps == 0
    true_rel = float(np.linalg.norm(b - apply_A(x))) / nb
    return PcgResult(x, it, converged, hist, true_rel)
