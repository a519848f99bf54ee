"""Oracle-side k-space synthesis for tests (test infrastructure only).

y_c = R (F S_c x + sigma n_c), sigma = 0.005 max_c,k |F S_c x| over the fully sampled
k-space (BASELINE.json config 1 noise; reading A21), unsampled entries exactly zero
(PAPER.md:95).  The GPU-side bench forms the same recipe with the library's sb_encode.
"""
from __future__ import annotations

import numpy as np

from .fft import fftn_u

__all__ = ["make_kspace", "NOISE_REL"]

NOISE_REL = 0.005


def make_kspace(phantom, sens, mask, noise, noise_rel=NOISE_REL):
    nd = mask.ndim
    full = fftn_u(sens * phantom[None], nd)
    sigma = noise_rel * float(np.max(np.abs(full)))
    return mask * (full + sigma * noise)
