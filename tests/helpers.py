"""Shared test helpers: seeded problems (synth) + oracle k-space and references."""
import numpy as np

import synth
from oracle import problems


def relerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make_problem(config=1, shape=None, coils=None, amp=None, slice_=0, mask_kind=None, seed_mask=None):
    """Seeded problem: phantom, sens (normalised, complex), mask, oracle k-space y."""
    p = synth.problem2d(config, slice_, shape=shape, coils=coils, amplitude=amp)
    if mask_kind == "random":
        shp = p["mask"].shape
        p["mask"] = synth.random_vd_mask2d(shp, 4, max(2, min(shp) // 8),
                                           synth.rng_for(config, slice_ if seed_mask is None else seed_mask, 5))
    p["y"] = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    return p


def batch(config, B, shape=None, coils=None, amp=None, mask_kind=None):
    ps = [make_problem(config, shape, coils, amp, slice_=s, mask_kind=mask_kind) for s in range(B)]
    return ps
