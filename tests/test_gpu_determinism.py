"""Run-to-run determinism of the cluster kernels (reading A24: fixed reduction orders).

The plane kernels (K1P, k_plane.cu) exchange tile rows between the CTAs of a cluster with
asynchronous bulk copies completed on mbarriers, and K1 (k_matvec.cu) sums the coil groups of a
cluster through DSMEM in a fixed order. Repeating an operator, or a whole fixed-count solve, on
the same inputs must therefore give bitwise-identical results — a missed wait or a reordered
sum would show up here as a difference in the last bits, before it shows up against the oracle.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg


def _ctx(sens, mask):
    return SbPcg(torch.from_numpy(sens).to(torch.complex64).cuda(), torch.from_numpy(mask).cuda(),
                 1.0, 0.02, 0.02, 1)


def _plane2d(B, shape, coils, seed):
    rng = np.random.default_rng(seed)
    sens = rng.standard_normal((B, coils) + shape) + 1j * rng.standard_normal((B, coils) + shape)
    mask = (rng.random((B,) + shape) < 0.3).astype(np.uint8)
    mask[:, 0, 0], mask[:, 0, 1] = 1, 0  # non-separable
    return sens, mask


def _line(B, shape, coils, seed):
    rng = np.random.default_rng(seed)
    sens = rng.standard_normal((B, coils) + shape) + 1j * rng.standard_normal((B, coils) + shape)
    rows = (rng.random((B, shape[0])) < 0.3).astype(np.uint8)
    rows[:, 0] = 1
    return sens, np.repeat(rows[:, :, None], shape[1], axis=2)


def _vol3d(shape, coils):
    p = synth.problem3d(5, shape=shape, coils=coils)
    return p["sens"][None], p["mask"][None]


CASES = {
    "plane2d_256x128_G16": lambda: _plane2d(3, (256, 128), 6, 1),
    "plane3d_8x192x192_G8": lambda: _vol3d((8, 192, 192), 4),
    "line_256x256_K1G8_pre2d": lambda: _line(1, (256, 256), 12, 2),
    "line_256x256_batch": lambda: _line(20, (256, 256), 3, 3),
}


@pytest.mark.parametrize("name", list(CASES))
def test_operators_and_solve_bitwise_repeatable(name):
    sens, mask = CASES[name]()
    ctx = _ctx(sens, mask)
    shape = (sens.shape[0],) + sens.shape[2:]
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).to(torch.complex64).cuda()
    ya = [ctx.apply_A(x) for _ in range(4)]
    za = [ctx.apply_Pinv(x) for _ in range(4)]
    for y in ya[1:]:
        assert torch.equal(y, ya[0])
    for z in za[1:]:
        assert torch.equal(z, za[0])
    x0 = torch.zeros_like(x)
    xs = [ctx.solve(x, x0, eps=0.0, max_iters=8)[0] for _ in range(2)]
    assert torch.isfinite(torch.view_as_real(xs[0])).all()
    assert torch.equal(xs[0], xs[1])
    ctx.close()
