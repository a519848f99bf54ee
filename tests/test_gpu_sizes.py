"""Parity sweep over every plane size the plane kernels instantiate (k_plane.cu): 2D problems
with a non-separable random mask and 3D volumes with a readout-constant mask — apply_A and
M^{-1} against the oracle (per-operator relative L2 <= 1e-5), one fixed-count PCG (<= 1e-3)."""
import numpy as np
import pytest
import torch

import synth
from oracle import ops, precond
from oracle.pcg import pcg
from tests.helpers import relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg

SIZES2 = [(8, 8), (8, 16), (8, 32), (8, 64), (16, 8), (16, 16), (16, 32), (16, 64), (16, 128), (16, 256),
          (32, 8), (32, 16), (32, 32), (32, 64), (32, 128), (32, 256), (64, 8), (64, 16), (64, 32), (64, 64),
          (64, 128), (64, 256), (128, 8), (128, 16), (128, 32), (128, 64), (128, 128), (128, 256), (256, 8),
          (256, 16), (256, 32), (256, 64), (256, 128), (256, 256)]
SIZES3 = [(8, 16, 16), (8, 32, 32), (8, 48, 48), (8, 64, 64), (8, 128, 128), (8, 192, 192), (8, 256, 256),
          (192, 16, 16)]


def _c32(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _check(sens, mask, shape, seed):
    mu, lam, gam = 1.0, 0.03, 0.02
    ctx = SbPcg(torch.from_numpy(sens[None]).to(torch.complex64).cuda(), torch.from_numpy(mask[None]).cuda(),
                mu, lam, gam, 1)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    xt = torch.from_numpy(x[None]).to(torch.complex64).cuda()
    s32 = _c32(sens)
    y = ctx.apply_A(xt).cpu().numpy()[0]
    assert relerr(y, ops.apply_A(_c32(x), s32, mask, mu, lam, gam)) <= 1e-5
    k = precond.build_k(s32, mask, mu, lam, gam)
    z = ctx.apply_Pinv(xt).cpu().numpy()[0]
    assert relerr(z, precond.apply_Minv(_c32(x), k)) <= 1e-5
    xs, st = ctx.solve(xt, torch.zeros_like(xt), eps=0.0, max_iters=6)
    ref = pcg(lambda v: ops.apply_A(v, s32, mask, mu, lam, gam), _c32(x), np.zeros(shape, complex),
              lambda v: precond.apply_Minv(v, k), 0.0, 6)
    assert relerr(xs.cpu().numpy()[0], ref.x) <= 1e-3
    ctx.close()


@pytest.mark.parametrize("shape", SIZES2, ids=lambda s: f"{s[0]}x{s[1]}")
def test_plane2d_sizes(shape):
    rng = np.random.default_rng(sum(shape))
    sens = rng.standard_normal((2,) + shape) + 1j * rng.standard_normal((2,) + shape)
    mask = (rng.random(shape) < 0.4).astype(np.uint8)
    mask[0, 0], mask[0, 1] = 1, 0           # non-separable: rows are not constant
    mask[1, 0], mask[1, 1] = 0, 1
    _check(sens, mask, shape, 1)


@pytest.mark.parametrize("shape", SIZES3, ids=lambda s: "x".join(map(str, s)))
def test_plane3d_sizes(shape):
    p = synth.problem3d(5, shape=shape, coils=2)
    _check(p["sens"], p["mask"], shape, 2)


SIZESL = [(8, 8), (16, 64), (32, 32), (64, 256), (128, 16), (256, 8), (256, 128), (128, 256)]


@pytest.mark.parametrize("coils", [1, 5])
@pytest.mark.parametrize("shape", SIZESL, ids=lambda s: f"{s[0]}x{s[1]}")
def test_line_mask_sizes(shape, coils):
    # K1 (line masks) at every column length it instantiates, with coil-group clusters G in
    # {1..8} chosen by the batch (B = 1 here) and both preconditioner forms (fused for B = 1)
    rng = np.random.default_rng(7 * shape[0] + shape[1] + coils)
    sens = rng.standard_normal((coils,) + shape) + 1j * rng.standard_normal((coils,) + shape)
    rows = (rng.random(shape[0]) < 0.4).astype(np.uint8)
    rows[0] = 1
    mask = np.repeat(rows[:, None], shape[1], axis=1)
    _check(sens, mask, shape, 3)
