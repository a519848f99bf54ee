"""GPU parity of the persistent per-problem cluster PCG (KC, k_pcgc.cu: 256 x 256 line masks,
circulant preconditioner — BASELINE configs 2 and 3; opt-in with SBPCG_KC=1) against the
oracle and against the default kernel-sequence path (K1 -> K2a/b/c in a CUDA-graph while
loop)."""
import os

import numpy as np
import pytest
import torch

from oracle import ops, precond, sb
from oracle.pcg import pcg
from tests.helpers import batch, relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg

DEV = "cuda"


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.complex64).to(DEV)


def _c32(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _ctx(ps, mu, lam, gam, levels, kc=True):
    old = os.environ.get("SBPCG_KC")
    os.environ["SBPCG_KC"] = "1" if kc else "0"
    try:
        sens = np.stack([p["sens"] for p in ps])
        masks = np.stack([p["mask"] for p in ps])
        return SbPcg(_t(sens), torch.from_numpy(masks).to(DEV), mu, lam, gam, levels)
    finally:
        if old is None:
            del os.environ["SBPCG_KC"]
        else:
            os.environ["SBPCG_KC"] = old


def _crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_kc_pcg_fixed_count_parity():
    ps = batch(2, 2, (256, 256), 12)
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = _ctx(ps, mu, lam, gam, 3)
    rng = np.random.default_rng(31)
    bvec = np.stack([_crandn(rng, 256, 256) for _ in ps])
    x0 = np.stack([ops.rss_init(p["y"]) for p in ps])
    x, st = ctx.solve(_t(bvec), _t(x0), eps=0.0, max_iters=15, precond=1, history=True)
    assert st["iters"] == [15, 15]
    xg = x.cpu().numpy()
    for b, p in enumerate(ps):
        s32 = _c32(p["sens"])
        k = precond.build_k(s32, p["mask"], mu, lam, gam)
        ref = pcg(lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam), _c32(bvec[b]), _c32(x0[b]),
                  lambda v: precond.apply_Minv(v, k), 0.0, 15)
        assert relerr(xg[b], ref.x) <= 1e-3, relerr(xg[b], ref.x)
        np.testing.assert_allclose(st["relres_hist"][b][:16], ref.relres, rtol=2e-2, atol=1e-6)
    ctx.close()


def test_kc_matches_kernel_sequence_in_tolerance_mode():
    ps = batch(2, 3, (256, 256), 12)
    mu, lam, gam = 1.0, 0.02, 0.02
    rng = np.random.default_rng(32)
    bvec = _t(np.stack([_crandn(rng, 256, 256) for _ in ps]))
    x0 = torch.zeros_like(bvec)
    a, b = _ctx(ps, mu, lam, gam, 3, kc=True), _ctx(ps, mu, lam, gam, 3, kc=False)
    xa, sa = a.solve(bvec, x0, eps=1e-4, max_iters=100)
    xb, sb_ = b.solve(bvec, x0, eps=1e-4, max_iters=100)
    assert sa["iters"] == sb_["iters"] and all(sa["converged"])
    assert relerr(xa.cpu().numpy(), xb.cpu().numpy()) <= 1e-5
    a.close(), b.close()


def test_kc_batch_equals_single():
    ps = batch(2, 3, (256, 256), 12)
    mu, lam, gam = 1.0, 0.02, 0.02
    rng = np.random.default_rng(33)
    bvec = np.stack([_crandn(rng, 256, 256) * (10 ** i) for i in range(3)])
    x0 = np.zeros_like(bvec)
    ctx = _ctx(ps, mu, lam, gam, 3)
    xb, stb = ctx.solve(_t(bvec), _t(x0), eps=1e-5, max_iters=100)
    ctx.close()
    for i, p in enumerate(ps):
        c1 = _ctx([p], mu, lam, gam, 3)
        x1, st1 = c1.solve(_t(bvec[i:i + 1]), _t(x0[i:i + 1]), eps=1e-5, max_iters=100)
        assert st1["iters"][0] == stb["iters"][i]
        assert torch.equal(x1[0], xb[i])  # bitwise: each problem is one independent cluster
        c1.close()


@pytest.mark.parametrize("eager", [False, True])
def test_kc_sb_recon_fixed_counts(eager):
    ps = batch(2, 2, (256, 256), 12, amp=100.0)
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = _ctx(ps, mu, lam, gam, 3)
    y = np.stack([p["y"] for p in ps])
    xg, log = ctx.recon(_t(y), 3, eps=0.0, max_iters=10, use_graph=not eager)
    assert log["pcg_iters"] == [[10, 10]] * 3
    for b, p in enumerate(ps):
        ref, _ = sb.sb_recon(_c32(p["y"]), _c32(p["sens"]), p["mask"], mu, lam, gam, 3, 1, 3, 0.0, 10, "circulant")
        assert relerr(xg.cpu().numpy()[b], ref) <= 1e-3
    ctx.close()
