"""GPU parity for the plane-cluster path (k_plane.cu): 3D problems (BASELINE config 5
geometry, mask constant along the readout d0) and 2D problems with a non-separable shared
mask (BASELINE config 4 geometry), through the C ABI binding, against the oracle.

Tolerances (BASELINE.json north_star): per operator relative L2 <= 1e-5; k relative <= 1e-6;
fixed-count PCG / SB image relative L2 <= 1e-3.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import ops, precond, problems, sb
from oracle.pcg import pcg
from tests.helpers import relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbError, SbPcg

DEV = "cuda"


def _t(a, dtype=torch.complex64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dtype).to(DEV)


def _np(t):
    return t.detach().cpu().numpy().astype(np.complex128)


def _c32(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# (shape, coils, levels): single-CTA planes, a 2-CTA cluster with a radix-3 plane (48^2),
# a 2-CTA cluster (64^2); d0 spans several column tiles
CASES3 = [((8, 32, 32), 3, 2), ((16, 48, 48), 2, 3), ((8, 64, 64), 2, 1), ((32, 16, 16), 2, 1)]


def _prob3(shape, coils, amp=1.0, B=1):
    ps = []
    for b in range(B):
        p = synth.problem3d(5, shape=shape, coils=coils, amplitude=amp)
        if b:  # a second, different problem: rotate the maps and the phantom
            p["sens"] = np.roll(p["sens"], b, axis=0)
            p["phantom"] = np.roll(p["phantom"], 3 * b, axis=1)
        p["y"] = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
        ps.append(p)
    return ps


def _ctx3(ps, mu, lam, gam, levels):
    sens = np.stack([p["sens"] for p in ps])
    mask = np.stack([p["mask"] for p in ps])
    return SbPcg(_t(sens), torch.from_numpy(mask).to(DEV), mu, lam, gam, levels)


def _id3(c):
    return "x".join(map(str, c[0])) + f"c{c[1]}"


@pytest.mark.parametrize("case", CASES3, ids=_id3)
def test_3d_apply_A_Pinv_k(case):
    shape, coils, L = case
    ps = _prob3(shape, coils, B=2)
    mu, lam, gam = 1.0, 0.03, 0.02
    ctx = _ctx3(ps, mu, lam, gam, L)
    rng = np.random.default_rng(11)
    x = np.stack([_crandn(rng, *shape) for _ in ps])
    y = _np(ctx.apply_A(_t(x)))
    z = _np(ctx.apply_Pinv(_t(x)))
    kg = ctx.get_k().numpy()
    for b, p in enumerate(ps):
        s32 = _c32(p["sens"])
        ref = ops.apply_A(_c32(x[b]), s32, p["mask"], mu, lam, gam)
        assert relerr(y[b], ref) <= 1e-5, ("apply_A", b, relerr(y[b], ref))
        kref = precond.build_k(s32, p["mask"], mu, lam, gam)
        assert relerr(kg[b], kref) <= 1e-6, ("k", b, relerr(kg[b], kref))
        assert np.max(np.abs(kg[b] - kref) / kref) <= 1e-5
        zref = precond.apply_Minv(_c32(x[b]), kref)
        assert relerr(z[b], zref) <= 1e-5, ("Pinv", b, relerr(z[b], zref))
    ctx.close()


@pytest.mark.parametrize("case", CASES3[:3], ids=_id3)
def test_3d_encode_adjoint(case):
    shape, coils, L = case
    ps = _prob3(shape, coils)
    p = ps[0]
    ctx = _ctx3(ps, 1.0, 0.01, 0.01, L)
    x = p["phantom"][None]
    y = _np(ctx.encode(_t(x)))[0]
    yf = _np(ctx.encode(_t(x), full=True))[0]
    u = _np(ctx.adjoint(_t(p["y"][None])))[0]
    s32 = _c32(p["sens"])
    assert relerr(y, ops.encode(_c32(x[0]), s32, p["mask"])) <= 1e-5
    assert relerr(yf, ops.encode(_c32(x[0]), s32, np.ones_like(p["mask"]))) <= 1e-5
    assert relerr(u, ops.encode_adj(_c32(p["y"]), s32, p["mask"])) <= 1e-5
    ctx.close()


@pytest.mark.parametrize("precond_kind", [1, 0, 2])
def test_3d_pcg_fixed_count(precond_kind):
    shape, coils, L = CASES3[0]
    ps = _prob3(shape, coils, B=2)
    mu, lam, gam = 1.0, 0.01, 0.01
    ctx = _ctx3(ps, mu, lam, gam, L)
    rng = np.random.default_rng(12)
    bvec = np.stack([_crandn(rng, *shape) for _ in ps])
    x0 = np.stack([ops.rss_init(p["y"]) for p in ps])
    x, st = ctx.solve(_t(bvec), _t(x0), eps=0.0, max_iters=10, precond=precond_kind, history=True)
    assert st["iters"] == [10, 10]
    xg = _np(x)
    for b, p in enumerate(ps):
        s32 = _c32(p["sens"])
        A = lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam)  # noqa: E731
        Minv = None
        if precond_kind == 1:
            k = precond.build_k(s32, p["mask"], mu, lam, gam)
            Minv = lambda v: precond.apply_Minv(v, k)  # noqa: E731
        elif precond_kind == 2:
            dj = precond.jacobi_diag(s32, p["mask"], mu, lam, gam)
            Minv = lambda v: v / dj  # noqa: E731
        ref = pcg(A, _c32(bvec[b]), _c32(x0[b]), Minv, 0.0, 10)
        assert relerr(xg[b], ref.x) <= 1e-3, relerr(xg[b], ref.x)
        np.testing.assert_allclose(st["relres_hist"][b][:11], ref.relres, rtol=2e-2, atol=1e-6)
    ctx.close()


def test_3d_sb_update_parity():
    shape, L = (8, 32, 32), 3
    ps = _prob3(shape, 2, amp=100.0)
    lam, gam = 0.05, 0.05
    ctx = _ctx3(ps, 1.0, lam, gam, L)
    rng = np.random.default_rng(13)
    x = ps[0]["phantom"][None]
    bs = [_crandn(rng, 1, *shape) * 3 for _ in range(4)]  # bx, by, bz, bw
    gbx, gby, gbw, grhs, gbz = (_np(t) for t in ctx.sb_update(_t(x), _t(bs[0]), _t(bs[1]), _t(bs[3]), bz=_t(bs[2])))
    xs = _c32(x[0])
    rb = [_c32(bs[a][0]) for a in range(3)]
    dd = []
    for a in range(3):
        z = ops.diff(xs, a) + rb[a]
        d = ops.shrink(z, 1 / lam)
        rb[a] = z - d
        dd.append(d)
    zw = ops.haar_fwd(xs, L) + _c32(bs[3][0])
    dw = ops.shrink(zw, 1 / gam)
    rbw = zw - dw
    rhs = lam * sum(ops.diff_adj(dd[a] - rb[a], a) for a in range(3)) + gam * ops.haar_inv(dw - rbw, L)
    assert relerr(gbx[0], rb[0]) <= 1e-5 and relerr(gby[0], rb[1]) <= 1e-5 and relerr(gbz[0], rb[2]) <= 1e-5
    assert relerr(gbw[0], rbw) <= 1e-5
    assert relerr(grhs[0], rhs) <= 1e-5
    ctx.close()


@pytest.mark.parametrize("amp", [1.0, 100.0])
def test_3d_sb_recon_fixed_counts(amp):
    # config-5 recipe (3D TV + 3D Haar, mu=1, lambda=gamma=0.01) at a reduced size
    shape, coils, L = (16, 48, 48), 3, 3
    ps = _prob3(shape, coils, amp=amp)
    p = ps[0]
    mu, lam, gam = 1.0, 0.01, 0.01
    ctx = _ctx3(ps, mu, lam, gam, L)
    xg, log = ctx.recon(_t(p["y"][None]), 3, eps=0.0, max_iters=8, precond=1)
    assert log["pcg_iters"] == [[8]] * 3
    ref, _ = sb.sb_recon(_c32(p["y"]), _c32(p["sens"]), p["mask"], mu, lam, gam, 3, 1, L, 0.0, 8, "circulant")
    assert relerr(_np(xg)[0], ref) <= 1e-3, relerr(_np(xg)[0], ref)
    ctx.close()


def test_3d_mask_must_be_readout_constant():
    shape = (8, 32, 32)
    p = _prob3(shape, 2)[0]
    mask = p["mask"].copy()
    mask[3, 0, 5] ^= 1
    with pytest.raises(SbError):
        SbPcg(_t(p["sens"][None]), torch.from_numpy(mask[None]).to(DEV), 1.0, 0.01, 0.01, 1)


# ---------------------------------------------------------------- 2D non-separable shared mask
def _c4(volume, coils, slices, amp=1.0):
    q = synth.problem_c4(slices, volume=volume, coils=coils, amplitude=amp)
    ys = [problems.make_kspace(q["phantom"][i], q["sens"][i].astype(np.complex128), q["mask"],
                               q["noise"][i].astype(np.complex128)) for i in range(len(slices))]
    return q, np.stack(ys)


def test_config4_geometry_plane2d_parity():
    # readout planes of a 3D volume, one shared (d1, d2) mask, 2D per-plane problems
    q, y = _c4((3, 128, 64), 4, [0, 1, 2])
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = SbPcg(_t(q["sens"]), torch.from_numpy(q["mask"]).to(DEV), mu, lam, gam, 3)
    rng = np.random.default_rng(14)
    x = np.stack([_crandn(rng, 128, 64) for _ in range(3)])
    ya = _np(ctx.apply_A(_t(x)))
    kg = ctx.get_k().numpy()
    xg, log = ctx.recon(_t(y), 3, eps=0.0, max_iters=8)
    xg = _np(xg)
    for b in range(3):
        s32 = _c32(q["sens"][b])
        assert relerr(ya[b], ops.apply_A(_c32(x[b]), s32, q["mask"], mu, lam, gam)) <= 1e-5
        kref = precond.build_k(s32, q["mask"], mu, lam, gam)
        assert relerr(kg[b], kref) <= 1e-6
        ref, _ = sb.sb_recon(_c32(y[b]), s32, q["mask"], mu, lam, gam, 3, 1, 3, 0.0, 8, "circulant")
        assert relerr(xg[b], ref) <= 1e-3, (b, relerr(xg[b], ref))
    ctx.close()


def test_config4_full_size_sampled():
    # BASELINE config 4 at full size (256 readout planes of 256x128, 16 coils) in the launch
    # configuration bench.py times; two sampled planes checked against the oracle
    spec = synth.CONFIGS[4]
    slices = list(range(spec.batch))
    q = synth.problem_c4(slices)
    mu, lam, gam = spec.params.mu, spec.params.lam, spec.params.gamma
    ctx = SbPcg(_t(q["sens"]), torch.from_numpy(q["mask"]).to(DEV), mu, lam, gam, spec.params.wavelet_levels)
    x = q["phantom"]
    ya = _np(ctx.apply_A(_t(x)))
    kg = ctx.get_k().numpy()
    for b in (0, 173):
        s32 = _c32(q["sens"][b])
        assert relerr(ya[b], ops.apply_A(_c32(x[b]), s32, q["mask"], mu, lam, gam)) <= 1e-5
        assert relerr(kg[b], precond.build_k(s32, q["mask"], mu, lam, gam)) <= 1e-6
    ctx.close()


def test_3d_sb_recon_d4_fixed_counts():
    shape, coils, L = (16, 32, 32), 2, 2
    p = _prob3(shape, coils, amp=300.0)[0]
    mu, lam, gam = 1.0, 0.01, 0.01
    ctx = SbPcg(_t(p["sens"][None]), torch.from_numpy(p["mask"][None]).to(DEV), mu, lam, gam, L, wavelet="d4")
    xg, log = ctx.recon(_t(p["y"][None]), 3, eps=0.0, max_iters=6)
    ref, _ = sb.sb_recon(_c32(p["y"]), _c32(p["sens"]), p["mask"], mu, lam, gam, 3, 1, L, 0.0, 6, "circulant",
                         wavelet="d4")
    assert relerr(_np(xg)[0], ref) <= 1e-3, relerr(_np(xg)[0], ref)
    ctx.close()
