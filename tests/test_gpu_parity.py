"""GPU (libsbpcg, sm_100a) vs oracle parity, through the C ABI binding.

Tolerances (BASELINE.json north_star): per operator application relative L2 <= 1e-5;
Lambda (k) relative <= 1e-6; fixed-count PCG / SB image relative L2 <= 1e-3.
"""
import numpy as np
import pytest
import torch

from oracle import ops, precond, sb
from oracle.pcg import pcg
from tests.helpers import batch, make_problem, relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbError, SbPcg

DEV = "cuda"


def _t(a, dtype=torch.complex64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dtype).to(DEV)


def _np(t):
    return t.detach().cpu().numpy().astype(np.complex128)


def _ctx(ps, mu, lam, gam, levels):
    sens = np.stack([p["sens"] for p in ps])
    masks = np.stack([p["mask"] for p in ps])
    return SbPcg(_t(sens), torch.from_numpy(masks).to(DEV), mu, lam, gam, levels)


def _crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# sizes spanning several tiles; (8,8)/(16,16) are single-tile edge cases
CASES = [
    dict(config=1, shape=(64, 64), coils=4, mask=None),
    dict(config=1, shape=(8, 8), coils=2, mask=None),
    dict(config=1, shape=(16, 32), coils=3, mask=None),
    dict(config=2, shape=(256, 256), coils=12, mask=None),
    dict(config=1, shape=(64, 64), coils=4, mask="random"),
    dict(config=2, shape=(128, 64), coils=5, mask="random"),
]


def _case_id(c):
    return f"{c['shape'][0]}x{c['shape'][1]}c{c['coils']}{'R' if c['mask'] else 'L'}"


@pytest.mark.parametrize("case", CASES, ids=_case_id)
def test_apply_A_and_Pinv_and_k(case):
    ps = batch(case["config"], 2, case["shape"], case["coils"], mask_kind=case["mask"])
    mu, lam, gam = 1.0, 0.05, 0.02
    ctx = _ctx(ps, mu, lam, gam, 1)
    rng = np.random.default_rng(1)
    x = np.stack([_crandn(rng, *case["shape"]) for _ in ps])
    y = _np(ctx.apply_A(_t(x)))
    kg = ctx.get_k().numpy()
    z = _np(ctx.apply_Pinv(_t(x)))
    for b, p in enumerate(ps):
        ref = ops.apply_A(x[b].astype(np.complex64).astype(np.complex128), p["sens"].astype(np.complex64),
                          p["mask"], mu, lam, gam)
        assert relerr(y[b], ref) <= 1e-5, ("apply_A", b)
        sens32 = p["sens"].astype(np.complex64).astype(np.complex128)
        kref = precond.build_k(sens32, p["mask"], mu, lam, gam)
        assert relerr(kg[b], kref) <= 1e-6, ("k", b)
        assert np.max(np.abs(kg[b] - kref) / kref) <= 1e-5
        zref = precond.apply_Minv(x[b].astype(np.complex64).astype(np.complex128), kref)
        assert relerr(z[b], zref) <= 1e-5, ("Pinv", b)
    ctx.close()


@pytest.mark.parametrize("case", CASES[:3] + CASES[4:5], ids=_case_id)
def test_encode_adjoint(case):
    ps = batch(case["config"], 2, case["shape"], case["coils"], mask_kind=case["mask"])
    ctx = _ctx(ps, 1.0, 0.05, 0.05, 1)
    x = np.stack([p["phantom"] for p in ps])
    y = _np(ctx.encode(_t(x)))
    yfull = _np(ctx.encode(_t(x), full=True))
    yin = np.stack([p["y"] for p in ps])
    u = _np(ctx.adjoint(_t(yin)))
    for b, p in enumerate(ps):
        s32 = p["sens"].astype(np.complex64).astype(np.complex128)
        x32 = x[b].astype(np.complex64).astype(np.complex128)
        assert relerr(y[b], ops.encode(x32, s32, p["mask"])) <= 1e-5
        assert relerr(yfull[b], ops.encode(x32, s32, np.ones_like(p["mask"]))) <= 1e-5
        y32 = yin[b].astype(np.complex64).astype(np.complex128)
        assert relerr(u[b], ops.encode_adj(y32, s32, p["mask"])) <= 1e-5
    ctx.close()


@pytest.mark.parametrize("precond_kind", [1, 0, 2])
@pytest.mark.parametrize("use_graph", [True, False])
def test_pcg_fixed_count_parity(precond_kind, use_graph):
    ps = batch(1, 3, (64, 64), 4)
    mu, lam, gam = 1.0, 0.05, 0.05
    ctx = _ctx(ps, mu, lam, gam, 1)
    rng = np.random.default_rng(2)
    bvec = np.stack([_crandn(rng, 64, 64) for _ in ps])
    x0 = np.stack([ops.rss_init(p["y"]) for p in ps])
    x, st = ctx.solve(_t(bvec), _t(x0), eps=0.0, max_iters=15, precond=precond_kind, use_graph=use_graph,
                      history=True)
    xg = _np(x)
    assert st["iters"] == [15, 15, 15]
    for b, p in enumerate(ps):
        s32 = p["sens"].astype(np.complex64).astype(np.complex128)
        A = lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam)  # noqa: E731
        Minv = None
        if precond_kind == 1:
            k = precond.build_k(s32, p["mask"], mu, lam, gam)
            Minv = lambda v: precond.apply_Minv(v, k)  # noqa: E731
        elif precond_kind == 2:  # Jacobi
            dj = precond.jacobi_diag(s32, p["mask"], mu, lam, gam)
            Minv = lambda v: v / dj  # noqa: E731
        ref = pcg(A, bvec[b].astype(np.complex64).astype(np.complex128),
                  x0[b].astype(np.complex64).astype(np.complex128), Minv, 0.0, 15)
        assert relerr(xg[b], ref.x) <= 1e-3
        np.testing.assert_allclose(st["relres_hist"][b][:16], ref.relres, rtol=2e-2, atol=1e-6)
    ctx.close()


def test_pcg_tolerance_mode_counts():
    ps = batch(2, 2, (128, 128), 8)
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = _ctx(ps, mu, lam, gam, 3)
    rng = np.random.default_rng(3)
    bvec = np.stack([_crandn(rng, 128, 128) for _ in ps])
    x0 = np.zeros_like(bvec)
    for pk in (1, 0):
        x, st = ctx.solve(_t(bvec), _t(x0), eps=1e-4, max_iters=200, precond=pk)
        for b, p in enumerate(ps):
            s32 = p["sens"].astype(np.complex64).astype(np.complex128)
            k = precond.build_k(s32, p["mask"], mu, lam, gam)
            ref = pcg(lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam),
                      bvec[b].astype(np.complex64).astype(np.complex128), x0[b],
                      (lambda v: precond.apply_Minv(v, k)) if pk else None, 1e-4, 200)
            assert abs(st["iters"][b] - ref.iters) <= 1, (pk, b, st["iters"][b], ref.iters)
            assert st["converged"][b]
            assert relerr(_np(x)[b], ref.x) <= 1e-3
    ctx.close()


def test_pcg_edge_cases():
    ps = batch(1, 2, (32, 32), 2)
    ctx = _ctx(ps, 1.0, 0.05, 0.05, 1)
    zero = torch.zeros((2, 32, 32), dtype=torch.complex64, device=DEV)
    rng = np.random.default_rng(4)
    x0 = _t(np.stack([_crandn(rng, 32, 32) for _ in ps]))
    x, st = ctx.solve(zero, x0, eps=1e-4, max_iters=10)
    assert torch.count_nonzero(x).item() == 0 and st["converged"] == [True, True] and st["iters"] == [0, 0]
    # mixed: problem 0 has b = 0, problem 1 random -> independent convergence
    bb = zero.clone()
    bb[1] = x0[1]
    x, st = ctx.solve(bb, torch.zeros_like(x0), eps=1e-5, max_iters=100)
    assert st["iters"][0] == 0 and st["iters"][1] > 0 and torch.count_nonzero(x[0]).item() == 0
    # already converged start: x0 = exact-ish solution -> 0 iterations
    x2, st2 = ctx.solve(bb, x, eps=1e-3, max_iters=100)
    assert st2["iters"][1] == 0
    ctx.close()
    # argument errors
    with pytest.raises(SbError):
        SbPcg(_t(np.stack([ps[0]["sens"]])), torch.from_numpy(ps[0]["mask"][None]).to(DEV), 1.0, 0.1, 0.0, 1)
    with pytest.raises(SbError):
        SbPcg(torch.zeros((1, 1, 48, 48), dtype=torch.complex64, device=DEV),
              torch.ones((1, 48, 48), dtype=torch.uint8, device=DEV), 1.0, 0.1, 0.1, 1)


def test_batch_equals_single():
    ps = batch(1, 3, (64, 64), 4)
    mu, lam, gam = 1.0, 0.05, 0.05
    ctx = _ctx(ps, mu, lam, gam, 1)
    rng = np.random.default_rng(5)
    bvec = np.stack([_crandn(rng, 64, 64) * (10 ** b) for b in range(3)])
    x0 = np.zeros_like(bvec)
    xb, stb = ctx.solve(_t(bvec), _t(x0), eps=1e-5, max_iters=100)
    ctx.close()
    for b, p in enumerate(ps):
        c1 = _ctx([p], mu, lam, gam, 1)
        x1, st1 = c1.solve(_t(bvec[b:b + 1]), _t(x0[b:b + 1]), eps=1e-5, max_iters=100)
        assert st1["iters"][0] == stb["iters"][b]
        assert torch.equal(x1[0], xb[b])  # bitwise: frozen problems are not touched
        c1.close()


def test_sb_update_parity():
    ps = batch(1, 2, (64, 64), 4, amp=100.0)
    lam, gam, L = 0.05, 0.05, 3
    ctx = _ctx(ps, 1.0, lam, gam, L)
    rng = np.random.default_rng(6)
    x = np.stack([p["phantom"] for p in ps])
    bx = np.stack([_crandn(rng, 64, 64) for _ in ps]) * 3
    by = np.stack([_crandn(rng, 64, 64) for _ in ps]) * 3
    bw = np.stack([_crandn(rng, 64, 64) for _ in ps]) * 3
    gbx, gby, gbw, grhs = (_np(t) for t in ctx.sb_update(_t(x), _t(bx), _t(by), _t(bw)))
    for b in range(2):
        xs = x[b].astype(np.complex64).astype(np.complex128)
        c = lambda a: a[b].astype(np.complex64).astype(np.complex128)  # noqa: E731
        rb = [c(bx), c(by)]
        dd = []
        for a in range(2):
            z = ops.diff(xs, a) + rb[a]
            d = ops.shrink(z, 1 / lam)
            rb[a] = z - d
            dd.append(d)
        zw = ops.haar_fwd(xs, L) + c(bw)
        dw = ops.shrink(zw, 1 / gam)
        rbw = zw - dw
        rhs = lam * sum(ops.diff_adj(dd[a] - rb[a], a) for a in range(2)) + gam * ops.haar_inv(dw - rbw, L)
        assert relerr(gbx[b], rb[0]) <= 1e-5 and relerr(gby[b], rb[1]) <= 1e-5
        assert relerr(gbw[b], rbw) <= 1e-5
        assert relerr(grhs[b], rhs) <= 1e-5
    ctx.close()


@pytest.mark.parametrize("precond_kind", [1, 0, 2])
@pytest.mark.parametrize("amp", [1.0, 100.0])
def test_sb_recon_config1_fixed_counts(precond_kind, amp):
    # BASELINE config 1: 64x64, 4 coils, TV + 1-level Haar, mu=1, lam=gam=0.05, 5 outer, CG 15
    ps = batch(1, 2, (64, 64), 4, amp=amp)
    mu, lam, gam = 1.0, 0.05, 0.05
    ctx = _ctx(ps, mu, lam, gam, 1)
    y = np.stack([p["y"] for p in ps])
    xg, log = ctx.recon(_t(y), 5, eps=0.0, max_iters=15, precond=precond_kind)
    xg = _np(xg)
    assert log["pcg_iters"] == [[15, 15]] * 5
    for b, p in enumerate(ps):
        s32 = p["sens"].astype(np.complex64).astype(np.complex128)
        ref, rlog = sb.sb_recon(p["y"].astype(np.complex64).astype(np.complex128), s32, p["mask"], mu, lam, gam,
                                5, 1, 1, 0.0, 15, ["none", "circulant", "jacobi"][precond_kind])
        assert relerr(xg[b], ref) <= 1e-3, relerr(xg[b], ref)
    ctx.close()


def test_sb_recon_tolerance_mode_config2_geometry():
    # config-2 geometry (256x256, 12 coils, VD lines R=4, 3-level Haar), reduced outer count
    p = make_problem(2)
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = _ctx([p], mu, lam, gam, 3)
    xg, log = ctx.recon(_t(p["y"][None]), 3, eps=1e-4, max_iters=50, precond=1)
    s32 = p["sens"].astype(np.complex64).astype(np.complex128)
    ref, rlog = sb.sb_recon(p["y"].astype(np.complex64).astype(np.complex128), s32, p["mask"], mu, lam, gam,
                            3, 1, 3, 1e-4, 50, "circulant")
    got = [r[0] for r in log["pcg_iters"]]
    assert all(abs(a - b) <= 1 for a, b in zip(got, rlog.pcg_iters)), (got, rlog.pcg_iters)
    assert relerr(_np(xg)[0], ref) <= 1e-2
    ctx.close()


def test_host_pointer_entry_points_match_device():
    ps = batch(1, 1, (64, 64), 4)
    ctx = _ctx(ps, 1.0, 0.05, 0.05, 1)
    rng = np.random.default_rng(7)
    x = np.stack([_crandn(rng, 64, 64)])
    yd = ctx.apply_A(_t(x)).cpu()
    xh = torch.from_numpy(x).to(torch.complex64).pin_memory()
    yh = ctx.apply_A(xh)
    assert yh.device.type == "cpu" and torch.equal(yh, yd)
    y = ps[0]["y"][None]
    x1, l1 = ctx.recon(_t(y), 2, eps=0.0, max_iters=5)
    x2, l2 = ctx.recon(torch.from_numpy(y).to(torch.complex64), 2, eps=0.0, max_iters=5,
                       out=torch.empty((1, 64, 64), dtype=torch.complex64))
    assert torch.equal(x1.cpu(), x2)
    ctx.close()


@pytest.mark.parametrize("amp", [100.0, 1000.0])
def test_sb_recon_d4_fixed_counts(amp):
    # the paper's wavelet (Daubechies-4; reading A32), shrinkage active
    ps = batch(1, 2, (64, 64), 4, amp=amp)
    mu, lam, gam = 1.0, 0.05, 0.05
    sens = np.stack([p["sens"] for p in ps])
    masks = np.stack([p["mask"] for p in ps])
    ctx = SbPcg(_t(sens), torch.from_numpy(masks).to(DEV), mu, lam, gam, 2, wavelet="d4")
    y = np.stack([p["y"] for p in ps])
    xg, log = ctx.recon(_t(y), 4, eps=0.0, max_iters=10)
    xg = _np(xg)
    for b, p in enumerate(ps):
        s32 = p["sens"].astype(np.complex64).astype(np.complex128)
        ref, _ = sb.sb_recon(p["y"].astype(np.complex64).astype(np.complex128), s32, p["mask"], mu, lam, gam,
                             4, 1, 2, 0.0, 10, "circulant", wavelet="d4")
        haar, _ = sb.sb_recon(p["y"].astype(np.complex64).astype(np.complex128), s32, p["mask"], mu, lam, gam,
                              4, 1, 2, 0.0, 10, "circulant", wavelet="haar")
        assert relerr(xg[b], ref) <= 1e-3, relerr(xg[b], ref)
        assert relerr(ref, haar) > 10 * relerr(xg[b], ref)  # the test discriminates D4 from Haar
    ctx.close()


def test_update_sens_equals_fresh_context():
    # a context reused for new coil maps (same geometry/mask): Lambda rebuilt, cached graphs
    # still valid; results equal a context created from the new maps
    ps = batch(2, 2, (128, 128), 6)
    mask = ps[0]["mask"]
    ctx = SbPcg(_t(ps[0]["sens"][None]), torch.from_numpy(mask[None]).to(DEV), 1.0, 0.02, 0.02, 3)
    y1 = make_problem(2, (128, 128), 6, slice_=1)
    yk = _t(problems_kspace(ps[1], mask)[None])
    ctx.recon(yk, 2, eps=1e-4, max_iters=30)           # captures graphs with the old maps
    ctx.update_sens(_t(ps[1]["sens"][None]))
    xa, la = ctx.recon(yk, 3, eps=1e-4, max_iters=30)
    fresh = SbPcg(_t(ps[1]["sens"][None]), torch.from_numpy(mask[None]).to(DEV), 1.0, 0.02, 0.02, 3)
    xb, lb = fresh.recon(yk, 3, eps=1e-4, max_iters=30)
    assert la["pcg_iters"] == lb["pcg_iters"]
    assert torch.equal(xa, xb)
    assert np.array_equal(ctx.get_k().numpy(), fresh.get_k().numpy())
    del y1
    ctx.close(), fresh.close()


def problems_kspace(p, mask):
    from oracle import problems
    return problems.make_kspace(p["phantom"], p["sens"], mask, p["noise"])


def test_singular_k_reporting():
    # k >= gamma > 0 for finite maps, so only non-finite coil maps make Lambda singular
    # (SB_E_SINGULAR_K): reported by create (synchronous), and after the asynchronous rebuild of
    # sb_pcg_update_sens by the next synchronising call (include/sbpcg.h)
    ps = batch(1, 1, (64, 64), 4)
    bad = np.stack([ps[0]["sens"]]).copy()
    bad[0, 1, 5, 7] = np.nan
    with pytest.raises(SbError) as ei:
        _ctx([dict(sens=bad[0], mask=ps[0]["mask"])], 1.0, 0.05, 0.05, 1)
    assert ei.value.status == 5
    ctx = _ctx(ps, 1.0, 0.05, 0.05, 1)
    ctx.update_sens(_t(bad))
    y = _t(ps[0]["y"][None])
    with pytest.raises(SbError) as ei:
        ctx.recon(y, 1, eps=0.0, max_iters=2)
    assert ei.value.status == 5
    ctx.update_sens(_t(np.stack([ps[0]["sens"]])))  # healthy maps again: the context recovers
    x, log = ctx.recon(y, 1, eps=0.0, max_iters=2)
    assert torch.isfinite(x).all()
    ctx.close()


@pytest.mark.parametrize("shape,coils,nb", [((256, 256), 12, 1), ((64, 64), 4, 3), ((8, 8), 2, 2), ((128, 32), 5, 1)],
                         ids=["256c12b1", "64c4b3", "8c2b2", "128x32c5b1"])
def test_separable_lambda_build_equals_2d_build(monkeypatch, shape, coils, nb):
    """K4S (k_lambda.cu: the one-dimensional form of k_c for line masks, Parseval along d1)
    against the general 2D correlation build (C + 3 2D FFTs) on the same maps, both fp64 on the
    device: equal to rounding.  The oracle pin of both is test_apply_A_and_Pinv_and_k."""
    ps = batch(2, nb, shape, coils)
    mu, lam, gam = 1.0, 0.02, 0.02
    monkeypatch.setenv("SBPCG_LSEP", "1")
    ctx = _ctx(ps, mu, lam, gam, 1)
    k_sep = ctx.get_k().numpy()
    ctx.close()
    monkeypatch.setenv("SBPCG_LSEP", "0")
    ctx = _ctx(ps, mu, lam, gam, 1)
    k_2d = ctx.get_k().numpy()
    ctx.close()
    assert np.max(np.abs(k_sep - k_2d) / np.abs(k_2d)) <= 1e-12
    for b, p in enumerate(ps):
        kref = precond.build_k(p["sens"].astype(np.complex64).astype(np.complex128), p["mask"], mu, lam, gam)
        assert relerr(k_sep[b], kref) <= 1e-6
