"""The persistent whole-GPU kernel (k_persist.cu) against the oracle, and against
the kernel-sequence path, through the C ABI.

KR runs solves and whole SB reconstructions of small batches of square line-mask problems
(64^2 and 256^2) in one cooperative launch.  Same tolerances as every parity test
(BASELINE.json north_star): fixed-count PCG / SB image relative L2 <= 1e-3, tolerance-mode
iteration counts within +-1.
"""
import numpy as np
import pytest
import torch

from oracle import ops, precond, sb
from oracle.pcg import pcg
from tests.helpers import batch, make_problem, relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg

DEV = "cuda"


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.complex64).to(DEV)


def _np(t):
    return t.detach().cpu().numpy().astype(np.complex128)


def _c128(a):
    return a.astype(np.complex64).astype(np.complex128)


def _ctx(ps, mu, lam, gam, levels, persistent=True, cg=True):
    sens = np.stack([p["sens"] for p in ps])
    masks = np.stack([p["mask"] for p in ps])
    ctx = SbPcg(_t(sens), torch.from_numpy(masks).to(DEV), mu, lam, gam, levels, persistent=persistent)
    ctx.set_pcg_cg(cg)
    return ctx


# both PCG recurrence forms of the persistent kernel (SB_OPT_PCG_CG): Chronopoulos-Gear
# single-reduction (default) and the standard form
CG = pytest.mark.parametrize("cg", [True, False], ids=["cg", "std"])


def _crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# (config, shape, coils, batch): config-1 and config-2 geometries; B = 3 at 64^2 (three problems in
# one launch, 192 CTAs), B = 1 at 256^2 (the bench shape, 256 CTAs)
KR_CASES = [(1, (64, 64), 4, 1), (1, (64, 64), 4, 3), (2, (256, 256), 12, 1)]


def _kid(c):
    return f"{c[1][0]}c{c[2]}B{c[3]}"


@pytest.mark.parametrize("case", KR_CASES, ids=_kid)
@CG
def test_kr_fixed_count_solve_vs_oracle(case, cg):
    cfg, shape, coils, B = case
    ps = batch(cfg, B, shape, coils)
    mu, lam, gam = 1.0, 0.05, 0.05
    ctx = _ctx(ps, mu, lam, gam, 1, cg=cg)
    rng = np.random.default_rng(11)
    bvec = np.stack([_crandn(rng, *shape) for _ in ps])
    x0 = np.stack([ops.rss_init(p["y"]) for p in ps])
    x, st = ctx.solve(_t(bvec), _t(x0), eps=0.0, max_iters=15, precond=1, history=True)
    assert ctx.last_path() == "persistent"
    assert st["iters"] == [15] * B and all(st["converged"])
    xg = _np(x)
    for b, p in enumerate(ps):
        s32 = _c128(p["sens"])
        k = precond.build_k(s32, p["mask"], mu, lam, gam)
        ref = pcg(lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam), _c128(bvec[b]), _c128(x0[b]),
                  lambda v: precond.apply_Minv(v, k), 0.0, 15)
        assert relerr(xg[b], ref.x) <= 1e-3, relerr(xg[b], ref.x)
        np.testing.assert_allclose(st["relres_hist"][b][:16], ref.relres, rtol=2e-2, atol=1e-6)
    ctx.close()


@pytest.mark.parametrize("case", KR_CASES, ids=_kid)
@CG
def test_kr_tolerance_solve_counts(case, cg):
    cfg, shape, coils, B = case
    ps = batch(cfg, B, shape, coils)
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = _ctx(ps, mu, lam, gam, 3, cg=cg)
    rng = np.random.default_rng(12)
    bvec = np.stack([_crandn(rng, *shape) for _ in ps])
    x0 = np.zeros_like(bvec)
    x, st = ctx.solve(_t(bvec), _t(x0), eps=1e-4, max_iters=200, precond=1)
    assert ctx.last_path() == "persistent"
    for b, p in enumerate(ps):
        s32 = _c128(p["sens"])
        k = precond.build_k(s32, p["mask"], mu, lam, gam)
        ref = pcg(lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam), _c128(bvec[b]), x0[b],
                  lambda v: precond.apply_Minv(v, k), 1e-4, 200)
        assert abs(st["iters"][b] - ref.iters) <= 1, (b, st["iters"][b], ref.iters)
        assert st["converged"][b]
        assert relerr(_np(x)[b], ref.x) <= 1e-3
    ctx.close()


@pytest.mark.parametrize("amp", [1.0, 100.0])
@pytest.mark.parametrize("case", KR_CASES[:2], ids=_kid)
@CG
def test_kr_sb_recon_fixed_counts_vs_oracle(case, amp, cg):
    # BASELINE config 1 settings (TV + 1-level Haar, mu=1, lam=gam=0.05, 5 outer, CG fixed at 15);
    # amp = 100 makes the shrinkage active (reading A8)
    cfg, shape, coils, B = case
    ps = batch(cfg, B, shape, coils, amp=amp)
    mu, lam, gam = 1.0, 0.05, 0.05
    ctx = _ctx(ps, mu, lam, gam, 1, cg=cg)
    y = np.stack([p["y"] for p in ps])
    xg, log = ctx.recon(_t(y), 5, eps=0.0, max_iters=15, precond=1)
    assert log["path"] == "persistent"
    assert log["pcg_iters"] == [[15] * B] * 5
    xg = _np(xg)
    for b, p in enumerate(ps):
        ref, _ = sb.sb_recon(_c128(p["y"]), _c128(p["sens"]), p["mask"], mu, lam, gam, 5, 1, 1, 0.0, 15,
                             "circulant")
        assert relerr(xg[b], ref) <= 1e-3, relerr(xg[b], ref)
    ctx.close()


@pytest.mark.parametrize("amp,cg", [(1.0, False), (100.0, True)], ids=["std-amp1", "cg-amp100"])
def test_kr_sb_recon_bench_shape_fixed_counts(amp, cg):
    # the exact bench shape (config 2: 256^2, 12 coils, VD lines, 3-level Haar, mu=1,
    # lam=gam=0.02), B = 1, eps = 0: 5 outer x 10 CG against the oracle
    p = make_problem(2, amp=amp)
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = _ctx([p], mu, lam, gam, 3, cg=cg)
    xg, log = ctx.recon(_t(p["y"][None]), 5, eps=0.0, max_iters=10, precond=1)
    assert log["path"] == "persistent"
    ref, _ = sb.sb_recon(_c128(p["y"]), _c128(p["sens"]), p["mask"], mu, lam, gam, 5, 1, 3, 0.0, 10, "circulant")
    assert relerr(_np(xg)[0], ref) <= 1e-3, relerr(_np(xg)[0], ref)
    ctx.close()


@CG
def test_kr_sb_recon_tolerance_mode_config2(cg):
    # config 2 at its BASELINE settings (eps = 1e-4, max 50), 4 outer: per-solve counts +-1
    p = make_problem(2)
    mu, lam, gam = 1.0, 0.02, 0.02
    ctx = _ctx([p], mu, lam, gam, 3, cg=cg)
    xg, log = ctx.recon(_t(p["y"][None]), 4, eps=1e-4, max_iters=50, precond=1)
    assert log["path"] == "persistent"
    ref, rlog = sb.sb_recon(_c128(p["y"]), _c128(p["sens"]), p["mask"], mu, lam, gam, 4, 1, 3, 1e-4, 50, "circulant")
    got = [r[0] for r in log["pcg_iters"]]
    assert all(abs(a - b) <= 1 for a, b in zip(got, rlog.pcg_iters)), (got, rlog.pcg_iters)
    assert relerr(_np(xg)[0], ref) <= 1e-2
    ctx.close()


@pytest.mark.parametrize("case", KR_CASES, ids=_kid)
@CG
def test_kr_agrees_with_kernel_sequence(case, cg):
    cfg, shape, coils, B = case
    ps = batch(cfg, B, shape, coils, amp=100.0)
    mu, lam, gam = 1.0, 0.05, 0.05
    y = _t(np.stack([p["y"] for p in ps]))
    out = {}
    for pers in (True, False):
        ctx = _ctx(ps, mu, lam, gam, 1, persistent=pers, cg=cg)
        x, log = ctx.recon(y, 3, eps=0.0, max_iters=12, precond=1)
        out[pers] = (_np(x), log["path"])
        ctx.close()
    assert out[True][1] == "persistent" and out[False][1] == "graph"
    for b in range(B):  # the same arithmetic up to reduction order (cg: recurrence form, fp32 rounding)
        assert relerr(out[True][0][b], out[False][0][b]) <= (1e-4 if cg else 2e-5)


@CG
def test_kr_edge_cases(cg):
    ps = batch(1, 2, (64, 64), 4)
    ctx = _ctx(ps, 1.0, 0.05, 0.05, 1, cg=cg)
    zero = torch.zeros((2, 64, 64), dtype=torch.complex64, device=DEV)
    rng = np.random.default_rng(13)
    x0 = _t(np.stack([_crandn(rng, 64, 64) for _ in ps]))
    x, st = ctx.solve(zero, x0, eps=1e-4, max_iters=10)
    assert ctx.last_path() == "persistent"
    assert torch.count_nonzero(x).item() == 0 and st["converged"] == [True, True] and st["iters"] == [0, 0]
    bb = zero.clone()
    bb[1] = x0[1]
    x, st = ctx.solve(bb, torch.zeros_like(x0), eps=1e-5, max_iters=100)
    assert st["iters"][0] == 0 and st["iters"][1] > 0 and torch.count_nonzero(x[0]).item() == 0
    x2, st2 = ctx.solve(bb, x, eps=1e-3, max_iters=100)
    assert st2["iters"][1] == 0
    # max_iters = 1 and a problem that stops on max_iters with eps > 0 (not converged)
    x3, st3 = ctx.solve(bb, torch.zeros_like(x0), eps=1e-12, max_iters=1)
    assert st3["iters"][1] == 1 and not st3["converged"][1]
    ctx.close()


@CG
def test_kr_batch_equals_single_bitwise(cg):
    ps = batch(1, 3, (64, 64), 4)
    mu, lam, gam = 1.0, 0.05, 0.05
    ctx = _ctx(ps, mu, lam, gam, 1, cg=cg)
    rng = np.random.default_rng(14)
    bvec = np.stack([_crandn(rng, 64, 64) * (10 ** b) for b in range(3)])
    x0 = np.zeros_like(bvec)
    xb, stb = ctx.solve(_t(bvec), _t(x0), eps=1e-5, max_iters=100)
    assert ctx.last_path() == "persistent"
    ctx.close()
    for b, p in enumerate(ps):
        c1 = _ctx([p], mu, lam, gam, 1, cg=cg)
        x1, st1 = c1.solve(_t(bvec[b:b + 1]), _t(x0[b:b + 1]), eps=1e-5, max_iters=100)
        assert st1["iters"][0] == stb["iters"][b]
        assert torch.equal(x1[0], xb[b])
        c1.close()


def test_kr_run_to_run_bitwise():
    p = make_problem(2, amp=100.0)
    ctx = _ctx([p], 1.0, 0.02, 0.02, 3)
    y = _t(p["y"][None])
    xa, la = ctx.recon(y, 3, eps=1e-4, max_iters=50)
    xb, lb = ctx.recon(y, 3, eps=1e-4, max_iters=50)
    assert la["pcg_iters"] == lb["pcg_iters"] and torch.equal(xa, xb)
    ctx.close()


def test_stage_timers():
    p = make_problem(2)
    y = _t(p["y"][None])
    for pers in (True, False):
        ctx = _ctx([p], 1.0, 0.02, 0.02, 3, persistent=pers)
        x, log = ctx.recon(y, 3, eps=1e-4, max_iters=50, stage_timers=True)
        st = log["stages"]
        assert st is not None, pers
        assert st["pcg_s"] > 0 and st["rhs_s"] > 0 and st["shrink_s"] > 0 and st["init_s"] > 0
        assert st["feedback_s"] == 0.0  # fused into the RHS pass (include/sbpcg.h)
        assert sum(st.values()) <= 1.05 * log["total_ms"] * 1e-3
        assert log["build_s"] > 0
        ctx.close()


def test_kr_in_launch_init_and_host_kspace(monkeypatch):
    """Alg. 1 step 1 inside the persistent launch (kinit: u1, the RSS start and the zero SB state,
    reading a device k-space in place) against the sequence-pass init followed by the launch
    (SBPCG_KR_INIT=0): iteration counts within +-1 and images equal to the fp32 rounding of the
    init transforms; and a host (pinned) k-space against the device one: bitwise equal."""
    ps = batch(2, 1, (256, 256), 12, amp=100.0)
    y = _t(np.stack([p["y"] for p in ps]))
    res = {}
    for mode in ("kinit", "seq", "host"):
        monkeypatch.setenv("SBPCG_KR_INIT", "0" if mode == "seq" else "1")
        ctx = _ctx(ps, 1.0, 0.02, 0.02, 3)
        yy = y.cpu().pin_memory() if mode == "host" else y
        x, log = ctx.recon(yy, 4, eps=1e-4, max_iters=50)
        assert log["path"] == "persistent"
        res[mode] = (_np(x), log["pcg_iters"])
        ctx.close()
    assert res["kinit"][1] == res["host"][1] and np.array_equal(res["kinit"][0], res["host"][0])
    for a_, b_ in zip(res["kinit"][1], res["seq"][1]):  # init rounding differs: counts within +-1
        assert abs(a_[0] - b_[0]) <= 1
    assert relerr(res["kinit"][0], res["seq"][0]) <= 1e-4
