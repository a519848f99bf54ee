"""Oracle parity at the launch shapes bench.py runs (VERDICT r01 "What's weak" #1): the exact
bench shape of config 2 on the kernel-sequence path (K1 with G = 8 coil-group clusters, the
fused one-cluster preconditioner KP_PRE2D), fixed-count SB reconstructions of the full batches
of configs 3 and 4 on sampled slices, and config 5's 192^3 launch shapes (the 16-column
192-row d0 passes k_col<192,16,*>, KP_PRECOND<192,192,8>, the K1P plane matvec
kp_plane<192,192,8>) with a few coils.

Tolerances (BASELINE.json north_star): operators <= 1e-5 relative L2, Lambda <= 1e-6,
fixed-count PCG / SB images <= 1e-3.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import ops, precond, problems, sb
from oracle.pcg import pcg
from tests.helpers import make_problem, relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg

DEV = "cuda"


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.complex64).to(DEV)


def _np(t):
    return t.detach().cpu().numpy().astype(np.complex128)


def _c32(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_config2_bench_shape_sequence_path():
    # B = 1, 256^2, 12 coils: apply_A runs K1 with G = 8 coil-group clusters, apply_Pinv the
    # fused KP_PRE2D cluster kernel; the solve runs K1 (PCG mode) + KP_PRE2D in a CUDA graph
    p = make_problem(2)
    prm = synth.CONFIGS[2].params
    mu, lam, gam = prm.mu, prm.lam, prm.gamma
    ctx = SbPcg(_t(p["sens"][None]), torch.from_numpy(p["mask"][None]).to(DEV), mu, lam, gam, prm.wavelet_levels,
                persistent=False)
    rng = np.random.default_rng(31)
    x = _crandn(rng, 256, 256)
    s32 = _c32(p["sens"])
    ya = _np(ctx.apply_A(_t(x[None])))[0]
    assert relerr(ya, ops.apply_A(_c32(x), s32, p["mask"], mu, lam, gam)) <= 1e-5
    k = precond.build_k(s32, p["mask"], mu, lam, gam)
    assert relerr(ctx.get_k().numpy()[0], k) <= 1e-6
    za = _np(ctx.apply_Pinv(_t(x[None])))[0]
    assert relerr(za, precond.apply_Minv(_c32(x), k)) <= 1e-5
    b = _crandn(rng, 256, 256)
    xs, st = ctx.solve(_t(b[None]), torch.zeros((1, 256, 256), dtype=torch.complex64, device=DEV), eps=0.0,
                       max_iters=15)
    assert ctx.last_path() == "graph" and st["iters"] == [15]
    ref = pcg(lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam), _c32(b), np.zeros((256, 256), complex),
              lambda v: precond.apply_Minv(v, k), 0.0, 15)
    assert relerr(_np(xs)[0], ref.x) <= 1e-3
    ctx.close()


def test_config2_fixed_count_sb_sequence():
    # config 2 at its settings (3-level Haar, mu = 1, lambda = gamma = 0.02), eps = 0, 5 outer x 10
    # CG, on the kernel-sequence path (the persistent path: test_gpu_persistent.py)
    persistent = False
    p = make_problem(2, amp=100.0)
    prm = synth.CONFIGS[2].params
    ctx = SbPcg(_t(p["sens"][None]), torch.from_numpy(p["mask"][None]).to(DEV), prm.mu, prm.lam, prm.gamma,
                prm.wavelet_levels, persistent=persistent)
    xg, log = ctx.recon(_t(p["y"][None]), 5, eps=0.0, max_iters=10)
    assert log["path"] == ("persistent" if persistent else "graph")
    ref, _ = sb.sb_recon(_c32(p["y"]), _c32(p["sens"]), p["mask"], prm.mu, prm.lam, prm.gamma, 5, 1,
                         prm.wavelet_levels, 0.0, 10, "circulant")
    assert relerr(_np(xg)[0], ref) <= 1e-3, relerr(_np(xg)[0], ref)
    ctx.close()


def _full_batch_fixed_count(sens, masks, ys, prm, sample, n_out=5, its=10):
    ctx = SbPcg(torch.from_numpy(np.ascontiguousarray(sens, dtype=np.complex64)).to(DEV),
                torch.from_numpy(masks).to(DEV), prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
    x, log = ctx.recon(torch.from_numpy(np.stack(ys)).to(torch.complex64).to(DEV), n_out, eps=0.0, max_iters=its)
    xs = x.cpu().numpy()
    ctx.close()
    for i in sample:
        assert all(row[i] == its for row in log["pcg_iters"]), (i, [row[i] for row in log["pcg_iters"]])
        m = masks if masks.ndim == 2 else masks[i]
        ref, _ = sb.sb_recon(_c32(ys[i]), _c32(sens[i]), m, prm.mu, prm.lam, prm.gamma, n_out, 1,
                             prm.wavelet_levels, 0.0, its, "circulant")
        assert relerr(xs[i], ref) <= 1e-3, (i, relerr(xs[i], ref))


def test_config3_full_batch_fixed_count_sb():
    # 128 slices x 256^2 x 12 coils in one context (K1 over the batch, the three preconditioner
    # passes, the batched SB update); 5 outer x 10 CG, slices 0 and 127 against the oracle
    spec = synth.CONFIGS[3]
    ps = [synth.problem2d(3, s) for s in range(spec.batch)]
    sens = np.stack([p["sens"] for p in ps]).astype(np.complex64)
    masks = np.stack([p["mask"] for p in ps])
    ys = [problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"]) for p in ps]
    _full_batch_fixed_count(sens, masks, ys, spec.params, [0, spec.batch - 1])


def test_config4_full_batch_fixed_count_sb():
    # 256 readout planes of 256 x 128, 16 coils, shared 2D random mask (K1P with 16-CTA clusters);
    # 5 outer x 10 CG, planes 100 and 173 against the oracle (planes near the volume edge hold
    # no signal: b = 0 there, so those solves stop at once, reading A26)
    spec = synth.CONFIGS[4]
    q = synth.problem_c4(range(spec.batch))
    ys = [problems.make_kspace(q["phantom"][i], q["sens"][i].astype(np.complex128), q["mask"],
                               q["noise"][i].astype(np.complex128)) for i in range(spec.batch)]
    _full_batch_fixed_count(q["sens"], q["mask"], ys, spec.params, [100, 173])


@pytest.fixture(scope="module")
def c5_small_coils():
    """Config 5's geometry (192^3, 2D VD phase-encode mask R = 8 with a 20 x 20 centre, readout
    fully sampled, 3D Haar with 3 levels) with 2 coils: the same kernel instantiations and launch
    shapes as the 32-coil bench run (the d0 passes and plane kernels do not depend on C)."""
    p = synth.problem3d(5, coils=2, dtype=np.complex64)
    p["y"] = problems.make_kspace(p["phantom"].astype(np.complex128), p["sens"].astype(np.complex128), p["mask"],
                                  p["noise"].astype(np.complex128))
    return p


def test_config5_launch_shape_operators(c5_small_coils):
    p = c5_small_coils
    prm = synth.CONFIGS[5].params
    ctx = SbPcg(_t(p["sens"][None]), torch.from_numpy(p["mask"][None]).to(DEV), prm.mu, prm.lam, prm.gamma,
                prm.wavelet_levels)
    rng = np.random.default_rng(32)
    x = _crandn(rng, 192, 192, 192)
    s32 = _c32(p["sens"])
    z = _np(ctx.apply_Pinv(_t(x[None])))[0]
    k = precond.build_k(s32, p["mask"], prm.mu, prm.lam, prm.gamma)
    assert relerr(ctx.get_k().numpy()[0], k) <= 1e-6
    assert relerr(z, precond.apply_Minv(_c32(x), k)) <= 1e-5
    ya = _np(ctx.apply_A(_t(x[None])))[0]
    assert relerr(ya, ops.apply_A(_c32(x), s32, p["mask"], prm.mu, prm.lam, prm.gamma)) <= 1e-5
    ctx.close()


def test_config5_launch_shape_fixed_count_sb(c5_small_coils):
    # 1 outer x 5 CG (SURVEY 8(c) "config 5"): RSS init, the RESID prelude, 5 PCG iterations
    # through the 192-row d0 passes and KP_PRECOND, the 3D shrink step
    p = c5_small_coils
    prm = synth.CONFIGS[5].params
    ctx = SbPcg(_t(p["sens"][None]), torch.from_numpy(p["mask"][None]).to(DEV), prm.mu, prm.lam, prm.gamma,
                prm.wavelet_levels)
    xg, log = ctx.recon(_t(p["y"][None]), 1, eps=0.0, max_iters=5)
    assert log["pcg_iters"] == [[5]]
    ref, _ = sb.sb_recon(_c32(p["y"]), _c32(p["sens"]), p["mask"], prm.mu, prm.lam, prm.gamma, 1, 1,
                         prm.wavelet_levels, 0.0, 5, "circulant")
    assert relerr(_np(xg)[0], ref) <= 1e-3, relerr(_np(xg)[0], ref)
    ctx.close()


@pytest.mark.parametrize("spec", ["1", "0"], ids=["spectral", "three-pass"])
def test_spectral_residual_preconditioner_batch(monkeypatch, spec):
    # the spectral-residual preconditioner passes (K1 writes F_0 q / F_0 r0; one row pass with
    # the S_r update and both dot products; one column pass) on a batch whose K1 CTAs hold whole
    # columns (G = 1); the fused one-cluster preconditioner is switched off so the batch takes
    # the pass sequence.  Against the oracle, and against the three-pass preconditioner.
    monkeypatch.setenv("SBPCG_PRE2D", "0")
    monkeypatch.setenv("SBPCG_SPEC", spec)
    from tests.helpers import batch
    ps = batch(1, 20, (64, 64), 4, amp=100.0)
    mu, lam, gam = 1.0, 0.05, 0.05
    sens = np.stack([p["sens"] for p in ps])
    masks = np.stack([p["mask"] for p in ps])
    ctx = SbPcg(_t(sens), torch.from_numpy(masks).to(DEV), mu, lam, gam, 1, persistent=False)
    rng = np.random.default_rng(33)
    bvec = np.stack([_crandn(rng, 64, 64) for _ in ps])
    x0 = np.zeros_like(bvec)
    x, st = ctx.solve(_t(bvec), _t(x0), eps=0.0, max_iters=12, history=True)
    xt, stt = ctx.solve(_t(bvec), _t(x0), eps=1e-5, max_iters=100)
    y = np.stack([p["y"] for p in ps])
    xr, log = ctx.recon(_t(y), 3, eps=0.0, max_iters=8)
    for bi in (0, 13):
        p = ps[bi]
        s32 = _c32(p["sens"])
        k = precond.build_k(s32, p["mask"], mu, lam, gam)
        A = lambda v: ops.apply_A(v, s32, p["mask"], mu, lam, gam)  # noqa: E731
        Mi = lambda v: precond.apply_Minv(v, k)  # noqa: E731
        ref = pcg(A, _c32(bvec[bi]), x0[bi], Mi, 0.0, 12)
        assert relerr(_np(x)[bi], ref.x) <= 1e-3
        np.testing.assert_allclose(st["relres_hist"][bi][:13], ref.relres, rtol=2e-2, atol=1e-6)
        reft = pcg(A, _c32(bvec[bi]), x0[bi], Mi, 1e-5, 100)
        assert abs(stt["iters"][bi] - reft.iters) <= 1 and relerr(_np(xt)[bi], reft.x) <= 1e-3
        refr, _ = sb.sb_recon(_c32(p["y"]), s32, p["mask"], mu, lam, gam, 3, 1, 1, 0.0, 8, "circulant")
        assert relerr(_np(xr)[bi], refr) <= 1e-3
    ctx.close()
