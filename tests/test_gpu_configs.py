"""Full-size GPU parity at BASELINE.json's configs, in the launch configuration bench.py times
(whole batch in one context), on outputs the oracle can compute one by one (sampled slices /
planes) or via properties that hold at any size.

Tolerance-mode recon (SURVEY 8(c) "tolerance mode"): per-solve iteration counts within +-1
and the image within 1e-2 (one stop-iteration difference moves the image ~2e-3).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import ops, problems, sb
from tests.helpers import relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg

DEV = "cuda"


def _c32(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _recon_check(sens, masks, phantoms, noises, prm, sample, n_out=4):
    """Full-batch GPU recon (oracle k-space) vs the oracle on the sampled problems."""
    B = sens.shape[0]
    ys = []
    for i in range(B):
        m = masks if masks.ndim == 2 else masks[i]
        ys.append(problems.make_kspace(phantoms[i], sens[i].astype(np.complex128), m, noises[i].astype(np.complex128)))
    ctx = SbPcg(torch.from_numpy(np.ascontiguousarray(sens, dtype=np.complex64)).to(DEV),
                torch.from_numpy(masks).to(DEV), prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
    x, log = ctx.recon(torch.from_numpy(np.stack(ys)).to(torch.complex64).to(DEV), n_out, eps=prm.eps,
                       max_iters=prm.max_iters)
    its = np.array(log["pcg_iters"])
    xs = x.cpu().numpy()
    ctx.close()
    for i in sample:
        m = masks if masks.ndim == 2 else masks[i]
        xr, lg = sb.sb_recon(_c32(ys[i]), sens[i].astype(np.complex128), m, prm.mu, prm.lam, prm.gamma, n_out, 1,
                             prm.wavelet_levels, prm.eps, prm.max_iters, "circulant")
        assert all(abs(a - b) <= 1 for a, b in zip(its[:, i], lg.pcg_iters)), (i, its[:, i], lg.pcg_iters)
        assert relerr(xs[i], xr) <= 1e-2, (i, relerr(xs[i], xr))


def test_config3_full_batch_tolerance_mode():
    spec = synth.CONFIGS[3]
    ps = [synth.problem2d(3, s) for s in range(spec.batch)]
    sens = np.stack([p["sens"] for p in ps]).astype(np.complex64)
    masks = np.stack([p["mask"] for p in ps])
    _recon_check(sens, masks, [p["phantom"] for p in ps], [p["noise"] for p in ps], spec.params,
                 [0, 61, spec.batch - 1])


def test_config4_full_batch_tolerance_mode():
    spec = synth.CONFIGS[4]
    q = synth.problem_c4(range(spec.batch))
    _recon_check(q["sens"], q["mask"], q["phantom"], q["noise"], spec.params, [0, 97, spec.batch - 1])


def test_config5_full_size_sampled_planes():
    # 192^3 x 32 coils.  With a readout-constant mask the data term is exactly per d0 plane
    # (F_3 = F_0 (x) F_12 unitary, R = I_0 (x) R_12), so A p at plane x is
    #   mu sum_c conj(s_c(x)) F_12^H R_12 F_12 (s_c(x) p(x)) + lambda (L_3D p)(x) + gamma p(x),
    # which the oracle computes plane by plane (2D data term + its own 3D Laplacian).
    spec = synth.CONFIGS[5]
    prm = spec.params
    p = synth.problem3d(5, dtype=np.complex64)
    ctx = SbPcg(torch.from_numpy(p["sens"][None]).to(DEV), torch.from_numpy(p["mask"][None]).to(DEV),
                prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
    rng = np.random.default_rng(21)
    x = (rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape)).astype(np.complex64)
    xt = torch.from_numpy(x[None]).to(DEV)
    ya = ctx.apply_A(xt)[0].cpu().numpy()
    lap = ops.tv_normal(x.astype(np.complex128))
    for xp in (0, 77, spec.shape[0] - 1):
        dn = ops.data_normal(x[xp].astype(np.complex128), p["sens"][:, xp].astype(np.complex128), p["mask"][xp])
        ref = prm.mu * dn + prm.lam * lap[xp] + prm.gamma * x[xp]
        assert relerr(ya[xp], ref) <= 1e-5, (xp, relerr(ya[xp], ref))
    # invariants at full size: A Hermitian; M^{-1} Hermitian; k >= gamma; mean(k_c) = sampled
    # fraction f when sum_c |s_c|^2 = 1 (SURVEY 8(c) full-size invariants)
    u = (rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape)).astype(np.complex64)
    ut = torch.from_numpy(u[None]).to(DEV)
    au = ctx.apply_A(ut)[0].cpu().numpy().astype(np.complex128)
    lhs = np.vdot(u.astype(np.complex128), ya.astype(np.complex128))
    rhs = np.vdot(au, x.astype(np.complex128))
    assert abs(lhs - rhs) <= 1e-5 * np.linalg.norm(u) * np.linalg.norm(ya)
    zu = ctx.apply_Pinv(ut)[0].cpu().numpy().astype(np.complex128)
    zx = ctx.apply_Pinv(xt)[0].cpu().numpy().astype(np.complex128)
    assert abs(np.vdot(x.astype(np.complex128), zu) - np.vdot(zx, u.astype(np.complex128))) <= \
        1e-5 * np.linalg.norm(x) * np.linalg.norm(zu)
    k = ctx.get_k()[0].numpy()
    assert k.min() >= prm.gamma * (1 - 1e-12)
    from oracle.precond import k_d_closed
    kc = (k - prm.lam * k_d_closed(spec.shape) - prm.gamma) / prm.mu
    f = p["mask"].mean()
    assert abs(kc.mean() - f) <= 1e-6 * f
    ctx.close()
