"""The paper's preconditioner comparison on the GPU against
the oracle, with the paper's coil model: maps normalised inside the subject's support and zero
outside for a posterior-array-like half ring of coils, so diag(A) is not
constant and the Jacobi preconditioner is a non-trivial diagonal scaling
(VERDICT r01 "What's missing" #6).  Parameter set 1, eps = 1e-3, phantom x1e3
(shrinkage active), at a reduced geometry the oracle runs in seconds (64^2, 8 coils, VD lines
R = 4).  Per-solve iteration counts must match within +-1 for none / Jacobi / circulant (the
tolerance-mode check of SURVEY 8(c)); the images within 1e-2.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import preprocess, problems, sb
from tests.helpers import relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg, normalize_sens


def _support(phantom, grow=2):
    s = np.abs(phantom) > 0
    out = s.copy()
    for dy in range(-grow, grow + 1):
        for dx in range(-grow, grow + 1):
            out |= np.roll(np.roll(s, dy, 0), dx, 1)
    return out.astype(np.uint8)


@pytest.fixture(scope="module")
def support_problem():
    p = synth.problem2d(2, 0, shape=(64, 64), coils=8, amplitude=1e3)
    sens_half = p["sens"][:4]  # half of the ring: a posterior-array-like coil set
    sup = _support(p["phantom"])
    s_or = preprocess.normalize_sens(sens_half, sup)
    s_gpu = normalize_sens(torch.from_numpy(sens_half[None]).to(torch.complex64).cuda(),
                           torch.from_numpy(sup).cuda())[0].cpu().numpy()
    assert relerr(s_gpu, s_or) <= 1e-6
    rss2 = np.sum(np.abs(s_or) ** 2, axis=0)
    assert set(np.unique(np.round(rss2, 12))) <= {0.0, 1.0} and 0 < rss2.mean() < 1
    y = problems.make_kspace(p["phantom"], s_or, p["mask"], p["noise"][:4])
    return dict(sens=s_gpu.astype(np.complex64), mask=p["mask"], y=y)


@pytest.mark.parametrize("pk", [0, 2, 1], ids=["none", "jacobi", "circulant"])
def test_paper_set1_support_masked_counts(support_problem, pk):
    p = support_problem
    mu, lam, gam = synth.PAPER_SET[1]
    n_outer = 8
    ctx = SbPcg(torch.from_numpy(p["sens"][None]).cuda(), torch.from_numpy(p["mask"][None]).cuda(), mu, lam, gam, 3)
    x, log = ctx.recon(torch.from_numpy(p["y"][None]).to(torch.complex64).cuda(), n_outer, eps=1e-3, max_iters=200,
                       precond=pk)
    got = [r[0] for r in log["pcg_iters"]]
    s32 = p["sens"].astype(np.complex128)
    ref, rlog = sb.sb_recon(p["y"].astype(np.complex64).astype(np.complex128), s32, p["mask"], mu, lam, gam, n_outer,
                            1, 3, 1e-3, 200, ["none", "circulant", "jacobi"][pk])
    assert all(abs(a - b) <= 1 for a, b in zip(got, rlog.pcg_iters)), (got, rlog.pcg_iters)
    assert relerr(x[0].cpu().numpy(), ref) <= 1e-2
    ctx.close()


def test_jacobi_differs_from_none_with_support_masked_maps(support_problem):
    # diag(A) = mu f sum|S_hat|^2 + 4 lambda + gamma takes two values here: Jacobi changes the
    # iteration (unlike with sum|S|^2 = 1 everywhere, where it is a pure rescaling)
    p = support_problem
    mu, lam, gam = synth.PAPER_SET[1]
    ctx = SbPcg(torch.from_numpy(p["sens"][None]).cuda(), torch.from_numpy(p["mask"][None]).cuda(), mu, lam, gam, 3)
    b = ctx.adjoint(torch.from_numpy(p["y"][None]).to(torch.complex64).cuda())
    _, s0 = ctx.solve(b, torch.zeros_like(b), eps=1e-6, max_iters=300, precond=0, history=True)
    _, s2 = ctx.solve(b, torch.zeros_like(b), eps=1e-6, max_iters=300, precond=2, history=True)
    h0, h2 = s0["relres_hist"][0], s2["relres_hist"][0]
    k = min(s0["iters"][0], s2["iters"][0], 10)
    assert max(abs(h0[i] - h2[i]) / h0[i] for i in range(1, k)) > 1e-3
    ctx.close()
