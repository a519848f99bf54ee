"""GPU parity of the preprocessing of PAPER.md Methods (k_prep.cu)
against oracle/preprocess.py, and the paper's coil-compression claim (PCG iteration
counts nearly unchanged with half of the coils)."""
import numpy as np
import pytest
import torch

import synth
from oracle import preprocess, problems, sb
from tests.helpers import relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg, coil_compress, normalize_coil_images, normalize_sens


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.complex64).cuda()


def _c32(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def test_normalize_sens_and_coil_images():
    rng = np.random.default_rng(8)
    s = rng.standard_normal((2, 5, 48, 64)) + 1j * rng.standard_normal((2, 5, 48, 64))
    sup = (rng.random((2, 48, 64)) < 0.7).astype(np.uint8)
    g = normalize_sens(_t(s), torch.from_numpy(sup).cuda()).cpu().numpy()
    for b in range(2):
        ref = preprocess.normalize_sens(_c32(s[b]), sup[b])
        assert relerr(g[b], ref) <= 1e-6
        rss = np.sum(np.abs(g[b]) ** 2, axis=0)
        assert np.allclose(rss[sup[b] == 1], 1, atol=1e-5) and np.all(rss[sup[b] == 0] == 0)
    gs = normalize_sens(_t(s), torch.from_numpy(sup[0]).cuda()).cpu().numpy()  # shared support
    assert relerr(gs[1], preprocess.normalize_sens(_c32(s[1]), sup[0])) <= 1e-6
    m = rng.standard_normal(s.shape) + 1j * rng.standard_normal(s.shape)
    gm = normalize_coil_images(_t(m), torch.from_numpy(g).cuda()).cpu().numpy()
    for b in range(2):
        assert relerr(gm[b], preprocess.normalize_coil_images(_c32(m[b]), _c32(g[b]))) <= 1e-5


def test_coil_compress_parity_and_invariants():
    p = synth.problem2d(2, 0, shape=(128, 128), coils=12)
    y = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    yo, so, ev = coil_compress(_t(y[None]), _t(p["sens"][None]), 6)
    A, w = preprocess.compression_matrix(_c32(y), 6)
    assert np.allclose(ev.numpy()[0], w, rtol=1e-5, atol=1e-6 * w[0])
    yo = yo.cpu().numpy()[0].astype(np.complex128)
    G = yo.reshape(6, -1) @ yo.reshape(6, -1).conj().T          # diagonalised covariance
    assert np.allclose(G, np.diag(w[:6]), atol=2e-5 * w[0])
    # eigenvectors are unique up to a phase per virtual coil: compare the projector A^H A
    yref = preprocess.compress(_c32(y), A)
    Pg = np.einsum("kn,km->nm", yo.reshape(6, -1)[:, :64].conj(), yo.reshape(6, -1)[:, :64])
    Pr = np.einsum("kn,km->nm", yref.reshape(6, -1)[:, :64].conj(), yref.reshape(6, -1)[:, :64])
    assert relerr(Pg, Pr) <= 1e-4


def test_coil_compressed_recon_matches_oracle_and_keeps_iterations():
    # config-2 geometry at paper set 1 (the paper's coil-compression experiment keeps half the
    # coils): iteration counts nearly unchanged, images equal the oracle's
    # recon from the oracle-compressed inputs (phase-invariant)
    p = synth.problem2d(2, 0, amplitude=1e3)
    y = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    mu, lam, gam = synth.PAPER_SET[1]
    yo, so, _ = coil_compress(_t(y[None]), _t(p["sens"][None]), 6)
    ctx = SbPcg(so, torch.from_numpy(p["mask"][None]).cuda(), mu, lam, gam, 3)
    xg, log = ctx.recon(yo, 20, eps=1e-3, max_iters=200)
    full = SbPcg(_t(p["sens"][None]), torch.from_numpy(p["mask"][None]).cuda(), mu, lam, gam, 3)
    xf, logf = full.recon(_t(y[None]), 20, eps=1e-3, max_iters=200)
    it_c, it_f = sum(r[0] for r in log["pcg_iters"]), sum(r[0] for r in logf["pcg_iters"])
    assert abs(it_c - it_f) <= 0.2 * it_f, (it_c, it_f)
    A, _ = preprocess.compression_matrix(_c32(y), 6)
    xr, lr = sb.sb_recon(preprocess.compress(_c32(y), A), preprocess.compress(_c32(p["sens"]), A), p["mask"],
                         mu, lam, gam, 20, 1, 3, 1e-3, 200, "circulant")
    assert relerr(xg.cpu().numpy()[0], xr) <= 1e-2
    assert all(abs(a[0] - b) <= 1 for a, b in zip(log["pcg_iters"], lr.pcg_iters))
    ctx.close(), full.close()
