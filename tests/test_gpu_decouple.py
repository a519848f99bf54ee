"""K7 readout decoupling (sb_readout_decouple; BASELINE config 4): a 3D acquisition
with a readout-constant mask splits exactly into independent 2D problems on the readout planes
after a unitary 1D IFFT along d0.  Checked against the plain definition of the decoupled
problem computed by the oracle (per-plane 2D encoding of the plane's phantom with the plane's
maps), against the oracle's own 1D IFFT of the 3D k-space, and end to end: the decoupled batch
reconstructed on the GPU vs the oracle's 2D reconstruction of sampled planes."""
import numpy as np
import pytest
import torch

import synth
from oracle import fft, ops, problems, sb
from tests.helpers import relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbPcg, readout_decouple


@pytest.fixture(scope="module")
def vol():
    # config 5's generator at a small shape: 3D phantom, 3D coil maps, (d1, d2) phase-encode mask
    # repeated along the fully sampled readout d0
    return synth.problem3d(5, shape=(16, 32, 16), coils=3, amplitude=100.0)


def test_decouple_equals_definition(vol):
    p = vol
    D0 = p["phantom"].shape[0]
    y3 = problems.make_kspace(p["phantom"], p["sens"], p["mask"], 0 * p["noise"])  # noise-free
    y2, s2 = readout_decouple(torch.from_numpy(y3).to(torch.complex64).cuda(),
                              torch.from_numpy(p["sens"]).to(torch.complex64).cuda())
    y2 = y2.cpu().numpy().astype(np.complex128)
    s2 = s2.cpu().numpy()
    m2 = p["mask"][0]
    y3_32 = y3.astype(np.complex64).astype(np.complex128)
    ref_ifft = np.moveaxis(fft.ifft(y3_32, axis=1) / np.sqrt(D0), 1, 0)  # the oracle's own 1D IFFT
    assert relerr(y2, ref_ifft) <= 1e-5
    # plain definition of plane x's 2D problem: R_12 F_12 (s_c(x) . phantom(x)) (planes at the
    # volume edge hold no signal, so the error is measured against the whole stack)
    ref = np.stack([ops.encode(p["phantom"][x], p["sens"][:, x], m2) for x in range(D0)])
    assert relerr(y2, ref) <= 2e-5
    scale = np.linalg.norm(ref) / np.sqrt(D0)
    assert all(np.linalg.norm(y2[x] - ref[x]) <= 2e-5 * scale for x in range(D0))
    for x in range(D0):
        assert np.array_equal(s2[x], p["sens"][:, x].astype(np.complex64))


def test_decoupled_batch_recon_matches_oracle(vol):
    p = vol
    y3 = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    y2, s2 = readout_decouple(torch.from_numpy(y3).to(torch.complex64).cuda(),
                              torch.from_numpy(p["sens"]).to(torch.complex64).cuda())
    m2 = p["mask"][0]
    mu, lam, gam, L = 1.0, 0.02, 0.02, 2
    ctx = SbPcg(s2, torch.from_numpy(m2).cuda(), mu, lam, gam, L)  # D0 problems, shared mask
    x, log = ctx.recon(y2, 3, eps=0.0, max_iters=8)
    assert log["pcg_iters"][0] == [8] * p["phantom"].shape[0]
    xs = x.cpu().numpy()
    y2n = y2.cpu().numpy().astype(np.complex128)
    s2n = s2.cpu().numpy().astype(np.complex128)
    for xp in (3, 11):
        ref, _ = sb.sb_recon(y2n[xp], s2n[xp], m2, mu, lam, gam, 3, 1, L, 0.0, 8, "circulant")
        assert relerr(xs[xp], ref) <= 1e-3, (xp, relerr(xs[xp], ref))
    ctx.close()
