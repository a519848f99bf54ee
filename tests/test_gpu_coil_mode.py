"""Coil-sharded mode (SURVEY 8(e), config 5 over G GPUs) on one GPU: a world-size-1 NCCL
communicator exercises the whole sharded data path (the plane kernel's partial sums in plane
chunks -> per-chunk ncclAllReduce on the comm stream -> epilogue kernel; the loop captured in
CUDA graphs of U iterations, or eager; all-reduced Lambda marginal / u_1 / RSS); results must
equal the unsharded context.  The multi-rank decomposition itself is covered on CPU by
tests/test_coil_shard_gloo.py."""
import numpy as np
import pytest
import torch

import synth
from oracle import problems
from tests.helpers import relerr

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1710_01758_b200 import SbComm, SbPcg


def _ctx(p, comm=None):
    c = SbPcg(torch.from_numpy(p["sens"][None]).to(torch.complex64).cuda(),
              torch.from_numpy(p["mask"][None]).cuda(), 1.0, 0.01, 0.01, 2)
    if comm is not None:
        c.set_comm(comm)
    return c


def test_coil_mode_world1_equals_unsharded():
    p = synth.problem3d(5, shape=(8, 32, 32), coils=4, amplitude=100.0)
    y = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    comm = SbComm(SbComm.unique_id(), 0, 1)
    a, b = _ctx(p), _ctx(p, comm)
    np.testing.assert_allclose(a.get_k().numpy(), b.get_k().numpy(), rtol=1e-12)
    rng = np.random.default_rng(3)
    x = torch.from_numpy((rng.standard_normal((1, 8, 32, 32)) + 1j * rng.standard_normal((1, 8, 32, 32)))
                         .astype(np.complex64)).cuda()
    assert relerr(b.apply_A(x).cpu().numpy(), a.apply_A(x).cpu().numpy()) <= 1e-6
    yt = torch.from_numpy(y[None]).to(torch.complex64).cuda()
    xa, la = a.recon(yt, 3, eps=0.0, max_iters=6)
    xb, lb = b.recon(yt, 3, eps=0.0, max_iters=6)
    assert la["pcg_iters"] == lb["pcg_iters"]
    assert relerr(xb.cpu().numpy(), xa.cpu().numpy()) <= 1e-5
    xa, la = a.recon(yt, 3, eps=1e-4, max_iters=40)
    xb, lb = b.recon(yt, 3, eps=1e-4, max_iters=40)
    assert la["pcg_iters"] == lb["pcg_iters"]
    assert relerr(xb.cpu().numpy(), xa.cpu().numpy()) <= 1e-5
    a.close(), b.close(), comm.close()


@pytest.mark.parametrize("chunks", [1, 3])
@pytest.mark.parametrize("graph", [True, False], ids=["graph", "eager"])
def test_coil_mode_chunked_and_graph(monkeypatch, chunks, graph):
    # comm given at create (sb_pcg_create's comm argument); chunked all-reduce; graphs or eager
    p = synth.problem3d(5, shape=(8, 32, 32), coils=3, amplitude=100.0)
    y = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    monkeypatch.setenv("SBPCG_COIL_CHUNKS", str(chunks))
    monkeypatch.setenv("SBPCG_COIL_UNROLL", "3")
    comm = SbComm(SbComm.unique_id(), 0, 1)
    a = _ctx(p)
    b = SbPcg(torch.from_numpy(p["sens"][None]).to(torch.complex64).cuda(), torch.from_numpy(p["mask"][None]).cuda(),
              1.0, 0.01, 0.01, 2, comm=comm)
    yt = torch.from_numpy(y[None]).to(torch.complex64).cuda()
    for eps, mx in ((0.0, 7), (1e-4, 40)):
        xa, la = a.recon(yt, 3, eps=eps, max_iters=mx)
        xb, lb = b.recon(yt, 3, eps=eps, max_iters=mx, use_graph=graph)
        assert lb["path"] == "coil-sharded"
        assert la["pcg_iters"] == lb["pcg_iters"]
        assert relerr(xb.cpu().numpy(), xa.cpu().numpy()) <= 1e-5
    # the solve entry point through the same path
    rng = np.random.default_rng(4)
    bb = torch.from_numpy((rng.standard_normal((1, 8, 32, 32)) + 1j * rng.standard_normal((1, 8, 32, 32)))
                          .astype(np.complex64)).cuda()
    xa, sa = a.solve(bb, torch.zeros_like(bb), eps=1e-5, max_iters=60)
    xb, sb_ = b.solve(bb, torch.zeros_like(bb), eps=1e-5, max_iters=60, use_graph=graph)
    assert sa["iters"] == sb_["iters"] and relerr(xb.cpu().numpy(), xa.cpu().numpy()) <= 1e-5
    a.close(), b.close(), comm.close()


def test_coil_mode_guards():
    # coil sharding is the 3D mode; Jacobi needs every rank's coils and is rejected there
    from paper_1710_01758_b200 import SbError
    comm = SbComm(SbComm.unique_id(), 0, 1)
    p2 = synth.problem2d(1, 0, shape=(32, 32), coils=2)
    m2 = synth.random_vd_mask2d((32, 32), 4, 4, synth.rng_for(1, 0, 9))
    c2 = SbPcg(torch.from_numpy(p2["sens"][None]).to(torch.complex64).cuda(), torch.from_numpy(m2[None]).cuda(),
               1.0, 0.02, 0.02, 1)
    with pytest.raises(SbError):
        c2.set_comm(comm)
    c2.close()
    p3 = synth.problem3d(5, shape=(8, 32, 32), coils=2)
    c3 = _ctx(p3, comm)
    b = torch.ones((1, 8, 32, 32), dtype=torch.complex64, device="cuda")
    with pytest.raises(SbError):
        c3.solve(b, torch.zeros_like(b), eps=1e-4, max_iters=5, precond=2)
    c3.close(), comm.close()
