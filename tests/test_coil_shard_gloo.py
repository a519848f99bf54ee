"""Host-side logic of the coil-sharded mode on CPU with world_size 2 (gloo): each rank takes
its contiguous coil shard (the rule of paper_1710_01758_b200.coil_shard, mirrored here for the
spawned workers and checked equal to the binding's function below), computes its partial data
term sum_{c in shard} E_c^H E_c x with the oracle, and one all-reduce gives the full operator
 — the decomposition the library's per-matvec NCCL all-reduce relies on; Lambda's
coil marginal decomposes the same way (k is affine in sum_c |F s_c|^2).
The reference for the coil marginal g uses numpy.fft (a library FFT), so this checks the
decomposition, not the library's FFT."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import ops, precond


def coil_shard(coils, rank, world):
    # same rule as paper_1710_01758_b200.sbpcg.coil_shard (test_mirror_equals_binding)
    base, extra = divmod(coils, world)
    c0 = rank * base + min(rank, extra)
    return c0, c0 + base + (1 if rank < extra else 0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = synth.problem3d(5, shape=(8, 16, 16), coils=5)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((8, 16, 16)) + 1j * rng.standard_normal((8, 16, 16))
    c0, c1 = coil_shard(5, rank, world)
    part = ops.data_normal(x, p["sens"][c0:c1], p["mask"])
    t = torch.from_numpy(np.stack([part.real, part.imag]))
    dist.all_reduce(t)
    g = np.sum(np.abs(np.fft.fftn(p["sens"][c0:c1], axes=(1, 2, 3))) ** 2, axis=0)
    tg = torch.from_numpy(g)
    dist.all_reduce(tg)
    if rank == 0:
        full = ops.data_normal(x, p["sens"], p["mask"])
        red = t[0].numpy() + 1j * t[1].numpy()
        gfull = np.sum(np.abs(np.fft.fftn(p["sens"], axes=(1, 2, 3))) ** 2, axis=0)
        out.put((float(np.linalg.norm(red - full) / np.linalg.norm(full)),
                 float(np.linalg.norm(tg.numpy() - gfull) / np.linalg.norm(gfull))))
    dist.destroy_process_group()


def test_coil_shard_partition():
    for C in (1, 5, 12, 32):
        for W in (1, 2, 3, 4, 8):
            if W > C:
                continue
            rs = [coil_shard(C, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == C
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_mirror_equals_binding():
    # the binding loads libsbpcg.so without a GPU (ctypes; no compute call is made)
    from paper_1710_01758_b200 import coil_shard as lib_coil_shard
    for C in (1, 5, 12, 16, 32):
        for W in (1, 2, 3, 4, 8):
            for r in range(W):
                assert coil_shard(C, r, W) == lib_coil_shard(C, r, W)


def test_coil_sharded_data_term_allreduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    mp.start_processes(_worker, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    e_op, e_g = q.get(timeout=60)
    assert e_op <= 1e-12 and e_g <= 1e-12
