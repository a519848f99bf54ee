"""Host-side logic on CPU: slice sharding of the batched configs over ranks (gloo, world 2),
and the isolation of the product path (no oracle imports; no CPU fallback)."""
import os
import shutil
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _slices_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import bench
    out = {}
    for cfg in (2, 3, 4):
        spec, per, first = bench.workload(cfg, world, rank, 0)
        mine = torch.zeros(max(spec.batch, world), dtype=torch.int64)
        mine[first:first + per] = 1
        dist.all_reduce(mine)
        out[cfg] = (per, mine.tolist())
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_slice_sharding_partitions_each_batch_world2():
    # configs 3-4: contiguous slice ranges, every slice on exactly one rank, no
    # data-path collective; config 2 (replicas only): one independent slice per rank
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 200
    mp.start_processes(_slices_worker, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    out = q.get(timeout=60)
    assert out[3][0] == 64 and all(v == 1 for v in out[3][1])
    assert out[4][0] == 128 and all(v == 1 for v in out[4][1])
    assert out[2][0] == 1 and out[2][1] == [1, 1]


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1710_01758_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn


def test_binding_fails_loudly_without_the_library(tmp_path):
    # a copy of the package without libsbpcg.so: using the compute path must raise, not fall
    # back to anything on the CPU
    dst = tmp_path / "paper_1710_01758_b200"
    shutil.copytree(os.path.join(ROOT, "paper_1710_01758_b200"), dst,
                    ignore=shutil.ignore_patterns("*.so", "build_obj", "csrc", "__pycache__"))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_1710_01758_b200 as p\n"
            "try:\n    p.SbPcg\nexcept ImportError as e:\n    print('RAISED', e)\n") % str(tmp_path)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert "RAISED" in r.stdout and "libsbpcg.so not built" in r.stdout, r.stdout + r.stderr


def test_reference_arm_under_torchrun_world2_prints_one_line():
    # `bench.py --impl reference` launched the way the driver launches N > 1: rank 0 alone runs
    # the oracle and prints ONE JSON line; the other rank exits 0 without work (config 1, the
    # small case, so the CPU suite stays short)
    import json
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["unit"] == "PCG iters/s"
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
