#!/usr/bin/env python
"""bench.py — PCG iterations/s and SB reconstruction time on B200 (BASELINE.json metric).

One STEP = one pass of the whole hot path on one batch of synthetic input:
  Lambda build + Split Bregman reconstruction (a1-a13): 20 outer
  iterations, each a device-driven PCG solve (tol 1e-4, max 50) with the circulant
  preconditioner, shrink/Bregman updates and data feedback.
Default workload: BASELINE.json configs[1] ("config 2"): 256x256, 12 coils, VD line mask
R=4 with a 24-line centre, TV + 3-level Haar, mu=1, lambda=gamma=0.02.  Inputs are seeded
synthetic phantoms/coil maps/masks (synth/), k-space formed on the GPU with the library's
own encoder (sb_encode).

Multi-GPU: `--gpus N` without a torchrun environment relaunches itself under
torch.distributed.run with N ranks (one per GPU, NCCL).  The main line is config 2 as
replicas (weak scaling: one slice per rank, no collective); the `extra` object adds config 3
sharded by slice (128 slices over the ranks, no collective), config 4 sharded by readout plane
and config 5 sharded by coil (one NCCL all-reduce per matvec), each timed as the max over
ranks (`--no-extra` skips them).

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle instead (bounded
sample per step on all host cores).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = ("PCG iters/s & SB recon time (256²×12-coil); "
          "HBM GB/s as fraction of B200 peak")
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precond", type=int, default=1, choices=[0, 1, 2], help="0 none, 1 circulant, 2 Jacobi")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-persistent", action="store_true", help="force the kernel-sequence path")
    ap.add_argument("--std-pcg", action="store_true", help="persistent kernel: standard PCG recurrences")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--full-cpu-baseline", action="store_true",
                    help="oracle baseline with complete SB reconstructions (BASELINE.md §3; minutes)")
    ap.add_argument("--no-extra", action="store_true", help="skip the configs 3-5 extra measurements")
    ap.add_argument("--extra", default="3,4,5", help="configs measured in the extra object")
    ap.add_argument("--slices", type=int, default=0, help="override problems per rank")
    return ap.parse_args()


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run with N ranks
    (rendezvous on 127.0.0.1) and pass its output through; rank 0 prints the JSON line."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def workload(cfg: int, ws: int, rank: int, slices_override: int):
    """(spec, problems on this rank, first problem index).  Configs 3-4 shard their batch over
    the ranks (strong scaling); configs 1-2 give every rank its own slice (weak scaling);
    config 5 is one volume (coil-sharded when ws > 1)."""
    spec = synth.CONFIGS[cfg]
    if cfg in (3, 4):
        per = slices_override or max(1, spec.batch // ws)
        first = rank * per
    else:
        per = slices_override or 1
        first = rank * per
    return spec, per, first


def make_inputs(cfg, first, per):
    if cfg == 5:  # one fully 3D problem (synth.problem3d), complex64 to bound host memory
        p = synth.problem3d(5, dtype=np.complex64)
        return p["phantom"][None], p["sens"][None], p["mask"][None], p["noise"][None]
    if cfg == 4:  # readout planes of one 3D volume, shared 2D mask (synth.problem_c4)
        p = synth.problem_c4(range(first, first + per))
        return p["phantom"], p["sens"], p["mask"], p["noise"]
    ps = [synth.problem2d(cfg, s) for s in range(first, first + per)]
    phantom = np.stack([p["phantom"] for p in ps])
    sens = np.stack([p["sens"] for p in ps])
    mask = np.stack([p["mask"] for p in ps])
    noise = np.stack([p["noise"] for p in ps])
    return phantom, sens, mask, noise


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out, _ = self.p.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_pipes(cfg):
    """FP32-issue co-limit of the dominant kernel: FMA-pipe busy %, issue-active %,
    warps-active % from the last ncu metric pass (tools/gpu_pipes.sh -> profiles/ncu_pipes.json)."""
    path = os.path.join(ROOT, "profiles", "ncu_pipes.json")
    if os.path.exists(path):
        d = json.load(open(path)).get(f"config{cfg}")
        if d:
            return {k: d[k] for k in ("kernel", "fma_pipe_busy_pct", "issue_active_pct", "warps_active_pct",
                                      "fma_inst_share", "source")}
    return None


def load_traffic(cfg):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get(f"config{cfg}")
    return None


# ---------------------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline): oracle/ as it stands, one process per host core
def _oracle_worker(job):
    """One oracle SB reconstruction (Alg. 1, literal per-coil k-space feedback) of slice s."""
    cfg, s, n_outer, precond = job
    from oracle import problems, sb
    spec = synth.CONFIGS[cfg]
    prm = spec.params
    if cfg == 4:
        q = synth.problem_c4([s])
        p = dict(phantom=q["phantom"][0], sens=q["sens"][0].astype(np.complex128), mask=q["mask"],
                 noise=q["noise"][0].astype(np.complex128))
    else:
        p = synth.problem2d(cfg, s)
    y = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    t = time.perf_counter()
    _, log = sb.sb_recon(y, p["sens"], p["mask"], prm.mu, prm.lam, prm.gamma, n_outer, 1,
                         prm.wavelet_levels, prm.eps, prm.max_iters, ["none", "circulant", "jacobi"][precond])
    return time.perf_counter() - t, int(sum(log.pcg_iters))


def _oracle_pool(jobs):
    """Run oracle jobs on all host cores (one single-threaded numpy process per core);
    returns (wall seconds, total PCG iterations, per-job seconds, processes)."""
    import multiprocessing as mp
    env_keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in env_keys}
    for k in env_keys:
        os.environ[k] = "1"
    procs = min(len(jobs), os.cpu_count() or 1)
    try:
        ctx = mp.get_context("spawn")
        t = time.perf_counter()
        with ctx.Pool(procs) as pool:
            res = pool.map(_oracle_worker, jobs)
        wall = time.perf_counter() - t
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return wall, sum(r[1] for r in res), [r[0] for r in res], procs


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_3d(cfg, precond):
    """Config 5: one oracle PCG iteration at 192^3 x 32 coils is minutes of numpy, so the bounded
    sample times ONE coil's data-term pair E_c^H E_c p plus the regulariser and one M^{-1}
    application and extrapolates t_iter = C * t_coil + t_rest (labelled as such); the coil
    terms are independent, so on P cores t_iter = ceil(C/P) t_coil + t_rest."""
    from oracle import ops, precond as opre
    p = synth.problem3d(cfg, dtype=np.complex64)
    spec = synth.CONFIGS[cfg]
    prm = spec.params
    s0 = p["sens"][:1].astype(np.complex128)
    x = p["phantom"].astype(np.complex128)
    t = time.perf_counter()
    ops.data_normal(x, s0, p["mask"])
    t_coil = time.perf_counter() - t
    t = time.perf_counter()
    ops.tv_normal(x)
    t_reg = time.perf_counter() - t
    t_pre = 0.0
    if precond:
        kd = opre.k_d_closed(spec.shape)
        k = prm.mu * 0.5 + prm.lam * kd + prm.gamma  # stand-in diagonal: M^{-1} cost only
        t = time.perf_counter()
        opre.apply_Minv(x, k)
        t_pre = time.perf_counter() - t
    cores = os.cpu_count() or 1
    t_iter = math.ceil(spec.coils / cores) * t_coil + t_reg + t_pre
    return {"value": 1.0 / t_iter, "unit": "PCG iters/s", "cores": cores, "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"extrapolated: 1 coil data-term pair ({t_coil:.1f} s) x ceil({spec.coils}/{cores} cores) + "
                      f"regulariser ({t_reg:.1f} s) + one M^-1 ({t_pre:.1f} s) = {t_iter:.0f} s per PCG "
                      f"iteration at 192^3 (numpy fp64, own FFT; coil terms in parallel over the cores)"}


def cpu_baseline(cfg, precond, full=False):
    """The oracle on all host cores, one independent slice per core (single-threaded numpy
    processes): by default a bounded sample of 2 SB outer iterations per slice (~10-15 s);
    `full` (--full-cpu-baseline) runs complete SB reconstructions (~100 s for
    config 2).  Config 5 extrapolates from one coil's data-term pair."""
    if cfg == 5:
        return cpu_baseline_3d(cfg, precond)
    spec = synth.CONFIGS[cfg]
    cores = os.cpu_count() or 1
    n_outer = spec.params.n_outer if full else 2
    jobs = [(cfg, s, n_outer, precond) for s in range(cores)]
    wall, its, per, procs = _oracle_pool(jobs)
    return {"value": its / wall, "unit": "PCG iters/s", "cores": procs, "kind": "oracle", "cpu": cpu_model(),
            "sb_recon_s": statistics.median(per),
            "sample": f"{procs} independent slices in parallel, one single-threaded numpy fp64 process per core, "
                      f"{n_outer} SB outer iterations each ({'full reconstruction' if n_outer == spec.params.n_outer else 'partial'}); "
                      f"{its} PCG iterations in {wall:.1f} s wall; median per-slice sb_recon {statistics.median(per):.1f} s"}


def run_reference(args):
    """CPU oracle arm (oracle/ as it stands) on the box's host cores; each step runs one SB
    outer iteration of one slice per core (a bounded sample of the same workload)."""
    ws, rank, _ = dist_setup()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            return
    spec, per, first = workload(args.config, 1, 0, args.slices)
    if args.config == 5:
        cb = cpu_baseline_3d(args.config, args.precond)
        value = cb["value"]
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": "PCG iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded phantom/coils/mask)",
            "config": {"workload": spec.name, "sample": cb["sample"]},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "PCG iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
    else:
        cores = os.cpu_count() or 1
        jobs = [(args.config, s, 1, args.precond) for s in range(cores)]
        for _ in range(min(args.warmup, 1)):
            _oracle_pool(jobs)
        tot_t, tot_it = 0.0, 0
        for _ in range(args.steps):
            wall, its, _, procs = _oracle_pool(jobs)
            tot_t += wall
            tot_it += its
        value = tot_it / tot_t
        sample = f"1 SB outer iteration of {cores} independent slices per step, one numpy process per core"
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": "PCG iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded phantom/coils/mask)",
            "config": {"workload": spec.name, "sample": sample,
                       "mask": "VD lines" if spec.mask_kind == "lines" else "random2d"},
            "cpu_baseline": {"value": value, "unit": "PCG iters/s", "cores": cores, "kind": "oracle",
                             "cpu": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": "PCG iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------------------
def kspace_gpu(ctx, spec, phantom, mask_d, noise, dev, coil_group=None):
    """y = R (F S x + sigma n), sigma = 0.005 max|F S x| (reading A21; A29 for a shared
    mask), formed on the GPU with the library's own encoder (input synthesis, untimed)."""
    import torch
    x_d = torch.from_numpy(phantom).to(torch.complex64).to(dev)
    yfull = ctx.encode(x_d, full=True)
    if spec.mask_shared:  # reading A29: one noise level over the whole hybrid (x0, k1, k2) data
        sigma = 0.005 * yfull.abs().amax()
        mask_c = mask_d.to(torch.complex64)[None, None]
    else:
        sigma = 0.005 * yfull.abs().flatten(1).amax(dim=1).view((-1,) + (1,) * (yfull.dim() - 1))
        mask_c = mask_d.to(torch.complex64).unsqueeze(1)
    if coil_group is not None:  # coil shards: the max runs over every rank's coils
        coil_group.all_reduce(sigma, op=coil_group.ReduceOp.MAX)
    yfull.add_(sigma * torch.from_numpy(noise).to(torch.complex64).to(dev))
    yfull.mul_(mask_c)
    return yfull


def bench_config(cfg, args, ws, rank, dist, dev, main):
    """Time `steps` whole-hot-path steps of config `cfg` on this rank (max over ranks); main =
    the headline line (clock sampling, e2e); otherwise a short extra measurement."""
    import torch
    from paper_1710_01758_b200 import SbPcg

    steps = args.steps if main else min(args.steps, 3)
    warmup = args.warmup if main else 3
    spec, per, first = workload(cfg, ws, rank, args.slices if main else 0)
    prm = spec.params
    phantom, sens, mask, noise = make_inputs(cfg, first, per)
    coil_mode = cfg == 5 and ws > 1
    comm = None
    if coil_mode:  # config 5 over G GPUs: coil shards + one all-reduce per matvec
        from paper_1710_01758_b200 import SbComm, coil_shard
        c0, c1 = coil_shard(spec.coils, rank, ws)
        sens, noise = np.ascontiguousarray(sens[:, c0:c1]), np.ascontiguousarray(noise[:, c0:c1])
        obj = [SbComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = SbComm(obj[0], rank, ws)
    sens_d = torch.from_numpy(sens).to(torch.complex64).to(dev)
    mask_d = torch.from_numpy(mask).to(dev)
    ctx = SbPcg(sens_d, mask_d, prm.mu, prm.lam, prm.gamma, prm.wavelet_levels, comm=comm,
                persistent=not args.no_persistent)
    if args.std_pcg:
        ctx.set_pcg_cg(False)
    y_d = kspace_gpu(ctx, spec, phantom, mask_d, noise, dev, dist if coil_mode else None)
    del phantom, noise
    out = torch.empty((per,) + tuple(spec.shape), dtype=torch.complex64, device=dev)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    use_graph = not args.no_graph

    # config 4 on one GPU: the step starts from the 3D acquisition -- k-space [C][D0][D1][D2] with
    # the fully sampled readout d0 -- and decouples it into the 256 plane problems with the
    # library's readout decoupling (sb_readout_decouple, a unitary 1D IFFT along d0); the 3D
    # k-space is synthesised once from the plane data by a forward 1D FFT (input synthesis)
    y3 = None
    if cfg == 4 and ws == 1:
        from paper_1710_01758_b200 import readout_decouple
        y3 = torch.fft.fft(y_d.permute(1, 0, 2, 3), dim=1, norm="ortho").contiguous()

    def step():
        yv = y_d
        if y3 is not None:
            yv, _ = readout_decouple(y3)
        ctx.build_precond()
        _, log = ctx.recon(yv, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters,
                           precond=args.precond, use_graph=use_graph, out=out)
        return log

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    clock = ClockSampler(dev.index) if main else None
    if clock:
        clock.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    total_ms, iters, step_ms = 0.0, 0, []
    l0 = ctx.launches()
    log = None
    for _ in range(steps):
        flush.fill_(1.0)  # L2 flush between timed steps (inputs < L2 at config 2)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        log = step()
        e1.record(st)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        total_ms += step_ms[-1]
        iters += sum(sum(r) for r in log["pcg_iters"])
    torch.cuda.synchronize()
    launches = ctx.launches() - l0
    path = log["path"]
    stages = log["stages"]
    build_s = log["build_s"]
    if dist:
        dist.barrier()
    clocks = None
    if clock:
        # keep the GPU loaded ~1.5 s so the sampler sees the steady state: a step count that
        # every rank agrees on (the coil-sharded mode runs collectives inside each step)
        n_probe = max(1, int(math.ceil(1500.0 / max(total_ms / steps, 1e-3))))
        if dist:
            t = torch.tensor([n_probe], device=dev, dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            n_probe = int(t.item())
        for _ in range(min(n_probe, 2000)):
            step()
        torch.cuda.synchronize()
        clocks = clock.stop()

    # max over ranks of the device time; sum of work (coil mode: every rank iterates on the
    # same single problem, so the iterations are not summed)
    t_max, it_sum = total_ms, iters
    if dist:
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        ii = torch.tensor([iters], device=dev, dtype=torch.float64)
        dist.all_reduce(ii, op=dist.ReduceOp.MAX if coil_mode else dist.ReduceOp.SUM)
        it_sum = int(ii.item())
    value = it_sum / (t_max / 1e3)

    # ---- per-PCG-iteration rate and HBM fraction (north star: ">= 60% of the B200 HBM roofline
    # per PCG iteration"): fixed-count solves (eps = 0) with K = 10 and 50 iterations,
    # t_iter = (t50 - t10) / 40 (the prelude/exit of a solve cancel), best of 3;
    # bytes per iteration = B_iter of SURVEY 8(a), 8N(C+10) + 4N + mask bytes, per problem
    pk, peak_kind = peaks()
    nimg = int(np.prod(spec.shape))
    mask_b = 4.0 * spec.shape[0] if spec.mask_kind == "lines" else float(
        np.prod(spec.shape[1:] if len(spec.shape) == 3 else spec.shape))
    coils_here = sens.shape[1]
    b_iter = per * (8.0 * nimg * (coils_here + 10) + 4.0 * nimg + mask_b)
    pcg_iter = None
    if not coil_mode:
        bsolve = ctx.adjoint(y_d)
        x0 = torch.zeros_like(bsolve)

        def t_solve(K):
            best = float("inf")
            for _ in range(3):
                flush.fill_(1.0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                ctx.solve(bsolve, x0, eps=0.0, max_iters=K, precond=args.precond, use_graph=use_graph)
                e1.record(st)
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            return best
        t_solve(10)  # graph capture
        t10, t50 = t_solve(10), t_solve(50)
        t_it = max(t50 - t10, 1e-9) / 40.0 / 1e3  # s
        pcg_iter = {"us_per_iteration": t_it * 1e6, "problem_iters_per_s": per / t_it,
                    "bytes_per_iteration": b_iter, "achieved_gbs": b_iter / t_it / 1e9,
                    "hbm_frac": b_iter / t_it / 1e9 / pk, "path": ctx.last_path(),
                    "method": "fixed-count solves (eps=0) K=10 and K=50, (t50-t10)/40, best of 3, L2 flushed"}

    # ---- dominant-kernel roofline, timed with CUDA events per launch on the context stream:
    # the persistent kernel KR when the step runs it (its algorithmic bytes: B_iter per PCG
    # iteration + the solve prelude and SB step per solve), else the matvec
    # kernel K1 / K1P (eager pass)
    which = 2 if path == "persistent" else 0
    ctx.set_kernel_timing(True)
    for _ in range(max(1, min(steps, 5))):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    k_ms, k_n, k_bytes = ctx.kernel_time(which)
    ctx.set_kernel_timing(False)
    k_avg_s = (k_ms / max(k_n, 1)) / 1e3
    achieved = k_bytes / k_avg_s / 1e9 if k_avg_s > 0 else 0.0
    kname = {2: "k_persist (whole SB recon in one cooperative launch: coil FFT matvec, preconditioner, "
                "PCG scalars, shrink)",
             0: ("k1_matvec (fused coil FFT matvec, line-mask 1D FFTs)" if spec.mask_kind == "lines"
                 else "kp_plane (cluster plane matvec: per-coil 2D FFT via DSMEM)")}[which]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": pk, "unit": "GB/s", "frac": achieved / pk,
                "traffic": load_traffic(cfg) if which == 0 else load_traffic(f"{cfg}_kr"),
                "peak_kind": peak_kind, "kernel": kname, "kernel_avg_us": k_avg_s * 1e6,
                "kernel_launches_timed": k_n, "alg_bytes_per_launch": k_bytes,
                "fp32_colimit": load_pipes(cfg)}

    res = {"value": value, "ms_per_step": t_max / steps, "steps": steps, "warmup": warmup,
           "problems_per_gpu": per, "pcg_iters_per_step": it_sum / steps / (1 if coil_mode else ws),
           "path": path, "step_ms": [round(t, 3) for t in step_ms], "pcg_iteration": pcg_iter,
           "roofline": roofline, "gpu_launches": int(launches), "clocks": clocks,
           "stages_s_per_step": stages, "lambda_build_s": build_s,
           "parallelism": (f"coil-sharded x{ws} (NCCL all-reduce per matvec)" if coil_mode
                           else (f"slice-sharded x{ws}" if ws > 1 and cfg in (3, 4)
                                 else (f"replicas x{ws}" if ws > 1 else "1 GPU")))}

    # ---- e2e: public API with HOST (pinned) buffers, copies inside the timed region
    if main and not args.no_e2e:
        sens_h = torch.from_numpy(sens).to(torch.complex64).pin_memory()
        mask_h = torch.from_numpy(mask).pin_memory()
        y_h = y_d.cpu().pin_memory()
        x_h = torch.empty((per,) + tuple(spec.shape), dtype=torch.complex64).pin_memory()
        # one context for the geometry (as a user would keep it); every step uploads that
        # step's coil maps (+ Lambda rebuild) and k-space from pinned host memory and reads
        # the image back (sb_pcg_update_sens + sb_recon with host pointers)
        c2 = SbPcg(sens_h, mask_h, prm.mu, prm.lam, prm.gamma, prm.wavelet_levels, comm=comm,
                   persistent=not args.no_persistent)
        if args.std_pcg:
            c2.set_pcg_cg(False)

        def e2e_step():
            c2.update_sens(sens_h)
            _, lg = c2.recon(y_h, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters,
                             precond=args.precond, use_graph=use_graph, out=x_h)
            return lg
        for _ in range(min(args.warmup, 3)):
            e2e_step()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_it = 0
        for _ in range(steps):
            lg = e2e_step()
            e_it += sum(sum(r) for r in lg["pcg_iters"])
        torch.cuda.synchronize()
        e_dt = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([e_dt, e_it], device=dev, dtype=torch.float64)
            mx = tt.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
            e_dt, e_it = float(mx[0].item()), float((mx if coil_mode else tt)[1].item())
        c2.close()
        h2d = sens_h.numel() * 8 + y_h.numel() * 8
        res["e2e"] = {"value": e_it / e_dt, "unit": "PCG iters/s", "h2d_bytes_per_step": int(h2d),
                      "d2h_bytes_per_step": int(x_h.numel() * 8), "ms_per_step": 1e3 * e_dt / steps}
    ctx.close()
    if comm is not None:
        comm.close()
    del sens_d, y_d, out, flush
    torch.cuda.empty_cache()
    return res, spec


def mask_desc(spec):
    return {"lines": "VD lines R=%d, %d-line centre" % (spec.accel, spec.center),
            "random2d": "shared 2D VD random R=%d, %dx%d centre" % (spec.accel, spec.center, spec.center),
            "pe2d": "2D VD phase-encode R=%d, %dx%d centre, readout fully sampled"
                    % (spec.accel, spec.center, spec.center)}[spec.mask_kind]


def run_ours(args):
    # reading A24: a fixed reduction order for the coil-sharded all-reduce (a pinned ring); set
    # before any NCCL communicator (torch's or the library's) reads the environment
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")
    import torch
    ws, rank, local = dist_setup()
    dist = None
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    main, spec = bench_config(args.config, args, ws, rank, dist, dev, main=True)

    extra = {}
    if not args.no_extra and args.config == 2:
        for c in [int(v) for v in args.extra.split(",") if v.strip()]:
            if c == args.config:
                continue
            try:
                r, sp = bench_config(c, args, ws, rank, dist, dev, main=False)
                extra[f"config{c}"] = {
                    "workload": sp.name, "value": r["value"], "unit": "PCG iters/s",
                    "ms_per_step": r["ms_per_step"], "steps": r["steps"], "warmup": r["warmup"],
                    "scaling": "strong" if c in (3, 4, 5) and ws > 1 else "weak",
                    "parallelism": r["parallelism"], "problems_per_gpu": r["problems_per_gpu"],
                    "pcg_iters_per_step": r["pcg_iters_per_step"], "path": r["path"],
                    "pcg_iteration": r["pcg_iteration"], "roofline": r["roofline"],
                    "stages_s_per_step": r["stages_s_per_step"], "lambda_build_s": r["lambda_build_s"],
                    "gpu_launches": r["gpu_launches"], "n_gpus": ws}
            except Exception as e:  # an extra must not lose the main line
                extra[f"config{c}"] = {"error": f"{type(e).__name__}: {e}"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.precond, full=args.full_cpu_baseline)

    if rank == 0:
        prm = spec.params
        line = {
            "metric": METRIC, "value": main["value"], "unit": "PCG iters/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
            "higher_is_better": True, "scaling": "weak" if args.config not in (3, 4, 5) else "strong",
            "vs_baseline": None, "dtype": "c64 (fp32 complex; Lambda built in f64)",
            "data": "synthetic (seeded phantoms, coil maps, masks; k-space by sb_encode)",
            "config": {"workload": spec.name, "problems_per_gpu": main["problems_per_gpu"],
                       "shape": list(spec.shape), "coils": spec.coils, "mask": mask_desc(spec),
                       "mu": prm.mu, "lambda": prm.lam, "gamma": prm.gamma, "n_outer": prm.n_outer,
                       "pcg_eps": prm.eps, "pcg_max_iters": prm.max_iters,
                       "precond": ["none", "circulant", "jacobi"][args.precond],
                       "pcg_iters_per_step": main["pcg_iters_per_step"],
                       "parallelism": main["parallelism"],
                       "sb_recon_ms": main["ms_per_step"], "step_ms": main["step_ms"],
                       "l2": "flushed between timed steps (256 MiB write)",
                       "path": main["path"],
                       "loop": {"persistent": "one cooperative launch per reconstruction (k_persist)",
                                "graph": "CUDA graph, conditional while node",
                                "eager": "eager kernel sequence",
                                "coil-sharded": "coil-sharded kernel sequence"}.get(main["path"], main["path"])},
            "stages_s_per_step": main["stages_s_per_step"],
            "lambda_build_s": main["lambda_build_s"],
            "roofline": main["roofline"],
            "pcg_iteration": main["pcg_iteration"],
            "cpu_baseline": cpu,
            "e2e": main.get("e2e"),
            "gpu_launches": main["gpu_launches"],
            "clocks": main["clocks"],
            "extra": extra or None,
        }
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
