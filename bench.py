#!/usr/bin/env python
"""bench.py — PCG iterations/s and SB reconstruction time on B200 (BASELINE.json metric).

One STEP = one pass of the whole hot path on one batch of synthetic input:
  Lambda build + Split Bregman reconstruction (a1-a13): 20 outer
  iterations, each a device-driven PCG solve (tol 1e-4, max 50) with the circulant
  preconditioner, shrink/Bregman updates and data feedback.
Default workload: BASELINE.json configs[1] ("config 2"): 256x256, 12 coils, VD line mask
R=4 with a 24-line centre, TV + 3-level Haar, mu=1, lambda=gamma=0.02.  Inputs are seeded
synthetic phantoms/coil maps/masks (synth/), k-space formed on the GPU with the library's
own encoder (sb_encode).  With --gpus N (torchrun), each rank reconstructs its own
independent slice (weak scaling, no data-path collective).

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle instead
(bounded sample per step).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = synth_metric = ("PCG iters/s & SB recon time (256²×12-coil); "
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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slices", type=int, default=0, help="override problems per rank")
    return ap.parse_args()


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(cfg: int, ws: int, rank: int, slices_override: int):
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


def load_traffic(cfg):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get(f"config{cfg}")
    return None


# ---------------------------------------------------------------------------------------
def run_reference(args):
    """CPU oracle arm (oracle/ as it stands), bounded sample per step: one SB outer iteration
    (Alg. 1 steps 4-15, literal per-coil k-space feedback) of the same workload."""
    ws, rank, _ = dist_setup()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            return
    spec, per, first = workload(args.config, 1, 0, args.slices)
    prm = spec.params
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
        return
    from oracle import sb
    p, y = oracle_problem(args.config, first)

    def sample():
        t = time.perf_counter()
        x, log = sb.sb_recon(y, p["sens"], p["mask"], prm.mu, prm.lam, prm.gamma, 1, 1,
                             prm.wavelet_levels, prm.eps, prm.max_iters,
                             ["none", "circulant", "jacobi"][args.precond])
        return time.perf_counter() - t, sum(log.pcg_iters)

    for _ in range(args.warmup):
        sample()
    tot_t, tot_it = 0.0, 0
    for _ in range(args.steps):
        dt, it = sample()
        tot_t += dt
        tot_it += it
    value = tot_it / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "PCG iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded phantom/coils/mask)",
        "config": {"workload": spec.name, "sample": "1 SB outer iteration per step (oracle)",
                   "mask": "VD lines" if spec.mask_kind == "lines" else "random2d"},
        "cpu_baseline": {"value": value, "unit": "PCG iters/s", "cores": 1, "kind": "oracle",
                         "sample": "1 SB outer iteration of slice 0 per step"},
        "e2e": {"value": value, "unit": "PCG iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def oracle_problem(cfg, s):
    """One problem of the workload for the oracle arm: (inputs, oracle k-space y)."""
    from oracle import problems
    if cfg == 4:
        q = synth.problem_c4([s])
        p = dict(phantom=q["phantom"][0], sens=q["sens"][0].astype(np.complex128), mask=q["mask"],
                 noise=q["noise"][0].astype(np.complex128))
    else:
        p = synth.problem2d(cfg, s)
    return p, problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])


def cpu_baseline_3d(cfg, precond):
    """Config 5: one oracle PCG iteration at 192^3 x 32 coils is ~7 min of single-thread numpy
    (64 own-FFT 3D transforms), so the bounded sample times ONE coil's data-term pair
    E_c^H E_c p plus the regulariser, and one M^{-1} application, and extrapolates
    t_iter = C * t_coil + t_rest (labelled as such)."""
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
    t_iter = spec.coils * t_coil + t_reg + t_pre
    return {"value": 1.0 / t_iter, "unit": "PCG iters/s", "cores": 1, "kind": "oracle",
            "sample": f"extrapolated: 1 coil data-term pair ({t_coil:.1f} s) x {spec.coils} coils + "
                      f"regulariser ({t_reg:.1f} s) + one M^-1 ({t_pre:.1f} s) = {t_iter:.0f} s per PCG "
                      f"iteration at 192^3, numpy fp64 single thread (own FFT)"}


def cpu_baseline_sample(cfg, precond):
    """Oracle PCG iterations/s on a bounded sample: the first 2 SB outer iterations of slice 0
    (about 10-30 s of single-threaded numpy work at config 2)."""
    if cfg == 5:
        return cpu_baseline_3d(cfg, precond)
    from oracle import sb
    spec = synth.CONFIGS[cfg]
    p, y = oracle_problem(cfg, 0)
    prm = spec.params
    n_outer = 2
    t = time.perf_counter()
    _, log = sb.sb_recon(y, p["sens"], p["mask"], prm.mu, prm.lam, prm.gamma, n_outer, 1,
                         prm.wavelet_levels, prm.eps, prm.max_iters, ["none", "circulant", "jacobi"][precond])
    dt = time.perf_counter() - t
    it = sum(log.pcg_iters)
    return {"value": it / dt, "unit": "PCG iters/s", "cores": 1, "kind": "oracle",
            "sample": f"{n_outer} SB outer iterations of slice 0 ({it} PCG iterations, {dt:.1f} s), "
                      f"numpy fp64 single thread; sb_recon time extrapolates to "
                      f"{dt / n_outer * prm.n_outer:.1f} s for {prm.n_outer} outer"}


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


def run_ours(args):
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
    from paper_1710_01758_b200 import SbPcg

    spec, per, first = workload(args.config, ws, rank, args.slices)
    prm = spec.params
    phantom, sens, mask, noise = make_inputs(args.config, first, per)
    coil_mode = args.config == 5 and ws > 1
    comm = None
    if coil_mode:  # config 5 over G GPUs: coil shards + one all-reduce per matvec
        from paper_1710_01758_b200 import SbComm, coil_shard
        c0, c1 = coil_shard(spec.coils, rank, ws)
        sens, noise = np.ascontiguousarray(sens[:, c0:c1]), np.ascontiguousarray(noise[:, c0:c1])
    sens_d = torch.from_numpy(sens).to(torch.complex64).to(dev)
    mask_d = torch.from_numpy(mask).to(dev)
    ctx = SbPcg(sens_d, mask_d, prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
    if coil_mode:
        obj = [SbComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = SbComm(obj[0], rank, ws)
        ctx.set_comm(comm)
    y_d = kspace_gpu(ctx, spec, phantom, mask_d, noise, dev, dist if coil_mode else None)
    out = torch.empty((per,) + tuple(spec.shape), dtype=torch.complex64, device=dev)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    use_graph = not args.no_graph

    def step():
        ctx.build_precond()
        _, log = ctx.recon(y_d, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters,
                           precond=args.precond, use_graph=use_graph, out=out)
        return log

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clock = ClockSampler(dev.index)
    clock.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    total_ms = 0.0
    iters = 0
    step_ms = []
    l0 = ctx.launches()
    for _ in range(args.steps):
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
    if dist:
        dist.barrier()
    # clock probe: keep the GPU loaded ~1.5 s so the sampler sees the steady state
    t_end = time.perf_counter() + 1.5
    while time.perf_counter() < t_end:
        step()
    torch.cuda.synchronize()
    clocks = clock.stop()

    # max over ranks of the device time; sum of work
    t_max = total_ms
    it_sum = iters
    if dist:
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        ii = torch.tensor([iters], device=dev, dtype=torch.float64)
        dist.all_reduce(ii, op=dist.ReduceOp.MAX if coil_mode else dist.ReduceOp.SUM)
        it_sum = int(ii.item())  # coil mode: every rank iterates on the same single problem
    value = it_sum / (t_max / 1e3)
    ms_per_step = t_max / args.steps

    # ---- per-PCG-iteration rate and HBM fraction (BASELINE north_star target: ">= 60% of the
    # B200 HBM roofline per PCG iteration"): fixed-count solves (eps = 0, CUDA graph) with
    # K = 10 and 50 iterations, t_iter = (t50 - t10) / 40 (SURVEY 8(d) timing procedure; the
    # prelude/post of a solve cancel), best of 3; bytes per iteration = B_iter of SURVEY 8(a),
    # 8N(C+10) + 4N + mask bytes, per problem
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
        nimg = int(np.prod(spec.shape))
        mask_b = 4.0 * spec.shape[0] if spec.mask_kind == "lines" else float(np.prod(spec.shape[1:] if len(spec.shape) == 3 else spec.shape))
        b_iter = per * (8.0 * nimg * (spec.coils + 10) + 4.0 * nimg + mask_b)
        pk, _ = peaks()
        pcg_iter = {"us_per_iteration": t_it * 1e6, "problem_iters_per_s": per / t_it,
                    "bytes_per_iteration": b_iter, "achieved_gbs": b_iter / t_it / 1e9,
                    "hbm_frac": b_iter / t_it / 1e9 / pk,
                    "method": "fixed-count solves (eps=0) K=10 and K=50, (t50-t10)/40, best of 3, L2 flushed"}

    # ---- dominant-kernel roofline: K1 (fused matvec) timed with CUDA events per launch on the
    # context stream (eager mode for this pass)
    ctx.set_kernel_timing(True)
    for _ in range(max(1, min(args.steps, 5))):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    k_ms, k_n, k_bytes = ctx.kernel_time(0)
    ctx.set_kernel_timing(False)
    peak, peak_kind = peaks()
    k_avg_s = (k_ms / max(k_n, 1)) / 1e3
    achieved = k_bytes / k_avg_s / 1e9 if k_avg_s > 0 else 0.0
    traffic = load_traffic(args.config)

    # ---- e2e: public API with HOST (pinned) buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        sens_h = torch.from_numpy(sens).to(torch.complex64).pin_memory()
        mask_h = torch.from_numpy(mask).pin_memory()
        y_h = y_d.cpu().pin_memory()
        x_h = torch.empty((per,) + tuple(spec.shape), dtype=torch.complex64).pin_memory()

        # one context for the geometry (as a user would keep it); every step uploads that
        # step's coil maps (+ Lambda rebuild) and k-space from pinned host memory and reads
        # the image back (sb_pcg_update_sens + sb_recon with host pointers)
        c2 = SbPcg(sens_h, mask_h, prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
        if comm is not None:
            c2.set_comm(comm)

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
        for _ in range(args.steps):
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
        e2e = {"value": e_it / e_dt, "unit": "PCG iters/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(x_h.numel() * 8),
               "ms_per_step": 1e3 * e_dt / args.steps}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(args.config, args.precond)

    if rank == 0:
        mask_desc = {"lines": "VD lines R=%d, %d-line centre" % (spec.accel, spec.center),
                     "random2d": "shared 2D VD random R=%d, %dx%d centre" % (spec.accel, spec.center, spec.center),
                     "pe2d": "2D VD phase-encode R=%d, %dx%d centre, readout fully sampled"
                             % (spec.accel, spec.center, spec.center)}[spec.mask_kind]
        line = {
            "metric": METRIC, "value": value, "unit": "PCG iters/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak" if args.config not in (3, 4, 5) else "strong",
            "vs_baseline": None, "dtype": "c64 (fp32 complex; Lambda built in f64)",
            "data": "synthetic (seeded phantoms, coil maps, masks; k-space by sb_encode)",
            "config": {"workload": spec.name, "problems_per_gpu": per, "shape": list(spec.shape),
                       "coils": spec.coils, "mask": mask_desc,
                       "mu": prm.mu, "lambda": prm.lam, "gamma": prm.gamma, "n_outer": prm.n_outer,
                       "pcg_eps": prm.eps, "pcg_max_iters": prm.max_iters,
                       "precond": ["none", "circulant", "jacobi"][args.precond],
                       "pcg_iters_per_step": it_sum / args.steps / (1 if coil_mode else ws),
                       "parallelism": (f"coil-sharded x{ws} (NCCL all-reduce per matvec)" if coil_mode
                                       else (f"slice-sharded x{ws}" if ws > 1 else "1 GPU")),
                       "sb_recon_ms": ms_per_step, "step_ms": [round(t, 3) for t in step_ms],
                       "l2": "flushed between timed steps (256 MiB write)",
                       "loop": "CUDA graph, conditional while node" if use_graph else "eager"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": ("k1_matvec (fused coil FFT matvec, line-mask 1D FFTs)" if spec.mask_kind == "lines"
                                    else "kp_plane (cluster plane matvec: per-coil 2D FFT via DSMEM)"),
                         "kernel_avg_us": k_avg_s * 1e6, "kernel_launches_timed": k_n,
                         "alg_bytes_per_launch": k_bytes},
            "pcg_iteration": pcg_iter,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line))
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
