#!/usr/bin/env python
"""Benchmark of the IPM hot path (arXiv 1912.09238) on B200.

One step = one ipm_step over every cell of the workload: per-cell Newton solve of the IPM dual
problem (FULL, tau = 1e-10), CFL dt, kinetic-flux moment update (all rows of DESIGN.md §Path).
Default workload: BASELINE config 3 (2D Euler Riemann, 1024^2 cells, N=15 x m=4, Q=10x10 GL)
started from the seeded dual-solve stress state so that every cell iterates.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the reference arm of
this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_TFLOPS = 37.2  # derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--nx", type=int, default=0, help="override grid size (cartesian nx = ny)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=32, help="ipm_step_host copy/solve ranges (e2e, N=1)")
    ap.add_argument("--e2e-max-gb", type=float, default=16.0, help="largest state (uhat + lambda) the e2e leg pins")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=9238)
    ap.add_argument("--no-alt", action="store_true", help="skip the L-BFGS comparison line (N=1, Newton runs)")
    ap.add_argument("--hessian", default="newton", choices=["newton", "lbfgs"],
                    help="dual-solve direction: exact Newton (the paper's method, default) or L-BFGS "
                         "(reading 35, SURVEY 8(f) NEXT-4)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = every rank a block of the configured grid; strong = the configured grid "
                         "split into N blocks (fixed total work)")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
def flops_per_iteration(N, m, Q):
    """Algorithmic fp64 flops of one Newton iteration of one cell:
    reconstruction 2QNm, gradient 2QNm, Hessian unique entries 2Q N(N+1)/2 m(m+1)/2,
    Cholesky n^3/3 and two triangular solves 2n^2 (n = N m).  Transcendentals not counted."""
    n = N * m
    return 2 * Q * N * m + 2 * Q * N * m + 2 * Q * (N * (N + 1) // 2) * (m * (m + 1) // 2) + n ** 3 / 3 + 2 * n * n


def flops_executed_per_iteration(N, m, Q, p, q1, kernel):
    """fp64 flops the kernels actually execute per Newton iteration: the Hessian
    is sum-factorised over the tensor Gauss-Legendre rule for p = 2, 3 (k_dual_mma / k_dual_big), the
    DMMA Cholesky works on the 8-padded n.  Reported next to the algorithmic figure, so the fraction
    of the fp64 pipe the kernel really uses is visible (SURVEY §8d note on sum factorisation)."""
    n = N * m
    MM = m * (m + 1) // 2
    sf = None
    if p in (2, 3) and kernel in ("k_dual_mma", "k_dual_group", "k_dual_big"):
        # degree M from N = C(M+p, p)
        from math import comb
        M = next(mm for mm in range(0, 40) if comb(mm + p, p) == N)
        npr = (M + 1) * (M + 2) // 2
        npairs = N * (N + 1) // 2
        if p == 2:
            sf = q1 * MM * q1 * npr * 2 + npairs * MM * q1 * 2
        else:
            sf = q1 * q1 * MM * q1 * npr * 2 + q1 * npr * MM * q1 * npr * 2 + npairs * MM * q1 * 2
    hess = sf if sf is not None else 2 * Q * (N * (N + 1) // 2) * MM
    nc = 8 * ((n + 7) // 8) if kernel == "k_dual_mma" else n
    return 4 * Q * N * m + hess + nc ** 3 / 3 + 2 * nc * nc


def flops_lbfgs_per_iteration(N, m, Q, mh=8):
    """fp64 flops of one L-BFGS iteration of one cell (reading 35): reconstruction 2QNm, gradient 2QNm,
    Jbar = sum_k omega_k J_k 2Q m(m+1)/2, two-loop recursion over mh pairs (two dot products and two
    axpys of length n each: 8 n mh), H0 = I (x) Jbar^{-1} by two m x m triangular solves per moment
    (2 N m^2).  Executed = algorithmic (no sum factorisation, the DMMA gradient pads N to 8)."""
    n = N * m
    return 4 * Q * N * m + 2 * Q * (m * (m + 1) // 2) + 8 * n * mh + 2 * N * m * m


def flops_initial(N, m, Q):
    """every cell evaluates the reconstruction and gradient once before its first test (a2 + a3)"""
    return 4 * Q * N * m


def flux_bytes_per_cell(N, m, Q):
    """algorithmic HBM bytes of the flux kernel per cell: node states read once, uhat read + write"""
    return 8 * (Q * m + 2 * N * m)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.samples, self.index, self._stop = [], index, threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nme, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(nme)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------
def workload(args):
    from inputs import configs

    cfg = configs.get(args.config)
    cfg["hessian"] = args.hessian
    if args.nx and cfg["mesh"]["kind"] == "cart2d":
        cfg["mesh"].update(nx=args.nx, ny=args.nx)
    elif args.nx and cfg["mesh"]["kind"] == "1d":
        cfg["mesh"].update(nx=args.nx)
    return cfg


def mesh_arrays(cfg):
    """triangle meshes (config 4) are generated from their seeded recipe (inputs/generators.py)"""
    from inputs.generators import bump_channel_mesh

    m = cfg["mesh"]
    return bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"]) if m["kind"] == "tri" else None


def stress_kind(cfg):
    if cfg["closure"] != "euler":
        return "burgers"
    if cfg["mesh"]["kind"] == "tri":
        return "bump"
    return "euler1d" if cfg["m"] == 3 else "euler2d"


def centres(cfg, ma):
    from inputs.generators import cell_centres

    return cell_centres(cfg["mesh"], *(ma[:2] if ma is not None else (None, None)))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands, on a bounded sample."""
    import oracle
    from inputs import configs
    from inputs.generators import STRESS_AMP, cell_centres, stress_state

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    cfg = workload(args)
    kind = stress_kind(cfg)
    if cfg["mesh"]["kind"] == "tri":
        full_cells = len(mesh_arrays(cfg)[1])
        sample = dict(configs.parity_variant(args.config), hessian=args.hessian)
        side = None
    else:
        full_cells = cfg["mesh"]["nx"] * cfg["mesh"].get("ny", 1)
        side = (128 if cfg["p"] <= 2 else 8) if cfg["mesh"]["kind"] == "cart2d" else min(cfg["mesh"]["nx"], 4096)
        if args.nx:
            side = min(side, args.nx)
        sample = configs.get(args.config, mesh=dict(nx=side, ny=side), hessian=args.hessian)
    ma = mesh_arrays(sample)
    o = oracle.Oracle(sample, ma)
    base, z = stress_state(kind, centres(sample, ma), o.N, o.m, args.seed, sample.get("gamma", 1.4))
    amp = STRESS_AMP[kind]
    lam_star = o.stress_dual(base, z, amp)
    uhat = o.moments_from_dual_all(lam_star)
    lam = o.warm_start(uhat)
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    iters = 0
    for _ in range(steps):
        w, it, _, _, _ = o.step(uhat, lam)
        iters += int(it.sum())
    dt = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    value = o.cells * steps / dt
    line = {
        "impl": "reference", "metric": "IPM cell-steps/s (= cell dual-solves/s)", "value": value,
        "unit": "cell-steps/s", "n_gpus": args.gpus, "steps": steps, "warmup": 0,
        "ms_per_step": dt / steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "cells_full": full_cells, "sample_cells": o.cells},
        "cpu_baseline": {"value": value, "unit": "cell-steps/s", "cores": cores, "kind": "oracle",
                         "cpu": cpu_model(),
                         "sample": f"{o.cells} cells of the {args.config} stress state, {steps} steps "
                                   f"({iters} Newton iterations), OpenMP over cells"},
        "e2e": {"value": value, "unit": "cell-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def cpu_baseline(args, cfg):
    """Oracle timed on the host cores on a bounded sample (~10-30 s of CPU work)."""
    ref = run_reference(args)
    if ref is None:
        return None
    return ref["cpu_baseline"]


def _allreduce(t, op):
    """all-reduce of a device tensor (staged through the host on gloo, the one-GPU functional test)"""
    import torch.distributed as dist

    if dist.get_backend() == "gloo" and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)


def decompose(world):
    """px x py block decomposition of the 2D grid (py >= px; rows of cells are contiguous in y)."""
    py = 1
    while py * py * 2 <= world and world % (py * 2) == 0:
        py *= 2
    return world // py, py


def _local_centres(mesh, ids):
    nx = mesh["nx"]
    dx = (mesh["x1"] - mesh["x0"]) / nx
    dy = (mesh["y1"] - mesh["y0"]) / mesh["ny"]
    ix, iy = ids % nx, ids // nx
    return np.stack([mesh["x0"] + (ix + 0.5) * dx, mesh["y0"] + (iy + 0.5) * dy], axis=1)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from inputs.generators import STRESS_AMP, cell_centres, stress_state
    from paper_1912_09238_b200 import Context

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("IPM_DIST_BACKEND", "nccl") != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink; IPM_DIST_BACKEND=gloo runs the multi-rank path on one GPU (functional test)
        backend = os.environ.get("IPM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = workload(args)
    px, py = decompose(world)
    if world > 1 and cfg["mesh"]["kind"] == "cart2d" and args.scaling == "weak":
        # weak scaling: every rank owns a block of the single-GPU size, halos exchanged over NVLink
        cfg["mesh"].update(nx=cfg["mesh"]["nx"] * px, ny=cfg["mesh"]["ny"] * py)
    ma = mesh_arrays(cfg)
    g = Context(cfg, ma, rank=rank, nranks=world, px=px, py=py)
    kind = stress_kind(cfg)
    if world == 1:
        xy = centres(cfg, ma)
    elif cfg["mesh"]["kind"] == "cart2d":
        xy = _local_centres(cfg["mesh"], g.cell_ids())
    else:
        xy = centres(cfg, ma)[g.cell_ids()]
    base, z = stress_state(kind, xy, g.N, g.m, args.seed + rank, cfg.get("gamma", 1.4))
    amp = STRESS_AMP[kind]
    dev = torch.device("cuda", local)
    # two state arrays only (config 5 at 4096^2: 30 GB each): lambda* -> uhat = h(lambda*) -> warm start
    lam = g.zeros()
    d_base, d_z = torch.from_numpy(base).to(dev), torch.from_numpy(z).to(dev)
    del base, z
    g.ipm_stress_dual(d_base, d_z, amp[0], amp[1], lam)
    del d_base, d_z
    uhat = g.zeros()
    g.ipm_moments_from_dual(lam, uhat)
    g.ipm_warm_start(uhat, lam)
    torch.cuda.synchronize()
    state_gb = 2 * uhat.numel() * 8 / 1e9
    # small problems (configs 1, 2) replay each step from a CUDA graph (ipm.h IPM_GRAPH_MAX_CELLS), which
    # per-kernel event timing disables: their kernel times come from a separate pass after the timed one
    graph_step = world == 1 and g.cells < 65536 and not cfg.get("levels")
    g.enable_timing(not graph_step)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (starts from the stress state)
    for _ in range(args.warmup):
        g.ipm_step(uhat, lam, None, sync=False)
    barrier()
    # the starting state of the timed steps: the e2e leg below re-runs exactly these steps
    t_start = g.time()
    do_e2e = not args.no_e2e and state_gb <= args.e2e_max_gb
    if do_e2e:
        u_start, l_start = uhat.cpu().pin_memory(), lam.cpu().pin_memory()
    # timed region: K consecutive steps (Algorithm 1), device-timed with CUDA events
    # inputs smaller than L2 (configs 1, 2, small windows): every step is timed on its own after an
    # L2 flush (a write of twice the L2 size), and the step times are summed
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    state_bytes = g.cells * (g.Q * g.m + 2 * g.N * g.m) * 8
    flush = state_bytes < 2 * l2
    fbuf = torch.empty(2 * l2 // 4, dtype=torch.int32, device=dev) if flush else None
    dual_ms, flux_ms, iters, local_iters, failed, halvings = [], [], 0, 0, 0, 0
    hist = np.zeros(16, np.int64)
    ms = 0.0
    with ClockSampler(local) as clk:
        barrier()
        if not flush:
            e0.record(stream)
        for k in range(args.steps):
            if flush:
                fbuf.fill_(k)
                e0.record(stream)
            info = g.ipm_step(uhat, lam, None, sync=True)
            if flush:
                e1.record(stream)
                e1.synchronize()
                ms += e0.elapsed_time(e1)
            # info holds global sums (the binding all-reduces across ranks once); the rank's own count
            # is kept for the imbalance
            iters += info.newton_iters
            local_iters += g.last_local_newton_iters if world > 1 else info.newton_iters
            failed += info.failed_cells
            halvings += info.halvings
            hist += np.array(info.newton_hist[:], dtype=np.int64)
            if not graph_step:
                d, f = g.last_kernel_ms()
                dual_ms.append(d)
                flux_ms.append(f)
        if not flush:
            e1.record(stream)
        barrier()
    if not flush:
        ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        _allreduce(t, dist.ReduceOp.MAX)
    ms = float(t.item())
    cells_total = g.cells * world
    value = cells_total * args.steps / (ms / 1e3)
    if graph_step:  # kernel times of the same kind of steps, launched kernel by kernel (untimed pass)
        g.enable_timing(True)
        uc, lc = uhat.clone(), lam.clone()
        for _ in range(args.steps):
            g.ipm_step(uc, lc, None, sync=True)
            d, f = g.last_kernel_ms()
            dual_ms.append(d)
            flux_ms.append(f)
        del uc, lc
        g.enable_timing(False)
    if failed:
        raise SystemExit(f"bench: {failed} failed cells in the timed steps (worst status "
                         f"{g.get_status()[0]}): the step did not do the method's work")
    # Newton-iteration balance across ranks (the scaling risk is the imbalance): the
    # per-rank counts reduced exactly once (MAX), the total is already global
    imbalance, iters_all = None, iters
    if world > 1:
        it_max = torch.tensor([float(local_iters)], device=dev, dtype=torch.float64)
        _allreduce(it_max, dist.ReduceOp.MAX)
        imbalance = float(it_max.item()) / max(1e-30, iters_all / world)

    # end-to-end through the C-ABI with host buffers: H2D of the step inputs (uhat, lambda) from
    # pinned memory, ipm_step, D2H of the step result (uhat, lambda), every step
    e2e = None if do_e2e or args.no_e2e else {
        "value": None, "skipped": f"state {state_gb:.0f} GB exceeds --e2e-max-gb {args.e2e_max_gb} of pinned host memory"}
    if do_e2e:
        # the SAME K steps from the same starting state (host copies of the state after warm-up)
        h_u, h_l = u_start, l_start
        g.set_time(t_start)
        e2e_iters, e2e_failed = 0, 0
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            if world == 1:
                # the C-ABI host-buffer step: copies in cell ranges overlapped with the dual solves
                info = g.ipm_step_host(h_u, h_l, uhat, lam, None, nchunks=args.e2e_chunks)
            else:
                uhat.copy_(h_u, non_blocking=True)
                lam.copy_(h_l, non_blocking=True)
                info = g.ipm_step(uhat, lam, None, sync=True)
                h_u.copy_(uhat, non_blocking=True)
                h_l.copy_(lam, non_blocking=True)
            e2e_iters += info.newton_iters
            e2e_failed += info.failed_cells
        e1.record(stream)
        barrier()
        if e2e_failed:
            raise SystemExit(f"bench e2e: {e2e_failed} failed cells")
        ms_e = e0.elapsed_time(e1)
        te = torch.tensor([ms_e], device=dev, dtype=torch.float64)
        if world > 1:
            _allreduce(te, dist.ReduceOp.MAX)
        nbytes = (uhat.numel() + lam.numel()) * 8
        e2e = {"value": cells_total * args.steps / (float(te.item()) / 1e3), "unit": "cell-steps/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "path": f"ipm_step_host, {args.e2e_chunks} copy/solve cell ranges" if world == 1
               else "cudaMemcpyAsync + ipm_step",
               "same_steps_as_value": True, "newton_iters": int(e2e_iters),
               "newton_iters_match_value": int(e2e_iters) == int(iters)}

    N, m, Q = g.N, g.m, g.Q
    dual_avg = float(np.mean(dual_ms))
    kname = Context.last_dual_kernel()
    if args.hessian == "lbfgs":
        flops = flops_ex = iters / args.steps * flops_lbfgs_per_iteration(N, m, Q) + g.cells * flops_initial(N, m, Q)
    else:
        flops = iters / args.steps * flops_per_iteration(N, m, Q) + g.cells * flops_initial(N, m, Q)
        flops_ex = iters / args.steps * flops_executed_per_iteration(N, m, Q, cfg["p"], cfg["q1d"], kname) + \
            g.cells * flops_initial(N, m, Q)
    achieved = flops / (dual_avg / 1e3) / 1e12
    achieved_ex = flops_ex / (dual_avg / 1e3) / 1e12
    traffic = traffic_flux = ncu_pipe = None
    if os.path.exists(NCU_SUMMARY) and not args.nx and args.hessian == "newton":  # the bench configuration only
        try:
            ent = json.load(open(NCU_SUMMARY)).get(args.config, {})
            traffic, traffic_flux = ent.get("dual_dram_bytes_per_launch"), ent.get("flux_dram_bytes_per_launch")
            ncu_pipe = ent.get("dual_fp64_pipe_active_pct")
        except Exception:
            traffic = traffic_flux = ncu_pipe = None
    flux_avg = float(np.mean(flux_ms))
    hbm = json.load(open(MEASURED))["hbm_gbs"] if os.path.exists(MEASURED) else 6650.0
    flux_gbs = g.cells * flux_bytes_per_cell(N, m, Q) / (flux_avg / 1e3) / 1e9
    line = None
    if rank == 0:
        line = {
            "metric": "IPM cell-steps/s (= cell dual-solves/s)", "value": value, "unit": "cell-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.config, "cells_per_gpu": g.cells, "N": N, "m": m, "Q": Q,
                       "newton": cfg["newton"], "tau": cfg["tau"], "hessian": args.hessian,
                       "state": "seeded dual-solve stress state (SURVEY §8d), steps continue Algorithm 1",
                       "l2": ("L2 flushed before every timed step (step state %.1f MB < 2x L2)" % (state_bytes / 1e6))
                       if flush else "inputs larger than L2 (node states %.1f GB)" % (g.cells * Q * m * 8 / 1e9),
                       "parallelism": f"domain decomposition {px}x{py}, {os.environ.get('IPM_DIST_BACKEND', 'nccl').upper()} halo exchange" if world > 1
                       else "single", "global_cells": g.cells * world,
                       "node_state_bands": g.node_band_rows(),
                       "step_launch": "CUDA graph replay" if graph_step else "kernel launches"},
            "newton_iters_per_cell_step": iters_all / (cells_total * args.steps),
            "cell_newton_iters_per_s": iters_all / (ms / 1e3),
            "newton_imbalance_max_over_mean": imbalance,
            "failed_cells": int(failed),
            "newton_hist": [int(x) for x in hist],
            "linesearch_halvings": int(halvings),
            # the dual kernel's fp64 roofline: led by the flops the kernel EXECUTES (the Hessian is
            # sum-factorised, SURVEY §8d note), the algorithmic count of §8d beside it
            "roofline": {"bound": "alu", "kernel": kname, "achieved": achieved_ex,
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved_ex / FP64_PEAK_TFLOPS,
                         "flops": ("L-BFGS iteration (reading 35): node pass, gradient, Jbar, two-loop recursion"
                                   if args.hessian == "lbfgs" else
                                   "as executed: sum-factorised Hessian, 8-padded DMMA Cholesky"),
                         "peak_note": "derived 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz; measured DMMA 37.06, "
                                      "DFMA 33.7, DGEMM 35.5 TF/s (profiles/r01_fp64_peak.json)",
                         "algorithmic": {"achieved": achieved, "frac": achieved / FP64_PEAK_TFLOPS,
                                         "flops": "SURVEY §8d: direct unique-entry Hessian, Cholesky n^3/3"},
                         "ncu_fp64_pipe_active": ncu_pipe,
                         "traffic": traffic, "dual_ms_avg": dual_avg,
                         "share_of_step": dual_avg / (ms / args.steps)},
            "roofline_flux": {"bound": "hbm", "kernel": Context.last_flux_kernel(), "achieved": flux_gbs, "peak": hbm,
                              "unit": "GB/s", "frac": flux_gbs / hbm, "traffic": traffic_flux,
                              "bytes_per_launch": g.cells * flux_bytes_per_cell(N, m, Q), "flux_ms_avg": flux_avg},
            "e2e": e2e,
            "gpu_launches": (4 if world == 1 else 6) * args.steps,
            "clocks": clk.summary(),
        }
    if line is not None and world == 1 and args.hessian == "newton" and not args.no_alt:
        del uhat, lam
        torch.cuda.empty_cache()
        line["lbfgs"] = run_alt_lbfgs(args, cfg, ma, dev)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def run_alt_lbfgs(args, cfg, ma, dev):
    """The same workload, warm-up and timed steps with the quasi-Newton dual solve (reading 35,
    SURVEY 8(f) NEXT-4: L-BFGS directions instead of the exact Hessian): a comparison line, not the
    headline (the paper's method is Newton).  Same stress state, same device timing."""
    import torch

    from inputs.generators import STRESS_AMP, stress_state
    from paper_1912_09238_b200 import Context

    c2 = dict(cfg, hessian="lbfgs")
    try:
        g = Context(c2, ma)
    except Exception as e:  # (configurations the quasi-Newton kernels do not cover)
        return {"skipped": str(e)[:200]}
    kind = stress_kind(cfg)
    base, z = stress_state(kind, centres(cfg, ma), g.N, g.m, args.seed, cfg.get("gamma", 1.4))
    amp = STRESS_AMP[kind]
    lam = g.zeros()
    g.ipm_stress_dual(torch.from_numpy(base).to(dev), torch.from_numpy(z).to(dev), amp[0], amp[1], lam)
    uhat = g.zeros()
    g.ipm_moments_from_dual(lam, uhat)
    g.ipm_warm_start(uhat, lam)
    g.enable_timing(True)
    for _ in range(args.warmup):
        g.ipm_step(uhat, lam, None, sync=False)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = g.cells * (g.Q * g.m + 2 * g.N * g.m) * 8 < 2 * l2
    fbuf = torch.empty(2 * l2 // 4, dtype=torch.int32, device=dev) if flush else None
    ms, iters, failed, dual_ms, flux_ms = 0.0, 0, 0, [], []
    for k in range(args.steps):
        if flush:
            fbuf.fill_(k)
        e0.record(stream)
        info = g.ipm_step(uhat, lam, None, sync=True)
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        iters += info.newton_iters
        failed += info.failed_cells
        d, f = g.last_kernel_ms()
        dual_ms.append(d)
        flux_ms.append(f)
    N, m, Q = g.N, g.m, g.Q
    dual_avg = float(np.mean(dual_ms))
    flops = iters / args.steps * flops_lbfgs_per_iteration(N, m, Q) + g.cells * flops_initial(N, m, Q)
    return {"hessian": "lbfgs", "what": "quasi-Newton dual solve (reading 35, PAPER.md:843), same workload and steps; "
                                         "it pays far from the warm start (this stress state, One-Shot), not on "
                                         "smooth time stepping from the IC (DESIGN.md §8 full runs)",
            "value": g.cells * args.steps / (ms / 1e3), "unit": "cell-steps/s", "ms_per_step": ms / args.steps,
            "newton_iters_per_cell_step": iters / (g.cells * args.steps), "failed_cells": int(failed),
            "kernel": Context.last_dual_kernel(), "dual_ms_avg": dual_avg, "flux_ms_avg": float(np.mean(flux_ms)),
            "dual_tflops": flops / (dual_avg / 1e3) / 1e12}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        # not under torchrun: launch N ranks (one process per GPU) the way the driver does
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    if world and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        line = run_reference(args)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    line = run_ours(args)
    if line is not None:
        line["cpu_baseline"] = None if args.no_cpu_baseline else cpu_baseline(args, None)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
