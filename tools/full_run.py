"""Full runs of the BASELINE configurations from their initial conditions (Algorithm 1 to t_end, or a
window of pseudo-time steps for config 4) on one GPU: steps, Newton iterations, wall time, and the
mean / min of the zeroth moment of the density as a sanity summary.  Evidence for DESIGN.md §5
(the bench uses the dual-solve stress state instead; real runs have mostly 0-1 Newton iterations).

usage: python tools/full_run.py [cfg1 cfg2 cfg3 ...] [--nx N] [--steps K]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

from inputs import configs  # noqa: E402
from inputs.generators import bump_channel_mesh  # noqa: E402
from paper_1912_09238_b200 import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["cfg1", "cfg2", "cfg3"])
    ap.add_argument("--nx", type=int, default=0)
    ap.add_argument("--steps", type=int, default=0, help="cap on the number of steps (0: to t_end)")
    ap.add_argument("--hessian", default="newton", choices=["newton", "lbfgs"])
    args = ap.parse_args()
    for name in args.names:
        cfg = configs.get(name, hessian=args.hessian)
        if args.nx and cfg["mesh"]["kind"] == "cart2d":
            cfg["mesh"].update(nx=args.nx, ny=args.nx)
        ma = None
        if cfg["mesh"]["kind"] == "tri":
            m = cfg["mesh"]
            ma = bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"])
        g = Context(cfg, ma)
        uhat = g.zeros()
        g.ipm_project_ic(uhat)
        lam = g.zeros()
        g.ipm_warm_start(uhat, lam)
        t_end = cfg.get("t_end")
        steps = args.steps or (None if t_end else 1000)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n, iters, t = 0, 0, 0.0
        res0 = None
        while True:
            if steps is not None and n >= steps:
                break
            if t_end is not None and t >= t_end * (1 - 1e-14):
                break
            info = g.ipm_step(uhat, lam, t_end)
            if info.failed_cells:
                raise RuntimeError(f"{name} step {n}: {info.failed_cells} failed cells")
            t, n, iters = info.t, n + 1, iters + info.newton_iters
            res0 = res0 or info.residual
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        rho = uhat[:, 0, 0]
        out = {"config": name, "hessian": args.hessian, "cells": g.cells, "steps": n, "t": t, "wall_s": wall,
               "cell_steps_per_s": g.cells * n / wall, "newton_iters_per_cell_step": iters / max(1, g.cells * n),
               "mean_rho0": float(rho.mean()), "min_rho0": float(rho.min()), "dual_kernel": Context.last_dual_kernel()}
        if t_end is None:
            out["residual_drop"] = info.residual / res0 if res0 else None
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
