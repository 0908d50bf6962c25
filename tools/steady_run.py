"""Steady config 4 (One-Shot IPM, adaptive degree 2-5) from the free-stream initial state until the
steady residual (reading 23: area-weighted 1-norm of the change of the density
mean) has dropped by the BASELINE factor 1e-8 relative to the first pseudo-time step,
or a step cap.  Prints one JSON line per `--every` steps (residual drop, level histogram, wall time)
and a final summary line.  Evidence for VERDICT r01 Missing #7 (convergence of the One-Shot
adaptive path).

usage: python tools/steady_run.py [--drop 1e-8] [--max-steps 300000] [--every 2000] [--no-adaptive]
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
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--drop", type=float, default=1e-8)
    ap.add_argument("--max-steps", type=int, default=300000)
    ap.add_argument("--max-seconds", type=float, default=1500.0)
    ap.add_argument("--every", type=int, default=2000)
    ap.add_argument("--no-adaptive", action="store_true")
    ap.add_argument("--pts", default="", help="mesh points NXxNY of the bump channel (default: BASELINE 548x183)")
    ap.add_argument("--hessian", default="newton", choices=["newton", "lbfgs"])
    ap.add_argument("--farfield", action="store_true",
                    help="characteristic far-field ghosts at the inlet and outlet (reading 37) instead of Dirichlet")
    ap.add_argument("--newton", default="", choices=["", "full", "one_step"], help="override the config's mode")
    args = ap.parse_args()
    cfg = configs.get(args.config)
    if args.no_adaptive:
        cfg.pop("levels", None)
    if args.pts:
        nxp, nyp = (int(v) for v in args.pts.split("x"))
        cfg["mesh"].update(nx_pts=nxp, ny_pts=nyp)
    cfg["hessian"] = args.hessian
    if args.farfield:
        cfg["bc"] = [("farfield", sp) if k == "state" else (k, sp) for k, sp in cfg["bc"]]
    if args.newton:
        cfg["newton"] = args.newton
    m = cfg["mesh"]
    g = Context(cfg, bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"]))
    uhat = g.zeros()
    g.ipm_project_ic(uhat)
    lam = g.zeros()
    g.ipm_warm_start(uhat, lam)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res1, n, iters, info = None, 0, 0, None
    drop = None
    while n < args.max_steps:
        info = g.ipm_step(uhat, lam, None)
        if info.failed_cells:
            raise RuntimeError(f"step {n}: {info.failed_cells} failed cells")
        n += 1
        iters += info.newton_iters
        res1 = res1 or info.residual
        drop = info.residual / res1
        if n % args.every == 0 or drop <= args.drop:
            rec = {"step": n, "residual": info.residual, "drop": drop, "wall_s": time.perf_counter() - t0,
                   "newton_iters_per_cell_step": iters / (g.cells * n)}
            if g.cfg.get("levels"):
                lv = g.levels().cpu()
                rec["level_hist"] = torch.bincount(lv.long(), minlength=4).tolist()
            print(json.dumps(rec), flush=True)
        if drop <= args.drop or time.perf_counter() - t0 > args.max_seconds:
            break
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    rho = uhat[:, 0, 0]
    print(json.dumps({"summary": True, "config": args.config, "hessian": args.hessian, "newton": cfg["newton"],
                      "cells": g.cells, "steps": n, "converged": drop <= args.drop,
                      "residual_drop": drop, "target_drop": args.drop, "wall_s": wall,
                      "cell_steps_per_s": g.cells * n / wall, "adaptive": bool(g.cfg.get("levels")),
                      "mean_rho0": float(rho.mean()), "min_rho0": float(rho.min())}), flush=True)


if __name__ == "__main__":
    main()
