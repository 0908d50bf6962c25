"""Where does the steady config-4 residual plateau live?  (DESIGN.md §8 "Next" 3)

Runs the One-Shot adaptive iteration of tools/steady_run.py on the bump-channel mesh to pseudo-step
--start, then for a window of --window pseudo-steps records every step's residual (reading 23) and,
every --snap steps, the per-cell one-step change |rho_mean^{n+1} - rho_mean^n| / dt-free (the summand
of the residual) and the density means themselves.  Writes gpurun_out/<tag>.npz (centroids, areas,
tags of boundary cells, the residual series, the per-cell maps) for analysis on the host.

usage: python tools/steady_diag.py [--pts 548x183] [--hessian lbfgs] [--start 240000] [--window 20000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

from inputs import configs  # noqa: E402
from inputs.generators import bump_channel_mesh  # noqa: E402
from paper_1912_09238_b200 import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pts", default="")
    ap.add_argument("--hessian", default="lbfgs", choices=["newton", "lbfgs"])
    ap.add_argument("--start", type=int, default=240000)
    ap.add_argument("--window", type=int, default=20000)
    ap.add_argument("--snap", type=int, default=1000)
    ap.add_argument("--out", default="gpurun_out/steady_diag")
    ap.add_argument("--cfl", type=float, default=0.0, help="pseudo-time CFL number (default: the config's)")
    args = ap.parse_args()
    cfg = configs.get("cfg4")
    if args.pts:
        nxp, nyp = (int(v) for v in args.pts.split("x"))
        cfg["mesh"].update(nx_pts=nxp, ny_pts=nyp)
    cfg["hessian"] = args.hessian
    if args.cfl > 0:
        cfg["cfl"] = args.cfl
    m = cfg["mesh"]
    vert, tri, tags = bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"])
    g = Context(cfg, (vert, tri, tags))
    uhat = g.zeros()
    g.ipm_project_ic(uhat)
    lam = g.zeros()
    g.ipm_warm_start(uhat, lam)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res1 = None
    for n in range(args.start):
        info = g.ipm_step(uhat, lam, None)
        res1 = res1 or info.residual
        if (n + 1) % 20000 == 0:
            print(json.dumps({"step": n + 1, "drop": info.residual / res1, "wall_s": time.perf_counter() - t0}),
                  flush=True)
    res, dts, maps, rhos, steps = [], [], [], [], []
    for k in range(args.window):
        before = uhat[:, 0, 0].clone() if k % args.snap == 0 else None
        t_before = g.time()
        info = g.ipm_step(uhat, lam, None)
        if info.failed_cells:
            raise RuntimeError(f"{info.failed_cells} failed cells")
        res.append(info.residual)
        dts.append(g.time() - t_before)
        if before is not None:
            maps.append((uhat[:, 0, 0] - before).abs().float().cpu().numpy())
            if not rhos or k + args.snap >= args.window:
                rhos.append(uhat[:, 0, 0].cpu().numpy())
            steps.append(args.start + k)
    cen = vert[tri].mean(axis=1)
    a, b, c = vert[tri[:, 0]], vert[tri[:, 1]], vert[tri[:, 2]]
    area = 0.5 * np.abs((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))
    lv = g.levels().cpu().numpy()
    np.savez_compressed(args.out + ".npz", centroid=cen, area=area, tags=tags, residual=np.array(res),
                        dt=np.array(dts), dmap=np.array(maps), rho=np.array(rhos), steps=np.array(steps),
                        levels=lv, res1=res1)
    print(json.dumps({"summary": True, "cells": g.cells, "start": args.start, "window": args.window,
                      "drop_first": res[0] / res1, "drop_last": res[-1] / res1,
                      "drop_min": min(res) / res1, "drop_max": max(res) / res1,
                      "wall_s": time.perf_counter() - t0}), flush=True)


if __name__ == "__main__":
    main()
