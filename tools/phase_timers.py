"""Per-phase cycle breakdown of the dual kernel (needs libipm_timers.so: build.py --timers)."""
import os, sys, json
os.environ.setdefault("IPM_LIB", os.path.join(os.path.dirname(__file__), "..", "paper_1912_09238_b200", "libipm_timers.so"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from inputs import configs
from inputs.generators import STRESS_AMP, cell_centres, stress_state
from paper_1912_09238_b200 import Context
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
nx = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = configs.get(name, mesh=dict(nx=nx, ny=nx))
g = Context(cfg)
kind = "euler2d" if cfg["closure"] == "euler" else "burgers"
base, z = stress_state(kind, cell_centres(cfg["mesh"]), g.N, g.m, 9238)
lam = g.zeros(); g.ipm_stress_dual(torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda"), *STRESS_AMP[kind], lam)
u = g.zeros(); g.ipm_moments_from_dual(lam, u); l0 = g.zeros(); g.ipm_warm_start(u, l0)
g.debug_phase_cycles()
g.enable_timing(True)
info = g.ipm_step(u, l0)
d, f = g.last_kernel_ms()
c = g.debug_phase_cycles().astype(float)
names = (["eval/grad/linesearch", "hessian", "cholesky", "backsub", "final linesearch", "end", "-", "epilogue+fetch"] if os.environ.get("IPM_DUAL_KERNEL") == "group" else ["top (eval/grad)", "hessian", "chol+solve", "linesearch", "[gather+diag0]", "[factor loop]", "[backsub]", "epilogue+fetch"])
tot = c.sum()
print(json.dumps({"cfg": name, "cells": g.cells, "iters": int(info.newton_iters), "dual_ms": d,
                  "cycles_per_cell_iter": tot / max(1, info.newton_iters),
                  "share": {n: round(v / tot, 3) for n, v in zip(names, c) if v}}))
