"""L-BFGS dual solve on the bench workload (config 3 stress state): per-step status histogram, iteration
histogram, and the failing cells' counts (diagnostic for reading 35's iteration cap)."""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from inputs import configs
from inputs.generators import STRESS_AMP, cell_centres, stress_state
from paper_1912_09238_b200 import Context
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = configs.get("cfg3", mesh=dict(nx=nx, ny=nx), hessian="lbfgs", max_newton=maxit)
g = Context(cfg)
base, z = stress_state("euler2d", cell_centres(cfg["mesh"]), g.N, g.m, 9238)
lam = g.zeros(); g.ipm_stress_dual(torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda"), *STRESS_AMP["euler2d"], lam)
u = g.zeros(); g.ipm_moments_from_dual(lam, u); g.ipm_warm_start(u, lam)
for step in range(8):
    info = g.ipm_step(u, lam, None)
    it, st = (x.cpu().numpy() for x in g.last_cell_stats())
    hv, ia = (x.cpu().numpy() for x in g.last_cell_linesearch())
    bad = np.nonzero(st)[0]
    print(json.dumps({"step": step, "maxit": maxit, "status_hist": np.bincount(st, minlength=5).tolist(),
                      "iters_mean": float(it.mean()), "iters_p99": float(np.percentile(it, 99)), "iters_max": int(it.max()),
                      "failed_iters": it[bad][:10].tolist(), "failed_halvings": hv[bad][:10].tolist(),
                      "failed_inadm": ia[bad][:10].tolist(), "halvings_total": int(hv.sum())}), flush=True)
