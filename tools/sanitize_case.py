"""Small invocations of every product kernel for compute-sanitizer (racecheck / synccheck / memcheck,
one tool per run): k_dual_mma (fixed-shape config-3 and bucketed config-4 instances), k_dual_big
(config 5), k_flux_strip (IPM and SC walks), k_flux_cart, k_flux_warp (triangles, banded), small kernels.
usage: compute-sanitizer --tool racecheck python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from inputs import configs  # noqa: E402
from inputs.generators import bump_channel_mesh  # noqa: E402
from paper_1912_09238_b200 import Context  # noqa: E402


def run(cfg, steps, ma=None, env=None):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        g = Context(cfg, ma)
    finally:
        for k, v in old.items():
            os.environ.pop(k) if v is None else os.environ.__setitem__(k, v)
    u, lam, info = g.run(n_steps=steps)
    torch.cuda.synchronize()
    print(cfg["name"], env or "", "steps", info["steps"], "t", info["t"], "dual", Context.last_dual_kernel(),
          "flux", Context.last_flux_kernel(), flush=True)
    return g


run(configs.get("cfg3", mesh=dict(nx=24, ny=16)), 2)                                  # k_dual_mma fixed, k_flux_strip
run(configs.get("cfg3", mesh=dict(nx=24, ny=16)), 1, env={"IPM_FLUX_KERNEL": "cart"})  # k_flux_cart
run(configs.get("cfg1"), 2)                                                            # 1D, CUDA graph
c4 = configs.parity_variant("cfg4")
m = c4["mesh"]
run(c4, 2, bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"]))                     # bucketed levels, k_flux_warp
run(configs.get("cfg5", mesh=dict(nx=6, ny=5)), 1, env={"IPM_BAND_ROWS": "2"})         # k_dual_big, banded flux
g = Context(configs.get("cfg3", mesh=dict(nx=24, ny=16)))                              # SC strip walk
a, b = g.sc_zeros(), g.sc_zeros()
g.ipm_sc_init(a)
g.ipm_sc_step(a, b)
torch.cuda.synchronize()
print("sc ok", flush=True)
