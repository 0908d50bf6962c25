"""Helpers for the GPU parity tests: run the same seeded inputs through the CUDA path (C-ABI via
paper_1912_09238_b200.ipm) and the oracle, and compare with the tolerances of DESIGN.md."""
from __future__ import annotations

import numpy as np

from inputs import configs
from inputs.generators import STRESS_AMP, bump_channel_mesh, cell_centres, stress_state


def mesh_arrays(cfg):
    if cfg["mesh"]["kind"] != "tri":
        return None
    m = cfg["mesh"]
    return bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"])


def stress_kind(cfg):
    if cfg["closure"] != "euler":
        return "burgers"
    if cfg["mesh"]["kind"] == "tri":
        return "bump"
    return "euler1d" if cfg["m"] == 3 else "euler2d"


def stress_inputs(cfg, seed, ma=None):
    """Seeded base states and normal draws for every cell (inputs/generators.py)."""
    from oracle import num_basis

    N = num_basis(cfg["p"], cfg["M"])
    xy = cell_centres(cfg["mesh"], *(ma[:2] if ma is not None else (None, None)))
    kind = stress_kind(cfg)
    base, z = stress_state(kind, xy, N, cfg["m"], seed, cfg.get("gamma", 1.4))
    return base, z, STRESS_AMP[kind]


def state_scale(u_ref):
    """per-state scale max_j |uhat_{j,0,a}| (reading 27)"""
    return np.maximum(np.abs(u_ref[:, 0, :]).max(axis=0), 1e-300)


def assert_moments_close(u_gpu, u_ora, rel=1e-9, what=""):
    sc = state_scale(u_ora)
    err = (np.abs(u_gpu - u_ora) / sc[None, None, :]).max()
    assert err <= rel, f"{what}: max relative moment difference {err:.3e} > {rel:.0e}"
    return err


def to_np(t):
    return t.detach().cpu().numpy()
