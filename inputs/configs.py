"""Workload descriptions for BASELINE.json configs 1-5 and their parity-sized variants.

Pure data: no arithmetic of the method lives here.  Both the CPU oracle
(``oracle/oracle.py``) and the CUDA path (``paper_1912_09238_b200/ipm.py``)
translate these dicts into their own structures.  Readings of the paper used to
fill gaps are numbered as in DESIGN.md ("Readings", = SURVEY.md §8(c)).

State specs are primitive states, optionally affine in xi:
  ``{"prim": (q...), "dprim": {(comp, dim): coeff}}``  scalar: (u,); Euler 1D (rho,v,p);
  Euler 2D (rho,vx,vy,p);   or ``{"freestream": dict(rho, p, mach0, dmach, dim_mach,
  theta0_deg, dtheta_deg, dim_theta)}``.
"""
from __future__ import annotations

import copy

GAMMA = 1.4

_NEWTON = dict(tau=1e-10, armijo_c=1e-4, max_newton=100, max_halvings=30)  # readings 2, 3, 5

# Lax-Liu 2D Riemann configuration of BASELINE cfg 3: NE, NW, SW, SE (reading 18)
_QUAD_STATES = [
    {"prim": (1.5, 0.0, 0.0, 1.5)},
    {"prim": (0.5323, 1.206, 0.0, 0.3)},
    {"prim": (0.138, 1.206, 1.206, 0.029)},
    {"prim": (0.5323, 0.0, 1.206, 0.3)},
]


def _cfg1():
    # BASELINE cfg 1: Burgers, bounded-barrier entropy, global LF (reading 14), Dirichlet 12 / 3
    return dict(
        name="cfg1_burgers", p=1, M=5, q1d=20, m=1, closure="barrier", umin=2.9, umax=12.1,
        gamma=GAMMA, flux="lf_global",
        mesh=dict(kind="1d", nx=200, x0=0.0, x1=3.0, periodic=False),
        bc=[("state", {"prim": (12.0,)}), ("state", {"prim": (3.0,)})],
        ic=dict(kind="step1d", xs0=0.5, xs1=(0.2,), states=[{"prim": (12.0,)}, {"prim": (3.0,)}]),
        cfl=0.5, t_end=0.11, newton="full", update="conservative", **_NEWTON)


def _cfg2():
    # BASELINE cfg 2: Sod, interface 0.5+0.05 xi, HLL (reading 14), transmissive
    return dict(
        name="cfg2_sod", p=1, M=9, q1d=30, m=3, closure="euler", gamma=GAMMA, flux="hll",
        mesh=dict(kind="1d", nx=2000, x0=0.0, x1=1.0, periodic=False),
        bc=[("transmissive", None), ("transmissive", None)],
        ic=dict(kind="step1d", xs0=0.5, xs1=(0.05,),
                states=[{"prim": (1.0, 0.0, 1.0)}, {"prim": (0.125, 0.0, 0.1)}]),
        cfl=0.4, t_end=0.14, newton="full", update="conservative", **_NEWTON)


def _cfg3():
    # BASELINE cfg 3: 2D Riemann, x_s = 0.5+0.05 xi1, y_s = 0.5+0.05 xi2, Rusanov (reading 14)
    return dict(
        name="cfg3_riemann2d", p=2, M=4, q1d=10, m=4, closure="euler", gamma=GAMMA, flux="rusanov",
        mesh=dict(kind="cart2d", nx=1024, ny=1024, x0=0.0, x1=1.0, y0=0.0, y1=1.0, periodic=False),
        bc=[("transmissive", None)] * 4,
        ic=dict(kind="quad2d", xs0=0.5, xs1=(0.05, 0.0), ys0=0.5, ys1=(0.0, 0.05),
                states=copy.deepcopy(_QUAD_STATES)),
        cfl=0.4, t_end=0.25, newton="full", update="conservative", **_NEWTON)


def _cfg4():
    # BASELINE cfg 4: steady bump channel, One-Shot + adaptive degree 2..5 (readings 18, 20, 22-24)
    fs = {"freestream": dict(rho=1.0, p=1.0 / GAMMA, mach0=0.5, dmach=0.05, dim_mach=0,
                             theta0_deg=0.0, dtheta_deg=1.0, dim_theta=1)}
    return dict(
        name="cfg4_bump", p=2, M=5, q1d=12, m=4, closure="euler", gamma=GAMMA, flux="rusanov",
        mesh=dict(kind="tri", generator="bump_channel", nx_pts=548, ny_pts=183, seed=9238),
        # tri tags: 0 bottom wall (incl. bump), 1 outlet (x=3), 2 top wall, 3 inlet (x=0)
        bc=[("slip", None), ("state", fs), ("slip", None), ("state", fs)],
        ic=dict(kind="uniform", states=[fs]),
        cfl=0.5, t_end=None, steady_drop=1e-8, newton="one_step", update="paper_c",
        levels=[2, 3, 4, 5], initial_level=0, delta_dec=1e-5, delta_inc=1e-4, **_NEWTON)


def _cfg5():
    # BASELINE cfg 5: cfg 3 + rho x (1 + 0.1 xi3) for x < x_s (NW, SW) (readings 18, 28)
    st = copy.deepcopy(_QUAD_STATES)
    st[1]["dprim"] = {(0, 2): 0.1 * 0.5323}
    st[2]["dprim"] = {(0, 2): 0.1 * 0.138}
    return dict(
        name="cfg5_riemann2d_p3", p=3, M=5, q1d=10, m=4, closure="euler", gamma=GAMMA, flux="rusanov",
        mesh=dict(kind="cart2d", nx=4096, ny=4096, x0=0.0, x1=1.0, y0=0.0, y1=1.0, periodic=False),
        bc=[("transmissive", None)] * 4,
        ic=dict(kind="quad2d", xs0=0.5, xs1=(0.05, 0.0, 0.0), ys0=0.5, ys1=(0.0, 0.05, 0.0), states=st),
        cfl=0.4, t_end=0.25, newton="full", update="conservative", **_NEWTON)


CONFIGS = {"cfg1": _cfg1, "cfg2": _cfg2, "cfg3": _cfg3, "cfg4": _cfg4, "cfg5": _cfg5}


def get(name: str, **overrides) -> dict:
    """A fresh copy of a config; ``mesh`` overrides are merged, the rest replace."""
    cfg = CONFIGS[name]()
    for k, v in overrides.items():
        if k == "mesh":
            cfg["mesh"].update(v)
        else:
            cfg[k] = v
    return cfg


def parity_variant(name: str) -> dict:
    """Parity-sized versions the oracle finishes in seconds (SURVEY §8c parity protocol)."""
    if name == "cfg1":
        return get("cfg1")
    if name == "cfg2":
        return get("cfg2", mesh=dict(nx=200), t_end=0.04)
    if name == "cfg3":
        return get("cfg3", mesh=dict(nx=24, ny=20), t_end=0.02)
    if name == "cfg4":
        return get("cfg4", mesh=dict(nx_pts=40, ny_pts=14))
    if name == "cfg5":
        return get("cfg5", mesh=dict(nx=6, ny=5), t_end=0.01)
    raise KeyError(name)


def steady1d(newton: str = "full", nx: int = 40) -> dict:
    """Test-only steady problem for the One-Shot pins (Theorems 1-2):
    supersonic Burgers inflow u_L(xi) = 9 + 2 xi washing out the IC u = 8 + 1.5 xi, bounded-barrier
    entropy of cfg 1, Dirichlet inflow ghost, transmissive outflow, global LF flux."""
    uL = {"prim": (9.0,), "dprim": {(0, 0): 2.0}}
    u0 = {"prim": (8.0,), "dprim": {(0, 0): 1.5}}
    return dict(
        name="steady1d_burgers", p=1, M=4, q1d=10, m=1, closure="barrier", umin=2.9, umax=12.1,
        gamma=GAMMA, flux="lf_global",
        mesh=dict(kind="1d", nx=nx, x0=0.0, x1=1.0, periodic=False),
        bc=[("state", uL), ("transmissive", None)],
        ic=dict(kind="uniform", states=[u0]),
        cfl=0.5, t_end=None, steady_drop=1e-8, newton=newton,
        update="paper_c" if newton == "one_step" else "conservative", **_NEWTON)
