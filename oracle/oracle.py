"""ctypes binding of the plain C oracle (ipm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product path
(paper_1912_09238_b200/).  Shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ORACLE_LIB: a prebuilt oracle library instead of the in-tree one (tests/test_oracle_mutants.py
# points it at deliberately mutated builds to show that the pins catch those mistakes)
LIB = os.environ.get("ORACLE_LIB") or os.path.join(HERE, "libipm_oracle.so")
SRC = os.path.join(HERE, "ipm_oracle.c")
HDR = os.path.join(HERE, "ipm_oracle.h")

CLOSURE = {"quadratic": 0, "barrier": 1, "euler": 2}
FLUX = {"lf_global": 0, "hll": 1, "rusanov": 2}
MESH = {"1d": 0, "cart2d": 1, "tri": 2}
BC = {"transmissive": 0, "state": 1, "slip": 2, "farfield": 3}
IC = {"uniform": 0, "step1d": 1, "quad2d": 2}
NEWTON = {"full": 0, "one_step": 1}
UPDATE = {"conservative": 0, "paper_c": 1}
STATUS = {0: "ok", 1: "nonconvergence", 2: "illconditioned", 3: "linesearch", 4: "inadmissible"}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, OpenMP over cells)."""
    if os.environ.get("ORACLE_LIB"):
        return LIB
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class StateSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim_a", C.c_int32), ("dim_b", C.c_int32), ("pad", C.c_int32),
                ("q0", C.c_double * 6), ("q1", (C.c_double * 3) * 5)]


class Problem(C.Structure):
    _fields_ = [
        ("p", C.c_int32), ("M", C.c_int32), ("q1d", C.c_int32),
        ("m", C.c_int32), ("closure", C.c_int32), ("flux", C.c_int32),
        ("gamma", C.c_double), ("umin", C.c_double), ("umax", C.c_double),
        ("mesh_kind", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
        ("n_vert", C.c_int32), ("n_tri", C.c_int32), ("periodic", C.c_int32),
        ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
        ("vert", C.POINTER(C.c_double)), ("tri", C.POINTER(C.c_int32)), ("tri_tag", C.POINTER(C.c_int32)),
        ("bc_kind", C.c_int32 * 4), ("bc_state", StateSpec * 4),
        ("tau", C.c_double), ("armijo_c", C.c_double),
        ("max_newton", C.c_int32), ("max_halvings", C.c_int32),
        ("newton_mode", C.c_int32), ("update_form", C.c_int32),
        ("cfl", C.c_double),
        ("n_levels", C.c_int32), ("level_M", C.c_int32 * 8), ("pad1", C.c_int32),
        ("delta_dec", C.c_double), ("delta_inc", C.c_double),
        ("n_threads", C.c_int32),
        ("n_retard", C.c_int32), ("retard_level", C.c_int32 * 8), ("retard_eps", C.c_double * 8),
        ("quad_kind", C.c_int32), ("quad_level", C.c_int32),
        ("hessian_kind", C.c_int32), ("lbfgs_m", C.c_int32),
        ("level_q1d", C.c_int32 * 8),
    ]


class ICSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32),
                ("xs0", C.c_double), ("xs1", C.c_double * 3),
                ("ys0", C.c_double), ("ys1", C.c_double * 3),
                ("state", StateSpec * 4)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P, D, I = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32)
        sig = {
            "orc_create": (P, [C.POINTER(Problem)]), "orc_destroy": (None, [P]),
            "orc_N": (C.c_int, [P]), "orc_Q": (C.c_int, [P]), "orc_cells": (C.c_int, [P]),
            "orc_gauss_legendre": (None, [C.c_int, D, D]),
            "orc_clenshaw_curtis": (None, [C.c_int, D, D]),
            "orc_smolyak_cc": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p]), "orc_num_basis": (C.c_int, [C.c_int, C.c_int]),
            "orc_multi_indices": (None, [C.c_int, C.c_int, I]),
            "orc_get_quadrature": (None, [P, D, D, D]), "orc_get_geometry": (None, [P, I, D, D, D]),
            "orc_closure_u": (C.c_int, [P, D, D]), "orc_closure_du": (C.c_int, [P, D, D]),
            "orc_closure_sstar": (C.c_double, [P, D]), "orc_closure_grad_s": (C.c_int, [P, D, D]),
            "orc_euler_paper_grad_s": (None, [C.c_double, C.c_int, D, D]),
            "orc_euler_paper_u": (C.c_int, [C.c_double, C.c_int, D, D]),
            "orc_dual_objective": (C.c_int, [P, C.c_int, D, D, D]),
            "orc_dual_gradient": (C.c_int, [P, C.c_int, D, D, D]),
            "orc_dual_hessian": (C.c_int, [P, C.c_int, D, D]),
            "orc_dual_solve_cell": (C.c_int, [P, C.c_int, C.c_int, D, D, I, D]),
            "orc_moments_from_dual": (C.c_int, [P, C.c_int, D, D]),
            "orc_flux_g": (None, [P, D, D, D, C.c_double, D]),
            "orc_project_ic": (None, [P, C.POINTER(ICSpec), D]),
            "orc_warm_start": (None, [P, D, D]),
            "orc_indicator": (C.c_double, [P, C.c_int, D]),
            "orc_farfield_ghost": (None, [C.c_double, D, D, D, D]),
            "orc_set_levels": (None, [P, I]), "orc_get_levels": (None, [P, I]),
            "orc_retard_stage": (C.c_int, [P]),
            "orc_problem_size": (C.c_size_t, []),
            "orc_lbfgs_direction": (C.c_int, [P, C.c_int, D, D, D, D, C.c_int, D]),
            "orc_lbfgs_jbar": (C.c_int, [P, C.c_int, D, D]),
            "orc_lbfgs_history": (C.c_int, [P, C.c_int, C.c_void_p, C.c_void_p]),
            "orc_lbfgs_reset": (None, [P]),
            "orc_level_rule": (C.c_int, [P, C.c_int, C.c_void_p, C.c_void_p]),
            "orc_sc_init": (None, [P, C.POINTER(ICSpec), D]),
            "orc_sc_step": (C.c_double, [P, D, D, C.c_double, D]),
            "orc_sc_moments": (None, [P, D, D]),
            "orc_dual_solve_all": (None, [P, D, D, I, I, D]),
            "orc_dual_solve_all_ls": (None, [P, D, D, I, I, D, I, I]),
            "orc_compute_dt": (C.c_double, [P, D, C.c_double]),
            "orc_cell_rates": (None, [P, D, D]),
            "orc_flux_update": (None, [P, D, D, D, C.c_double]),
            "orc_step": (C.c_int, [P, D, D, C.c_double, I, I, D, D]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype, f.argtypes = res, args
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def farfield_ghost(gamma, ui, uf, n):
    """characteristic far-field ghost state (reading 37) of interior ui, free stream uf, outward normal n"""
    ui, uf, n = (np.ascontiguousarray(x, np.float64) for x in (ui, uf, n))
    ug = np.zeros(4)
    lib().orc_farfield_ghost(float(gamma), _d(ui), _d(uf), _d(n), _d(ug))
    return ug


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _spec(s: dict | None) -> StateSpec:
    out = StateSpec()
    if s is None:
        return out
    if "freestream" in s:
        f = s["freestream"]
        out.kind, out.dim_a, out.dim_b = 1, f["dim_mach"], f["dim_theta"]
        for k, v in enumerate([f["rho"], f["p"], f["mach0"], f["dmach"], f["theta0_deg"], f["dtheta_deg"]]):
            out.q0[k] = v
        return out
    out.kind = 0
    for k, v in enumerate(s["prim"]):
        out.q0[k] = v
    for (comp, dim), v in s.get("dprim", {}).items():
        out.q1[comp][dim] = v
    return out


def num_basis(p: int, M: int) -> int:
    return lib().orc_num_basis(p, M)


def multi_indices(p: int, M: int) -> np.ndarray:
    n = num_basis(p, M)
    out = np.zeros((n, p), dtype=np.int32)
    lib().orc_multi_indices(p, M, _i(out))
    return out


def clenshaw_curtis(n: int):
    x, w = np.zeros(n), np.zeros(n)
    lib().orc_clenshaw_curtis(n, _d(x), _d(w))
    return x, w


def smolyak_cc(p: int, L: int):
    Q = lib().orc_smolyak_cc(p, L, None, None)
    xi, w = np.zeros((Q, p)), np.zeros(Q)
    lib().orc_smolyak_cc(p, L, xi.ctypes.data, w.ctypes.data)
    return xi, w


def gauss_legendre(q: int):
    x, w = np.zeros(q), np.zeros(q)
    lib().orc_gauss_legendre(q, _d(x), _d(w))
    return x, w


class Oracle:
    """One oracle context for a config dict from inputs/configs.py."""

    def __init__(self, cfg: dict, mesh_arrays=None, n_threads: int = 0):
        L = lib()
        self.cfg = cfg
        P = Problem()
        P.p, P.M, P.q1d, P.m = cfg["p"], cfg["M"], cfg["q1d"], cfg["m"]
        P.closure, P.flux = CLOSURE[cfg["closure"]], FLUX[cfg["flux"]]
        P.gamma, P.umin, P.umax = cfg.get("gamma", 1.4), cfg.get("umin", 0.0), cfg.get("umax", 1.0)
        mesh = cfg["mesh"]
        P.mesh_kind = MESH[mesh["kind"]]
        self._keep = []
        if mesh["kind"] == "tri":
            vert, tri, tags = mesh_arrays
            vert = np.ascontiguousarray(vert, dtype=np.float64)
            tri = np.ascontiguousarray(tri, dtype=np.int32)
            tags = np.ascontiguousarray(tags, dtype=np.int32)
            self._keep += [vert, tri, tags]
            P.n_vert, P.n_tri = vert.shape[0], tri.shape[0]
            P.vert, P.tri, P.tri_tag = _d(vert), _i(tri), _i(tags)
        else:
            P.nx, P.ny = mesh["nx"], mesh.get("ny", 1)
            P.x0, P.x1 = mesh["x0"], mesh["x1"]
            P.y0, P.y1 = mesh.get("y0", 0.0), mesh.get("y1", 1.0)
            P.periodic = int(mesh.get("periodic", False))
        for t, (kind, spec) in enumerate(cfg["bc"]):
            P.bc_kind[t] = BC[kind]
            P.bc_state[t] = _spec(spec)
        P.tau, P.armijo_c = cfg["tau"], cfg["armijo_c"]
        P.max_newton, P.max_halvings = cfg["max_newton"], cfg["max_halvings"]
        P.newton_mode, P.update_form = NEWTON[cfg["newton"]], UPDATE[cfg["update"]]
        P.cfl = cfg["cfl"]
        levels = cfg.get("levels") or []
        P.n_levels = len(levels)
        for k, Mk in enumerate(levels):
            P.level_M[k] = Mk
        P.delta_dec, P.delta_inc = cfg.get("delta_dec", 0.0), cfg.get("delta_inc", 0.0)
        P.n_threads = n_threads
        # quadrature (reading 33): "gl" tensor Gauss-Legendre, "cc" tensor Clenshaw-Curtis (q1d points),
        # "smolyak" sparse grid of nested Clenshaw-Curtis rules of level quad_level
        P.quad_kind = {"gl": 0, "cc": 1, "smolyak": 2}[cfg.get("quad", "gl")]
        P.quad_level = cfg.get("quad_level", 0)
        # dual-solve direction (reading 35): "newton" exact Hessian, "lbfgs" limited-memory BFGS
        P.hessian_kind = {"newton": 0, "lbfgs": 1}[cfg.get("hessian", "newton")]
        P.lbfgs_m = cfg.get("lbfgs_m", 8)
        # per-level nested Clenshaw-Curtis rules (reading 36): points per dimension of every level
        for k, q in enumerate(cfg.get("level_q1d") or []):
            P.level_q1d[k] = q
        # refinement retardation (Alg. 4): [(eps_l, level index cap l*_l), ...]
        retard = cfg.get("retard") or []
        P.n_retard = len(retard)
        for k, (eps, lv) in enumerate(retard):
            P.retard_eps[k], P.retard_level[k] = eps, lv
        self._P = P
        self.ctx = L.orc_create(C.byref(P))
        if not self.ctx:
            raise ValueError("orc_create rejected the problem (per-level rules need nested tensor CC)")
        self.N, self.Q, self.cells, self.m = L.orc_N(self.ctx), L.orc_Q(self.ctx), L.orc_cells(self.ctx), cfg["m"]
        self.p = cfg["p"]
        if levels:
            self.Nl = [num_basis(self.p, Mk) for Mk in levels]
            self.set_levels(np.full(self.cells, cfg.get("initial_level", 0), dtype=np.int32))
        else:
            self.Nl = [self.N]

    def __del__(self):
        try:
            lib().orc_destroy(self.ctx)
        except Exception:
            pass

    # --- accessors -------------------------------------------------------
    def quadrature(self):
        xi, om, Phi = np.zeros((self.Q, self.p)), np.zeros(self.Q), np.zeros((self.Q, self.N))
        lib().orc_get_quadrature(self.ctx, _d(xi), _d(om), _d(Phi))
        return xi, om, Phi

    def geometry(self):
        F = {"1d": 2, "cart2d": 4, "tri": 3}[self.cfg["mesh"]["kind"]]
        nbr = np.zeros((self.cells, F), dtype=np.int32)
        nrm, coef, area = np.zeros((self.cells, F, 2)), np.zeros((self.cells, F)), np.zeros(self.cells)
        lib().orc_get_geometry(self.ctx, _i(nbr), _d(nrm), _d(coef), _d(area))
        return nbr, nrm, coef, area

    def zeros(self):
        return np.zeros((self.cells, self.N, self.m))

    # --- closures ---------------------------------------------------------
    def closure_u(self, Lam):
        Lam = np.ascontiguousarray(Lam, dtype=np.float64)
        u = np.zeros(self.m)
        ok = lib().orc_closure_u(self.ctx, _d(Lam), _d(u))
        return u, bool(ok)

    def closure_du(self, Lam):
        Lam = np.ascontiguousarray(Lam, dtype=np.float64)
        J = np.zeros((self.m, self.m))
        ok = lib().orc_closure_du(self.ctx, _d(Lam), _d(J))
        return J, bool(ok)

    def closure_sstar(self, Lam):
        Lam = np.ascontiguousarray(Lam, dtype=np.float64)
        return lib().orc_closure_sstar(self.ctx, _d(Lam))

    def closure_grad_s(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        L = np.zeros(self.m)
        ok = lib().orc_closure_grad_s(self.ctx, _d(u), _d(L))
        return L, bool(ok)

    # --- dual problem (one cell) ------------------------------------------
    def dual_objective(self, lam, uhat, Nl=None):
        Nl = Nl or self.N
        lam, uhat = np.ascontiguousarray(lam, np.float64), np.ascontiguousarray(uhat, np.float64)
        out = C.c_double()
        lib().orc_dual_objective(self.ctx, Nl, _d(lam), _d(uhat), C.byref(out))
        return out.value

    def dual_gradient(self, lam, uhat, Nl=None):
        Nl = Nl or self.N
        lam, uhat = np.ascontiguousarray(lam, np.float64), np.ascontiguousarray(uhat, np.float64)
        g = np.zeros((Nl, self.m))
        ok = lib().orc_dual_gradient(self.ctx, Nl, _d(lam), _d(uhat), _d(g))
        return g, bool(ok)

    def dual_hessian(self, lam, Nl=None):
        Nl = Nl or self.N
        lam = np.ascontiguousarray(lam, np.float64)
        H = np.zeros((Nl * self.m, Nl * self.m))
        ok = lib().orc_dual_hessian(self.ctx, Nl, _d(lam), _d(H))
        return H, bool(ok)

    def dual_solve_cell(self, uhat, lam0, mode="full", Nl=None):
        Nl = Nl or self.N
        uhat = np.ascontiguousarray(uhat, np.float64)
        lam = np.array(lam0, dtype=np.float64, copy=True, order="C")
        it, crit = C.c_int32(), C.c_double()
        st = lib().orc_dual_solve_cell(self.ctx, Nl, NEWTON[mode], _d(uhat), _d(lam), C.byref(it), C.byref(crit))
        return lam, int(it.value), float(crit.value), int(st)

    # --- L-BFGS dual solve (reading 35, NEXT-4) ---------------------------
    def lbfgs_jbar(self, lam, Nl=None):
        Nl = Nl or self.N
        J = np.zeros((self.m, self.m))
        ok = lib().orc_lbfgs_jbar(self.ctx, Nl, _d(np.ascontiguousarray(lam, np.float64)), _d(J))
        return J, bool(ok)

    def lbfgs_direction(self, lam, g, S, Y, Nl=None):
        """two-loop direction -H g over the pairs S, Y [cnt][n] (newest first)"""
        Nl = Nl or self.N
        n = Nl * self.m
        S = np.ascontiguousarray(S, np.float64).reshape(-1, n)
        Y = np.ascontiguousarray(Y, np.float64).reshape(-1, n)
        d = np.zeros(n)
        ok = lib().orc_lbfgs_direction(self.ctx, Nl, _d(np.ascontiguousarray(lam, np.float64)),
                                       _d(np.ascontiguousarray(g, np.float64)), _d(S), _d(Y), S.shape[0], _d(d))
        return d, bool(ok)

    def lbfgs_history(self, j):
        mh, n = self._P.lbfgs_m, self.N * self.m
        S, Y = np.zeros((mh, n)), np.zeros((mh, n))
        cnt = lib().orc_lbfgs_history(self.ctx, j, S.ctypes.data, Y.ctypes.data)
        return S[:cnt], Y[:cnt]

    def level_rule(self, lvl):
        """(finest-rule node indices, weights) of level lvl's nested rule (reading 36)"""
        Ql = lib().orc_level_rule(self.ctx, lvl, None, None)
        kf, w = np.zeros(Ql, np.int32), np.zeros(Ql)
        lib().orc_level_rule(self.ctx, lvl, kf.ctypes.data, w.ctypes.data)
        return kf, w

    def lbfgs_reset(self):
        lib().orc_lbfgs_reset(self.ctx)

    def moments_from_dual(self, lam, Nl=None):
        Nl = Nl or self.N
        lam = np.ascontiguousarray(lam, np.float64)
        u = np.zeros((Nl, self.m))
        ok = lib().orc_moments_from_dual(self.ctx, Nl, _d(lam), _d(u))
        return u, bool(ok)

    def flux_g(self, ul, ur, n=(1.0, 0.0), dx_over_dt=0.0):
        ul, ur = np.ascontiguousarray(ul, np.float64), np.ascontiguousarray(ur, np.float64)
        n = np.ascontiguousarray(n, np.float64)
        g = np.zeros(self.m)
        lib().orc_flux_g(self.ctx, _d(ul), _d(ur), _d(n), dx_over_dt, _d(g))
        return g

    # --- fields -------------------------------------------------------------
    def _ic_spec(self, ic):
        spec = ICSpec()
        spec.kind = IC[ic["kind"]]
        spec.xs0, spec.ys0 = ic.get("xs0", 0.0), ic.get("ys0", 0.0)
        for d, v in enumerate(ic.get("xs1", ())):
            spec.xs1[d] = v
        for d, v in enumerate(ic.get("ys1", ())):
            spec.ys1[d] = v
        for r, s in enumerate(ic["states"]):
            spec.state[r] = _spec(s)
        return spec

    # --- Stochastic Collocation (reading 32) -------------------
    def sc_init(self, ic: dict | None = None):
        """node states [cells][Q][m] of the IC (cell averages at every quadrature point)"""
        spec = self._ic_spec(ic or self.cfg["ic"])
        U = np.zeros((self.cells, self.Q, self.m))
        lib().orc_sc_init(self.ctx, C.byref(spec), _d(U))
        return U

    def sc_step(self, U, t_remaining=np.inf):
        """one coupled collocation step; returns (new states, dt, residual)"""
        Un = np.zeros_like(U)
        res = C.c_double()
        dt = lib().orc_sc_step(self.ctx, _d(U), _d(Un), float(t_remaining), C.byref(res))
        return Un, dt, res.value

    def sc_moments(self, U):
        u = self.zeros()
        lib().orc_sc_moments(self.ctx, _d(U), _d(u))
        return u

    def project_ic(self, ic: dict | None = None):
        ic = ic or self.cfg["ic"]
        spec = ICSpec()
        spec.kind = IC[ic["kind"]]
        spec.xs0, spec.ys0 = ic.get("xs0", 0.0), ic.get("ys0", 0.0)
        for d, v in enumerate(ic.get("xs1", ())):
            spec.xs1[d] = v
        for d, v in enumerate(ic.get("ys1", ())):
            spec.ys1[d] = v
        for r, s in enumerate(ic["states"]):
            spec.state[r] = _spec(s)
        u = self.zeros()
        lib().orc_project_ic(self.ctx, C.byref(spec), _d(u))
        return u

    def warm_start(self, uhat):
        lam = self.zeros()
        lib().orc_warm_start(self.ctx, _d(np.ascontiguousarray(uhat)), _d(lam))
        return lam

    def set_levels(self, levels):
        lv = np.ascontiguousarray(levels, dtype=np.int32)
        lib().orc_set_levels(self.ctx, _i(lv))

    def indicator(self, lvl, h):
        h = np.ascontiguousarray(h, np.float64)
        return lib().orc_indicator(self.ctx, lvl, _d(h))

    def retard_stage(self) -> int:
        """refinement retardation stage (Algorithm 4)"""
        return lib().orc_retard_stage(self.ctx)

    def levels(self):
        lv = np.zeros(self.cells, dtype=np.int32)
        lib().orc_get_levels(self.ctx, _i(lv))
        return lv

    def dual_solve_all(self, uhat, lam):
        """in-place on lam; returns iters, status, crit"""
        it = np.zeros(self.cells, np.int32)
        st = np.zeros(self.cells, np.int32)
        cr = np.zeros(self.cells)
        lib().orc_dual_solve_all(self.ctx, _d(uhat), _d(lam), _i(it), _i(st), _d(cr))
        return it, st, cr

    def dual_solve_all_ls(self, uhat, lam):
        """in-place on lam; returns iters, status, crit, rejected line-search trials, inadmissible trials"""
        it = np.zeros(self.cells, np.int32)
        st = np.zeros(self.cells, np.int32)
        cr = np.zeros(self.cells)
        hv = np.zeros(self.cells, np.int32)
        ia = np.zeros(self.cells, np.int32)
        lib().orc_dual_solve_all_ls(self.ctx, _d(uhat), _d(lam), _i(it), _i(st), _d(cr), _i(hv), _i(ia))
        return it, st, cr, hv, ia

    def compute_dt(self, lam, t_remaining=np.inf):
        return lib().orc_compute_dt(self.ctx, _d(lam), t_remaining)

    def cell_rates(self, lam):
        r = np.zeros(self.cells)
        lib().orc_cell_rates(self.ctx, _d(np.ascontiguousarray(lam)), _d(r))
        return r

    def flux_update(self, lam, uhat_old, dt):
        new = self.zeros()
        lib().orc_flux_update(self.ctx, _d(lam), _d(uhat_old), _d(new), dt)
        return new

    def step(self, uhat, lam, t_remaining=np.inf):
        """in place on uhat, lam; returns (worst status, iters, status, dt, residual)"""
        it = np.zeros(self.cells, np.int32)
        st = np.zeros(self.cells, np.int32)
        dt, res = C.c_double(), C.c_double()
        w = lib().orc_step(self.ctx, _d(uhat), _d(lam), t_remaining, _i(it), _i(st), C.byref(dt), C.byref(res))
        return int(w), it, st, float(dt.value), float(res.value)

    def run(self, n_steps: int | None = None, t_end: float | None = None, uhat=None, lam=None,
            record=False):
        """Algorithm 1 from the IC (or given state) for n_steps or until t_end."""
        uhat = self.project_ic() if uhat is None else uhat
        lam = self.warm_start(uhat) if lam is None else lam
        t, n, hist = 0.0, 0, []
        t_end = self.cfg.get("t_end") if (t_end is None and n_steps is None) else t_end
        while True:
            if n_steps is not None and n >= n_steps:
                break
            if t_end is not None and t >= t_end * (1 - 1e-14):
                break
            rem = (t_end - t) if t_end is not None else np.inf
            w, it, st, dt, res = self.step(uhat, lam, rem)
            if w != 0:
                raise RuntimeError(f"oracle step {n}: status {STATUS.get(w, w)}")
            t += dt
            n += 1
            if record:
                hist.append((dt, it.copy(), res))
        return uhat, lam, dict(t=t, steps=n, hist=hist)

    # --- stress state -----------------------------------------
    def stress_dual(self, base, z, amp):
        """lambda*_0 = grad s(base); lambda*_{i,a} = (rel|lambda*_{0,a}| + abs) 2^-|i| z_{i,a};
        higher modes scaled so that max_k Lambda_E <= 1/2 lambda*_{0,E} (Euler)."""
        rel, ab = amp
        idx = multi_indices(self.p, self.cfg["M"])
        deg = idx.sum(axis=1)
        _, _, Phi = self.quadrature()
        lam = np.zeros((self.cells, self.N, self.m))
        for j in range(self.cells):
            l0, ok = self.closure_grad_s(base[j])
            assert ok
            lam[j, 0] = l0
            for i in range(1, self.N):
                lam[j, i] = (rel * np.abs(l0) + ab) * 2.0 ** (-deg[i]) * z[j, i]
            if self.cfg["closure"] == "euler":
                hi = Phi[:, 1:] @ lam[j, 1:, self.m - 1]
                r = hi.max()
                lim = 0.5 * abs(l0[self.m - 1])
                if r > lim:
                    lam[j, 1:] *= lim / r
        return lam

    def moments_from_dual_all(self, lam):
        out = self.zeros()
        for j in range(self.cells):
            u, ok = self.moments_from_dual(lam[j])
            assert ok
            out[j] = u
        return out
