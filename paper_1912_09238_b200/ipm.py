"""Thin ctypes binding of libipm (include/ipm.h).  Argument marshalling only: every step of the
path runs in the CUDA kernels behind the C-ABI; there is no CPU fallback.

Names follow the C entry points (ipm_init, ipm_dual_solve, ipm_flux_update, ipm_step, ...).
Device arrays are torch tensors (float64, contiguous, on the context's device); PyTorch is used
only for device memory, streams and torch.distributed.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IPM_LIB", os.path.join(HERE, "libipm.so"))

CLOSURE = {"quadratic": 0, "barrier": 1, "euler": 2}
FLUX = {"lf_global": 0, "hll": 1, "rusanov": 2}
MESH = {"1d": 0, "cart2d": 1, "tri": 2}
BC = {"transmissive": 0, "state": 1, "slip": 2, "farfield": 3}
NEWTON = {"full": 0, "one_step": 1}
UPDATE = {"conservative": 0, "paper_c": 1}
IC = {"uniform": 0, "step1d": 1, "quad2d": 2}
CELL_STATUS = {0: "ok", 1: "nonconvergence", 2: "illconditioned", 3: "linesearch", 4: "inadmissible"}

EXPORTS = [
    "ipm_init", "ipm_destroy", "ipm_status_string", "ipm_last_error", "ipm_sizes", "ipm_get_basis",
    "ipm_get_cell_ids", "ipm_dual_solve", "ipm_flux_update", "ipm_step", "ipm_step_host", "ipm_sc_init", "ipm_sc_step", "ipm_sc_moments", "ipm_project_ic", "ipm_warm_start",
    "ipm_moments_from_dual", "ipm_stress_dual", "ipm_get_levels", "ipm_set_levels", "ipm_last_cell_stats",
    "ipm_get_time", "ipm_set_time", "ipm_last_kernel_ms", "ipm_enable_timing", "ipm_last_dual_kernel", "ipm_last_flux_kernel", "ipm_struct_size", "ipm_retard_stage", "ipm_retard_advance",
    "ipm_debug_phase_cycles", "ipm_step_dual", "ipm_step_flux", "ipm_halo_layout", "ipm_partition_query",
    "ipm_get_status", "ipm_last_cell_linesearch", "ipm_node_band_rows", "ipm_lbfgs_reset", "ipm_lbfgs_history",
    "ipm_step_dual_boundary", "ipm_step_dual_interior",
]
HIST_BUCKETS = 16  # IPM_HIST_BUCKETS


class IPMError(RuntimeError):
    pass


class ipm_state(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim_a", C.c_int32), ("dim_b", C.c_int32), ("reserved", C.c_int32),
                ("q0", C.c_double * 6), ("q1", (C.c_double * 3) * 5)]


class ipm_config(C.Structure):
    _fields_ = [
        ("p", C.c_int32), ("M", C.c_int32), ("q1d", C.c_int32), ("m", C.c_int32),
        ("closure", C.c_int32), ("flux", C.c_int32),
        ("gamma", C.c_double), ("u_minus", C.c_double), ("u_plus", C.c_double),
        ("mesh_kind", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("periodic", C.c_int32),
        ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
        ("n_vert", C.c_int32), ("n_tri", C.c_int32),
        ("h_vert", C.c_void_p), ("h_tri", C.c_void_p), ("h_tri_tag", C.c_void_p),
        ("bc_kind", C.c_int32 * 4), ("bc_state", ipm_state * 4),
        ("tau", C.c_double), ("armijo_c", C.c_double),
        ("max_newton", C.c_int32), ("max_halvings", C.c_int32),
        ("newton_mode", C.c_int32), ("update_form", C.c_int32),
        ("cfl", C.c_double),
        ("n_levels", C.c_int32), ("level_M", C.c_int32 * 8),
        ("delta_dec", C.c_double), ("delta_inc", C.c_double),
        ("rank", C.c_int32), ("nranks", C.c_int32), ("px", C.c_int32), ("py", C.c_int32),
        ("reserved_ptr", C.c_void_p), ("stream", C.c_void_p),
        ("n_retard", C.c_int32), ("retard_level", C.c_int32 * 8), ("retard_eps", C.c_double * 8),
        ("quad_kind", C.c_int32), ("quad_level", C.c_int32),
        ("hessian_kind", C.c_int32), ("lbfgs_m", C.c_int32),
        ("level_q1d", C.c_int32 * 8),
    ]


class ipm_step_info(C.Structure):
    _fields_ = [("dt", C.c_double), ("t", C.c_double), ("residual", C.c_double),
                ("newton_iters", C.c_int64), ("failed_cells", C.c_int64),
                ("worst_status", C.c_int32), ("reserved", C.c_int32),
                ("newton_hist", C.c_int64 * HIST_BUCKETS), ("halvings", C.c_int64),
                ("inadmissible_trials", C.c_int64)]


class ipm_ic(C.Structure):
    _fields_ = [("kind", C.c_int32), ("initial_level", C.c_int32),
                ("xs0", C.c_double), ("xs1", C.c_double * 3), ("ys0", C.c_double), ("ys1", C.c_double * 3),
                ("state", ipm_state * 4)]


_lib = None


def lib():
    """Load libipm.so (built in-tree by paper_1912_09238_b200/build.py).  Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise IPMError(f"libipm.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P, D, I = C.c_void_p, C.c_void_p, C.c_void_p
        st = C.c_int
        sig = {
            "ipm_init": (st, [C.POINTER(ipm_config), C.POINTER(C.c_void_p)]),
            "ipm_destroy": (None, [P]),
            "ipm_status_string": (C.c_char_p, [C.c_int]),
            "ipm_last_error": (C.c_char_p, []),
            "ipm_sizes": (st, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                               C.POINTER(C.c_int32)]),
            "ipm_get_basis": (st, [P, D, D, D]),
            "ipm_get_cell_ids": (st, [P, P]),
            "ipm_dual_solve": (st, [P, D, D, C.c_int32, I, I, D]),
            "ipm_flux_update": (st, [P, D, D, D, C.c_double, D]),
            "ipm_step": (st, [P, D, D, C.c_double, C.POINTER(ipm_step_info)]),
            "ipm_step_host": (st, [P, D, D, D, D, C.c_double, C.c_int32, C.POINTER(ipm_step_info)]),
            "ipm_project_ic": (st, [P, C.POINTER(ipm_ic), D]),
            "ipm_sc_init": (st, [P, C.POINTER(ipm_ic), D]),
            "ipm_sc_step": (st, [P, D, D, C.c_double, C.POINTER(ipm_step_info)]),
            "ipm_sc_moments": (st, [P, D, D]),
            "ipm_warm_start": (st, [P, D, D]),
            "ipm_moments_from_dual": (st, [P, D, D]),
            "ipm_stress_dual": (st, [P, D, D, C.c_double, C.c_double, D]),
            "ipm_get_levels": (st, [P, I]),
            "ipm_set_levels": (st, [P, I]),
            "ipm_last_cell_stats": (st, [P, I, I]),
            "ipm_get_time": (st, [P, C.POINTER(C.c_double)]),
            "ipm_set_time": (st, [P, C.c_double]),
            "ipm_step_dual": (st, [P, D, D, D, D]),
            "ipm_step_flux": (st, [P, D, D, D, D, C.c_double, C.POINTER(ipm_step_info)]),
            "ipm_halo_layout": (st, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64), P, P, P]),
            "ipm_partition_query": (st, [C.POINTER(ipm_config), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int64), P, P, P, P, P, P]),
            "ipm_last_kernel_ms": (st, [P, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
            "ipm_enable_timing": (st, [P, C.c_int32]),
            "ipm_last_dual_kernel": (C.c_char_p, []),
            "ipm_last_flux_kernel": (C.c_char_p, []),
            "ipm_struct_size": (C.c_size_t, [C.c_int32]),
            "ipm_retard_stage": (st, [P, C.POINTER(C.c_int32)]),
            "ipm_retard_advance": (st, [P, C.c_double]),
            "ipm_debug_phase_cycles": (st, [P]),
            "ipm_get_status": (st, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
            "ipm_last_cell_linesearch": (st, [P, I, I]),
            "ipm_node_band_rows": (st, [P, C.POINTER(C.c_int64)]),
            "ipm_lbfgs_reset": (st, [P]),
            "ipm_lbfgs_history": (st, [P, P, P, P]),
            "ipm_step_dual_boundary": (st, [P, P, P, P]),
            "ipm_step_dual_interior": (st, [P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        for which, st_ in ((0, ipm_config), (1, ipm_ic), (2, ipm_step_info)):
            if L.ipm_struct_size(which) != C.sizeof(st_):
                raise IPMError(f"struct mirror {st_.__name__} ({C.sizeof(st_)} B) does not match libipm "
                               f"({L.ipm_struct_size(which)} B): rebuild libipm.so")
        _lib = L
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise IPMError(f"{what}: {L.ipm_status_string(rc).decode()}: {L.ipm_last_error().decode()}")


def _state(s: dict | None) -> ipm_state:
    out = ipm_state()
    if s is None:
        return out
    if "freestream" in s:
        f = s["freestream"]
        out.kind, out.dim_a, out.dim_b = 1, f["dim_mach"], f["dim_theta"]
        for k, v in enumerate([f["rho"], f["p"], f["mach0"], f["dmach"], f["theta0_deg"], f["dtheta_deg"]]):
            out.q0[k] = v
        return out
    for k, v in enumerate(s["prim"]):
        out.q0[k] = v
    for (comp, dim), v in s.get("dprim", {}).items():
        out.q1[comp][dim] = v
    return out


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _dev(t, ctx, shape, dtype, name):
    """device pointer of a tensor argument after checking what the C-ABI assumes (ipm.h conventions):
    dtype, contiguity, the context's device and the element count; None passes NULL"""
    if t is None:
        return 0
    if t.dtype != dtype:
        raise IPMError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise IPMError(f"{name}: not contiguous")
    if t.device != ctx.device:
        raise IPMError(f"{name}: on {t.device}, the context is on {ctx.device}")
    n = 1
    for d in shape:
        n *= d
    if t.numel() != n:
        raise IPMError(f"{name}: {t.numel()} elements, expected {n} {tuple(shape)}")
    return t.data_ptr()


def _host(t, shape, name):
    """host tensor of the ipm_step_host path: float64, contiguous, CPU, page-locked"""
    if t.dtype.is_floating_point is False or t.element_size() != 8 or t.device.type != "cpu":
        raise IPMError(f"{name}: expected a float64 CPU tensor")
    if not t.is_contiguous() or not t.is_pinned():
        raise IPMError(f"{name}: must be contiguous and pinned (pin_memory()) for the overlapped copies")
    n = 1
    for d in shape:
        n *= d
    if t.numel() != n:
        raise IPMError(f"{name}: {t.numel()} elements, expected {n}")
    return t.data_ptr()


def make_config(cfg: dict, mesh_arrays=None, rank=0, nranks=1, px=1, py=1):
    """ipm_config for a config dict (inputs/configs.py format); returns (config, arrays to keep alive)."""
    c = ipm_config()
    keep = []
    c.p, c.M, c.q1d, c.m = cfg["p"], cfg["M"], cfg["q1d"], cfg["m"]
    c.closure, c.flux = CLOSURE[cfg["closure"]], FLUX[cfg["flux"]]
    c.gamma, c.u_minus, c.u_plus = cfg.get("gamma", 1.4), cfg.get("umin", 0.0), cfg.get("umax", 1.0)
    mesh = cfg["mesh"]
    c.mesh_kind = MESH[mesh["kind"]]
    if mesh["kind"] == "tri":
        vert, tri, tags = mesh_arrays
        vert = np.ascontiguousarray(vert, np.float64)
        tri = np.ascontiguousarray(tri, np.int32)
        tags = np.ascontiguousarray(tags, np.int32)
        keep += [vert, tri, tags]
        c.n_vert, c.n_tri = vert.shape[0], tri.shape[0]
        c.h_vert, c.h_tri, c.h_tri_tag = vert.ctypes.data, tri.ctypes.data, tags.ctypes.data
    else:
        c.nx, c.ny = mesh["nx"], mesh.get("ny", 1)
        c.x0, c.x1 = mesh["x0"], mesh["x1"]
        c.y0, c.y1 = mesh.get("y0", 0.0), mesh.get("y1", 1.0)
        c.periodic = int(mesh.get("periodic", False))
    for t, (kind, spec) in enumerate(cfg["bc"]):
        c.bc_kind[t] = BC[kind]
        c.bc_state[t] = _state(spec)
    c.tau, c.armijo_c = cfg["tau"], cfg["armijo_c"]
    c.max_newton, c.max_halvings = cfg["max_newton"], cfg["max_halvings"]
    c.newton_mode, c.update_form = NEWTON[cfg["newton"]], UPDATE[cfg["update"]]
    c.cfl = cfg["cfl"]
    levels = cfg.get("levels") or []
    c.n_levels = len(levels)
    for k, Mk in enumerate(levels):
        c.level_M[k] = Mk
    c.delta_dec, c.delta_inc = cfg.get("delta_dec", 0.0), cfg.get("delta_inc", 0.0)
    c.quad_kind = {"gl": 0, "cc": 1, "smolyak": 2}[cfg.get("quad", "gl")]  # quadrature (reading 33)
    c.quad_level = cfg.get("quad_level", 0)
    # dual-solve direction (reading 35): "newton" exact Hessian (default), "lbfgs" limited-memory BFGS
    c.hessian_kind = {"newton": 0, "lbfgs": 1}[cfg.get("hessian", "newton")]
    c.lbfgs_m = cfg.get("lbfgs_m", 8)
    # per-level nested Clenshaw-Curtis rules (reading 36)
    for k, q in enumerate(cfg.get("level_q1d") or []):
        c.level_q1d[k] = q
    retard = cfg.get("retard") or []  # refinement retardation (Alg. 4): [(eps_l, level index cap), ...]
    c.n_retard = len(retard)
    for k, (eps, lv) in enumerate(retard):
        c.retard_eps[k], c.retard_level[k] = eps, lv
    c.rank, c.nranks, c.px, c.py = rank, nranks, px, py
    return c, keep


def partition_query(cfg: dict, rank: int, nranks: int, px: int = 0, py: int = 0, mesh_arrays=None) -> dict:
    """Host-only: the partition libipm builds for this rank (no CUDA needed)."""
    c, keep = make_config(cfg, mesh_arrays, rank, nranks, px, py)
    cells, nhalo, nsend = C.c_int64(), C.c_int64(), C.c_int64()
    npeers = C.c_int32()
    L = lib()
    check(L.ipm_partition_query(C.byref(c), C.byref(cells), C.byref(nhalo), C.byref(npeers), C.byref(nsend),
                                None, None, None, None, None, None), "ipm_partition_query")
    local = np.zeros(cells.value, np.int64)
    halo = np.zeros(nhalo.value, np.int64)
    send = np.zeros(nsend.value, np.int64)
    peers = np.zeros(npeers.value, np.int32)
    sc = np.zeros(npeers.value, np.int32)
    rc = np.zeros(npeers.value, np.int32)
    check(L.ipm_partition_query(C.byref(c), C.byref(cells), C.byref(nhalo), C.byref(npeers), C.byref(nsend),
                                local.ctypes.data, halo.ctypes.data, peers.ctypes.data, sc.ctypes.data,
                                rc.ctypes.data, send.ctypes.data), "ipm_partition_query")
    return dict(local=local, halo=halo, send=send, peers=peers, send_count=sc, recv_count=rc)


class Context:
    """One libipm context for a config dict (inputs/configs.py format)."""

    def __init__(self, cfg: dict, mesh_arrays=None, device=None, stream=None, rank=0, nranks=1, px=1, py=1,
                 group=None):
        import torch

        self.torch = torch
        self.cfg = cfg
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        c, self._keep = make_config(cfg, mesh_arrays, rank, nranks, px, py)
        self.rank, self.nranks, self.group = rank, nranks, group
        c.stream = self.stream.cuda_stream
        self._c = c
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(lib().ipm_init(C.byref(c), C.byref(h)), "ipm_init")
        self.h = h
        cells, N, Q, m = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        check(lib().ipm_sizes(h, C.byref(cells), C.byref(N), C.byref(Q), C.byref(m)), "ipm_sizes")
        self.cells, self.N, self.Q, self.m = cells.value, N.value, Q.value, m.value

    def close(self):
        if getattr(self, "h", None):
            lib().ipm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- arrays -----------------------------------------------------------------------------
    def zeros(self, *shape, dtype=None):
        t = self.torch
        shape = shape or (self.cells, self.N, self.m)
        return t.zeros(shape, dtype=dtype or t.float64, device=self.device)

    def basis(self):
        p = self.cfg["p"]
        xi, om, phi = np.zeros((self.Q, p)), np.zeros(self.Q), np.zeros((self.Q, self.N))
        check(lib().ipm_get_basis(self.h, xi.ctypes.data, om.ctypes.data, phi.ctypes.data), "ipm_get_basis")
        return xi, om, phi

    def cell_ids(self):
        ids = np.zeros(self.cells, np.int64)
        check(lib().ipm_get_cell_ids(self.h, ids.ctypes.data), "ipm_get_cell_ids")
        return ids

    # --- the path ---------------------------------------------------------------------------
    def _state(self, t, name):
        return _dev(t, self, (self.cells, self.N, self.m), self.torch.float64, name)

    def _cellv(self, t, name, dtype=None):
        return _dev(t, self, (self.cells,), dtype or self.torch.int32, name)

    def ipm_dual_solve(self, uhat, lam, mode=None, iters=None, status=None, crit=None):
        mode = NEWTON[mode or self.cfg["newton"]]
        with self.torch.cuda.device(self.device):
            check(lib().ipm_dual_solve(self.h, self._state(uhat, "uhat"), self._state(lam, "lambda"), mode,
                                       self._cellv(iters, "iters"), self._cellv(status, "status"),
                                       self._cellv(crit, "crit", self.torch.float64)), "ipm_dual_solve")

    def ipm_flux_update(self, lam, uhat_old, uhat_new, dt=-1.0, dt_out=None):
        with self.torch.cuda.device(self.device):
            check(lib().ipm_flux_update(self.h, self._state(lam, "lambda"), self._state(uhat_old, "uhat_old"),
                                        self._state(uhat_new, "uhat_new"), float(dt),
                                        _dev(dt_out, self, (1,), self.torch.float64, "dt_out")), "ipm_flux_update")

    def node_band_rows(self) -> int:
        """0: whole node-state buffer; else rows per band of the banded node states"""
        r = C.c_int64()
        check(lib().ipm_node_band_rows(self.h, C.byref(r)), "ipm_node_band_rows")
        return r.value

    def get_status(self):
        """(worst ipm_cell_status, failed cells) of the last dual solve (synchronous, ipm_get_status)"""
        w, n = C.c_int32(), C.c_int64()
        check(lib().ipm_get_status(self.h, C.byref(w), C.byref(n)), "ipm_get_status")
        return w.value, n.value

    def lbfgs_reset(self):
        """forget every cell's L-BFGS pairs (hessian="lbfgs" contexts)"""
        check(lib().ipm_lbfgs_reset(self.h), "ipm_lbfgs_reset")

    def lbfgs_history(self):
        """(S, Y [cells][lbfgs_m][N m], count [cells]) of the L-BFGS pairs, newest first"""
        mh = self.cfg.get("lbfgs_m", 8)
        S = self.zeros(self.cells, mh, self.N * self.m)
        Y = self.zeros(self.cells, mh, self.N * self.m)
        cnt = self.zeros(self.cells, dtype=self.torch.int32)
        check(lib().ipm_lbfgs_history(self.h, _ptr(S), _ptr(Y), _ptr(cnt)), "ipm_lbfgs_history")
        return S, Y, cnt

    def last_cell_linesearch(self):
        """per-cell (rejected Armijo trials, inadmissible trials) of the last dual solve"""
        hv = self.zeros(self.cells, dtype=self.torch.int32)
        ia = self.zeros(self.cells, dtype=self.torch.int32)
        check(lib().ipm_last_cell_linesearch(self.h, _ptr(hv), _ptr(ia)), "ipm_last_cell_linesearch")
        return hv, ia

    def _halo_setup(self):
        npeers, nsend, nrecv = C.c_int32(), C.c_int64(), C.c_int64()
        check(lib().ipm_halo_layout(self.h, C.byref(npeers), C.byref(nsend), C.byref(nrecv), None, None, None),
              "ipm_halo_layout")
        peers = np.zeros(npeers.value, np.int32)
        sc = np.zeros(npeers.value, np.int32)
        rc = np.zeros(npeers.value, np.int32)
        check(lib().ipm_halo_layout(self.h, C.byref(npeers), C.byref(nsend), C.byref(nrecv), peers.ctypes.data,
                                    sc.ctypes.data, rc.ctypes.data), "ipm_halo_layout")
        t = self.torch
        row = self.N * self.m
        self.halo = dict(peers=peers.tolist(), send_count=sc.tolist(), recv_count=rc.tolist())
        self.sendbuf = t.zeros((max(int(nsend.value), 1), row), dtype=t.float64, device=self.device)
        self.recvbuf = t.zeros((max(int(nrecv.value), 1), row), dtype=t.float64, device=self.device)
        self.rate = t.zeros(1, dtype=t.int64, device=self.device)

    def ipm_step(self, uhat, lam, t_end=None, sync=True):
        """One step; for nranks > 1 the halo exchange and the dt all-reduce run in between
        (paper_1912_09238_b200.dist, torch.distributed)."""
        info = ipm_step_info() if sync else None
        te = -1.0 if t_end is None else float(t_end)
        pu, pl = self._state(uhat, "uhat"), self._state(lam, "lambda")
        if self.nranks <= 1:
            with self.torch.cuda.device(self.device):
                rc = lib().ipm_step(self.h, pu, pl, te, C.byref(info) if sync else None)
        else:
            from . import dist

            if not hasattr(self, "sendbuf"):
                self._halo_setup()
            # boundary cells first; their duals travel while the interior cells solve
            check(lib().ipm_step_dual_boundary(self.h, pu, pl, _ptr(self.sendbuf)), "ipm_step_dual_boundary")
            reqs = dist.halo_exchange(self.sendbuf, self.recvbuf, self.halo, self.group, async_op=True)
            check(lib().ipm_step_dual_interior(self.h, pu, pl, _ptr(self.rate)), "ipm_step_dual_interior")
            dist.wait_all(reqs)
            dist.allreduce_max_(self.rate, self.group)
            rc = lib().ipm_step_flux(self.h, pu, pl, _ptr(self.recvbuf), _ptr(self.rate), te,
                                     C.byref(info) if sync else None)
            if sync and rc in (0, 5):
                # this rank's own count, before info becomes the global sums (bench: imbalance)
                self.last_local_newton_iters = int(info.newton_iters)
                dist.reduce_info_(info, self.device, self.group)
                rc = 5 if info.failed_cells else 0
                if self.cfg.get("retard"):  # Alg. 4 stage from the global residual
                    check(lib().ipm_retard_advance(self.h, info.residual), "ipm_retard_advance")
        if rc == 5:  # IPM_ERR_NUMERIC: report, caller decides
            return info
        check(rc, "ipm_step")
        return info

    def retard_stage(self) -> int:
        """current refinement retardation stage (Algorithm 4)"""
        st = C.c_int32()
        check(lib().ipm_retard_stage(self.h, C.byref(st)), "ipm_retard_stage")
        return st.value

    def ipm_step_host(self, h_uhat, h_lam, d_uhat, d_lam, t_end=None, nchunks=32):
        """One step with the state in (pinned) host tensors h_uhat / h_lam, d_uhat / d_lam device work
        buffers; copies overlapped with the dual solves in nchunks cell ranges (synchronous)."""
        info = ipm_step_info()
        te = -1.0 if t_end is None else float(t_end)
        shape = (self.cells, self.N, self.m)
        with self.torch.cuda.device(self.device):
            rc = lib().ipm_step_host(self.h, _host(h_uhat, shape, "h_uhat"), _host(h_lam, shape, "h_lambda"),
                                     self._state(d_uhat, "d_uhat"), self._state(d_lam, "d_lambda"), te, int(nchunks),
                                     C.byref(info))
        if rc == 5:
            return info
        check(rc, "ipm_step_host")
        return info

    # --- helpers ----------------------------------------------------------------------------
    def _ic(self, ic):
        s = ipm_ic()
        s.kind = IC[ic["kind"]]
        s.initial_level = self.cfg.get("initial_level", 0)
        s.xs0, s.ys0 = ic.get("xs0", 0.0), ic.get("ys0", 0.0)
        for d, v in enumerate(ic.get("xs1", ())):
            s.xs1[d] = v
        for d, v in enumerate(ic.get("ys1", ())):
            s.ys1[d] = v
        for r, st in enumerate(ic["states"]):
            s.state[r] = _state(st)
        return s

    # --- Stochastic Collocation (ipm.h ipm_sc_*) ----------------------------------------------
    def sc_zeros(self):
        """node-state buffer [cells][m][Q]"""
        return self.torch.zeros((self.cells, self.m, self.Q), dtype=self.torch.float64, device=self.device)

    def ipm_sc_init(self, nodes, ic: dict | None = None):
        check(lib().ipm_sc_init(self.h, C.byref(self._ic(ic or self.cfg["ic"])), _ptr(nodes)), "ipm_sc_init")

    def ipm_sc_step(self, nodes_in, nodes_out, t_end=None, sync=True):
        info = ipm_step_info() if sync else None
        te = -1.0 if t_end is None else float(t_end)
        check(lib().ipm_sc_step(self.h, _ptr(nodes_in), _ptr(nodes_out), te, C.byref(info) if sync else None),
              "ipm_sc_step")
        return info

    def ipm_sc_moments(self, nodes, uhat):
        check(lib().ipm_sc_moments(self.h, _ptr(nodes), _ptr(uhat)), "ipm_sc_moments")

    def ipm_project_ic(self, uhat, ic: dict | None = None):
        ic = ic or self.cfg["ic"]
        s = ipm_ic()
        s.kind = IC[ic["kind"]]
        s.initial_level = self.cfg.get("initial_level", 0)
        s.xs0, s.ys0 = ic.get("xs0", 0.0), ic.get("ys0", 0.0)
        for d, v in enumerate(ic.get("xs1", ())):
            s.xs1[d] = v
        for d, v in enumerate(ic.get("ys1", ())):
            s.ys1[d] = v
        for r, st in enumerate(ic["states"]):
            s.state[r] = _state(st)
        check(lib().ipm_project_ic(self.h, C.byref(s), self._state(uhat, "uhat")), "ipm_project_ic")

    def ipm_warm_start(self, uhat, lam):
        check(lib().ipm_warm_start(self.h, self._state(uhat, "uhat"), self._state(lam, "lambda")), "ipm_warm_start")

    def ipm_moments_from_dual(self, lam, uhat):
        check(lib().ipm_moments_from_dual(self.h, self._state(lam, "lambda"), self._state(uhat, "uhat")),
              "ipm_moments_from_dual")

    def ipm_stress_dual(self, base, z, rel, abs_, lam):
        check(lib().ipm_stress_dual(self.h, _ptr(base), _ptr(z), float(rel), float(abs_), _ptr(lam)),
              "ipm_stress_dual")

    def levels(self):
        out = self.zeros(self.cells, dtype=self.torch.int32)
        check(lib().ipm_get_levels(self.h, _ptr(out)), "ipm_get_levels")
        return out

    def set_levels(self, lv):
        check(lib().ipm_set_levels(self.h, _ptr(lv)), "ipm_set_levels")

    def last_cell_stats(self):
        it = self.zeros(self.cells, dtype=self.torch.int32)
        st = self.zeros(self.cells, dtype=self.torch.int32)
        check(lib().ipm_last_cell_stats(self.h, _ptr(it), _ptr(st)), "ipm_last_cell_stats")
        return it, st

    def time(self):
        t = C.c_double()
        check(lib().ipm_get_time(self.h, C.byref(t)), "ipm_get_time")
        return t.value

    def set_time(self, t):
        check(lib().ipm_set_time(self.h, float(t)), "ipm_set_time")

    def enable_timing(self, on=True):
        check(lib().ipm_enable_timing(self.h, int(on)), "ipm_enable_timing")

    @staticmethod
    def last_dual_kernel() -> str:
        """name of the dual kernel of the last launch (process-wide)"""
        return lib().ipm_last_dual_kernel().decode()

    @staticmethod
    def last_flux_kernel() -> str:
        """name of the flux kernel of the last launch (process-wide)"""
        return lib().ipm_last_flux_kernel().decode()

    def last_kernel_ms(self):
        a, b = C.c_float(), C.c_float()
        check(lib().ipm_last_kernel_ms(self.h, C.byref(a), C.byref(b)), "ipm_last_kernel_ms")
        return a.value, b.value

    def debug_phase_cycles(self):
        out = np.zeros(8, np.uint64)
        check(lib().ipm_debug_phase_cycles(out.ctypes.data), "ipm_debug_phase_cycles")
        return out

    def run(self, uhat=None, lam=None, t_end=None, n_steps=None, record=False):
        """Algorithm 1 from the IC (or a given state) until t_end or for n_steps (synchronous steps)."""
        if uhat is None:
            uhat = self.zeros()
            self.ipm_project_ic(uhat)
        if lam is None:
            lam = self.zeros()
            self.ipm_warm_start(uhat, lam)
        t_end = self.cfg.get("t_end") if (t_end is None and n_steps is None) else t_end
        hist, n, t = [], 0, self.time()
        while True:
            if n_steps is not None and n >= n_steps:
                break
            if t_end is not None and t >= t_end * (1 - 1e-14):
                break
            info = self.ipm_step(uhat, lam, t_end)
            if info.failed_cells:
                raise IPMError(f"step {n}: {info.failed_cells} failed cells, worst "
                               f"{CELL_STATUS.get(info.worst_status)}")
            t = info.t
            n += 1
            if record:
                it, _ = self.last_cell_stats()
                hist.append((info.dt, it.cpu().numpy(), info.residual))
        return uhat, lam, dict(t=t, steps=n, hist=hist)
