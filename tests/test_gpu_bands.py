"""Banded node states (ipm_api.cu band_flux; the memory-light flux path that makes config 5 at
4096^2 fit one B200: its whole [cells][m][Q] node-state buffer would be 537 GB).  The node states are
recomputed from lambda band by band (k_nodes) and the flux runs on each band's cells; the result must
match the whole-buffer path and the oracle (1e-9, reading 27), single context and virtual ranks."""
import os

import numpy as np
import pytest

from inputs import configs

from .gpu_common import assert_moments_close, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("GPU test needs CUDA (no CPU fallback exists)")
    return t


def ctx(cfg, band_rows=None, **kw):
    from paper_1912_09238_b200 import Context

    old = os.environ.get("IPM_BAND_ROWS")
    if band_rows:
        os.environ["IPM_BAND_ROWS"] = str(band_rows)
    try:
        return Context(cfg, **kw)
    finally:
        if old is None:
            os.environ.pop("IPM_BAND_ROWS", None)
        else:
            os.environ["IPM_BAND_ROWS"] = old


@pytest.mark.parametrize("name,nx,ny,rows,steps", [("cfg5", 12, 10, 3, 3), ("cfg3", 24, 20, 5, 8), ("cfg3", 24, 20, 1, 3)])
def test_banded_node_states_match_whole_buffer_and_oracle(torch, name, nx, ny, rows, steps):
    import oracle

    cfg = configs.get(name, mesh=dict(nx=nx, ny=ny))
    whole = ctx(cfg)
    band = ctx(cfg, rows)
    assert whole.node_band_rows() == 0 and band.node_band_rows() == rows
    u_w, _, iw = whole.run(n_steps=steps)
    u_b, _, ib = band.run(n_steps=steps)
    assert abs(iw["t"] - ib["t"]) <= 1e-13 * iw["t"]
    np.testing.assert_allclose(to_np(u_b), to_np(u_w), rtol=0, atol=1e-12 * np.abs(to_np(u_w)).max())
    u_o, _, _ = oracle.Oracle(cfg).run(n_steps=steps)
    assert_moments_close(to_np(u_b), u_o, 1e-9, f"{name} bands of {rows} rows")


def test_banded_flux_update_entry_point(torch):
    """ipm_flux_update (separate output array) in band mode = whole-buffer mode"""
    cfg = configs.get("cfg3", mesh=dict(nx=16, ny=12))
    out = []
    for rows in (None, 4):
        g = ctx(cfg, rows)
        u = g.zeros()
        g.ipm_project_ic(u)
        lam = g.zeros()
        g.ipm_warm_start(u, lam)
        g.ipm_dual_solve(u, lam)
        new = g.zeros()
        g.ipm_flux_update(lam, u, new)
        out.append(to_np(new))
    np.testing.assert_allclose(out[1], out[0], rtol=0, atol=1e-12 * np.abs(out[0]).max())


def test_banded_virtual_ranks(torch):
    """2 x 1 ranks on one GPU, each with bands of 3 rows and its halo buffer, against one context"""
    from paper_1912_09238_b200.ipm import _ptr, check, ipm_step_info, lib

    import ctypes as C

    cfg = configs.get("cfg3", mesh=dict(nx=16, ny=14))
    ref = ctx(cfg)
    u_ref, _, _ = ref.run(n_steps=4, t_end=1e9)
    ctxs, us, lams = [], [], []
    for r in range(2):
        g = ctx(cfg, 3, rank=r, nranks=2, px=2, py=1)
        assert g.node_band_rows() == 3
        g._halo_setup()
        u = g.zeros()
        g.ipm_project_ic(u)
        lam = g.zeros()
        g.ipm_warm_start(u, lam)
        ctxs.append(g)
        us.append(u)
        lams.append(lam)
    L = lib()
    for _ in range(4):
        for g, u, lam in zip(ctxs, us, lams):
            check(L.ipm_step_dual(g.h, _ptr(u), _ptr(lam), _ptr(g.sendbuf), _ptr(g.rate)), "ipm_step_dual")
        torch.cuda.synchronize()
        for r, g in enumerate(ctxs):
            s0 = 0
            for p, ns in zip(g.halo["peers"], g.halo["send_count"]):
                gp = ctxs[p]
                k = gp.halo["peers"].index(r)
                r0 = sum(gp.halo["recv_count"][:k])
                gp.recvbuf[r0:r0 + ns].copy_(g.sendbuf[s0:s0 + ns])
                s0 += ns
        rate = torch.stack([g.rate for g in ctxs]).max()
        for g in ctxs:
            g.rate.copy_(rate.reshape(1))
        for g, u, lam in zip(ctxs, us, lams):
            info = ipm_step_info()
            check(L.ipm_step_flux(g.h, _ptr(u), _ptr(lam), _ptr(g.recvbuf), _ptr(g.rate), 1e9, C.byref(info)),
                  "ipm_step_flux")
    ur = to_np(u_ref)
    for g, u in zip(ctxs, us):
        np.testing.assert_allclose(to_np(u), ur[g.cell_ids()], rtol=0, atol=1e-12 * np.abs(ur).max())
