"""Distributed CUDA path on one GPU: R contexts own the parts of one mesh (ipm_init with rank/nranks),
the host moves the packed boundary duals between their send/receive buffers and takes the max of the
CFL rates (what torch.distributed does across GPUs), and the owned cells must equal a single-context
run bit for bit — including the adaptive config-4 path (halo duals at the old level, truncation
after the flux) — and the assembled result must match the oracle (1e-9, reading 27).  No kernel waits
on another context."""
import ctypes as C

import numpy as np
import pytest

from inputs import configs
from inputs.generators import bump_channel_mesh

from .gpu_common import assert_moments_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("GPU test needs CUDA")
    return t


def _case(name):
    if name == "cart":
        return configs.parity_variant("cfg3"), None
    if name == "cart_lbfgs":
        return dict(configs.parity_variant("cfg3"), hessian="lbfgs"), None
    cfg = configs.parity_variant("cfg4")
    if name == "tri_retard":  # refinement retardation: the stage advances from the global residual
        cfg.update(delta_inc=1e-9, delta_dec=0.0, initial_level=0, retard=[(1.9e-4, 0), (1.8759e-4, 1)])
    m = cfg["mesh"]
    return cfg, bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"])


@pytest.mark.parametrize("name,R,px,py,split", [("cart", 2, 2, 1, False), ("cart", 4, 2, 2, False),
                                               ("tri", 3, 0, 0, False), ("tri_retard", 3, 0, 0, False),
                                               ("cart", 4, 2, 2, True), ("cart_lbfgs", 2, 2, 1, True),
                                               ("tri", 3, 0, 0, True)])
def test_virtual_ranks_match_single_context(torch, name, R, px, py, split):
    """split: the boundary cells' dual solves first (ipm_step_dual_boundary), the exchange, then the
    interior cells' (ipm_step_dual_interior) — the overlap order of the binding's distributed step"""
    from paper_1912_09238_b200 import Context
    from paper_1912_09238_b200.ipm import _ptr, check, ipm_step_info, lib

    cfg, ma = _case(name)
    steps = 6
    ref = Context(cfg, ma)
    u_ref, _, _ = ref.run(n_steps=steps, t_end=1e9)
    ctxs, us, lams = [], [], []
    for r in range(R):
        g = Context(cfg, ma, rank=r, nranks=R, px=px, py=py)
        g._halo_setup()
        u = g.zeros()
        g.ipm_project_ic(u)
        lam = g.zeros()
        g.ipm_warm_start(u, lam)
        ctxs.append(g)
        us.append(u)
        lams.append(lam)
    L = lib()
    for _ in range(steps):
        for g, u, lam in zip(ctxs, us, lams):
            if split:
                check(L.ipm_step_dual_boundary(g.h, _ptr(u), _ptr(lam), _ptr(g.sendbuf)), "ipm_step_dual_boundary")
            else:
                check(L.ipm_step_dual(g.h, _ptr(u), _ptr(lam), _ptr(g.sendbuf), _ptr(g.rate)), "ipm_step_dual")
        torch.cuda.synchronize()
        # exchange: slice of r's send buffer for peer p -> slice of p's receive buffer from r
        for r, g in enumerate(ctxs):
            s0 = 0
            for p, ns in zip(g.halo["peers"], g.halo["send_count"]):
                gp = ctxs[p]
                k = gp.halo["peers"].index(r)
                r0 = sum(gp.halo["recv_count"][:k])
                assert gp.halo["recv_count"][k] == ns
                gp.recvbuf[r0:r0 + ns].copy_(g.sendbuf[s0:s0 + ns])
                s0 += ns
        if split:
            for g, u, lam in zip(ctxs, us, lams):
                check(L.ipm_step_dual_interior(g.h, _ptr(u), _ptr(lam), _ptr(g.rate)), "ipm_step_dual_interior")
            torch.cuda.synchronize()
        rate = torch.stack([g.rate for g in ctxs]).max()
        for g in ctxs:
            g.rate.copy_(rate.reshape(1))
        res = 0.0
        for g, u, lam in zip(ctxs, us, lams):
            info = ipm_step_info()
            rc = L.ipm_step_flux(g.h, _ptr(u), _ptr(lam), _ptr(g.recvbuf), _ptr(g.rate), 1e9, C.byref(info))
            check(rc, "ipm_step_flux")
            res += info.residual
        if cfg.get("retard"):  # what the binding does after its residual all-reduce
            for g in ctxs:
                check(L.ipm_retard_advance(g.h, res), "ipm_retard_advance")
    seen = np.zeros(ref.cells, bool)
    ur = u_ref.cpu().numpy()
    assembled = np.zeros_like(ur)
    for g, u in zip(ctxs, us):
        ids = g.cell_ids()
        assert not seen[ids].any()
        seen[ids] = True
        np.testing.assert_array_equal(u.cpu().numpy(), ur[ids])
        assembled[ids] = u.cpu().numpy()
    assert seen.all()
    # the assembled R-rank result against the oracle (not only against the GPU's single context)
    import oracle

    o = oracle.Oracle(cfg, ma)
    u_o, _, _ = o.run(n_steps=steps, t_end=1e9)
    assert_moments_close(assembled, u_o, 1e-9, f"{name} {R} ranks vs oracle")
    if cfg.get("retard"):
        assert ref.retard_stage() == 2 and all(g.retard_stage() == 2 for g in ctxs)
