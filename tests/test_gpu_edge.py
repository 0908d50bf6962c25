"""GPU edge cases through the C-ABI, against the oracle on the same seeded inputs: ragged cell counts
(not multiples of the kernels' cells per CTA / per warp), inputs that are already converged, cells
whose starting dual is inadmissible, and the One-Shot mode (a single Newton step)."""
import numpy as np
import pytest

from inputs import configs

from .gpu_common import assert_moments_close, stress_inputs, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("GPU test needs CUDA (no CPU fallback exists)")
    return t


@pytest.fixture(params=["group", "mma"])
def dual_kernel(request, monkeypatch):
    monkeypatch.setenv("IPM_DUAL_KERNEL", request.param)
    return request.param


def _pair(cfg):
    import oracle
    from paper_1912_09238_b200 import Context

    return Context(cfg), oracle.Oracle(cfg)


def _stress(torch, g, o, cfg, seed):
    base, z, amp = stress_inputs(cfg, seed=seed)
    lam_star = o.stress_dual(base, z, amp)
    u_o = o.moments_from_dual_all(lam_star)
    lam_s = g.zeros()
    g.ipm_stress_dual(torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda"), amp[0], amp[1], lam_s)
    u_g = g.zeros()
    g.ipm_moments_from_dual(lam_s, u_g)
    return lam_star, u_o, lam_s, u_g


@pytest.mark.parametrize("name,mesh", [("cfg3", dict(nx=7, ny=3)), ("cfg2", dict(nx=33)), ("cfg1", dict(nx=13))])
def test_ragged_cell_counts_full_steps(torch, dual_kernel, name, mesh):
    cfg = configs.get(name, mesh=mesh)
    g, o = _pair(cfg)
    u_o, _, io = o.run(n_steps=4)
    u_g, _, ig = g.run(n_steps=4)
    assert io["steps"] == ig["steps"] == 4
    assert_moments_close(to_np(u_g), u_o, 1e-9, f"{name} {mesh}")


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_converged_input_takes_no_newton_step(torch, dual_kernel, name):
    cfg = configs.get(name, mesh=dict(nx=9, ny=5) if name == "cfg3" else dict(nx=37))
    g, o = _pair(cfg)
    lam_star, u_o, lam_s, u_g = _stress(torch, g, o, cfg, seed=11)
    it_g = g.zeros(g.cells, dtype=torch.int32)
    st_g = g.zeros(g.cells, dtype=torch.int32)
    lam_g = lam_s.clone()
    g.ipm_dual_solve(u_g, lam_g, "full", it_g, st_g)
    lam_o = lam_star.copy()
    it_o, st_o, _ = o.dual_solve_all(u_o, lam_o)
    torch.cuda.synchronize()
    # the exact dual satisfies the gradient test up to rounding: at most one polishing step
    assert (it_o <= 1).all() and (to_np(it_g) <= 1).all()
    assert np.abs(to_np(it_g) - it_o).max() <= 1
    np.testing.assert_array_equal(to_np(st_g), st_o)
    scale = np.abs(lam_star).max(axis=(0, 1))
    assert (np.abs(to_np(lam_g) - lam_star) / scale).max() < 1e-9


def test_inadmissible_start_is_reported_per_cell(torch, dual_kernel):
    """Euler duals with v_E >= 0 have no state (reading 9): status 4 on both sides, the other cells
    solve normally."""
    cfg = configs.get("cfg3", mesh=dict(nx=6, ny=4))
    g, o = _pair(cfg)
    lam_star, u_o, lam_s, u_g = _stress(torch, g, o, cfg, seed=12)
    lam0_o = o.warm_start(u_o)
    bad = np.zeros(g.cells, bool)
    bad[[1, 7, 18]] = True
    lam0_o[bad, 0, 3] = 0.25  # lambda_{0,E} > 0: inadmissible at every node
    lam_g = torch.tensor(lam0_o, device="cuda")
    it_g = g.zeros(g.cells, dtype=torch.int32)
    st_g = g.zeros(g.cells, dtype=torch.int32)
    g.ipm_dual_solve(torch.tensor(u_o, device="cuda"), lam_g, "full", it_g, st_g)
    it_o, st_o, _ = o.dual_solve_all(u_o, lam0_o)
    torch.cuda.synchronize()
    assert (st_o[bad] == 4).all() and (st_o[~bad] == 0).all()
    np.testing.assert_array_equal(to_np(st_g), st_o)
    assert (to_np(it_g)[bad] == 0).all()
    scale = np.abs(lam_star).max(axis=(0, 1))
    assert (np.abs(to_np(lam_g)[~bad] - lam0_o[~bad]) / scale).max() < 1e-9


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_one_step_mode_matches_oracle(torch, dual_kernel, name):
    cfg = configs.get(name, mesh=dict(nx=9, ny=5) if name == "cfg3" else dict(nx=37), newton="one_step")
    g, o = _pair(cfg)
    lam_star, u_o, lam_s, u_g = _stress(torch, g, o, cfg, seed=13)
    lam0_o = o.warm_start(u_o)
    lam_g = g.zeros()
    g.ipm_warm_start(u_g, lam_g)
    it_g = g.zeros(g.cells, dtype=torch.int32)
    st_g = g.zeros(g.cells, dtype=torch.int32)
    g.ipm_dual_solve(u_g, lam_g, "one_step", it_g, st_g)
    it_o, st_o, _ = o.dual_solve_all(u_o, lam0_o)
    torch.cuda.synchronize()
    assert (it_o <= 1).all()
    np.testing.assert_array_equal(to_np(it_g), it_o)
    np.testing.assert_array_equal(to_np(st_g), st_o)
    scale = np.abs(lam_star).max(axis=(0, 1))
    assert (np.abs(to_np(lam_g) - lam0_o) / scale).max() < 1e-9


@pytest.mark.parametrize("nchunks", [1, 3, 7])
def test_step_host_matches_device_step(torch, nchunks):
    """ipm_step_host (host buffers, copies overlapped with the dual solves of earlier cell ranges)
    gives ipm_step's result bit for bit"""
    from paper_1912_09238_b200 import Context

    cfg = configs.get("cfg3", mesh=dict(nx=13, ny=11))
    g = Context(cfg)
    o = __import__("oracle").Oracle(cfg)
    _, _, lam_s, u_g = _stress(torch, g, o, cfg, seed=3)
    lam0 = g.zeros()
    g.ipm_warm_start(u_g, lam0)
    ref_u, ref_l = u_g.clone(), lam0.clone()
    h_u, h_l = u_g.cpu().pin_memory(), lam0.cpu().pin_memory()
    d_u, d_l = g.zeros(), g.zeros()
    for _ in range(2):
        ia = g.ipm_step(ref_u, ref_l)
        ib = g.ipm_step_host(h_u, h_l, d_u, d_l, None, nchunks=nchunks)
        assert ia.newton_iters == ib.newton_iters and ia.dt == ib.dt
    assert torch.equal(h_u, ref_u.cpu()) and torch.equal(h_l, ref_l.cpu())


def test_step_host_matches_device_step_adaptive(torch):
    """the adaptive path of ipm_step_host (duals copied back after the flux, which truncates them to
    the new levels) on config 4's One-Shot ladder"""
    from paper_1912_09238_b200 import Context

    from .gpu_common import mesh_arrays

    cfg = dict(configs.parity_variant("cfg4"), delta_inc=1e-9, delta_dec=0.0, initial_level=0)
    ma = mesh_arrays(cfg)
    ga, gb = Context(cfg, ma), Context(cfg, ma)
    u = ga.zeros()
    ga.ipm_project_ic(u)
    gb.ipm_project_ic(gb.zeros())  # levels / time of the second context
    lam = ga.zeros()
    ga.ipm_warm_start(u, lam)
    ref_u, ref_l = u.clone(), lam.clone()
    h_u, h_l = u.cpu().pin_memory(), lam.cpu().pin_memory()
    d_u, d_l = gb.zeros(), gb.zeros()
    for _ in range(3):
        ia = ga.ipm_step(ref_u, ref_l)
        ib = gb.ipm_step_host(h_u, h_l, d_u, d_l, None, nchunks=5)
        assert ia.newton_iters == ib.newton_iters and ia.dt == ib.dt
    assert torch.equal(h_u, ref_u.cpu()) and torch.equal(h_l, ref_l.cpu())
    assert torch.equal(ga.levels(), gb.levels())
