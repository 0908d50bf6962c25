"""GPU parity: the CUDA path through the C-ABI against the oracle on the same seeded inputs.

Tolerances: moments 1e-9 relative to the state's scale (reading 27), Newton
counts +-1, statuses equal, zeroth-moment conservation 1e-12 on periodic meshes.
"""
import numpy as np
import pytest

from inputs import configs

from .gpu_common import assert_moments_close, mesh_arrays, stress_inputs, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("GPU test needs CUDA (no CPU fallback exists)")
    return t


def ctx_and_oracle(cfg):
    import oracle
    from paper_1912_09238_b200 import Context

    ma = mesh_arrays(cfg)
    return Context(cfg, ma), oracle.Oracle(cfg, ma), ma


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_basis_tables_match(torch, name):
    cfg = configs.parity_variant(name)
    g, o, _ = ctx_and_oracle(cfg)
    xg, wg, pg = g.basis()
    xo, wo, po = o.quadrature()
    np.testing.assert_allclose(xg, xo, atol=2e-15)
    np.testing.assert_allclose(wg, wo, rtol=1e-13, atol=1e-17)
    np.testing.assert_allclose(pg, po, rtol=1e-12, atol=1e-12)


QUAD_VARIANTS = {"cc17_cfg1": ("cfg1", dict(quad="cc", q1d=17)), "cc9_cfg3": ("cfg3", dict(quad="cc", q1d=9)),
                 "smolyak6_cfg3": ("cfg3", dict(quad="smolyak", quad_level=6)),
                 "smolyak7_cfg3": ("cfg3", dict(quad="smolyak", quad_level=7))}


@pytest.mark.parametrize("variant", list(QUAD_VARIANTS))
def test_quadrature_variants_tables_match(torch, variant):
    """reading 33: the device's Clenshaw-Curtis (moment-fitted weights) and Smolyak rules against the
    oracle's (cosine-sum weights): the same points in the same order, weights and basis values"""
    name, kw = QUAD_VARIANTS[variant]
    cfg = dict(configs.parity_variant(name), **kw)
    g, o, _ = ctx_and_oracle(cfg)
    xg, wg, pg = g.basis()
    xo, wo, po = o.quadrature()
    np.testing.assert_allclose(xg, xo, atol=2e-15)
    np.testing.assert_allclose(wg, wo, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(pg, po, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("variant", list(QUAD_VARIANTS))
def test_quadrature_variants_dual_solve_parity(torch, variant):
    """the dual solve under the chosen rule: per-cell statuses (Smolyak's negative weights make some
    Hessians indefinite: IPM_CELL_ILLCONDITIONED, the failure mode of PAPER.md:753-773) and duals"""
    name, kw = QUAD_VARIANTS[variant]
    cfg = dict(configs.parity_variant(name), **kw)
    g, o, ma = ctx_and_oracle(cfg)
    base, z, amp = stress_inputs(cfg, seed=3, ma=ma)
    lam_star = o.stress_dual(base, z, amp)
    u_o = o.moments_from_dual_all(lam_star)
    lam_o = o.warm_start(u_o)
    it_o, st_o, _ = o.dual_solve_all(u_o, lam_o)
    lam_s = g.zeros()
    g.ipm_stress_dual(torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda"), amp[0], amp[1], lam_s)
    u_g = g.zeros()
    g.ipm_moments_from_dual(lam_s, u_g)
    lam_g = g.zeros()
    g.ipm_warm_start(u_g, lam_g)
    it_g = g.zeros(g.cells, dtype=torch.int32)
    st_g = g.zeros(g.cells, dtype=torch.int32)
    g.ipm_dual_solve(u_g, lam_g, "full", it_g, st_g)
    torch.cuda.synchronize()
    st_g = to_np(st_g)
    assert (st_g == st_o).mean() >= 0.99  # a pivot at the rounding level may flip a cell
    if variant.startswith("smolyak"):
        assert (st_o == 2).any()
    ok = (st_o == 0) & (st_g == 0)
    assert np.abs(to_np(it_g)[ok] - it_o[ok]).max() <= 1
    scale = np.abs(lam_star).max(axis=(0, 1))
    err = (np.abs(to_np(lam_g)[ok] - lam_o[ok]) / scale).max()
    assert err < 1e-9, err


@pytest.fixture(params=["group", "mma"])
def dual_kernel(request, monkeypatch):
    """both dual-solve kernels (IPM_DUAL_KERNEL is read at every launch)"""
    monkeypatch.setenv("IPM_DUAL_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_dual_solve_stress_parity(torch, name, dual_kernel):
    """manufactured lambda* per cell: uhat = h(lambda*), solve from e0 (x) grad s(uhat_0)."""
    cfg = configs.parity_variant(name)
    if name == "cfg4":
        cfg["levels"] = None  # whole basis in every cell; adaptivity is covered by the run test
        cfg["newton"] = "full"
    g, o, ma = ctx_and_oracle(cfg)
    base, z, amp = stress_inputs(cfg, seed=9238 + int(name[-1]), ma=ma)
    # oracle side
    lam_star = o.stress_dual(base, z, amp)
    u_o = o.moments_from_dual_all(lam_star)
    lam_o = o.warm_start(u_o)
    it_o, st_o, _ = o.dual_solve_all(u_o, lam_o)
    # GPU side, from the same seeded draws
    tb, tz = torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda")
    lam_s = g.zeros()
    g.ipm_stress_dual(tb, tz, amp[0], amp[1], lam_s)
    np.testing.assert_allclose(to_np(lam_s), lam_star, rtol=1e-13, atol=1e-13)
    u_g = g.zeros()
    g.ipm_moments_from_dual(lam_s, u_g)
    assert_moments_close(to_np(u_g), u_o, 1e-13, "h(lambda*)")
    lam_g = g.zeros()
    g.ipm_warm_start(u_g, lam_g)
    it_g = g.zeros(g.cells, dtype=torch.int32)
    st_g = g.zeros(g.cells, dtype=torch.int32)
    g.ipm_dual_solve(u_g, lam_g, "full", it_g, st_g)
    torch.cuda.synchronize()
    assert (st_o == 0).all()
    np.testing.assert_array_equal(to_np(st_g), st_o)
    assert np.abs(to_np(it_g) - it_o).max() <= 1
    assert (it_o >= 1).mean() > 0.9  # the stress input makes every cell iterate
    scale = np.abs(lam_star).max(axis=(0, 1))
    err = (np.abs(to_np(lam_g) - lam_o) / scale).max()
    assert err < 1e-9, err


def _run_both(cfg, n_steps=None):
    g, o, _ = ctx_and_oracle(cfg)
    u_o, l_o, info_o = o.run(n_steps=n_steps, record=True)
    u_g, l_g, info_g = g.run(n_steps=n_steps, record=True)
    return g, o, (u_o, l_o, info_o), (to_np(u_g), to_np(l_g), info_g)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_full_run_parity(torch, name, dual_kernel):
    cfg = configs.parity_variant(name)
    g, o, (u_o, l_o, io), (u_g, l_g, ig) = _run_both(cfg)
    assert io["steps"] == ig["steps"]
    assert abs(io["t"] - ig["t"]) < 1e-14
    assert_moments_close(u_g, u_o, 1e-9, name)
    for (dto, ito, _), (dtg, itg, _) in zip(io["hist"], ig["hist"]):
        assert abs(dto - dtg) <= 1e-12 * dto
        assert np.abs(ito - itg).max() <= 1


def test_cfg5_window_parity(torch):
    cfg = configs.parity_variant("cfg5")
    g, o, (u_o, _, io), (u_g, _, ig) = _run_both(cfg, n_steps=3)
    assert_moments_close(u_g, u_o, 1e-9, "cfg5")


def test_one_shot_adaptive_cfg4_parity(torch):
    cfg = configs.parity_variant("cfg4")
    g, o, (u_o, l_o, io), (u_g, l_g, ig) = _run_both(cfg, n_steps=15)
    lv_o = o.levels()
    lv_g = to_np(g.levels())
    assert (lv_o != lv_g).mean() < 0.01
    assert_moments_close(u_g, u_o, 1e-9, "cfg4")
    for (_, ito, ro), (_, itg, rg) in zip(io["hist"], ig["hist"]):
        assert np.abs(ito - itg).max() <= 1
        assert abs(ro - rg) <= 1e-9 * max(ro, 1e-300)


def test_refinement_retardation_cfg4_parity(torch):
    """Algorithm 4: the stage caps and their residual-driven advance on the GPU
    (device-side stage) against the oracle; the schedule moves the stage twice within the run"""
    cfg = dict(configs.parity_variant("cfg4"), delta_inc=1e-9, delta_dec=0.0, initial_level=0,
               retard=[(1.9e-4, 0), (1.8759e-4, 1)])
    g, o, (u_o, l_o, io), (u_g, l_g, ig) = _run_both(cfg, n_steps=8)
    assert o.retard_stage() == g.retard_stage() == 2
    assert (o.levels() != to_np(g.levels())).mean() < 0.01
    assert_moments_close(u_g, u_o, 1e-9, "cfg4 retardation")
    for (_, ito, ro), (_, itg, rg) in zip(io["hist"], ig["hist"]):
        assert np.abs(ito - itg).max() <= 1
        assert abs(ro - rg) <= 1e-9 * max(ro, 1e-300)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg3_smolyak6", "cfg3_wide"])
def test_stochastic_collocation_parity(torch, name):
    """Stochastic Collocation (reading 32) through the C-ABI against the oracle:
    node states of the IC, coupled CFL steps with the same numerical flux, quadrature moments"""
    if name == "cfg3_smolyak6":  # SC on a sparse grid (negative weights are harmless for SC)
        cfg = dict(configs.parity_variant("cfg3"), quad="smolyak", quad_level=6)
    elif name == "cfg3_wide":  # more strips than CTAs: the strip walk's contiguous work split
        cfg = configs.get("cfg3", mesh=dict(nx=1201, ny=3))
    else:
        cfg = configs.parity_variant(name)
    g, o, _ = ctx_and_oracle(cfg)
    steps = 6
    U = o.sc_init()
    a, b = g.sc_zeros(), g.sc_zeros()
    g.ipm_sc_init(a)
    np.testing.assert_allclose(to_np(a).transpose(0, 2, 1), U, rtol=1e-15, atol=0)  # FMA contraction: 1 ulp
    for _ in range(steps):
        U, dt_o, res_o = o.sc_step(U)
        info = g.ipm_sc_step(a, b)
        a, b = b, a
        assert abs(info.dt - dt_o) <= 1e-12 * dt_o
        assert abs(info.residual - res_o) <= 1e-9 * max(res_o, 1e-300)
    u_g = g.zeros()
    g.ipm_sc_moments(a, u_g)
    assert_moments_close(to_np(u_g), o.sc_moments(U), 1e-10, f"SC {name}")


def test_one_shot_steady_fixed_point(torch):
    from paper_1912_09238_b200 import Context

    res = {}
    for mode in ("full", "one_step"):
        g = Context(configs.steady1d(mode))
        u = g.zeros()
        g.ipm_project_ic(u)
        lam = g.zeros()
        g.ipm_warm_start(u, lam)
        r1, total = None, 0
        for _ in range(5000):
            info = g.ipm_step(u, lam)
            assert info.failed_cells == 0
            total += info.newton_iters
            r1 = info.residual if r1 is None else r1
            if info.residual <= 1e-8 * r1:
                break
        res[mode] = (to_np(u), total)
    assert res["one_step"][1] < res["full"][1]
    np.testing.assert_allclose(res["one_step"][0], res["full"][0], atol=1e-6)


def test_periodic_conservation(torch):
    cfg = configs.get("cfg3", mesh=dict(nx=16, ny=12, periodic=True))
    from paper_1912_09238_b200 import Context

    g = Context(cfg)
    u = g.zeros()
    g.ipm_project_ic(u)
    lam = g.zeros()
    g.ipm_warm_start(u, lam)
    tot0 = to_np(u)[:, 0, :].sum(axis=0)
    for _ in range(10):
        info = g.ipm_step(u, lam)
        assert info.failed_cells == 0
    tot = to_np(u)[:, 0, :].sum(axis=0)
    np.testing.assert_allclose(tot, tot0, rtol=1e-12, atol=1e-12)


def test_uniform_state_bit_exact(torch):
    from paper_1912_09238_b200 import Context

    cfg = configs.get("cfg3", mesh=dict(nx=8, ny=6, periodic=True))
    cfg["ic"] = dict(kind="uniform", states=[cfg["ic"]["states"][0]])
    g = Context(cfg)
    u = g.zeros()
    g.ipm_project_ic(u)
    u0 = u.clone()
    lam = g.zeros()
    g.ipm_warm_start(u, lam)
    for _ in range(3):
        info = g.ipm_step(u, lam)
        assert info.newton_iters == 0
    assert torch.equal(u, u0)


@pytest.mark.parametrize("deltas", [(1e-4, 1e-5), (1e-9, 1e-12)])
def test_adaptive_levels_stepwise_exact(torch, deltas):
    """Alg. 3 line 15 (readings 19-20, 34) step by step: after every step the GPU's
    levels equal the oracle's except on borderline cells, whose oracle indicator S (computed from the
    oracle's lambda at the old level) lies within 1e-6 relative of delta_inc or delta_dec (a decision
    taken by floating point on both sides); the GPU is then reset to the oracle's levels so one flip
    cannot cascade.  The second pair of thresholds forces level changes (the check is not vacuous)."""
    d_inc, d_dec = deltas
    cfg = dict(configs.parity_variant("cfg4"), delta_inc=d_inc, delta_dec=d_dec)
    g, o, _ = ctx_and_oracle(cfg)
    u_o = o.project_ic()
    l_o = o.warm_start(u_o)
    u_g, l_g = g.zeros(), g.zeros()
    g.ipm_project_ic(u_g)
    g.ipm_warm_start(u_g, l_g)
    changed = borderline = 0
    for step in range(10):
        lv_old = o.levels()
        w, _, st, _, _ = o.step(u_o, l_o)
        assert w == 0
        info = g.ipm_step(u_g, l_g)
        assert info.failed_cells == 0
        lv_o, lv_g = o.levels(), to_np(g.levels())
        changed += int((lv_o != lv_old).sum())
        for j in np.nonzero(lv_o != lv_g)[0]:
            h, ok = o.moments_from_dual(l_o[j], o.Nl[lv_old[j]])
            assert ok
            S = o.indicator(int(lv_old[j]), h)
            near = min(abs(S - d_inc) / d_inc, abs(S - d_dec) / max(d_dec, 1e-300))
            assert near <= 1e-6, f"step {step} cell {j}: levels {lv_o[j]} vs {lv_g[j]}, S = {S:.6e}"
            borderline += 1
        if borderline:
            g.set_levels(torch.from_numpy(lv_o).to(u_g.device))
        assert_moments_close(to_np(u_g), u_o, 1e-9, f"cfg4 step {step}")
    if d_inc < 1e-6:
        assert changed > 0


def _farfield(cfg):
    cfg = dict(cfg)
    cfg["bc"] = [("farfield", s) if k == "state" else (k, s) for k, s in cfg["bc"]]
    return cfg


def test_farfield_cfg4_parity(torch):
    """Reading 37 (characteristic far-field ghosts at the bump channel's inlet and outlet) on the GPU
    (k_flux_warp) against the oracle: One-Shot config 4, 15 pseudo-steps, from the seeded stress state
    so that the interior node states differ from the free stream at the boundary (whole basis in
    every cell, as in the stress parity tests: the stress duals carry every mode)"""
    cfg = _farfield(configs.parity_variant("cfg4"))
    cfg["levels"] = None
    g, o, ma = ctx_and_oracle(cfg)
    base, z, amp = stress_inputs(cfg, 37, ma)
    lam_o = o.stress_dual(base, z, amp)
    u0 = o.moments_from_dual_all(lam_o)
    u_o, l_o, io = o.run(n_steps=15, uhat=u0.copy(), lam=lam_o.copy(), record=True)
    u_g = torch.from_numpy(u0.copy()).cuda()
    l_g = torch.from_numpy(lam_o.copy()).cuda()
    _, _, ig = g.run(uhat=u_g, lam=l_g, n_steps=15, record=True)
    assert_moments_close(to_np(u_g), u_o, 1e-9, "cfg4 farfield")
    for (dto, ito, ro), (dtg, itg, rg) in zip(io["hist"], ig["hist"]):
        assert abs(dto - dtg) <= 1e-12 * dto
        assert np.abs(ito - itg).max() <= 1
        assert abs(ro - rg) <= 1e-9 * max(ro, 1e-300)
    # the far-field ghosts differ from the Dirichlet ones on this state: the runs must differ
    cfg_d = dict(configs.parity_variant("cfg4"), levels=None)
    od = __import__("oracle").Oracle(cfg_d, ma)
    u_d, _, _ = od.run(n_steps=15, uhat=u0.copy(), lam=lam_o.copy())
    assert np.abs(u_d - u_o).max() > 1e-6


def test_farfield_refused_off_triangles(torch):
    from paper_1912_09238_b200 import Context, IPMError

    cfg = _farfield(dict(configs.parity_variant("cfg3"), bc=[("state", configs.parity_variant("cfg4")["bc"][1][1])] * 4))
    with pytest.raises(IPMError):
        Context(cfg)
