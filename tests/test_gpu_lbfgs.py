"""GPU parity of the quasi-Newton (L-BFGS) dual solve (reading 35):
k_dual_lbfgs through the C-ABI against the oracle's L-BFGS iteration on the same seeded inputs, with
the per-cell pair history carried across (pseudo-)time steps on both sides.

Tolerances as the Newton parity tests: duals 1e-9 of the state scale, moments 1e-9
(reading 27), iteration counts +-1 (an L-BFGS count depends on every earlier iterate's rounding, so a
small fraction of cells may differ by more: bounded below), statuses equal.
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


def _stress_both(torch, g, o, cfg, ma, seed):
    base, z, amp = stress_inputs(cfg, seed=seed, ma=ma)
    lam_star = o.stress_dual(base, z, amp)
    u_o = o.moments_from_dual_all(lam_star)
    lam_s = g.zeros()
    g.ipm_stress_dual(torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda"), amp[0], amp[1], lam_s)
    u_g = g.zeros()
    g.ipm_moments_from_dual(lam_s, u_g)
    return lam_star, u_o, u_g


def _counts_close(it_g, it_o, frac=0.99, dmax=4):
    d = np.abs(it_g - it_o)
    far = int((d > 1).sum())
    assert far <= max(2, (1.0 - frac) * d.size), f"{far} of {d.size} cells differ by more than one iteration"
    assert d.max() <= dmax


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_lbfgs_stress_steps_parity(torch, name):
    """the stress state, then three steps of Algorithm 1 (FULL) with the histories carried along"""
    cfg = dict(configs.parity_variant(name), hessian="lbfgs")
    if name == "cfg4":
        cfg.update(levels=None, newton="full", update="conservative")
    g, o, ma = ctx_and_oracle(cfg)
    lam_star, u_o, u_g = _stress_both(torch, g, o, cfg, ma, seed=9300 + int(name[-1]))
    assert_moments_close(to_np(u_g), u_o, 1e-13, "h(lambda*)")
    lam_o = o.warm_start(u_o)
    lam_g = g.zeros()
    g.ipm_warm_start(u_g, lam_g)
    scale = np.abs(lam_star).max(axis=(0, 1))
    for step in range(3):
        w, it_o, st_o, dt_o, res_o = o.step(u_o, lam_o)
        info = g.ipm_step(u_g, lam_g)
        it_g, st_g = (to_np(x) for x in g.last_cell_stats())
        assert w == 0 and info.failed_cells == 0
        np.testing.assert_array_equal(st_g, st_o)
        err = (np.abs(to_np(lam_g) - lam_o) / scale).max()
        assert err < 1e-9, f"step {step}: duals {err:.2e}"
        assert_moments_close(to_np(u_g), u_o, 1e-9, f"{name} step {step}")
        assert abs(info.dt - dt_o) <= 1e-10 * dt_o
        # counts: config 5's 20-35 quasi-Newton steps per solve amplify rounding differences most (its
        # node pass and gradient are sum-factorised on the GPU, direct sums in the oracle)
        _counts_close(it_g, it_o, frac=0.8 if name == "cfg5" else 0.99, dmax=10 if name == "cfg5" else 4)
    assert it_o.mean() > 1.0  # the stress state makes the cells iterate
    # history: pair counts agree (a borderline curvature test may flip one cell)
    _, _, cnt_g = g.lbfgs_history()
    cnt_o = np.array([len(o.lbfgs_history(j)[0]) for j in range(o.cells)])
    assert (to_np(cnt_g) == cnt_o).mean() >= 0.99


@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_lbfgs_newton_fallback_parity(torch, name):
    """reading 35: with the cap at 8 steps most cells continue with Newton after 8 quasi-Newton steps
    (the k_dual_mma / k_dual_big pass over the device-built fallback list); statuses, summed counts
    and duals as the oracle, pairs dropped"""
    cfg = dict(configs.parity_variant(name), hessian="lbfgs", max_newton=8)
    g, o, ma = ctx_and_oracle(cfg)
    lam_star, u_o, u_g = _stress_both(torch, g, o, cfg, ma, seed=35)
    lam_o = o.warm_start(u_o)
    it_o, st_o, _ = o.dual_solve_all(u_o, lam_o)
    lam_g = g.zeros()
    g.ipm_warm_start(u_g, lam_g)
    it_g = g.zeros(g.cells, dtype=torch.int32)
    st_g = g.zeros(g.cells, dtype=torch.int32)
    g.ipm_dual_solve(u_g, lam_g, "full", it_g, st_g)
    torch.cuda.synchronize()
    assert (st_o == 0).all()
    np.testing.assert_array_equal(to_np(st_g), st_o)
    assert (it_o > 8).mean() > 0.5
    _counts_close(to_np(it_g), it_o)
    scale = np.abs(lam_star).max(axis=(0, 1))
    assert (np.abs(to_np(lam_g) - lam_o) / scale).max() < 1e-9
    cnt = to_np(g.lbfgs_history()[2])
    assert (cnt[to_np(it_g) > 8] == 0).all()
    w, nf = g.get_status()
    assert w == 0 and nf == 0


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_lbfgs_full_run_parity(torch, name):
    cfg = dict(configs.parity_variant(name), hessian="lbfgs")
    g, o, _ = ctx_and_oracle(cfg)
    u_o, l_o, io = o.run(record=True)
    u_g, l_g, ig = g.run(record=True)
    assert io["steps"] == ig["steps"]
    assert_moments_close(to_np(u_g), u_o, 1e-9, name)
    for (dto, ito, _), (dtg, itg, _) in zip(io["hist"], ig["hist"]):
        # the two sides' final iterates agree to the stopping tolerance only (superlinear convergence),
        # so dt, a max over the reconstructed states, differs more than Newton's 1e-12
        # (the oracle against itself under a 1e-15 perturbation: dt differs by 3.0e-9 on config 1,
        # 2.5e-10 on config 2 — the GPU gets a few times that spread)
        assert abs(dto - dtg) <= 2e-8 * dto
        # over a whole run the histories carry every earlier rounding difference (measured: up to 6 % of
        # the config-1 cells differ by 2 iterations in some steps of 25-iteration solves)
        # the counts of a superlinear iteration near tau are not reproducible across summation orders:
        # the oracle against ITSELF with the initial moments perturbed by 1e-15 (relative) differs by up
        # to 16 iterations, 17 % of a step's cells by more than one (config 1, whose barrier-closure duals
        # near u-, u+ are the worst conditioned; tests/test_oracle_lbfgs.py::
        # test_counts_are_rounding_sensitive) — the GPU must stay within that spread; the moments agree
        # to 1e-9
        _counts_close(itg, ito, frac=0.8, dmax=20)
        assert abs(itg.sum() - ito.sum()) <= 0.15 * max(ito.sum(), 20)


def test_lbfgs_one_shot_adaptive_cfg4_parity(torch):
    """One-Shot (one quasi-Newton step per pseudo-time step) with adaptive degree, bucketed launches:
    a level change clears the cell's pairs on both sides"""
    cfg = dict(configs.parity_variant("cfg4"), hessian="lbfgs")
    g, o, _ = ctx_and_oracle(cfg)
    u_o, l_o, io = o.run(n_steps=15, record=True)
    u_g, l_g, ig = g.run(n_steps=15, record=True)
    assert (o.levels() != to_np(g.levels())).mean() < 0.01
    assert_moments_close(to_np(u_g), u_o, 1e-9, "cfg4 lbfgs")
    for (_, ito, ro), (_, itg, rg) in zip(io["hist"], ig["hist"]):
        assert np.abs(ito - itg).max() <= 1
        assert abs(ro - rg) <= 1e-9 * max(ro, 1e-300)


def test_lbfgs_matches_newton_solution(torch):
    """both iterations stop at ||grad L|| < tau: the GPU's L-BFGS duals equal its Newton duals to the
    conditioning of the dual problem (same unique minimiser)"""
    from paper_1912_09238_b200 import Context

    cfg = configs.parity_variant("cfg3")
    gb, gn = Context(dict(cfg, hessian="lbfgs")), Context(cfg)
    import oracle

    o = oracle.Oracle(cfg)
    lam_star, _, u = _stress_both(torch, gb, o, cfg, None, seed=77)
    lb, ln = gb.zeros(), gn.zeros()
    gb.ipm_warm_start(u, lb)
    gn.ipm_warm_start(u, ln)
    gb.ipm_dual_solve(u, lb, "full")
    gn.ipm_dual_solve(u, ln, "full")
    scale = np.abs(lam_star).max(axis=(0, 1))
    assert (np.abs(to_np(lb) - to_np(ln)) / scale).max() < 1e-8
    w, nf = gb.get_status()
    assert w == 0 and nf == 0
    gb.lbfgs_reset()
    assert int(gb.lbfgs_history()[2].sum()) == 0


def test_lbfgs_step_host_matches_device_step(torch):
    """ipm_step_host (chunked copy/solve ranges: L-BFGS histories and the Newton-fallback lists of
    each range offset into the context's arrays) equals ipm_step bit for bit"""
    from paper_1912_09238_b200 import Context

    cfg = dict(configs.get("cfg3", mesh=dict(nx=17, ny=13)), hessian="lbfgs", max_newton=12)
    ga, gb = Context(cfg), Context(cfg)
    import oracle

    o = oracle.Oracle(cfg)
    _, _, u = _stress_both(torch, ga, o, cfg, None, seed=41)
    lam = ga.zeros()
    ga.ipm_warm_start(u, lam)
    ref_u, ref_l = u.clone(), lam.clone()
    h_u, h_l = u.cpu().pin_memory(), lam.cpu().pin_memory()
    d_u, d_l = gb.zeros(), gb.zeros()
    for _ in range(3):
        ia = ga.ipm_step(ref_u, ref_l)
        ib = gb.ipm_step_host(h_u, h_l, d_u, d_l, None, nchunks=7)
        assert ia.newton_iters == ib.newton_iters and ia.dt == ib.dt and ia.failed_cells == 0
    assert torch.equal(h_u, ref_u.cpu()) and torch.equal(h_l, ref_l.cpu())
