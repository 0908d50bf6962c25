"""GPU parity of the per-level nested quadrature (reading 36):
the adaptive One-Shot path of config 4 with level l integrating on its own tensor Clenshaw-Curtis rule
(5 x 5 for degree 2, 9 x 9 for degrees 3-5, nested in the finest), against the oracle on the same
seeded inputs.  Cells start on random levels so that the stencils mix levels and the ladder moves both
ways.  Tolerances as the other parity tests."""
import numpy as np
import pytest

from inputs import configs

from .gpu_common import assert_moments_close, mesh_arrays, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("GPU test needs CUDA (no CPU fallback exists)")
    return t


def _nested_cfg(**kw):
    cfg = configs.parity_variant("cfg4")
    cfg.update(quad="cc", q1d=9, level_q1d=[5, 9, 9, 9])
    cfg.update(kw)
    return cfg


@pytest.mark.parametrize("hessian", ["newton", "lbfgs"])
def test_nested_rules_mixed_levels_parity(torch, hessian):
    import oracle
    from paper_1912_09238_b200 import Context

    cfg = _nested_cfg(hessian=hessian)
    ma = mesh_arrays(cfg)
    g, o = Context(cfg, ma), oracle.Oracle(cfg, ma)
    # IC at the initial level, then random levels on both sides (mixed stencils)
    u_o = o.project_ic()
    u_g = g.zeros()
    g.ipm_project_ic(u_g)
    # (the free stream's mean y-momentum vanishes: absolute tolerance, not reading 27's state scale)
    np.testing.assert_allclose(to_np(u_g), u_o, rtol=0, atol=1e-13 * np.abs(u_o).max())
    lv = np.random.default_rng(36).integers(0, 4, o.cells).astype(np.int32)
    o.set_levels(lv)
    g.set_levels(torch.tensor(lv, device="cuda"))
    l_o = o.warm_start(u_o)
    l_g = g.zeros()
    g.ipm_warm_start(u_g, l_g)
    moved = 0
    for step in range(10):
        w, it_o, st_o, dt_o, res_o = o.step(u_o, l_o)
        info = g.ipm_step(u_g, l_g)
        assert w == 0 and info.failed_cells == 0
        it_g, st_g = (to_np(x) for x in g.last_cell_stats())
        assert abs(info.dt - dt_o) <= 1e-12 * dt_o
        assert abs(info.residual - res_o) <= 1e-9 * max(res_o, 1e-300)
        assert np.abs(it_g - it_o).max() <= 1
        lv_o, lv_g = o.levels(), to_np(g.levels())
        assert (lv_o != lv_g).mean() < 0.01
        moved += int((lv_o != lv).sum())
        lv = lv_o
        assert_moments_close(to_np(u_g), u_o, 1e-9, f"step {step}")
    assert moved > 0  # the ladder moved


def test_nested_rules_single_rule_ladder_equals_plain_cc(torch):
    """equal rules on every level = the adaptive path on one CC rule (GPU against GPU and oracle)"""
    from paper_1912_09238_b200 import Context

    a = _nested_cfg(level_q1d=[9, 9, 9, 9])
    b = _nested_cfg(level_q1d=None)
    ma = mesh_arrays(a)
    ga, gb = Context(a, ma), Context(b, ma)
    ua, _, _ = ga.run(n_steps=5)
    ub, _, _ = gb.run(n_steps=5)
    assert_moments_close(to_np(ua), to_np(ub), 1e-12, "equal rules")
