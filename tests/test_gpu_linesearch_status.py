"""GPU parity of the per-cell outcome record and the step bookkeeping (ipm.h: ipm_get_status,
ipm_last_cell_linesearch, ipm_step_info.newton_hist / halvings; the CUDA-graph step replay):

* the Armijo line search (reading 3') really backtracks and really meets inadmissible trials
  (reading 4) on the GPU, with the oracle's per-cell counts;
* an INADMISSIBLE cell is reported by ipm_get_status and keeps its level on both sides (reading 34);
* the step statistics are consistent with the per-cell arrays;
* the graph-replayed step (small problems) is bit-identical to the launched one;
* ipm_step_host at 256^2 with 32 and 64 copy/solve ranges is bit-identical to ipm_step.
"""
import os

import numpy as np
import pytest

from inputs import configs

from .gpu_common import mesh_arrays, stress_inputs, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("GPU test needs CUDA (no CPU fallback exists)")
    return t


def make(cfg, env=None):
    import oracle
    from paper_1912_09238_b200 import Context

    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        ma = mesh_arrays(cfg)
        return Context(cfg, ma), oracle.Oracle(cfg, ma), ma
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def stressed(torch, g, o, cfg, ma, amp, seed):
    """the same seeded stress problem on both sides (each side forms its own moments h(lambda*))"""
    base, z, _ = stress_inputs(cfg, seed=seed, ma=ma)
    lam_star = o.stress_dual(base, z, amp)
    u_o = o.moments_from_dual_all(lam_star)
    lam_o = o.warm_start(u_o)
    lam_s = g.zeros()
    g.ipm_stress_dual(torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda"), amp[0], amp[1], lam_s)
    u_g = g.zeros()
    g.ipm_moments_from_dual(lam_s, u_g)
    lam_g = g.zeros()
    g.ipm_warm_start(u_g, lam_g)
    return u_o, lam_o, u_g, lam_g


@pytest.mark.parametrize("name,amp,env", [("cfg3", (0.3, 0.0), None), ("cfg3", (0.3, 0.0), {"IPM_DUAL_KERNEL": "group"}),
                                          ("cfg2", (0.4, 0.0), None)])
def test_linesearch_backtracks_and_rejects_inadmissible_trials_like_the_oracle(torch, name, amp, env):
    """Large higher dual modes (SURVEY §8d recipe, amplitude raised): the full Newton step from the
    warm start overshoots, so most cells halve alpha and many trials leave the admissible set
    (Lambda_E >= 0, reading 4).  Per cell: status equal, Newton count +-1, and where the counts are
    equal the rejected / inadmissible trial counts equal."""
    cfg = configs.get(name, mesh=dict(nx=16, ny=16) if name == "cfg3" else dict(nx=256))
    g, o, ma = make(cfg, env)
    u_o, lam_o, u_g, lam_g = stressed(torch, g, o, cfg, ma, amp, seed=5)
    it_o, st_o, _, hv_o, ia_o = o.dual_solve_all_ls(u_o, lam_o)
    it_g = g.zeros(g.cells, dtype=torch.int32)
    st_g = g.zeros(g.cells, dtype=torch.int32)
    g.ipm_dual_solve(u_g, lam_g, "full", it_g, st_g)
    hv_g, ia_g = (to_np(x) for x in g.last_cell_linesearch())
    it_g, st_g = to_np(it_g), to_np(st_g)
    assert (st_g == st_o).all() and (st_o == 0).all()
    assert np.abs(it_g - it_o).max() <= 1
    assert (hv_o > 0).sum() >= g.cells // 2 and (ia_o > 0).sum() >= g.cells // 4  # the inputs do stress it
    same = it_g == it_o
    assert same.mean() > 0.95
    np.testing.assert_array_equal(hv_g[same], hv_o[same])
    np.testing.assert_array_equal(ia_g[same], ia_o[same])
    scale = np.abs(to_np(lam_g)).max()
    assert np.abs(to_np(lam_g)[same] - lam_o[same]).max() / scale < 1e-9
    w, nf = g.get_status()
    assert (w, nf) == (0, 0)


def test_step_statistics_are_consistent(torch):
    """newton_hist sums to the cell count, its first moment is newton_iters, and it is the histogram
    of the per-cell counts; ipm_get_status agrees with info"""
    cfg = configs.get("cfg3", mesh=dict(nx=32, ny=32))
    g, o, ma = make(cfg)
    _, _, u, lam = stressed(torch, g, o, cfg, ma, (0.3, 0.0), seed=7)
    info = g.ipm_step(u, lam)
    hist = np.array(info.newton_hist[:])
    it, st = (to_np(x) for x in g.last_cell_stats())
    assert hist.sum() == g.cells and info.failed_cells == 0
    ref = np.bincount(np.minimum(it, 15), minlength=16)
    np.testing.assert_array_equal(hist, ref)
    assert info.newton_iters == it.sum()
    hv, ia = (to_np(x) for x in g.last_cell_linesearch())
    assert info.halvings == hv.sum() > 0 and info.inadmissible_trials == ia.sum() > 0
    assert g.get_status() == (0, 0)


def test_inadmissible_cell_is_reported_and_keeps_its_level(torch):
    """Config 4 (adaptive One-Shot): one cell's duals give Lambda_E > 0 (no admissible state,
    IPM_CELL_INADMISSIBLE).  ipm_get_status reports it; the step completes; every cell's next level
    equals the oracle's, the inadmissible cell keeping its own (reading 34)."""
    cfg = configs.parity_variant("cfg4")
    g, o, ma = make(cfg)
    u_o = o.project_ic()
    lam_o = o.warm_start(u_o)
    for _ in range(3):  # a few One-Shot steps so that levels move
        assert o.step(u_o, lam_o)[0] == 0
    lv = o.levels()
    bad = 5
    lam_o[bad, 0, 3] = 1.0  # Lambda_E = +1 at every node: outside the Euler closure's domain
    u_g = torch.tensor(u_o, device="cuda")
    lam_g = torch.tensor(lam_o, device="cuda")
    g.set_levels(torch.tensor(lv, device="cuda"))
    st_g = g.zeros(g.cells, dtype=torch.int32)
    g.ipm_dual_solve(u_g, lam_g.clone(), "one_step", None, st_g)
    assert to_np(st_g)[bad] == 4 and (np.delete(to_np(st_g), bad) == 0).all()
    assert g.get_status() == (4, 1)
    w_o, _, st_o, _, _ = o.step(u_o, lam_o)
    info = g.ipm_step(u_g, lam_g)
    assert w_o == 4 and info.worst_status == 4 and info.failed_cells == 1 and st_o[bad] == 4
    lv_g, lv_o = to_np(g.levels()), o.levels()
    assert lv_o[bad] == lv[bad] and lv_g[bad] == lv[bad]
    np.testing.assert_array_equal(lv_g, lv_o)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_graph_replay_is_bit_identical_to_launches(torch, name):
    """configs 1-2 replay ipm_step from a CUDA graph; with kernel timing on the same step is launched
    kernel by kernel.  30 steps of Algorithm 1 from the IC: identical bits."""
    cfg = configs.get(name, mesh=dict(nx=400) if name == "cfg2" else {})
    out = []
    for timing in (False, True):
        g, _, _ = make(cfg)
        g.enable_timing(timing)
        u, lam, info = g.run(n_steps=30)
        out.append((to_np(u), to_np(lam), info["t"]))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


@pytest.mark.parametrize("nchunks", [32, 64])
def test_step_host_256_chunks_is_bit_identical(torch, nchunks):
    """ipm_step_host (host buffers, 32 copy/solve ranges: the bench's e2e path, and 64) against ipm_step
    on a 256^2 config-3 stress state, 2 steps"""
    cfg = configs.get("cfg3", mesh=dict(nx=256, ny=256))
    g, o, ma = make(cfg)
    base, z, amp = stress_inputs(cfg, seed=2, ma=ma)
    lam_s = g.zeros()
    g.ipm_stress_dual(torch.tensor(base, device="cuda"), torch.tensor(z, device="cuda"), amp[0], amp[1], lam_s)
    u0 = g.zeros()
    g.ipm_moments_from_dual(lam_s, u0)
    l0 = g.zeros()
    g.ipm_warm_start(u0, l0)
    u1, l1 = u0.clone(), l0.clone()
    for _ in range(2):
        g.ipm_step(u1, l1)
    g.set_time(0.0)
    h_u, h_l = u0.cpu().pin_memory(), l0.cpu().pin_memory()
    du, dl = g.zeros(), g.zeros()
    for _ in range(2):
        info = g.ipm_step_host(h_u, h_l, du, dl, None, nchunks=nchunks)
        assert info.failed_cells == 0
    np.testing.assert_array_equal(h_u.numpy(), to_np(u1))
    np.testing.assert_array_equal(h_l.numpy(), to_np(l1))


@pytest.mark.parametrize("thresholds", [None, (1e-8, 1e-7)])
def test_bucketed_levels_match_single_launch_and_oracle(torch, thresholds):
    """Adaptive degree (north star (c), Alg. 3): the per-level launches over uniform-degree buckets
    (default) against the single N_max launch (IPM_BUCKET=0) and the oracle, 30 One-Shot steps of the
    config-4 parity mesh; with the lower thresholds cells move between levels during the run"""
    cfg = configs.parity_variant("cfg4")
    if thresholds:
        cfg["delta_dec"], cfg["delta_inc"] = thresholds
    out = []
    for env in (None, {"IPM_BUCKET": "0"}):
        g, o, _ = make(cfg, env)
        u, lam, info = g.run(n_steps=30)
        out.append((to_np(u), to_np(g.levels())))
    u_o, _, _ = o.run(n_steps=30)
    np.testing.assert_array_equal(out[0][1], out[1][1])
    np.testing.assert_allclose(out[0][0], out[1][0], rtol=0, atol=1e-12 * np.abs(out[1][0]).max())
    from .gpu_common import assert_moments_close

    assert_moments_close(out[0][0], u_o, 1e-9, "bucketed cfg4")
    assert (o.levels() != out[0][1]).mean() < 0.01
