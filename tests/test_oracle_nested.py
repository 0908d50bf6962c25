"""Oracle pins: per-level nested quadrature for the adaptive method (reading 36; SURVEY 8(f) NEXT-3;
PAPER.md:385-398 "nested quadrature rules ... evaluate the neighboring cell at the finer quadrature
level", "Order 2 uses 5 quadrature points, orders 3 to 6 use 9").

What fixes it, independently of the oracle's own code:
  * each level's rule: its nodes are Clenshaw-Curtis points (written out here with numpy) found among
    the finest rule's nodes, weights sum to one, exact for the polynomials a CC rule integrates;
  * equal rules on every level reduce to the single-rule adaptive path bit for bit;
  * a frozen level ladder reproduces the non-adaptive method with that level's degree and rule;
  * the moment update of eq. (adaptiveFVUpdate), recomputed by hand for cells whose
    neighbours sit on other levels (states from the neighbours' duals at their own degree, evaluated
    at the nodes of the updated cell's rule; pinned closure, flux and basis values as primitives).
"""
import numpy as np
import pytest

from inputs import configs
from inputs.generators import bump_channel_mesh


def _cfg4_nested(**kw):
    cfg = configs.parity_variant("cfg4")
    cfg.update(quad="cc", q1d=9, level_q1d=[5, 9, 9, 9])
    cfg.update(kw)
    return cfg


def _mesh(cfg):
    m = cfg["mesh"]
    return bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"])


def _cc_points(n):
    return -np.cos(np.pi * np.arange(n) / (n - 1))


def test_level_rules_are_nested_cc_rules(oracle_mod):
    cfg = _cfg4_nested()
    o = oracle_mod.Oracle(cfg, _mesh(cfg))
    xi, om, _ = o.quadrature()
    assert xi.shape[0] == 81
    for lvl, n in enumerate(cfg["level_q1d"]):
        kf, w = o.level_rule(lvl)
        assert len(kf) == n * n and len(set(kf.tolist())) == n * n
        pts = xi[kf]
        x1 = _cc_points(n)
        ref = np.stack(np.meshgrid(x1, x1, indexing="ij"), axis=-1).reshape(-1, 2)  # last dim fastest
        np.testing.assert_allclose(pts, ref, atol=1e-15)
        assert abs(w.sum() - 1.0) < 1e-14
        # CC with n (odd) points integrates degree n per dimension exactly (uniform density 1/4)
        for a in range(n + 1):
            for b in range(n + 1 - a):
                exact = (0.0 if a % 2 else 1.0 / (a + 1)) * (0.0 if b % 2 else 1.0 / (b + 1))
                assert abs(w @ (pts[:, 0] ** a * pts[:, 1] ** b) - exact) < 1e-13


def test_equal_level_rules_reduce_to_the_single_rule(oracle_mod):
    a = _cfg4_nested(level_q1d=[9, 9, 9, 9])
    b = _cfg4_nested(level_q1d=None)
    ma = _mesh(a)
    oa, ob = oracle_mod.Oracle(a, ma), oracle_mod.Oracle(b, ma)
    ua, _, ia = oa.run(n_steps=6, record=True)
    ub, _, ib = ob.run(n_steps=6, record=True)
    np.testing.assert_array_equal(ua, ub)
    np.testing.assert_array_equal(oa.levels(), ob.levels())


def test_frozen_level_is_the_nonadaptive_method_on_that_rule(oracle_mod):
    # levels never change (thresholds out of reach): level 0 = degree 2 on the 5 x 5 CC rule
    a = _cfg4_nested(delta_dec=-1.0, delta_inc=1e300, initial_level=0)
    b = configs.parity_variant("cfg4")
    b.update(levels=None, M=2, quad="cc", q1d=5)
    ma = _mesh(a)
    oa, ob = oracle_mod.Oracle(a, ma), oracle_mod.Oracle(b, ma)
    ua, _, ia = oa.run(n_steps=5, record=True)
    ub, _, ib = ob.run(n_steps=5, record=True)
    assert (oa.levels() == 0).all()
    for (dta, _, ra), (dtb, _, rb) in zip(ia["hist"], ib["hist"]):
        assert dta == dtb and ra == rb
    np.testing.assert_array_equal(ua[:, : ob.N], ub)
    assert (ua[:, ob.N:] == 0).all()


def test_adaptive_update_by_hand(oracle_mod):
    """eq. (adaptiveFVUpdate) for interior cells whose neighbours have other levels (c-form)"""
    cfg = _cfg4_nested()
    ma = _mesh(cfg)
    o = oracle_mod.Oracle(cfg, ma)
    rng = np.random.default_rng(36)
    levels = rng.integers(0, 4, o.cells).astype(np.int32)
    o.set_levels(levels)
    # smooth admissible duals: free stream plus small random higher modes, truncated to each level
    u0 = o.project_ic()
    lam = o.warm_start(u0)
    Nl = o.Nl
    for j in range(o.cells):
        lam[j, 1:Nl[levels[j]]] = 1e-3 * rng.standard_normal((Nl[levels[j]] - 1, o.m)) * np.abs(lam[j, 0])
        lam[j, Nl[levels[j]]:] = 0.0
    uhat_old = o.moments_from_dual_all(lam)
    dt = 1e-3
    new = o.flux_update(lam, uhat_old, dt)
    xi, _, Phi = o.quadrature()
    nbr, nrm, coef, area = o.geometry()
    interior = [j for j in range(o.cells) if (nbr[j] >= 0).all()]
    checked = 0
    for j in interior:
        lv_nb = levels[nbr[j]]
        if (lv_nb == levels[j]).all():
            continue
        kf, w = o.level_rule(levels[j])
        def state(c, k):
            u, ok = o.closure_u(Phi[k, : Nl[levels[c]]] @ lam[c, : Nl[levels[c]]])
            assert ok
            return np.asarray(u)
        acc = np.zeros((Nl[levels[j]], o.m))
        for q, k in enumerate(kf):
            uj = state(j, k)
            r = np.zeros(o.m)
            for f in range(3):
                r += coef[j, f] * np.asarray(o.flux_g(uj, state(nbr[j, f], k), nrm[j, f]))
            acc += w[q] * np.outer(Phi[k, : Nl[levels[j]]], uj - dt * r)
        np.testing.assert_allclose(new[j, : Nl[levels[j]]], acc, rtol=1e-12, atol=1e-13 * np.abs(acc).max())
        assert (new[j, Nl[levels[j]]:] == 0).all()
        checked += 1
        if checked >= 12:
            break
    assert checked >= 12


def test_nested_rules_need_a_nested_cc_ladder(oracle_mod):
    cfg = _cfg4_nested(level_q1d=[5, 7, 9, 9])  # 7 points do not nest in 9
    with pytest.raises(ValueError):
        oracle_mod.Oracle(cfg, _mesh(cfg))
