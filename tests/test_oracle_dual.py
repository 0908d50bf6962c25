"""Oracle pins: the dual problem and Newton's method.

Pins: quadratic entropy reproduces stochastic-Galerkin; xi-constant cells
need no iteration (reading 6); grad L and H equal finite differences of L and grad L;
manufactured lambda* is recovered; quadratic convergence; monotone ||grad L||.
"""
import numpy as np
import pytest

from inputs import configs


def _oracle(oracle_mod, kind, M=None, q1d=None):
    if kind == "quadratic":
        cfg = configs.get("cfg1", mesh=dict(nx=2), closure="quadratic", flux="lf_global")
    elif kind == "barrier":
        cfg = configs.get("cfg1", mesh=dict(nx=2))
    elif kind == "euler1d":
        cfg = configs.get("cfg2", mesh=dict(nx=2))
    elif kind == "euler2d":
        cfg = configs.get("cfg3", mesh=dict(nx=2, ny=2))
    elif kind == "euler2d_p3":
        cfg = configs.get("cfg5", mesh=dict(nx=2, ny=2))
    if M is not None:
        cfg["M"] = M
    if q1d is not None:
        cfg["q1d"] = q1d
    return oracle_mod.Oracle(cfg)


def _manufactured(o, rng, kind):
    """lambda* = e0 (x) grad s(base) + small random higher modes (SURVEY §8d recipe)."""
    if kind in ("barrier", "quadratic"):
        base = np.array([rng.uniform(4.0, 11.0)])
    else:
        d = o.m - 2
        rho, v, p = rng.uniform(0.3, 1.4), rng.uniform(-0.8, 0.8, d), rng.uniform(0.2, 1.2)
        base = np.concatenate([[rho], rho * v, [p / 0.4 + 0.5 * rho * v @ v]])
    z = rng.standard_normal((1, o.N, o.m)).clip(-3, 3)
    amp = (0.0, 0.5) if kind in ("barrier", "quadratic") else (0.05, 0.0)
    lam = o.stress_dual(np.tile(base, (o.cells, 1)), np.tile(z, (o.cells, 1, 1)), amp)[0]
    return lam


def test_quadratic_entropy_is_stochastic_galerkin(oracle_mod):
    # s = u^2/2: u_s = Lambda, H = Gram = I, so one Newton step gives lambda = uhat
    o = _oracle(oracle_mod, "quadratic")
    rng = np.random.default_rng(0)
    for _ in range(10):
        uhat = rng.standard_normal((o.N, 1))
        lam, it, crit, st = o.dual_solve_cell(uhat, np.zeros((o.N, 1)))
        assert st == 0 and it == 1 and crit < 1e-10
        np.testing.assert_allclose(lam, uhat, atol=1e-13)
        H, _ = o.dual_hessian(lam)
        np.testing.assert_allclose(H, np.eye(o.N), atol=1e-13)


@pytest.mark.parametrize("kind", ["barrier", "euler1d", "euler2d"])
def test_xi_constant_cell_needs_no_iteration(oracle_mod, kind):
    o = _oracle(oracle_mod, kind)
    rng = np.random.default_rng(1)
    lam_star = _manufactured(o, rng, kind)
    lam_star[1:] = 0.0
    uhat, ok = o.moments_from_dual(lam_star)
    assert ok
    lam0 = o.warm_start(np.tile(uhat, (o.cells, 1, 1)))[0]
    lam, it, crit, st = o.dual_solve_cell(uhat, lam0)
    assert st == 0 and it == 0 and crit < 1e-12
    # reconstruction is the constant cell mean
    u0, _ = o.closure_u(o.quadrature()[2][0] @ lam)
    np.testing.assert_allclose(u0, uhat[0], rtol=1e-13)


@pytest.mark.parametrize("kind,M,q1d", [("barrier", 3, 6), ("euler1d", 2, 5), ("euler2d", 1, 3)])
def test_gradient_is_fd_of_dual_objective(oracle_mod, kind, M, q1d):
    o = _oracle(oracle_mod, kind, M, q1d)
    rng = np.random.default_rng(2)
    lam = _manufactured(o, rng, kind)
    uhat = _manufactured(o, rng, kind)
    uhat, _ = o.moments_from_dual(uhat)
    g, ok = o.dual_gradient(lam, uhat)
    assert ok
    h = 1e-6
    fd = np.zeros_like(lam)
    for i in range(o.N):
        for a in range(o.m):
            e = np.zeros_like(lam)
            e[i, a] = h
            fd[i, a] = (o.dual_objective(lam + e, uhat) - o.dual_objective(lam - e, uhat)) / (2 * h)
    np.testing.assert_allclose(g, fd, rtol=1e-6, atol=1e-7 * max(1.0, np.abs(g).max()))


@pytest.mark.parametrize("kind", ["barrier", "euler1d", "euler2d"])
def test_hessian_is_fd_jacobian_of_gradient(oracle_mod, kind):
    o = _oracle(oracle_mod, kind)
    rng = np.random.default_rng(3)
    lam = _manufactured(o, rng, kind)
    uhat = np.zeros_like(lam)
    H, ok = o.dual_hessian(lam)
    assert ok
    n = o.N * o.m
    h = 1e-6
    J = np.zeros((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = h
        gp, _ = o.dual_gradient(lam + e.reshape(lam.shape), uhat)
        gm, _ = o.dual_gradient(lam - e.reshape(lam.shape), uhat)
        J[:, c] = (gp - gm).ravel() / (2 * h)
    np.testing.assert_allclose(H, J, rtol=1e-5, atol=1e-5 * np.abs(H).max())
    np.testing.assert_allclose(H, H.T, atol=1e-14 * np.abs(H).max())
    assert np.linalg.eigvalsh(H).min() > 0


@pytest.mark.parametrize("kind", ["barrier", "euler1d", "euler2d"])
def test_manufactured_dual_is_recovered(oracle_mod, kind):
    o = _oracle(oracle_mod, kind)
    rng = np.random.default_rng(4)
    for _ in range(5):
        lam_star = _manufactured(o, rng, kind)
        uhat, ok = o.moments_from_dual(lam_star)
        assert ok
        lam0 = o.warm_start(np.tile(uhat, (o.cells, 1, 1)))[0]
        lam, it, crit, st = o.dual_solve_cell(uhat, lam0)
        assert st == 0 and crit < 1e-10 and 1 <= it <= 20
        np.testing.assert_allclose(lam, lam_star, rtol=0, atol=1e-8 * max(1.0, np.abs(lam_star).max()))


def test_manufactured_dual_p3_n224(oracle_mod):
    o = _oracle(oracle_mod, "euler2d_p3", M=2, q1d=4)
    rng = np.random.default_rng(5)
    lam_star = _manufactured(o, rng, "euler2d")
    uhat, _ = o.moments_from_dual(lam_star)
    lam0 = o.warm_start(np.tile(uhat, (o.cells, 1, 1)))[0]
    lam, it, crit, st = o.dual_solve_cell(uhat, lam0)
    assert st == 0 and crit < 1e-10
    np.testing.assert_allclose(lam, lam_star, atol=1e-8 * np.abs(lam_star).max())


@pytest.mark.parametrize("kind", ["barrier", "euler2d"])
def test_newton_quadratic_convergence_and_monotone_gradient(oracle_mod, kind):
    """Iterates of FULL mode are reproduced by repeated ONE_STEP calls (Alg. 2 line 5);
    the error to lambda* contracts quadratically and ||grad L|| decreases strictly."""
    o = _oracle(oracle_mod, kind)
    rng = np.random.default_rng(6)
    lam_star = _manufactured(o, rng, kind)
    uhat, _ = o.moments_from_dual(lam_star)
    lam = o.warm_start(np.tile(uhat, (o.cells, 1, 1)))[0]
    errs, crits = [], []
    for _ in range(12):
        lam, it, crit, st = o.dual_solve_cell(uhat, lam, mode="one_step")
        assert st == 0
        crits.append(crit)
        errs.append(np.abs(lam - lam_star).max())
        if it == 0:
            break
    crits = np.array(crits)
    assert (np.diff(crits[:-1]) < 0).all()
    e = np.array(errs)
    big = e > 1e-12
    ratios = e[1:][big[1:]] / e[:-1][big[1:]] ** 2
    # quadratic: e_{k+1} <= C e_k^2 once in the basin (last few iterates)
    assert ratios[-2:].max() < 1e3
    full_lam, full_it, _, _ = o.dual_solve_cell(uhat, o.warm_start(np.tile(uhat, (o.cells, 1, 1)))[0])
    np.testing.assert_array_equal(full_lam, lam)


def test_one_step_mode_skips_converged_cell(oracle_mod):
    # reading 8: ONE_STEP returns without a step if crit < tau already
    o = _oracle(oracle_mod, "euler2d")
    rng = np.random.default_rng(7)
    lam_star = _manufactured(o, rng, "euler2d")
    uhat, _ = o.moments_from_dual(lam_star)
    lam, it, crit, st = o.dual_solve_cell(uhat, lam_star, mode="one_step")
    assert it == 0 and st == 0
    np.testing.assert_array_equal(lam, lam_star)


def test_inadmissible_start_is_reported(oracle_mod):
    o = _oracle(oracle_mod, "euler2d")
    lam = np.zeros((o.N, o.m))
    lam[0] = [1.0, 0.0, 0.0, 0.5]  # v_E > 0: no admissible state
    _, it, _, st = o.dual_solve_cell(np.zeros((o.N, o.m)), lam)
    assert st == 4 and it == 0
