"""Oracle pins: entropy closures u_s = (grad s)^{-1}, grad u_s, s_* (App. B).

Each pin differentiates an entropy written out in this file from its printed
definition (BASELINE cfg 1 barrier, BASELINE cfg 2 U = -rho S/(gamma-1),
PAPER.md:887-890) by central finite differences, or checks an inverse pair.
"""
import numpy as np
import pytest

from inputs import configs

G = 1.4


def _cl(oracle_mod, closure, m):
    if closure == "barrier":
        cfg = configs.get("cfg1", mesh=dict(nx=2))
    elif m == 3:
        cfg = configs.get("cfg2", mesh=dict(nx=2))
    else:
        cfg = configs.get("cfg3", mesh=dict(nx=2, ny=2))
    return oracle_mod.Oracle(cfg)


def fd_grad(f, x, h=1e-6):
    g = np.zeros_like(x)
    for i in range(x.size):
        e = np.zeros_like(x)
        e[i] = h
        g[i] = (f(x + e) - f(x - e)) / (2 * h)
    return g


def fd_jac(f, x, h=1e-6):
    cols = []
    for i in range(x.size):
        e = np.zeros_like(x)
        e[i] = h
        cols.append((f(x + e) - f(x - e)) / (2 * h))
    return np.stack(cols, axis=1)


# --- bounded barrier (BASELINE cfg 1) --------------------------------------------------------
UM, UP = 2.9, 12.1


def barrier_entropy(u):
    return (u - UM) * np.log(u - UM) + (UP - u) * np.log(UP - u)


def test_barrier_ansatz_is_printed_formula(oracle_mod):
    o = _cl(oracle_mod, "barrier", 1)
    for L in [-30.0, -4.5, -1.0, 0.0, 0.3, 4.511, 25.0]:
        u, ok = o.closure_u(np.array([L]))
        assert ok
        # BASELINE cfg 1: u(Lambda) = u- + (u+ - u-)/(1 + exp(-Lambda))
        assert abs(u[0] - (UM + (UP - UM) / (1 + np.exp(-L)))) < 1e-13


def test_barrier_inverse_pair_and_derivatives(oracle_mod):
    o = _cl(oracle_mod, "barrier", 1)
    rng = np.random.default_rng(1)
    for u in rng.uniform(3.0, 12.0, 50):
        L, ok = o.closure_grad_s(np.array([u]))
        assert ok
        # grad s of the barrier entropy, by FD of the entropy written above
        assert abs(L[0] - fd_grad(lambda x: barrier_entropy(x[0]), np.array([u]))[0]) < 1e-7
        ub, _ = o.closure_u(L)
        assert abs(ub[0] - u) < 1e-13  # u_s(grad s(u)) = u
        J, _ = o.closure_du(L)
        assert abs(J[0, 0] - fd_jac(lambda x: o.closure_u(x)[0], L)[0, 0]) < 1e-7 * max(1, J[0, 0])
        # grad s_* = u_s and the Legendre identity s_* = Lambda u - s(u)
        assert abs(fd_grad(lambda x: o.closure_sstar(x), L)[0] - u) < 1e-7
        assert abs(o.closure_sstar(L) - (L[0] * u - barrier_entropy(u))) < 1e-11


# --- Euler, BASELINE scaling U = -rho S / (gamma - 1) ------------------------------------------

def euler_U(u, d):
    rho, mom, E = u[0], u[1:1 + d], u[1 + d]
    p = (G - 1) * (E - 0.5 * mom @ mom / rho)
    S = np.log(p) - G * np.log(rho)
    return -rho * S / (G - 1)


def random_states(rng, d, n):
    out = []
    for _ in range(n):
        rho = rng.uniform(0.1, 2.0)
        v = rng.uniform(-1.5, 1.5, d)
        p = rng.uniform(0.02, 2.0)
        out.append(np.concatenate([[rho], rho * v, [p / (G - 1) + 0.5 * rho * v @ v]]))
    return out


@pytest.mark.parametrize("d", [1, 2])
def test_euler_entropy_variables_are_fd_gradient(oracle_mod, d):
    o = _cl(oracle_mod, "euler", d + 2)
    for u in random_states(np.random.default_rng(d), d, 40):
        v, ok = o.closure_grad_s(u)
        assert ok
        np.testing.assert_allclose(v, fd_grad(lambda x: euler_U(x, d), u), rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("d", [1, 2])
def test_euler_inverse_pair(oracle_mod, d):
    o = _cl(oracle_mod, "euler", d + 2)
    for u in random_states(np.random.default_rng(10 + d), d, 200):
        v, _ = o.closure_grad_s(u)
        ub, ok = o.closure_u(v)
        assert ok
        np.testing.assert_allclose(ub, u, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("d", [1, 2])
def test_euler_jacobian_and_legendre_transform(oracle_mod, d):
    o = _cl(oracle_mod, "euler", d + 2)
    for u in random_states(np.random.default_rng(20 + d), d, 30):
        v, _ = o.closure_grad_s(u)
        J, ok = o.closure_du(v)
        assert ok
        np.testing.assert_allclose(J, J.T, atol=0)  # symmetric by construction
        assert np.linalg.eigvalsh(J).min() > 0  # positive definite
        Jfd = fd_jac(lambda x: o.closure_u(x)[0], v, h=1e-6)
        np.testing.assert_allclose(J, Jfd, rtol=2e-6, atol=2e-6 * np.abs(J).max())
        # U_* = rho(v), grad U_* = u_s, Legendre identity U_* = v.u - U(u)
        assert abs(o.closure_sstar(v) - u[0]) < 1e-13
        np.testing.assert_allclose(fd_grad(lambda x: o.closure_sstar(x), v), u, rtol=1e-6, atol=1e-7)
        assert abs(o.closure_sstar(v) - (v @ u - euler_U(u, d))) < 1e-10


def test_euler_inadmissible_dual(oracle_mod):
    o = _cl(oracle_mod, "euler", 4)
    _, ok = o.closure_u(np.array([0.1, 0.2, 0.3, 0.0]))
    assert not ok
    _, ok = o.closure_u(np.array([0.1, 0.2, 0.3, 0.5]))
    assert not ok


# --- App. B (paper scaling), readings 9 and 10 ---------------------------------------------------

def paper_s(u, d):
    # s(u) = -rho ln(rho^{-gamma} (E - |m|^2 / (2 rho)))
    rho, mom, E = u[0], u[1:1 + d], u[1 + d]
    return -rho * np.log(rho ** (-G) * (E - mom @ mom / (2 * rho)))


def test_app_b_gradient_with_corrected_dsde(oracle_mod):
    """Reading 9: the printed dS/dE = -(1/rho)(E - |m|^2/(2rho)) is a misprint; the oracle's
    corrected component equals the FD gradient of the printed entropy, the printed one does not."""
    L = oracle_mod.oracle.lib()
    import ctypes as C
    for u in random_states(np.random.default_rng(3), 2, 20):
        lam = np.zeros(4)
        L.orc_euler_paper_grad_s(G, 2, u.ctypes.data_as(C.POINTER(C.c_double)), lam.ctypes.data_as(C.POINTER(C.c_double)))
        fd = fd_grad(lambda x: paper_s(x, 2), u)
        np.testing.assert_allclose(lam, fd, rtol=1e-6, atol=1e-6)
        rho, m1, m2, E = u
        printed_dsde = -(1 / rho) * (E - (m1 ** 2 + m2 ** 2) / (2 * rho))
        assert abs(printed_dsde - fd[3]) > 1e-3 * abs(fd[3])


def test_app_b_alpha_with_corrected_sign(oracle_mod):
    """Reading 10: with +2 Lambda_4 gamma in alpha, u_s inverts grad s of App. B; as printed
    (-2 Lambda_4 gamma) it does not.  Also the BASELINE/paper scalings are related by
    v = (Lambda - ln(gamma-1) e_1)/(gamma-1) (reading 11)."""
    import ctypes as C
    L = oracle_mod.oracle.lib()
    o = _cl(oracle_mod, "euler", 4)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    for u in random_states(np.random.default_rng(4), 2, 50):
        lam = np.zeros(4)
        L.orc_euler_paper_grad_s(G, 2, dp(u), dp(lam))
        ub = np.zeros(4)
        assert L.orc_euler_paper_u(G, 2, dp(lam), dp(ub)) == 1
        np.testing.assert_allclose(ub, u, rtol=1e-12, atol=1e-12)
        # printed alpha (gamma-term sign as in PAPER.md:899)
        L1, L2, L3, L4 = lam
        a_pr = np.exp((L2 ** 2 + L3 ** 2 - 2 * L1 * L4 - 2 * L4 * G) / (2 * L4 * (1 - G))) * (-L4) ** (1 / (1 - G))
        assert abs(a_pr - u[0]) > 1e-3 * u[0]
        v = (lam - np.array([np.log(G - 1), 0, 0, 0])) / (G - 1)
        ubase, ok = o.closure_u(v)
        assert ok
        np.testing.assert_allclose(ubase, u, rtol=1e-12, atol=1e-12)
