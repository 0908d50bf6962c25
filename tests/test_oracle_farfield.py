"""Pins of the oracle's characteristic far-field ghost state (reading 37; PAPER.md:490, 753
far-field boundaries).  The ghost is checked through what characteristic boundary theory fixes, not
by re-typing its formula: the outgoing Riemann invariant R+ = v_n + 2c/(g-1) equals the interior's,
the incoming R- = v_n - 2c/(g-1) equals the free stream's, entropy p/rho^g and tangential velocity
come from the upwind side; a free-stream interior gives the free stream back; supersonic inflow
takes the free stream, supersonic outflow the interior state."""
import numpy as np
import pytest

from oracle import farfield_ghost
from oracle.oracle import build

G = 1.4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build()


def cons(rho, vx, vy, p):
    return np.array([rho, rho * vx, rho * vy, p / (G - 1) + 0.5 * rho * (vx * vx + vy * vy)])


def prim(u):
    rho, vx, vy = u[0], u[1] / u[0], u[2] / u[0]
    return rho, vx, vy, (G - 1) * (u[3] - 0.5 * rho * (vx * vx + vy * vy))


def invariants(u, n):
    rho, vx, vy, p = prim(u)
    c = np.sqrt(G * p / rho)
    vn = vx * n[0] + vy * n[1]
    vt = np.array([vx, vy]) - vn * np.asarray(n)
    return vn + 2 * c / (G - 1), vn - 2 * c / (G - 1), p / rho ** G, vt


def unit(a):
    return np.array([np.cos(a), np.sin(a)])


def test_free_stream_interior_is_fixed_point():
    rng = np.random.default_rng(37)
    for _ in range(50):
        uf = cons(rng.uniform(0.5, 2), *rng.uniform(-0.4, 0.4, 2), rng.uniform(0.5, 1.5))
        ug = farfield_ghost(G, uf, uf, unit(rng.uniform(0, 2 * np.pi)))
        np.testing.assert_allclose(ug, uf, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("outflow", [True, False])
def test_subsonic_riemann_invariants_and_upwind_entropy(outflow):
    rng = np.random.default_rng(11 + outflow)
    for _ in range(100):
        n = unit(rng.uniform(0, 2 * np.pi))
        c0 = 1.0
        vn = (0.3 if outflow else -0.3) * c0
        t = np.array([-n[1], n[0]])
        ui = cons(rng.uniform(0.95, 1.05), *(vn * n + rng.uniform(-0.3, 0.3) * t + rng.uniform(-0.05, 0.05, 2)),
                  rng.uniform(0.68, 0.72))
        uf = cons(rng.uniform(0.95, 1.05), *(vn * n + rng.uniform(-0.3, 0.3) * t + rng.uniform(-0.05, 0.05, 2)),
                  rng.uniform(0.68, 0.72))
        ug = farfield_ghost(G, ui, uf, n)
        rpg, rmg, sg, vtg = invariants(ug, n)
        rpi, _, si, vti = invariants(ui, n)
        _, rmf, sf, vtf = invariants(uf, n)
        assert abs(rpg - rpi) <= 1e-12 * abs(rpi)  # outgoing invariant from the interior
        assert abs(rmg - rmf) <= 1e-12 * abs(rmf)  # incoming invariant from the free stream
        vng = 0.5 * (rpg + rmg)
        assert (vng > 0) == outflow
        s_up, vt_up = (si, vti) if outflow else (sf, vtf)
        assert abs(sg - s_up) <= 1e-12 * s_up
        np.testing.assert_allclose(vtg, vt_up, atol=1e-13)


def test_supersonic_in_and_outflow():
    n = unit(0.3)
    uf = cons(1.0, *(0.5 * n), 1.0 / G)
    ui_out = cons(1.1, *(2.0 * n), 0.5 / G)   # |v_n| = 2 > c ~ 0.67: outflow
    ui_in = cons(1.1, *(-2.0 * n), 0.5 / G)   # inflow
    np.testing.assert_array_equal(farfield_ghost(G, ui_out, uf, n), ui_out)
    np.testing.assert_array_equal(farfield_ghost(G, ui_in, uf, n), uf)


def test_ghost_is_rotation_covariant():
    rng = np.random.default_rng(5)
    ui, uf = cons(1.1, 0.3, 0.1, 0.7), cons(1.0, 0.4, -0.05, 1 / G)
    n = unit(0.7)
    ug = farfield_ghost(G, ui, uf, n)
    for a in rng.uniform(0, 2 * np.pi, 5):
        R = np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]])
        rot = lambda u: np.array([u[0], *(R @ u[1:3]), u[3]])  # noqa: E731
        np.testing.assert_allclose(farfield_ghost(G, rot(ui), rot(uf), R @ n), rot(ug), rtol=1e-13, atol=1e-14)
