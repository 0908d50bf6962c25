"""Oracle pins against the published values in tests/golden/ (each fixture cites its source)."""
import json
import os

import numpy as np
import pytest

from inputs import configs

from .test_oracle_fv import sod_exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def oracle_mod():
    import oracle

    oracle.build()
    return oracle


def test_basis_counts(oracle_mod):
    for c in load("basis_counts.json")["cases"]:
        assert oracle_mod.num_basis(c["p"], c["M"]) == c["N"]
        assert len(oracle_mod.multi_indices(c["p"], c["M"])) == c["N"]


def test_gauss_legendre_rules(oracle_mod):
    for r in load("gauss_legendre.json")["rules"]:
        x, w = oracle_mod.gauss_legendre(r["q"])
        np.testing.assert_allclose(np.sort(x), r["x"], atol=1e-15)
        np.testing.assert_allclose(np.asarray(w)[np.argsort(x)], r["w"], atol=1e-15)


def test_sod_star_state():
    g = load("sod_star_state.json")
    _, (p, u, rl, rr, S) = sod_exact(np.array([0.0]))
    tol = g["tol"]
    assert abs(p - g["p_star"]) < tol and abs(u - g["u_star"]) < tol
    assert abs(rl - g["rho_star_left"]) < tol and abs(rr - g["rho_star_right"]) < tol
    assert abs(S - g["shock_speed"]) < tol


def test_burgers_shock_speed_from_the_oracle_scheme(oracle_mod):
    """a deterministic (xi-independent) Burgers shock in the oracle's FV scheme moves at the
    Rankine-Hugoniot speed: the front position after t is x0 + s t within a few cells"""
    g = load("burgers_riemann.json")
    case = g["shocks"][1]  # the BASELINE cfg-1 states 12 | 3
    cfg = configs.get("cfg1", mesh=dict(nx=600))
    cfg["ic"] = dict(kind="step1d", xs0=0.5, xs1=(0.0,), states=[{"prim": (case["ul"],)}, {"prim": (case["ur"],)}])
    o = oracle_mod.Oracle(cfg)
    u, _, info = o.run(t_end=0.11)
    dx = 3.0 / 600
    mean = u[:, 0, 0]  # xi-independent: the mean is the state
    front = (np.argmax(mean < 0.5 * (case["ul"] + case["ur"])) + 0.5) * dx
    assert abs(front - (0.5 + case["speed"] * info["t"])) < 4 * dx
