"""Oracle pins: basis and quadrature.

Pinned against closed forms and an independent library routine
(numpy.polynomial.legendre.leggauss), never against the oracle itself.
"""
import math

import numpy as np
import pytest

from inputs import configs


@pytest.mark.parametrize("p,M", [(1, 5), (1, 9), (2, 4), (2, 5), (2, 9), (3, 5), (3, 0), (4, 3)])
def test_basis_count_is_binomial(oracle_mod, p, M):
    # N = binom(M+p, p); N = 55 at M = 9, p = 2
    assert oracle_mod.num_basis(p, M) == math.comb(M + p, p)
    idx = oracle_mod.multi_indices(p, M)
    assert idx.shape == (math.comb(M + p, p), p)
    assert len({tuple(r) for r in idx}) == idx.shape[0]
    assert (idx.sum(axis=1) <= M).all()
    assert (np.diff(idx.sum(axis=1)) >= 0).all()  # graded


def test_basis_55_at_total_degree_9_p2(oracle_mod):
    assert oracle_mod.num_basis(2, 9) == 55


def test_multi_index_order_degree2_p2(oracle_mod):
    # graded, then lexicographically descending (prefix property for adaptivity)
    idx = oracle_mod.multi_indices(2, 2).tolist()
    assert idx == [[0, 0], [1, 0], [0, 1], [2, 0], [1, 1], [0, 2]]


@pytest.mark.parametrize("q", [2, 5, 10, 12, 20, 30])
def test_gauss_legendre_matches_numpy(oracle_mod, q):
    x, w = oracle_mod.gauss_legendre(q)
    xr, wr = np.polynomial.legendre.leggauss(q)
    np.testing.assert_allclose(x, xr, atol=1e-14)
    np.testing.assert_allclose(w, wr, atol=1e-14)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_quadrature_weights_and_moments(oracle_mod, name):
    cfg = configs.get(name, mesh=dict(nx=2, ny=2))
    o = oracle_mod.Oracle(cfg)
    xi, om, Phi = o.quadrature()
    assert abs(om.sum() - 1.0) < 1e-14  # <1>_Q = 1
    for d in range(cfg["p"]):
        assert abs(om @ xi[:, d] ** 2 - 1.0 / 3.0) < 1e-14  # <xi^2> = 1/3 for U(-1,1)
        assert abs(om @ xi[:, d] ** 4 - 1.0 / 5.0) < 1e-14


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_gram_matrix_is_identity(oracle_mod, name):
    # <phi phi^T>_Q = I: all configs' GL rules are exact to degree 2M
    cfg = configs.get(name)
    if cfg["mesh"]["kind"] == "tri":
        from inputs.generators import bump_channel_mesh
        o = oracle_mod.Oracle(cfg, bump_channel_mesh(6, 4, 1))
    else:
        o = oracle_mod.Oracle(configs.get(name, mesh=dict(nx=2, ny=2)))
    _, om, Phi = o.quadrature()
    G = Phi.T @ (om[:, None] * Phi)
    np.testing.assert_allclose(G, np.eye(G.shape[0]), atol=1e-13)


def test_phi1_at_one_is_sqrt3(oracle_mod):
    # univariate orthonormal Legendre: phi_1(1) = sqrt(3); checked through Phi of a
    # 1-node-per-side rule is not possible, so use the GL nodes: phi_1(x) = sqrt(3) x exactly.
    o = oracle_mod.Oracle(configs.get("cfg1"))
    xi, _, Phi = o.quadrature()
    np.testing.assert_allclose(Phi[:, 1], np.sqrt(3.0) * xi[:, 0], atol=1e-14)
    np.testing.assert_allclose(Phi[:, 0], 1.0, atol=0)
    # phi_2 = sqrt(5) (3x^2-1)/2
    np.testing.assert_allclose(Phi[:, 2], np.sqrt(5.0) * (3 * xi[:, 0] ** 2 - 1) / 2, atol=1e-13)


def test_tensor_rule_last_dimension_fastest(oracle_mod):
    o = oracle_mod.Oracle(configs.get("cfg3", mesh=dict(nx=2, ny=2)))
    xi, om, Phi = o.quadrature()
    x1, w1 = np.polynomial.legendre.leggauss(10)
    np.testing.assert_allclose(xi[:10, 0], x1[0], atol=1e-15)
    np.testing.assert_allclose(xi[:10, 1], x1, atol=1e-14)
    np.testing.assert_allclose(om.reshape(10, 10), np.outer(w1, w1) / 4, atol=1e-15)
    # phi_(1,1) = 3 xi1 xi2 ; index of (1,1) is 4 in the graded order
    np.testing.assert_allclose(Phi[:, 4], 3.0 * xi[:, 0] * xi[:, 1], atol=1e-14)


# ------------------------------------------------------------------ Clenshaw-Curtis and Smolyak (reading 33)
def _mono_exact(a):  # int_{-1}^{1} x^a dx
    return 0.0 if a % 2 else 2.0 / (a + 1)


def test_clenshaw_curtis_textbook_weights_and_exactness():
    import oracle

    x, w = oracle.clenshaw_curtis(3)
    np.testing.assert_allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=0, atol=1e-15)
    x, w = oracle.clenshaw_curtis(5)
    np.testing.assert_allclose(x, [-1, -np.sqrt(0.5), 0, np.sqrt(0.5), 1], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, np.array([1, 8, 12, 8, 1]) / 15, rtol=0, atol=1e-15)
    for n in (3, 5, 9, 17, 33):
        x, w = oracle.clenshaw_curtis(n)
        for a in range(n + 1):  # odd n: exact through degree n (symmetry), fails at n + 1
            assert abs((w * x**a).sum() - _mono_exact(a)) < 1e-13, (n, a)
        if n <= 9:
            assert abs((w * x ** (n + 1)).sum() - _mono_exact(n + 1)) > 1e-8


@pytest.mark.parametrize("p,counts", [(1, [1, 3, 5, 9, 17]), (2, [1, 5, 13, 29, 65]), (3, [1, 7, 25, 69])])
def test_smolyak_point_counts_weights_and_exactness(p, counts):
    """nested Clenshaw-Curtis sparse grids: the classical point counts, weights summing to 2^p, exact
    integration of every monomial of total degree <= 2(L - p) + 1 (Smolyak/Novak-Ritter)"""
    import itertools

    import oracle

    for L, cnt in zip(range(p, p + len(counts)), counts):
        xi, w = oracle.smolyak_cc(p, L)
        assert len(w) == cnt
        assert abs(w.sum() - 2.0**p) < 1e-13
        for deg in range(2 * (L - p) + 2):
            for a in itertools.product(range(deg + 1), repeat=p):
                if sum(a) != deg:
                    continue
                v = (w * np.prod([xi[:, d] ** a[d] for d in range(p)], axis=0)).sum()
                assert abs(v - np.prod([_mono_exact(ad) for ad in a])) < 1e-12, (p, L, a)
    if p == 1:  # one dimension: the Clenshaw-Curtis rule itself
        xi, w = oracle.smolyak_cc(1, 4)
        x, wc = oracle.clenshaw_curtis(9)
        np.testing.assert_allclose(xi[:, 0], x, atol=1e-15)
        np.testing.assert_allclose(w, wc, atol=1e-15)
    else:  # from level p + 2 on the combination has negative weights (the failure mode of PAPER.md:753-773)
        assert (oracle.smolyak_cc(p, p + 2)[1] < 0).any()


def test_oracle_uses_the_chosen_rule():
    import oracle
    from inputs import configs

    cfg = dict(configs.parity_variant("cfg3"), quad="smolyak", quad_level=6)
    o = oracle.Oracle(cfg)
    xi, om, _ = o.quadrature()
    xs, ws = oracle.smolyak_cc(2, 6)
    np.testing.assert_array_equal(xi, xs)
    np.testing.assert_allclose(om, ws / 4.0, rtol=0, atol=1e-17)
    cfg = dict(configs.parity_variant("cfg1"), quad="cc", q1d=9)
    xi, om, _ = oracle.Oracle(cfg).quadrature()
    np.testing.assert_allclose(om, oracle.clenshaw_curtis(9)[1] / 2.0, rtol=0, atol=1e-17)
