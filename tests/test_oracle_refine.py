"""Oracle pins for global refinement (NEXT-1, SPEC global_refine S:359-366).

Refinement is `run` from a finished layout with gamma / rho overridden, so its arithmetic
is the pinned force step; these tests pin the override itself (closed forms on two nodes)
and the paper's qualitative effects as paired statistics on fixed seeds.
"""
import math

import numpy as np
import pytest

import oracle as O
from synth import path_graph, two_cluster_graph, uniform_disc


def _two_nodes(d):
    X = np.array([[-d / 2, 0.0], [d / 2, 0.0]])
    rp, col = O.csr_build(2, np.array([0], np.int32), np.array([1], np.int32))
    return X, rp, col


@pytest.mark.parametrize("gamma,rho", [(2.0, 4.0), (4.0, 1.0), (8.0, 0.5), (2.5, 3.0)])
def test_one_iteration_closed_form(gamma, rho):
    """T = 1: x1 = x0 + eta0 (rho d s^-gamma - alpha (1 + beta/s) d) along the pair axis,
    s = 1 + d^2 (eta_0 = eta0 at t = 0, R2)."""
    d = 1.3
    X, rp, col = _two_nodes(d)
    s = 1.0 + d * d
    push = rho * d * s ** (-gamma) - 0.1 * (1.0 + 8.0 / s) * d
    X1 = O.global_refine(X, rp, col, O.Params(), gamma=gamma, rho=rho, T=1)
    assert X1[1, 0] - X[1, 0] == pytest.approx(0.1 * push, rel=1e-13)
    assert X1[0, 0] - X[0, 0] == pytest.approx(-0.1 * push, rel=1e-13)
    assert np.all(X1[:, 1] == 0.0)


def test_identity_override_bounded_step():
    """identity override with T = 1 moves every node by at most eta0 max|F|."""
    u, v = path_graph(20)
    rp, col = O.csr_build(20, u, v)
    X = uniform_disc(20, 5.0, 11).astype(np.float64)
    R, A = O.forces_exact(X, rp, col)
    X1 = O.global_refine(X, rp, col, O.Params(), T=1)
    step = np.linalg.norm(X1 - X, axis=1)
    assert step.max() <= 0.1 * np.linalg.norm(R + A, axis=1).max() * (1 + 1e-12)
    assert step.max() > 0


def test_equilibrium_moves_with_rho():
    """Two connected nodes settle where rho s^-2 = alpha (1 + beta/s) (gamma = 2):
    u = (-alpha beta + sqrt(alpha^2 beta^2 + 4 alpha rho)) / (2 alpha), d* = sqrt(u - 1).
    Refining with rho = 4 moves the pair from d*(1) = 0.3147 to d*(4)."""
    a, b = 0.1, 8.0
    X, rp, col = _two_nodes(3.0)
    for rho in (1.0, 4.0):
        uu = (-a * b + math.sqrt(a * a * b * b + 4 * a * rho)) / (2 * a)
        dstar = math.sqrt(uu - 1.0)
        Xr = O.global_refine(X, rp, col, O.Params(), rho=rho, T=3000, cooling="constant")
        assert np.linalg.norm(Xr[0] - Xr[1]) == pytest.approx(dstar, rel=1e-6)


def test_gamma_le_one_rejected():
    X, rp, col = _two_nodes(1.0)
    for g in (1.0, 0.5):
        with pytest.raises(ValueError):
            O.global_refine(X, rp, col, O.Params(), gamma=g, T=1)
    with pytest.raises(ValueError):
        O.global_refine(X, rp, col, O.Params(), rho=0.0, T=1)


def test_large_rho_evens_edge_lengths_P20():
    """P:15-17 'a large repulsive t-force will distribute nearby nodes evenly':
    on P20, rho = 4 refinement lowers the variance (and the coefficient of variation) of
    the consecutive-edge lengths of the base layout."""
    u, v = path_graph(20)
    rp, col = O.csr_build(20, u, v)
    Xb = O.run(uniform_disc(20, 5.0, 11).astype(np.float64), rp, col, O.Params(), T=300)
    Xr = O.global_refine(Xb, rp, col, O.Params(), rho=4.0, T=300)
    lb = np.linalg.norm(Xb[u] - Xb[v], axis=1)
    lr = np.linalg.norm(Xr[u] - Xr[v], axis=1)
    assert lr.var() < 0.5 * lb.var()
    assert lr.std() / lr.mean() < 0.5 * lb.std() / lb.mean()


def test_larger_gamma_tightens_clusters():
    """P:20-21 'a repulsive force with a shorter range (larger gamma) allows to display a
    clear skeleton structure': on a weakly linked 2-block SBM (DESIGN.md reading
    R21: p_in = 0.1, p_out = 0.002, 100 + 100 nodes) gamma = 4 refinement lowers the mean
    intra-cluster / mean inter-cluster distance ratio."""
    u, v, lab = two_cluster_graph(100, 0.1, 0.002, 12)
    n = 200
    rp, col = O.csr_build(n, u, v)
    Xb = O.run(uniform_disc(n, 8.0, 13).astype(np.float64), rp, col, O.Params(), T=300)
    Xr = O.global_refine(Xb, rp, col, O.Params(), gamma=4.0, T=300)

    def ratio(X):
        D = np.linalg.norm(X[:, None] - X[None], axis=2)
        same = lab[:, None] == lab[None]
        off = ~np.eye(n, dtype=bool)
        return D[same & off].mean() / D[~same].mean()

    assert ratio(Xr) < 0.9 * ratio(Xb)
