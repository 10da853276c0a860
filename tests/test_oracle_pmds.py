"""Oracle pins for the PivotMDS initialisation (NEXT-2, SPEC init_pivot_mds
S:110-118).  Pinned by: the published SplitMix64 output, BFS against scipy's shortest
paths, the max-min pivot rule against brute force on all-pairs distances, PivotMDS
exactness on a 1-D metric (a path: equally spaced collinear positions), and the SPEC
invariants (centred, mean edge length 1, orthogonal Gram fixed points)."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

import oracle as O
from synth import grid_graph, random_graph


def test_splitmix64_reference_values():
    # SplitMix64 (Steele, Lea, Flood 2014) from state 0: first outputs
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF
    assert O.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def _csr(n, u, v):
    return O.csr_build(n, u, v)


def test_bfs_against_scipy():
    n = 400
    u, v = random_graph(n, 500, 3)  # sparse: several components
    rp, col = _csr(n, u, v)
    A = sp.csr_matrix((np.ones(len(col)), col, rp), shape=(n, n))
    ref = shortest_path(A, unweighted=True, directed=False)
    for s in (0, 7, 123, 399):
        d = O.bfs_hops(rp, col, s)
        want = np.where(np.isinf(ref[s]), -1, ref[s]).astype(np.int64)
        np.testing.assert_array_equal(d, want)


def test_pivots_max_min_brute_force():
    n = 300
    u, v = random_graph(n, 700, 5)
    rp, col = _csr(n, u, v)
    A = sp.csr_matrix((np.ones(len(col)), col, rp), shape=(n, n))
    ref = shortest_path(A, unweighted=True, directed=False)
    pivots, D = O.pmds_pivots(rp, col, 12, seed=9)
    assert pivots[0] == O.splitmix64(9) % n
    mind = np.full(n, np.inf)
    for j, p in enumerate(pivots):
        d = ref[p].copy()
        d[np.isinf(d)] = d[~np.isinf(d)].max() + 1
        np.testing.assert_array_equal(D[:, j], d)
        mind = np.minimum(mind, d)
        if j + 1 < len(pivots):
            cand = np.nonzero(mind == mind.max())[0]
            assert pivots[j + 1] == cand[0]


@pytest.mark.parametrize("p", [3, 5, 10])
def test_path_is_exact_1d(p):
    """A path's hop metric is 1-D Euclidean: PivotMDS recovers it exactly (any >= 2 pivots):
    x_i = +-(i - 4.5), y = 0 at mean edge length 1."""
    rp, col = _csr(10, list(range(9)), list(range(1, 10)))
    X, piv = O.pivot_mds(rp, col, p, seed=1)
    want = np.arange(10) - 4.5
    assert np.allclose(np.abs(X[:, 0]), np.abs(want), atol=1e-9)
    assert np.allclose(X[:, 0] * np.sign(X[-1, 0]), want, atol=1e-9)
    assert np.abs(X[:, 1]).max() < 1e-9


def test_invariants_grid():
    u, v = grid_graph(20, 10)
    n = 200
    rp, col = _csr(n, u, v)
    X, piv = O.pivot_mds(rp, col, 25, seed=3)
    assert np.abs(X.mean(0)).max() < 1e-9  # centred
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.linalg.norm(X[rows] - X[col], axis=1).mean() == pytest.approx(1.0, abs=1e-9)
    assert abs(X[:, 0] @ X[:, 1]) < 1e-6 * np.linalg.norm(X[:, 0]) * np.linalg.norm(X[:, 1])
    # the long side of the 20 x 10 grid is the first axis
    assert np.ptp(X[:, 0]) > 1.5 * np.ptp(X[:, 1])
    X2, piv2 = O.pivot_mds(rp, col, 25, seed=3)
    np.testing.assert_array_equal(X, X2)  # deterministic
    with pytest.raises(ValueError):
        O.pivot_mds(rp, col, 0)
