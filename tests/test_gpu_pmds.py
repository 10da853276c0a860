"""GPU PivotMDS (NEXT-2, tfdp_pivot_mds) against the oracle's pivot_mds on the
same graphs: the pivots (integer max-min decisions) bit-exact, the layout within rel-L2
1e-5 (fp64 pipeline, fp32 output; eigenvector signs fixed by the same rule)."""
import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from synth import grid_graph, random_graph, rgg_graph

pytestmark = pytest.mark.gpu


def _gpu_pmds(n, rp, col, p, seed, **kw):
    with P.Layout(n, rp, col, np.zeros((n, 2), np.float32), P.Params(**kw)) as L:
        piv = L.pivot_mds(p, seed)
        X = L.layout()
    return X, piv


def test_path_exact():
    rp, col = O.csr_build(10, np.arange(9, dtype=np.int32), np.arange(1, 10, dtype=np.int32))
    X, piv = _gpu_pmds(10, rp, col, 4, 1)
    want = np.arange(10) - 4.5
    assert np.allclose(X[:, 0] * np.sign(X[-1, 0]), want, atol=1e-5)
    assert np.abs(X[:, 1]).max() < 1e-5
    _, po = O.pivot_mds(rp, col, 4, 1)
    np.testing.assert_array_equal(piv, po)


@pytest.mark.parametrize("n,m,p,seed", [(300, 700, 12, 9), (500, 400, 20, 2), (1000, 2500, 64, 5)])
def test_pivots_and_layout_random(n, m, p, seed):
    """Random graphs, some disconnected (unreachable rule R24)."""
    u, v = random_graph(n, m, seed + 10)
    rp, col = O.csr_build(n, u, v)
    X, piv = _gpu_pmds(n, rp, col, p, seed)
    Xo, po = O.pivot_mds(rp, col, p, seed)
    np.testing.assert_array_equal(piv, po)
    assert O.rel_l2(X, Xo) < 1e-5, O.rel_l2(X, Xo)


def test_grid_and_rgg_layouts():
    u, v = grid_graph(30, 12)
    rp, col = O.csr_build(360, u, v)
    X, piv = _gpu_pmds(360, rp, col, 30, 4)
    Xo, po = O.pivot_mds(rp, col, 30, 4)
    np.testing.assert_array_equal(piv, po)
    assert O.rel_l2(X, Xo) < 1e-5
    n = 20000
    u, v, xy = rgg_graph(n, np.sqrt(8 / np.pi), np.sqrt(n), 7)
    rp, col = O.csr_build(n, u, v)
    X, piv = _gpu_pmds(n, rp, col, 20, 11)
    Xo, po = O.pivot_mds(rp, col, 20, 11)
    np.testing.assert_array_equal(piv, po)
    assert O.rel_l2(X, Xo) < 1e-5
    # SPEC invariants on the device output
    assert np.abs(X.astype(np.float64).mean(0)).max() < 1e-5
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.linalg.norm(X[rows] - X[col], axis=1).mean() == pytest.approx(1.0, rel=1e-5)


def test_reordered_context_and_errors():
    n = 70000  # >= 65536: the ibFFT context renumbers nodes internally
    u, v, xy = rgg_graph(n, np.sqrt(8 / np.pi), np.sqrt(n), 8)
    rp, col = O.csr_build(n, u, v)
    X1, p1 = _gpu_pmds(n, rp, col, 16, 3)
    with P.Layout(n, rp, col, xy, P.Params(solver="ibfft", k=1, iterations=20)) as L:
        L.step(10)  # renumbered
        p2 = L.pivot_mds(16, 3)
        X2 = L.layout()
        L.step(2)  # the PMDS layout is a valid state
        for bad in (0, 65):
            with pytest.raises(P.TfdpError) as e:
                L.pivot_mds(bad, 0)
            assert e.value.status == 1
    np.testing.assert_array_equal(p1, p2)
    np.testing.assert_array_equal(X1, X2)
