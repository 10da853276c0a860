"""GPU NP1 (NEXT-3) through the C ABI (tfdp_np1) against the oracle's
brute-force np1_hits on the same inputs.  The kNN set decisions are taken on fp32 d^2 on
both sides (R22), so the per-node hit counts are compared bit-exactly; the NP1
value is their fixed-order mean."""
import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config, random_graph, random_layout

pytestmark = pytest.mark.gpu


def _gpu_hits(n, rp, col, X, **kw):
    with P.Layout(n, rp, col, X, P.Params(**kw)) as L:
        h = np.empty(L.hi - L.lo, np.int32)
        v = L.np1(h)
    return v, h


def test_hand_examples():
    cases = [
        (3, [(0, 1), (1, 2), (0, 2)], [[0, 0], [1, 0], [0.3, 0.9]], 1.0, [2, 2, 2]),
        (3, [(0, 1), (1, 2)], [[0, 0], [1, 0], [2, 0]], 1.0, [1, 2, 1]),
        (4, [(0, 1), (2, 3)], [[0, 0], [10, 0], [1, 0], [11, 0]], 0.0, [0, 0, 0, 0]),
    ]
    for n, e, X, np1, hits in cases:
        u, v = np.array(e, np.int32).T
        rp, col = O.csr_build(n, u, v)
        val, h = _gpu_hits(n, rp, col, np.array(X, np.float32))
        assert h.tolist() == hits and val == pytest.approx(np1, abs=1e-15)


@pytest.mark.parametrize("name", ["C1", "C2", "C2rgg"])
def test_small_configs_bit_exact(name):
    w = make_config(name)
    rp, col = O.csr_build(w.n, w.u, w.v)
    val, h = _gpu_hits(w.n, rp, col, w.xy)
    ho = O.np1_hits(w.xy, rp, col, dist="fp32")
    np.testing.assert_array_equal(h, ho)
    assert val == pytest.approx(O.np1_from_hits(ho, rp), abs=1e-14)


@pytest.mark.parametrize("n,m,scale", [(1, 0, 1.0), (2, 1, 1.0), (33, 40, 3.0), (1025, 3000, 20.0),
                                       (4099, 2000, 40.0)])
def test_ragged_and_isolated(n, m, scale):
    """Sizes off every block / warp multiple; m < n leaves degree-0 nodes (contribute 1)."""
    X = random_layout(n, n + 5, scale)
    u, v = random_graph(n, m, n + 6) if m else (np.zeros(0, np.int32),) * 2
    rp, col = O.csr_build(n, u, v)
    val, h = _gpu_hits(n, rp, col, X)
    ho = O.np1_hits(X, rp, col, dist="fp32")
    np.testing.assert_array_equal(h, ho)
    assert val == pytest.approx(O.np1_from_hits(ho, rp), abs=1e-14)


def test_lattice_ties_and_coincident_points():
    """Integer lattice positions (fp32-exact distances: many exact ties, broken by id) with
    duplicated points, and a hub of degree n - 1."""
    g = np.random.default_rng(5)
    n = 3000
    X = g.integers(0, 40, (n, 2)).astype(np.float32)  # ~1.9 points per lattice site
    u, v = random_graph(n, 4 * n, 9)
    hub_u = np.zeros(n - 1, np.int32)
    hub_v = np.arange(1, n, dtype=np.int32)
    rp, col = O.csr_build(n, np.concatenate([u, hub_u]), np.concatenate([v, hub_v]))
    val, h = _gpu_hits(n, rp, col, X)
    ho = O.np1_hits(X, rp, col, dist="fp32")
    np.testing.assert_array_equal(h, ho)
    assert h[0] == n - 1  # the hub's layout neighbourhood is everyone
    # all points coincident: every distance ties at 0 -> the k lowest other ids
    Xc = np.zeros((500, 2), np.float32)
    u, v = random_graph(500, 1500, 10)
    rp, col = O.csr_build(500, u, v)
    val, h = _gpu_hits(500, rp, col, Xc)
    np.testing.assert_array_equal(h, O.np1_hits(Xc, rp, col, dist="fp32"))


def test_c3_sampled_and_value():
    """C3 (n = 1e5, RGG, random node order): 2000 sampled nodes bit-exact against the
    brute-force oracle; the NP1 value against the oracle's fp64 KD-tree NP1."""
    w = make_config("C3")
    rp, col = O.csr_build(w.n, w.u, w.v)
    val, h = _gpu_hits(w.n, rp, col, w.xy)
    idx = np.random.default_rng(3).choice(w.n, 2000, replace=False)
    np.testing.assert_array_equal(h[idx], O.np1_hits(w.xy, rp, col, nodes=idx, dist="fp32"))
    assert val == pytest.approx(O.np1_from_hits(h, rp), abs=1e-12)
    assert abs(val - O.np1(w.xy.astype(np.float64), rp, col)) < 1e-4


def test_reordered_context_and_shards():
    """Internal Morton renumbering (ibFFT, n >= 65536) keeps the caller's order and ids for
    the tie rule; virtual shards partition the hits and the value."""
    w = make_config("C3")
    rp, col = O.csr_build(w.n, w.u, w.v)
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=1, iterations=20)) as L:
        L.step(10)  # renumbers at the first step call
        X = L.layout()
        h = np.empty(w.n, np.int32)
        val = L.np1(h)
    idx = np.random.default_rng(4).choice(w.n, 2000, replace=False)
    np.testing.assert_array_equal(h[idx], O.np1_hits(X, rp, col, nodes=idx, dist="fp32"))
    val_k, h_k = _gpu_hits(w.n, rp, col, X, solver="ibfft", k=1, node_order="keep")
    np.testing.assert_array_equal(h, h_k)
    assert val == pytest.approx(val_k, abs=1e-14)  # same hits, summed in internal slot order
    parts, hs = [], []
    for r in range(3):
        with P.Layout(w.n, rp, col, X, dist=P.Dist(r, 3, 0, None)) as L:
            hh = np.empty(L.hi - L.lo, np.int32)
            parts.append(L.np1(hh))
            hs.append(hh)
    np.testing.assert_array_equal(np.concatenate(hs), h)
    assert sum(parts) == pytest.approx(val, abs=1e-12)
