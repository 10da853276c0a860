"""Pins of the fp64 oracle against things other than itself:
closed forms, paper/SPEC worked examples (tests/golden/force_pins.json, each cited),
invariants, special cases that reduce to textbook identities, and brute force.
CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from synth import random_graph, random_layout

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "force_pins.json")))
P0 = O.Params()


def csr_of(n, edges):
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    return O.csr_build(n, e[:, 0], e[:, 1])


# ---------------------------------------------------------------- force model (P1-P11)
def test_t_force_worked_examples():
    for d, phi, f in GOLD["t_force"]["values"]:
        assert O.t_force(d, phi) == pytest.approx(f, abs=1e-15)
    for phi, (dstar, fmax) in GOLD["t_force"]["argmax"].items():
        phi = float(phi)
        d = np.linspace(1e-6, 10, 2_000_001)
        f = O.t_force(d, phi)
        assert d[np.argmax(f)] == pytest.approx(dstar, abs=1e-5)
        assert f.max() == pytest.approx(fmax, rel=1e-9)


@pytest.mark.parametrize("phi", [1.0, 2.0, 4.0, 8.0])
def test_t_force_requirements_R1_R3(phi):
    """P:252-258 requirements: R1 bounded (< 1, max in [0,1] P:274), R2 ~ d^-(2phi-1), R3 ~ d."""
    d = np.logspace(-6, 4, 1_000_000)
    f = O.t_force(d, phi)
    dstar = 1 / math.sqrt(2 * phi - 1)
    assert f.max() <= O.t_force(dstar, phi) * (1 + 1e-12) and f.max() < 1 and dstar <= 1
    assert O.t_force(1e3, phi) * 1e3 ** (2 * phi - 1) == pytest.approx(1.0, rel=1e-2)
    assert O.t_force(1e-4, phi) / 1e-4 == pytest.approx(1.0, rel=1e-6)


def test_two_points():
    g = GOLD["two_points"]
    R = O.repulsion_exact(np.array(g["X"]), g["gamma"])
    np.testing.assert_allclose(R, g["R"], atol=1e-15)
    np.testing.assert_allclose(O.repulsion_exact_loops(np.array(g["X"]), g["gamma"]), g["R"], atol=1e-15)


def test_edge_attraction_and_resultant():
    g = GOLD["edge_d1"]
    rp, col = csr_of(2, [[0, 1]])
    R, A = O.forces_exact(np.array(g["X"]), rp, col, P0)
    np.testing.assert_allclose(A[0], g["A0"], atol=1e-15)
    np.testing.assert_allclose(R[0] + A[0], g["D0"], atol=1e-15)
    np.testing.assert_allclose(A[0], -A[1], atol=1e-15)


def test_parameter_constraint_defaults():
    assert P0.alpha * (1 + P0.beta) == pytest.approx(GOLD["alpha_beta"]["value"])
    assert P0.alpha * (1 + P0.beta) < 1 and P0.gamma > 1  # Eqs. limitweight / exponentcondiction


def test_two_node_equilibrium_closed_form_and_run():
    dstar = GOLD["equilibrium"]["d_star"]
    assert O.equilibrium_distance(P0) == pytest.approx(dstar, rel=1e-9)
    assert O.equilibrium_distance(O.Params(gamma=2.0000001)) == pytest.approx(dstar, rel=1e-5)
    rp, col = csr_of(2, [[0, 1]])
    for d, sign in ((dstar, 0), (0.5 * dstar, +1), (2 * dstar, -1)):
        R, A = O.forces_exact(np.array([[d, 0.0], [0.0, 0.0]]), rp, col, P0)
        Dx = R[0, 0] + A[0, 0]
        if sign == 0:
            assert abs(Dx) < 1e-9
        else:
            assert np.sign(Dx) == sign  # repulsive inside d*, attractive outside (P3 crossover)
    # S:355 example: two connected nodes from distance 3 end within 5% of d*
    X = O.run(np.array([[3.0, 0.0], [0.0, 0.0]]), rp, col, P0, T=300, eta0=0.1)
    assert np.linalg.norm(X[0] - X[1]) == pytest.approx(dstar, rel=0.05)


def test_equilateral_triangle():
    X = np.array([[0.0, 0.0], [1.0, 0.0], [0.5, math.sqrt(3) / 2]])
    R = O.repulsion_exact(X)
    c = X.mean(0)
    for i in range(3):
        radial = (X[i] - c) / np.linalg.norm(X[i] - c)
        assert np.linalg.norm(R[i]) == pytest.approx(GOLD["triangle"]["magnitude"], rel=1e-9)
        assert np.dot(R[i], radial) == pytest.approx(np.linalg.norm(R[i]), rel=1e-12)


def test_unit_square_corner():
    X = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    np.testing.assert_allclose(O.repulsion_exact(X)[0], GOLD["unit_square"]["R_corner"], rtol=1e-9)


def _rand_case(n=40, m=90, seed=0, scale=2.0):
    X = random_layout(n, seed, scale).astype(np.float64)
    u, v = random_graph(n, m, seed + 100)
    rp, col = O.csr_build(n, u, v)
    return X, rp, col


def test_newton_third_law_and_centroid():
    X, rp, col = _rand_case(200, 500, 1)
    R, A = O.forces_exact(X, rp, col, P0)
    scale = np.abs(R).sum() + np.abs(A).sum()
    assert np.abs(R.sum(0)).max() < 1e-12 * scale
    assert np.abs(A.sum(0)).max() < 1e-12 * scale
    X1 = O.step(X, rp, col, P0, 0.1)
    np.testing.assert_allclose(X1.mean(0), X.mean(0), atol=1e-12)


@pytest.mark.parametrize("gamma", [2.0, 3.0, 1.5])
def test_displacement_is_minus_energy_gradient(gamma):
    p = O.Params(alpha=0.1, beta=8.0, gamma=gamma, rho=1.3)
    X, rp, col = _rand_case(12, 25, 2, 1.5)
    R, A = O.forces_exact(X, rp, col, p)
    D = R + A
    h = 1e-6
    G = np.zeros_like(X)
    for i in range(X.shape[0]):
        for a in range(2):
            Xp, Xm = X.copy(), X.copy()
            Xp[i, a] += h
            Xm[i, a] -= h
            G[i, a] = (O.energy(Xp, rp, col, p) - O.energy(Xm, rp, col, p)) / (2 * h)
    np.testing.assert_allclose(D, -G, rtol=1e-5, atol=1e-8)


def test_symmetries():
    X, rp, col = _rand_case(60, 150, 3)
    R, A = O.forces_exact(X, rp, col, P0)
    # translation invariance
    R2, A2 = O.forces_exact(X + np.array([3.25, -7.5]), rp, col, P0)
    np.testing.assert_allclose(R2, R, atol=1e-12)
    np.testing.assert_allclose(A2, A, atol=1e-12)
    # rotation equivariance
    th = 0.7
    Q = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    R3, A3 = O.forces_exact(X @ Q.T, rp, col, P0)
    np.testing.assert_allclose(R3, R @ Q.T, atol=1e-12)
    np.testing.assert_allclose(A3, A @ Q.T, atol=1e-12)
    # permutation equivariance
    n = X.shape[0]
    perm = np.random.default_rng(5).permutation(n)
    inv = np.argsort(perm)
    deg = np.diff(rp)
    rows = np.repeat(np.arange(n), deg)
    rp4, col4 = O.csr_build(n, inv[rows], inv[col])
    R4, A4 = O.forces_exact(X[perm], rp4, col4, P0)
    np.testing.assert_allclose(R4, R[perm], atol=1e-12)
    np.testing.assert_allclose(A4, A[perm], atol=1e-12)


@pytest.mark.parametrize("gamma", [2.0, 1.0, 4.0])
def test_vectorized_equals_literal_loops(gamma):
    X, rp, col = _rand_case(64, 160, 4)
    X[5] = X[9]  # a coincident pair: zero contribution (R12)
    np.testing.assert_allclose(O.repulsion_exact(X, gamma, 1.7), O.repulsion_exact_loops(X, gamma, 1.7),
                               rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(O.attraction(X, rp, col, 0.2, 3.0), O.attraction_loops(X, rp, col, 0.2, 3.0),
                               rtol=1e-12, atol=1e-13)


def test_target_restriction_matches_full():
    X, rp, col = _rand_case(300, 700, 6)
    R, A = O.forces_exact(X, rp, col, P0)
    idx = np.array([0, 17, 299, 5, 5])
    R2, A2 = O.forces_exact(X, rp, col, P0, targets=idx)
    np.testing.assert_array_equal(R2, R[idx])
    np.testing.assert_array_equal(A2, A[idx])


# ---------------------------------------------------------------- schedule (P14)
def test_k_schedule_and_cooling():
    for T, (a, b, c) in GOLD["schedule"]["cases"].items():
        ks = O.k_schedule(int(T))
        assert [(ks == 1).sum(), (ks == 2).sum(), (ks == 3).sum()] == [a, b, c]
        assert np.all(np.diff(ks) >= 0)
    etas = [O.eta(t, 300) for t in range(300)]
    assert etas[0] == pytest.approx(0.1) and np.all(np.diff(etas) < 0) and etas[-1] > 0


# ---------------------------------------------------------------- CSR + shards (P16)
def test_csr_golden():
    for c in GOLD["csr"]["cases"]:
        rp, col = O.csr_build(c["n"], c["u"], c["v"])
        assert rp.tolist() == c["row_ptr"] and col.tolist() == c["col"]


def test_csr_against_set_construction():
    n = 300
    u, v = random_graph(n, 2000, 7)
    rp, col = O.csr_build(n, u, v)
    adj = [set() for _ in range(n)]
    for a, b in zip(u.tolist(), v.tolist()):
        if a != b:
            adj[a].add(b)
            adj[b].add(a)
    assert rp[0] == 0 and rp.dtype == np.int64 and col.dtype == np.int32
    for i in range(n):
        assert col[rp[i]:rp[i + 1]].tolist() == sorted(adj[i])
    assert rp[-1] == sum(len(a) for a in adj)


def test_shard_ranges_partition():
    for n in (1, 2, 7, 100, 1_000_003):
        for p in (1, 2, 3, 4, 8):
            rs = [O.shard_range(n, p, r) for r in range(p)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(p - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


# ---------------------------------------------------------------- NP1 (P15)
def test_np1_hand_examples():
    for c in GOLD["np1"]["cases"]:
        rp, col = csr_of(c["n"], c["edges"])
        assert O.np1(np.array(c["X"], dtype=np.float64), rp, col) == pytest.approx(c["np1"])


def test_np1_isolated_and_kdtree_path():
    X, rp, col = _rand_case(3000, 6000, 8, 20.0)
    a = O.np1(X, rp, col)
    b = O.np1(X, rp, col, brute_max=0)
    assert a == pytest.approx(b, abs=1e-12)
    rp1, col1 = O.csr_build(3, [0], [1])  # node 2 isolated -> contributes 1
    assert O.np1(np.array([[0, 0], [1, 0], [5, 5.0]]), rp1, col1) == pytest.approx(1.0)


def test_np1_hits_hand_examples_and_consistency():
    """Per-node hits reproduce S:427-429 (K3: 2,2,2; P3: 1,2,1; two far pairs: 0) and the
    brute-force / KD-tree np1 through NP1 = mean |∩| / (2k - |∩|)."""
    want = [[2, 2, 2], [1, 2, 1], [0, 0, 0, 0]]
    for c, w in zip(GOLD["np1"]["cases"], want):
        rp, col = csr_of(c["n"], c["edges"])
        X = np.array(c["X"], dtype=np.float64)
        for dist in ("fp64", "fp32"):
            h = O.np1_hits(X, rp, col, dist=dist)
            assert h.tolist() == w
            assert O.np1_from_hits(h, rp) == pytest.approx(c["np1"])
    X, rp, col = _rand_case(3000, 6000, 8, 20.0)
    h64 = O.np1_hits(X, rp, col)
    assert O.np1_from_hits(h64, rp) == pytest.approx(O.np1(X, rp, col, brute_max=0), abs=1e-12)
    # no near-ties in generic fp32 data: both precisions take the same decisions
    h32 = O.np1_hits(X.astype(np.float32), rp, col, dist="fp32")
    assert (h32 != h64).sum() <= 3


def test_np1_hits_tie_rule():
    """Equal distances are broken by the lower node id: node 0 at the origin with
    nodes 1, 2, 3 at distance 1 (exact in fp32) and k_0 = 1."""
    X = np.array([[0, 0], [0, 1], [-1, 0], [1, 0], [5, 5]], dtype=np.float64)
    for nb, hit in ((3, 0), (1, 1), (2, 0)):
        rp, col = O.csr_build(5, [0], [nb])
        assert O.np1_hits(X, rp, col, nodes=[0], dist="fp32")[0] == hit
    # coincident nodes: distance 0 ties, again by id
    X = np.array([[0, 0], [2, 0], [2, 0], [9, 9]], dtype=np.float64)
    rp, col = O.csr_build(4, [0, 3], [2, 1])  # node 1's nearest: node 2 (d=0), then 0
    assert O.np1_hits(X, rp, col, nodes=[1], dist="fp32")[0] == 0
    rp, col = O.csr_build(4, [2], [1])  # node 2's nearest other: node 1 (d=0, lower id)
    assert O.np1_hits(X, rp, col, nodes=[2], dist="fp32")[0] == 1
