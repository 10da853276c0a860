"""GPU parity of the exact path (SURVEY.md §8(c) parity criteria) through the C ABI:
libtfdp's tfdp_forces / tfdp_step vs the fp64 oracle on the same seeded inputs.
Bar: rel-L2 <= 1e-4 per force field (north_star), bitwise determinism across shard counts
(R15), full-run NP1 within 0.01 (C1)."""
import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config, random_graph, random_layout

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _case(name):
    w = make_config(name)
    rp, col = O.csr_build(w.n, w.u, w.v)
    return w, rp, col


def _check(R, A, X, rp, col, p=O.Params(), targets=None, tol=TOL):
    Re, Ae = O.forces_exact(X.astype(np.float64), rp, col, p, targets=targets)
    eR, eA = O.rel_l2(R, Re), O.rel_l2(A, Ae)
    assert eR <= tol and eA <= tol, (eR, eA)
    return eR, eA


@pytest.mark.parametrize("name", ["C1", "C2", "C2rgg"])
def test_forces_small_configs(name):
    w, rp, col = _case(name)
    with P.Layout(w.n, rp, col, w.xy) as L:
        R, A = L.forces()
    _check(R, A, w.xy, rp, col)


@pytest.mark.parametrize("n", [1, 2, 31, 1023, 1025, 4097, 20011])
def test_forces_ragged_sizes(n):
    """Tile / chunk / block tails: n not a multiple of 1024 sources or 1024 targets."""
    X = random_layout(n, n, 3.0 + n ** 0.5 / 2)
    u, v = random_graph(n, 3 * n, n + 1) if n > 1 else (np.zeros(0, np.int32),) * 2
    rp, col = O.csr_build(n, u, v)
    with P.Layout(n, rp, col, X) as L:
        R, A = L.forces()
    if n == 1:
        assert np.all(R == 0) and np.all(A == 0)
    else:
        _check(R, A, X, rp, col)


@pytest.mark.parametrize("gamma,rho,alpha,beta", [(1.0, 1.0, 0.1, 8.0), (3.0, 2.0, 0.05, 4.0),
                                                  (4.0, 1.0, 0.1, 8.0), (8.0, 1.0, 0.1, 8.0),
                                                  (1.5, 1.0, 0.1, 8.0), (2.5, 0.7, 0.2, 1.0)])
def test_forces_parameters(gamma, rho, alpha, beta):
    """Integer-gamma templates and the general exp2/log2 path (NEXT-1 global refinement uses
    larger gamma / rho)."""
    n = 3000
    X = random_layout(n, 7, 20.0)
    u, v = random_graph(n, 4 * n, 8)
    rp, col = O.csr_build(n, u, v)
    prm = P.Params(gamma=gamma, rho=rho, alpha=alpha, beta=beta)
    with P.Layout(n, rp, col, X, prm) as L:
        R, A = L.forces()
        warn = L.warnings
    _check(R, A, X, rp, col, O.Params(alpha=alpha, beta=beta, gamma=gamma, rho=rho),
           tol=TOL if gamma == int(gamma) else 3e-4)
    assert bool(warn & 2) == (gamma <= 1)  # TFDP_WARN_GAMMA


def test_coincident_and_isolated_nodes():
    """d = 0 pairs contribute 0 (R12); degree-0 nodes feel repulsion only (R13)."""
    n = 500
    X = random_layout(n, 11, 5.0)
    X[10:20] = X[5]  # coincident cluster
    u, v = random_graph(n, 300, 12)  # many isolated nodes
    rp, col = O.csr_build(n, u, v)
    with P.Layout(n, rp, col, X) as L:
        R, A = L.forces()
    _check(R, A, X, rp, col)
    assert np.all(np.isfinite(R))


def test_c3_snapshot_sampled():
    w, rp, col = _case("C3")
    with P.Layout(w.n, rp, col, w.xy) as L:
        R, A = L.forces()
    idx = np.random.default_rng(0).choice(w.n, 2048, replace=False)
    _check(R[idx], A[idx], w.xy, rp, col, targets=idx)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_virtual_shards_bitwise(world):
    """Every target keeps the same source order, so each shard equals the p=1 slice
    bit for bit (R15); shard ranges follow the rule of §8(b)."""
    n = 5000
    X = random_layout(n, 21, 15.0)
    u, v = random_graph(n, 5 * n, 22)
    rp, col = O.csr_build(n, u, v)
    with P.Layout(n, rp, col, X) as L:
        R1, A1 = L.forces()
    for r in range(world):
        d = P.Dist(r, world, 0, None)
        with P.Layout(n, rp, col, X, dist=d) as L:
            lo, hi = L.lo, L.hi
            assert (lo, hi) == O.shard_range(n, world, r)
            R, A = L.forces()
            with pytest.raises(P.TfdpError):
                L.step(1)  # virtual shard has no communicator
        np.testing.assert_array_equal(R, R1[lo:hi])
        np.testing.assert_array_equal(A, A1[lo:hi])


def test_step_matches_oracle_and_is_deterministic():
    w, rp, col = _case("C2")
    outs = []
    for _ in range(2):
        with P.Layout(w.n, rp, col, w.xy) as L:
            L.step(5)
            assert L.iteration == 5
            outs.append(L.layout())
    np.testing.assert_array_equal(outs[0], outs[1])
    Xo = O.run(w.xy, rp, col, O.Params(), T=300, t_end=5)
    assert O.rel_l2(outs[0] - w.xy, Xo - w.xy) < 1e-4  # displacement parity


def test_full_run_np1_C1():
    """C1: 300 exact iterations (T=300, eta0=0.1, linear cooling R2); NP1 within 0.01."""
    w, rp, col = _case("C1")
    with P.Layout(w.n, rp, col, w.xy) as L:
        L.step(300)
        Xg = L.layout()
    Xo = O.run(w.xy, rp, col, O.Params(), T=300)
    ng, no = O.np1(Xg, rp, col), O.np1(Xo, rp, col)
    assert abs(ng - no) <= 0.01, (ng, no)


def test_resume_and_errors():
    w, rp, col = _case("C1")
    with P.Layout(w.n, rp, col, w.xy) as L:
        L.step(10)
        X10 = L.layout()
        L.step(10)
        X20 = L.layout()
    with P.Layout(w.n, rp, col, X10, P.Params(t0=10)) as L:  # checkpoint = layout + t
        L.step(10)
        np.testing.assert_array_equal(L.layout(), X20)
        with pytest.raises(P.TfdpError) as e:
            L.step(290)  # t would exceed T under linear cooling
        assert e.value.status == 5
    with P.Layout(w.n, rp, col, w.xy, P.Params(step0=1e30)) as L:
        with pytest.raises(P.TfdpError) as e:
            L.step(5)
        assert e.value.status == 4 and "diverged at iter" in str(e.value)
        with pytest.raises(P.TfdpError) as e:
            L.step(1)
        assert e.value.status == 5  # errored context


def test_device_buffers_and_stream():
    import torch

    w, rp, col = _case("C2")
    X = torch.from_numpy(w.xy).cuda()
    s = torch.cuda.Stream()
    with P.Layout(w.n, rp, col, X, stream=s.cuda_stream) as L:
        R = torch.empty((w.n, 2), dtype=torch.float32, device="cuda")
        A = torch.empty_like(R)
        L.forces(R, A)
        s.synchronize()
        _check(R.cpu().numpy(), A.cpu().numpy(), w.xy, rp, col)
        out = torch.empty_like(R)
        L.layout(out)
        s.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), w.xy)


@pytest.mark.slow
def test_c5_sampled_targets():
    """4M-node Chung-Lu graph: 1024 seeded sampled targets against all n sources (fp64)."""
    w, rp, col = _case("C5")
    idx = np.random.default_rng(4).choice(w.n, 1024, replace=False)
    with P.Layout(w.n, rp, col, w.xy) as L:
        R, A = L.forces()
    _check(R[idx], A[idx], w.xy, rp, col, targets=idx)
