"""Multi-rank paths on one device: the p virtual ranks of a
world driven in lockstep by tfdp_group_step / tfdp_group_forces run the same kernels, phases,
buffer layouts and message boundaries as the NCCL path, with device copies in place of the
NCCL calls.  Parity: against the one-rank context and the oracle; the exact path and the
renumbering are bitwise across rank counts (R15)."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config

pytestmark = pytest.mark.gpu


def _case(name):
    w = make_config(name)
    rp, col = O.csr_build(w.n, w.u, w.v)
    return w, rp, col


def _group(w, rp, col, X, world, prm, stream):
    return [P.Layout(w.n, rp, col, X, prm, dist=P.Dist(r, world, 0, None), stream=stream)
            for r in range(world)]


def _close(G):
    for L in G:
        L.close()


@pytest.fixture(scope="module")
def stream():
    import torch
    s = torch.cuda.Stream()
    yield s.cuda_stream
    torch.cuda.synchronize()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("k", [1, 3])
def test_slab_forces_match_one_rank_and_oracle(world, k, stream):
    """Slab-distributed convolution (row slabs, column chunks, two transposes, potential
    rows exchange) on C3 in the caller's order: every rank's shard equals the one-rank
    forces up to fp32 atomics order and the oracle within the ibFFT bar."""
    w, rp, col = _case("C3")
    prm = P.Params(solver="ibfft", k=k)
    with P.Layout(w.n, rp, col, w.xy, prm) as L1:
        R1, A1 = L1.forces()
    G = _group(w, rp, col, w.xy, world, prm, stream)
    try:
        out = P.group_forces(G)
        tol = {1: 1e-4, 3: 3e-4}[k]  # fp32 atomics noise floor of two runs (R15; k^2 terms)
        for L, (R, A) in zip(G, out):
            assert O.rel_l2(R, R1[L.lo:L.hi]) <= tol, (L.lo, O.rel_l2(R, R1[L.lo:L.hi]))
            np.testing.assert_array_equal(A, A1[L.lo:L.hi])
        R = np.concatenate([o[0] for o in out])
        e = O.rel_l2(R, O.repulsion_ibfft(w.xy.astype(np.float64), k))
        print(f"[dist] slab p={world} k={k} rel_l2 vs oracle {e:.3e}")
        assert e <= 1e-3
    finally:
        _close(G)


@pytest.mark.parametrize("world", [2, 4])
def test_slab_step_renumbered(world, stream):
    """Steps of the slab mode with the internal renumbering (n >= 65536: rank 0's Morton
    permutation broadcast to every rank): all ranks hold bitwise the same layout, the forces
    after the steps match the oracle at that layout, and the short trajectory matches the
    one-rank context's."""
    w, rp, col = _case("C3")
    prm = P.Params(solver="ibfft", k=0, iterations=20, step0=1e-3)
    with P.Layout(w.n, rp, col, w.xy, prm) as L1:
        L1.step(19)
        X1 = L1.layout()
    G = _group(w, rp, col, w.xy, world, prm, stream)
    try:
        P.group_step(G, 19)  # k = 1 x 18, then k = 2
        Xs = [L.layout() for L in G]
        for X in Xs[1:]:
            np.testing.assert_array_equal(X, Xs[0])
        assert O.rel_l2(Xs[0] - w.xy, X1 - w.xy) <= 1e-3  # fp32 atomics order (R15)
        out = P.group_forces(G)  # k = 3 at t = 19
        R = np.concatenate([o[0] for o in out])
        A = np.concatenate([o[1] for o in out])
        X = Xs[0].astype(np.float64)
        e = O.rel_l2(R, O.repulsion_ibfft(X, 3))
        print(f"[dist] slab step p={world} rel_l2 vs oracle {e:.3e}")
        assert e <= 1e-3
        assert O.rel_l2(A, O.attraction(X, rp, col)) <= 1e-4
    finally:
        _close(G)


@pytest.mark.parametrize("mode", ["spread_all", "slab"])
def test_modes_small_graph(mode, stream):
    """C2rgg (n < 65536: no renumbering), k = 2, three ranks: forces and 5 steps per mode
    against the one-rank context."""
    w, rp, col = _case("C2rgg")
    prm = P.Params(solver="ibfft", k=2, dist_mode=mode, step0=1e-2)
    with P.Layout(w.n, rp, col, w.xy, prm) as L1:
        R1, _ = L1.forces()
        L1.step(5)
        X1 = L1.layout()
    G = _group(w, rp, col, w.xy, 3, prm, stream)
    try:
        out = P.group_forces(G)
        for L, (R, _) in zip(G, out):
            assert O.rel_l2(R, R1[L.lo:L.hi]) <= 1e-5
        P.group_step(G, 5)
        # fp32 atomics order (R15) is ~1e-5 here (tools/dist_noise.py), but a node within
        # an ulp of an interval edge can take either side (the k >= 2 interpolant jumps at
        # interval edges): one such node moves the displacement rel-L2 by ~1e-3
        Xs = [L.layout() for L in G]
        for X in Xs[1:]:
            np.testing.assert_array_equal(X, Xs[0])
        assert O.rel_l2(Xs[0] - w.xy, X1 - w.xy) <= 5e-3
    finally:
        _close(G)


@pytest.mark.parametrize("p2p", ["1", "0"])
def test_exact_group_step_bitwise(p2p, stream, monkeypatch):
    """Exact path: 4 ranks x 3 steps through the group equal the one-rank steps bit for bit
    (fixed per-target source order, R15), with the position all-gather fused into the update
    (peer stores, TFDP_P2P=1) or as device copies (TFDP_P2P=0)."""
    monkeypatch.setenv("TFDP_P2P", p2p)
    w, rp, col = _case("C2")
    prm = P.Params(solver="exact")
    with P.Layout(w.n, rp, col, w.xy, prm) as L1:
        L1.step(3)
        X1 = L1.layout()
    G = _group(w, rp, col, w.xy, 4, prm, stream)
    try:
        P.group_step(G, 3)
        for L in G:
            np.testing.assert_array_equal(L.layout(), X1)
    finally:
        _close(G)


def test_group_errors(stream):
    w, rp, col = _case("C2rgg")
    prm = P.Params(solver="ibfft", k=1, dist_mode="grid_allreduce")
    G = _group(w, rp, col, w.xy, 2, prm, stream)
    try:
        with pytest.raises(P.TfdpError):  # the all-reduce mode needs a communicator
            P.group_forces(G)
    finally:
        _close(G)
    G = _group(w, rp, col, w.xy, 2, P.Params(solver="ibfft", k=1), stream)
    try:
        with pytest.raises(P.TfdpError):  # ranks out of order
            P.group_step(G[::-1], 1)
        with pytest.raises(P.TfdpError):  # a lone slab rank cannot step
            G[0].step(1)
    finally:
        _close(G)


@pytest.mark.slow
def test_slab_c4_k2(stream):
    """C4 (the bench graph) at k = 2 (P = 4096) over 2 ranks, renumbered."""
    w, rp, col = _case("C4")
    prm = P.Params(solver="ibfft", k=2, step0=1e-5)
    G = _group(w, rp, col, w.xy, 2, prm, stream)
    try:
        P.group_step(G, 8)
        X = G[0].layout().astype(np.float64)
        R = np.concatenate([o[0] for o in P.group_forces(G)])
        e = O.rel_l2(R, O.repulsion_ibfft(X, 2))
        print(f"[dist] C4 slab k=2 rel_l2 vs oracle {e:.3e}")
        assert e <= 1e-3
    finally:
        _close(G)


def test_slab_heavy_rows_renumbered(stream):
    """Slab mode on a power-law graph (Chung-Lu, hubs above the 128-edge split): the heavy
    chunk index follows the broadcast renumbering on every rank, each rank sums only its own
    shard's heavy rows; attraction and repulsion against the oracle."""
    from synth import chung_lu_graph
    n = 80_000
    u, v = chung_lu_graph(n, 17.35, 2.5, 81)
    rp, col = O.csr_build(n, u, v)
    assert np.diff(rp).max() > 500
    X = (np.random.default_rng(82).random((n, 2)) * np.sqrt(n)).astype(np.float32)

    class W:  # minimal workload record for _group
        pass
    w = W()
    w.n, w.xy = n, X
    G = _group(w, rp, col, X, 3, P.Params(solver="ibfft", k=1, step0=1e-6), stream)
    try:
        P.group_step(G, 8)
        Xg = G[0].layout().astype(np.float64)
        out = P.group_forces(G)
        R = np.concatenate([o[0] for o in out])
        A = np.concatenate([o[1] for o in out])
        assert O.rel_l2(A, O.attraction(Xg, rp, col)) <= 1e-4
        assert O.rel_l2(R, O.repulsion_ibfft(Xg, 1)) <= 1e-3
    finally:
        _close(G)


@pytest.mark.parametrize("p2p", ["1", "0"])
def test_slab_group_grows_through_replans(p2p, stream, monkeypatch):
    """A group whose layout expands far beyond the first plan (strong repulsion, rho = 50):
    every rank re-plans at the same step (identical boxes), buffers are re-allocated and the
    peer routes refreshed; the forces at the final layout match the oracle."""
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, oracle as O, paper_2303_03964_b200 as P
from synth import random_layout, random_graph
n = 2000
X = random_layout(n, 41, 3.0); u, v = random_graph(n, 2 * n, 42); rp, col = O.csr_build(n, u, v)
s = torch.cuda.Stream().cuda_stream
prm = P.Params(solver="ibfft", k=1, rho=50.0, iterations=300)
G = [P.Layout(n, rp, col, X, prm, dist=P.Dist(r, 2, 0, None), stream=s) for r in range(2)]
P0 = G[0].fft_plan(1)[0]
P.group_step(G, 96)
Xg = G[0].layout()
assert np.array_equal(Xg, G[1].layout())
R = np.concatenate([o[0] for o in P.group_forces(G)])
assert G[0].fft_plan(1)[0] > P0, (P0, G[0].fft_plan(1))
e = O.rel_l2(R, O.repulsion_ibfft(Xg.astype(np.float64), 1, rho=50.0))
print("rel", e); assert e <= 1e-3
print("grow ok")
"""
    env = dict(os.environ, TFDP_P2P=p2p)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0 and "grow ok" in r.stdout
