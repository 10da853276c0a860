"""The library's NCCL code paths on one GPU.

Real NCCL refuses two ranks on one device, so these tests load the in-process NCCL stand-in
tests/nccl_loopback (TFDP_NCCL_LIB): every rank is a host thread of one process with its own
context, stream and communicator, created from one unique id exactly as on a multi-GPU node.
That runs the product's NCCL exchanges — position and permutation broadcasts, slab
send/recv transposes, the phase-barrier / divergence / ok all-reduces, the grid all-reduce
mode, the shard gathers of forces and NP1, and the peer-route handle exchange — which the
virtual-rank tests replace by device copies.  Peer routes: TFDP_IPC_LOOPBACK=1 exchanges raw
pointers (threads of one process share an address space), so the fused peer-store path runs
behind NCCL barriers; without it CUDA IPC cannot open the process's own allocations and every
rank takes the collective fallback (also tested).  Each case runs in a subprocess under a
timeout: a mismatched collective would hang rather than fail.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOOPBACK = os.path.join(ROOT, "tests", "nccl_loopback", "libnccl_loopback.so")

PRELUDE = r"""
import threading, numpy as np, oracle as O, paper_2303_03964_b200 as P
from synth import make_config

def group(p, n, rp, col, X, prm, fn):
    uid = P.nccl_unique_id()
    res, err = [None] * p, [None] * p
    def work(r):
        try:
            with P.Layout(n, rp, col, X, prm, dist=P.Dist(r, p, 0, uid)) as L:
                res[r] = fn(L)
        except Exception as e:  # reported by the main thread
            err[r] = e
    th = [threading.Thread(target=work, args=(r,)) for r in range(p)]
    for t in th: t.start()
    for t in th: t.join()
    for e in err:
        if e is not None: raise e
    return res

def one(n, rp, col, X, prm, fn):
    with P.Layout(n, rp, col, X, prm) as L:
        return fn(L)

def case(name):
    w = make_config(name); rp, col = O.csr_build(w.n, w.u, w.v); return w, rp, col
"""


def _run(code, timeout=600, **env):
    if not os.path.exists(LOOPBACK):
        from paper_2303_03964_b200 import build as B
        B.build_nccl_loopback()
    e = dict(os.environ, TFDP_NCCL_LIB=LOOPBACK, **env)
    r = subprocess.run([sys.executable, "-c", PRELUDE + code], env=e, capture_output=True,
                       text=True, cwd=ROOT, timeout=timeout)
    print(r.stdout, r.stderr[-3000:])
    assert r.returncode == 0 and "ALL OK" in r.stdout


EXACT = r"""
w, rp, col = case("C2")
prm = P.Params(solver="exact")
def fn(L):
    R, A = L.forces(); L.step(3); return R, A, L.layout(), (L.lo, L.hi)
R1, A1, X1, _ = one(w.n, rp, col, w.xy, prm, fn)
for p in (2, 3):
    out = group(p, w.n, rp, col, w.xy, prm, fn)
    for R, A, X, (lo, hi) in out:
        assert np.array_equal(R, R1[lo:hi]) and np.array_equal(A, A1[lo:hi])
        assert np.array_equal(X, X1), p  # bitwise (R15)
    print("exact", p, "ok", flush=True)
print("ALL OK")
"""


@pytest.mark.parametrize("mode", ["p2p", "copy", "ipc_fallback"])
def test_exact_nccl(mode):
    """Exact path, p = 2, 3: shard forces and 3 steps bitwise equal to one rank, with the
    position all-gather as fused peer stores (p2p), NCCL broadcasts (copy), or the fallback
    after a failed IPC mapping."""
    env = {"p2p": dict(TFDP_IPC_LOOPBACK="1"), "copy": dict(TFDP_P2P="0"),
           "ipc_fallback": dict(TFDP_IPC_LOOPBACK="0")}[mode]
    _run(EXACT, **env)


IBFFT = r"""
import os
w, rp, col = case("C3")  # n = 10^5: renumbered (rank-0 permutation broadcast)
for mode, k, p in (("slab", 1, 2), ("slab", 2, 3), ("slab", 3, 2), ("spread_all", 1, 2),
                   ("grid_allreduce", 2, 2)):
    prm = P.Params(solver="ibfft", k=k, dist_mode=mode, step0=1e-2)
    def fn(L):
        R, A = L.forces(); L.step(8); R2, _ = L.forces()
        return R, A, L.layout(), R2, (L.lo, L.hi), L.fft_geometry()
    R1, A1, X1, R21, _, g1 = one(w.n, rp, col, w.xy, prm, fn)
    out = group(p, w.n, rp, col, w.xy, prm, fn)
    R = np.concatenate([o[0] for o in out]); A = np.concatenate([o[1] for o in out])
    e = O.rel_l2(R, R1); ea = O.rel_l2(A, A1)
    Xs = [o[2] for o in out]
    for X in Xs[1:]: assert np.array_equal(X, Xs[0])
    ex = O.rel_l2(Xs[0] - w.xy, X1 - w.xy)
    R2 = np.concatenate([o[3] for o in out])
    eo = O.rel_l2(R2, O.repulsion_ibfft(Xs[0].astype(np.float64), k))
    assert all(o[5]["P"] == g1["P"] for o in out)
    print(mode, k, p, "forces", e, "att", ea, "layout", ex, "vs oracle after 8 steps", eo, flush=True)
    tol = {1: 1e-4, 2: 3e-4, 3: 3e-4}[k]  # fp32 atomics noise floor of two runs (R15)
    assert e <= tol and ea <= 1e-6 and ex <= 5e-3 and eo <= 1e-3, (mode, k, p)
print("ALL OK")
"""


@pytest.mark.parametrize("mode", ["p2p", "copy", "ipc_fallback"])
def test_ibfft_nccl(mode):
    """ibFFT path at p = 2, 3 over the NCCL code paths: slab (k = 1, 2, 3; fused peer stores,
    NCCL send/recv copies, or the IPC fallback), spread_all and grid_allreduce: forces against
    one rank (fp32 atomics order, R15), 8 renumbered steps identical on every rank and within
    the interval-edge bar of one rank, the final forces against the oracle."""
    env = {"p2p": dict(TFDP_IPC_LOOPBACK="1"), "copy": dict(TFDP_P2P="0"),
           "ipc_fallback": dict(TFDP_IPC_LOOPBACK="0")}[mode]
    _run(IBFFT, timeout=900, **env)


MISC = r"""
w, rp, col = case("C3")
# NP1 over the shards (per-rank hits gathered with NCCL) equals one rank's
prm = P.Params(solver="ibfft", k=1)
def fn(L):
    L.step(8); return L.layout(), L.np1()
out = group(2, w.n, rp, col, w.xy, prm, fn)
X, vs = out[0][0], [o[1] for o in out]
v1 = one(w.n, rp, col, X, prm, lambda L: L.np1())  # the same layout on one rank
print("np1", v1, vs, flush=True)
assert np.array_equal(out[1][0], X) and vs[0] == vs[1] and abs(vs[0] - v1) <= 1e-12
# divergence on any rank fails every rank together (divergence word all-reduced)
prm = P.Params(solver="exact", step0=1e30)
def fdiv(L):
    try:
        L.step(4)
    except P.TfdpError as e:
        return str(e)
    return None
msgs = group(2, w.n, rp, col, w.xy, prm, fdiv)
print("diverged", msgs, flush=True)
assert all(m is not None and "diverged" in m for m in msgs)
print("ALL OK")
"""


def test_np1_and_divergence_nccl():
    """NP1 gathered over the communicator equals one rank's on the same layout; a diverging
    layout fails both ranks at the same check (divergence word all-reduced)."""
    _run(MISC, TFDP_IPC_LOOPBACK="1")


GROW = r"""
from synth import random_layout, random_graph
n = 2000
X = random_layout(n, 41, 3.0); u, v = random_graph(n, 2 * n, 42); rp, col = O.csr_build(n, u, v)
prm = P.Params(solver="ibfft", k=1, rho=50.0, iterations=300)
def fn(L):
    P0 = L.fft_plan(1)[0]
    L.step(96)
    R, _ = L.forces()
    return P0, L.fft_plan(1)[0], L.layout(), R
out = group(2, n, rp, col, X, prm, fn)
assert np.array_equal(out[0][2], out[1][2])
assert out[0][1] > out[0][0] and out[1][1] == out[0][1], [(o[0], o[1]) for o in out]
R = np.concatenate([o[3] for o in out])
e = O.rel_l2(R, O.repulsion_ibfft(out[0][2].astype(np.float64), 1, rho=50.0))
print("grow", out[0][0], "->", out[0][1], "rel", e, flush=True); assert e <= 1e-3
# host-path set_layout + PivotMDS at p = 2: every rank holds the same layout as one rank
w, rp, col = case("C3")
prm = P.Params(solver="ibfft", k=1)
def fp(L):
    L.pivot_mds(20, seed=5); Xp = L.layout()
    L.set_layout(w.xy); Xs = L.layout()
    return Xp, Xs
Xp1, _ = one(w.n, rp, col, w.xy, prm, fp)
out = group(2, w.n, rp, col, w.xy, prm, fp)
for Xp, Xs in out:
    assert np.array_equal(Xs, w.xy.astype(np.float32))
    assert O.rel_l2(Xp, Xp1) <= 1e-5
print("pmds/set_layout ok", flush=True)
print("ALL OK")
"""


def test_replans_pmds_set_layout_nccl():
    """A layout growing far beyond its first plan re-plans on every rank at the same step
    (buffers re-allocated, peer routes re-exchanged over the communicator); PivotMDS and a
    host set_layout at p = 2 leave every rank with one rank's layout."""
    _run(GROW, TFDP_IPC_LOOPBACK="1")


REFINE = r"""
w, rp, col = case("C2rgg")
focal = [10, 900]
# local (fisheye) refinement at p = 2, 3: exact steps bitwise equal to one rank
prm = P.Params(solver="exact", iterations=40)
def fl(L):
    L.step(10); L.local_refine(focal, 4.0, 2.0, 2.0, iterations=4); return L.layout()
X1 = one(w.n, rp, col, w.xy, prm, fl)
for p in (2, 3):
    for X in group(p, w.n, rp, col, w.xy, prm, fl):
        assert np.array_equal(X, X1), p
print("local_refine exact ok", flush=True)
# global refinement (gamma / rho overrides) on the slab-distributed ibFFT path at p = 2
w, rp, col = case("C3")
prm = P.Params(solver="ibfft", k=1, iterations=20)
def fg(L):
    L.step(4); L.global_refine(gamma=4.0, rho=2.0, iterations=4); R, _ = L.forces()
    return L.layout(), R
out = group(2, w.n, rp, col, w.xy, prm, fg)
assert np.array_equal(out[0][0], out[1][0])
Xg = out[0][0]
R = np.concatenate([o[1] for o in out])
# one rank at the group's final layout, same overrides (the trajectories themselves part by
# the atomics order, R15)
R1 = one(w.n, rp, col, Xg, P.Params(solver="ibfft", k=1, gamma=4.0, rho=2.0),
         lambda L: L.forces()[0])
e1 = O.rel_l2(R, R1)
e = O.rel_l2(R, O.repulsion_ibfft(Xg.astype(np.float64), 1, gamma=4.0, rho=2.0))
print("global_refine", e1, e, flush=True); assert e1 <= 1e-4 and e <= 1e-3
print("ALL OK")
"""


def test_refinement_nccl():
    """Local refinement (exact, p = 2, 3: bitwise equal to one rank) and global refinement
    (ibFFT slab, p = 2: the γ / ρ overrides against the oracle) over the NCCL paths."""
    _run(REFINE, TFDP_IPC_LOOPBACK="1")
