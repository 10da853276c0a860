"""GPU parity of the ibFFT path: libtfdp's tfdp_forces vs the oracle's
step-by-step ibFFT at identical (box, N_int, k) — the box and interval index are decided in
fp32 on both sides (R19) — and vs the exact oracle within the oracle's own ibFFT error.
Bar: (i) rel-L2 <= 1e-3 vs oracle-ibFFT; (ii) <= e_k + 1e-3 vs exact; full-run NP1 within
0.01 (C3, dynamic k, T=300)."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from synth import blob_layout, make_config, random_graph, random_layout

pytestmark = pytest.mark.gpu
TOL_IB = 1e-3
# Per-node bars (DESIGN.md §2 "per-node tolerance").  (a) VERDICT r1's measure
# e_i = |R_i - Ro_i| / (|Ro_i| + med |Ro|) at the 99.9th percentile and the worst node, on
# the dense (unit-density, clustered, bench-shaped) layouts.  (b) everywhere, the error
# relative to the two terms whose difference is F_i (R11: F = rho (x~ psi_1 - psi_x~)):
# c_i = |R_i - Ro_i| / (rho |(|x~_i| psi_1 + |psi_x~|, |y~_i| psi_1 + |psi_y~|)|), the
# cancellation fp32 can resolve — on sparse layouts (|x~| ~ 500, |F_i| << |x~_i| psi_1)
# (a) measures that cancellation, not the kernels.
TOL_NODE_Q = 5e-3
TOL_NODE_MAX = 2e-2
TOL_COND_Q = 2e-5
TOL_COND_MAX = 3e-4


def _case(name):
    w = make_config(name)
    rp, col = O.csr_build(w.n, w.u, w.v)
    return w, rp, col


def _fft_forces(w_n, rp, col, X, k, **kw):
    with P.Layout(w_n, rp, col, X, P.Params(solver="ibfft", k=k, **kw)) as L:
        R, A = L.forces()
        geo = L.fft_geometry()
    return R, A, geo


def pernode(R, Ro):
    """(99.9th percentile, max) of e_i = |R_i - Ro_i| / (|Ro_i| + median_j |Ro_j|): a global
    rel-L2 can hide a handful of wrong nodes (e.g. a mis-assigned interval); this cannot."""
    a = np.linalg.norm(np.asarray(R, np.float64) - Ro, axis=1)
    m = np.linalg.norm(Ro, axis=1)
    e = a / (m + np.median(m))
    return float(np.quantile(e, 0.999)), float(e.max())


def percond(R, Ro, X, info, rho=1.0):
    """(99.9th percentile, max) of c_i (see above) from the oracle's psi and box."""
    psi, xt = info["psi"], np.asarray(X, np.float64) - info["box"].center
    s = rho * np.hypot(np.abs(xt[:, 0] * psi[0]) + np.abs(psi[1]), np.abs(xt[:, 1] * psi[0]) + np.abs(psi[2]))
    c = np.linalg.norm(np.asarray(R, np.float64) - Ro, axis=1) / s
    return float(np.quantile(c, 0.999)), float(c.max())


def oracle_ib(X, k, **kw):
    """Oracle ibFFT forces + the info percond needs."""
    Ro, info = O.repulsion_ibfft(np.asarray(X, np.float64), k, return_info=True, **kw)
    return Ro, (X, info, kw.get("rho", 1.0))


def check_ib(R, Ro, tag="", cond=None, dense=True):
    """Global rel-L2 <= TOL_IB; per-node (a) on dense layouts; per-node (b) given cond."""
    if isinstance(Ro, tuple):
        Ro, cond = Ro
    e = O.rel_l2(R, Ro)
    q, mx = pernode(R, Ro)
    cq, cmx = percond(R, Ro, *cond) if cond else (float("nan"), float("nan"))
    # R11 conditioning: F = x~ psi_1 - psi_x~ cancels terms of size |x~| psi_1, so the fp32
    # rel-L2 grows linearly with the box half-width at fixed density (measured 8.6e-4 at
    # C4 k = 3, span 1000; 1.0e-3 at span 2100, k = 2) while c_i stays ~1e-6: the global
    # bar is 1e-3 up to a span of 1000 and scales with the span beyond
    tol = TOL_IB * max(1.0, float(cond[1]["box"].L) / 1000.0) if cond else TOL_IB
    print(f"[parity] {tag} rel_l2={e:.3e} (bar {tol:.2e}) node_q999={q:.3e} node_max={mx:.3e} "
          f"cond_q999={cq:.3e} cond_max={cmx:.3e}")
    assert e <= tol, (tag, e)
    if dense:
        assert q <= TOL_NODE_Q and mx <= TOL_NODE_MAX, (tag, q, mx)
    if cond:
        assert cq <= TOL_COND_Q and cmx <= TOL_COND_MAX, (tag, cq, cmx)


@pytest.mark.parametrize("name", ["C2", "C2rgg"])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_c2_vs_oracle_ibfft_and_exact(name, k):
    w, rp, col = _case(name)
    X = w.xy.astype(np.float64)
    R, A, geo = _fft_forces(w.n, rp, col, w.xy, k)
    box = O.box_rule(w.xy)
    assert geo["n_int"] == box.n_int and geo["k"] == k
    assert np.float32(geo["L"]) == box.L and np.float32(geo["w"]) == box.w
    assert (np.float32(geo["lo"][0]), np.float32(geo["lo"][1])) == (box.lo[0], box.lo[1])
    assert geo["P"] >= 2 * box.n_int * k - 1
    Ro, cond = oracle_ib(X, k)
    Re = O.repulsion_exact(X)
    e_k = O.rel_l2(Ro, Re)
    check_ib(R, Ro, f"{name} k={k}", cond)
    assert O.rel_l2(R, Re) <= e_k + 1e-3
    assert O.rel_l2(A, O.attraction(X, rp, col)) <= 1e-4


@pytest.mark.parametrize("k", [1, 2, 3])
def test_fixed_grid_and_fft_size(k):
    """n_int_fixed / fft_size overrides: any P >= 2M-1 gives the same linear convolution."""
    n = 4000
    X = random_layout(n, 31, 8.0)
    u, v = random_graph(n, 4 * n, 32)
    rp, col = O.csr_build(n, u, v)
    Ro = O.repulsion_ibfft(X.astype(np.float64), k, n_int_fixed=64)
    outs = []
    for P_ in (0, {1: 512, 2: 768, 3: 1280}[k]):
        R, _, geo = _fft_forces(n, rp, col, X, k, n_int_fixed=64, fft_size=P_)
        assert geo["n_int"] == 64
        outs.append(R)
        assert O.rel_l2(R, Ro) <= TOL_IB
    assert O.rel_l2(outs[0], outs[1]) <= 2e-5


def test_c3_snapshot_all_k():
    w, rp, col = _case("C3")
    X = w.xy.astype(np.float64)
    for k in (1, 3):
        R, A, geo = _fft_forces(w.n, rp, col, w.xy, k)
        box = O.box_rule(w.xy)
        assert geo["n_int"] == box.n_int and np.float32(geo["w"]) == box.w == 1.0  # R5'
        check_ib(R, oracle_ib(X, k), f"C3 k={k}")


@pytest.mark.parametrize("k", [1, 3])
def test_c3_span_rule(k):
    """interval_rule='span' (reading R5, w = L / N_int) against the oracle's rule='span'."""
    w, rp, col = _case("C3")
    R, _, geo = _fft_forces(w.n, rp, col, w.xy, k, interval_rule="span")
    box = O.box_rule(w.xy, rule="span")
    assert geo["n_int"] == box.n_int and np.float32(geo["w"]) == box.w != 1.0
    check_ib(R, oracle_ib(w.xy, k, rule="span"), f"C3 span k={k}")


def test_kernel_spectrum_reuse_and_invalidation():
    """The kernel spectrum is recomputed only when (P, h, gamma) change (setup's key):
    every evaluation must match the oracle across gamma changes, a grid re-plan, small
    layouts whose w = L / 50 (h) changes with every layout, and k switches."""
    n = 20000
    u, v = random_graph(n, 4 * n, 51)
    rp, col = O.csr_build(n, u, v)
    X = (np.random.default_rng(52).random((n, 2)) * 180.0).astype(np.float32)
    with P.Layout(n, rp, col, X, P.Params(solver="ibfft", k=1)) as L:
        for rep in range(2):  # the second evaluation reuses the spectrum
            R, _ = L.forces()
            check_ib(R, oracle_ib(X, 1), f"reuse {rep}")
        for g in (3.0, 2.0):
            L.set_params(P.Params(solver="ibfft", k=1, gamma=g))
            R, _ = L.forces()
            check_ib(R, oracle_ib(X, 1, gamma=g), f"gamma {g}")
        for scale in (0.2, 0.23, 2.5):  # L ~ 36, 41 (w = L/50 differs) then a re-plan
            Xs = (X * scale).astype(np.float32)
            L.set_layout(Xs)
            for _ in range(2):
                R, _ = L.forces()
            check_ib(R, oracle_ib(Xs, 1), f"scale {scale}")
        for k in (2, 3, 1):
            L.set_params(P.Params(solver="ibfft", k=k))
            R, _ = L.forces()
            check_ib(R, oracle_ib(Xs, k), f"k {k}")


@pytest.mark.parametrize("layout", ["c3", "blobs"])
@pytest.mark.parametrize("k", [2, 3])
def test_morton_ordered_k23_forces(layout, k):
    """Forces after the internal Morton renumbering at k = 2, 3: the only node order in
    which the spread's warp pre-aggregation forms groups (same-interval lanes).  On C3
    (unit density) ~60 % of a warp's nodes share an interval; the clustered layout puts up
    to 32 lanes in one interval.  Compared with the oracle at the layout the context holds."""
    w, rp, col = _case("C3")
    X0 = w.xy if layout == "c3" else blob_layout(w.n, 60, 2.0, 300.0, 53)
    with P.Layout(w.n, rp, col, X0, P.Params(solver="ibfft", k=k, step0=1e-4)) as L:
        L.step(8)  # renumbers (n >= 65536) at the first step call
        R, A = L.forces()
        X = L.layout().astype(np.float64)
    check_ib(R, oracle_ib(X, k), f"morton {layout} k={k}")
    assert O.rel_l2(A, O.attraction(X, rp, col)) <= 1e-4


def test_coincident_and_degenerate():
    n = 300
    X = np.tile(np.array([[2.5, -1.0]], np.float32), (n, 1))
    u, v = random_graph(n, 600, 3)
    rp, col = O.csr_build(n, u, v)
    R, A, geo = _fft_forces(n, rp, col, X, 3)
    assert geo["L"] == 1.0 and geo["n_int"] == 50  # unit square
    assert np.abs(R).max() < 1e-4 and np.abs(A).max() == 0
    R1, _, _ = _fft_forces(1, np.zeros(2, np.int64), np.zeros(0, np.int32), X[:1], 1)
    assert np.abs(R1).max() < 1e-6


@pytest.mark.parametrize("world", [2, 5])
def test_virtual_shards(world):
    w, rp, col = _case("C2rgg")
    R1, A1, _ = _fft_forces(w.n, rp, col, w.xy, 2)
    for r in range(world):
        prm = P.Params(solver="ibfft", k=2, dist_mode="spread_all")  # a lone virtual rank
        with P.Layout(w.n, rp, col, w.xy, prm, dist=P.Dist(r, world, 0, None)) as L:
            R, A = L.forces()
            lo, hi = L.lo, L.hi
        assert O.rel_l2(R, R1[lo:hi]) <= 1e-5  # atomics order only (R15)
        np.testing.assert_array_equal(A, A1[lo:hi])


def test_step_and_dynamic_schedule():
    """Iterations follow the 90/5/5 schedule with the fused box of the update."""
    w, rp, col = _case("C2")
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0, iterations=20)) as L:
        L.step(18)
        L.forces()
        assert L.fft_geometry()["k"] == 2  # T=20 -> 18/1/1
        L.step(1)
        L.forces()
        assert L.fft_geometry()["k"] == 3
        Xg = L.layout()
    Xo = O.run(w.xy, rp, col, O.Params(), T=20, solver="ibfft", k=0, t_end=19)
    assert O.rel_l2(Xg - w.xy, Xo - w.xy) < 1e-2  # chaotic amplification is small over 19 steps


def test_grid_replans():
    """A layout that outgrows the preallocated grid: tfdp_set_layout re-plans at once (no
    capped iteration), and a layout that grows while stepping is re-planned by
    the in-step check; forces stay on the oracle's rule."""
    n = 2000
    X = random_layout(n, 41, 3.0)
    u, v = random_graph(n, 2 * n, 42)
    rp, col = O.csr_build(n, u, v)
    with P.Layout(n, rp, col, X, P.Params(solver="ibfft", k=1)) as L:
        big = (X * 60.0).astype(np.float32)  # span ~ 1000 >> initial cap
        L.set_layout(big)
        R, _ = L.forces()
        assert not L.warnings & 4
        geo = L.fft_geometry()
        box = O.box_rule(big)
        assert geo["n_int"] == box.n_int
        check_ib(R, oracle_ib(big, 1), "set_layout replan", dense=False)  # 2000 nodes, span 1000
        # strong repulsion expands the layout by far more than the 8-interval headroom
        L.set_params(P.Params(solver="ibfft", k=1, rho=50.0, iterations=300))
        L.set_layout(X)
        L.step(96)
        Xg = L.layout()
        R, _ = L.forces()
        assert L.fft_geometry()["n_int"] == O.box_rule(Xg).n_int > O.box_rule(X).n_int
    check_ib(R, oracle_ib(Xg, 1, rho=50.0), "grown", dense=False)


@pytest.mark.slow
@pytest.mark.parametrize("k", [1, 2, 3])
def test_c4_forces_vs_oracle(k):
    """1M-node RGG at the bench configuration, every k (P = 2048 / 4096 / 6144: the three
    FFT specialisations the bench runs), in the Morton order the bench runs (after 8
    iterations at a tiny step) and in the caller's order."""
    w, rp, col = _case("C4")
    X = w.xy.astype(np.float64)
    R, A, geo = _fft_forces(w.n, rp, col, w.xy, k)
    assert geo["n_int"] == O.box_rule(w.xy).n_int and geo["P"] == {1: 2048, 2: 4096, 3: 6144}[k]
    check_ib(R, oracle_ib(X, k), f"C4 k={k}")
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=k, step0=1e-5)) as L:
        L.step(8)
        R, _ = L.forces()
        Xm = L.layout().astype(np.float64)
    check_ib(R, oracle_ib(Xm, k), f"C4 morton k={k}")


@pytest.mark.slow
def test_full_run_np1_C3():
    """C3: 300 iterations, dynamic k; the NP1 of EVERY GPU run within 0.01 of the fp64
    oracle's (north star).  Measured under reading R5' (tools/np1_spread_c3.py,
    tools/np1_offset_c3.py): 8 GPU runs 0.8470 - 0.8477 (std 0.0002) vs the oracle's 0.8469;
    the oracle with fp32-stored positions 0.8470 and from 1e-7-perturbed inputs 0.8472 +-
    0.0003 (R22')."""
    w, rp, col = _case("C3")
    ngs = []
    for _ in range(3):
        with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0)) as L:
            L.step(300)
            ngs.append(O.np1(L.layout(), rp, col))
    Xo = O.run(w.xy, rp, col, O.Params(), T=300, solver="ibfft", k=0)
    no = O.np1(Xo, rp, col)
    print(f"[np1] gpu {ngs} oracle {no}")
    assert all(abs(g - no) <= 0.01 for g in ngs), (ngs, no)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_internal_node_order_is_invisible(k):
    """n >= 65536 triggers the internal Morton renumbering at the first tfdp_step call of
    >= 8 iterations.  Afterwards tfdp_set_layout / tfdp_forces / tfdp_layout must still speak
    the caller's node order: forces at a caller-supplied layout match the oracle and the
    node_order='keep' context, and the layout round-trips."""
    w, rp, col = _case("C3")
    X = w.xy.astype(np.float64)
    Ro, Ao = oracle_ib(X, k), O.attraction(X, rp, col)
    out = {}
    # step0 = 1e-3: at the default 0.1 the first iterations of C3 are chaotic enough that two
    # identical node_order='keep' runs already differ by ~2% in displacement after 8
    # iterations (fp32 atomics, R15); a small step keeps the trajectory comparison meaningful.
    for order in ("auto", "keep"):
        prm = P.Params(solver="ibfft", k=k, node_order=order, step0=1e-3)
        with P.Layout(w.n, rp, col, w.xy, prm) as L:
            L.step(8)  # renumbers (auto) and moves the layout
            moved = L.layout()
            assert not np.array_equal(moved, w.xy)
            L.set_layout(w.xy)  # back to the caller's input layout
            np.testing.assert_array_equal(L.layout(), w.xy)
            R, A = L.forces()
        check_ib(R, Ro, f"order {order} k={k}")
        assert O.rel_l2(A, Ao) <= 1e-4, order
        out[order] = (R, A, moved)
    # fp32 spread atomics (R15): two node_order='keep' runs already differ by ~3e-5 at C3
    # and k = 1; the noise floor grows with the k^2 contributions per node (1.1e-4 / 1.4e-4
    # measured at k = 2 / 3, each run within 2.2e-4 of the oracle)
    assert O.rel_l2(out["auto"][0], out["keep"][0]) <= {1: 1e-4, 2: 3e-4, 3: 3e-4}[k]
    # the 8 iterations themselves agree up to fp32 summation order (atomics, R15), and with
    # the oracle's 8 ibFFT iterations
    Xo = O.run(w.xy, rp, col, O.Params(), T=300, eta0=1e-3, solver="ibfft", k=k, t_end=8)
    da, dk, do = out["auto"][2] - w.xy, out["keep"][2] - w.xy, Xo - w.xy
    assert O.rel_l2(da, dk) <= 1e-3
    # vs the fp64 oracle: the device keeps positions in fp32 (R14), so each of the 8 updates
    # rounds by up to ulp(x)/2 -- at |x| ~ 100 that is ~1e-3 of these small displacements
    ulp = np.spacing(np.maximum(np.abs(w.xy), np.abs(out["auto"][2])).astype(np.float32))
    bound = np.linalg.norm(8 * 0.5 * ulp.astype(np.float64)) / np.linalg.norm(do)
    assert O.rel_l2(da, do) <= bound + 1e-3, bound


def test_charges_cleared_between_evaluations():
    """The interleaved charge grid is re-zeroed by every evaluation (rows_inv), whatever k:
    repeated force calls, and calls after the dynamic schedule switched k (18/1/1 at T = 20,
    P:545), match a fresh context on the same layout — leftover charges would add up."""
    w, rp, col = _case("C2rgg")
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0, iterations=20)) as L:
        R1, _ = L.forces()
        R1b, _ = L.forces()
        assert O.rel_l2(R1b, R1) <= 1e-5  # fp32 atomics order only (R15)
        L.step(18)  # k = 1 iterations; the next one is k = 2
        X = L.layout()
        R2, _ = L.forces()
        R2b, _ = L.forces()
        L.step(1)
        X3 = L.layout()
        R3, _ = L.forces()
    # the fresh context plans its FFT size from the moved layout (R9: any P >= 2M - 1 gives
    # the same kept outputs up to fp32 rounding, measured 1e-5); leftover charges would
    # shift the forces by O(1)
    for Xs, Rs, k in ((X, R2, 2), (X, R2b, 2), (X3, R3, 3)):
        Rf, _, _ = _fft_forces(w.n, rp, col, Xs, k)
        assert O.rel_l2(Rs, Rf) <= 1e-4, k
    assert O.rel_l2(R1, O.repulsion_ibfft(w.xy.astype(np.float64), 1)) <= TOL_IB


def test_spread_tile_variant_subprocess():
    """The shared-memory privatised spread (TFDP_SPREAD=tile, measured slower and kept as an
    A/B variant) is parity-tested too: Morton-ordered C3 and clustered layouts, k = 1, 3,
    including the per-node fallback of random-order contexts."""
    import subprocess
    import sys
    code = r"""
import numpy as np, oracle as O, paper_2303_03964_b200 as P
from synth import make_config, blob_layout
w = make_config("C3"); rp, col = O.csr_build(w.n, w.u, w.v)
for X0 in (w.xy, blob_layout(w.n, 60, 2.0, 300.0, 53)):
    for k in (1, 3):
        for order in ("auto", "keep"):
            with P.Layout(w.n, rp, col, X0, P.Params(solver="ibfft", k=k, step0=1e-4, node_order=order)) as L:
                L.step(8); R, _ = L.forces(); X = L.layout().astype(np.float64)
            e = O.rel_l2(R, O.repulsion_ibfft(X, k))
            print(k, order, e); assert e <= 1e-3, (k, order, e)
print("tile ok")
"""
    env = dict(os.environ, TFDP_SPREAD="tile")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0 and "tile ok" in r.stdout


@pytest.mark.parametrize("env", ["TFDP_ATTR_SIDE=0", "TFDP_HEAVY=0", "TFDP_PDL=0",
                                 "TFDP_KSPEC_OVERLAP=0", "TFDP_ROWS_RB=1", "TFDP_ROWS_RB=4",
                                 "TFDP_PDL_MAX_FFT=8192", "TFDP_ATTR_AT=1", "TFDP_ATTR_AT=2",
                                 "TFDP_ATTR_BLOCKS=296"])
def test_env_variants_subprocess(env):
    """Every A/B switch of DESIGN §7 keeps parity: Morton-ordered C3 forces at k = 1, 2, 3
    against the oracle after 8 steps, 40 iterations of the dynamic schedule, and the
    attraction (exact definition) on a Chung-Lu graph with hub rows."""
    import subprocess
    import sys
    code = r"""
import numpy as np, oracle as O, paper_2303_03964_b200 as P
from synth import make_config, random_layout
w = make_config("C3"); rp, col = O.csr_build(w.n, w.u, w.v)
for k in (1, 2, 3):
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=k, step0=1e-4)) as L:
        L.step(8); R, A = L.forces(); X = L.layout().astype(np.float64)
    e = O.rel_l2(R, O.repulsion_ibfft(X, k)); ea = O.rel_l2(A, O.attraction(X, rp, col))
    print(k, e, ea); assert e <= 1e-3 and ea <= 1e-4, (k, e, ea)
with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0, iterations=40)) as L:
    L.step(40); assert np.isfinite(L.layout()).all()
from synth import chung_lu_graph
n = 20000
u, v = chung_lu_graph(n, 12.0, 2.1, 9)  # power-law degrees: hub rows above the 128 split
rp, col = O.csr_build(n, u, v)
assert np.diff(rp).max() > 300
X = random_layout(n, 7, 40.0)
with P.Layout(n, rp, col, X, P.Params(solver="ibfft", k=1)) as L:
    _, A = L.forces()
ea = O.rel_l2(A, O.attraction(X.astype(np.float64), rp, col)); print("hubs", ea); assert ea <= 1e-4
print("variant ok")
"""
    k, v = env.split("=")
    e = dict(os.environ, **{k: v})
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0 and "variant ok" in r.stdout


def test_cols_register_variant_subprocess():
    """The register four-step column kernel (TFDP_COLS=reg, P = 2048; measured slower and
    kept as an A/B variant) is parity-tested too: forced P = 2048 grids at k = 1, 2, 3, equal
    to the radix-16 kernel up to fp32 rounding, and the slab mode's routed stores (3 virtual
    ranks)."""
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, oracle as O, paper_2303_03964_b200 as P
from synth import random_layout, random_graph
n = 6000
X = random_layout(n, 31, 30.0); u, v = random_graph(n, 4 * n, 32); rp, col = O.csr_build(n, u, v)
for k, nf in ((1, 1000), (2, 500), (3, 333)):
    prm = P.Params(solver="ibfft", k=k, n_int_fixed=nf, fft_size=2048)
    with P.Layout(n, rp, col, X, prm) as L:
        R, _ = L.forces(); assert L.fft_geometry()["P"] == 2048
    e = O.rel_l2(R, O.repulsion_ibfft(X.astype(np.float64), k, n_int_fixed=nf))
    print(k, e); assert e <= 1e-4, (k, e)
    s = torch.cuda.Stream().cuda_stream
    G = [P.Layout(n, rp, col, X, prm, dist=P.Dist(r, 3, 0, None), stream=s) for r in range(3)]
    Rg = np.concatenate([o[0] for o in P.group_forces(G)])
    for L in G: L.close()
    eg = O.rel_l2(Rg, R); print("slab", k, eg); assert eg <= 1e-4, (k, eg)  # atomics order (R15)
print("reg ok")
"""
    env = dict(os.environ, TFDP_COLS="reg")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0 and "reg ok" in r.stdout


@pytest.mark.parametrize("P_", [9216, 12288, 16384])
@pytest.mark.parametrize("k", [1, 3])
def test_large_fft_sizes_forced(P_, k):
    """FFT sizes above 8192 (the AoS one-FFT kernel spectrum / column pass, 1024-thread row
    passes), forced on a small grid: any P >= 2M - 1 gives the same linear convolution (R9),
    so the oracle runs at its own small P."""
    n = 4000
    X = random_layout(n, 61, 8.0)
    u, v = random_graph(n, 4 * n, 62)
    rp, col = O.csr_build(n, u, v)
    R, _, geo = _fft_forces(n, rp, col, X, k, n_int_fixed=100, fft_size=P_)
    assert geo["P"] == P_ and geo["n_int"] == 100
    check_ib(R, oracle_ib(X, k, n_int_fixed=100), f"P={P_} k={k}")


@pytest.mark.slow
def test_large_span_auto_plan():
    """A layout of span ~2100 (the span of the paper's 4M-node LiveJournal layout at unit
    density): the rule N_int = ceil L (R5') needs P = 9216 at k = 2, beyond the
    round-1 cap of 8192; planned automatically, no capped warning."""
    n = 105000  # unit density on a 2100 x 50 strip (the span sets N_int)
    g = np.random.default_rng(63)
    X = (g.random((n, 2)) * np.array([2100.0, 50.0])).astype(np.float32)
    u, v = random_graph(n, 3 * n, 64)
    rp, col = O.csr_build(n, u, v)
    with P.Layout(n, rp, col, X, P.Params(solver="ibfft", k=2)) as L:
        R, _ = L.forces()
        geo = L.fft_geometry()
        assert not L.warnings & 4
    assert geo["P"] == 9216 and geo["n_int"] == O.box_rule(X).n_int
    check_ib(R, oracle_ib(X, 2), "span 2100 k=2")


def test_layout_level_band_C2_gpu():
    """P:655 on the device: full C2 layouts (T = 300, constant step R2') from the exact path
    and from the ibFFT path with the dynamic 90/5/5 schedule agree on NP1 within +-4 %
    relative (the oracle's own pin: tests/test_oracle_ibfft.py::test_layout_level_band_C2),
    and each device NP1 is within 0.01 of the oracle's run of the same path (north star)."""
    w, rp, col = _case("C2")
    np1 = {}
    for solver in ("exact", "ibfft"):
        prm = P.Params(solver=solver, k=0, cooling="constant", iterations=300)
        with P.Layout(w.n, rp, col, w.xy, prm) as L:
            L.step(300)
            np1[solver] = L.np1()
    assert abs(np1["ibfft"] - np1["exact"]) / np1["exact"] <= 0.04, np1
    X0 = w.xy.astype(np.float64)
    for solver in ("exact", "ibfft"):
        Xo = O.run(X0, rp, col, O.Params(), T=300, solver=solver, k=0, cooling="constant")
        no = O.np1(Xo, rp, col)
        print(f"[np1] C2 {solver}: gpu {np1[solver]:.4f} oracle {no:.4f}")
        assert abs(np1[solver] - no) <= 0.01, (solver, np1[solver], no)
