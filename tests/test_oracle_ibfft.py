"""Pins of the oracle's ibFFT path.

The interpolation scheme is an approximation with no paper force-error bound, so it is
pinned by exact special cases (partition of unity, polynomial exactness, coincident
points, P-independence, translation invariance), by the direct-sum definition of the
grid convolution, by the textbook convergence order of piecewise Lagrange
interpolation, and at layout level by the paper's +-4% band."""
import math

import numpy as np
import pytest

import oracle as O
from synth import make_config, random_layout


def _uniform(n, side, seed):
    return (np.random.default_rng(seed).random((n, 2)) * side).astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_partition_of_unity(k):
    """K == 1 => psi_1 = n and psi_x = sum x~ exactly, whatever the interpolation."""
    X = _uniform(500, 30.0, 1)
    R, info = O.repulsion_ibfft(X, k, kernel=lambda dx, dy: np.ones_like(dx + dy), return_info=True)
    psi = info["psi"]
    xt = X - info["box"].center
    np.testing.assert_allclose(psi[0], 500.0, rtol=1e-11)
    np.testing.assert_allclose(psi[1], xt[:, 0].sum(), rtol=1e-9, atol=1e-8)
    np.testing.assert_allclose(psi[2], xt[:, 1].sum(), rtol=1e-9, atol=1e-8)
    # and then F = n x~_i - sum_j x~_j, the K == 1 repulsion, exactly
    np.testing.assert_allclose(R, 500.0 * xt - xt.sum(0), rtol=1e-9, atol=1e-8)


def test_polynomial_exactness():
    """K(D) = |D|^2 is degree 2 per axis: the k=3 (quadratic) interpolation is exact,
    k <= 2 is not.  Dyadic coordinates with L = 12 = N_int make the fp32 box
    arithmetic of R19 exact, so the only error left would be interpolation error."""
    X = np.random.default_rng(2).integers(0, 12 * 64 + 1, (300, 2)) / 64.0
    X[0], X[1] = (0.0, 0.0), (12.0, 12.0)
    K2 = lambda dx, dy: dx * dx + dy * dy
    box = O.box_rule(X, n_int_min=10)
    xt = X - box.center
    d2 = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    psi_exact = np.stack([d2.sum(1), d2 @ xt[:, 0], d2 @ xt[:, 1]])
    errs = {}
    for k in (1, 2, 3):
        _, info = O.repulsion_ibfft(X, k, kernel=K2, n_int_min=10, backend="direct", return_info=True)
        errs[k] = np.abs(info["psi"] - psi_exact).max() / np.abs(psi_exact).max()
    assert errs[3] < 1e-12
    assert errs[1] > 1e-3 and errs[2] > 1e-3


@pytest.mark.parametrize("k", [1, 2, 3])
def test_coincident_points_zero(k):
    X = np.tile(np.array([[3.5, -1.25]]), (50, 1))
    R = O.repulsion_ibfft(X, k)
    assert np.abs(R).max() < 1e-9
    box = O.box_rule(X)
    assert box.L == 1.0 and box.n_int == 50  # degenerate box -> unit square


@pytest.mark.parametrize("k", [1, 2, 3])
def test_direct_convolution_equals_fft(k):
    X = _uniform(400, 20.0, 3)
    for nint in (7, 20 // k):
        a = O.repulsion_ibfft(X, k, n_int_fixed=nint, backend="direct")
        b = O.repulsion_ibfft(X, k, n_int_fixed=nint, backend="fft")
        np.testing.assert_allclose(b, a, rtol=1e-10, atol=1e-10)


def test_fft_size_independence():
    X = _uniform(400, 20.0, 4)
    M = 50 * 3
    ref = O.repulsion_ibfft(X, 3, P=2 * M - 1)
    for P in (2 * M, 2 * M + 37, 512):
        np.testing.assert_allclose(O.repulsion_ibfft(X, 3, P=P), ref, rtol=1e-10, atol=1e-11)
    with pytest.raises(ValueError):
        O.repulsion_ibfft(X, 3, P=2 * M - 2)


def test_convergence_order_and_k_ordering():
    """SPEC's case: 5000 uniform points in [0,50]^2.  Piecewise Lagrange
    interpolation with k nodes per interval converges as w^k: the log-log slope of the
    field error over N_int in {50, 100, 200} is ~1, 2, 3 for k = 1, 2, 3."""
    X = _uniform(5000, 50.0, 0)
    E = O.repulsion_exact(X)
    errs = {k: [O.rel_l2(O.repulsion_ibfft(X, k, n_int_fixed=ni), E) for ni in (50, 100, 200)]
            for k in (1, 2, 3)}
    for k in (1, 2, 3):
        slope = -np.polyfit(np.log([50, 100, 200]), np.log(errs[k]), 1)[0]
        assert abs(slope - k) < 0.3, (k, slope, errs[k])
    e1, e2, e3 = errs[1][0], errs[2][0], errs[3][0]
    assert e1 > e2 > e3  # S:298 "k=1 error strictly larger than k=3 error"
    assert errs[3][2] < 1e-3


def test_two_points_within_2pct():
    X = np.array([[0.0, 0.0], [1.0, 0.0]])
    assert O.rel_l2(O.repulsion_ibfft(X, 3), O.repulsion_exact(X)) < 0.02


def test_translation_invariance_exact():
    """Dyadic coordinates + a dyadic shift: every fp32 subtraction is exact, so the
    box-anchored scheme gives bit-identical forces."""
    g = np.random.default_rng(5)
    X = g.integers(0, 40 * 64, (800, 2)) / 64.0
    for k in (1, 3):
        a = O.repulsion_ibfft(X, k)
        b = O.repulsion_ibfft(X + np.array([1024.0, -512.0]), k)
        np.testing.assert_allclose(b, a, rtol=1e-12, atol=1e-12)


def test_interval_rule_and_top_edge():
    X = np.array([[0.0, 0.0], [100.0, 10.0], [50.0, 5.0]], dtype=np.float32)
    box = O.box_rule(X)
    assert box.L == 100.0 and box.n_int == 100 and box.w == 1.0  # N_int = max(50, ceil L)
    b, u = O.interval_coords(X, box)
    assert b[1, 0] == 99 and u[1, 0] == 1.0  # x = x_max -> last interval (R7)
    assert O.box_rule(X[:, ::-1] * 0.2).n_int == 50
    assert O.box_rule(np.array([[0, 0], [50.2, 1]], np.float32)).n_int == 51
    # Lagrange basis: l_c(t_c') = delta, sums to 1
    for k in (1, 2, 3):
        t = (np.arange(k) + 0.5) / k
        np.testing.assert_allclose(O.lagrange_weights(t, k), np.eye(k), atol=1e-15)
        np.testing.assert_allclose(O.lagrange_weights(np.linspace(0, 1, 11), k).sum(-1), 1.0, atol=1e-14)


@pytest.mark.slow
def test_layout_level_band_C2():
    """layouts from ibFFT and exact agree on NP1 within [-4%, +4%] relative.
    C2 mesh, T=300, dynamic k vs exact.  Integrator reading R2' (constant step):
    under linear cooling (R2) the k=2/3 iterations run at eta <= 0.01 and the dynamic
    run stays ~10% below exact, contradicting P:680."""
    w = make_config("C2")
    rp, col = O.csr_build(w.n, w.u, w.v)
    X0 = w.xy.astype(np.float64)
    Xe = O.run(X0, rp, col, O.Params(), T=300, solver="exact", cooling="constant")
    Xf = O.run(X0, rp, col, O.Params(), T=300, solver="ibfft", k=0, cooling="constant")
    ne, nf = O.np1(Xe, rp, col), O.np1(Xf, rp, col)
    assert abs(nf - ne) / ne <= 0.04, (ne, nf)
    assert ne > O.np1(X0, rp, col)  # the run improves neighbourhood preservation


# ---------------------------------------------------------------- reading R5' (unit width)
@pytest.mark.parametrize("side", [0.3, 7.0, 49.6, 50.0, 50.2, 123.4, 1000.7])
def test_unit_rule_box(side):
    """R5': N_int = max(50, ceil L) either way; when the span sets the count the
    intervals have unit width and the square (side N_int >= L) holds every point; below
    50 intervals the span is divided (w = L / 50, the R5 box)."""
    X = _uniform(2000, side, 11)
    X[0], X[1] = (0.0, 0.0), (side, 0.25 * side)
    u, s = O.box_rule(X, rule="unit"), O.box_rule(X, rule="span")
    assert u.n_int == s.n_int and u.L == s.L and np.array_equal(u.lo, s.lo)
    if math.ceil(float(u.L)) >= 50:
        assert u.w == np.float32(1.0)
        assert float(u.L) <= u.n_int < float(u.L) + 1.0
        np.testing.assert_allclose(u.center, u.lo.astype(np.float64) + u.n_int / 2, rtol=0, atol=0)
    else:
        assert u.w == s.w and np.array_equal(u.center, s.center)
    t = ((X.astype(np.float32) - u.lo) / u.w).astype(np.float32)
    assert t.min() >= 0.0 and t.max() <= u.n_int
    b, uu = O.interval_coords(X, u)
    assert b.min() >= 0 and b.max() <= u.n_int - 1 and uu.min() >= 0.0 and uu.max() <= 1.0


@pytest.mark.parametrize("k", [1, 2, 3])
def test_unit_equals_span_on_integer_span(k):
    """An integer span L >= 50 gives w = L / N_int = 1 under both readings: the same box,
    centre and forces, bit for bit."""
    g = np.random.default_rng(12)
    X = g.integers(0, 64 * 64 + 1, (600, 2)) / 64.0
    X[0], X[1] = (0.0, 0.0), (64.0, 3.0)
    a = O.repulsion_ibfft(X, k, rule="unit")
    b = O.repulsion_ibfft(X, k, rule="span")
    np.testing.assert_array_equal(a, b)


def test_unit_rule_polynomial_exactness_and_translation():
    """Under R5' with a non-integer span (side N_int > L): K = |D|^2 is reproduced exactly
    at k = 3 (a wrong width, anchor or centre would break it), and a dyadic shift leaves the
    forces bit-identical."""
    X = np.random.default_rng(13).integers(0, 60 * 64 + 33, (300, 2)) / 64.0
    X[0], X[1] = (0.0, 0.0), (60.5, 60.5)
    box = O.box_rule(X)
    assert box.n_int == 61 and box.w == 1.0
    K2 = lambda dx, dy: dx * dx + dy * dy
    xt = X - box.center
    d2 = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    psi_exact = np.stack([d2.sum(1), d2 @ xt[:, 0], d2 @ xt[:, 1]])
    _, info = O.repulsion_ibfft(X, 3, kernel=K2, return_info=True)
    assert np.abs(info["psi"] - psi_exact).max() / np.abs(psi_exact).max() < 1e-12
    for k in (1, 3):
        a = O.repulsion_ibfft(X, k)
        b = O.repulsion_ibfft(X + np.array([1024.0, -512.0]), k)
        np.testing.assert_allclose(b, a, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_unit_rule_partition_of_unity(k):
    X = _uniform(500, 130.0, 14)
    R, info = O.repulsion_ibfft(X, k, kernel=lambda dx, dy: np.ones_like(dx + dy), return_info=True)
    assert info["box"].w == 1.0
    xt = X - info["box"].center
    np.testing.assert_allclose(info["psi"][0], 500.0, rtol=1e-11)
    np.testing.assert_allclose(R, 500.0 * xt - xt.sum(0), rtol=1e-9, atol=1e-7)


def test_unit_rule_accuracy_matches_span():
    """Unit-width intervals (w = 1) and span-divided ones (w = L / ceil L, here 0.996) are
    the same approximation up to that width ratio: e_k differ by a few percent at most and
    keep the order e1 > e2 > e3."""
    X = _uniform(4000, 120.5, 15)
    E = O.repulsion_exact(X)
    eu = [O.rel_l2(O.repulsion_ibfft(X, k, rule="unit"), E) for k in (1, 2, 3)]
    es = [O.rel_l2(O.repulsion_ibfft(X, k, rule="span"), E) for k in (1, 2, 3)]
    assert eu[0] > eu[1] > eu[2]
    for a, b in zip(eu, es):
        assert abs(a - b) <= 0.1 * b, (eu, es)


def test_run_round_fp32_diagnostic():
    """run(round_fp32=True) (diagnostic of the device's fp32 position storage, R14): every
    stored position is an fp32 value and the trajectory stays within the accumulated
    rounding (<= 1/2 ulp per update) of the fp64 one over a few iterations."""
    w = make_config("C1")
    rp, col = O.csr_build(w.n, w.u, w.v)
    X0 = w.xy.astype(np.float64)
    a = O.run(X0, rp, col, O.Params(), T=300, t_end=3, round_fp32=True)
    b = O.run(X0, rp, col, O.Params(), T=300, t_end=3)
    np.testing.assert_array_equal(a, a.astype(np.float32).astype(np.float64))
    assert np.abs(a - b).max() <= 3 * 4 * np.spacing(np.float32(8.0))
