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
