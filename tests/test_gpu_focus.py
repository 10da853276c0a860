"""GPU parity of local (fisheye) refinement (NEXT-4, tfdp_set_focus /
tfdp_local_refine) against the oracle's masked forces on the same seeded inputs.
Bars as for the base path: exact rel-L2 <= 1e-4, ibFFT <= 1e-3 vs the oracle's masked ibFFT
(reading R23) at the same geometry, bitwise identity for boosts (1, 1, 1) and across shards."""
import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config

pytestmark = pytest.mark.gpu

BOOSTS = [(4.0, 2.0, 2.0), (1.0, 3.0, 1.0), (2.0, 1.0, 5.0)]


def _case(name):
    w = make_config(name)
    rp, col = O.csr_build(w.n, w.u, w.v)
    return w, rp, col


@pytest.mark.parametrize("boosts", BOOSTS)
def test_exact_masked_forces(boosts):
    w, rp, col = _case("C2")
    focal = [100, 600, 601]
    fo = O.Focus(tuple(focal), *boosts)
    X = w.xy.astype(np.float64)
    lab = O.focus_region(w.n, rp, col, focal)
    with P.Layout(w.n, rp, col, w.xy, P.Params(gamma=2.5, rho=1.5)) as L:
        L.set_focus(focal, *boosts)
        R, A = L.forces()
    Re, Ae = O.forces_masked(X, rp, col, lab, fo, O.Params(gamma=2.5, rho=1.5))
    assert O.rel_l2(R, Re) <= 1e-4 and O.rel_l2(A, Ae) <= 1e-4, (O.rel_l2(R, Re), O.rel_l2(A, Ae))


@pytest.mark.parametrize("k", [1, 2, 3])
def test_ibfft_masked_forces(k):
    w, rp, col = _case("C2")
    focal = [7, 512]
    boosts = (4.0, 2.0, 3.0)
    fo = O.Focus(tuple(focal), *boosts)
    X = w.xy.astype(np.float64)
    lab = O.focus_region(w.n, rp, col, focal)
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=k)) as L:
        L.set_focus(focal, *boosts)
        R, A = L.forces()
    Ro, Ao = O.forces_masked(X, rp, col, lab, fo, solver="ibfft", k=k)
    assert O.rel_l2(R, Ro) <= 1e-3 and O.rel_l2(A, Ao) <= 1e-4, (O.rel_l2(R, Ro), O.rel_l2(A, Ao))


def test_identity_boosts_bitwise_and_clear():
    w, rp, col = _case("C2")
    for solver in ("exact", "ibfft"):
        with P.Layout(w.n, rp, col, w.xy, P.Params(solver=solver, k=1)) as L:
            R0, A0 = L.forces()
            L.set_focus([3, 4], 1.0, 1.0, 1.0)
            R1, A1 = L.forces()
            L.set_focus([3, 4], 4.0, 2.0, 2.0)
            R2, _ = L.forces()
            L.set_focus([])  # clear
            R3, A3 = L.forces()
        if solver == "exact":  # deterministic path: bitwise
            np.testing.assert_array_equal(R0, R1)
            np.testing.assert_array_equal(R0, R3)
        np.testing.assert_array_equal(A0, A1)
        np.testing.assert_array_equal(A0, A3)
        assert O.rel_l2(R2, R0) > 1e-3


def test_local_refine_matches_oracle_exact():
    w, rp, col = _case("C1")
    focal = [44, 55]
    boosts = (4.0, 2.0, 2.0)
    with P.Layout(w.n, rp, col, w.xy, P.Params(iterations=40)) as L:
        L.step(40)
        Xb = L.layout()
        L.local_refine(focal, *boosts, iterations=6)
        assert L.iteration == 6
        Xr = L.layout()
    Xo = O.local_refine(Xb.astype(np.float64), rp, col, O.Focus(tuple(focal), *boosts), T=6)
    assert O.rel_l2(Xr - Xb, Xo - Xb) < 1e-4


def test_shards_bitwise_exact():
    w, rp, col = _case("C2rgg")
    focal = [10, 900]
    with P.Layout(w.n, rp, col, w.xy) as L:
        L.set_focus(focal, 4.0, 2.0, 2.0)
        R1, A1 = L.forces()
    for world in (2, 3):
        for r in range(world):
            with P.Layout(w.n, rp, col, w.xy, dist=P.Dist(r, world, 0, None)) as L:
                L.set_focus(focal, 4.0, 2.0, 2.0)
                R, A = L.forces()
                np.testing.assert_array_equal(R, R1[L.lo:L.hi])
                np.testing.assert_array_equal(A, A1[L.lo:L.hi])


def test_reordered_context_c3():
    """Internal Morton renumbering (ibFFT, n >= 65536): the mask follows the renumbering."""
    w, rp, col = _case("C3")
    focal = [12345, 67890]
    boosts = (4.0, 2.0, 2.0)
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=1, iterations=20)) as L:
        L.set_focus(focal, *boosts)
        L.step(10)  # renumbers at the first step call
        X = L.layout()
        R, A = L.forces()
    lab = O.focus_region(w.n, rp, col, focal)
    Ro, Ao = O.forces_masked(X.astype(np.float64), rp, col, lab, O.Focus(tuple(focal), *boosts),
                             solver="ibfft", k=1)
    assert O.rel_l2(R, Ro) <= 1e-3 and O.rel_l2(A, Ao) <= 1e-4


def test_star_center_pulls_leaves_on_device():
    n = 31
    rp, col = O.csr_build(n, np.zeros(n - 1, np.int32), np.arange(1, n, dtype=np.int32))
    from synth import uniform_disc
    with P.Layout(n, rp, col, uniform_disc(n, 4.0, 21)) as L:
        L.step(300)
        X0 = L.layout()
    with P.Layout(n, rp, col, X0, P.Params(iterations=100)) as L:
        L.local_refine([0], 4.0, 1.0, 1.0, iterations=100)
        Xr = L.layout()
    with P.Layout(n, rp, col, X0, P.Params(iterations=100)) as L:
        L.step(100)
        Xc = L.layout()
    dr = np.linalg.norm(Xr[1:] - Xr[0], axis=1).mean()
    dc = np.linalg.norm(Xc[1:] - Xc[0], axis=1).mean()
    assert dr < 0.8 * dc


def test_errors():
    w, rp, col = _case("C1")
    with P.Layout(w.n, rp, col, w.xy) as L:
        for args in (([], 2.0, 1.0, 1.0), ([1], 0.5, 1.0, 1.0), ([1], 1.0, float("nan"), 1.0),
                     ([100], 2.0, 1.0, 1.0), ([-1], 2.0, 1.0, 1.0)):
            with pytest.raises(P.TfdpError) as e:
                L.local_refine(*args, iterations=1)
            assert e.value.status == 1
        L.local_refine([1], 2.0, 1.0, 1.0, iterations=2)  # still usable
        assert L.iteration == 2
