"""Oracle pins for local (fisheye) refinement (NEXT-4, SPEC RefinementMask S:155-158,
local_refine S:368-376).  The masked forces are pinned by brute force, Newton's third law
(the weights are symmetric), D = -grad E_masked, the identity mask, the ibFFT correction
rule against the exact masked sum, and the paired statistics of S:375-376."""
import numpy as np
import pytest

import oracle as O
from synth import make_config, random_graph, random_layout, two_cluster_graph, uniform_disc


def _case(n=40, m=80, seed=3, scale=3.0):
    X = random_layout(n, seed, scale).astype(np.float64)
    u, v = random_graph(n, m, seed + 1)
    rp, col = O.csr_build(n, u, v)
    return X, rp, col


def test_region_hand_example():
    rp, col = O.csr_build(6, [0, 1, 2, 3, 4], [1, 2, 3, 4, 5])  # path 0-1-2-3-4-5
    assert O.focus_region(6, rp, col, [2]).tolist() == [0, 1, 1, 1, 0, 0]
    assert O.focus_region(6, rp, col, [0, 5]).tolist() == [1, 1, 0, 0, 1, 1]


@pytest.mark.parametrize("la,lf,ls", [(1, 1, 1), (4, 2, 2), (1, 3, 1), (2, 1, 5)])
def test_masked_equals_loops_and_newton(la, lf, ls):
    X, rp, col = _case()
    fo = O.Focus((3, 17), la, lf, ls)
    lab = O.focus_region(40, rp, col, fo.focal)
    R = O.repulsion_masked_exact(X, lab, fo, 2.5, 1.5)
    np.testing.assert_allclose(R, O.repulsion_masked_loops(X, lab, fo, 2.5, 1.5), rtol=1e-11, atol=1e-13)
    A = O.attraction_masked(X, rp, col, lab, fo)
    assert np.abs(R.sum(0)).max() < 1e-12 * np.abs(R).sum()
    assert np.abs(A.sum(0)).max() < 1e-12 * np.abs(A).sum()
    if (la, lf, ls) == (1, 1, 1):  # identity mask
        np.testing.assert_allclose(R, O.repulsion_exact(X, 2.5, 1.5), rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(A, O.attraction(X, rp, col), rtol=1e-12, atol=1e-14)


def test_masked_forces_are_minus_gradient():
    X, rp, col = _case(30, 60, 7)
    fo = O.Focus((4,), 4.0, 2.0, 3.0)
    lab = O.focus_region(30, rp, col, fo.focal)
    p = O.Params(gamma=2.0, rho=1.3)
    R, A = O.forces_masked(X, rp, col, lab, fo, p)
    D = R + A
    h = 1e-6
    G = np.zeros_like(X)
    for i in range(30):
        for d in range(2):
            Xp, Xm = X.copy(), X.copy()
            Xp[i, d] += h
            Xm[i, d] -= h
            G[i, d] = (O.energy_masked(Xp, rp, col, lab, fo, p) - O.energy_masked(Xm, rp, col, lab, fo, p)) / (2 * h)
    assert O.rel_l2(D, -G) < 1e-6


def test_masked_ibfft_correction_rule():
    """The FFT-path rule (R23) is exact when the FFT sum is exact: with S_all replaced by
    the exact sum it reproduces the definition, and on C2 (k = 3) its error against the
    exact masked forces stays at the unmasked ibFFT error level."""
    w = make_config("C2")
    rp, col = O.csr_build(w.n, w.u, w.v)
    X = w.xy.astype(np.float64)
    fo = O.Focus((100, 600), 4.0, 2.0, 2.0)
    lab = O.focus_region(w.n, rp, col, fo.focal)
    Rex = O.repulsion_masked_exact(X, lab, fo)
    Rib = O.repulsion_masked_ibfft(X, lab, fo, 3)
    e_mask = O.rel_l2(Rib, Rex)
    e_plain = O.rel_l2(O.repulsion_ibfft(X, 3), O.repulsion_exact(X))
    assert e_mask < 2.0 * e_plain + 1e-6, (e_mask, e_plain)
    # identity mask: the correction vanishes
    fo1 = O.Focus((100,), 1.0, 1.0, 1.0)
    lab1 = O.focus_region(w.n, rp, col, fo1.focal)
    np.testing.assert_allclose(O.repulsion_masked_ibfft(X, lab1, fo1, 3), O.repulsion_ibfft(X, 3),
                               rtol=1e-12, atol=1e-12)


def test_errors():
    X, rp, col = _case()
    with pytest.raises(ValueError):
        O.local_refine(X, rp, col, O.Focus(()), T=1)
    with pytest.raises(ValueError):
        O.local_refine(X, rp, col, O.Focus((1,), 0.5, 1, 1), T=1)


def test_identity_boosts_equal_run_continuation():
    """boosts (1, 1, 1) -> plain run continuation."""
    X, rp, col = _case(40, 80, 9)
    Xa = O.local_refine(X, rp, col, O.Focus((5,), 1, 1, 1), T=20)
    Xb = O.run(X, rp, col, O.Params(), T=20)
    np.testing.assert_allclose(Xa, Xb, rtol=1e-12, atol=1e-12)


def test_star_center_pulls_leaves():
    """star graph, centre focal, lambda_a = 4: the mean centre-leaf distance falls
    below that of the unrefined continuation."""
    n = 31
    rp, col = O.csr_build(n, [0] * (n - 1), list(range(1, n)))
    X0 = O.run(uniform_disc(n, 4.0, 21).astype(np.float64), rp, col, O.Params(), T=300)
    Xr = O.local_refine(X0, rp, col, O.Focus((0,), 4.0, 1.0, 1.0), T=100)
    Xc = O.run(X0, rp, col, O.Params(), T=100)
    dr = np.linalg.norm(Xr[1:] - Xr[0], axis=1).mean()
    dc = np.linalg.norm(Xc[1:] - Xc[0], axis=1).mean()
    assert dr < 0.8 * dc


def test_two_cluster_fisheye():
    """two focal nodes in different clusters, boosts (4, 2, 2): the region's mean
    pairwise distance falls, and the other nodes' mean pairwise distance relative to the
    bounding-box diagonal falls (compression), both against the unrefined continuation."""
    u, v, lab_c = two_cluster_graph(100, 0.1, 0.002, 12)
    n = 200
    rp, col = O.csr_build(n, u, v)
    X0 = O.run(uniform_disc(n, 8.0, 13).astype(np.float64), rp, col, O.Params(), T=300)
    fo = O.Focus((5, 150), 4.0, 2.0, 2.0)
    Xr = O.local_refine(X0, rp, col, fo, T=100)
    Xc = O.run(X0, rp, col, O.Params(), T=100)
    lab = O.focus_region(n, rp, col, fo.focal)

    def stats(X):
        D = np.linalg.norm(X[:, None] - X[None], axis=2)
        reg = np.nonzero(lab)[0]
        oth = np.nonzero(lab == 0)[0]
        diag = np.linalg.norm(X.max(0) - X.min(0))
        dreg = D[np.ix_(reg, reg)][np.triu_indices(reg.size, 1)].mean()
        doth = D[np.ix_(oth, oth)][np.triu_indices(oth.size, 1)].mean() / diag
        return dreg, doth

    (rr, ro), (cr, co) = stats(Xr), stats(Xc)
    assert rr < cr and ro < co, (rr, cr, ro, co)
