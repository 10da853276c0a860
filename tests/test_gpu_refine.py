"""GPU parity of global refinement (NEXT-1; tfdp_set_params / tfdp_global_refine)
through the C ABI against the oracle's global_refine on the same seeded inputs.
Bars as for the base path: exact rel-L2 <= 1e-4 per force field, ibFFT <= 1e-3 vs the
oracle's ibFFT at the same geometry, short runs by displacement parity."""
import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config, path_graph, two_cluster_graph, uniform_disc

pytestmark = pytest.mark.gpu


def _case(name):
    w = make_config(name)
    rp, col = O.csr_build(w.n, w.u, w.v)
    return w, rp, col


@pytest.mark.parametrize("gamma,rho", [(4.0, 1.0), (8.0, 4.0), (2.5, 4.0), (2.0, 0.25)])
def test_set_params_forces_exact(gamma, rho):
    """Forces after tfdp_set_params equal the oracle's with the new weights (C2)."""
    w, rp, col = _case("C2")
    X = w.xy.astype(np.float64)
    with P.Layout(w.n, rp, col, w.xy) as L:
        L.forces()
        L.set_params(P.Params(gamma=gamma, rho=rho, alpha=0.05, beta=4.0))
        R, A = L.forces()
    Re, Ae = O.forces_exact(X, rp, col, O.Params(alpha=0.05, beta=4.0, gamma=gamma, rho=rho))
    assert O.rel_l2(R, Re) <= 1e-4 and O.rel_l2(A, Ae) <= 1e-4


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("gamma,rho", [(4.0, 4.0), (2.5, 1.0)])
def test_set_params_forces_ibfft(k, gamma, rho):
    """ibFFT after set_params (gamma enters the kernel spectrum, rho the assembly) and a
    k change (re-plan) vs the oracle's ibFFT at the same geometry."""
    w, rp, col = _case("C2")
    X = w.xy.astype(np.float64)
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=1)) as L:
        L.forces()
        L.set_params(P.Params(solver="ibfft", k=k, gamma=gamma, rho=rho))
        R, _ = L.forces()
        geo = L.fft_geometry()
    assert geo["k"] == k
    Ro = O.repulsion_ibfft(X, k, gamma, rho)
    assert O.rel_l2(R, Ro) <= 1e-3, O.rel_l2(R, Ro)


def test_global_refine_matches_oracle_exact():
    """C1: base run of 40 iterations, then a rho = 4 / gamma = 4 refinement of T = 6."""
    w, rp, col = _case("C1")
    with P.Layout(w.n, rp, col, w.xy, P.Params(iterations=40)) as L:
        L.step(40)
        Xb = L.layout()
        L.global_refine(gamma=4.0, rho=4.0, iterations=6)
        assert L.iteration == 6
        Xr = L.layout()
    Xo = O.global_refine(Xb.astype(np.float64), rp, col, O.Params(), gamma=4.0, rho=4.0, T=6)
    assert O.rel_l2(Xr - Xb, Xo - Xb) < 1e-4


def test_global_refine_ibfft_short():
    """C2 ibFFT refinement (k = 3 throughout, T < 20) vs the oracle over 4 iterations."""
    w, rp, col = _case("C2")
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0)) as L:
        L.global_refine(rho=4.0, iterations=4)
        Xr = L.layout()
    Xo = O.global_refine(w.xy.astype(np.float64), rp, col, O.Params(), rho=4.0, T=4,
                         solver="ibfft", k=0)
    assert O.rel_l2(Xr - w.xy, Xo - w.xy) < 1e-3


def test_refinement_effects_on_device():
    """The paired statistics of the oracle pins, measured on the GPU path."""
    u, v = path_graph(20)
    rp, col = O.csr_build(20, u, v)
    with P.Layout(20, rp, col, uniform_disc(20, 5.0, 11)) as L:
        L.step(300)
        Xb = L.layout()
        L.global_refine(rho=4.0, iterations=300)
        Xr = L.layout()
    lb = np.linalg.norm(Xb[u] - Xb[v], axis=1)
    lr = np.linalg.norm(Xr[u] - Xr[v], axis=1)
    assert lr.var() < 0.5 * lb.var()

    u, v, lab = two_cluster_graph(100, 0.1, 0.002, 12)
    n = 200
    rp, col = O.csr_build(n, u, v)
    with P.Layout(n, rp, col, uniform_disc(n, 8.0, 13)) as L:
        L.step(300)
        Xb = L.layout().astype(np.float64)
        L.global_refine(gamma=4.0, iterations=300)
        Xr = L.layout().astype(np.float64)

    def ratio(X):
        D = np.linalg.norm(X[:, None] - X[None], axis=2)
        same = lab[:, None] == lab[None]
        off = ~np.eye(n, dtype=bool)
        return D[same & off].mean() / D[~same].mean()

    assert ratio(Xr) < 0.9 * ratio(Xb)


def test_refine_errors_keep_context_usable():
    w, rp, col = _case("C1")
    with P.Layout(w.n, rp, col, w.xy) as L:
        for g in (1.0, 0.5, float("nan")):
            with pytest.raises(P.TfdpError) as e:
                L.global_refine(gamma=g, iterations=1)
            assert e.value.status == 1
        with pytest.raises(P.TfdpError) as e:
            L.global_refine(rho=-1.0, iterations=1)
        assert e.value.status == 1
        with pytest.raises(P.TfdpError) as e:
            L.set_params(P.Params(solver="ibfft"))  # solver fixed at init
        assert e.value.status == 1
        L.global_refine(gamma=3.0, iterations=2)  # still usable
        assert L.iteration == 2
        assert not (L.warnings & 2)
        L.set_params(P.Params(gamma=1.0))  # allowed outside refinement: warning only
        assert L.warnings & 2
