"""Host-side checks of libtfdp.so that need no GPU: the library loads and exports every
symbol include/tfdp.h declares, the host CSR builder and shard rule are bit-exact with
the oracle, argument errors are reported (no compute calls)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
import paper_2303_03964_b200 as P
from paper_2303_03964_b200 import _lib
from synth import make_config, random_graph


def test_library_exports_every_declared_symbol():
    L = P.lib()
    syms = P.declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s


def test_params_default_matches_paper():
    p = _lib.tfdp_params()
    assert P.lib().tfdp_params_default(C.byref(p)) == 0
    assert (p.dim, p.alpha, p.beta, p.gamma, p.rho) == (2, 0.1, 8.0, 2.0, 1.0)
    assert (p.n_int_min, p.step0, p.iterations, p.k) == (50, 0.1, 300, 0)  # P:540, R3
    assert p.interval_rule == 0  # reading R5' (unit-width intervals)
    assert P.lib().tfdp_params_default(None) == 1


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_csr_build_bit_exact(seed):
    n = [1, 50, 3000][seed]
    u, v = random_graph(n, 5 * n, seed)
    rp, col = P.csr_build(n, u, v)
    rp2, col2 = O.csr_build(n, u, v)
    np.testing.assert_array_equal(rp, rp2)
    np.testing.assert_array_equal(col, col2)


def test_csr_build_configs_bit_exact():
    for name in ("C1", "C2", "C2rgg", "C3"):
        w = make_config(name)
        rp, col = P.csr_build(w.n, w.u, w.v)
        rp2, col2 = O.csr_build(w.n, w.u, w.v)
        assert np.array_equal(rp, rp2) and np.array_equal(col, col2), name


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C4", "C5"])
def test_csr_build_bench_configs_bit_exact(name):
    """The bench's graphs (C4: 8.0M, C5: 69.3M directed entries) build bit-identically."""
    w = make_config(name)
    rp, col = P.csr_build(w.n, w.u, w.v)
    rp2, col2 = O.csr_build(w.n, w.u, w.v)
    assert np.array_equal(rp, rp2) and np.array_equal(col, col2), name
    del w, rp, col, rp2, col2


def test_csr_build_errors():
    with pytest.raises(P.TfdpError):
        P.csr_build(3, np.array([0, 5]), np.array([1, 1]))
    rp, col = P.csr_build(2, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert rp.tolist() == [0, 0, 0] and col.size == 0


def test_shard_range_bit_exact():
    for n in (1, 7, 1000, 4_000_000, 2**31 - 1):
        for p in (1, 2, 3, 8):
            for r in range(p):
                assert P.shard_range(n, p, r) == O.shard_range(n, p, r)
    with pytest.raises(P.TfdpError):
        P.shard_range(10, 2, 2)


def test_init_argument_errors_without_gpu():
    """Validation happens before any device work: bad CSR / params are TFDP_ERR_ARG."""
    xy = np.zeros((3, 2), np.float32)
    rp, col = O.csr_build(3, [0], [1])
    bad_col = col.copy()
    bad_col[0] = 0  # self-loop in row 0
    with pytest.raises(P.TfdpError) as e:
        P.Layout(3, rp, bad_col, xy)
    assert e.value.status == 1
    with pytest.raises(P.TfdpError) as e:
        P.Layout(3, rp, col, xy, P.Params(iterations=0))
    assert e.value.status == 1
    with pytest.raises(P.TfdpError) as e:
        P.Layout(3, rp, col, xy, P.Params(dim=3))
    assert e.value.status == 7
    asym_rp = np.array([0, 1, 1, 1], np.int64)  # 0 -> 1 without 1 -> 0
    with pytest.raises(P.TfdpError) as e:
        P.Layout(3, asym_rp, np.array([1], np.int32), xy)
    assert e.value.status == 1


def test_status_strings():
    L = P.lib()
    assert L.tfdp_status_string(4) == b"TFDP_ERR_DIVERGED"
    assert L.tfdp_last_error(None) is not None


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("rows,Pf", [(1001, 2048), (2002, 4096), (3003, 6144), (150, 512)])
def test_slab_plan(world, rows, Pf):
    """Slab plan of the multi-GPU FFT path (host only): grid-row slabs of whole 24-row units
    (CA row tiles of 8 and whole intervals at k = 1, 2, 3) covering [0, rows rounded up to 24),
    even-starting half-spectrum column chunks covering [0, P/2 + 1), balanced to one unit."""
    row0, q0 = P.slab_plan(rows, Pf, world)
    H = Pf // 2 + 1
    assert row0[0] == 0 and row0[-1] == (rows + 23) // 24 * 24 and q0[0] == 0 and q0[-1] == H
    d_rows = np.diff(row0)
    d_cols = np.diff(q0)
    assert (d_rows >= 0).all() and (np.asarray(row0) % 24 == 0).all()
    assert (d_cols >= 0).all() and all(q % 2 == 0 for q in q0[:-1])
    assert d_rows.max() - d_rows.min() <= 24 and d_cols.max() - d_cols.min() <= 3
    with pytest.raises(P.TfdpError):
        P.slab_plan(rows, Pf, 0)


def test_c_example_builds_and_links():
    """examples/*.c compile against include/tfdp.h alone and link libtfdp.so (no GPU needed)."""
    from paper_2303_03964_b200 import build as B
    exes = B.build_examples()
    assert exes and all(os.path.exists(e) for e in exes)


def test_nccl_loopback_builds_and_exports():
    """The tests' in-process NCCL stand-in (tests/nccl_loopback) builds with g++ and exports
    every NCCL entry point libtfdp.so resolves (csrc/nccl_shim.cpp)."""
    import ctypes
    from paper_2303_03964_b200 import build as B
    path = B.build_nccl_loopback()
    lb = ctypes.CDLL(path)
    for s in ("ncclGetUniqueId", "ncclCommInitRank", "ncclCommDestroy", "ncclGroupStart",
              "ncclGroupEnd", "ncclBroadcast", "ncclAllReduce", "ncclSend", "ncclRecv",
              "ncclGetErrorString"):
        assert hasattr(lb, s), s
