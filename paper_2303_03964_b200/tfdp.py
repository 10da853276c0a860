"""Python binding of libtfdp (include/tfdp.h) — argument marshalling only.

    from paper_2303_03964_b200 import Params, Layout, csr_build
    row_ptr, col = csr_build(n, u, v)
    L = Layout(n, row_ptr, col, xy0, Params(solver="ibfft"))
    L.step(300); xy = L.layout()

Arrays may be NumPy (host) or torch tensors (host or CUDA); torch supplies device memory
and the stream (torch.cuda.current_stream()) — the computation is libtfdp's kernels.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import _lib as _L
from ._lib import check, lib


@dataclasses.dataclass
class Params:
    """Mirror of tfdp_params (defaults: P:372 alpha=0.1 beta=8 gamma=2; S:340 eta0=0.1;
    T=300 (R3); N_int >= 50)."""
    alpha: float = 0.1
    beta: float = 8.0
    gamma: float = 2.0
    rho: float = 1.0
    solver: str = "exact"  # "exact" | "ibfft"
    k: int = 0  # 0 = dynamic 90/5/5
    n_int_min: int = 50
    n_int_fixed: int = 0
    fft_size: int = 0
    step0: float = 0.1
    iterations: int = 300
    t0: int = 0
    cooling: str = "linear"  # "linear" (R2) | "constant" (R2')
    dist_mode: str = "slab"  # "slab" | "spread_all" | "grid_allreduce" (ibFFT, p > 1)
    node_order: str = "auto"  # "auto" (internal Morton renumbering, ibFFT) | "keep"
    interval_rule: str = "unit"  # "unit" (R5', unit-width intervals) | "span" (R5)
    dim: int = 2

    def to_c(self) -> _L.tfdp_params:
        p = _L.tfdp_params()
        check(lib().tfdp_params_default(C.byref(p)))
        p.dim = self.dim
        p.alpha, p.beta, p.gamma, p.rho = self.alpha, self.beta, self.gamma, self.rho
        p.solver = {"exact": _L.EXACT, "ibfft": _L.IBFFT}[self.solver]
        p.k, p.n_int_min, p.n_int_fixed, p.fft_size = self.k, self.n_int_min, self.n_int_fixed, self.fft_size
        p.step0, p.iterations, p.t0 = self.step0, self.iterations, self.t0
        p.cooling = {"linear": _L.COOL_LINEAR, "constant": _L.COOL_CONSTANT}[self.cooling]
        p.dist_mode = {"spread_all": _L.DIST_SPREAD_ALL, "grid_allreduce": _L.DIST_GRID_ALLREDUCE,
                       "slab": _L.DIST_SLAB}[self.dist_mode]
        p.node_order = {"auto": 0, "keep": 1}[self.node_order]
        p.interval_rule = {"unit": 0, "span": 1}[self.interval_rule]
        return p


def _ptr(a):
    """(pointer, keepalive) of a NumPy array or torch tensor (contiguous)."""
    if a is None:
        return None, None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            a = np.ascontiguousarray(a)
        return a.ctypes.data, a
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr(), a
    raise TypeError(f"unsupported array type {type(a)}")


def csr_build(n: int, u, v):
    """Symmetric CSR via the library (tfdp_csr_build)."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    m = int(u.shape[0])
    row_ptr = np.empty(n + 1, dtype=np.int64)
    col = np.empty(max(2 * m, 1), dtype=np.int32)
    nnz = C.c_int64(0)
    check(lib().tfdp_csr_build(n, m, u.ctypes.data, v.ctypes.data, row_ptr.ctypes.data,
                               col.ctypes.data, C.byref(nnz)))
    return row_ptr, col[: nnz.value].copy()


def shard_range(n: int, world: int, rank: int):
    lo, hi = C.c_int64(), C.c_int64()
    check(lib().tfdp_shard_range(n, world, rank, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def slab_plan(rows: int, fft_size: int, world: int):
    """tfdp_slab_plan: (row0, q0) int lists of world + 1 entries (host only)."""
    r0 = (C.c_int32 * (world + 1))()
    q0 = (C.c_int32 * (world + 1))()
    check(lib().tfdp_slab_plan(int(rows), int(fft_size), int(world), C.cast(r0, C.c_void_p),
                               C.cast(q0, C.c_void_p)))
    return list(r0), list(q0)


def group_step(layouts, n_iters: int = 1):
    """tfdp_group_step over the virtual ranks 0..p-1 (Layout objects in rank order)."""
    arr = (C.c_void_p * len(layouts))(*[L._ctx.value for L in layouts])
    check(lib().tfdp_group_step(C.cast(arr, C.c_void_p), len(layouts), int(n_iters)), layouts[0]._ctx)


def group_forces(layouts):
    """tfdp_group_forces: [(R, A)] per virtual rank (NumPy float32 (hi - lo, 2))."""
    outs = [(np.empty((L.hi - L.lo, 2), np.float32), np.empty((L.hi - L.lo, 2), np.float32)) for L in layouts]
    rp = (C.c_void_p * len(layouts))(*[o[0].ctypes.data for o in outs])
    ap = (C.c_void_p * len(layouts))(*[o[1].ctypes.data for o in outs])
    arr = (C.c_void_p * len(layouts))(*[L._ctx.value for L in layouts])
    check(lib().tfdp_group_forces(C.cast(arr, C.c_void_p), len(layouts), C.cast(rp, C.c_void_p),
                                  C.cast(ap, C.c_void_p)), layouts[0]._ctx)
    return outs


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    check(lib().tfdp_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Dist:
    """rank/world/device + the 128-byte NCCL unique id (see dist.bootstrap)."""

    def __init__(self, rank: int, world: int, device: int, uid: bytes | None):
        self._uid = (C.c_ubyte * 128).from_buffer_copy(uid) if uid else None
        self.c = _L.tfdp_dist(rank, world, device, C.cast(self._uid, C.c_void_p) if uid else None)
        self.rank, self.world, self.device = rank, world, device


class Layout:
    """One t-FDP layout context (tfdp_init ... tfdp_destroy)."""

    def __init__(self, n: int, row_ptr, col, xy0, params: Params | None = None,
                 dist: Dist | None = None, stream: int | None = None):
        self.n = int(n)
        self.params = params or Params()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cl = np.ascontiguousarray(col, dtype=np.int32)
        if rp.shape[0] != self.n + 1:
            raise ValueError("row_ptr must have n+1 entries")
        xp, keep = _ptr(xy0 if not isinstance(xy0, np.ndarray) else np.ascontiguousarray(xy0, np.float32))
        self._ctx = C.c_void_p()
        pc = self.params.to_c()
        st = lib().tfdp_init(C.byref(self._ctx), self.n, rp.ctypes.data,
                             cl.ctypes.data if cl.size else None, xp, C.byref(pc),
                             C.byref(dist.c) if dist else None, stream)
        if st != _L.TFDP_OK:
            m = lib().tfdp_last_error(None)
            raise _L.TfdpError(st, m.decode() if m else "")
        del keep
        lo, hi = C.c_int64(), C.c_int64()
        check(lib().tfdp_shard(self._ctx, C.byref(lo), C.byref(hi)), self._ctx)
        self.lo, self.hi = lo.value, hi.value

    # -- lifecycle --------------------------------------------------------------------
    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            lib().tfdp_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- calls --------------------------------------------------------------------------
    def step(self, n_iters: int = 1):
        check(lib().tfdp_step(self._ctx, int(n_iters)), self._ctx)

    def forces(self, rep=None, att=None):
        """(R, A) for this rank's shard.  With no arguments returns NumPy float32 (hi-lo, 2)."""
        own = rep is None and att is None
        if own:
            m = self.hi - self.lo
            rep = np.empty((m, 2), np.float32)
            att = np.empty((m, 2), np.float32)
        rp, k1 = _ptr(rep)
        ap, k2 = _ptr(att)
        check(lib().tfdp_forces(self._ctx, rp, ap), self._ctx)
        return rep, att

    def layout(self, out=None):
        if out is None:
            out = np.empty((self.n, 2), np.float32)
        p, k = _ptr(out)
        check(lib().tfdp_layout(self._ctx, p), self._ctx)
        return out

    def set_layout(self, xy):
        if isinstance(xy, np.ndarray):
            xy = np.ascontiguousarray(xy, np.float32)
        p, k = _ptr(xy)
        check(lib().tfdp_set_layout(self._ctx, p), self._ctx)

    def set_iteration(self, t: int):
        check(lib().tfdp_set_iteration(self._ctx, int(t)), self._ctx)

    def set_params(self, params: Params):
        """tfdp_set_params: new weights / schedule for the live layout (solver fixed)."""
        pc = params.to_c()
        check(lib().tfdp_set_params(self._ctx, C.byref(pc)), self._ctx)
        self.params = params

    def global_refine(self, gamma: float | None = None, rho: float | None = None,
                      iterations: int | None = None):
        """Global refinement (tfdp_global_refine): re-run the layout loop from the
        current layout with repulsion exponent gamma and/or scale rho (None = unchanged)."""
        g = self.params.gamma if gamma is None else float(gamma)
        r = self.params.rho if rho is None else float(rho)
        T = self.params.iterations if iterations is None else int(iterations)
        check(lib().tfdp_global_refine(self._ctx, g, r, T), self._ctx)
        self.params = dataclasses.replace(self.params, gamma=g, rho=r, iterations=T, t0=0)

    def pivot_mds(self, n_pivots: int = 50, seed: int = 0):
        """tfdp_pivot_mds: replace the layout by the PivotMDS initialisation.
        Returns the pivots (caller ids)."""
        p = min(int(n_pivots), self.n)
        piv = np.empty(max(p, 1), np.int32)
        check(lib().tfdp_pivot_mds(self._ctx, int(n_pivots), int(seed) & ((1 << 64) - 1),
                                   piv.ctypes.data), self._ctx)
        return piv[:p]

    def set_focus(self, focal, la: float = 1.0, lf: float = 1.0, ls: float = 1.0):
        """tfdp_set_focus: local-refinement mask on F u N(F); focal=[] clears it."""
        f = np.ascontiguousarray(np.asarray(focal, dtype=np.int32).ravel())
        check(lib().tfdp_set_focus(self._ctx, f.ctypes.data if f.size else None, int(f.size),
                                   float(la), float(lf), float(ls)), self._ctx)

    def local_refine(self, focal, la: float = 1.0, lf: float = 1.0, ls: float = 1.0,
                     iterations: int | None = None):
        """Local (fisheye) refinement (tfdp_local_refine)."""
        f = np.ascontiguousarray(np.asarray(focal, dtype=np.int32).ravel())
        T = self.params.iterations if iterations is None else int(iterations)
        check(lib().tfdp_local_refine(self._ctx, f.ctypes.data if f.size else None, int(f.size),
                                      float(la), float(lf), float(ls), T), self._ctx)
        self.params = dataclasses.replace(self.params, iterations=T, t0=0)

    def np1(self, hits=None):
        """NP1 of the current layout on the device (tfdp_np1).  Returns the float;
        with hits (int32 array / tensor of hi - lo entries) also fills the per-node counts."""
        v = C.c_double(0.0)
        hp, keep = _ptr(hits)
        check(lib().tfdp_np1(self._ctx, C.byref(v), hp), self._ctx)
        return v.value

    @property
    def iteration(self) -> int:
        return int(lib().tfdp_iteration(self._ctx))

    @property
    def warnings(self) -> int:
        return int(lib().tfdp_warnings(self._ctx))

    def fft_geometry(self):
        box = (C.c_float * 4)()
        ni, k, P = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib().tfdp_fft_geometry(self._ctx, C.cast(box, C.c_void_p), C.byref(ni), C.byref(k),
                                      C.byref(P)), self._ctx)
        return dict(lo=(box[0], box[1]), L=box[2], w=box[3], n_int=ni.value, k=k.value, P=P.value)

    def fft_plan(self, k: int):
        P, cap = C.c_int32(), C.c_int32()
        check(lib().tfdp_fft_plan(self._ctx, int(k), C.byref(P), C.byref(cap)), self._ctx)
        return P.value, cap.value

    def profile(self, enable: bool = True):
        check(lib().tfdp_profile(self._ctx, int(enable)), self._ctx)

    def kernel_kinds(self) -> list:
        """Names of the kernel kinds, in the bit order of profile_only()."""
        cap = 32
        names = (C.c_char_p * cap)()
        k = lib().tfdp_profile_read(self._ctx, names, None, None, cap)
        return [names[i].decode() for i in range(k)]

    def profile_only(self, kinds):
        """Time only the named kernel kinds (CUDA events around those launches alone)."""
        order = self.kernel_kinds()
        mask = 0
        for name in kinds:
            mask |= 1 << order.index(name)
        check(lib().tfdp_profile_mask(self._ctx, mask), self._ctx)

    def kinds_mask(self, kinds) -> int:
        order = self.kernel_kinds()
        mask = 0
        for name in kinds:
            mask |= 1 << order.index(name)
        return mask

    def profile_select(self, mask: int):
        """tfdp_profile_select: switch the timed kinds without reset or sync."""
        check(lib().tfdp_profile_select(self._ctx, int(mask)), self._ctx)

    def profile_read(self) -> dict:
        cap = 32
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        cnt = (C.c_int64 * cap)()
        k = lib().tfdp_profile_read(self._ctx, names, ms, cnt, cap)
        return {names[i].decode(): (ms[i], cnt[i]) for i in range(k) if cnt[i] > 0}

    @property
    def launch_count(self) -> int:
        return int(lib().tfdp_launch_count(self._ctx))
