"""ORACLE (test infrastructure only) — plain fp64 NumPy t-FDP force step.

Written from the paper, arXiv 2303.03964 (/root/reference/PAPER.md = P:<line>), with
SPEC.md (S:<line>) for interfaces and worked examples, and the readings R1..R19 of
DESIGN.md where the paper is silent/ambiguous.  Nothing here is blocked, fused or
reordered beyond what the definitions state.  Imported only by tests/, smoke() and
bench.py's CPU-baseline legs; never by the product path.

Notation:  r_ij = x_i - x_j,  s_ij = 1 + |r_ij|^2,
    R_i = rho * sum_{j != i} r_ij s_ij^-gamma                      (P:463-465 Eq. repfK)
    A_i = -alpha * sum_{j in adj(i)} (1 + beta / s_ij) r_ij         (P:286-288 Eq. newforce, x alpha P:299-303)
    D_i = R_i + A_i          (physical displacement, reading R1)
    x_i <- x_i + eta_t D_i,  eta_t = eta0 (1 - t/T)                 (reading R2)
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Params", "csr_build", "shard_range", "t_force", "repulsion_exact",
    "repulsion_exact_loops", "attraction", "attraction_loops", "forces_exact",
    "energy", "eta", "k_schedule", "Box", "box_rule", "interval_coords",
    "lagrange_weights", "spread", "kernel_tdist", "convolve_direct", "convolve_fft",
    "gather", "repulsion_ibfft", "forces", "step", "run", "np1", "rel_l2",
    "equilibrium_distance", "global_refine", "np1_hits", "np1_from_hits",
    "Focus", "focus_region", "repulsion_masked_exact", "repulsion_masked_loops",
    "attraction_masked", "repulsion_masked_ibfft", "forces_masked", "energy_masked",
    "local_refine", "splitmix64", "bfs_hops", "pmds_pivots", "pivot_mds",
]


@dataclasses.dataclass
class Params:
    """Force weights; defaults alpha=0.1, beta=8, gamma=2, rho=1."""
    alpha: float = 0.1
    beta: float = 8.0
    gamma: float = 2.0
    rho: float = 1.0


# ---------------------------------------------------------------------------------------
# Graph substrate: CSR + shard ranges (S:22-27 invariants; SURVEY §8(b) sharding rule)
# ---------------------------------------------------------------------------------------
def csr_build(n: int, u, v):
    """Undirected simple graph -> symmetric CSR: self-loops dropped, duplicate
    unordered pairs collapsed, each row's columns sorted ascending.
    Returns (row_ptr int64[n+1], col int32[2m])."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    if u.shape != v.shape:
        raise ValueError("u and v must have equal length")
    if u.size and (u.min() < 0 or v.min() < 0 or u.max() >= n or v.max() >= n):
        raise ValueError("edge endpoint out of range")
    keep = u != v
    a = np.minimum(u[keep], v[keep])
    b = np.maximum(u[keep], v[keep])
    pairs = np.unique(a * n + b)  # each unordered pair once
    a, b = pairs // n, pairs % n
    src = np.concatenate([a, b])
    dst = np.concatenate([b, a])
    order = np.lexsort((dst, src))  # by row, then column
    src, dst = src[order], dst[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, src + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, dst.astype(np.int32)


def shard_range(n: int, world: int, rank: int):
    """Rank r of p owns targets [floor(r n / p), floor((r+1) n / p))."""
    return (rank * n) // world, ((rank + 1) * n) // world


# ---------------------------------------------------------------------------------------
# Force model
# ---------------------------------------------------------------------------------------
def t_force(d, phi):
    """t-force f(d) = d / (1 + d^2)^phi (P:268 Eq. forcefunction)."""
    d = np.asarray(d, dtype=np.float64)
    return d / (1.0 + d * d) ** phi


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


def repulsion_exact(X, gamma=2.0, rho=1.0, targets=None, block_elems=1 << 22):
    """Exact O(n^2) repulsion (P:463-465 Eq. repfK):
    R_i = rho * sum_j (x_i - x_j) (1 + |x_i - x_j|^2)^-gamma.  The j = i term is 0
    (r_ii = 0), so summing over all j equals the paper's j != i sum.
    `targets` (optional int array) restricts the output rows; sources are always all n."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    tgt = np.arange(n) if targets is None else np.asarray(targets, dtype=np.int64)
    out = np.zeros((tgt.size, 2))
    bs = max(1, block_elems // max(n, 1))
    for s in range(0, tgt.size, bs):
        ti = tgt[s:s + bs]
        r = X[ti, None, :] - X[None, :, :]  # (B, n, 2)
        sij = 1.0 + (r * r).sum(-1)
        out[s:s + bs] = rho * (r * (sij ** (-gamma))[..., None]).sum(1)
    return out


def repulsion_exact_loops(X, gamma=2.0, rho=1.0):
    """Literal double loop of Eq. repfK with the j != i restriction (brute force, n <= 64)."""
    X = [tuple(map(float, p)) for p in np.asarray(X, dtype=np.float64)]
    n = len(X)
    out = np.zeros((n, 2))
    for i in range(n):
        fx = fy = 0.0
        for j in range(n):
            if j == i:
                continue
            dx, dy = X[i][0] - X[j][0], X[i][1] - X[j][1]
            d = math.sqrt(dx * dx + dy * dy)
            if d == 0.0:
                continue  # vector form r s^-gamma is 0 at d = 0 (reading R12)
            mag = d / (1.0 + d * d) ** gamma  # t-force magnitude
            fx += mag * dx / d
            fy += mag * dy / d
        out[i] = (rho * fx, rho * fy)
    return out


def attraction(X, row_ptr, col, alpha=0.1, beta=8.0, targets=None):
    """A_i = -alpha * sum_{j in adj(i)} (1 + beta/(1 + d^2)) (x_i - x_j)
    (P:286-288 Eq. newforce with phi=1 t-force term (reading R17), x alpha P:301-303)."""
    X = np.asarray(X, dtype=np.float64)
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    n = X.shape[0]
    tgt = np.arange(n) if targets is None else np.asarray(targets, dtype=np.int64)
    deg = row_ptr[1:] - row_ptr[:-1]
    rows = np.repeat(np.arange(n), deg)
    r = X[rows] - X[col]
    s = 1.0 + (r * r).sum(1)
    contrib = -alpha * (1.0 + beta / s)[:, None] * r
    out = np.zeros((n, 2))
    np.add.at(out, rows, contrib)
    return out[tgt]


def attraction_loops(X, row_ptr, col, alpha=0.1, beta=8.0):
    """Literal per-edge loop of Eq. newforce (brute force for small graphs)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    out = np.zeros((n, 2))
    for i in range(n):
        for e in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            j = int(col[e])
            dx, dy = X[i, 0] - X[j, 0], X[i, 1] - X[j, 1]
            d = math.sqrt(dx * dx + dy * dy)
            if d == 0.0:
                continue
            mag = d + beta * d / (1.0 + d * d)
            out[i, 0] -= alpha * mag * dx / d  # pulls x_i toward x_j (reading R1)
            out[i, 1] -= alpha * mag * dy / d
    return out


def forces_exact(X, row_ptr, col, p: Params = Params(), targets=None):
    """(R, A) for the exact path (SURVEY §8(c) definition)."""
    R = repulsion_exact(X, p.gamma, p.rho, targets)
    A = attraction(X, row_ptr, col, p.alpha, p.beta, targets)
    return R, A


def energy(X, row_ptr, col, p: Params = Params()):
    """E with D = -grad E (pin P9): rho sum_{i<j} s^(1-gamma)/(2(gamma-1))
    + alpha sum_edges (d^2/2 + (beta/2) ln s)  (potentials of S:214-219; gamma > 1)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    r = X[:, None, :] - X[None, :, :]
    s = 1.0 + (r * r).sum(-1)
    iu = np.triu_indices(n, 1)
    e_rep = p.rho * (s[iu] ** (1.0 - p.gamma)).sum() / (2.0 * (p.gamma - 1.0))
    deg = np.diff(row_ptr)
    rows = np.repeat(np.arange(n), deg)
    cols = np.asarray(col, dtype=np.int64)
    up = rows < cols  # each undirected edge once
    d2 = ((X[rows[up]] - X[cols[up]]) ** 2).sum(1)
    e_att = p.alpha * (0.5 * d2 + 0.5 * p.beta * np.log1p(d2)).sum()
    return e_rep + e_att


def equilibrium_distance(p: Params = Params()):
    """Two connected nodes: net force 0 where rho u^-gamma = alpha (1 + beta/u), u = 1 + d^2
    (P:345-355 crossover; closed form for gamma = 2, rho = 1: alpha u^2 + alpha beta u - 1 = 0)."""
    a, b = p.alpha, p.beta
    if p.gamma == 2.0 and p.rho == 1.0:
        u = (-a * b + math.sqrt(a * a * b * b + 4.0 * a)) / (2.0 * a)
        return math.sqrt(u - 1.0)
    lo, hi = 1e-9, 1e3  # bisection on net(d) = rep - att (repulsive for small d)
    f = lambda d: p.rho * (1 + d * d) ** (-p.gamma) - a * (1 + b / (1 + d * d))
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if f(mid) > 0 else (lo, mid)
    return 0.5 * (lo + hi)


# ---------------------------------------------------------------------------------------
# Schedules (reading R2/R4)
# ---------------------------------------------------------------------------------------
def eta(t: int, T: int, eta0: float = 0.1, cooling: str = "linear") -> float:
    """Step size.  The paper never states its integrator ("the resultant force will
    move the node until convergence").  Reading R2 (default): linear cooling
    eta_t = eta0 (1 - t/T).  Reading R2' ("constant"): eta_t = eta0, which is what
    the P:680 observation (NP1 recovers in the last 30 iterations) needs; see DESIGN.md."""
    if cooling == "linear":
        return eta0 * (1.0 - t / T)
    if cooling == "constant":
        return eta0
    raise ValueError(cooling)


def k_schedule(T: int) -> np.ndarray:
    """Dynamic k: k=1 for ceil(0.9T) iterations, k=2 for ceil(0.05T), k=3 for the
    rest; T < 20 -> k=3 throughout (reading R4)."""
    if T < 1:
        raise ValueError("T >= 1")
    if T < 20:
        return np.full(T, 3, dtype=np.int32)
    n1 = math.ceil(0.9 * T - 1e-9)
    n2 = math.ceil(0.05 * T - 1e-9)
    n1 = min(n1, T)
    n2 = min(n2, T - n1)
    return np.array([1] * n1 + [2] * n2 + [3] * (T - n1 - n2), dtype=np.int32)


# ---------------------------------------------------------------------------------------
# ibFFT — step by step
# ---------------------------------------------------------------------------------------
@dataclasses.dataclass
class Box:
    lo: np.ndarray  # float32[2]  lower-left corner of the bounding square (R6)
    L: np.float32  # span max(span_x, span_y) of the points (R6)
    n_int: int  # intervals per axis (R5)
    w: np.float32  # interval width: 1 (R5') or L / n_int (R5)
    center: np.ndarray  # float64[2] = lo + side/2, side = n_int w (R11)


def box_rule(X, n_int_min: int = 50, n_int_fixed: int = 0, rule: str = "unit") -> Box:
    """Bounding square + interval rule.  P:531 divides "[x_min,x_max] x [x_min,x_max]" into
    N_int x N_int intervals; P:540 N_int = max(50, [y_max - y_min]).  Readings: R6 square
    anchored at (min x, min y), L = max(span_x, span_y); R5 bracket = ceil.
    rule = "unit" (reading R5', the default): when the span sets the count (ceil L >=
    n_int_min) the N_int intervals have unit width, w = 1, and the square has side
    N_int >= L; otherwise (N_int = n_int_min, or n_int_fixed) the N_int intervals divide
    the span, w = L / N_int.  rule = "span" (reading R5): always w = L / N_int.
    R19: lo, L, w are computed in fp32 (the kernel's precision) because they decide the
    integer interval index; degenerate L = 0 -> unit square centred on the point."""
    if rule not in ("unit", "span"):
        raise ValueError("rule is 'unit' (R5') or 'span' (R5)")
    X32 = np.asarray(X, dtype=np.float32)
    mn = X32.min(0)
    mx = X32.max(0)
    span = (mx - mn).astype(np.float32)  # fp32 subtraction
    L = np.float32(max(span[0], span[1]))
    lo = mn.astype(np.float32)
    if L == np.float32(0.0):
        lo = (mn - np.float32(0.5)).astype(np.float32)
        L = np.float32(1.0)
    cl = int(math.ceil(float(L)))
    n_int = int(n_int_fixed) if n_int_fixed > 0 else max(int(n_int_min), cl)
    if rule == "unit" and n_int_fixed <= 0 and cl >= n_int_min:
        w = np.float32(1.0)  # R5': unit-width intervals, side N_int
        side = float(n_int)
    else:
        w = np.float32(L / np.float32(n_int))  # IEEE fp32 division
        side = float(L)
    center = lo.astype(np.float64) + 0.5 * side
    return Box(lo=lo, L=L, n_int=n_int, w=w, center=center)


def interval_coords(X, box: Box):
    """Interval index b = min(floor((x - lo)/w), N_int - 1) (top edge -> last interval, R7)
    and local coordinate u = (x - lo)/w - b in [0, 1].  (x - lo)/w is evaluated in fp32
    (R19) so the integer decision matches the device bit for bit; u is then exact."""
    X32 = np.asarray(X, dtype=np.float32)
    t32 = ((X32 - box.lo) / box.w).astype(np.float32)
    b = np.minimum(np.floor(t32).astype(np.int64), box.n_int - 1)
    b = np.maximum(b, 0)
    u = t32.astype(np.float64) - b
    return b, u


def lagrange_weights(u, k: int):
    """Lagrange basis on k equispaced nodes t_c = (c + 1/2)/k of the unit interval
    ("k x k equi-spaced nodes"; node placement reading R8):
    l_c(u) = prod_{c' != c} (u - t_c') / (t_c - t_c').  Returns array (..., k)."""
    u = np.asarray(u, dtype=np.float64)
    t = (np.arange(k) + 0.5) / k
    out = np.ones(u.shape + (k,))
    for c in range(k):
        for cp in range(k):
            if cp != c:
                out[..., c] *= (u - t[cp]) / (t[c] - t[cp])
    return out


def spread(X, box: Box, k: int):
    """Step 1 ("projecting all data points onto the grid by using Lagrange
    polynomials"): C_v[b_x k + a, b_y k + c] += l_a(u_x) l_c(u_y) v_i for v in
    {1, x~, y~} (x~ = x - center, R11).  Each node touches only its own interval's k x k
    nodes.  Returns C[3, M, M] indexed [channel, gx, gy], M = N_int k."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    M = box.n_int * k
    b, u = interval_coords(X, box)
    lx = lagrange_weights(u[:, 0], k)  # (n, k)
    ly = lagrange_weights(u[:, 1], k)
    xt = X - box.center
    vals = np.stack([np.ones(n), xt[:, 0], xt[:, 1]], 0)  # (3, n)
    C = np.zeros((3, M, M))
    for a in range(k):
        for c in range(k):
            gx = b[:, 0] * k + a
            gy = b[:, 1] * k + c
            wgt = lx[:, a] * ly[:, c]
            for ch in range(3):
                np.add.at(C[ch], (gx, gy), wgt * vals[ch])
    return C


def kernel_tdist(gamma: float):
    """K(x_i, x_j) = 1 / (1 + |x_i - x_j|^2)^gamma as a function of (dx, dy)."""
    return lambda dx, dy: (1.0 + dx * dx + dy * dy) ** (-gamma)


def convolve_direct(C, h: float, kernel):
    """Step 2 by definition ("computing the interaction of the grid nodes"):
    Phi_v[a, b] = sum_{a', b'} K(h (a - a'), h (b - b')) C_v[a', b']  (linear, R9).
    Dense M^2 x M^2 matrix — small M only."""
    M = C.shape[1]
    if M > 64:
        raise ValueError("direct convolution is for M <= 64")
    a = np.arange(M)
    gx, gy = np.meshgrid(a, a, indexing="ij")
    gx, gy = gx.ravel(), gy.ravel()
    Kmat = kernel(h * (gx[:, None] - gx[None, :]), h * (gy[:, None] - gy[None, :]))
    return np.stack([(Kmat @ C[ch].ravel()).reshape(M, M) for ch in range(C.shape[0])])


def convolve_fft(C, h: float, kernel, P: int | None = None):
    """Step 2 "accelerated by FFT": the same linear convolution via a
    zero-padded P x P circular convolution, P >= 2M - 1 (R9), numpy.fft in fp64."""
    M = C.shape[1]
    if P is None:
        P = 2 * M
    if P < 2 * M - 1:
        raise ValueError("P must be >= 2M-1 for a linear convolution")
    off = np.arange(-(M - 1), M)
    dx, dy = np.meshgrid(off, off, indexing="ij")
    Kp = np.zeros((P, P))
    Kp[dx % P, dy % P] = kernel(h * dx, h * dy)
    Khat = np.fft.rfft2(Kp)
    out = np.empty_like(C)
    for ch in range(C.shape[0]):
        Cp = np.zeros((P, P))
        Cp[:M, :M] = C[ch]
        out[ch] = np.fft.irfft2(np.fft.rfft2(Cp) * Khat, s=(P, P))[:M, :M]
    return out


def gather(Phi, X, box: Box, k: int):
    """Step 3 ("back-projecting the interaction of all grid nodes to the original
    points"): psi_v(x_i) = sum_{a,c} l_a(u_x) l_c(u_y) Phi_v[b_x k + a, b_y k + c]."""
    b, u = interval_coords(X, box)
    lx = lagrange_weights(u[:, 0], k)
    ly = lagrange_weights(u[:, 1], k)
    psi = np.zeros((Phi.shape[0], b.shape[0]))
    for a in range(k):
        for c in range(k):
            wgt = lx[:, a] * ly[:, c]
            psi += wgt[None, :] * Phi[:, b[:, 0] * k + a, b[:, 1] * k + c]
    return psi


def repulsion_ibfft(X, k: int, gamma: float = 2.0, rho: float = 1.0, n_int_min: int = 50,
                    n_int_fixed: int = 0, P: int | None = None, backend: str = "fft",
                    kernel=None, return_info: bool = False, rule: str = "unit"):
    """ibFFT repulsion.  F^r(i) = x_i psi_1(i) - psi_x(i)
    (P:465 Eq. repfK, P:474-475 Eqs. Fr1/Fr2) with the three kernel sums of Eq.
    kernelproduct approximated by spread -> grid convolution -> gather.
    The j = i term is kept in psi and cancels exactly (R10).  Coordinates are
    box-centred (R11; exact by translation invariance)."""
    if k not in (1, 2, 3):
        raise ValueError("k in {1,2,3}")
    X = np.asarray(X, dtype=np.float64)
    box = box_rule(X, n_int_min, n_int_fixed, rule)
    M = box.n_int * k
    h = float(box.w) / k
    K = kernel_tdist(gamma) if kernel is None else kernel
    C = spread(X, box, k)
    Phi = convolve_direct(C, h, K) if backend == "direct" else convolve_fft(C, h, K, P)
    psi = gather(Phi, X, box, k)
    xt = X - box.center
    R = rho * np.stack([xt[:, 0] * psi[0] - psi[1], xt[:, 1] * psi[0] - psi[2]], 1)
    if return_info:
        return R, dict(box=box, M=M, h=h, psi=psi, C=C, Phi=Phi)
    return R


# ---------------------------------------------------------------------------------------
# Runner
# ---------------------------------------------------------------------------------------
def forces(X, row_ptr, col, p: Params = Params(), solver: str = "exact", k: int = 3,
           n_int_min: int = 50, n_int_fixed: int = 0, P: int | None = None,
           rule: str = "unit"):
    """(R, A) for either repulsion path."""
    if solver == "exact":
        R = repulsion_exact(X, p.gamma, p.rho)
    elif solver == "ibfft":
        R = repulsion_ibfft(X, k, p.gamma, p.rho, n_int_min, n_int_fixed, P, rule=rule)
    else:
        raise ValueError(solver)
    return R, attraction(X, row_ptr, col, p.alpha, p.beta)


def step(X, row_ptr, col, p: Params, eta_t: float, **kw):
    """One Jacobi iteration x <- x + eta_t (R + A), all forces from the snapshot."""
    R, A = forces(X, row_ptr, col, p, **kw)
    return np.asarray(X, dtype=np.float64) + eta_t * (R + A)


def run(X0, row_ptr, col, p: Params = Params(), T: int = 300, eta0: float = 0.1,
        t0: int = 0, solver: str = "exact", k: int = 0, n_int_min: int = 50,
        n_int_fixed: int = 0, P: int | None = None, t_end: int | None = None,
        cooling: str = "linear", rule: str = "unit", round_fp32: bool = False):
    """Iterations t = t0 .. t_end-1 (default T-1) of the layout loop.
    k = 0 -> dynamic 90/5/5 schedule; raises on a non-finite position with the
    iteration and node.  round_fp32: store the positions in fp32 after every update
    (the device's storage precision, R14) — a diagnostic of the storage rounding alone."""
    if T < 1 or eta0 <= 0:
        raise ValueError("T >= 1 and eta0 > 0")
    X = np.asarray(X0, dtype=np.float64).copy()
    ks = k_schedule(T)
    for t in range(t0, T if t_end is None else t_end):
        kt = int(ks[t]) if k == 0 else k
        X = step(X, row_ptr, col, p, eta(t, T, eta0, cooling), solver=solver, k=kt,
                 n_int_min=n_int_min, n_int_fixed=n_int_fixed, P=P, rule=rule)
        if round_fp32:
            X = X.astype(np.float32).astype(np.float64)
        bad = ~np.isfinite(X).all(1)
        if bad.any():
            raise FloatingPointError(f"diverged at iter {t} node {int(np.argmax(bad))}")
    return X


def global_refine(X, row_ptr, col, p: Params = Params(), gamma: float | None = None,
                  rho: float | None = None, T: int = 300, **kw):
    """Global refinement: "Taking a t-FDP layout as initialization ... re-applying
    t-FDP with repulsive t-forces of different values"; SPEC global_refine:
    `run` from the given layout with gamma and/or rho overridden, t = 0 .. T-1.
    gamma <= 1 -> ValueError."""
    g = p.gamma if gamma is None else float(gamma)
    r = p.rho if rho is None else float(rho)
    if not (g > 1.0) or not (r > 0.0):
        raise ValueError("global refinement needs gamma > 1 and rho > 0 (S:362)")
    return run(X, row_ptr, col, dataclasses.replace(p, gamma=g, rho=r), T=T, **kw)


# ---------------------------------------------------------------------------------------
# Local (fisheye) refinement (SPEC RefinementMask S:155-158, local_refine S:368-376)
# ---------------------------------------------------------------------------------------
@dataclasses.dataclass
class Focus:
    """RefinementMask: focal node set F and boosts lambda_a (attraction on edges
    with both ends in F u N(F)), lambda_f (repulsion among F u N(F)), lambda_s (repulsion
    among the other nodes); every boost >= 1.  Pairs with one end in the region keep
    weight 1 (reading R23)."""
    focal: tuple
    la: float = 1.0
    lf: float = 1.0
    ls: float = 1.0


def focus_region(n, row_ptr, col, focal):
    """label_i = 1 for i in F u N(F) (the focal nodes and their graph neighbours), else 0."""
    lab = np.zeros(n, dtype=np.int64)
    for f in focal:
        f = int(f)
        lab[f] = 1
        lab[col[row_ptr[f]:row_ptr[f + 1]]] = 1
    return lab


def _rep_weights(lab_i, lab_j, fo: Focus):
    """w_ij = lambda_f if both in the region, lambda_s if both outside, else 1."""
    both_in = (lab_i == 1) & (lab_j == 1)
    both_out = (lab_i == 0) & (lab_j == 0)
    return np.where(both_in, fo.lf, np.where(both_out, fo.ls, 1.0))


def repulsion_masked_exact(X, lab, fo: Focus, gamma=2.0, rho=1.0):
    """Masked repulsion, the definition written out: R_i = rho sum_j w_ij (x_i - x_j) s_ij^-gamma
    (Eq. repfK P:463 with the per-pair boosts of the refinement mask)."""
    X = np.asarray(X, dtype=np.float64)
    lab = np.asarray(lab)
    r = X[:, None, :] - X[None, :, :]
    sij = 1.0 + (r * r).sum(-1)
    w = _rep_weights(lab[:, None], lab[None, :], fo)
    return rho * (r * (w * sij ** (-gamma))[..., None]).sum(1)


def repulsion_masked_loops(X, lab, fo: Focus, gamma=2.0, rho=1.0):
    """Literal double loop of the masked repulsion (brute force, small n)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    out = np.zeros((n, 2))
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            if lab[i] and lab[j]:
                w = fo.lf
            elif not lab[i] and not lab[j]:
                w = fo.ls
            else:
                w = 1.0
            dx, dy = X[i, 0] - X[j, 0], X[i, 1] - X[j, 1]
            f = w * (1.0 + dx * dx + dy * dy) ** (-gamma)
            out[i, 0] += rho * f * dx
            out[i, 1] += rho * f * dy
    return out


def attraction_masked(X, row_ptr, col, lab, fo: Focus, alpha=0.1, beta=8.0):
    """A_i = -alpha sum_{j in adj(i)} a_ij (1 + beta/s_ij)(x_i - x_j), a_ij = lambda_a if both
    ends are in F u N(F) else 1 (P:26 'we enhance the attractive forces between the focal
    nodes and their neighbors')."""
    X = np.asarray(X, dtype=np.float64)
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    n = X.shape[0]
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    r = X[rows] - X[col]
    s = 1.0 + (r * r).sum(1)
    a = np.where((lab[rows] == 1) & (lab[col] == 1), fo.la, 1.0)
    out = np.zeros((n, 2))
    np.add.at(out, rows, -alpha * (a * (1.0 + beta / s))[:, None] * r)
    return out


def repulsion_masked_ibfft(X, lab, fo: Focus, k: int, gamma=2.0, rho=1.0, **kw):
    """Masked repulsion on the interpolation/FFT path (reading R23): the grid cannot carry
    per-pair weights, so with S_all the unmasked sum (ibFFT) and S1_i the exact sum over the
    region's sources j in F u N(F),
      R_i = rho [w0(i) (S_all,i - S1_i) + w1(i) S1_i],  w0/w1 = the weight of (i, j) for j
    outside / inside the region (exact masked corrections inside the region)."""
    X = np.asarray(X, dtype=np.float64)
    lab = np.asarray(lab)
    R_all = repulsion_ibfft(X, k, gamma, 1.0, **kw)
    src = np.nonzero(lab == 1)[0]
    r = X[:, None, :] - X[None, src, :]
    S1 = (r * ((1.0 + (r * r).sum(-1)) ** (-gamma))[..., None]).sum(1)
    w0 = np.where(lab == 1, 1.0, fo.ls)[:, None]
    w1 = np.where(lab == 1, fo.lf, 1.0)[:, None]
    return rho * (w0 * (R_all - S1) + w1 * S1)


def forces_masked(X, row_ptr, col, lab, fo: Focus, p: Params = Params(), solver="exact",
                  k: int = 3, **kw):
    if solver == "exact":
        R = repulsion_masked_exact(X, lab, fo, p.gamma, p.rho)
    else:
        R = repulsion_masked_ibfft(X, lab, fo, k, p.gamma, p.rho, **kw)
    return R, attraction_masked(X, row_ptr, col, lab, fo, p.alpha, p.beta)


def energy_masked(X, row_ptr, col, lab, fo: Focus, p: Params = Params()):
    """E with D = -grad E for the masked forces (constant weights; gamma > 1):
    rho sum_{i<j} w_ij s^(1-gamma)/(2(gamma-1)) + alpha sum_edges a_ij (d^2/2 + (beta/2) ln s)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    iu, ju = np.triu_indices(n, 1)
    r = X[iu] - X[ju]
    s = 1.0 + (r * r).sum(1)
    w = _rep_weights(lab[iu], lab[ju], fo)
    Er = p.rho * (w * s ** (1.0 - p.gamma)).sum() / (2.0 * (p.gamma - 1.0))
    rows = np.repeat(np.arange(n), np.diff(np.asarray(row_ptr)))
    col = np.asarray(col)
    keep = rows < col
    r = X[rows[keep]] - X[col[keep]]
    s = 1.0 + (r * r).sum(1)
    a = np.where((lab[rows[keep]] == 1) & (lab[col[keep]] == 1), fo.la, 1.0)
    Ea = p.alpha * (a * (0.5 * (s - 1.0) + 0.5 * p.beta * np.log(s))).sum()
    return Er + Ea


def local_refine(X, row_ptr, col, fo: Focus, p: Params = Params(), T: int = 300,
                 eta0: float = 0.1, solver: str = "exact", k: int = 0, cooling: str = "linear",
                 **kw):
    """Local refinement (SPEC local_refine S:368-372): re-run from the given layout
    for t = 0 .. T-1 with the refinement mask.  Empty focal set -> ValueError."""
    if len(fo.focal) == 0:
        raise ValueError("empty focal set (S:372)")
    if min(fo.la, fo.lf, fo.ls) < 1.0:
        raise ValueError("boosts must be >= 1 (S:156)")
    X = np.asarray(X, dtype=np.float64).copy()
    n = X.shape[0]
    lab = focus_region(n, row_ptr, col, fo.focal)
    ks = k_schedule(T)
    for t in range(T):
        kt = int(ks[t]) if k == 0 else k
        R, A = forces_masked(X, row_ptr, col, lab, fo, p, solver=solver, k=kt, **kw)
        X = X + eta(t, T, eta0, cooling) * (R + A)
        bad = ~np.isfinite(X).all(1)
        if bad.any():
            raise FloatingPointError(f"diverged at iter {t} node {int(np.argmax(bad))}")
    return X


# ---------------------------------------------------------------------------------------
# PivotMDS initialisation (SPEC init_pivot_mds S:110-118; Brandes & Pich 2006)
# ---------------------------------------------------------------------------------------
def splitmix64(x: int) -> int:
    """SplitMix64 output for counter x (the counter-based generator both sides implement)."""
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def bfs_hops(row_ptr, col, src: int):
    """Hop distances from src (-1 = unreachable), plain queue BFS."""
    from collections import deque

    n = len(row_ptr) - 1
    d = np.full(n, -1, dtype=np.int64)
    d[src] = 0
    q = deque([src])
    while q:
        u = q.popleft()
        for v in col[row_ptr[u]:row_ptr[u + 1]]:
            if d[v] < 0:
                d[v] = d[u] + 1
                q.append(int(v))
    return d


def pmds_pivots(row_ptr, col, n_pivots: int, seed: int):
    """Max-min farthest-point pivots: the first is splitmix64(seed) mod n, each next
    one maximises the hop distance to the chosen set (ties: lowest index).  Returns
    (pivots, D) with D[:, j] the hop distances from pivot j; unreachable nodes get the
    pivot's eccentricity + 1 (reading R24)."""
    n = len(row_ptr) - 1
    p = min(int(n_pivots), n)
    D = np.zeros((n, p), dtype=np.int64)
    mind = np.full(n, np.iinfo(np.int64).max)
    piv = splitmix64(int(seed)) % n
    pivots = []
    for j in range(p):
        pivots.append(int(piv))
        d = bfs_hops(row_ptr, col, piv)
        d[d < 0] = d.max() + 1
        D[:, j] = d
        mind = np.minimum(mind, d)
        piv = int(np.argmax(mind))  # first index of the maximum
    return np.array(pivots, dtype=np.int64), D


def pivot_mds(row_ptr, col, n_pivots: int = 50, seed: int = 0):
    """PivotMDS layout: squared hop distances to the pivots, double-centred
    C = -1/2 (D2 - row means - column means + grand mean) (n x p), the top-2 eigenvectors
    v_1, v_2 of C^T C (library eigh; the right singular vectors of C), positions C v_k,
    centred and scaled to mean edge length 1.  Eigenvector signs: the largest-|.| component
    positive (lowest index on ties).  Returns (X, pivots)."""
    if n_pivots < 1:
        raise ValueError("pivot_count >= 1 (S:117)")
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    n = len(row_ptr) - 1
    pivots, D = pmds_pivots(row_ptr, col, n_pivots, seed)
    D2 = D.astype(np.float64) ** 2
    C = -0.5 * (D2 - D2.mean(1, keepdims=True) - D2.mean(0, keepdims=True) + D2.mean())
    w, V = np.linalg.eigh(C.T @ C)
    order = np.argsort(-w, kind="stable")
    X = np.zeros((n, 2))
    for a in range(min(2, V.shape[1])):
        v = V[:, order[a]]
        if w[order[a]] <= 1e-12 * max(w[order[0]], 1e-300):
            continue  # rank < 2: that axis stays 0 (reading R24)
        m = np.abs(v)
        if v[int(np.argmax(m))] < 0:
            v = -v
        X[:, a] = C @ v
    X -= X.mean(0)
    if row_ptr[-1] > 0:
        rows = np.repeat(np.arange(n), np.diff(row_ptr))
        L = np.linalg.norm(X[rows] - X[col], axis=1).mean()
        if L > 0:
            X /= L
    return X, pivots


# ---------------------------------------------------------------------------------------
# Neighbourhood preservation NP1
# ---------------------------------------------------------------------------------------
def np1(X, row_ptr, col, brute_max: int = 4096):
    """NP = (1/n) sum_i |N_G(i,1) ∩ N_L(x_i,k_i)| / |N_G(i,1) ∪ N_L(x_i,k_i)|, k_i = deg(i);
    layout kNN excludes i; ties by lower index; k_i = 0 contributes 1."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    deg = np.diff(row_ptr)
    total = 0.0
    if n <= brute_max:
        for i in range(n):
            ki = int(deg[i])
            if ki == 0:
                total += 1.0
                continue
            d2 = ((X - X[i]) ** 2).sum(1)
            d2[i] = np.inf
            nn = np.argsort(d2, kind="stable")[:ki]  # stable: ties -> lower index
            G = set(col[row_ptr[i]:row_ptr[i + 1]].tolist())
            Lset = set(nn.tolist())
            total += len(G & Lset) / len(G | Lset)
        return total / n
    from scipy.spatial import cKDTree  # library kNN primitive for large n (pinned vs brute force)

    tree = cKDTree(X)
    order = np.argsort(deg, kind="stable")
    for kval in np.unique(deg):
        idx = order[deg[order] == kval]
        if kval == 0:
            total += idx.size
            continue
        kq = int(min(n, kval + 1))
        for s in range(0, idx.size, 65536):
            ii = idx[s:s + 65536]
            _, nb = tree.query(X[ii], k=kq)
            nb = np.asarray(nb).reshape(ii.size, kq)
            for r, i in enumerate(ii):
                cand = [j for j in nb[r].tolist() if j != i][: int(kval)]
                G = set(col[row_ptr[i]:row_ptr[i + 1]].tolist())
                Lset = set(cand)
                total += len(G & Lset) / len(G | Lset)
    return total / n


def np1_hits(X, row_ptr, col, nodes=None, dist: str = "fp64"):
    """Per node i: |N_G(i,1) ∩ N_L(x_i, k_i)|, k_i = deg(i), by brute force —
    the layout kNN excludes i, ties by lower index, k_i = 0 -> 0.
    dist = "fp64": d^2 in fp64.  dist = "fp32": the kNN decisions are taken on
    d^2 = (dx*dx) + (dy*dy) with dx = x_j - x_i and every operation rounded to IEEE fp32
    (the device kernel's precision; R22)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = row_ptr.shape[0] - 1
    if dist == "fp32":
        Xc = np.asarray(X, dtype=np.float32)
    elif dist == "fp64":
        Xc = np.asarray(X, dtype=np.float64)
    else:
        raise ValueError(dist)
    nodes = np.arange(n) if nodes is None else np.asarray(nodes, dtype=np.int64)
    out = np.zeros(nodes.shape[0], dtype=np.int64)
    for r, i in enumerate(nodes.tolist()):
        ki = int(row_ptr[i + 1] - row_ptr[i])
        if ki == 0:
            continue
        dx = Xc[:, 0] - Xc[i, 0]
        dy = Xc[:, 1] - Xc[i, 1]
        d2 = dx * dx + dy * dy  # numpy: each op rounded in the array dtype, no contraction
        d2[i] = np.inf
        nn = np.argsort(d2, kind="stable")[:ki]  # stable: equal distances -> lower index
        G = set(col[row_ptr[i]:row_ptr[i + 1]].tolist())
        out[r] = len(G & set(nn.tolist()))
    return out


def np1_from_hits(hits, row_ptr):
    """NP1 = (1/n) sum_i |∩| / |∪| with |∪| = 2 k_i - |∩| (both sets have k_i elements) and
    k_i = 0 contributing 1."""
    deg = np.diff(np.asarray(row_ptr, dtype=np.int64))
    h = np.asarray(hits, dtype=np.float64)
    per = np.where(deg == 0, 1.0, h / np.maximum(2 * deg - h, 1))
    return float(per.mean())
