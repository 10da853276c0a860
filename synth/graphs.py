"""Seeded graph + position generators for configs C1..C5.

Every function returns raw data only:
  * ``u, v``  int32 arrays of undirected edge endpoints (may contain duplicates /
    self-loops only where documented -- cleaning them is the CSR builder's job);
  * ``xy``    float32 (n, 2) starting positions, centred at the origin.
No t-FDP arithmetic lives here.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class Workload:
    name: str
    n: int
    u: np.ndarray  # int32 [m_raw]
    v: np.ndarray  # int32 [m_raw]
    xy: np.ndarray  # float32 [n, 2]
    note: str = ""

    @property
    def m_raw(self) -> int:
        return int(self.u.shape[0])


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform_disc(n: int, radius: float, seed: int) -> np.ndarray:
    """i.i.d. uniform points in a disc of `radius` centred at 0 (SPEC S:101-104 init_random)."""
    g = _rng(seed)
    r = radius * np.sqrt(g.random(n))
    th = 2.0 * math.pi * g.random(n)
    return np.stack([r * np.cos(th), r * np.sin(th)], axis=1).astype(np.float32)


def uniform_square(n: int, side: float, seed: int) -> np.ndarray:
    g = _rng(seed)
    return ((g.random((n, 2)) - 0.5) * side).astype(np.float32)


def grid_graph(rows: int, cols: int):
    """rows x cols grid: node r*cols+c, right and down edges (C1: 10x10 -> m=180)."""
    idx = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    right_u, right_v = idx[:, :-1].ravel(), idx[:, 1:].ravel()
    down_u, down_v = idx[:-1, :].ravel(), idx[1:, :].ravel()
    u = np.concatenate([right_u, down_u]).astype(np.int32)
    v = np.concatenate([right_v, down_v]).astype(np.int32)
    return u, v


def mesh_graph(side: int):
    """side x side grid plus one diagonal per cell (qh882/cage8-shaped mesh).

    32x32 -> n=1024, m = 2*32*31 + 31*31 = 2945, mean degree 5.75.
    """
    u, v = grid_graph(side, side)
    idx = np.arange(side * side, dtype=np.int64).reshape(side, side)
    du, dv = idx[:-1, :-1].ravel(), idx[1:, 1:].ravel()
    return (np.concatenate([u, du.astype(np.int32)]),
            np.concatenate([v, dv.astype(np.int32)]))


def rgg_graph(n: int, radius: float, side: float, seed: int):
    """Random geometric graph: n uniform points in a side x side square (random node
    order), an edge for every pair closer than `radius`.  Returns (u, v, xy_centred)."""
    from scipy.spatial import cKDTree

    g = _rng(seed)
    pts = g.random((n, 2)) * side
    pairs = cKDTree(pts).query_pairs(radius, output_type="ndarray")
    xy = (pts - side / 2.0).astype(np.float32)
    return pairs[:, 0].astype(np.int32), pairs[:, 1].astype(np.int32), xy


def chung_lu_graph(n: int, mean_degree: float, exponent: float, seed: int):
    """Chung-Lu power-law graph: expected degree w_i ~ (i+i0)^(-1/(exponent-1)),
    m = n*mean_degree/2 endpoint pairs drawn with probability ~ w.  Raw pairs keep
    duplicates and self-loops (the CSR builder drops them), so the cleaned mean
    degree is slightly below `mean_degree`."""
    g = _rng(seed)
    i0 = 10.0
    w = (np.arange(n, dtype=np.float64) + i0) ** (-1.0 / (exponent - 1.0))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    m = int(round(n * mean_degree / 2.0))
    u = np.searchsorted(cdf, g.random(m), side="right").astype(np.int32)
    v = np.searchsorted(cdf, g.random(m), side="right").astype(np.int32)
    np.minimum(u, n - 1, out=u)
    np.minimum(v, n - 1, out=v)
    # random relabelling so hubs are spread over the id space (no sorted-degree order)
    perm = g.permutation(n).astype(np.int32)
    return perm[u], perm[v]


def _mean_edge_len(xy: np.ndarray, u: np.ndarray, v: np.ndarray) -> float:
    d = xy[u].astype(np.float64) - xy[v].astype(np.float64)
    return float(np.sqrt((d * d).sum(1)).mean())


def make_config(name: str) -> Workload:
    """The five configs of SURVEY.md §8(d)."""
    if name == "C1":
        u, v = grid_graph(10, 10)
        xy = uniform_disc(100, 5.0, seed=0)
        return Workload("C1", 100, u, v, xy, "10x10 grid, uniform disc r=5, seed 0")
    if name == "C2":
        side = 32
        u, v = mesh_graph(side)
        g = _rng(1)
        gy, gx = np.divmod(np.arange(side * side), side)
        xy = np.stack([gx, gy], 1).astype(np.float64)
        xy += 0.15 * (g.random(xy.shape) - 0.5)  # break exact ties of the lattice
        xy = xy / _mean_edge_len(xy, u, v)  # mean edge length 1
        xy -= xy.mean(0)
        return Workload("C2", side * side, u, v, xy.astype(np.float32),
                        "32x32 mesh + diagonals, lattice coords jittered, mean edge 1, seed 1")
    if name == "C2rgg":
        n = 1015
        side = math.sqrt(n)
        r = math.sqrt(10.0 / math.pi)  # mean degree 10 at unit density
        u, v, xy = rgg_graph(n, r, side, seed=1)
        return Workload("C2rgg", n, u, v, xy, "RGG n=1015 mean degree 10, seed 1")
    if name in ("C3", "C4"):
        n = 100_000 if name == "C3" else 1_000_000
        seed = 2 if name == "C3" else 3
        side = math.sqrt(n)
        r = math.sqrt(8.0 / math.pi)  # mean degree 8 at unit density
        u, v, xy = rgg_graph(n, r, side, seed=seed)
        return Workload(name, n, u, v, xy, f"RGG n={n} unit density mean degree 8, seed {seed}")
    if name == "C5":
        n = 4_000_000
        u, v = chung_lu_graph(n, 17.35, 2.5, seed=4)
        xy = uniform_square(n, 2000.0, seed=4)
        return Workload("C5", n, u, v, xy, "Chung-Lu n=4M exp 2.5 mean deg 17.35, square side 2000, seed 4")
    raise ValueError(f"unknown config {name}")


CONFIGS = ("C1", "C2", "C2rgg", "C3", "C4", "C5")


def random_layout(n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """Generic seeded Gaussian layout for small tests."""
    return (_rng(seed).standard_normal((n, 2)) * scale).astype(np.float32)


def blob_layout(n: int, n_blobs: int, sigma: float, side: float, seed: int) -> np.ndarray:
    """Clustered layout: n points in n_blobs Gaussian clusters (std sigma) with centres
    uniform in [0, side]^2, random node order — many nodes per unit interval (the shape of
    a converged layout's dense clusters)."""
    g = _rng(seed)
    centres = g.random((n_blobs, 2)) * side
    which = g.integers(0, n_blobs, n)
    return (centres[which] + g.standard_normal((n, 2)) * sigma).astype(np.float32)


def path_graph(n: int):
    """Path P_n: edges (i, i+1) (SPEC S:365 refinement example P20)."""
    u = np.arange(n - 1, dtype=np.int32)
    return u, u + 1


def two_cluster_graph(n_per: int, p_in: float, p_out: float, seed: int):
    """Two-block stochastic block model (SPEC S:366 '2-cluster synthetic graph'): nodes
    [0, n_per) and [n_per, 2 n_per); each pair is an edge with probability p_in inside a
    block and p_out across.  Returns (u, v, label)."""
    g = _rng(seed)
    n = 2 * n_per
    iu, ju = np.triu_indices(n, 1)
    lab = (np.arange(n) >= n_per).astype(np.int32)
    p = np.where(lab[iu] == lab[ju], p_in, p_out)
    keep = g.random(iu.shape[0]) < p
    return iu[keep].astype(np.int32), ju[keep].astype(np.int32), lab


def random_graph(n: int, m: int, seed: int):
    """Generic seeded random edge list (raw; may contain duplicates / self-loops)."""
    g = _rng(seed)
    return (g.integers(0, n, m).astype(np.int32), g.integers(0, n, m).astype(np.int32))
