"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the t-FDP method (no forces, no interpolation, no
CSR construction): it only draws graphs (raw undirected edge lists, possibly with
duplicates/self-loops for the CSR builder to clean) and starting positions, with
NumPy PCG64 and fixed seeds.  See DESIGN.md "Input recipe" and SURVEY.md §8(d).
"""
from .graphs import (  # noqa: F401
    Workload,
    grid_graph,
    mesh_graph,
    rgg_graph,
    chung_lu_graph,
    uniform_disc,
    uniform_square,
    random_layout,
    blob_layout,
    random_graph,
    path_graph,
    two_cluster_graph,
    make_config,
    CONFIGS,
)
