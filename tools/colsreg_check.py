"""A/B check of the column-pass cores at P = 2048 (TFDP_COLS=reg / smem): forces against the
oracle at k = 1, 2, 3 on a forced grid; saves the forces under gpurun_out/."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import oracle as O, paper_2303_03964_b200 as P
from synth import random_layout, random_graph
n = 6000
X = random_layout(n, 31, 30.0)
u, v = random_graph(n, 4 * n, 32)
rp, col = O.csr_build(n, u, v)
for k in (1, 2, 3):
    nf = {1: 1000, 2: 500, 3: 333}[k]
    prm = P.Params(solver="ibfft", k=k, n_int_fixed=nf, fft_size=2048)
    with P.Layout(n, rp, col, X, prm) as L:
        R, _ = L.forces(); geo = L.fft_geometry()
    Ro = O.repulsion_ibfft(X.astype(np.float64), k, n_int_fixed=nf)
    print(os.environ.get("TFDP_COLS", "smem"), k, geo["P"], geo["n_int"], "rel", O.rel_l2(R, Ro), flush=True)
    np.save(f"gpurun_out/cr_{os.environ.get('TFDP_COLS','smem')}_{k}.npy", R)
