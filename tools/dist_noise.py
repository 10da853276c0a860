"""Noise floor of short ibFFT trajectories: single-rank runs against each other, a 3-rank
virtual group (each dist mode) and the oracle (developer tool behind tests/test_gpu_dist.py)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, oracle as O, paper_2303_03964_b200 as P
from synth import make_config
w = make_config("C2rgg"); rp, col = O.csr_build(w.n, w.u, w.v)
s = torch.cuda.Stream().cuda_stream
for step0 in (1e-2, 1e-3):
  for mode in ("spread_all", "slab"):
    prm = P.Params(solver="ibfft", k=2, dist_mode=mode, step0=step0)
    runs = []
    for rep in range(3):
        with P.Layout(w.n, rp, col, w.xy, prm) as L1:
            L1.step(5); runs.append(L1.layout() - w.xy)
    G = [P.Layout(w.n, rp, col, w.xy, prm, dist=P.Dist(r, 3, 0, None), stream=s) for r in range(3)]
    P.group_step(G, 5); Xg = G[2].layout() - w.xy
    for L in G: L.close()
    Xo = O.run(w.xy, rp, col, O.Params(), T=300, eta0=step0, solver="ibfft", k=2, t_end=5) - w.xy
    print(step0, mode, "single-single", [O.rel_l2(runs[0], r) for r in runs[1:]], "group-single", O.rel_l2(Xg, runs[0]), "single-oracle", O.rel_l2(runs[0], Xo), "group-oracle", O.rel_l2(Xg, Xo))
# the test's sequence: forces, then steps
for mode in ("spread_all", "slab"):
    prm = P.Params(solver="ibfft", k=2, dist_mode=mode, step0=1e-2)
    with P.Layout(w.n, rp, col, w.xy, prm) as L1:
        R1, _ = L1.forces(); L1.step(5); X1 = L1.layout() - w.xy
    G = [P.Layout(w.n, rp, col, w.xy, prm, dist=P.Dist(r, 3, 0, None), stream=s) for r in range(3)]
    out = P.group_forces(G)
    P.group_step(G, 5)
    Xs = [L.layout() - w.xy for L in G]
    print(mode, "forces then step: group-single per rank", [O.rel_l2(X, X1) for X in Xs],
          "iters", [L.iteration for L in G], [L.fft_geometry() for L in G][0], L1 if False else "")
    for L in G: L.close()
