"""Runs a few fixed-k ibFFT iterations at C4 (developer tool for ncu captures of the FFT
passes).  Usage: python tools/fft_iter.py [k] [iters]; iters >= 8 so that the first
tfdp_step call renumbers the nodes (Morton order, as in the bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2303_03964_b200 as P
from synth import make_config

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = max(8, int(sys.argv[2]) if len(sys.argv) > 2 else 8)
w = make_config("C4")
rp, col = P.csr_build(w.n, w.u, w.v)
prm = P.Params(solver="ibfft", k=k, cooling="constant", step0=1e-3)
with P.Layout(w.n, rp, col, w.xy, prm) as L:
    L.step(iters)
    torch.cuda.synchronize()
print("done", k, iters)
