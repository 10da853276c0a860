"""One exact all-pairs force evaluation at C3 (developer tool for ncu captures of the exact
kernels).  Usage: python tools/exact_iter.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2303_03964_b200 as P
from synth import make_config

w = make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
rp, col = P.csr_build(w.n, w.u, w.v)
with P.Layout(w.n, rp, col, w.xy, P.Params(solver="exact")) as L:
    L.forces()
    torch.cuda.synchronize()
print("done")
