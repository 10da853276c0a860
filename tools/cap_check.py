"""Does a full dynamic-k run hit the grid cap (TFDP_WARN_NINT_CAPPED, R20)?  Developer tool:
runs C3 for T = 300 in blocks and reports the warning bit, N_int and the plan per block."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 300
w = make_config(name)
rp, col = P.csr_build(w.n, w.u, w.v)
with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0)) as L:
    done = 0
    while done < 300:
        L.step(min(blk, 300 - done))
        done += min(blk, 300 - done)
        g = L.fft_geometry()
        X = L.layout()
        b = O.box_rule(X)
        print(done, "warn", L.warnings, "n_int", g["n_int"], "oracle n_int", b.n_int, "plans", [L.fft_plan(k) for k in (1, 2, 3)], flush=True)
    print("NP1", O.np1(L.layout(), rp, col))
