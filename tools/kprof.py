"""Per-k kernel timing of one ibFFT force evaluation (developer tool, not the bench).
Usage: python tools/kprof.py [C4] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2303_03964_b200 as P
from synth import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = make_config(name)
rp, col = P.csr_build(w.n, w.u, w.v)
for k in (1, 2, 3):
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=k, cooling="constant", step0=1e-3)) as L:
        for _ in range(3):
            L.step(1)
        L.profile(True)
        L.step(reps)
        prof = L.profile_read()
        geo = L.fft_geometry()
        tot = sum(v[0] for v in prof.values())
        print(f"k={k} M={geo['n_int']*k} P={geo['P']} total {1e3*tot/reps:.1f} us/iter :: " +
              " ".join(f"{n}={1e3*v[0]/v[1]:.1f}" for n, v in prof.items()), flush=True)
