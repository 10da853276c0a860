"""Developer check: NP1 of full C3 runs (GPU x3 vs oracle) to size run-to-run spread."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config
w = make_config("C3")
rp, col = P.csr_build(w.n, w.u, w.v)
print("np1 init", O.np1(w.xy, rp, col), flush=True)
for rep in range(3):
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0)) as L:
        L.step(300)
        Xg = L.layout()
    print("gpu", rep, O.np1(Xg, rp, col), flush=True)
t = time.time()
Xo = O.run(w.xy, rp, col, O.Params(), T=300, solver="ibfft", k=0)
print("oracle", O.np1(Xo, rp, col), time.time() - t, flush=True)
