"""NP1 scatter of full C3 runs (300 iterations, dynamic k) over repeated GPU runs (developer
tool behind the bar of tests/test_gpu_fft.py::test_full_run_np1_C3)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config
w = make_config("C3")
rp, col = O.csr_build(w.n, w.u, w.v)
rule = "span" if "--span" in sys.argv else "unit"
ngs = []
for r in range(8):
    with P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0, interval_rule=rule)) as L:
        L.step(300)
        ngs.append(O.np1(L.layout(), rp, col))
print(rule, "GPU NP1 runs", [round(x, 4) for x in ngs], "mean", np.mean(ngs), "std", np.std(ngs))
Xo = O.run(w.xy, rp, col, O.Params(), T=300, solver="ibfft", k=0, rule=rule) if "--oracle" in sys.argv else None
if Xo is not None:
    print("oracle NP1", O.np1(Xo, rp, col))
