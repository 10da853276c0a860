"""Diagnostic of the C3 full-run NP1 offset (VERDICT r1 'what's weak' 2): is the device's
NP1 above the fp64 oracle's because of fp32 position storage (R14) or because the run is
chaotic and every valid trajectory lands elsewhere?  Oracle only (no GPU):
  - the fp64 oracle run (the test's reference),
  - the same run with positions stored in fp32 after every update (round_fp32=True),
  - fp64 runs from inputs perturbed by 1e-7 relative (an ensemble of equally valid runs).
Usage: python tools/np1_offset_c3.py [n_perturbed]  -> prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np

import oracle as O
from synth import make_config

w = make_config("C3")
rp, col = O.csr_build(w.n, w.u, w.v)
n_pert = int(sys.argv[1]) if len(sys.argv) > 1 else 6
res = {}
t0 = time.time()
X = O.run(w.xy, rp, col, O.Params(), T=300, solver="ibfft", k=0)
res["fp64"] = O.np1(X, rp, col)
X = O.run(w.xy, rp, col, O.Params(), T=300, solver="ibfft", k=0, round_fp32=True)
res["fp32_storage"] = O.np1(X, rp, col)
g = np.random.default_rng(99)
pert = []
for i in range(n_pert):
    X0 = w.xy.astype(np.float64) * (1.0 + 1e-7 * g.standard_normal(w.xy.shape))
    pert.append(O.np1(O.run(X0, rp, col, O.Params(), T=300, solver="ibfft", k=0), rp, col))
res["fp64_perturbed"] = pert
res["perturbed_mean"] = float(np.mean(pert))
res["perturbed_std"] = float(np.std(pert))
res["seconds"] = time.time() - t0
print(json.dumps(res))
