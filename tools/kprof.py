"""Per-k timing of ibFFT iterations (developer tool, not the bench): wall time per
iteration (CUDA events around tfdp_step, no per-kernel instrumentation), then a separate
instrumented pass for the per-kernel breakdown.  Usage: python tools/kprof.py [C4] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2303_03964_b200 as P
from synth import blob_layout, make_config

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lay = sys.argv[3] if len(sys.argv) > 3 else "input"
w = make_config(name)
rp, col = P.csr_build(w.n, w.u, w.v)
X0 = w.xy
if lay == "blobs":
    span = float((w.xy.max(0) - w.xy.min(0)).max())
    X0 = blob_layout(w.n, 1000, 2.0, span, 7)
for k in (1, 2, 3):
    s = torch.cuda.Stream()
    prm = P.Params(solver="ibfft", k=k, cooling="constant", step0=1e-3)
    with P.Layout(w.n, rp, col, X0, prm, stream=s.cuda_stream) as L:
        for _ in range(3):
            L.step(reps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        L.step(reps)
        e1.record(s)
        torch.cuda.synchronize()
        wall = 1e3 * e0.elapsed_time(e1) / reps
        L.profile(True)
        L.step(reps)
        prof = L.profile_read()
        geo = L.fft_geometry()
        print(f"[{lay}] k={k} M={geo['n_int']*k} P={geo['P']} wall {wall:.1f} us/iter :: " +
              " ".join(f"{n}={1e3*v[0]/v[1]:.1f}" for n, v in prof.items()), flush=True)
