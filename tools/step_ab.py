"""Iterations/s of the bench's stationary C4 step (set_layout + set_iteration(0) + step(20),
dynamic k 18/1/1) without any per-kernel events, for A/B runs of launch modes (e.g.
TFDP_GRAPH=0/1).  Usage: python tools/step_ab.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import oracle as O
import paper_2303_03964_b200 as P
from synth import make_config

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
w = make_config("C4")
rp, col = O.csr_build(w.n, w.u, w.v)
s = torch.cuda.Stream()
L = P.Layout(w.n, rp, col, w.xy, P.Params(solver="ibfft", k=0, iterations=20), stream=s.cuda_stream)
x0 = torch.from_numpy(w.xy).cuda()


def one():
    L.set_layout(x0)
    L.set_iteration(0)
    L.step(20)


for _ in range(4):
    one()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
for _ in range(steps):
    one()
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"GRAPH={os.environ.get('TFDP_GRAPH', '1')} {steps * 20 / (ms / 1e3):.1f} it/s ({ms / steps:.3f} ms/step)")
L.close()
