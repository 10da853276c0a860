"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 NumPy implementation of the t-FDP force step written from the
paper (arXiv 2303.03964, /root/reference/PAPER.md, cited as P:<line>) and, for
interfaces/worked examples, SPEC.md (S:<line>).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The product path
(``paper_2303_03964_b200``) never imports, calls or links this package and shares no
code with it; the only shared module is ``synth`` (seeded input generators, no method
arithmetic).

Pins: every function here is pinned by ``tests/test_oracle_*.py`` against closed
forms, paper/SPEC worked examples, invariants or brute force (see DESIGN.md
"Oracle pins").  No function is "parity unpinned".
"""
from .tfdp_oracle import *  # noqa: F401,F403
