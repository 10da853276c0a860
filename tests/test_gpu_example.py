"""The C ABI from a plain C program (examples/tfdp_layout.c, built by build() against the
in-tree libtfdp.so): CSR build, init, a full dynamic-k layout, layout read-back and NP1, every
status checked — no Python or torch in the client."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("args", [("60", "300", "1"), ("30", "100", "0")])
def test_c_client(args):
    exe = os.path.join(ROOT, "examples", "tfdp_layout")
    if not os.path.exists(exe):
        from paper_2303_03964_b200 import build as B
        B.build_examples()
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    m = re.search(r"np1=([0-9.]+)", r.stdout)
    assert m and 0.3 < float(m.group(1)) <= 1.0  # a grid graph lays out its neighbourhoods
