"""Per-kernel registers / spills / smem from `nvcc -Xptxas -v` (rebuilds libtfdp.so)."""
import os, re, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03964_b200 import build as B
import io, contextlib
err = io.StringIO()
with contextlib.redirect_stderr(err):
    B.build(verbose=True, force=True)
cur = None
out = {}
for line in err.getvalue().splitlines():
    m = re.search(r"(?:Compiling entry function|Function properties for) '?(_Z\w+)", line)
    if m:
        cur = m.group(1)
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"tfdp::\(anonymous namespace\)::|tfdp::", "", name)
        cur = re.sub(r"\(.*", "", name)
        out.setdefault(cur, {})
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        out[cur]["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        out[cur]["regs"] = int(m.group(1))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in sorted(out.items()):
    if pat in k:
        print(f"{k:60s} regs={v.get('regs')} spill={v.get('spill', 0)}")
