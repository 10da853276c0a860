"""SASS opcode mix of one kernel from an ncu report (source page).
Usage: python tools/ncu_mix.py rep.ncu-rep kernel_regex"""
import collections, csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
i0 = rows.index(hdr)
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot, stall, total = collections.Counter(), collections.Counter(), 0
for r in rows[i0 + 1:]:
    try:
        e, w = int(r[iE]), int(r[iW])
    except (ValueError, IndexError):
        continue
    toks = r[iS].strip().split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    op = op.split(".")[0]
    tot[op] += e
    stall[op] += w
    total += e
print("total warp inst", total)
for op, c in tot.most_common(22):
    print(f"{op:10s} {c:10d} {100 * c / total:5.1f}%  stall_samples={stall[op]}")
