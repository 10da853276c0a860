"""Dynamic SASS opcode mix (instructions executed) and stall samples per opcode for one
kernel of an ncu report.  Usage: python tools/ncu_opmix.py rep.ncu-rep launch_index"""
import collections, csv, io, re, subprocess, sys
rep, idx = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 3 and r[2].isdigit()]
half = len(data) // 2 if len(data) % 2 == 0 and data[: len(data) // 2] == data[len(data) // 2:] else len(data)
data = data[:half]
isrc, ie, isamp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops, samp = collections.Counter(), collections.Counter()
for r in data:
    s = r[isrc].strip()
    s = re.sub(r"^@!?U?P\w+\s+", "", s)
    op = s.split()[0].split(".")[0] if s else "?"
    ops[op] += float(r[ie] or 0)
    samp[op] += float(r[isamp] or 0)
T, S = sum(ops.values()), sum(samp.values())
print(rows[0][1][:100], f"inst={T:.0f} samples={S:.0f}")
for op, v in ops.most_common(30):
    print(f"{op:10s} {100*v/T:5.1f}% inst  {100*samp[op]/S:5.1f}% stall-samples")
