"""Top SASS lines by warp-stall samples for one kernel of an ncu report (source page).
Usage: python tools/ncu_hot.py rep.ncu-rep launch_index [top]"""
import csv, io, subprocess, sys
rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
name = rows[0][1]
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 3 and r[2].isdigit()]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[isamp] or 0) for r in data)
print(name[:120], "samples", tot)
for k, r in enumerate(data):
    r.append(k)
for r in sorted(data, key=lambda r: -int(r[isamp] or 0))[:top]:
    print(f"{int(r[isamp]):6d} {100*int(r[isamp])/tot:5.1f}%  #{r[-1]:4d} {r[isrc].strip()[:90]}")
