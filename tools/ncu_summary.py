"""Summarise an ncu report: per kernel duration, instructions, IPC, occupancy, DRAM bytes,
smem conflicts and top stall reasons.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
# normalise the duration to microseconds (ncu picks ns / us / ms per report)
_it = hdr.index("gpu__time_duration.sum") if "gpu__time_duration.sum" in hdr else None
if _it is not None:
    _f = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
          "second": 1e6, "s": 1e6}.get(units[_it], 1.0)
    for r in data:
        r[_it] = f"{float(r[_it]) * _f:.3f}"
# DRAM bytes in MB
for _m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    if _m in hdr:
        _i = hdr.index(_m)
        _f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(units[_i], 1.0)
        for r in data:
            r[_i] = f"{float(r[_i]) * _f:.3f}"
def col(name):
    for i, h in enumerate(hdr):
        if h == name:
            return i
    return None
keys = [("time_us", "gpu__time_duration.sum"), ("inst", "smsp__inst_executed.sum"),
        ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("dram_rd_MB", "dram__bytes_read.sum"), ("dram_wr_MB", "dram__bytes_write.sum"),
        ("smem_wf", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        ("smem_confl_ld", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        ("smem_confl_st", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
        ("regs", "launch__registers_per_thread"), ("block", "launch__block_size"),
        ("grid", "launch__grid_size")]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
iname = col("Kernel Name")
for r in data:
    name = r[iname].split("(")[0][-40:]
    vals = []
    for k, m in keys:
        c = col(m)
        vals.append(f"{k}={r[c]}" if c is not None else f"{k}=?")
    st = sorted(((float(r[col(h)] or 0), h) for h in stalls), reverse=True)[:5]
    print(name, " ".join(vals))
    print("   stalls/issue:", ", ".join(f"{h.split('stalled_')[1].split('_per_issue')[0]}={v:.2f}" for v, h in st))
