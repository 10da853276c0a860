"""DRAM traffic per launch from `ncu --set full` raw CSV exports (one per fixed-k run of
tools/gpu_profile_fft.sh): dram__bytes_read.sum + dram__bytes_write.sum per kernel kind and
k, written as JSON for bench.py's roofline "traffic" field.
Usage: python tools/ncu_traffic.py out.json k1_raw.csv k2_raw.csv k3_raw.csv"""
import csv
import json
import re
import sys

KINDS = [("kspec_rows_kernel", "kspec_rows"), ("kspec_cols_kernel", "kspec_cols"),
         ("spread_kernel", "spread"), ("rows_fwd_kernel", "rows_fwd"), ("cols_kernel", "cols"),
         ("rows_inv_kernel", "rows_inv"), ("gather_update_kernel", "gather_update"), ("attraction_kernel", "attraction")]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kind_of(name):
    for pat, kind in KINDS:
        if re.search(r"\b" + pat + r"<", name) or ("::" + pat + "<") in name:
            return kind
    return None


def main():
    out, files = sys.argv[1], sys.argv[2:]
    res = {"source": "ncu --set full --clock-control none (tools/gpu_profile_r2.sh, C4, fixed k)",
           "unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)", "kernels": {}}
    for k, path in enumerate(files, start=1):
        rows = list(csv.reader(open(path)))
        h, units, data = rows[0], rows[1], rows[2:]
        iname, ird, iwr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        for r in data:
            if len(r) <= max(ird, iwr) or r[iname] == "Kernel Name":
                continue  # header / unit rows of concatenated exports
            kind = kind_of(r[iname])
            if kind is None:
                continue
            try:
                b = float(r[ird]) * SCALE[units[ird]] + float(r[iwr]) * SCALE[units[iwr]]
            except ValueError:
                continue
            res["kernels"].setdefault(kind, {})[str(k)] = round(b)
    # the bench times kspec_rows + kspec_cols under one scope
    ks = res["kernels"]
    if "kspec_rows" in ks and "kspec_cols" in ks:
        ks["kspec_rows"] = {k: ks["kspec_rows"][k] + ks["kspec_cols"].get(k, 0) for k in ks["kspec_rows"]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
