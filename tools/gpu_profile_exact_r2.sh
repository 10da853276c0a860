#!/bin/bash
# Round-2 exact-path profiling (run under gpurun from the repo root): ncu --set full of the
# all-pairs kernel at C3 and of exact_finish / heavy_attr at C5 (Chung-Lu hubs: the
# degree-skew split of the row walk), plus a launch list of one C5 force evaluation.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"exact_partial" -c 1 \
  -o /tmp/ex_c3 -f python tools/exact_iter.py C3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"exact_finish|heavy_attr" -c 2 \
  -o /tmp/ex_c5 -f python tools/exact_iter.py C5 > /dev/null 2>&1
{ python tools/ncu_summary.py /tmp/ex_c3.ncu-rep; python tools/ncu_summary.py /tmp/ex_c5.ncu-rep; } \
  > gpurun_out/r2_ncu_full_exact_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_launches_exact_c5.csv python tools/exact_iter.py C5 > /dev/null 2>&1
cat gpurun_out/r2_ncu_full_exact_summary.txt
