#!/bin/bash
# Round-2 profiling pass of the ibFFT path at C4 (run under gpurun from the repo root): one
# ncu --set full capture per hot kernel and k (the second launch of each, Morton-renumbered
# nodes as in the bench), summaries + DRAM traffic, and the launch list of the bench command.
mkdir -p gpurun_out
for k in 1 2 3; do
  for kern in "^cols_kernel" rows_fwd_kernel rows_inv_kernel gather_update_kernel spread_kernel; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$kern" -s 1 -c 1 \
      -o /tmp/r2_k${k}_$kern -f python tools/fft_iter.py $k 8 > /dev/null 2>&1
  done
  for kern in "^cols_kernel" rows_fwd_kernel rows_inv_kernel gather_update_kernel spread_kernel; do
    python tools/ncu_summary.py /tmp/r2_k${k}_$kern.ncu-rep
  done > gpurun_out/r2_ncu_full_c4_k${k}_summary.txt 2>&1
  for kern in "^cols_kernel" rows_fwd_kernel rows_inv_kernel gather_update_kernel spread_kernel; do
    ncu -i /tmp/r2_k${k}_$kern.ncu-rep --page raw --csv 2>/dev/null
  done > gpurun_out/r2_ncu_full_k${k}_raw.csv
done
cp /tmp/r2_k3_cols_kernel.ncu-rep gpurun_out/ 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 200 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-exact --no-e2e \
  --no-cpu-baseline --no-full > /dev/null 2>&1
ls -la gpurun_out
