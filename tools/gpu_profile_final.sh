#!/bin/bash
# Final-tree profiling pass (run under gpurun from the repo root): ncu --set full of the
# hot kernels at C4 k = 1, 2, 3 (second launch of each, Morton order, warm L2:
# --cache-control none), DRAM traffic, and the launch list of the bench command.
mkdir -p gpurun_out
for k in 1 2 3; do
  for kern in "^cols_kernel" rows_fwd_kernel rows_inv_kernel gather_update_kernel spread_kernel "^attraction_kernel"; do
    tag=$(echo $kern | tr -d '^')
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$kern" -s 1 -c 1 \
      -o /tmp/f_k${k}_$tag -f python tools/fft_iter.py $k 8 > /dev/null 2>&1
  done
  for tag in cols_kernel rows_fwd_kernel rows_inv_kernel gather_update_kernel spread_kernel attraction_kernel; do
    python tools/ncu_summary.py /tmp/f_k${k}_$tag.ncu-rep
  done > gpurun_out/final_ncu_c4_k${k}_summary.txt 2>&1
  for tag in cols_kernel rows_fwd_kernel rows_inv_kernel gather_update_kernel spread_kernel attraction_kernel; do
    ncu -i /tmp/f_k${k}_$tag.ncu-rep --page raw --csv 2>/dev/null
  done > gpurun_out/final_ncu_k${k}_raw.csv
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 240 --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-exact --no-e2e \
  --no-cpu-baseline --no-full > /dev/null 2>&1
ls -la gpurun_out | tail -12
