# ncu --set full of the column pass at C4 k = 1, 2, 3 (summary, raw and source pages under gpurun_out/)
mkdir -p gpurun_out
for k in 1 2 3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^cols_kernel" -s 1 -c 1 -o /tmp/r2c_k$k -f python tools/fft_iter.py $k 8 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/r2c_k$k.ncu-rep > gpurun_out/r2_cols_k${k}_summary.txt 2>&1
  ncu -i /tmp/r2c_k$k.ncu-rep --page raw --csv > gpurun_out/r2_cols_k${k}_raw.csv 2>/dev/null
  ncu -i /tmp/r2c_k$k.ncu-rep --page source --csv > gpurun_out/r2_cols_k${k}_source.csv 2>/dev/null
done
cat gpurun_out/r2_cols_k*_summary.txt
