# ncu --set full of the register column kernel (TFDP_COLS=reg, C4, k = 1), the A/B variant of DESIGN §6
mkdir -p gpurun_out
TFDP_COLS=reg timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cols_reg_kernel" -s 1 -c 1 -o /tmp/creg -f python tools/fft_iter.py 1 8 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/creg.ncu-rep > gpurun_out/creg_summary.txt 2>&1
ncu -i /tmp/creg.ncu-rep --page raw --csv > gpurun_out/creg_raw.csv 2>/dev/null
ncu -i /tmp/creg.ncu-rep --page source --csv > gpurun_out/creg_source.csv 2>/dev/null
cat gpurun_out/creg_summary.txt
