# Developer profiling pass of the ibFFT path at C4 (run under gpurun): per-k timing, one
# ncu --set full capture per k of the hot kernels (summarised on the box, raw CSV kept), and
# the launch list of the bench command.
set -x
mkdir -p gpurun_out
python tools/kprof.py C4 20 > gpurun_out/kprof.txt 2>&1
for k in 1 2 3; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cols_kernel|rows_fwd|rows_inv|gather_update|spread_kernel|kspec|setup_kernel" -s 7 -c 7 -o /tmp/full_k$k -f python tools/fft_iter.py $k 8 > gpurun_out/ncu_full_k$k.log 2>&1
python tools/ncu_summary.py /tmp/full_k$k.ncu-rep > gpurun_out/ncu_full_k${k}_summary.txt 2>&1
ncu -i /tmp/full_k$k.ncu-rep --page raw --csv > gpurun_out/ncu_full_k${k}_raw.csv 2>/dev/null
done
[ "$1" = "nolaunch" ] || timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-exact --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
