# A/B of the P = 4096 / 6144 row-pass register caps (k = 2 / 3): variant built with
# -DTFDP_ROWS_MINB4096=3 -DTFDP_ROWS_MINB6144=4 into paper_2303_03964_b200/libtfdp_rmbx.so
mkdir -p gpurun_out
for v in base rmbx base rmbx; do
  lib=paper_2303_03964_b200/libtfdp_$v.so; [ $v = base ] && lib=paper_2303_03964_b200/libtfdp.so
  echo "=== $v" >> gpurun_out/rows_ab23.log
  TFDP_LIB_PATH=$lib timeout 300 python tools/kprof.py C4 20 2>&1 | grep "^k=[23]" >> gpurun_out/rows_ab23.log
done
