# A/B of the P = 2048 row-pass register cap (blocks per SM); variants built with
# -DTFDP_ROWS_MINB2048=<mb> into paper_2303_03964_b200/libtfdp_rmb<mb>.so
mkdir -p gpurun_out
for v in base rmb5 rmb6 base; do
  lib=paper_2303_03964_b200/libtfdp_$v.so; [ $v = base ] && lib=paper_2303_03964_b200/libtfdp.so
  echo "=== $v" >> gpurun_out/rows_ab.log
  TFDP_LIB_PATH=$lib timeout 300 python tools/kprof.py C4 20 2>&1 | grep "^k=1" >> gpurun_out/rows_ab.log
done
for v in rmb5 rmb6; do
  TFDP_LIB_PATH=paper_2303_03964_b200/libtfdp_$v.so timeout 300 python -m pytest tests/test_gpu_fft.py -m gpu -x -q 2>&1 | tail -1 >> gpurun_out/rows_ab.log
done
