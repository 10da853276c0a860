# Round-2 re-tune of the row passes' blocks per SM (register cap) at P = 2048 / 4096 / 6144:
# libtfdp_more.so (6 / 4 / 4) and libtfdp_less.so (4 / 2 / 2) against the default (5 / 3 / 3),
# alternating, plus TFDP_ROWS_RB=1 on the default library.
mkdir -p gpurun_out
: > gpurun_out/rows_minb_ab.log
for rep in 1 2; do
  for v in base more less rb1; do
    lib=paper_2303_03964_b200/libtfdp.so; env=""
    [ $v = more ] && lib=paper_2303_03964_b200/libtfdp_more.so
    [ $v = less ] && lib=paper_2303_03964_b200/libtfdp_less.so
    [ $v = rb1 ] && env="TFDP_ROWS_RB=1"
    echo "=== $v" >> gpurun_out/rows_minb_ab.log
    env $env TFDP_LIB_PATH=$lib timeout 300 python tools/kprof.py C4 20 2>&1 | grep "k=" >> gpurun_out/rows_minb_ab.log
  done
done
cat gpurun_out/rows_minb_ab.log
