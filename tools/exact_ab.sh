# A/B of exact-kernel variants (developer tool, under gpurun): micro-benchmark, then the
# bench's C5 exact leg with each variant library.
[ -n "$MB" ] && ./tools/mb_exact > gpurun_out/mb_exact.txt 2>&1
for v in "$@"; do
  lib=$PWD/paper_2303_03964_b200/libtfdp_$v.so
  [ "$v" = "default" ] && lib=$PWD/paper_2303_03964_b200/libtfdp.so
  TFDP_LIB_PATH=$lib python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/exact_ab_$v.json 2> gpurun_out/exact_ab_$v.err
done
