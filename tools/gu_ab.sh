# Round-1 A/B of gather_update variants (libtfdp_<v>.so built with -D switches of that tree; the log is profiles/r1_gu_ab.txt)
mkdir -p gpurun_out
for v in base minb8 new; do
  lib=paper_2303_03964_b200/libtfdp_$v.so; [ $v = new ] && lib=paper_2303_03964_b200/libtfdp.so
  echo "=== $v" >> gpurun_out/ab.log
  TFDP_LIB_PATH=$lib timeout 300 python tools/kprof.py C4 20 >> gpurun_out/ab.log 2>&1
done
for v in base minb8 new; do
  lib=paper_2303_03964_b200/libtfdp_$v.so; [ $v = new ] && lib=paper_2303_03964_b200/libtfdp.so
  echo "=== bench $v" >> gpurun_out/ab.log
  TFDP_LIB_PATH=$lib timeout 300 python bench.py --no-exact 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e']['value'], d['kernels']['gather_update'])" >> gpurun_out/ab.log 2>&1
done
TFDP_LIB_PATH=paper_2303_03964_b200/libtfdp_minb8.so timeout 600 python -m pytest tests/test_gpu_fft.py tests/test_gpu_exact.py -m gpu -x -q > gpurun_out/ab_tests_minb8.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fft.py tests/test_gpu_exact.py -m gpu -x -q > gpurun_out/ab_tests_new.log 2>&1
