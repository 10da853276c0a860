# Where the side-stream attraction forks off the FFT chain (TFDP_ATTR_AT) and its grid
# (TFDP_ATTR_BLOCKS), C4 per-k wall; two alternating passes.
mkdir -p gpurun_out
: > gpurun_out/attr_ab.log
for rep in 1 2; do
  for v in "0 0" "1 0" "2 0" "0 296" "1 296" "0 148" "1 148" "1 592" "2 296"; do
    set -- $v
    echo "=== at=$1 blocks=$2" >> gpurun_out/attr_ab.log
    TFDP_ATTR_AT=$1 TFDP_ATTR_BLOCKS=$2 timeout 300 python tools/kprof.py C4 20 2>&1 | grep "k=" | sed 's/ ::.*//' >> gpurun_out/attr_ab.log
  done
done
cat gpurun_out/attr_ab.log
