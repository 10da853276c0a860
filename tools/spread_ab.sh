#!/bin/bash
# A/B of the spread variants: per-node v4 REDs (warp-aggregated for
# k >= 2) vs the shared-memory privatised tile kernel, C4 input layout and a clustered
# layout, per-kernel times from tools/kprof.py.  Run on the GPU box from the repo root.
for lay in input blobs; do
  for mode in red tile; do
    echo "== spread=$mode layout=$lay"
    TFDP_SPREAD=$mode python tools/kprof.py C4 20 $lay
  done
done
