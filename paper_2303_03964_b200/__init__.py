"""B200-native t-FDP force step (arXiv 2303.03964): exact all-pairs and interpolation/FFT
repulsion, CSR attraction and the position update, behind the C ABI of include/tfdp.h
(libtfdp.so, sm_100a kernels).  This package is the product path; it never imports the
test oracle."""
from .tfdp import (  # noqa: F401
    Dist, Layout, Params, csr_build, group_forces, group_step, nccl_unique_id, shard_range,
    slab_plan,
)
from ._lib import TfdpError, declared_symbols, lib  # noqa: F401
