"""B200-native t-FDP force step (arXiv 2303.03964): exact all-pairs and interpolation/FFT
repulsion, CSR attraction and the position update, behind the C ABI of include/tfdp.h
(libtfdp.so, sm_100a kernels).  This package is the product path; it never imports the
test oracle."""
from .tfdp import Dist, Layout, Params, csr_build, nccl_unique_id, shard_range  # noqa: F401
from ._lib import TfdpError, declared_symbols, lib  # noqa: F401
