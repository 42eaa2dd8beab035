"""B200-native abstract rendering of Gaussian splats (AbstractSplat, arXiv 2503.00308).

The compute path is libabsplat.so (CUDA, sm_100a); this package is its thin ctypes binding
(api.Context, same names as the C ABI in include/absplat.h) plus the tile-sharding driver
over torch.distributed (dist.py).
"""
from .api import AbsplatError, Context, as_lpt_assign, as_untile, as_version  # noqa: F401
from ._abi import AS_ASYNC, AS_PTR_DEVICE, LIB_PATH  # noqa: F401
