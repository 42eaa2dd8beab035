"""B200-native abstract rendering of Gaussian splats (AbstractSplat, arXiv 2503.00308).

The compute path is libabsplat.so (CUDA, sm_100a); this package is its thin ctypes binding
(api.Context, same names as the C ABI in include/absplat.h) plus the multi-GPU plumbing
(dist.py: the NCCL id handed to every rank over torch.distributed; the collective itself
runs inside the library).
"""
from .api import (AbsplatError, Context, as_lpt_assign, as_nccl_id, as_untile,  # noqa: F401
                  as_version)
from ._abi import AS_ASYNC, AS_PTR_DEVICE, LIB_PATH  # noqa: F401
