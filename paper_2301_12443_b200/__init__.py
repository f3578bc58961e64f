"""B200-native Pipe-BD blockwise-distillation hot path (arXiv 2301.12443).

Host core (profile / cost model / AHD partitioner / simulator) and the sm_100a
kernels + partition executor live in ``lib/libpbd.so``; this package is the
thin Python face over its C-ABI (include/pbd_capi.h, include/pbdk.h,
include/pbdx.h) plus the multi-GPU driver built on torch.distributed.
"""
__version__ = "0.1.0"
