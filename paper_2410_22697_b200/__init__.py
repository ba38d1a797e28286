"""B200-native halo feature pipeline of arXiv 2410.22697 (MassiveGNN prefetch + eviction).

The product is libmgnn.so (sm_100a CUDA kernels behind the C ABI in
include/mgnn.h); `pipeline` is its thin Python front-end.  There is no CPU
fallback: if the library is missing, `pipeline.Context` raises.
"""
from .pipeline import Context, alpha_default, build_context, device_view, exchange_tables  # noqa: F401

__all__ = ["Context", "alpha_default", "build_context", "device_view", "exchange_tables"]
