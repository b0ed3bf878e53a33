"""B200-native XPipe hot path (arXiv 1911.04610): C-ABI library libxpipe.so + thin binding.

The product path is the CUDA library only.  Importing this package never imports oracle/.
"""
from .xpipe import (XPipe, XPipeError, adam_predict, sgd_predict, gemm_bf16, conv2d_bf16, linear_bf16, lib, SO_PATH,  # noqa: F401
                    exchange_blobs, connect_pipeline)

__all__ = ["XPipe", "XPipeError", "adam_predict", "sgd_predict", "gemm_bf16", "conv2d_bf16", "linear_bf16", "exchange_blobs", "connect_pipeline", "lib", "SO_PATH"]
