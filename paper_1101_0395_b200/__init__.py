"""B200-native hot path of Celebi's fast exact k-means colour quantiser
(arXiv 1101.0395): unique-colour histogram, weighted sort-means Lloyd
iterations with exact integer centroid updates, and pixel mapping + MSE, as
hand-written sm_100a CUDA kernels behind a C-ABI (include/cqg.h, libcqg.so).

`quant` mirrors the reference's quant:: API; `cabi` is the ctypes binding.
"""
from . import cabi  # noqa: F401

__all__ = ["cabi", "quant", "synth"]
