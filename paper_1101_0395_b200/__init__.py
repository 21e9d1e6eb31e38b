"""B200-native hot path of Celebi's fast exact k-means colour quantiser
(arXiv 1101.0395): unique-colour histogram, weighted sort-means Lloyd
iterations with exact integer centroid updates, and pixel mapping + MSE, as
hand-written sm_100a CUDA kernels behind a C-ABI (include/cqg.h, libcqg.so).

`quant` mirrors the reference's quant:: API; `cabi` is the ctypes binding.
"""
import os as _os

# Several library contexts on one GPU (a batch of images quantized side by side)
# put 3 streams each on the device; with the driver's default of 8 hardware
# queues the streams alias and serialise (cfg2 batch of 16: 493 -> 668 MPix/s
# with 32). Read by the driver when the CUDA context is created, so it has to
# be in the environment before the first CUDA call of the process.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import cabi  # noqa: F401,E402

__all__ = ["cabi", "quant", "synth"]
