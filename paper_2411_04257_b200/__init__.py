"""B200-native LSHBloom hot path (arXiv 2411.04257).

``LSHBloom`` wraps the C-ABI in ``include/lshbloom.h`` (``liblshbloom.so``, hand-written CUDA
for sm_100a).  ``sharded`` adds the band-sharded multi-GPU layer (torch.distributed / NCCL).
"""
from ._native import EXPORTS, LSHBloom, LSHBloomError, load_library, optimal_params, plan  # noqa: F401

__all__ = ["LSHBloom", "LSHBloomError", "load_library", "EXPORTS", "optimal_params", "plan"]
