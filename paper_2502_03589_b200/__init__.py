"""paper_2502_03589_b200 -- B200-native (sm_100a) hot path of HACK (arXiv 2502.03589).

Homomorphic attention on per-partition asymmetric, stochastically rounded low-bit
KV codes: quantize_pack, prefill / decode attention, packed-KV send/recv.
Everything runs in libhack.so (csrc/, C ABI in include/hack.h); `hack` is a thin
ctypes binding.  There is no CPU fallback.
"""
from . import hack  # noqa: F401  (fails loudly if libhack.so is missing)
from .hack import *  # noqa: F401,F403
