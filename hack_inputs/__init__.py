"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws fp16 Q/K/V
tensors (and decode-step tokens) from numpy's PCG64 with fixed seeds, in the
shapes of the paper's workloads.  Both `oracle/`
and the CUDA tests/bench import it; neither imports the other.

Distributions (input recipe):
  normal   : N(0, 1), cast to fp16 (the paper is FP16 throughout).
  outlier  : normal, with 8 channels per head scaled x10 (KV outlier channels).
  grid     : values on a per-partition 2-bit / 8-bit grid that hit both min and
             max in every partition, so quantization is exact (SURVEY c-5).
  constant : every element equal (degenerate partitions, scale = 0).
"""
from __future__ import annotations

import numpy as np

DATA_SEED = 20250205          # SURVEY d: data seed per (config, rank)
QUANT_SEED = 0x48414B         # "HAK": Philox key used by the benches

__all__ = ["DATA_SEED", "QUANT_SEED", "rng", "tensor", "qkv", "decode_tokens"]


def rng(seed: int, *salt: int) -> np.random.Generator:
    """A PCG64 generator keyed by (seed, *salt) -- independent streams per use."""
    return np.random.default_rng([int(seed) & 0xFFFFFFFF, *[int(s) & 0xFFFFFFFF for s in salt]])


def tensor(g: np.random.Generator, shape, dist: str = "normal", grid_bits: int = 2,
           partition: int = 64) -> np.ndarray:
    """Draw one fp16 tensor whose LAST axis is the head dimension."""
    shape = tuple(int(s) for s in shape)
    if dist == "normal":
        x = g.standard_normal(shape, dtype=np.float32)
    elif dist == "outlier":
        x = g.standard_normal(shape, dtype=np.float32)
        d = shape[-1]
        ch = g.choice(d, size=min(8, d), replace=False)
        x[..., ch] *= 10.0
    elif dist == "uniform":
        x = g.uniform(-1.0, 1.0, size=shape).astype(np.float32)
    elif dist == "constant":
        x = np.full(shape, np.float32(g.standard_normal()))
    elif dist == "grid":
        # Every partition (last axis, chunks of `partition`) takes values
        # lo + k * 2^-e with k in [0, 2^b-1] and hits both k=0 and k=2^b-1.
        q = (1 << grid_bits) - 1
        k = g.integers(0, q + 1, size=shape)
        kk = k.reshape(shape[:-1] + (shape[-1] // partition, partition))
        kk[..., 0] = 0
        kk[..., 1] = q
        k = kk.reshape(shape)
        step = np.float32(2.0 ** -3) if grid_bits <= 4 else np.float32(2.0 ** -7)
        lo = (g.integers(-8, 8, size=shape[:-1] + (shape[-1] // partition, 1)) *
              np.float32(0.25)).astype(np.float32)
        lo = np.repeat(lo, partition, axis=-1).reshape(shape)
        x = lo + k.astype(np.float32) * step
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    return x.astype(np.float16)


def qkv(seed: int, L: int, Hq: int, Hkv: int, d: int = 128, dist: str = "normal",
        partition: int = 64, kv_bits: int = 2):
    """Prompt tensors Q [L,Hq,d], K [L,Hkv,d], V [L,Hkv,d] (fp16, token-major)."""
    g = rng(seed, L, Hq, Hkv, d)
    qd = "grid" if dist == "grid" else dist
    q = tensor(g, (L, Hq, d), qd, grid_bits=8, partition=partition)
    k = tensor(g, (L, Hkv, d), dist, grid_bits=kv_bits, partition=partition)
    v = tensor(g, (L, Hkv, d), "normal" if dist == "grid" else dist, partition=partition)
    return q, k, v


def decode_tokens(seed: int, steps: int, B: int, Hq: int, Hkv: int, d: int = 128,
                  dist: str = "normal"):
    """Per-step decode inputs: q [steps,B,Hq,d], k/v [steps,B,Hkv,d] (fp16)."""
    g = rng(seed, 0xDEC0DE, steps, B, Hq, Hkv, d)
    q = tensor(g, (steps, B, Hq, d), dist)
    k = tensor(g, (steps, B, Hkv, d), dist)
    v = tensor(g, (steps, B, Hkv, d), dist)
    return q, k, v
