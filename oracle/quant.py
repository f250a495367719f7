"""Partitioned asymmetric b-bit quantization and bit packing.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper, §5.2: "In each partition i, the method identifies the minimum
(min_i) and maximum (max_i) values ... computes the scale=(max_i-min_i)/(2^2-1).
Each original value x in a partition is quantized to an integer
x'=round((x-min_i)/scale).  The stochastic rounding round(*) rounds * to
floor(*) with probability (ceil(*)-*)/(ceil(*)-floor(*)) and to ceil(*)
otherwise."  (The printed probability has an unbalanced parenthesis; reading
R1: standard unbiased SR.)

Readings used here:
  R1  SR: c = floor(y) + [u < y - floor(y)], u a 24-bit uniform (bias <= 2^-24).
  R4  K/V meta is stored in FP16: m16 = fp16(lo), s16 = fp16(fp32(hi-lo)/(2^b-1));
      codes are computed against the stored fp16 (m, s).  Q/P meta is fp32.
  R5  scale == 0  ->  every code 0.
  R17 RN is round-half-to-even.
The code-producing arithmetic is specified in fp32 with no contraction, so the
CUDA path can reproduce every code bit-exactly:
      y = fp32( fp32(x - m) * fp32(1/s) ),   codes clamped to [0, 2^b-1].
Sums are exact integers.
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


def partition_stats(x: np.ndarray, bits: int, meta: str = "fp16"):
    """min and scale of each partition (last axis).  Returns float32 (m, s)
    (fp16-representable when meta == 'fp16')."""
    x = np.asarray(x, dtype=F32)
    lo = x.min(axis=-1)
    hi = x.max(axis=-1)
    qmax = F32((1 << bits) - 1)
    s32 = ((hi - lo).astype(F32) / qmax).astype(F32)          # fp32(fp32(hi-lo)/(2^b-1))
    if meta == "fp16":
        m = lo.astype(np.float16).astype(F32)
        s = s32.astype(np.float16).astype(F32)
    elif meta == "fp32":
        m, s = lo.astype(F32), s32
    else:
        raise ValueError(meta)
    return m, s


def quantize(x: np.ndarray, bits: int, meta: str, rnd: str, u: np.ndarray | None = None):
    """Quantize each partition (the LAST axis of x) with its own (m, s).

    x    : float32 values (fp16-exact for K/V/Q), shape [..., Pi]
    bits : code width b (2, 4 or 8)
    meta : 'fp16' (stored K/V) or 'fp32' (transient Q/P)
    rnd  : 'sr' (stochastic, needs u of x's shape) or 'rn' (nearest-even)
    Returns codes uint8 [..., Pi], m float32 [...], s float32 [...], sums int64 [...]
    """
    x = np.asarray(x, dtype=F32)
    m, s = partition_stats(x, bits, meta)
    qmax = (1 << bits) - 1
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = (F32(1.0) / s).astype(F32)                         # fp32(1/s)
        y = ((x - m[..., None]).astype(F32) * inv[..., None]).astype(F32)
    if rnd == "rn":
        c = np.rint(y)                                           # half-to-even
    elif rnd == "sr":
        if u is None or u.shape != x.shape:
            raise ValueError("stochastic rounding needs u with x's shape")
        fl = np.floor(y)
        frac = (y - fl).astype(F32)                              # exact
        c = fl + (np.asarray(u, dtype=F32) < frac)
    else:
        raise ValueError(rnd)
    zero = (s == 0)[..., None]
    c = np.where(zero | ~np.isfinite(y), 0.0, c)
    codes = np.clip(c, 0, qmax).astype(np.uint8)
    sums = codes.astype(np.int64).sum(axis=-1)
    return codes, m, s, sums


def dequantize(codes, m, s) -> np.ndarray:
    """x_hat = s * x' + m, fp64."""
    return np.asarray(s, np.float64)[..., None] * codes.astype(np.float64) + \
        np.asarray(m, np.float64)[..., None]


def sum_width_bits(bits: int, partition: int) -> int:
    """Storage for a code sum: b + ceil(log2 Pi) bits, rounded to a byte
    or to INT16 when it does not fit 8 bits."""
    need = bits + int(np.ceil(np.log2(partition)))
    return 8 if need <= 8 else 16


def pack(codes: np.ndarray, bits: int) -> np.ndarray:
    """Pack codes along the last axis LSB-first: the first logical code sits in
    the least-significant bits of its byte ([0,1,2,3] -> 228)."""
    codes = np.asarray(codes, dtype=np.uint8)
    if bits == 8:
        return codes.copy()
    per = 8 // bits
    n = codes.shape[-1]
    if n % per:
        raise ValueError("length must be a multiple of codes-per-byte")
    g = codes.reshape(codes.shape[:-1] + (n // per, per)).astype(np.uint32)
    out = np.zeros(g.shape[:-1], dtype=np.uint32)
    for j in range(per):
        out |= g[..., j] << np.uint32(j * bits)
    return out.astype(np.uint8)


def unpack(packed: np.ndarray, bits: int, n: int) -> np.ndarray:
    packed = np.asarray(packed, dtype=np.uint8)
    if bits == 8:
        return packed[..., :n].copy()
    per = 8 // bits
    mask = (1 << bits) - 1
    out = np.stack([(packed >> (j * bits)) & mask for j in range(per)], axis=-1)
    return out.reshape(packed.shape[:-1] + (packed.shape[-1] * per,))[..., :n].astype(np.uint8)
