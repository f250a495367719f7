"""Philox4x32-10 (Salmon et al., SC'11) and the position-keyed counter map.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper does not name an RNG for stochastic rounding (reading R3 in
DESIGN.md).  This build uses Philox4x32-10 keyed by the 64-bit seed, with the
counter keyed by the element's *position*, so codes never depend on launch
shape, sharding, or on whether a token was quantized by prefill or decode:

    key   = (seed & 0xffffffff, seed >> 32)
    ctr   = (n & 0xffffffff, n >> 32, rng_id, (layer << 16) | (tag << 12) | head)
    u     = (out[w] >> 8) * 2^-24                     (24-bit uniform in [0,1))

with tag Q=0, K=1, V=2, P=3 and, for an element at position t, channel c:
    K, Q : n = (t*d + c) >> 2,   w = c & 3      (4 consecutive channels / call)
    V    : n = (t >> 2)*d + c,   w = t & 3      (4 consecutive tokens / call)
    P    : n = (i << 30) | (t >> 2), w = t & 3  (query position i, key position t < 2^32;
                                                4 consecutive keys / call; head = query head)
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = 0xFFFFFFFF

TAG_Q, TAG_K, TAG_V, TAG_P = 0, 1, 2, 3


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32 with 10 rounds.  All args: uint32-valued arrays
    (or ints).  Returns four uint64 arrays holding the 32-bit output words."""
    c0 = np.asarray(c0, dtype=np.uint64)
    c1 = np.asarray(c1, dtype=np.uint64)
    c2 = np.asarray(c2, dtype=np.uint64)
    c3 = np.asarray(c3, dtype=np.uint64)
    k0 = np.asarray(k0, dtype=np.uint64)
    k1 = np.asarray(k1, dtype=np.uint64)
    m = np.uint64(MASK)
    for r in range(10):
        if r:  # key schedule: bump between rounds
            k0 = (k0 + np.uint64(W0)) & m
            k1 = (k1 + np.uint64(W1)) & m
        p0 = np.uint64(M0) * c0          # < 2^64: exact in uint64
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & m
        hi1, lo1 = p1 >> np.uint64(32), p1 & m
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & m, lo1, (hi0 ^ c3 ^ k1) & m, lo0
    return c0, c1, c2, c3


def uniform24(word) -> np.ndarray:
    """24-bit uniform in [0,1) from a 32-bit Philox word (exact in fp32)."""
    w = np.asarray(word, dtype=np.uint64) >> np.uint64(8)
    return (w.astype(np.float64) * 2.0 ** -24).astype(np.float32)


def stream_word(seed, rng_id, layer, tag, head):
    """The counter word c3 and key for one (request, layer, tag, head) stream."""
    c3 = ((int(layer) & 0xFFFF) << 16) | ((int(tag) & 0xF) << 12) | (int(head) & 0xFFF)
    return c3, int(seed) & MASK, (int(seed) >> 32) & MASK


def uniforms(seed, rng_id, layer, tag, head, n, w) -> np.ndarray:
    """u for elements with Philox block index n (int array) and word w."""
    c3, k0, k1 = stream_word(seed, rng_id, layer, tag, head)
    n = np.asarray(n, dtype=np.uint64)
    out = philox4x32_10(n & np.uint64(MASK), n >> np.uint64(32),
                        np.uint64(int(rng_id) & MASK), np.uint64(c3), k0, k1)
    w = np.asarray(w)
    word = np.where(w == 0, out[0], np.where(w == 1, out[1], np.where(w == 2, out[2], out[3])))
    return uniform24(word)


def uniforms_rowwise(seed, rng_id, layer, tag, head, positions, d) -> np.ndarray:
    """K / Q stream: u[t, c] for tokens at `positions` (1-D), channels 0..d-1."""
    t = np.asarray(positions, dtype=np.uint64)[:, None]
    c = np.arange(d, dtype=np.uint64)[None, :]
    n = (t * np.uint64(d) + c) >> np.uint64(2)
    return uniforms(seed, rng_id, layer, tag, head, n, (c & np.uint64(3)).astype(np.int64))


def uniforms_colwise(seed, rng_id, layer, head, positions, d) -> np.ndarray:
    """V stream: u[t, c] for tokens at `positions` (1-D), channels 0..d-1."""
    t = np.asarray(positions, dtype=np.uint64)[:, None]
    c = np.arange(d, dtype=np.uint64)[None, :]
    n = (t >> np.uint64(2)) * np.uint64(d) + c
    return uniforms(seed, rng_id, layer, TAG_V, head, n, (t & np.uint64(3)).astype(np.int64))


def uniforms_p(seed, rng_id, layer, head, qpos, keys) -> np.ndarray:
    """P stream (stochastic rounding of P, reading R6's selectable mode): u[r, t] for query
    rows at positions `qpos` (1-D) and key positions `keys` (1-D); `head` = the global
    query head.  Position-keyed like K/Q/V, so codes do not depend on tiling or on whether
    a row is a prefill row or a decode step."""
    i = np.asarray(qpos, dtype=np.uint64)[:, None]
    t = np.asarray(keys, dtype=np.uint64)[None, :]
    n = (i << np.uint64(30)) | (t >> np.uint64(2))
    return uniforms(seed, rng_id, layer, TAG_P, head, n, (t & np.uint64(3)).astype(np.int64))
