"""Byte image of the paged packed-KV layout.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written independently of
the CUDA path from the layout *specification* in DESIGN.md, so tests can
compare the GPU's page bytes with these bit-for-bit.

One page = Pi tokens of one (request, KV head) = exactly one V block.
Sections, in order, each starting at a 16-byte aligned offset:
  K_CODES  [Pi][d*b/8]      token-major; codes packed LSB-first along d
  K_META   [Pi][d/Pi][2]    fp16 (m, s) per (token, d-block)
  K_SUMS   [Pi][d/Pi]       u8, or u16 LE when b+ceil(log2 Pi) > 8
  V_CODES  [d][Pi*b/8]      channel-major; codes packed LSB-first along tokens
  V_META   [d][2]           fp16 (m, s) per channel
  V_SUMS   [d]              u8 / u16 LE
Unused bytes (alignment padding) are zero on the oracle side and are not
compared.  K rows of tokens not yet present and the V sections of the last,
partially filled page are undefined.
"""
from __future__ import annotations

import numpy as np

from . import quant


def _up16(x: int) -> int:
    return (x + 15) // 16 * 16


def layout(d: int, Pi: int, bits: int) -> dict:
    sw = quant.sum_width_bits(bits, Pi) // 8
    nb = d // Pi
    off = {}
    o = 0
    for name, size in (("k_codes", Pi * d * bits // 8), ("k_meta", Pi * nb * 4),
                       ("k_sums", Pi * nb * sw), ("v_codes", d * Pi * bits // 8),
                       ("v_meta", d * 4), ("v_sums", d * sw)):
        off[name] = (o, size)
        o = _up16(o + size)
    off["page_bytes"] = o
    off["sum_bytes"] = sw
    return off


def _f16_bytes(x) -> np.ndarray:
    return np.asarray(x, np.float32).astype(np.float16).view(np.uint8)


def _sum_bytes(s, sw: int) -> np.ndarray:
    s = np.asarray(s, np.int64)
    dt = np.uint8 if sw == 1 else np.dtype("<u2")
    return s.astype(dt).view(np.uint8)


def pack_request(state) -> tuple[np.ndarray, np.ndarray]:
    """Pages of one request: (bytes [npages, Hkv, page_bytes], defined-mask of
    the same shape).  npages = ceil(L / Pi)."""
    cfg = state.cfg
    d, Pi, b, Hkv = cfg.d, cfg.Pi, cfg.bits, cfg.Hkv
    a = state.arrays()
    L = a["kc"].shape[0]
    lay = layout(d, Pi, b)
    pb, sw = lay["page_bytes"], lay["sum_bytes"]
    npages = (L + Pi - 1) // Pi
    out = np.zeros((npages, Hkv, pb), np.uint8)
    mask = np.zeros((npages, Hkv, pb), bool)
    nb = d // Pi
    for p in range(npages):
        t0, t1 = p * Pi, min(L, (p + 1) * Pi)
        n = t1 - t0
        for h in range(Hkv):
            pg, mk = out[p, h], mask[p, h]
            o, sz = lay["k_codes"]
            row = d * b // 8
            pg[o:o + n * row] = quant.pack(a["kc"][t0:t1, h], b).reshape(-1)
            mk[o:o + n * row] = True
            o, sz = lay["k_meta"]
            mh = np.stack([a["km"][t0:t1, h], a["ks"][t0:t1, h]], -1)      # [n, nb, 2]
            pg[o:o + n * nb * 4] = _f16_bytes(mh).reshape(-1)
            mk[o:o + n * nb * 4] = True
            o, sz = lay["k_sums"]
            pg[o:o + n * nb * sw] = _sum_bytes(a["ksum"][t0:t1, h], sw).reshape(-1)
            mk[o:o + n * nb * sw] = True
            if p < a["vc"].shape[0]:                                        # committed V block
                o, sz = lay["v_codes"]
                pg[o:o + sz] = quant.pack(a["vc"][p, h], b).reshape(-1)
                mk[o:o + sz] = True
                o, sz = lay["v_meta"]
                pg[o:o + sz] = _f16_bytes(np.stack([a["vm"][p, h], a["vs"][p, h]], -1)).reshape(-1)
                mk[o:o + sz] = True
                o, sz = lay["v_sums"]
                pg[o:o + sz] = _sum_bytes(a["vsum"][p, h], sw).reshape(-1)
                mk[o:o + sz] = True
    return out, mask


def bytes_per_token(d: int, Pi: int, bits: int) -> float:
    """Packed K+V bytes per token per KV head (section padding included)."""
    return layout(d, Pi, bits)["page_bytes"] / Pi
