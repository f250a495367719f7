"""Prefill attention TOPS for shapes of equal algorithmic work (L^2 H_q fixed): separates the
per-CTA fixed costs (prologue, pipeline fill / drain) from the per-tile cost."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_03589_b200 import hack as h  # noqa: E402

shapes = [(4096, 32, 8), (8192, 8, 4), (16384, 2, 1), (2048, 128, 32)]
for L, Hq, Hkv in shapes:
    cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv)
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((L, Hq, 128), generator=g, device="cuda").half()
    k = torch.randn((L, Hkv, 128), generator=g, device="cuda").half()
    v = torch.randn((L, Hkv, 128), generator=g, device="cuda").half()
    cache = h.KVCache.allocate(cfg, 1, L // 64)
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    sl = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty((L, Hq, 128), dtype=torch.float16, device="cuda")
    h.cache_ingest(cfg, k, v, cu, sl, L, cache)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(8):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.prefill_attention_cached(cfg, q, cu, sl, L, cache, out)
        b.record()
        b.synchronize()
        if it >= 3:
            ts.append(a.elapsed_time(b))
    ms = sum(ts) / len(ts)
    ops = 2 * 2 * 128 * (L * (L + 1) // 2) * Hq
    print(f"L={L:6d} Hq={Hq:3d} Hkv={Hkv:2d}: {ms:.4f} ms  {ops / ms / 1e9:.1f} TOPS")
