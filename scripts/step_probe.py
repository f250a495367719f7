"""C2 prefill step decomposition: ingest alone, attention alone, the two back to back
(stream order), and hack_prefill_attention (attention a programmatic dependent of the
ingest).  L2 flushed before every timed call, CUDA events on the launching stream."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_03589_b200 import hack as h  # noqa: E402

L, Hq, Hkv = 4096, 32, 8
cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, out_fp32=False)
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((L, Hq, 128), generator=g, device="cuda").half()
k = torch.randn((L, Hkv, 128), generator=g, device="cuda").half()
v = torch.randn((L, Hkv, 128), generator=g, device="cuda").half()
cache = h.KVCache.allocate(cfg, 1, L // 64)
cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
sl = torch.zeros(1, dtype=torch.int32, device="cuda")
out = torch.empty((L, Hq, 128), dtype=torch.float16, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ops = 2 * 2 * 128 * (L * (L + 1) // 2) * Hq


def timed(fn, n=20, warm=3):
    ts = []
    for it in range(n + warm):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if it >= warm:
            ts.append(a.elapsed_time(b))
    ts.sort()
    return sum(ts) / len(ts), ts[len(ts) // 2]


cases = {
    "ingest": lambda: h.cache_ingest(cfg, k, v, cu, sl, L, cache),
    "attention_cached": lambda: h.prefill_attention_cached(cfg, q, cu, sl, L, cache, out),
    "ingest+attention (stream order)": lambda: (h.cache_ingest(cfg, k, v, cu, sl, L, cache),
                                                h.prefill_attention_cached(cfg, q, cu, sl, L, cache, out)),
    "prefill_attention (PDL)": lambda: h.prefill_attention(cfg, q, k, v, cu, sl, L, cache, out),
}
for name, fn in cases.items():
    avg, med = timed(fn)
    print(f"{name:34s} avg {avg * 1e3:8.1f} us  median {med * 1e3:8.1f} us  ({ops / avg / 1e9:6.1f} TOPS)")
