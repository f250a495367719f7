"""Probe: C3 decode at the per-rank shape of an N-GPU head-sharded run (B = 64 requests,
8K context, 8/N KV heads, 4 query heads each) on one GPU: time of append + attention
(CUDA graph of 20 steps over layer caches cycled past L2).  HACK_DECODE_GRID overrides
the persistent grid for the sweep."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_03589_b200 import hack as h

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
B, ctx, Hkv, G, Pi, steps = 64, 8192, 8 // N, 4, 64, 20
cfg = h.config(num_q_heads=Hkv * G, num_kv_heads=Hkv, partition=Pi, kv_bits=2, out_fp32=False, layer=1)
mp = (ctx + steps * 4 + Pi) // Pi + 1
layer_bytes = B * Hkv * mp * h.page_bytes(cfg)
nl = max(1, min(32, -(-2 * 126_000_000 // layer_bytes)))
slots = torch.arange(B, dtype=torch.int32, device="cuda")
caches = []
for _ in range(nl):
    c = h.KVCache.allocate(cfg, B, mp)
    caches.append(c)
    kk = torch.randn((B * ctx, Hkv, 128), device="cuda").half()
    cu = torch.arange(0, B + 1, dtype=torch.int32, device="cuda") * ctx
    h.cache_ingest(cfg, kk, kk, cu, slots, ctx, c)
qn = torch.randn((steps * 3, B, Hkv * G, 128), device="cuda").half()
kn = torch.randn((steps * 3, B, Hkv, 128), device="cuda").half()
out = torch.empty((B, Hkv * G, 128), dtype=torch.float16, device="cuda")
ws = torch.zeros(h.decode_workspace_size(cfg, B, ctx + steps * 4 + Pi), dtype=torch.uint8, device="cuda")
ML = ctx + steps * 4 + Pi
SEP = os.environ.get("PROBE_SEPARATE") == "1"   # append + attention as two calls (round-1 step)


def step(i):
    if SEP:
        h.decode_append(cfg, kn[i], kn[i], slots, caches[i % nl])
        h.decode_attention_cached(cfg, qn[i], slots, ML, caches[i % nl], out, workspace=ws)
    else:
        h.decode_attention(cfg, qn[i], kn[i], kn[i], slots, ML, caches[i % nl], out, workspace=ws)


for i in range(3):
    step(i)
torch.cuda.synchronize()
g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(g1):
    for i in range(steps):
        step(3 + i)
with torch.cuda.graph(g2):
    for i in range(steps):
        h.decode_attention_cached(cfg, qn[3 + i], slots, ML, caches[i % nl], out, workspace=ws)
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
e[0].record(); g1.replay(); e[1].record(); e[2].record(); g2.replay(); e[3].record()
torch.cuda.synchronize()
step, attn = e[0].elapsed_time(e[1]) / steps, e[2].elapsed_time(e[3]) / steps
gb = B * Hkv * ctx * 84 / (attn * 1e-3) / 1e9
print(json.dumps({"N": N, "step": "separate" if SEP else "fused", "grid": os.environ.get("HACK_DECODE_GRID", "default"), "step_us": round(step * 1e3, 1),
                  "attn_us": round(attn * 1e3, 1), "kv_gbs": round(gb, 1), "layers": nl}))
