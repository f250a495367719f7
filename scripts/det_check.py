"""Determinism probe: the same decode call repeated (production and debug instantiations)
on one cache must give bit-identical outputs (C4 70B shape, G = 8)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_03589_b200 import hack as h  # noqa: E402

L, HQ, HKV = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, 64, 8
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = h.config(num_q_heads=HQ, num_kv_heads=HKV, kv_bits=bits, out_fp32=True)
mp = (L + 2 + 63) // 64
cache = h.KVCache.allocate(cfg, 1, mp)
g = torch.Generator(device="cuda").manual_seed(1)
k = torch.randn((L, HKV, 128), generator=g, device="cuda").half()
v = torch.randn((L, HKV, 128), generator=g, device="cuda").half()
h.cache_ingest(cfg, k, v, torch.tensor([0, L], dtype=torch.int32, device="cuda"),
               torch.zeros(1, dtype=torch.int32, device="cuda"), L, cache)
q = torch.randn((1, HQ, 128), generator=g, device="cuda").half()
sl = torch.zeros(1, dtype=torch.int32, device="cuda")
outs, wss = [], []
nb = h.decode_workspace_size(cfg, 1, L + 2)
for dbg in (False, False, True, True, False):
    o = torch.zeros((1, HQ, 128), dtype=torch.float32, device="cuda")
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    if dbg:
        pc = torch.zeros((1, HQ, mp * 64), dtype=torch.uint8, device="cuda")
        h.decode_attention_cached(cfg, q, sl, L + 2, cache, o, workspace=ws, debug_pcodes=pc)
    else:
        h.decode_attention_cached(cfg, q, sl, L + 2, cache, o, workspace=ws)
    torch.cuda.synchronize()
    outs.append(o.cpu().numpy())
    wss.append(ws.cpu().numpy())
for i in range(1, len(wss)):
    w0, w1 = wss[0][256:].view(np.float32), wss[i][256:].view(np.float32)
    d = np.argwhere(w0.view(np.int32) != w1.view(np.int32))[:, 0]
    print("workspace", i, "differs at", d.size, "floats; first", d[:8], "vals", w0[d[:4]], w1[d[:4]],
          "slot offsets mod 130:", sorted(set((d % 130).tolist()))[:10])
for i in range(1, len(outs)):
    d = outs[i].view(np.int32) != outs[0].view(np.int32)
    print(i, "differs in", int(d.sum()), "elements; max |diff|", float(np.abs(outs[i] - outs[0]).max()),
          "rows", sorted(set(np.argwhere(d)[:, 1].tolist()))[:16])
