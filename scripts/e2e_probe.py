"""C2 e2e (host buffers) per chunking (head chunks, or position streaming): hack_prefill_attention_host vs copies +
hack_prefill_attention in stream order."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_03589_b200 import hack as h  # noqa: E402

L, Hq, Hkv = 4096, 32, 8
cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, out_fp32=False)
g = torch.Generator().manual_seed(1)
qh = torch.randn((L, Hq, 128), generator=g).half().pin_memory()
kh = torch.randn((L, Hkv, 128), generator=g).half().pin_memory()
vh = torch.randn((L, Hkv, 128), generator=g).half().pin_memory()
outh = torch.empty((L, Hq, 128), dtype=torch.float16).pin_memory()
cuh = torch.tensor([0, L], dtype=torch.int32).pin_memory()
slh = torch.zeros(1, dtype=torch.int32).pin_memory()
cache = h.KVCache.allocate(cfg, 1, L // 64)
ws = torch.empty(h.prefill_host_workspace_size(cfg, 1, L), dtype=torch.uint8, device="cuda")
qd, kd, vd = torch.empty((L, Hq, 128), dtype=torch.float16, device="cuda"), torch.empty((L, Hkv, 128), dtype=torch.float16, device="cuda"), torch.empty((L, Hkv, 128), dtype=torch.float16, device="cuda")
od = torch.empty_like(qd)
cud, sld = cuh.cuda(), slh.cuda()
ops = 2 * 2 * 128 * (L * (L + 1) // 2) * Hq


def timed(fn, n=10, warm=3):
    ts = []
    for it in range(n + warm):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if it >= warm:
            ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts)


def serial():
    qd.copy_(qh, non_blocking=True); kd.copy_(kh, non_blocking=True); vd.copy_(vh, non_blocking=True)
    h.prefill_attention(cfg, qd, kd, vd, cud, sld, L, cache, od)
    outh.copy_(od, non_blocking=True)


ms = timed(serial)
print(f"copies + prefill_attention    {ms:.3f} ms  {ops / ms / 1e9:.1f} TOPS")
# head_chunks > 0: query-head chunks; <= 0: the prompt streamed by position (-n: n chunks, 0: 8)
for c in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "1,2,4,8,0,-4,-8,-12,-16".split(","))]:
    ms = timed(lambda: h.prefill_attention_host(cfg, qh, kh, vh, cuh, slh, L, cache, outh, workspace=ws, head_chunks=c))
    print(f"prefill_attention_host {c:+3d}     {ms:.3f} ms  {ops / ms / 1e9:.1f} TOPS")
