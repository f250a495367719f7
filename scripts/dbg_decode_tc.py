import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["HACK_DECODE_IMPL"] = sys.argv[1] if len(sys.argv) > 1 else "tc"
import numpy as np, torch
import hack_inputs
from paper_2502_03589_b200 import hack as h
from tests.gpu_util import make_cache
def run(prompts, Hq=4, Hkv=2, steps=70):
    cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, out_fp32=True)
    B = len(prompts); maxL = max(prompts) + steps
    cache = make_cache(cfg, max_reqs=B + 2, max_len=maxL, seed=1)
    slots = np.arange(B, dtype=np.int32) + 1
    for i, L in enumerate(prompts):
        q, k, v = hack_inputs.qkv(3 + i, L, Hq, Hkv)
        cu = torch.tensor([0, L], dtype=torch.int32, device="cuda"); sl = torch.tensor([slots[i]], dtype=torch.int32, device="cuda")
        out = torch.zeros((L, Hq, 128), dtype=torch.float32, device="cuda")
        h.prefill_attention(cfg, torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), cu, sl, L, cache, out)
    torch.cuda.synchronize()
    sl = torch.from_numpy(slots).cuda()
    qd, kd, vd = hack_inputs.decode_tokens(5, steps, B, Hq, Hkv)
    for s in range(steps):
        out = torch.zeros((B, Hq, 128), dtype=torch.float32, device="cuda")
        h.decode_attention(cfg, torch.from_numpy(qd[s]).cuda(), torch.from_numpy(kd[s]).cuda(), torch.from_numpy(vd[s]).cuda(), sl, maxL, cache, out)
        torch.cuda.synchronize()
    print("ok", prompts, flush=True)
cases = [((5,), 4, 1, 3), ((5,), 2, 1, 3), ((5,), 4, 2, 3), ((70,), 4, 2, 3), ((5,), 8, 2, 3)]
for p, Hq, Hkv, st in cases:
    print("run", p, Hq, Hkv, flush=True)
    run(list(p), Hq, Hkv, st)
