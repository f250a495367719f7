"""The dequantize-first comparator (not the HACK path): hack_dequantize_cache
expands the same packed pages into dense fp16 K-hat / V-hat.  Bit-exact against the
oracle's codes and fp16 meta (fp16(m + s*c) with one fp32 rounding) and the FP16
last V block; attention over the expanded cache then matches the oracle's exact
attention on the same dequantized values."""
import numpy as np
import pytest
import torch

import hack_inputs
from oracle import attention as att

from .gpu_util import gpu_cfg, hk, make_cache

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bits", [2, 4])
def test_dequantize_cache_bit_exact(bits):
    h = hk()
    ocfg = att.Config(Hq=4, Hkv=2, Pi=64, bits=bits, seed=21)
    cfg = gpu_cfg(ocfg)
    prompts, steps = [200, 64, 130], 3
    maxL = max(prompts) + steps
    B = len(prompts)
    cache = make_cache(cfg, max_reqs=B, max_len=maxL, seed=5)
    rid = np.array([300 + i for i in range(B)], np.uint32)
    cache.rng_ids[:B] = torch.from_numpy(rid.view(np.int32)).cuda()
    states = []
    for i, L in enumerate(prompts):
        _, k, v = hack_inputs.qkv(60 + i, L, 1, ocfg.Hkv, partition=64, kv_bits=bits)
        h.cache_ingest(cfg, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                       torch.tensor([0, L], dtype=torch.int32, device="cuda"),
                       torch.tensor([i], dtype=torch.int32, device="cuda"), L, cache)
        states.append(att.ingest_prompt(ocfg, k, v, rng_id=int(rid[i])))
    _, kd, vd = hack_inputs.decode_tokens(6, steps, B, ocfg.Hq, ocfg.Hkv)
    sl = torch.arange(B, dtype=torch.int32, device="cuda")
    for s in range(steps):
        h.decode_append(cfg, torch.from_numpy(kd[s]).cuda(), torch.from_numpy(vd[s]).cuda(), sl, cache)
        for i in range(B):
            states[i].append_k(kd[s, i][None])
            states[i].append_v(vd[s, i])
    kh = torch.zeros((B, ocfg.Hkv, maxL, 128), dtype=torch.float16, device="cuda")
    vh = torch.zeros_like(kh)
    h.dequantize_cache(cfg, sl, maxL, cache, kh, vh)
    torch.cuda.synchronize()
    kh, vh = kh.cpu().numpy(), vh.cpu().numpy()
    for i in range(B):
        a = states[i].arrays()
        L = a["kc"].shape[0]
        beta = np.arange(128) // 64
        kref = (a["km"][:, :, beta] + a["ks"][:, :, beta] * a["kc"].astype(np.float32)).astype(np.float16)
        assert np.array_equal(kh[i, :, :L].transpose(1, 0, 2).view(np.uint16), kref.view(np.uint16))
        nb, T = a["vc"].shape[0], a["tail"].shape[0]
        vq = (a["vm"][..., None] + a["vs"][..., None] * a["vc"].astype(np.float32)).astype(np.float16)
        vref = np.concatenate([vq.transpose(0, 3, 1, 2).reshape(nb * 64, ocfg.Hkv, 128), a["tail"]], 0)
        assert vref.shape[0] == L
        assert np.array_equal(vh[i, :, :L].transpose(1, 0, 2).view(np.uint16), vref.view(np.uint16))
        # attention over the expanded cache (fp32 here) == exact attention on the same values
        q = hack_inputs.decode_tokens(7, 1, 1, ocfg.Hq, ocfg.Hkv)[0][0]
        O = att.exact_attention(q, kref, vref, causal=False)
        kt = torch.from_numpy(kh[i, :, :L]).float().repeat_interleave(ocfg.G, 0)
        vt = torch.from_numpy(vh[i, :, :L]).float().repeat_interleave(ocfg.G, 0)
        qt = torch.from_numpy(q[0].astype(np.float32))[:, None, :]
        og = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt)[:, 0].numpy()
        assert np.abs(og - O[0]).max() <= 1e-5 * max(1.0, np.abs(O[0]).max())
