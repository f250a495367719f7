"""GPU parity of the "HACK/RQE" ablation mode.

With HACK_DECODE_NO_RQE set, decode append requantizes the partially filled last V
block at every step (the work requantization elimination removes): the T tokens of
the FP16 tail form one partition per (head, channel), quantized with the same
quantizer and position-keyed Philox counters as a flush.  The codes, meta and sums it
writes into the partial page's V section must equal the oracle's quantizer applied to
those T tokens; committed pages, the tail and the flush stay bit-exact (compare_pages)."""
import numpy as np
import pytest
import torch

import hack_inputs
from oracle import attention as att
from oracle import pages as opages
from oracle import philox, quant

from .gpu_util import compare_pages, gpu_cfg, hk, make_cache

pytestmark = pytest.mark.gpu


def check_partial_v(cache, slot, state, ocfg, rid):
    a = state.arrays()
    T = a["tail"].shape[0]
    if T == 0:
        return
    lay = opages.layout(128, ocfg.Pi, ocfg.bits)
    blk = state.nblocks
    pid = int(cache.block_table[slot, blk])
    pg = cache.pages[pid].cpu().numpy()                              # [Hkv, page_bytes]
    pos = blk * ocfg.Pi + np.arange(T)
    x = np.transpose(a["tail"].astype(np.float32), (1, 2, 0))        # [Hkv, d, T]
    for h in range(ocfg.Hkv):
        u = philox.uniforms_colwise(ocfg.seed, rid, ocfg.layer, ocfg.head_base + h, pos, 128).T
        codes, m, s, sums = quant.quantize(x[h], ocfg.bits, "fp16", "sr", u)
        o, sz = lay["v_codes"]
        raw = pg[h, o:o + sz].reshape(128, -1)                       # per channel, LSB-first
        per = 8 // ocfg.bits
        got = np.stack([(raw[:, t // per] >> ((t % per) * ocfg.bits)) & ((1 << ocfg.bits) - 1)
                        for t in range(T)], 1)
        bad = np.argwhere(got != codes)
        assert not len(bad), (f"head {h}: {len(bad)} codes differ (T={T}, blk={blk}), first {bad[:4].tolist()} "
                              f"got {got[tuple(bad[:4].T)]} want {codes[tuple(bad[:4].T)]}")
        o, sz = lay["v_meta"]
        meta = pg[h, o:o + sz].view(np.float16).reshape(128, 2).astype(np.float32)
        assert np.array_equal(meta[:, 0], m) and np.array_equal(meta[:, 1], s)
        o, sz = lay["v_sums"]
        sw = sz // 128
        gs = pg[h, o:o + sz].view(np.uint16 if sw == 2 else np.uint8).astype(np.int64)
        assert np.array_equal(gs, sums)


@pytest.mark.parametrize("bits", [2, 4])
def test_no_rqe_requantizes_partial_block(bits, monkeypatch):
    monkeypatch.setenv("HACK_DECODE_NO_RQE", "1")
    h = hk()
    ocfg = att.Config(Hq=4, Hkv=2, Pi=64, bits=bits, seed=19)
    cfg = gpu_cfg(ocfg)
    prompts, steps = [100, 63, 1], 70                                 # crosses one flush each
    B = len(prompts)
    cache = make_cache(cfg, max_reqs=B, max_len=max(prompts) + steps, seed=8)
    rid = np.array([900 + 11 * i for i in range(B)], np.uint32)
    cache.rng_ids[:B] = torch.from_numpy(rid.view(np.int32)).cuda()
    states = []
    for i, L in enumerate(prompts):
        _, k, v = hack_inputs.qkv(40 + i, L, 1, ocfg.Hkv)
        cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
        h.cache_ingest(cfg, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), cu,
                       torch.tensor([i], dtype=torch.int32, device="cuda"), L, cache)
        states.append(att.ingest_prompt(ocfg, k, v, rng_id=int(rid[i])))
    _, kd, vd = hack_inputs.decode_tokens(3, steps, B, ocfg.Hq, ocfg.Hkv)
    sl = torch.arange(B, dtype=torch.int32, device="cuda")
    for s in range(steps):
        h.decode_append(cfg, torch.from_numpy(kd[s]).cuda(), torch.from_numpy(vd[s]).cuda(), sl, cache)
        torch.cuda.synchronize()
        for i in range(B):
            states[i].append_k(kd[s, i][None])
            states[i].append_v(vd[s, i])
            if s % 7 == 0 or s == steps - 1:
                check_partial_v(cache, i, states[i], ocfg, int(rid[i]))
    for i in range(B):
        compare_pages(cache, i, states[i])
