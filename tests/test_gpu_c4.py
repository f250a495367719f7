"""GPU parity at C4 (BASELINE configs[3]): Llama-3.1-70B-shaped attention -- 64 Q / 8 KV
heads (GQA group G = 8), d = 128, one 32K-token prompt, 2-bit and 4-bit K/V -- at full size
on one GPU (the 8-GPU layout gives every GPU one KV head, SURVEY e).

The oracle runs KV head 5 alone (head_base = 5 selects the same Philox streams, R3):
its page bytes must equal the GPU's bytes for that head, and sampled prefill rows plus two
decode steps of its 8 query heads must agree within 1e-3 (R18).  Prefill P codes are not
dumped at this size (the dump would be L x Hq x L bytes); rows this long are diffuse, so a
near-tie P-code flip moves a row by ~1e-6 and the plain error is asserted."""
import numpy as np
import pytest
import torch

import hack_inputs
from oracle import attention as att
from oracle import pages as opages

from .gpu_util import ROW_TOL, acc_buffers, check_acc, check_pcodes, gpu_cfg, hk, make_cache, row_rel_err

pytestmark = pytest.mark.gpu

L, HQ, HKV, G, HSEL = 32768, 64, 8, 8, 5


def compare_head_pages(cache, slot, state, head):
    ref, mask = opages.pack_request(state)                      # [npages, 1, page_bytes]
    bt = cache.block_table[slot, :ref.shape[0]].long()
    got = cache.pages[bt][:, head:head + 1].cpu().numpy()
    bad = (got != ref) & mask
    assert not bad.any(), f"{bad.sum()} page bytes differ for KV head {head}"
    T = state.arrays()["tail"].shape[0]
    if T:
        tail = cache.v_tail[slot, head, :T].cpu().numpy()
        assert np.array_equal(tail.view(np.uint16), state.arrays()["tail"][:, 0].view(np.uint16))


@pytest.mark.parametrize("bits", [2, 4])
def test_c4_long_prompt_one_kv_head(bits):
    h = hk()
    full = att.Config(Hq=HQ, Hkv=HKV, Pi=64, bits=bits, seed=7)
    one = att.Config(Hq=G, Hkv=1, Pi=64, bits=bits, seed=7, head_base=HSEL)
    cfg = gpu_cfg(full)
    q, k, v = hack_inputs.qkv(31, L, HQ, HKV)
    steps = 2
    cache = make_cache(cfg, max_reqs=1, max_len=L + steps, seed=4)
    rid = 4242
    cache.rng_ids[0] = rid
    sl = torch.zeros(1, dtype=torch.int32, device="cuda")
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    out = torch.zeros((L, HQ, 128), dtype=torch.float32, device="cuda")
    h.prefill_attention(cfg, torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                        cu, sl, L, cache, out)
    torch.cuda.synchronize()
    heads = slice(G * HSEL, G * (HSEL + 1))
    rows = np.array([0, 1, 63, 64, 4097, 16384, 30000, L - 1])
    O, state, _ = att.prefill(one, q[:, heads], k[:, HSEL:HSEL + 1], v[:, HSEL:HSEL + 1], rng_id=rid, rows=rows)
    compare_head_pages(cache, 0, state, HSEL)
    Og = out[torch.from_numpy(rows).cuda()][:, heads].cpu().numpy()
    err = row_rel_err(Og, O[rows]).max()
    print(f"C4 b={bits}: prefill sampled rows, max row error {err:.3g}")
    assert err <= ROW_TOL
    assert np.isfinite(out[::997].cpu().numpy()).all()

    qd, kd, vd = hack_inputs.decode_tokens(8, steps, 1, HQ, HKV)
    stride = (L + steps + 63) // 64 * 64
    form = h.debug_acc_form(cfg, "decode")   # decode_g8_kernel (b = 2) / decode_mma_kernel (b = 4)
    assert form != h.ACC_NONE
    for s in range(steps):
        # production instantiation first, then the debug one (P codes + MMA accumulators)
        dout = torch.zeros((1, HQ, 128), dtype=torch.float32, device="cuda")
        h.decode_attention(cfg, torch.from_numpy(qd[s]).cuda(), torch.from_numpy(kd[s]).cuda(),
                           torch.from_numpy(vd[s]).cuda(), sl, L + steps, cache, dout)
        pc = torch.zeros((1, HQ, stride), dtype=torch.uint8, device="cuda")
        qk, pv = acc_buffers(1, HQ, one, stride)
        ddbg = torch.zeros_like(dout)
        h.decode_attention_cached(cfg, torch.from_numpy(qd[s]).cuda(), sl, L + steps, cache, ddbg, debug_pcodes=pc,
                                  debug_qk=qk, debug_pv=pv)
        torch.cuda.synchronize()
        assert torch.equal(dout.view(torch.int32), ddbg.view(torch.int32)), "production and debug outputs differ"
        Od, diag = att.decode_step(state, qd[s, 0, heads], kd[s, 0, HSEL:HSEL + 1], vd[s, 0, HSEL:HSEL + 1],
                                   keep_diag=True)
        nf = state.nblocks * 64
        pcn = pc.cpu().numpy()[0, heads, :nf]
        for j in range(G):
            check_pcodes(pcn[j][None], diag[j]["pcodes"], diag[j]["py"])
        pos = state.length - 1
        qc, _, _, qsum = att.quantize_q(one, qd[s, 0, heads][None], np.array([pos]), rid)
        qkn, pvn = qk.cpu().numpy()[0, heads], pv.cpu().numpy()[0, heads]
        for j in range(G):
            check_acc(form, one, state, qc, qsum, [pos], j, qkn[j][None], pvn[j][None], pcn[j][None])
        derr = row_rel_err(dout.cpu().numpy()[0, heads], Od).max()
        if derr > ROW_TOL:
            O2, _ = att.decode_attend(state, qd[s, 0, heads], pcodes_override={j: pcn[j][None] for j in range(G)})
            derr = row_rel_err(dout.cpu().numpy()[0, heads], O2).max()
        print(f"C4 b={bits}: decode step {s}, max row error {derr:.3g}")
        assert derr <= ROW_TOL
    compare_head_pages(cache, 0, state, HSEL)
