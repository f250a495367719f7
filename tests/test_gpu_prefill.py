"""GPU parity: homomorphic prefill (a1-a7) through the C ABI vs the oracle.

Bit-exact: page bytes (K/V codes, fp16 meta, sums), FP16 tail, seq_lens.
Outputs: row-relative error <= 1e-3 (north star, R18) with every P-code mismatch a
near-tie."""
import numpy as np
import pytest
import torch

import hack_inputs
from oracle import attention as att

from .gpu_util import (ROW_TOL, acc_buffers, check_acc, check_pcodes, compare_pages, gpu_cfg, hk, make_cache,
                       row_rel_err)

pytestmark = pytest.mark.gpu


def run_prefill(ocfg, prompts, dist="normal", seed=11, rng_ids=None, debug=True, acc_head=-1):
    """prompts: list of lengths (one request each).  Runs the PRODUCTION call
    (hack_prefill_attention, no debug pointers), then -- with debug -- the debug
    instantiation on the same cache (hack_prefill_attention_cached with P codes and MMA
    accumulator dumps, all heads or only `acc_head`); the two outputs must be bit-identical.
    Returns the production out [T,Hq,d], pcodes, cache, per-request inputs, cu, slots, rng
    ids and the accumulator dumps (form, qk, pv) or None."""
    h = hk()
    cfg = gpu_cfg(ocfg)
    reqs = [hack_inputs.qkv(seed + i, L, ocfg.Hq, ocfg.Hkv, dist=dist, partition=ocfg.Pi, kv_bits=ocfg.bits)
            for i, L in enumerate(prompts)]
    q = np.concatenate([r[0] for r in reqs]); k = np.concatenate([r[1] for r in reqs])
    v = np.concatenate([r[2] for r in reqs])
    cu = np.concatenate([[0], np.cumsum(prompts)]).astype(np.int32)
    maxL = max(prompts)
    B = len(prompts)
    cache = make_cache(cfg, max_reqs=B + 1, max_len=maxL, seed=seed)
    slots = np.arange(B, dtype=np.int32)[::-1].copy()          # non-trivial slot mapping
    rid = np.array(rng_ids if rng_ids is not None else [1000 + i for i in range(B)], np.uint32)
    cache.rng_ids[torch.from_numpy(slots).long()] = torch.from_numpy(rid.view(np.int32)).cuda()
    out = torch.zeros((q.shape[0], ocfg.Hq, 128), dtype=torch.float32, device="cuda")
    stride = (maxL + ocfg.Pi - 1) // ocfg.Pi * ocfg.Pi
    qg, cug, slg = torch.from_numpy(q).cuda(), torch.from_numpy(cu).cuda(), torch.from_numpy(slots).cuda()
    h.prefill_attention(cfg, qg, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), cug, slg, maxL, cache, out)
    pc, acc = None, None
    if debug:
        pc = torch.zeros((q.shape[0], ocfg.Hq, stride), dtype=torch.uint8, device="cuda")
        form = h.debug_acc_form(cfg, "prefill")
        qk = pv = None
        if form != h.ACC_NONE:
            qk, pv = acc_buffers(q.shape[0], ocfg.Hq if acc_head < 0 else 1, ocfg, stride)
        dout = torch.zeros_like(out)
        h.prefill_attention_cached(cfg, qg, cug, slg, maxL, cache, dout, debug_pcodes=pc, debug_qk=qk,
                                   debug_pv=pv, debug_head=acc_head)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int32), dout.view(torch.int32)), "production and debug outputs differ"
        if qk is not None:
            acc = (form, qk.cpu().numpy(), pv.cpu().numpy())
        pc = pc.cpu().numpy()
    torch.cuda.synchronize()
    return out.cpu().numpy(), pc, cache, reqs, cu, slots, rid, acc


def check_request(ocfg, i, out, pc, cache, reqs, cu, slots, rid, acc=None, rows=None, heads=None, acc_head=-1):
    """Parity protocol: pages bit-exact; every P-code mismatch a near-tie;
    plain row error <= 1e-3, else the oracle re-run with the GPU's P codes (which differ
    from its own only at near-ties) must be within 1e-3.  With `acc`, the kernel's QK / PV
    accumulators of the checked rows (every head, or acc_head) are bit-exact."""
    q, k, v = reqs[i]
    O, state, diag = att.prefill(ocfg, q, k, v, rng_id=int(rid[i]), rows=rows, heads=heads, keep_diag=True)
    compare_pages(cache, int(slots[i]), state)
    assert int(cache.seq_lens[int(slots[i])]) == q.shape[0]
    rows = np.arange(q.shape[0]) if rows is None else np.asarray(rows)
    if acc is not None:
        form, qk, pv = acc
        qc, _, _, qsum = att.quantize_q(ocfg, q[rows], rows, int(rid[i]))
        for hq in (range(ocfg.Hq) if acc_head < 0 else [acc_head]):
            hs = hq if acc_head < 0 else 0
            nq, npv = check_acc(form, ocfg, state, qc, qsum, rows, hq, qk[cu[i] + rows, hs], pv[cu[i] + rows, hs],
                                pc[cu[i] + rows, hq])
        print(f"req {i}: accumulators bit-exact ({nq} QK + {npv} PV per head)")
    Og = out[cu[i]:cu[i + 1]]
    nfull = q.shape[0] // ocfg.Pi
    flips, worst_plain, override = 0, 0.0, {}
    for hq in diag:
        err = row_rel_err(Og[rows, hq], O[rows, hq])
        worst_plain = max(worst_plain, float(err.max()))
        if pc is not None and nfull:
            g = pc[cu[i] + rows, hq, :nfull * ocfg.Pi]
            flips += check_pcodes(g, diag[hq]["pcodes"], diag[hq]["py"], diag[hq]["pu"])
            override[hq] = g          # rows of `rows`, the order att.prefill computes them
    worst = worst_plain
    if worst_plain > ROW_TOL:
        assert pc is not None and flips > 0, f"row error {worst_plain:.3g} without any P-code flip"
        O2, _, _ = att.prefill(ocfg, q, k, v, rng_id=int(rid[i]), rows=rows, heads=list(override),
                               pcodes_override=override)
        worst = max(float(row_rel_err(Og[rows, hq], O2[rows, hq]).max()) for hq in override)
    print(f"req {i}: plain {worst_plain:.3g}, with GPU P codes {worst:.3g}, near-tie flips {flips}")
    assert worst <= ROW_TOL, f"max row-relative error {worst:.3g} (plain {worst_plain:.3g}, P flips {flips})"
    return worst, flips


@pytest.mark.parametrize("L", [512, 1, 63, 64, 65, 127, 500])
def test_c1_prefill_single_head(L):
    ocfg = att.Config(Hq=1, Hkv=1, Pi=64, bits=2)
    res = run_prefill(ocfg, [L])
    check_request(ocfg, 0, *res)


@pytest.mark.parametrize("Pi,bits", [(32, 2), (128, 2), (64, 4), (32, 4), (128, 4)])
def test_prefill_partition_and_bits(Pi, bits):
    ocfg = att.Config(Hq=4, Hkv=2, Pi=Pi, bits=bits)
    res = run_prefill(ocfg, [300])
    check_request(ocfg, 0, *res)


def test_prefill_gqa_varlen_batch():
    ocfg = att.Config(Hq=8, Hkv=2, Pi=64, bits=2, seed=12345, layer=3, head_base=1)
    res = run_prefill(ocfg, [200, 64, 333, 17])
    for i in range(4):
        check_request(ocfg, i, *res)


@pytest.mark.parametrize("dist", ["outlier", "constant", "grid"])
def test_prefill_adversarial_inputs(dist):
    ocfg = att.Config(Hq=2, Hkv=1, Pi=64, bits=2, kv_round="rn" if dist == "grid" else "sr")
    res = run_prefill(ocfg, [257], dist=dist)
    check_request(ocfg, 0, *res)


def test_prefill_rn_rounding():
    ocfg = att.Config(Hq=2, Hkv=2, Pi=64, bits=2, kv_round="rn", q_round="rn")
    res = run_prefill(ocfg, [190])
    check_request(ocfg, 0, *res)


def test_c2_full_size_sampled_rows():
    """Mistral-7B shape (32 Q / 8 KV heads, 4K tokens) at BASELINE size: all page bytes
    bit-exact, sampled query rows of sampled heads within tolerance."""
    ocfg = att.Config(Hq=32, Hkv=8, Pi=64, bits=2)
    res = run_prefill(ocfg, [4096], debug=True, acc_head=17)
    out, pc, cache, reqs, cu, slots, rid, acc = res
    rows = np.array([0, 1, 63, 64, 777, 2048, 3000, 4031, 4095])
    check_request(ocfg, 0, out, pc, cache, reqs, cu, slots, rid, acc, rows=rows, heads=[0, 5, 17, 31], acc_head=17)
    assert np.isfinite(out).all()


def test_prefill_simt_baseline_kernel(monkeypatch):
    # the CUDA-core baseline (used for Pi != 64) meets the same bar at Pi = 64
    monkeypatch.setenv("HACK_PREFILL_IMPL", "simt")
    ocfg = att.Config(Hq=4, Hkv=2, Pi=64, bits=2)
    res = run_prefill(ocfg, [300, 77])
    for i in range(2):
        check_request(ocfg, i, *res)


@pytest.mark.parametrize("L,Hq,Hkv,bits,Pi", [(300, 4, 2, 2, 64), (513, 8, 2, 4, 64), (64, 2, 1, 2, 64),
                                             (200, 4, 1, 2, 32), (300, 2, 1, 4, 128)])
def test_prefill_p_stochastic_rounding(L, Hq, Hkv, bits, Pi):
    """R6 selectable: the paper's stochastic rounding for P with the
    position-keyed P stream; near-ties are judged against the SR boundary y - u integer."""
    ocfg = att.Config(Hq=Hq, Hkv=Hkv, Pi=Pi, bits=bits, p_round="sr", seed=77)
    res = run_prefill(ocfg, [L])
    check_request(ocfg, 0, *res)


def test_prefill_p_sr_unsupported_on_the_cuda_core_kernel(monkeypatch):
    h = hk()
    monkeypatch.setenv("HACK_PREFILL_IMPL", "simt")   # the CUDA-core baseline has RN P only
    cfg = gpu_cfg(att.Config(Hq=2, Hkv=1, Pi=32, bits=2, p_round="sr"))
    cache = make_cache(cfg, 1, 64)
    q = torch.zeros((64, 2, 128), dtype=torch.float16, device="cuda")
    k = torch.zeros((64, 1, 128), dtype=torch.float16, device="cuda")
    cu = torch.tensor([0, 64], dtype=torch.int32, device="cuda")
    sl = torch.zeros(1, dtype=torch.int32, device="cuda")
    with pytest.raises(h.HackError) as e:
        h.prefill_attention(cfg, q, k, k, cu, sl, 64, cache, torch.zeros_like(q))
    assert e.value.status == h.ERR_UNSUPPORTED
    assert int(cache.seq_lens[0]) == 0                 # rejected before the ingest launch


@pytest.mark.parametrize("chunks", [1, 2, 4, 0])
def test_prefill_host_buffers_pipelined_equals_device_call(chunks):
    """hack_prefill_attention_host (host q/k/v/out, the e2e path): per query-head chunk
    uploads, attention of those heads (kc.hq_begin / hq_count) and downloads overlap on
    library streams; outputs and cache pages must equal hack_prefill_attention's bit for
    bit, for a ragged two-request batch and every chunking (0 = the default)."""
    h = hk()
    ocfg = att.Config(Hq=16, Hkv=4, Pi=64, bits=2, seed=23)
    cfg = gpu_cfg(ocfg)
    lens = [300, 77]
    T = sum(lens)
    q, k, v = hack_inputs.qkv(23, T, ocfg.Hq, ocfg.Hkv)
    cu = torch.tensor([0, lens[0], T], dtype=torch.int32)
    sl = torch.tensor([1, 0], dtype=torch.int32)
    caches = [make_cache(cfg, max_reqs=2, max_len=max(lens), seed=3) for _ in range(2)]
    for c in caches:   # (bytes neither call writes compare equal too)
        c.pages.zero_()
        c.v_tail.zero_()
    ref = torch.zeros((T, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
    h.prefill_attention(cfg, torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                        cu.cuda(), sl.cuda(), max(lens), caches[0], ref)
    qh, kh, vh = (torch.from_numpy(x).pin_memory() for x in (q, k, v))
    outh = torch.full((T, ocfg.Hq, 128), float("nan"), dtype=torch.float32).pin_memory()
    h.prefill_attention_host(cfg, qh, kh, vh, cu.pin_memory(), sl.pin_memory(), max(lens), caches[1], outh,
                             head_chunks=chunks)
    torch.cuda.synchronize()
    assert torch.equal(outh, ref.cpu())
    assert torch.equal(caches[0].pages, caches[1].pages)
    assert torch.equal(caches[0].v_tail, caches[1].v_tail)
    assert torch.equal(caches[0].seq_lens, caches[1].seq_lens)


@pytest.mark.parametrize("Pi,bits", [(64, 2), (32, 4), (128, 2)])
@pytest.mark.parametrize("L,chunks,extra", [(300, 0, 0), (1000, -3, 37), (64, 0, 0), (63, -2, 1), (1, 0, 0),
                                            (1000, -16, 0), (777, -1, 0)])
def test_prefill_host_position_streamed_equals_device_call(Pi, bits, L, chunks, extra):
    """hack_prefill_attention_host for ONE prompt streams it by position (head_chunks <= 0):
    K/V/Q rows [a, b) up, the ingest of those tokens (kc.tok_begin / tok_end), the attention of
    those query rows (kc.qt_begin / qt_count) and their output down, chunk after chunk.  Output,
    pages, FP16 tail and length must equal hack_prefill_attention's bit for bit, for ragged
    lengths, every partition size, chunk counts from 1 to more than the prompt has tiles, and
    a host bound max_seqlen above the length (extra)."""
    h = hk()
    ocfg = att.Config(Hq=16, Hkv=4, Pi=Pi, bits=bits, seed=29)
    cfg = gpu_cfg(ocfg)
    q, k, v = hack_inputs.qkv(29 + L, L, ocfg.Hq, ocfg.Hkv)
    cu = torch.tensor([0, L], dtype=torch.int32)
    sl = torch.tensor([1], dtype=torch.int32)
    ms = L + extra
    caches = [make_cache(cfg, max_reqs=2, max_len=ms, seed=5) for _ in range(2)]
    for c in caches:
        c.pages.zero_()
        c.v_tail.zero_()
    ref = torch.zeros((L, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
    h.prefill_attention(cfg, torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                        cu.cuda(), sl.cuda(), ms, caches[0], ref)
    qh, kh, vh = (torch.from_numpy(x).pin_memory() for x in (q, k, v))
    outh = torch.full((L, ocfg.Hq, 128), float("nan"), dtype=torch.float32).pin_memory()
    h.prefill_attention_host(cfg, qh, kh, vh, cu.pin_memory(), sl.pin_memory(), ms, caches[1], outh,
                             head_chunks=chunks)
    torch.cuda.synchronize()
    assert torch.equal(outh, ref.cpu())
    assert torch.equal(caches[0].pages, caches[1].pages)
    assert torch.equal(caches[0].v_tail, caches[1].v_tail)
    assert torch.equal(caches[0].seq_lens, caches[1].seq_lens)
