"""GPU parity: decode append/flush (a8) and decode attention (a9) vs the oracle.

Summation elimination: the GPU never re-sums codes (it reads the cached sums).
Requantization elimination: the tail is FP16 until it reaches Pi, then flushed once;
committed pages are bit-stable.  Outputs within 1e-3 row-relative (R18)."""
import numpy as np
import pytest
import torch

import hack_inputs
from oracle import attention as att

from .gpu_util import (ROW_TOL, acc_buffers, check_acc, check_pcodes, compare_pages, gpu_cfg, gpu_pages_of, hk, make_cache,
                       row_rel_err)

pytestmark = pytest.mark.gpu


def substituted_err(state, q, gpu_pcodes, O_gpu, Hq):
    """Near-tie protocol step 3: the oracle re-run with the GPU's P codes (every
    mismatch was already checked to be a near-tie)."""
    O2, _ = att.decode_attend(state, q, pcodes_override={hq: gpu_pcodes[hq][None] for hq in range(Hq)})
    return float(row_rel_err(O_gpu, O2).max())


def run_decode(ocfg, prompts, steps, seed=21, check_every=1, check_pages_at=()):
    """Every step runs the PRODUCTION call (no debug pointers: even steps the combined
    hack_decode_attention, odd steps hack_decode_append + hack_decode_attention_cached), then the
    debug instantiation on the same cache (P codes + MMA accumulator dumps).  The two outputs
    must be bit-identical; the production output is checked against the oracle; the dumped
    accumulators bit-exactly through their affine form (acc_expected)."""
    h = hk()
    cfg = gpu_cfg(ocfg)
    B = len(prompts)
    maxL = max(prompts) + steps
    cache = make_cache(cfg, max_reqs=B + 2, max_len=maxL, seed=seed)
    slots = (np.arange(B, dtype=np.int32) + 1)
    rid = np.array([7000 + 13 * i for i in range(B)], np.uint32)
    cache.rng_ids[torch.from_numpy(slots).long()] = torch.from_numpy(rid.view(np.int32)).cuda()
    states = []
    # prefill each request (the ingest path), oracle state alongside
    for i, L in enumerate(prompts):
        q, k, v = hack_inputs.qkv(seed + i, L, ocfg.Hq, ocfg.Hkv)
        cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
        sl = torch.tensor([slots[i]], dtype=torch.int32, device="cuda")
        out = torch.zeros((L, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
        if ocfg.p_round == "sr" and ocfg.Pi != 64:   # P-SR prefill runs at Pi = 64 only: ingest the prompt
            h.cache_ingest(cfg, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), cu, sl, L, cache)
        else:
            h.prefill_attention(cfg, torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                torch.from_numpy(v).cuda(), cu, sl, L, cache, out)
        states.append(att.ingest_prompt(ocfg, k, v, rng_id=int(rid[i])))
    qd, kd, vd = hack_inputs.decode_tokens(seed, steps, B, ocfg.Hq, ocfg.Hkv)
    sl = torch.from_numpy(slots).cuda()
    stride = (maxL + ocfg.Pi - 1) // ocfg.Pi * ocfg.Pi
    form = h.debug_acc_form(cfg, "decode")
    worst, flips, nacc = 0.0, 0, 0
    for s in range(steps):
        qs, ks, vs = (torch.from_numpy(x[s]).cuda() for x in (qd, kd, vd))
        out = torch.zeros((B, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
        if s % 2 == 0:
            h.decode_attention(cfg, qs, ks, vs, sl, maxL, cache, out)
        else:
            h.decode_append(cfg, ks, vs, sl, cache)
            h.decode_attention_cached(cfg, qs, sl, maxL, cache, out)
        check = s % check_every == 0 or s == steps - 1
        dout = torch.zeros_like(out)
        pc = torch.zeros((B, ocfg.Hq, stride), dtype=torch.uint8, device="cuda")
        qk, pv = acc_buffers(B, ocfg.Hq, ocfg, stride) if check and form != h.ACC_NONE else (None, None)
        h.decode_attention_cached(cfg, qs, sl, maxL, cache, dout, debug_pcodes=pc, debug_qk=qk, debug_pv=pv)
        torch.cuda.synchronize()
        og, pcn = out.cpu().numpy(), pc.cpu().numpy()
        assert np.array_equal(og.view(np.uint32), dout.cpu().numpy().view(np.uint32)), \
            f"step {s}: production and debug instantiations differ"
        qkn = qk.cpu().numpy() if qk is not None else None
        pvn = pv.cpu().numpy() if pv is not None else None
        for i in range(B):
            O, diag = att.decode_step(states[i], qd[s, i], kd[s, i], vd[s, i], keep_diag=True)
            if check:
                nf = states[i].nblocks * ocfg.Pi
                for hq in range(ocfg.Hq):
                    if nf:
                        flips += check_pcodes(pcn[i, hq, :nf][None], diag[hq]["pcodes"], diag[hq]["py"],
                                              diag[hq]["pu"])
                err = row_rel_err(og[i], O).max()
                worst = max(worst, float(err))
                if err > ROW_TOL and nf:
                    err = substituted_err(states[i], qd[s, i], pcn[i, :, :nf], og[i], ocfg.Hq)
                assert err <= ROW_TOL, f"step {s} req {i}: row error {err:.3g}"
                if qkn is not None:
                    pos = states[i].length - 1
                    qc, _, _, qsum = att.quantize_q(ocfg, qd[s, i][None], np.array([pos]), states[i].rng_id)
                    for hq in range(ocfg.Hq):
                        nq, npv = check_acc(form, ocfg, states[i], qc, qsum, [pos], hq, qkn[i, hq][None],
                                            pvn[i, hq][None], pcn[i, hq][None])
                        nacc += nq + npv
            assert int(cache.seq_lens[int(slots[i])]) == states[i].length
        if s in check_pages_at:
            for i in range(B):
                compare_pages(cache, int(slots[i]), states[i])
    for i in range(B):
        compare_pages(cache, int(slots[i]), states[i])
    if form != h.ACC_NONE:
        assert nacc > 0
    print(f"decode: worst row error {worst:.3g}, near-tie flips {flips}, accumulators checked {nacc}")
    return worst, flips


def test_c1_decode_512_plus_16():
    run_decode(att.Config(Hq=1, Hkv=1, Pi=64, bits=2), [512], 16)


@pytest.mark.parametrize("L", [1, 63, 64, 65, 127, 500])
def test_decode_crosses_flush(L):
    # 70 steps: every prompt crosses at least one Pi boundary (RQE flush)
    run_decode(att.Config(Hq=4, Hkv=1, Pi=64, bits=2), [L], 70, check_every=7, check_pages_at=(5, 40))


@pytest.mark.parametrize("merge", ["auto", "1", "0"])
def test_decode_batch_gqa_mixed_lengths(merge, monkeypatch):
    # merge: where the split partials are merged (decode_pair.cu): chosen by the launch, in
    # the main kernel (merge_units), or by decode_pair_combine
    if merge != "auto":
        monkeypatch.setenv("HACK_DECODE_MERGE", merge)
    run_decode(att.Config(Hq=8, Hkv=2, Pi=64, bits=2, seed=99, layer=1), [100, 1, 64, 255], 40, check_every=5)


@pytest.mark.parametrize("Pi,bits", [(32, 2), (128, 2), (64, 4), (128, 4), (32, 4)])
def test_decode_partition_and_bits(Pi, bits):
    # Pi in {32, 128}: decode_mma_kernel<BITS, Pi>; Pi = 64, b = 4: decode_mma too
    run_decode(att.Config(Hq=4, Hkv=2, Pi=Pi, bits=bits), [150, 129], 2 * Pi + 3, check_every=11)


@pytest.mark.parametrize("Pi,bits,Hq", [(32, 2, 8), (128, 4, 6), (128, 2, 1)])
def test_decode_partition_group_shapes(Pi, bits, Hq):
    # G = 8, 6 (two row pairs padded), 1 at the non-64 partitions; ragged lengths incl. 1 token
    run_decode(att.Config(Hq=Hq, Hkv=1, Pi=Pi, bits=bits, seed=13), [1, 2 * Pi + 5, 300], Pi + 2, check_every=17)


@pytest.mark.parametrize("Pi,bits", [(32, 2), (128, 4)])
def test_decode_simt_other_partitions(Pi, bits, monkeypatch):
    # the CUDA-core kernel stays a parity-checked baseline at Pi != 64
    monkeypatch.setenv("HACK_DECODE_IMPL", "simt")
    run_decode(att.Config(Hq=4, Hkv=2, Pi=Pi, bits=bits), [150, 129], Pi + 3, check_every=13)


def test_decode_group_16():
    run_decode(att.Config(Hq=16, Hkv=1, Pi=64, bits=2), [70], 10, check_every=3)


def test_decode_simt_baseline_kernel(monkeypatch):
    # the CUDA-core baseline (used for Pi != 64 or G > 8) meets the same bar at Pi = 64
    monkeypatch.setenv("HACK_DECODE_IMPL", "simt")
    run_decode(att.Config(Hq=4, Hkv=2, Pi=64, bits=2), [130, 64, 5], 70, check_every=9)


def test_decode_general_mma_kernel_g4(monkeypatch):
    # the general split-KV kernel (serves G > 4 and b = 4) at the shapes the paired kernel covers
    monkeypatch.setenv("HACK_DECODE_IMPL", "mma")
    run_decode(att.Config(Hq=4, Hkv=2, Pi=64, bits=2), [130, 64, 5, 1000], 70, check_every=9)


def test_decode_paired_kernel_edges():
    # G in {1, 2, 3}, odd/even committed page counts, splits with and without the tail page
    run_decode(att.Config(Hq=3, Hkv=1, Pi=64, bits=2, seed=5), [2047, 1, 128], 66, check_every=13)
    run_decode(att.Config(Hq=4, Hkv=2, Pi=64, bits=2, seed=6), [4096 + 64, 3000], 3)


def test_c3_full_size_sampled_requests():
    """Llama-3.1-8B decode shape at BASELINE size (batch 64, ~8K context, 32 Q / 8 KV
    heads, b = 2, Pi = 64) in the launch configuration bench.py times: two decode steps
    over ragged lengths near 8192; three sampled requests are checked on every head
    against the oracle (page bytes bit-exact, outputs <= 1e-3 row-relative)."""
    h = hk()
    ocfg = att.Config(Hq=32, Hkv=8, Pi=64, bits=2, seed=77)
    cfg = gpu_cfg(ocfg)
    B, steps = 64, 2
    lens = [8192 - (i * 29) % 64 for i in range(B)]
    sampled = [0, 37, 63]
    maxL = 8192 + steps
    cache = make_cache(cfg, max_reqs=B, max_len=maxL, seed=3)
    slots = np.arange(B, dtype=np.int32)
    rid = np.array([100 + 7 * i for i in range(B)], np.uint32)
    cache.rng_ids[:B] = torch.from_numpy(rid.view(np.int32)).cuda()
    gen = torch.Generator(device="cuda").manual_seed(1234)
    states = {}
    for i, L in enumerate(lens):
        if i in sampled:
            _, k, v = hack_inputs.qkv(500 + i, L, 1, ocfg.Hkv)
            states[i] = att.ingest_prompt(ocfg, k, v, rng_id=int(rid[i]))
            kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
        else:
            kd = torch.randn((L, ocfg.Hkv, 128), generator=gen, device="cuda").half()
            vd = torch.randn((L, ocfg.Hkv, 128), generator=gen, device="cuda").half()
        cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
        h.cache_ingest(cfg, kd, vd, cu, torch.tensor([i], dtype=torch.int32, device="cuda"), L, cache)
    qd, kd, vd = hack_inputs.decode_tokens(9, steps, B, ocfg.Hq, ocfg.Hkv)
    sl = torch.from_numpy(slots).cuda()
    stride = (maxL + 63) // 64 * 64
    form = h.debug_acc_form(cfg, "decode")
    assert form == h.ACC_CENTERED4          # the production decode_pair_kernel serves C3
    for s in range(steps):
        out = torch.zeros((B, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
        # production call first (no debug pointers), then the debug instantiation on the same cache
        h.decode_attention(cfg, torch.from_numpy(qd[s]).cuda(), torch.from_numpy(kd[s]).cuda(),
                           torch.from_numpy(vd[s]).cuda(), sl, maxL, cache, out)
        dout = torch.zeros_like(out)
        pc = torch.zeros((B, ocfg.Hq, stride), dtype=torch.uint8, device="cuda")
        qk, pv = acc_buffers(B, ocfg.Hq, ocfg, stride)
        h.decode_attention_cached(cfg, torch.from_numpy(qd[s]).cuda(), sl, maxL, cache, dout, debug_pcodes=pc,
                                  debug_qk=qk, debug_pv=pv)
        torch.cuda.synchronize()
        og, pcn = out.cpu().numpy(), pc.cpu().numpy()
        assert np.array_equal(og.view(np.uint32), dout.cpu().numpy().view(np.uint32))
        assert np.isfinite(og).all()
        qkn, pvn = qk.cpu().numpy(), pv.cpu().numpy()
        for i in sampled:
            O, diag = att.decode_step(states[i], qd[s, i], kd[s, i], vd[s, i], keep_diag=True)
            nf = states[i].nblocks * ocfg.Pi
            for hq in range(ocfg.Hq):
                check_pcodes(pcn[i, hq, :nf][None], diag[hq]["pcodes"], diag[hq]["py"])
            err = row_rel_err(og[i], O).max()
            if err > ROW_TOL:
                err = substituted_err(states[i], qd[s, i], pcn[i, :, :nf], og[i], ocfg.Hq)
            assert err <= ROW_TOL, f"step {s} req {i}: row error {err:.3g}"
            pos = states[i].length - 1
            qc, _, _, qsum = att.quantize_q(ocfg, qd[s, i][None], np.array([pos]), states[i].rng_id)
            for hq in range(ocfg.Hq):
                check_acc(form, ocfg, states[i], qc, qsum, [pos], hq, qkn[i, hq][None], pvn[i, hq][None],
                          pcn[i, hq][None])
    for i in sampled:
        compare_pages(cache, i, states[i])


def test_no_se_ablation_bit_identical(monkeypatch):
    """SURVEY f2, HACK/SE: recomputing the code sums on every decode step
    instead of reading the summation cache must give bit-identical outputs (same integers
    into the same Eq. 4 arithmetic); only the cost differs.  Also meets the oracle bar."""
    h = hk()
    ocfg = att.Config(Hq=8, Hkv=2, Pi=64, bits=2, seed=12)
    monkeypatch.setenv("HACK_DECODE_NO_SE", "1")
    run_decode(ocfg, [300, 64, 1000], 5, check_every=2)
    cfg = gpu_cfg(ocfg)
    cache = make_cache(cfg, max_reqs=3, max_len=2100, seed=2)
    L = [2047, 700, 129]
    for i, n in enumerate(L):
        _, k, v = hack_inputs.qkv(40 + i, n, 1, ocfg.Hkv)
        h.cache_ingest(cfg, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                       torch.tensor([0, n], dtype=torch.int32, device="cuda"),
                       torch.tensor([i], dtype=torch.int32, device="cuda"), n, cache)
    qd, _, _ = hack_inputs.decode_tokens(3, 1, 3, ocfg.Hq, ocfg.Hkv)
    sl = torch.arange(3, dtype=torch.int32, device="cuda")
    outs = []
    for flag in ("1", None):
        if flag:
            monkeypatch.setenv("HACK_DECODE_NO_SE", flag)
        else:
            monkeypatch.delenv("HACK_DECODE_NO_SE", raising=False)
        o = torch.zeros((3, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
        h.decode_attention_cached(cfg, torch.from_numpy(qd[0]).cuda(), sl, 2100, cache, o)
        outs.append(o.cpu().numpy())
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


def test_decode_long_context_tiny_cta_ranges():
    """One 96K-token request (G = 4): the persistent split gives every CTA a range of only
    a few pages (odd sizes, single-page items, segments that start mid-pair) and the
    merge combines ~600 CTAs x warps partials of one unit."""
    run_decode(att.Config(Hq=4, Hkv=1, Pi=64, bits=2, seed=31), [96000], 2)


@pytest.mark.parametrize("Hq,merge", [(8, "auto"), (6, "auto"), (8, "1")])
def test_decode_group8_paired_kernel(Hq, merge, monkeypatch):
    # decode_g8_kernel: G in (4, 8] (C4 70B shape has G = 8), flushes, tails, mixed lengths
    if merge != "auto":
        monkeypatch.setenv("HACK_DECODE_MERGE", merge)
    run_decode(att.Config(Hq=Hq, Hkv=1, Pi=64, bits=2, seed=14), [300, 64, 1000, 1], 70, check_every=9)


def test_decode_general_mma_kernel_g8(monkeypatch):
    monkeypatch.setenv("HACK_DECODE_IMPL", "mma")
    run_decode(att.Config(Hq=16, Hkv=2, Pi=64, bits=2, seed=15), [300, 129], 20, check_every=7)


@pytest.mark.parametrize("Pi,bits,Hq", [(64, 2, 4), (64, 4, 8), (32, 2, 2), (128, 4, 4)])
def test_decode_p_stochastic_rounding(Pi, bits, Hq):
    """R6 selectable: P stochastic rounding on decode_mma_kernel (the paired kernels keep RN),
    across flushes; near-ties judged against the SR boundary."""
    run_decode(att.Config(Hq=Hq, Hkv=2 if Hq < 8 else 1, Pi=Pi, bits=bits, p_round="sr", seed=19), [130, 64],
               Pi + 3, check_every=7)


@pytest.mark.parametrize("Hq,merge", [(8, "1"), (16, "1"), (8, "0")])
def test_decode_workspace_reuse_merge_counters(Hq, merge, monkeypatch):
    """The in-kernel merge counts CTAs per unit in the workspace and leaves the counters zero:
    one zero-filled workspace reused for many launches (mixed lengths, units split over many
    CTAs, G = 4 pair kernel and G = 8 kernel) gives bit-identical outputs to a fresh
    workspace per launch, and the counter region is zero afterwards."""
    monkeypatch.setenv("HACK_DECODE_MERGE", merge)
    h = hk()
    ocfg = att.Config(Hq=Hq, Hkv=2, Pi=64, bits=2, seed=5)
    cfg = gpu_cfg(ocfg)
    lens = [5000, 1, 64, 700, 129, 3000]
    B = len(lens)
    cache = make_cache(cfg, max_reqs=B, max_len=max(lens) + 4, seed=5)
    for i, n in enumerate(lens):
        _, k, v = hack_inputs.qkv(60 + i, n, 1, ocfg.Hkv)
        h.cache_ingest(cfg, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                       torch.tensor([0, n], dtype=torch.int32, device="cuda"),
                       torch.tensor([i], dtype=torch.int32, device="cuda"), n, cache)
    sl = torch.arange(B, dtype=torch.int32, device="cuda")
    nb = h.decode_workspace_size(cfg, B, max(lens) + 4)
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    qd, _, _ = hack_inputs.decode_tokens(9, 6, B, ocfg.Hq, ocfg.Hkv)
    for s in range(6):
        q = torch.from_numpy(qd[s]).cuda()
        o1 = torch.zeros((B, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
        o2 = torch.zeros_like(o1)
        h.decode_attention_cached(cfg, q, sl, max(lens) + 4, cache, o1, workspace=ws)
        h.decode_attention_cached(cfg, q, sl, max(lens) + 4, cache, o2)   # fresh zero workspace
        assert np.array_equal(o1.cpu().numpy().view(np.uint32), o2.cpu().numpy().view(np.uint32)), f"launch {s}"
    # counter region: after the header of (16 + 2 B) ints rounded to 256 B, B * H_kv ints
    off = ((16 + 2 * B) * 4 + 255) // 256 * 256
    assert int(ws[off:off + 4 * B * ocfg.Hkv].view(torch.int32).abs().sum()) == 0


@pytest.mark.parametrize("Hq,merge", [(8, "1"), (8, "0"), (16, "1"), (16, "0")])
def test_fused_decode_step_equals_separate(Hq, merge, monkeypatch):
    """hack_decode_attention fuses the append (a8) into the paired decode kernel (the CTA
    owning a unit's last page appends before loading it; seq_lens bumped after every CTA
    read it, by the last CTA or by the combine kernel).  Over 70 steps (every request
    crosses a flush) it must produce bit-identical outputs, pages, FP16 tails and lengths to
    the separate append kernel + attention (HACK_DECODE_FUSED=0), on both merge paths; the
    oracle comparison of the fused path is run_decode's even steps."""
    h = hk()
    monkeypatch.setenv("HACK_DECODE_MERGE", merge)
    ocfg = att.Config(Hq=Hq, Hkv=2, Pi=64, bits=2, seed=8)
    cfg = gpu_cfg(ocfg)
    lens = [1000, 1, 64, 63, 300]
    B, steps = len(lens), 70
    caches = [make_cache(cfg, max_reqs=B, max_len=max(lens) + steps, seed=8) for _ in range(2)]
    for c in caches:
        c.rng_ids.copy_(torch.arange(100, 100 + B, dtype=torch.int32, device="cuda"))
        for i, n in enumerate(lens):
            _, k, v = hack_inputs.qkv(80 + i, n, 1, ocfg.Hkv)
            h.cache_ingest(cfg, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                           torch.tensor([0, n], dtype=torch.int32, device="cuda"),
                           torch.tensor([i], dtype=torch.int32, device="cuda"), n, c)
    sl = torch.arange(B, dtype=torch.int32, device="cuda")
    qd, kd, vd = hack_inputs.decode_tokens(12, steps, B, ocfg.Hq, ocfg.Hkv)
    ML = max(lens) + steps
    ws = [torch.zeros(h.decode_workspace_size(cfg, B, ML), dtype=torch.uint8, device="cuda") for _ in range(2)]
    for s in range(steps):
        q, k, v = (torch.from_numpy(x[s]).cuda() for x in (qd, kd, vd))
        outs = []
        for j, fused in enumerate(("1", "0")):
            monkeypatch.setenv("HACK_DECODE_FUSED", fused)
            o = torch.zeros((B, ocfg.Hq, 128), dtype=torch.float32, device="cuda")
            h.decode_attention(cfg, q, k, v, sl, ML, caches[j], o, workspace=ws[j])
            outs.append(o.cpu().numpy())
        assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32)), f"step {s}"
    a, b = caches
    assert torch.equal(a.seq_lens, b.seq_lens)
    assert [int(x) for x in a.seq_lens[:B].cpu()] == [n + steps for n in lens]
    for i in range(B):
        npg = (lens[i] + steps + ocfg.Pi - 1) // ocfg.Pi
        assert np.array_equal(gpu_pages_of(a, i, npg), gpu_pages_of(b, i, npg)), f"request {i} pages"
        T = (lens[i] + steps) % ocfg.Pi  # valid FP16 tail rows
        assert torch.equal(a.v_tail[i, :, :T], b.v_tail[i, :, :T]), f"request {i} tail"
