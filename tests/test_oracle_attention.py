"""Pins for the oracle's HACK prefill / decode / exact attention and pages (no GPU)."""
import json
import os

import numpy as np
import pytest

import hack_inputs
from oracle import attention as att
from oracle import pages, quant

W = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def cfg(Hq=2, Hkv=1, Pi=64, bits=2, **kw):
    return att.Config(Hq=Hq, Hkv=Hkv, d=128, Pi=Pi, bits=bits, **kw)


def v_hat(state, h):
    """Dequantized V history of head h: committed blocks (s v' + m) then the
    FP16 tail -- an independent reconstruction for the closed forms."""
    a = state.arrays()
    rows = []
    for j in range(a["vc"].shape[0]):
        rows.append(quant.dequantize(a["vc"][j, h], a["vm"][j, h], a["vs"][j, h]).T)   # [Pi, d]
    if a["tail"].shape[0]:
        rows.append(a["tail"][:, h].astype(np.float64))
    return np.concatenate(rows, 0)


# ----------------------------------------------------------------- exact attention

def test_exact_attention_vs_naive_loops():
    # S:489 bypass oracle vs an independent triple loop
    q, k, v = hack_inputs.qkv(1, 9, 2, 1, d=8, partition=8)
    O = att.exact_attention(q, k, v)
    for i in range(9):
        for h in range(2):
            s = [sum(float(q[i, h, c]) * float(k[t, 0, c]) for c in range(8)) / np.sqrt(8)
                 for t in range(i + 1)]
            mx = max(s)
            e = [np.exp(x - mx) for x in s]
            z = sum(e)
            for c in range(8):
                o = sum(e[t] / z * float(v[t, 0, c]) for t in range(i + 1))
                assert abs(O[i, h, c] - o) < 1e-12


def test_softmax_closed_forms():
    # [0,0,0] -> 1/3 each; [1,2,3] with 2 valid -> [1/(1+e), e/(1+e), 0]
    d = 4
    q = np.zeros((3, 1, d), np.float16)
    k = np.zeros((3, 1, d), np.float16)
    v = np.eye(3, d, dtype=np.float16)[:, None, :]
    O = att.exact_attention(q, k, v, causal=False)
    assert np.allclose(O[0, 0, :3], 1 / 3, atol=1e-15)
    # scores [1,2,3]*sqrt(d) so that S/sqrt(d) = [1,2,3]; row position 1 sees 2 keys
    q = np.zeros((1, 1, d), np.float16); q[0, 0, 0] = 2.0      # sqrt(4) = 2
    k = np.zeros((3, 1, d), np.float16); k[:, 0, 0] = [1, 2, 3]
    O = att.exact_attention(q, k, v, causal=True, q_positions=[1])
    e = np.e
    assert np.allclose(O[0, 0, :3], [1 / (1 + e), e / (1 + e), 0], atol=1e-15)


# ----------------------------------------------------------------- HACK closed forms

def test_q_zero_gives_mean_of_visible_dequantized_v():
    # Q = 0 -> S = 0 -> uniform P -> O = mean of visible V_hat (R14)
    L = 150
    c = cfg(Hq=1, Hkv=1)
    _, k, v = hack_inputs.qkv(2, L, 1, 1)
    q = np.zeros((L, 1, 128), np.float16)
    O, st, _ = att.prefill(c, q, k, v)
    V = v_hat(st, 0)
    # for rows whose visible keys cover whole committed blocks + tail the mean is
    # exact; for partially visible (diagonal) blocks P' is {255, 0} -> also exact
    for i in (0, 5, 63, 64, 100, 127, 128, 149):
        assert np.allclose(O[i, 0], V[:i + 1].mean(0), rtol=1e-10, atol=1e-12)


def test_grid_exact_scores_match_exact_qk():
    # Q, K on their quantization grids (both extremes present per partition):
    # quantization is exact under RN and SR, so S == QK^T/sqrt(d) (SURVEY c-5)
    L = 96
    c = cfg(Hq=2, Hkv=1)
    q, k, v = hack_inputs.qkv(3, L, 2, 1, dist="grid")
    for rnd in ("rn", "sr"):
        c.kv_round = c.q_round = rnd
        _, st, dg = att.prefill(c, q, k, v, keep_diag=True)
        a = st.arrays()
        khat = np.concatenate([quant.dequantize(a["kc"][:, 0].reshape(L, 2, 64)[:, b],
                                                a["km"][:, 0, b], a["ks"][:, 0, b]) for b in range(2)], 1)
        assert np.array_equal(khat, k[:, 0].astype(np.float64))
        ex = att.exact_attention(q, k, v)  # noqa: F841 (P check below)
        for hq in range(2):
            S = q[:, hq].astype(np.float64) @ k[:, 0].astype(np.float64).T / np.sqrt(128)
            S = np.where(np.tril(np.ones((L, L), bool)), S, -np.inf)
            P = np.exp(S - S.max(1, keepdims=True)); P /= P.sum(1, keepdims=True)
            assert np.allclose(dg[hq]["P"], P, rtol=1e-12, atol=1e-15)


def test_one_hot_attention_returns_v_hat():
    # q = alpha k_t with large alpha -> p ~ e_t -> O = v_hat_t (P' codes 255/0)
    L = 140
    c = cfg(Hq=1, Hkv=1)
    _, k, v = hack_inputs.qkv(4, L, 1, 1)
    q = np.zeros((L, 1, 128), np.float16)
    tgt = {70: 10, 139: 20, 130: 130}       # row -> target key (committed, committed, tail)
    for i, t in tgt.items():
        q[i, 0] = (k[t, 0].astype(np.float32) * 40).astype(np.float16)
    O, st, dg = att.prefill(c, q, k, v, rows=list(tgt), keep_diag=True)
    V = v_hat(st, 0)
    for i, t in tgt.items():
        assert np.allclose(O[i, 0], V[t], rtol=1e-9, atol=1e-9), (i, t)


def test_constant_v_channels_pin_no_renormalisation():
    # V constant per channel -> s_v = 0 -> O_c = v_c * (sum of dequantized P) (R14)
    L = 200
    c = cfg(Hq=1, Hkv=1)
    q, k, _ = hack_inputs.qkv(5, L, 1, 1)
    vc = np.random.default_rng(0).standard_normal(128).astype(np.float16)
    v = np.tile(vc, (L, 1, 1))
    O, st, dg = att.prefill(c, q, k, v, keep_diag=True)
    P = dg[0]["P"]; pc = dg[0]["pcodes"]
    nfull = L // 64
    for i in (10, 100, 199):
        mass = 0.0
        for j in range(nfull):
            p = P[i, j * 64:(j + 1) * 64]
            m, s = p.min(), (p.max() - p.min()) / 255
            mass += (s * pc[i, j * 64:(j + 1) * 64] + m).sum()
        mass += P[i, nfull * 64:].sum()
        assert np.allclose(O[i, 0], vc.astype(np.float64) * mass, rtol=1e-12)
        assert abs(mass - 1) < 0.05 and mass != 1.0


def test_short_prompt_pv_is_exact_fp():
    # L < Pi: every V is in the FP16 tail -> O = softmax(S_hack) V exactly
    L = 50
    c = cfg(Hq=2, Hkv=1)
    q, k, v = hack_inputs.qkv(6, L, 2, 1)
    O, st, dg = att.prefill(c, q, k, v, keep_diag=True)
    assert st.nblocks == 0 and len(st.tail) == L
    for hq in range(2):
        assert np.allclose(O[:, hq], dg[hq]["P"] @ v[:, 0].astype(np.float64), rtol=1e-13)


def test_single_and_identical_tokens():
    # a single token, or identical tokens, output the v row
    c = cfg(Hq=1, Hkv=1)
    q, k, v = hack_inputs.qkv(7, 1, 1, 1)
    O, _, _ = att.prefill(c, q, k, v)
    assert np.array_equal(O[0, 0], v[0, 0].astype(np.float64))
    # identical tokens under RN (SR would give the copies different K codes,
    # hence unequal scores and a quantized P whose mass is not exactly 1, R14)
    L = 130
    q, k, v = hack_inputs.qkv(8, L, 1, 1)
    k = np.tile(k[:1], (L, 1, 1)); v = np.tile(v[:1], (L, 1, 1))
    O, _, _ = att.prefill(cfg(Hq=1, Hkv=1, kv_round="rn"), q, k, v)
    assert np.allclose(O[:, 0], v[0, 0].astype(np.float64), rtol=1e-12, atol=1e-12)


def test_pv_identity_twin():
    # O7': Eq. 4 for P V equals dequantize-then-multiply with P_hat, V_hat
    L = 192 + 17
    c = cfg(Hq=1, Hkv=1)
    q, k, v = hack_inputs.qkv(9, L, 1, 1)
    O, st, dg = att.prefill(c, q, k, v, keep_diag=True)
    P, pc = dg[0]["P"], dg[0]["pcodes"]
    V = v_hat(st, 0)
    nfull = st.nblocks
    Phat = P.copy()
    for j in range(nfull):
        sl = slice(j * 64, (j + 1) * 64)
        m = P[:, sl].min(1, keepdims=True); s = (P[:, sl].max(1, keepdims=True) - m) / 255
        Phat[:, sl] = s * pc[:, sl] + m
    assert np.allclose(O[:, 0], Phat @ V, rtol=1e-11, atol=1e-13)


def test_w6_p_partition_with_masked_zeros():
    ex = W["p_partition"]
    c, m, s, sm, y = att.quantize_p(np.array(ex["p"]))
    assert c.tolist() == ex["codes"] and int(sm) == ex["sum"] and m == 0.0


# ----------------------------------------------------------------- structure: RQE / SE

@pytest.mark.parametrize("L,blocks,tail", W["pages"]["prompt_blocks_tail"])
def test_prompt_blocks_and_tail(L, blocks, tail):
    c = cfg(Hq=1, Hkv=1)
    _, k, v = hack_inputs.qkv(10, L, 1, 1)
    st = att.ingest_prompt(c, k, v)
    assert st.nblocks == blocks and len(st.tail) == tail and st.length == L


def test_rqe_committed_state_is_bit_stable_and_flush_at_pi():
    # S:242-245 / S:592: appends never change committed codes/meta/sums;
    # tail < Pi after every op; flush exactly when the tail reaches Pi
    c = cfg(Hq=2, Hkv=2, Pi=32)
    _, k, v = hack_inputs.qkv(11, 500, 2, 2)
    st = att.ingest_prompt(c, k[:37], v[:37])
    snap = st.arrays()
    for t in range(37, 500):
        st.append_k(k[t:t + 1]); st.append_v(v[t])
        assert len(st.tail) < 32
        assert len(st.tail) == (t + 1) % 32 and st.nblocks == (t + 1) // 32
        a = st.arrays()
        nb0, L0 = snap["vc"].shape[0], snap["kc"].shape[0]
        for key in ("vc", "vm", "vs", "vsum"):
            assert np.array_equal(a[key][:nb0], snap[key])
        for key in ("kc", "km", "ks", "ksum"):
            assert np.array_equal(a[key][:L0], snap[key])
        snap = a


def test_w5_rqe_tail_keeps_fp16():
    ex = W["rqe_example"]
    c = att.Config(Hq=1, Hkv=1, d=4, Pi=4)
    st = att.KVState(c)
    for x in (-2.1, 1.7, -2.9):
        st.append_k(np.full((1, 1, 4), x, np.float16))
        st.append_v(np.full((1, 4), x, np.float16))
    assert st.nblocks == 0
    assert [float(r[0, 1]) for r in st.tail] == ex["tail_fp16"]


def test_sums_are_code_sums():
    c = cfg(Hq=2, Hkv=2, Pi=128, bits=2)
    _, k, v = hack_inputs.qkv(12, 300, 2, 2)
    a = att.ingest_prompt(c, k, v).arrays()
    assert np.array_equal(a["ksum"], a["kc"].reshape(300, 2, 1, 128).astype(np.int64).sum(-1))
    assert np.array_equal(a["vsum"], a["vc"].astype(np.int64).sum(-1))
    # at Pi=128 a sum can reach 127*3 = 381 > 255: the INT16 width
    assert max(a["vsum"].max(), a["ksum"].max()) <= 127 * 3
    assert quant.sum_width_bits(2, 128) == 16


def test_prefill_equals_token_by_token_appends():
    # position-keyed counters: prefill ingestion == decode-style appends, bit-exact
    c = cfg(Hq=4, Hkv=2)
    _, k, v = hack_inputs.qkv(13, 150, 4, 2)
    a1 = att.ingest_prompt(c, k, v, rng_id=5).arrays()
    st = att.KVState(c, rng_id=5)
    for t in range(150):
        st.append_k(k[t:t + 1]); st.append_v(v[t])
    a2 = st.arrays()
    for key in a1:
        assert np.array_equal(a1[key], a2[key]), key


def test_decode_step_equals_last_prefill_row():
    c = cfg(Hq=4, Hkv=2)
    L = 131
    q, k, v = hack_inputs.qkv(14, L, 4, 2)
    O, _, _ = att.prefill(c, q, k, v, rng_id=3)
    st = att.ingest_prompt(c, k[:L - 1], v[:L - 1], rng_id=3)
    o, _ = att.decode_step(st, q[L - 1], k[L - 1], v[L - 1])
    # same codes (position-keyed counters); fp64 GEMM order may differ by ulps
    assert np.allclose(o, O[L - 1], rtol=1e-13, atol=1e-15)


def test_causality_outside_the_diagonal_block():
    # Row i never depends on K of later tokens nor on V of later *blocks*.
    # (V of later tokens in i's own block shares i's V partition min/scale --
    # a property of partitioning V along the sequence.)
    c = cfg(Hq=1, Hkv=1)
    L = 200
    q, k, v = hack_inputs.qkv(15, L, 1, 1)
    O1, _, _ = att.prefill(c, q, k, v)
    k2, v2 = k.copy(), v.copy()
    k2[101:] *= 3
    v2[128:] *= -2
    O2, _, _ = att.prefill(c, q, k2, v2)
    assert np.array_equal(O1[:101], O2[:101])


def test_error_monotone_in_bits_and_partition():
    # mean error vs exact attention: 2-bit > 4-bit; Pi=32 <= Pi=128
    errs = {}
    for bits, Pi in ((2, 64), (4, 64), (2, 32), (2, 128)):
        e = []
        for seed in range(6):
            q, k, v = hack_inputs.qkv(100 + seed, 256, 1, 1)
            O, _, _ = att.prefill(cfg(Hq=1, Hkv=1, Pi=Pi, bits=bits), q, k, v)
            ex = att.exact_attention(q, k, v)
            e.append(np.abs(O - ex).mean())
        errs[(bits, Pi)] = np.mean(e)
    assert errs[(2, 64)] > errs[(4, 64)]
    assert errs[(2, 32)] <= errs[(2, 128)]


def test_hack_scores_unbiased_over_seeds():
    # SR unbiased + linearity of Eq. 4: with Q on its 8-bit grid
    # (exact) the seed-mean of S converges to Q K^T / sqrt(d).
    c = cfg(Hq=1, Hkv=1)
    q, k, _ = hack_inputs.qkv(16, 64, 1, 1, dist="grid")
    _, k, v = hack_inputs.qkv(17, 64, 1, 1)
    S_ex = q[-1:, 0].astype(np.float64) @ k[:, 0].astype(np.float64).T / np.sqrt(128)
    acc = []
    for seed in range(300):
        c.seed = seed
        st = att.ingest_prompt(c, k, v).arrays()
        qc, qm, qs, qsum = att.quantize_q(c, q[-1:], [63], 0)
        S = np.zeros(64)
        for b in range(2):
            sl = slice(b * 64, (b + 1) * 64)
            D = qc[0, 0, sl].astype(np.float64) @ st["kc"][:, 0, sl].T.astype(np.float64)
            S += (qs[0, 0, b] * st["ks"][:, 0, b] * D + st["km"][:, 0, b] * qs[0, 0, b] * qsum[0, 0, b]
                  + qm[0, 0, b] * st["ks"][:, 0, b] * st["ksum"][:, 0, b] + 64 * qm[0, 0, b] * st["km"][:, 0, b])
        acc.append(S / np.sqrt(128))
    acc = np.array(acc)
    se = acc.std(0) / np.sqrt(len(acc))
    assert np.all(np.abs(acc.mean(0) - S_ex[0]) <= 5 * se + 2e-3 * np.abs(S_ex[0]) + 1e-6)


# ----------------------------------------------------------------- pages

def test_page_layout_sizes_and_compression():
    ex = W["pages"]
    assert pages.layout(128, 64, 2)["page_bytes"] == ex["page_bytes_b2_pi64"]
    assert pages.layout(128, 64, 4)["page_bytes"] == ex["page_bytes_b4_pi64"]
    c = cfg(Hq=1, Hkv=1)
    _, k, v = hack_inputs.qkv(18, 512, 1, 1)
    pg, mk = pages.pack_request(att.ingest_prompt(c, k, v))
    assert pg.size == ex["c1_packed_bytes"] and k.nbytes + v.nbytes == ex["c1_fp16_bytes"]
    assert pg.size / (k.nbytes + v.nbytes) <= 0.17      # S:591, "~15%"
    assert pages.bytes_per_token(128, 64, 2) == 84


def test_pages_round_trip():
    c = cfg(Hq=2, Hkv=2, bits=4)
    _, k, v = hack_inputs.qkv(19, 150, 2, 2)
    st = att.ingest_prompt(c, k, v)
    pg, mk = pages.pack_request(st)
    a = st.arrays()
    lay = pages.layout(128, 64, 4)
    o, sz = lay["k_codes"]
    for p in range(pg.shape[0]):
        n = min(64, 150 - p * 64)
        kc = quant.unpack(pg[p, 1, o:o + n * 64].reshape(n, 64), 4, 128)
        assert np.array_equal(kc, a["kc"][p * 64:p * 64 + n, 1])
    ov, _ = lay["v_codes"]
    vc = quant.unpack(pg[1, 0, ov:ov + 128 * 32].reshape(128, 32), 4, 64)
    assert np.array_equal(vc, a["vc"][1, 0])
    om, _ = lay["v_meta"]
    vm = pg[1, 0, om:om + 512].view(np.float16).reshape(128, 2)
    assert np.array_equal(vm[:, 0].astype(np.float32), a["vm"][1, 0])
    assert not mk[2, 0, ov:ov + 16].any()        # partial page: V section undefined


# ----------------------------------------------------------------- P-code substitution

def test_pcodes_override_pins_the_near_tie_substitution():
    """The near-tie protocol's step 3 re-runs the oracle with the GPU's P codes
    (`pcodes_override`).  Pins: (1) substituting the oracle's own codes changes nothing;
    (2) raising one code p'_{r,t} by 1 in committed block j changes exactly row r, by the
    closed form s_p(r, j) * v_hat_t -- Eq. 4 with SP recomputed from the substituted codes
    (sum_t (s_p p'_t + m_p)(s_v v'_t + m_v)); keeping the old SP would give
    s_p s_v v'_t instead, an index mix-up would move another row or key; (3) the decode
    entry point substitutes the same way."""
    c = cfg(Hq=2, Hkv=1)
    L = 150                                   # 2 committed V blocks + 22 FP16 tail tokens
    q, k, v = hack_inputs.qkv(21, L, 2, 1)
    O, st, diag = att.prefill(c, q, k, v, rng_id=9, keep_diag=True)
    own = {hq: diag[hq]["pcodes"] for hq in diag}
    O1, _, _ = att.prefill(c, q, k, v, rng_id=9, pcodes_override=own)
    assert np.array_equal(O1, O)
    hq, r, t = 1, 140, 70                     # key 70 lies in block j = 1, visible to row 140
    j = t // c.Pi
    P = diag[hq]["P"][r, j * c.Pi:(j + 1) * c.Pi]
    s_p = (P.max() - P.min()) / 255.0
    bumped = {h: own[h].copy() for h in own}
    assert bumped[hq][r, t] < 255
    bumped[hq][r, t] += 1
    O2, _, _ = att.prefill(c, q, k, v, rng_id=9, pcodes_override=bumped)
    dO = O2 - O
    vh = v_hat(st, 0)[t]
    assert np.allclose(dO[r, hq], s_p * vh, rtol=1e-9, atol=1e-14)
    dO[r, hq] = 0
    assert np.abs(dO).max() < 1e-15
    a = st.arrays()
    assert not np.allclose(s_p * vh, s_p * a["vs"][j, 0] * a["vc"][j, 0, :, t - j * c.Pi])   # the SP term matters
    # decode: the last query row of a 150-token cache, same substitution
    st2 = att.ingest_prompt(c, k, v, rng_id=9)
    qn = hack_inputs.qkv(22, 1, 2, 1)[0][0]
    Od, dg = att.decode_attend(st2, qn, keep_diag=True)
    codes = {h: dg[h]["pcodes"].copy() for h in dg}
    Od1, _ = att.decode_attend(st2, qn, pcodes_override=codes)
    assert np.array_equal(Od1, Od)
    Pd = dg[0]["P"][0, j * c.Pi:(j + 1) * c.Pi]
    codes[0][0, t] = codes[0][0, t] + 1 if codes[0][0, t] < 255 else 254
    sgn = 1 if dg[0]["pcodes"][0, t] < 255 else -1
    Od2, _ = att.decode_attend(st2, qn, pcodes_override=codes)
    assert np.allclose(Od2[0] - Od[0], sgn * (Pd.max() - Pd.min()) / 255.0 * v_hat(st2, 0)[t], rtol=1e-9, atol=1e-14)
    assert np.array_equal(Od2[1], Od[1])


# ----------------------------------------------------------------- P stochastic rounding (R6, selectable)

def test_p_sr_extremes_and_rn_default():
    """quantize_p 'sr' is floor(y) + [u < frac(y)] (R1): u = 0 gives ceil(y) off the grid and
    y on it; u -> 1 gives floor(y); the default stays round-to-nearest-even."""
    g = np.random.default_rng(3)
    p = np.concatenate([[0.0, 1.0], g.random(62)])[None]               # lo = 0, hi = 1: y = 255 p
    y = 255.0 * p
    c0, *_ = att.quantize_p(p, "sr", np.zeros_like(p, np.float32))
    c1, *_ = att.quantize_p(p, "sr", np.full_like(p, 1 - 2.0 ** -24, np.float32))
    assert np.array_equal(c0, np.ceil(y).astype(np.uint8))
    assert np.array_equal(c1, np.floor(y).astype(np.uint8))
    crn, *_ = att.quantize_p(p)
    assert np.array_equal(crn, np.rint(y).astype(np.uint8))
    with pytest.raises(ValueError):
        att.quantize_p(p, "sr")


def test_p_sr_unbiased_over_streams():
    """E[p_hat] = p under SR: dequantized P averaged over 4000 independent
    position-keyed streams (rng ids) is within 4 sigma of p for every key."""
    from oracle import philox
    g = np.random.default_rng(4)
    p = g.random(64)
    n = 4000
    u = np.stack([philox.uniforms_p(7, rid, 0, 3, [100], np.arange(64))[0] for rid in range(n)])
    c, lo, s, _, y = att.quantize_p(np.broadcast_to(p, (n, 64)), "sr", u)
    phat = lo[:, None] + s[:, None] * c
    frac = y[0] - np.floor(y[0])
    sigma = s[0] * np.sqrt(frac * (1 - frac) / n) + 1e-15
    assert (np.abs(phat.mean(0) - p) <= 4 * sigma + 1e-12).all()


def test_p_sr_counter_map_is_position_keyed():
    """u(i, t) depends only on (query position, key position, head, request, layer): the
    same element drawn through different key ranges agrees; distinct elements differ."""
    from oracle import philox
    a = philox.uniforms_p(9, 5, 2, 1, [7, 300], np.arange(0, 128))
    b = philox.uniforms_p(9, 5, 2, 1, [300], np.arange(64, 192))
    assert np.array_equal(a[1, 64:], b[0, :64])
    grid = philox.uniforms_p(9, 5, 2, 1, np.arange(64), np.arange(256))
    assert len(np.unique(grid)) > 0.999 * grid.size
    assert not np.array_equal(philox.uniforms_p(9, 5, 2, 2, [7], np.arange(8)), a[:1, :8])


def test_p_sr_decode_row_equals_prefill_row():
    """With P stochastic rounding, the decode step's P codes are the last prefill row's
    (position-keyed counters), and the outputs agree (SR pins the same code choices)."""
    c = cfg(Hq=4, Hkv=2, p_round="sr")
    L = 200
    q, k, v = hack_inputs.qkv(41, L, 4, 2)
    O, _, dg = att.prefill(c, q, k, v, rng_id=3, rows=[L - 1], keep_diag=True)
    st = att.ingest_prompt(c, k[:L - 1], v[:L - 1], rng_id=3)
    o, dd = att.decode_step(st, q[L - 1], k[L - 1], v[L - 1], keep_diag=True)
    for hq in range(4):
        assert np.array_equal(dd[hq]["pcodes"], dg[hq]["pcodes"])
    assert np.allclose(o, O[L - 1], rtol=1e-12, atol=1e-14)
    Orn, _, _ = att.prefill(cfg(Hq=4, Hkv=2), q, k, v, rng_id=3, rows=[L - 1])
    assert not np.array_equal(O[L - 1], Orn[L - 1])                    # the mode changes the codes
