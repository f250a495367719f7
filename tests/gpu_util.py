"""Helpers for the GPU parity tests: run the CUDA path through the C ABI, run the
oracle on the same seeded inputs, compare."""
from __future__ import annotations

import numpy as np
import torch

from oracle import attention as att
from oracle import pages as opages

ROW_TOL = 1e-3          # north star: max relative error <= 1e-3 (R18 row-relative)
NEAR_TIE = 1e-2         # delta of the P-code near-tie protocol (SURVEY c-4)


def hk():
    from paper_2502_03589_b200 import hack
    return hack


def gpu_cfg(ocfg: att.Config, out_fp32=True):
    h = hk()
    return h.config(num_q_heads=ocfg.Hq, num_kv_heads=ocfg.Hkv, partition=ocfg.Pi, kv_bits=ocfg.bits,
                    kv_round=0 if ocfg.kv_round == "sr" else 1, q_round=0 if ocfg.q_round == "sr" else 1,
                    p_round=0 if ocfg.p_round == "sr" else 1,
                    seed=ocfg.seed, layer=ocfg.layer, head_base=ocfg.head_base, out_fp32=out_fp32)


def row_rel_err(O_gpu: np.ndarray, O_ref: np.ndarray) -> np.ndarray:
    """R18: per output row r, ||O_gpu - O_ref||_inf / max(||O_ref||_inf, 1e-6)."""
    num = np.abs(O_gpu - O_ref).max(-1)
    den = np.maximum(np.abs(O_ref).max(-1), 1e-6)
    return num / den


def check_pcodes(gpu_codes: np.ndarray, ora_codes: np.ndarray, ora_y: np.ndarray, ora_u: np.ndarray | None = None):
    """Every P-code mismatch must be a near-tie of the oracle's fp64 y and off by one: the
    RN boundary is k + 1/2; under stochastic rounding (ora_u given) c = ceil(y - u), so the
    boundary is y - u integer.  Returns the number of mismatches."""
    mism = gpu_codes != ora_codes
    if mism.any():
        y = ora_y[mism]
        if ora_u is None:
            dist = np.abs(y - (np.floor(y) + 0.5))
        else:
            z = y - np.asarray(ora_u, np.float64)[mism]
            dist = np.abs(z - np.rint(z))
        bad = (dist >= NEAR_TIE) | (np.abs(gpu_codes[mism].astype(int) - ora_codes[mism].astype(int)) > 1)
        assert not bad.any(), f"{bad.sum()} non-near-tie P-code mismatches (max dist {dist.max():.3g})"
    return int(mism.sum())


def make_cache(cfg, max_reqs, max_len, extra_pages=0, scramble=True, seed=0):
    """A cache whose block tables map to a shuffled page pool (exercises paging)."""
    h = hk()
    mp = (max_len + cfg.partition - 1) // cfg.partition
    n = max_reqs * mp + extra_pages
    cache = h.KVCache.allocate(cfg, max_reqs, mp, num_pages=n)
    if scramble:
        perm = torch.from_numpy(np.random.default_rng(seed).permutation(n)[: max_reqs * mp].astype(np.int32))
        cache.block_table.copy_(perm.reshape(max_reqs, mp).cuda())
    return cache


def gpu_pages_of(cache, slot, npages):
    bt = cache.block_table[slot, :npages].long()
    return cache.pages[bt].cpu().numpy()


def compare_pages(cache, slot, state):
    """GPU page bytes of one request == the oracle's packed pages (defined bytes)."""
    ref, mask = opages.pack_request(state)
    got = gpu_pages_of(cache, slot, ref.shape[0])
    bad = (got != ref) & mask
    assert not bad.any(), f"{bad.sum()} page bytes differ (first at {np.argwhere(bad)[0]})"
    # FP16 tail
    a = state.arrays()
    T = a["tail"].shape[0]
    if T:
        tail = cache.v_tail[slot, :, :T].cpu().numpy()              # [Hkv, T, d]
        assert np.array_equal(tail.transpose(1, 0, 2).view(np.uint16), a["tail"].view(np.uint16))


# ---------------------------------------------------------------- MMA accumulator dumps
# The hot kernels can dump their own int32 block accumulators (hack_debug_t.qk_acc /
# pv_acc).  Each kernel's accumulator is an exact affine function of the paper's integer
# block product D = sum_{z in block} a'_z b'_z (Eq. 4); the form is
# reported by hack_debug_acc_form.  D comes from
# oracle.homomm.int_blocks on the oracle's codes (QK) or on the GPU's own P codes with the
# oracle's V codes (PV: P codes may differ from the oracle's at near-ties).

def acc_expected(form, D, SA, SB, bits, Pi):
    h = hk()
    qkm = (1 << bits) - 1
    D = np.asarray(D, np.int64)
    if form == h.ACC_PLAIN:
        return D
    if form == h.ACC_S8_2B:                       # (a' - 128) x 2 b'
        return 2 * D - 256 * np.asarray(SB, np.int64)
    if form == h.ACC_CENTERED4:                   # 4 D - 2(2^b - 1) S_A + Pi 255 (2^b - 1)
        return 4 * D - 2 * qkm * np.asarray(SA, np.int64) + Pi * 255 * qkm
    raise AssertionError(f"no accumulator form {form}")


def acc_buffers(rows, heads, ocfg, stride):
    """Device int32 dump buffers: qk [rows, heads, d/Pi, stride], pv [rows, heads, stride/Pi, d]."""
    qk = torch.full((rows, heads, ocfg.nbeta, stride), -7, dtype=torch.int32, device="cuda")
    pv = torch.full((rows, heads, stride // ocfg.Pi, ocfg.d), -7, dtype=torch.int32, device="cuda")
    return qk, pv


def check_acc(form, ocfg, state, qc, qsum, pos, hq, got_qk, got_pv, gpu_pcodes):
    """One query head hq (local index), query rows at positions `pos` (one row per entry):
    got_qk [n, d/Pi, stride], got_pv [n, stride/Pi, d], gpu_pcodes [n, >= nfull*Pi].
    QK: every key t <= pos; PV: every committed block j with j*Pi <= pos.  Bit-exact."""
    from oracle import homomm
    a = state.arrays()
    Pi, b = ocfg.Pi, ocfg.bits
    hkv = hq // ocfg.G
    pos = np.asarray(pos)
    L = a["kc"].shape[0]
    D = homomm.int_blocks(qc[:, hq, :], a["kc"][:, hkv, :].T, Pi)           # [nb, n, L]
    exp = acc_expected(form, D, qsum[:, hq, :].T[:, :, None], a["ksum"][:, hkv, :].T[:, None, :], b, Pi)
    got = np.asarray(got_qk)[:, :, :L].transpose(1, 0, 2)
    vis = np.arange(L)[None, :] <= pos[:, None]
    bad = (got != exp) & vis[None]
    assert not bad.any(), f"QK accumulator: {bad.sum()} of {vis.sum() * ocfg.nbeta} differ (first {np.argwhere(bad)[0]})"
    nfull = a["vc"].shape[0]
    nchk = 0
    for j in range(nfull):
        rows = pos >= j * Pi
        if not rows.any():
            continue
        P = np.asarray(gpu_pcodes)[rows, j * Pi:(j + 1) * Pi]                # [n', Pi]
        Dp = homomm.int_blocks(P, a["vc"][j, hkv].T, Pi)[0]                  # [n', d]
        e = acc_expected(form, Dp, P.astype(np.int64).sum(1)[:, None], a["vsum"][j, hkv][None, :], b, Pi)
        g = np.asarray(got_pv)[rows, j]
        assert np.array_equal(g, e), f"PV accumulator block {j}: {(g != e).sum()} differ"
        nchk += rows.sum()
    return int(vis.sum()) * ocfg.nbeta, nchk * ocfg.d
