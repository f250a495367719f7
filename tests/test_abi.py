"""The C-ABI library loads, exports every symbol include/hack.h declares, and its
host-side logic (validation, layout, transfer sizes) agrees with the oracle /
closed forms.  No compute call needs a GPU here (and none falls back to CPU)."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hack.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hack_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def hk():
    from paper_2502_03589_b200 import hack
    return hack


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("hack_quantize_pack", "hack_prefill_attention", "hack_decode_attention", "hack_kv_send",
              "hack_kv_recv"):
        assert s in syms


def test_every_declared_symbol_is_exported(hk):
    lib = hk.library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and through a fresh dlopen (no python-side aliasing)
    raw = ctypes.CDLL(hk.LIB_PATH)
    for s in declared_symbols():
        getattr(raw, s)


def test_abi_version_and_default_config(hk):
    assert hk.abi_version() == 2
    c = hk.config()
    assert (c.head_dim, c.partition, c.kv_bits, c.kv_round, c.q_round, c.p_round) == (128, 64, 2, 0, 0, 1)
    hk.config_validate(c)


@pytest.mark.parametrize("kw,status", [
    (dict(kv_bits=3), 1),                       # S:545 '--bits 3 usage error' -> INVALID_ARG
    (dict(partition=16), 2),                    # R16: Pi=16 unsupported
    (dict(partition=48), 2),
    (dict(head_dim=64), 2),
    (dict(num_q_heads=6, num_kv_heads=4), 3),   # H_q % H_kv != 0 -> SHAPE
    (dict(num_q_heads=34, num_kv_heads=2), 2),  # G = 17 > 16
    (dict(p_round=5), 1),                       # P rounding: RN (R6 default) or SR
    (dict(kv_round=5), 1),
])
def test_config_validation_errors(hk, kw, status):
    c = hk.config(**kw)
    with pytest.raises(hk.HackError) as e:
        hk.config_validate(c)
    assert e.value.status == status
    assert len(hk.library().hack_last_error()) > 0


@pytest.mark.parametrize("Pi,bits", [(32, 2), (64, 2), (128, 2), (32, 4), (64, 4), (128, 4)])
def test_page_layout_matches_oracle_spec(hk, Pi, bits):
    from oracle import pages
    c = hk.config(partition=Pi, kv_bits=bits)
    lay = hk.page_layout(c)
    ref = pages.layout(128, Pi, bits)
    for k in ("k_codes", "k_meta", "k_sums", "v_codes", "v_meta", "v_sums"):
        assert lay[k] == ref[k], k
    assert hk.page_bytes(c) == ref["page_bytes"]


def test_kv_transfer_bytes_closed_form(hk):
    from oracle import pages
    c = hk.config(num_q_heads=32, num_kv_heads=8)
    for L in (1, 63, 64, 65, 4096, 16200):
        npages = (L + 63) // 64
        T = L % 64
        per_layer = npages * 8 * pages.layout(128, 64, 2)["page_bytes"] + 8 * T * 128 * 2
        assert hk.kv_transfer_bytes(c, 32, L) == 64 + 32 * per_layer
    # S:591 / P:896: packed bytes per token ~ 16.4% of fp16 K+V
    assert hk.kv_transfer_bytes(c, 1, 4096) / (4096 * 8 * 128 * 2 * 2) < 0.17
    assert hk.kv_transfer_bytes(c, 0, 10) == -1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_compute_without_gpu_fails_loudly(hk):
    # no CPU fallback: host pointers / no device -> HACK_ERR_CUDA, never a silent result
    c = hk.config()
    x = np.zeros((64, 1, 128), np.float16)
    out = np.zeros(64 * 32, np.uint8)
    meta = np.zeros(64 * 2 * 4, np.uint8)
    sums = np.zeros(64 * 2, np.uint8)
    with pytest.raises(hk.HackError) as e:
        hk.quantize_pack(c, hk.QMODE_K, torch.from_numpy(x), out.ctypes.data, meta.ctypes.data,
                         sums.ctypes.data, stream=0)
    assert e.value.status == hk.ERR_CUDA


def test_argument_errors_detected_before_launch(hk):
    c = hk.config()
    lib = hk.library()
    st = lib.hack_quantize_pack(ctypes.byref(c), 0, None, 4, 1, 0, 0, 0, None, None, None, None)
    assert st == hk.ERR_INVALID_ARG
    st = lib.hack_quantize_pack(ctypes.byref(c), 7, 1, 4, 1, 0, 0, 0, 1, 1, 1, None)
    assert st == hk.ERR_INVALID_ARG
    st = lib.hack_quantize_pack(ctypes.byref(c), hk.QMODE_V, 1, 65, 1, 0, 0, 0, 1, 1, 1, None)
    assert st == hk.ERR_SHAPE   # V rows must be a multiple of Pi


def test_debug_acc_form_follows_dispatch(hk, monkeypatch):
    """hack_debug_acc_form names the affine form of the accumulator dump of the kernel the
    next call dispatches to (include/hack.h); host logic only, no GPU needed."""
    c = hk.config(num_q_heads=4, num_kv_heads=1)
    assert hk.debug_acc_form(c, "prefill") == hk.ACC_S8_2B          # prefill_tc (tcgen05)
    assert hk.debug_acc_form(c, "decode") == hk.ACC_CENTERED4       # decode_pair (b = 2, Pi = 64)
    assert hk.debug_acc_form(hk.config(num_q_heads=8, num_kv_heads=1), "decode") == hk.ACC_CENTERED4  # g8
    assert hk.debug_acc_form(hk.config(kv_bits=4), "decode") == hk.ACC_PLAIN   # decode_mma
    assert hk.debug_acc_form(hk.config(partition=32), "decode") == hk.ACC_PLAIN
    assert hk.debug_acc_form(hk.config(num_q_heads=16, num_kv_heads=1), "decode") == hk.ACC_NONE  # simt
    monkeypatch.setenv("HACK_DECODE_IMPL", "simt")
    assert hk.debug_acc_form(c, "decode") == hk.ACC_NONE
    monkeypatch.setenv("HACK_PREFILL_IMPL", "simt")
    assert hk.debug_acc_form(c, "prefill") == hk.ACC_NONE


def test_prefill_host_rejects_bad_arguments_before_any_work(hk):
    """hack_prefill_attention_host validates its host index arrays and workspace before it
    enqueues anything (no GPU needed to reach these errors)."""
    cfg = hk.config(num_q_heads=4, num_kv_heads=1)
    assert hk.prefill_host_workspace_size(cfg, 1, 100) > 100 * 4 * 128 * 2 * 2
    assert hk.prefill_host_workspace_size(cfg, 0, 100) == 0
    lib = hk.library()
    cache = hk.CacheStruct(1, 1, 1, 1, 1, 4, 1, 2, hk.page_bytes(cfg))
    buf = (ctypes.c_uint8 * 64)()
    cu = (ctypes.c_int32 * 2)(0, 0)          # empty prompt
    sl = (ctypes.c_int32 * 1)(0)
    st = lib.hack_prefill_attention_host(ctypes.byref(cfg), buf, buf, buf, cu, sl, 1, 64, ctypes.byref(cache), buf,
                                         buf, 64, 0, None)
    assert st == 1, lib.hack_last_error().decode()        # INVALID_ARG
    cu = (ctypes.c_int32 * 2)(0, 64)
    st = lib.hack_prefill_attention_host(ctypes.byref(cfg), buf, buf, buf, cu, sl, 1, 64, ctypes.byref(cache), buf,
                                         buf, 64, 0, None)
    assert st == 4, lib.hack_last_error().decode()        # CAPACITY: workspace too small
