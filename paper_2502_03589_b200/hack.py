"""Thin ctypes binding of libhack.so (include/hack.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  torch supplies device memory and streams.  There is no CPU
fallback -- if libhack.so is missing the import fails, and on a machine without
an sm_100 GPU every compute call raises HackError(HACK_ERR_CUDA).

Names follow the C ABI without the `hack_` prefix.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhack.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2502_03589_b200/build.py` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_SHAPE, ERR_CAPACITY, ERR_PROTOCOL, ERR_CUDA, ERR_NCCL = range(8)
STATUS_NAMES = ["OK", "INVALID_ARG", "UNSUPPORTED", "SHAPE", "CAPACITY", "PROTOCOL", "CUDA", "NCCL"]
ROUND_STOCHASTIC, ROUND_NEAREST_EVEN = 0, 1
QMODE_K, QMODE_V, QMODE_Q = 0, 1, 2


class HackError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.hack_last_error().decode()
        super().__init__(f"{where}: HACK_ERR_{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("partition", C.c_int32), ("kv_bits", C.c_int32), ("kv_round", C.c_int32),
                ("q_round", C.c_int32), ("p_round", C.c_int32), ("seed", C.c_uint64),
                ("layer", C.c_int32), ("head_base", C.c_int32), ("out_dtype", C.c_int32),
                ("reserved", C.c_int32)]


class CacheStruct(C.Structure):
    _fields_ = [("pages", C.c_void_p), ("v_tail", C.c_void_p), ("block_table", C.c_void_p),
                ("seq_lens", C.c_void_p), ("rng_ids", C.c_void_p), ("num_pages", C.c_int32),
                ("max_reqs", C.c_int32), ("max_pages_per_req", C.c_int32), ("page_bytes", C.c_int32)]


class DebugStruct(C.Structure):
    _fields_ = [("pcodes", C.c_void_p), ("pcodes_stride", C.c_int64), ("qk_acc", C.c_void_p),
                ("pv_acc", C.c_void_p), ("acc_stride", C.c_int64), ("acc_head", C.c_int32),
                ("reserved", C.c_int32)]


# hack_acc_form_t: affine form of the dumped MMA accumulators (include/hack.h)
ACC_NONE, ACC_PLAIN, ACC_S8_2B, ACC_CENTERED4 = range(4)


_S = C.c_int
_P = C.c_void_p
_lib.hack_last_error.restype = C.c_char_p
_lib.hack_version.restype = C.c_char_p
_lib.hack_abi_version.restype = C.c_int32
_lib.hack_kernel_launches.restype = C.c_int64
_lib.hack_page_bytes.restype = C.c_int64
_lib.hack_kv_transfer_bytes.restype = C.c_int64
_lib.hack_prefill_workspace_size.restype = C.c_size_t
_lib.hack_decode_workspace_size.restype = C.c_size_t
_lib.hack_config_default.restype = None
_lib.hack_debug_acc_form.restype = C.c_int32
for _name in ("hack_config_validate", "hack_page_layout", "hack_quantize_pack", "hack_cache_ingest",
              "hack_prefill_attention", "hack_prefill_attention_cached", "hack_prefill_attention_host",
              "hack_decode_append",
              "hack_decode_attention", "hack_decode_attention_cached", "hack_homomorphic_matmul",
              "hack_comm_unique_id", "hack_comm_init", "hack_comm_destroy", "hack_kv_pack", "hack_kv_unpack",
              "hack_kv_send", "hack_kv_recv", "hack_kv_send_layer", "hack_kv_recv_layer", "hack_kv_pull",
              "hack_comm_recv_bytes", "hack_comm_group_start",
              "hack_comm_group_end"):
    getattr(_lib, _name).restype = _S

_lib.hack_quantize_pack.argtypes = [C.POINTER(Config), C.c_int32, _P, C.c_int64, C.c_int32, C.c_int64, C.c_int32,
                                    C.c_uint32, _P, _P, _P, _P]
_lib.hack_cache_ingest.argtypes = [C.POINTER(Config), _P, _P, _P, _P, C.c_int32, C.c_int32,
                                   C.POINTER(CacheStruct), _P]
_lib.hack_prefill_attention.argtypes = [C.POINTER(Config), _P, _P, _P, _P, _P, C.c_int32, C.c_int32,
                                        C.POINTER(CacheStruct), _P, _P, C.c_size_t, C.POINTER(DebugStruct), _P]
_lib.hack_prefill_attention_cached.argtypes = [C.POINTER(Config), _P, _P, _P, C.c_int32, C.c_int32,
                                               C.POINTER(CacheStruct), _P, _P, C.c_size_t,
                                               C.POINTER(DebugStruct), _P]
_lib.hack_prefill_attention_host.argtypes = [C.POINTER(Config), _P, _P, _P, _P, _P, C.c_int32, C.c_int32,
                                             C.POINTER(CacheStruct), _P, _P, C.c_size_t, C.c_int32, _P]
_lib.hack_prefill_host_workspace_size.restype = C.c_size_t
_lib.hack_prefill_host_workspace_size.argtypes = [C.POINTER(Config), C.c_int32, C.c_int32]
_lib.hack_decode_append.argtypes = [C.POINTER(Config), _P, _P, _P, C.c_int32, C.POINTER(CacheStruct), _P]
_lib.hack_decode_attention.argtypes = [C.POINTER(Config), _P, _P, _P, _P, C.c_int32, C.c_int32,
                                       C.POINTER(CacheStruct), _P, _P, C.c_size_t, C.POINTER(DebugStruct), _P]
_lib.hack_decode_attention_cached.argtypes = [C.POINTER(Config), _P, _P, C.c_int32, C.c_int32,
                                              C.POINTER(CacheStruct), _P, _P, C.c_size_t,
                                              C.POINTER(DebugStruct), _P]
_lib.hack_dequantize_cache.argtypes = [C.POINTER(Config), _P, C.c_int32, C.c_int32, C.POINTER(CacheStruct), _P, _P,
                                       _P]
_lib.hack_homomorphic_matmul.argtypes = [C.POINTER(Config), _P, _P, _P, _P, _P, _P, C.c_int32, C.c_int32,
                                         C.c_int32, _P, _P, _P]
_lib.hack_prefill_workspace_size.argtypes = [C.POINTER(Config), C.c_int32, C.c_int32]
_lib.hack_debug_acc_form.argtypes = [C.POINTER(Config), C.c_int32]
_lib.hack_decode_workspace_size.argtypes = [C.POINTER(Config), C.c_int32, C.c_int32]
_lib.hack_page_bytes.argtypes = [C.POINTER(Config)]
_lib.hack_page_layout.argtypes = [C.POINTER(Config), C.POINTER(C.c_int64 * 12)]
_lib.hack_kv_transfer_bytes.argtypes = [C.POINTER(Config), C.c_int32, C.c_int32]
_lib.hack_comm_init.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_char_p]
_lib.hack_comm_destroy.argtypes = [_P]
_lib.hack_kv_pack.argtypes = [C.POINTER(Config), C.POINTER(CacheStruct), C.c_int32, C.c_int32, C.c_int32,
                              C.c_int32, C.c_uint32, _P, _P]
_lib.hack_kv_unpack.argtypes = [C.POINTER(Config), C.POINTER(CacheStruct), C.c_int32, C.c_int32, C.c_int32, _P,
                                _P, _P]
_lib.hack_kv_send.argtypes = [_P, C.c_int32, C.POINTER(Config), C.POINTER(CacheStruct), C.c_int32, C.c_int32,
                              C.c_int32, C.c_int32, C.c_uint32, _P, _P]
_lib.hack_kv_recv.argtypes = [_P, C.c_int32, C.POINTER(Config), C.POINTER(CacheStruct), C.c_int32, C.c_int32,
                              C.c_int32, _P, _P, _P]
_lib.hack_comm_recv_bytes.argtypes = [_P, C.c_int32, _P, C.c_int64, _P]
_lib.hack_kv_pull.argtypes = [C.POINTER(Config), C.POINTER(CacheStruct), C.POINTER(CacheStruct), C.c_int32,
                              C.c_int32, C.c_int32, C.c_int32, _P]
_lib.hack_kv_layer_range.restype = C.c_int64
_lib.hack_kv_layer_range.argtypes = [C.POINTER(Config), C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]
_lib.hack_kv_send_layer.argtypes = [_P, C.c_int32, C.POINTER(Config), C.POINTER(CacheStruct), C.c_int32, C.c_int32,
                                    C.c_int32, C.c_int32, C.c_int32, C.c_uint32, _P, _P]
_lib.hack_kv_recv_layer.argtypes = [_P, C.c_int32, C.POINTER(Config), C.c_int32, C.c_int32, C.c_int32, _P, _P]


def _check(st: int, where: str):
    if st != OK:
        raise HackError(st, where)


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return int(t)


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def version() -> str:
    return _lib.hack_version().decode()


def abi_version() -> int:
    return int(_lib.hack_abi_version())


def kernel_launches() -> int:
    """Kernels libhack has launched in this process."""
    return int(_lib.hack_kernel_launches())


def library():
    """The loaded ctypes CDLL (symbol-export tests)."""
    return _lib


def config(num_q_heads=1, num_kv_heads=1, head_dim=128, partition=64, kv_bits=2, kv_round=ROUND_STOCHASTIC,
           q_round=ROUND_STOCHASTIC, p_round=ROUND_NEAREST_EVEN, seed=0x48414B, layer=0, head_base=0,
           out_fp32=False) -> Config:
    c = Config()
    _lib.hack_config_default(C.byref(c))
    c.num_q_heads, c.num_kv_heads, c.head_dim, c.partition, c.kv_bits = (num_q_heads, num_kv_heads, head_dim,
                                                                          partition, kv_bits)
    c.kv_round, c.q_round, c.p_round, c.seed = kv_round, q_round, p_round, seed
    c.layer, c.head_base, c.out_dtype = layer, head_base, 1 if out_fp32 else 0
    return c


def config_validate(cfg: Config):
    _check(_lib.hack_config_validate(C.byref(cfg)), "config_validate")


def page_bytes(cfg: Config) -> int:
    n = _lib.hack_page_bytes(C.byref(cfg))
    if n < 0:
        raise HackError(_lib.hack_config_validate(C.byref(cfg)), "page_bytes")
    return int(n)


def page_layout(cfg: Config) -> dict:
    arr = (C.c_int64 * 12)()
    _check(_lib.hack_page_layout(C.byref(cfg), C.byref(arr)), "page_layout")
    names = ("k_codes", "k_meta", "k_sums", "v_codes", "v_meta", "v_sums")
    return {n: (int(arr[2 * i]), int(arr[2 * i + 1])) for i, n in enumerate(names)}


def kv_transfer_bytes(cfg: Config, num_layers: int, prompt_len: int) -> int:
    return int(_lib.hack_kv_transfer_bytes(C.byref(cfg), num_layers, prompt_len))


def sum_bytes(cfg: Config) -> int:
    lay = page_layout(cfg)
    return lay["k_sums"][1] // (cfg.partition * (cfg.head_dim // cfg.partition))


# --------------------------------------------------------------------------- cache

@dataclass
class KVCache:
    """One layer's paged packed-KV cache in torch device memory (plumbing only)."""
    cfg: Config
    pages: torch.Tensor        # u8 [num_pages, H_kv, page_bytes]
    v_tail: torch.Tensor       # fp16 [max_reqs, H_kv, Pi, d]
    block_table: torch.Tensor  # i32 [max_reqs, max_pages_per_req]
    seq_lens: torch.Tensor     # i32 [max_reqs]
    rng_ids: torch.Tensor      # i32 (u32 bits) [max_reqs]

    @classmethod
    def allocate(cls, cfg: Config, max_reqs: int, max_pages_per_req: int, num_pages: int | None = None,
                 device="cuda", shared_tables: "KVCache | None" = None) -> "KVCache":
        pb = page_bytes(cfg)
        num_pages = num_pages if num_pages is not None else max_reqs * max_pages_per_req
        pages = torch.zeros((num_pages, cfg.num_kv_heads, pb), dtype=torch.uint8, device=device)
        tail = torch.zeros((max_reqs, cfg.num_kv_heads, cfg.partition, cfg.head_dim), dtype=torch.float16,
                           device=device)
        if shared_tables is not None:
            bt, sl, rid = shared_tables.block_table, shared_tables.seq_lens, shared_tables.rng_ids
        else:
            bt = torch.arange(max_reqs * max_pages_per_req, dtype=torch.int32, device=device).reshape(
                max_reqs, max_pages_per_req) % num_pages
            sl = torch.zeros(max_reqs, dtype=torch.int32, device=device)
            rid = torch.zeros(max_reqs, dtype=torch.int32, device=device)
        return cls(cfg, pages, tail, bt, sl, rid)

    def struct(self) -> CacheStruct:
        s = CacheStruct()
        s.pages, s.v_tail = self.pages.data_ptr(), self.v_tail.data_ptr()
        s.block_table, s.seq_lens, s.rng_ids = (self.block_table.data_ptr(), self.seq_lens.data_ptr(),
                                                self.rng_ids.data_ptr())
        s.num_pages = self.pages.shape[0]
        s.max_reqs, s.max_pages_per_req = self.block_table.shape
        s.page_bytes = self.pages.shape[2]
        return s


def _dbg(pcodes: torch.Tensor | None, qk_acc: torch.Tensor | None = None, pv_acc: torch.Tensor | None = None,
         acc_head: int = -1):
    """hack_debug_t: pcodes u8 [rows, H_q, stride]; qk_acc int32 [rows, H_q, d/Pi, acc_stride];
    pv_acc int32 [rows, H_q, acc_stride/Pi, d] (parity runs only).  acc_head >= 0 dumps only
    that query head's accumulators, into [rows, 1, ...] arrays."""
    if pcodes is None and qk_acc is None and pv_acc is None:
        return None
    d = DebugStruct()
    d.acc_head = acc_head
    if pcodes is not None:
        d.pcodes, d.pcodes_stride = pcodes.data_ptr(), pcodes.shape[-1]
    if qk_acc is not None:
        d.qk_acc, d.acc_stride = qk_acc.data_ptr(), qk_acc.shape[-1]
    if pv_acc is not None:
        if qk_acc is None:
            raise ValueError("pv_acc needs qk_acc (the shared acc_stride comes from it)")
        d.pv_acc = pv_acc.data_ptr()
    return C.byref(d)


def debug_acc_form(cfg: Config, op: str) -> int:
    """ACC_* form of the accumulator dump of the kernel the next prefill / decode call uses."""
    return int(_lib.hack_debug_acc_form(C.byref(cfg), {"prefill": 0, "decode": 1}[op]))


# --------------------------------------------------------------------------- calls

def quantize_pack(cfg: Config, mode: int, x: torch.Tensor, codes, meta, sums, pos0: int = 0, head0: int = 0,
                  rng_id: int = 0, stream=None):
    rows, heads = x.shape[0], x.shape[1]
    _check(_lib.hack_quantize_pack(C.byref(cfg), mode, _ptr(x), rows, heads, pos0, head0, rng_id & 0xFFFFFFFF,
                                   _ptr(codes), _ptr(meta), _ptr(sums), _stream(stream)), "quantize_pack")


def cache_ingest(cfg: Config, k, v, cu_seqlens, slots, max_seqlen: int, cache: KVCache, stream=None):
    cs = cache.struct()
    _check(_lib.hack_cache_ingest(C.byref(cfg), _ptr(k), _ptr(v), _ptr(cu_seqlens), _ptr(slots),
                                  slots.shape[0], max_seqlen, C.byref(cs), _stream(stream)), "cache_ingest")


def prefill_workspace_size(cfg: Config, batch: int, max_seqlen: int) -> int:
    return int(_lib.hack_prefill_workspace_size(C.byref(cfg), batch, max_seqlen))


def decode_workspace_size(cfg: Config, batch: int, max_seqlen: int) -> int:
    return int(_lib.hack_decode_workspace_size(C.byref(cfg), batch, max_seqlen))


def _ws(workspace, nbytes, device):
    if nbytes == 0:
        return None, 0
    if workspace is None:
        # zero-filled: the decode workspace holds merge counters that must start at zero
        # (hack.h); the library leaves them zero after every launch
        workspace = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    return workspace, workspace.numel()


def prefill_attention(cfg: Config, q, k, v, cu_seqlens, slots, max_seqlen: int, cache: KVCache, out,
                      workspace=None, debug_pcodes=None, debug_qk=None, debug_pv=None, debug_head=-1, stream=None):
    cs = cache.struct()
    ws, nb = _ws(workspace, prefill_workspace_size(cfg, slots.shape[0], max_seqlen), q.device)
    _check(_lib.hack_prefill_attention(C.byref(cfg), _ptr(q), _ptr(k), _ptr(v), _ptr(cu_seqlens), _ptr(slots),
                                       slots.shape[0], max_seqlen, C.byref(cs), _ptr(out), _ptr(ws), nb,
                                       _dbg(debug_pcodes, debug_qk, debug_pv, debug_head), _stream(stream)), "prefill_attention")


def prefill_host_workspace_size(cfg: Config, batch: int, total_tokens: int) -> int:
    return _lib.hack_prefill_host_workspace_size(C.byref(cfg), batch, total_tokens)


def prefill_attention_host(cfg: Config, q, k, v, cu_seqlens, slots, max_seqlen: int, cache: KVCache, out,
                           workspace=None, head_chunks: int = 0, stream=None):
    """hack_prefill_attention with HOST q / k / v / cu_seqlens / slots / out (CPU tensors, pinned for
    copy-compute overlap): the library stages them through `workspace` (device) and pipelines
    uploads, ingest, per-chunk attention and downloads (head_chunks > 0: query-head chunks;
    <= 0 for one prompt: query-position chunks, longest rows first, -n = n chunks)."""
    for t in (q, k, v, cu_seqlens, slots, out):
        if t.is_cuda:
            raise ValueError("prefill_attention_host takes host tensors")
    cs = cache.struct()
    T = int(cu_seqlens[-1])
    ws, nb = _ws(workspace, prefill_host_workspace_size(cfg, slots.shape[0], T), cache.pages.device)
    _check(_lib.hack_prefill_attention_host(C.byref(cfg), _ptr(q), _ptr(k), _ptr(v), _ptr(cu_seqlens), _ptr(slots),
                                            slots.shape[0], max_seqlen, C.byref(cs), _ptr(out), _ptr(ws), nb,
                                            head_chunks, _stream(stream)), "prefill_attention_host")


def prefill_attention_cached(cfg: Config, q, cu_seqlens, slots, max_seqlen: int, cache: KVCache, out,
                             workspace=None, debug_pcodes=None, debug_qk=None, debug_pv=None, debug_head=-1, stream=None):
    cs = cache.struct()
    ws, nb = _ws(workspace, prefill_workspace_size(cfg, slots.shape[0], max_seqlen), q.device)
    _check(_lib.hack_prefill_attention_cached(C.byref(cfg), _ptr(q), _ptr(cu_seqlens), _ptr(slots),
                                              slots.shape[0], max_seqlen, C.byref(cs), _ptr(out), _ptr(ws), nb,
                                              _dbg(debug_pcodes, debug_qk, debug_pv, debug_head), _stream(stream)),
           "prefill_attention_cached")


def decode_append(cfg: Config, k_new, v_new, slots, cache: KVCache, stream=None):
    cs = cache.struct()
    _check(_lib.hack_decode_append(C.byref(cfg), _ptr(k_new), _ptr(v_new), _ptr(slots), slots.shape[0],
                                   C.byref(cs), _stream(stream)), "decode_append")


def decode_attention(cfg: Config, q_new, k_new, v_new, slots, max_seqlen: int, cache: KVCache, out,
                     workspace=None, debug_pcodes=None, debug_qk=None, debug_pv=None, debug_head=-1, stream=None):
    cs = cache.struct()
    ws, nb = _ws(workspace, decode_workspace_size(cfg, slots.shape[0], max_seqlen), q_new.device)
    _check(_lib.hack_decode_attention(C.byref(cfg), _ptr(q_new), _ptr(k_new), _ptr(v_new), _ptr(slots),
                                      slots.shape[0], max_seqlen, C.byref(cs), _ptr(out), _ptr(ws), nb,
                                      _dbg(debug_pcodes, debug_qk, debug_pv, debug_head), _stream(stream)), "decode_attention")


def decode_attention_cached(cfg: Config, q_new, slots, max_seqlen: int, cache: KVCache, out, workspace=None,
                            debug_pcodes=None, debug_qk=None, debug_pv=None, debug_head=-1, stream=None):
    cs = cache.struct()
    ws, nb = _ws(workspace, decode_workspace_size(cfg, slots.shape[0], max_seqlen), q_new.device)
    _check(_lib.hack_decode_attention_cached(C.byref(cfg), _ptr(q_new), _ptr(slots), slots.shape[0], max_seqlen,
                                             C.byref(cs), _ptr(out), _ptr(ws), nb,
                                             _dbg(debug_pcodes, debug_qk, debug_pv, debug_head),
                                             _stream(stream)), "decode_attention_cached")


def dequantize_cache(cfg: Config, slots, max_seqlen: int, cache: KVCache, k_out, v_out, stream=None):
    """Comparator only (not the HACK path): dense fp16 K-hat / V-hat
    [batch, H_kv, max_seqlen, d] of every request, dequantized from the same pages."""
    cs = cache.struct()
    _check(_lib.hack_dequantize_cache(C.byref(cfg), _ptr(slots), slots.shape[0], max_seqlen, C.byref(cs),
                                      _ptr(k_out), _ptr(v_out), _stream(stream)), "dequantize_cache")


def homomorphic_matmul(cfg: Config, a_codes, a_meta, a_sums, b_packed, b_meta, b_sums, M, N, Z, c,
                       d_blocks=None, stream=None):
    _check(_lib.hack_homomorphic_matmul(C.byref(cfg), _ptr(a_codes), _ptr(a_meta), _ptr(a_sums), _ptr(b_packed),
                                        _ptr(b_meta), _ptr(b_sums), M, N, Z, _ptr(d_blocks), _ptr(c),
                                        _stream(stream)), "homomorphic_matmul")


# --------------------------------------------------------------------------- KV transfer (a10)

def _caches_array(caches):
    arr = (CacheStruct * len(caches))()
    for i, c in enumerate(caches):
        arr[i] = c.struct()
    return arr


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.hack_comm_unique_id(buf), "comm_unique_id")
    return buf.raw


def comm_init(nranks: int, rank: int, uid: bytes):
    h = C.c_void_p()
    _check(_lib.hack_comm_init(C.byref(h), nranks, rank, C.c_char_p(bytes(uid))), "comm_init")
    return h


def comm_destroy(comm):
    _check(_lib.hack_comm_destroy(comm), "comm_destroy")


def comm_group_start():
    _check(_lib.hack_comm_group_start(), "comm_group_start")


def comm_group_end():
    _check(_lib.hack_comm_group_end(), "comm_group_end")


def kv_pack(cfg, caches, slot, prompt_len, first_token, rng_id, staging, stream=None):
    arr = _caches_array(caches)
    _check(_lib.hack_kv_pack(C.byref(cfg), arr, len(caches), slot, prompt_len, first_token, rng_id & 0xFFFFFFFF,
                             _ptr(staging), _stream(stream)), "kv_pack")


def kv_unpack(cfg, caches, slot, prompt_len, staging, status=None, stream=None):
    arr = _caches_array(caches)
    _check(_lib.hack_kv_unpack(C.byref(cfg), arr, len(caches), slot, prompt_len, _ptr(staging), _ptr(status),
                               _stream(stream)), "kv_unpack")


def kv_send(comm, peer, cfg, caches, slot, prompt_len, first_token, rng_id, staging, stream=None):
    arr = _caches_array(caches)
    _check(_lib.hack_kv_send(comm, peer, C.byref(cfg), arr, len(caches), slot, prompt_len, first_token,
                             rng_id & 0xFFFFFFFF, _ptr(staging), _stream(stream)), "kv_send")


def kv_recv(comm, peer, cfg, caches, slot, prompt_len, staging, status=None, stream=None):
    arr = _caches_array(caches)
    _check(_lib.hack_kv_recv(comm, peer, C.byref(cfg), arr, len(caches), slot, prompt_len, _ptr(staging),
                             _ptr(status), _stream(stream)), "kv_recv")


def kv_layer_range(cfg: Config, num_layers: int, layer: int, prompt_len: int) -> tuple[int, int]:
    """(begin, nbytes) of one layer's slice of the wire buffer (layer 0 includes the header)."""
    b = C.c_int64(0)
    n = int(_lib.hack_kv_layer_range(C.byref(cfg), num_layers, layer, prompt_len, C.byref(b)))
    if n < 0:
        raise HackError(ERR_INVALID_ARG, "kv_layer_range: bad arguments")
    return int(b.value), n


def kv_pull(cfg, src_caches, dst_caches, src_slot, dst_slot, prompt_len, stream=None):
    """Fused transfer: src (e.g. a peer GPU's cache opened through CUDA IPC) -> dst, one kernel."""
    if len(src_caches) != len(dst_caches):
        raise ValueError("kv_pull: src and dst need the same number of layers")
    _check(_lib.hack_kv_pull(C.byref(cfg), _caches_array(src_caches), _caches_array(dst_caches), len(src_caches),
                             src_slot, dst_slot, prompt_len, _stream(stream)), "kv_pull")


def kv_send_layer(comm, peer, cfg, caches, layer, slot, prompt_len, first_token, rng_id, staging, stream=None):
    arr = _caches_array(caches)
    _check(_lib.hack_kv_send_layer(comm, peer, C.byref(cfg), arr, len(caches), layer, slot, prompt_len, first_token,
                                   rng_id & 0xFFFFFFFF, _ptr(staging), _stream(stream)), "kv_send_layer")


def kv_recv_layer(comm, peer, cfg, num_layers, layer, prompt_len, staging, stream=None):
    _check(_lib.hack_kv_recv_layer(comm, peer, C.byref(cfg), num_layers, layer, prompt_len, _ptr(staging),
                                   _stream(stream)), "kv_recv_layer")


def comm_recv_bytes(comm, peer, buf, nbytes, stream=None):
    _check(_lib.hack_comm_recv_bytes(comm, peer, _ptr(buf), nbytes, _stream(stream)), "comm_recv_bytes")
