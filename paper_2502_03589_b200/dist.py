"""Host-side multi-GPU / disaggregation logic (no compute).

* Head sharding (C3/C4): rank r owns a contiguous range of KV heads and their G query
  heads.  Philox counters use the GLOBAL head index (config.head_base), so codes and
  outputs are independent of the sharding (R3).
* Request sharding: independent requests per rank (weak scaling, no collective).
* Disaggregation (fig:overview): prefill ranks ship the packed KV of a
  request (hack_kv_send/hack_kv_recv over NCCL in libhack) to the decode rank chosen by
  shortest queued tokens.  The 64-byte wire header (S:350 fields) is mirrored
  here for host-side inspection and for transports other than NCCL (gloo in CPU tests).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

MAGIC = 0x4B434148          # "HACK" little-endian
WIRE_VERSION = 1
HEADER_BYTES = 64
_HDR = struct.Struct("<IHHHHHBBIIiIIIQQ8x")
assert _HDR.size == HEADER_BYTES


def head_shard(num_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """(head_base, local_kv_heads) of `rank` when KV heads are split across `world`
    ranks (contiguous blocks; every rank >= 1 head)."""
    if not (0 < world <= num_kv_heads) or num_kv_heads % world:
        raise ValueError("KV heads must split evenly across ranks")
    per = num_kv_heads // world
    return rank * per, per


def request_shard(num_requests: int, world: int, rank: int) -> list[int]:
    """Independent requests of `rank` (round robin)."""
    return list(range(rank, num_requests, world))


def page_bytes(d: int, Pi: int, bits: int) -> int:
    """Closed form of the page size (== hack_page_bytes)."""
    up = lambda x: (x + 15) // 16 * 16
    sw = 1 if bits + (Pi - 1).bit_length() <= 8 else 2
    nb = d // Pi
    return (up(Pi * d * bits // 8) + up(Pi * nb * 4) + up(Pi * nb * sw) + up(d * Pi * bits // 8) +
            up(d * 4) + up(d * sw))


def layer_bytes(Hkv: int, d: int, Pi: int, bits: int, prompt_len: int) -> int:
    npages = (prompt_len + Pi - 1) // Pi
    return npages * Hkv * page_bytes(d, Pi, bits) + Hkv * (prompt_len % Pi) * d * 2


def transfer_bytes(Hkv: int, d: int, Pi: int, bits: int, num_layers: int, prompt_len: int) -> int:
    """== hack_kv_transfer_bytes: header + per layer (pages + FP16 tail rows)."""
    return HEADER_BYTES + num_layers * layer_bytes(Hkv, d, Pi, bits, prompt_len)


def layer_range(Hkv: int, d: int, Pi: int, bits: int, num_layers: int, layer: int, prompt_len: int) -> tuple[int, int]:
    """== hack_kv_layer_range: (begin, nbytes) of layer `layer` in the wire buffer; layer 0
    carries the header.  The ranges of layers 0..num_layers-1 tile [0, transfer_bytes)."""
    if not 0 <= layer < num_layers:
        raise ValueError("layer out of range")
    lb = layer_bytes(Hkv, d, Pi, bits, prompt_len)
    begin = 0 if layer == 0 else HEADER_BYTES + layer * lb
    return begin, HEADER_BYTES + (layer + 1) * lb - begin


@dataclass
class WireHeader:
    num_layers: int
    num_kv_heads: int
    head_dim: int
    partition: int
    kv_bits: int
    prompt_len: int
    first_token: int
    rng_id: int
    head_base: int = 0
    seed: int = 0x48414B

    @property
    def sum_bytes(self) -> int:
        return 1 if self.kv_bits + (self.partition - 1).bit_length() <= 8 else 2

    @property
    def tail_len(self) -> int:
        return self.prompt_len % self.partition

    @property
    def payload_bytes(self) -> int:
        return self.num_layers * layer_bytes(self.num_kv_heads, self.head_dim, self.partition, self.kv_bits,
                                             self.prompt_len)

    def pack(self) -> bytes:
        return _HDR.pack(MAGIC, WIRE_VERSION, self.num_layers, self.num_kv_heads, self.head_dim, self.partition,
                         self.kv_bits, self.sum_bytes, self.prompt_len, self.tail_len, self.first_token,
                         self.rng_id & 0xFFFFFFFF, page_bytes(self.head_dim, self.partition, self.kv_bits),
                         self.head_base, self.payload_bytes, self.seed)

    @classmethod
    def unpack(cls, raw: bytes) -> "WireHeader":
        (magic, ver, nl, hkv, d, pi, bits, sb, plen, tail, first, rid, pb, hb, payload, seed) = \
            _HDR.unpack(bytes(raw[:HEADER_BYTES]))
        if magic != MAGIC:
            raise ValueError("bad magic (HACK_ERR_PROTOCOL)")
        if ver != WIRE_VERSION:
            raise ValueError("unknown wire version (HACK_ERR_PROTOCOL)")
        h = cls(nl, hkv, d, pi, bits, plen, first, rid, hb, seed)
        if sb != h.sum_bytes or tail != h.tail_len or pb != page_bytes(d, pi, bits) or payload != h.payload_bytes:
            raise ValueError("inconsistent header (HACK_ERR_PROTOCOL)")
        return h

    def check(self, expect: "WireHeader"):
        """The receiver's header check (libhack header_ok): dims, sizes, and the Philox seed
        and head_base -- this rank's later appends continue the same streams (R3)."""
        keys = ("num_layers", "num_kv_heads", "head_dim", "partition", "kv_bits", "prompt_len", "head_base", "seed")
        bad = [k for k in keys if getattr(self, k) != getattr(expect, k)]
        if bad:
            raise ValueError(f"header mismatch in {bad} (HACK_ERR_PROTOCOL)")


@dataclass
class DecodeScheduler:
    """Shortest-queue assignment of prefilled requests to decode ranks (the
    decode instance with the shortest queue of tokens still to process)."""
    decode_ranks: list[int]
    queued: dict = field(default_factory=dict)

    def __post_init__(self):
        self.queued = {r: 0 for r in self.decode_ranks}

    def assign(self, prompt_len: int, output_len: int) -> int:
        r = min(self.decode_ranks, key=lambda x: (self.queued[x], x))
        self.queued[r] += prompt_len + output_len
        return r

    def finish(self, rank: int, prompt_len: int, output_len: int):
        self.queued[rank] -= prompt_len + output_len
