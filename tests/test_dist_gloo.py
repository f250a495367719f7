"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host paths:
head sharding gives bit-identical codes/outputs to the unsharded run (position- and
global-head-keyed Philox, R3); the disaggregated prefill -> decode exchange of the
wire format (header + pages + FP16 tail) round-trips exactly; max-over-ranks timing.
The CUDA transport (hack_kv_send/recv over NCCL) is covered by test_gpu_kv_transfer."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hack_inputs
from oracle import attention as att
from oracle import pages as opages

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name):
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", world_size=world, rank=rank)
    try:
        globals()[fn_name](rank, world)
    finally:
        dist.destroy_process_group()


def run_gloo(fn_name, world=2):
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, fn_name), nprocs=world, join=True, start_method="spawn")


# ----------------------------------------------------------------------------- workers

def _head_sharding(rank, world):
    from paper_2502_03589_b200 import dist as hd
    Hq, Hkv, L = 8, 4, 130
    q, k, v = hack_inputs.qkv(9, L, Hq, Hkv)
    base, nloc = hd.head_shard(Hkv, world, rank)
    G = Hq // Hkv
    cfg = att.Config(Hq=nloc * G, Hkv=nloc, head_base=base, seed=77, layer=2)
    rows = np.array([0, 63, 64, 129])
    O, st, _ = att.prefill(cfg, q[:, base * G:(base + nloc) * G], k[:, base:base + nloc], v[:, base:base + nloc],
                           rng_id=5, rows=rows)
    kc = torch.from_numpy(st.arrays()["kc"].astype(np.int64))
    outs = torch.from_numpy(O[rows])
    gk = [torch.zeros_like(kc) for _ in range(world)]
    go = [torch.zeros_like(outs) for _ in range(world)]
    dist.all_gather(gk, kc)
    dist.all_gather(go, outs)
    if rank == 0:
        full = att.Config(Hq=Hq, Hkv=Hkv, seed=77, layer=2)
        Of, stf, _ = att.prefill(full, q, k, v, rng_id=5, rows=rows)
        assert np.array_equal(torch.cat(gk, 1).numpy(), stf.arrays()["kc"])      # codes bit-identical
        assert np.allclose(torch.cat(go, 1).numpy(), Of[rows], rtol=1e-13, atol=1e-15)


def _wire_bytes(states, hdr):
    parts = [np.frombuffer(hdr.pack(), np.uint8)]
    for st in states:
        pg, mask = opages.pack_request(st)
        pg = np.where(mask, pg, 0).astype(np.uint8)
        parts.append(pg.reshape(-1))
        tail = st.arrays()["tail"]                        # [T, Hkv, d] fp16
        parts.append(np.ascontiguousarray(tail.transpose(1, 0, 2)).view(np.uint8).reshape(-1))
    return np.concatenate(parts)


def _disagg_exchange(rank, world):
    from paper_2502_03589_b200 import dist as hd
    Hkv, L, layers = 2, 150, 2
    states = []
    for layer in range(layers):
        cfg = att.Config(Hq=4, Hkv=Hkv, layer=layer, seed=3)
        _, k, v = hack_inputs.qkv(20 + layer, L, 4, Hkv)
        states.append(att.ingest_prompt(cfg, k, v, rng_id=1234))
    nbytes = hd.transfer_bytes(Hkv, 128, 64, 2, layers, L)
    if rank == 0:   # prefill rank: pack + send
        hdr = hd.WireHeader(layers, Hkv, 128, 64, 2, L, first_token=42, rng_id=1234, seed=3)
        wire = _wire_bytes(states, hdr)
        assert wire.size == nbytes
        dist.send(torch.from_numpy(wire), dst=1)
    else:           # decode rank: recv (size from the closed form), validate, compare
        buf = torch.zeros(nbytes, dtype=torch.uint8)
        dist.recv(buf, src=0)
        raw = buf.numpy()
        hdr = hd.WireHeader.unpack(raw)
        assert (hdr.prompt_len, hdr.first_token, hdr.rng_id, hdr.num_layers, hdr.tail_len) == (L, 42, 1234, layers,
                                                                                                L % 64)
        ref = _wire_bytes(states, hdr)
        assert np.array_equal(raw, ref)
        bad = raw.copy()
        bad[0] ^= 1
        with pytest.raises(ValueError):
            hd.WireHeader.unpack(bad)


def _layer_pipelined_exchange(rank, world):
    """the prefill rank sends each layer's slice as soon as that layer is
    ingested (one message per layer, layer 0 with the header); the decode rank receives
    the slices into one buffer, which must equal the one-shot wire bytes."""
    from paper_2502_03589_b200 import dist as hd
    Hkv, L, layers = 2, 130, 3
    nbytes = hd.transfer_bytes(Hkv, 128, 64, 2, layers, L)
    hdr = hd.WireHeader(layers, Hkv, 128, 64, 2, L, first_token=7, rng_id=99, seed=5)
    states = []
    if rank == 0:
        wire = np.zeros(nbytes, np.uint8)
        for layer in range(layers):              # "prefill" of layer l, then its send
            cfg = att.Config(Hq=4, Hkv=Hkv, layer=layer, seed=5)
            _, k, v = hack_inputs.qkv(60 + layer, L, 4, Hkv)
            states.append(att.ingest_prompt(cfg, k, v, rng_id=99))
            full = _wire_bytes(states + [states[-1]] * (layers - len(states)), hdr)
            b, n = hd.layer_range(Hkv, 128, 64, 2, layers, layer, L)
            wire[b:b + n] = full[b:b + n]
            dist.send(torch.from_numpy(wire[b:b + n].copy()), dst=1)
    else:
        buf = np.zeros(nbytes, np.uint8)
        for layer in range(layers):
            b, n = hd.layer_range(Hkv, 128, 64, 2, layers, layer, L)
            t = torch.zeros(n, dtype=torch.uint8)
            dist.recv(t, src=0)
            buf[b:b + n] = t.numpy()
        for layer in range(layers):
            cfg = att.Config(Hq=4, Hkv=Hkv, layer=layer, seed=5)
            _, k, v = hack_inputs.qkv(60 + layer, L, 4, Hkv)
            states.append(att.ingest_prompt(cfg, k, v, rng_id=99))
        assert np.array_equal(buf, _wire_bytes(states, hdr))
        assert hd.WireHeader.unpack(buf).num_layers == layers


def _max_over_ranks(rank, world):
    t = torch.tensor([1.5 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    assert float(t) == 1.5 + world - 1


# ----------------------------------------------------------------------------- tests

def test_head_sharding_bit_identical_gloo():
    run_gloo("_head_sharding")


def test_disaggregated_wire_exchange_gloo():
    run_gloo("_disagg_exchange")


def test_layer_pipelined_exchange_gloo():
    run_gloo("_layer_pipelined_exchange")


def test_layer_ranges_tile_the_wire_buffer():
    from paper_2502_03589_b200 import dist as hd
    from paper_2502_03589_b200 import hack as h
    for (Hkv, Pi, bits) in ((8, 64, 2), (2, 32, 2), (8, 128, 4)):
        c = h.config(num_q_heads=Hkv, num_kv_heads=Hkv, partition=Pi, kv_bits=bits)
        for L in (1, 64, 1000):
            end = 0
            for layer in range(4):
                b, n = hd.layer_range(Hkv, 128, Pi, bits, 4, layer, L)
                assert b == end and n > 0 and (b, n) == h.kv_layer_range(c, 4, layer, L)
                end = b + n
            assert end == hd.transfer_bytes(Hkv, 128, Pi, bits, 4, L) == h.kv_transfer_bytes(c, 4, L)
    with pytest.raises(ValueError):
        hd.layer_range(8, 128, 64, 2, 4, 4, 10)


def test_max_over_ranks_gloo():
    run_gloo("_max_over_ranks")


def test_wire_sizes_match_library():
    from paper_2502_03589_b200 import dist as hd
    from paper_2502_03589_b200 import hack as h
    for (Hkv, Pi, bits) in ((8, 64, 2), (2, 32, 2), (8, 128, 4), (1, 64, 4)):
        c = h.config(num_q_heads=Hkv, num_kv_heads=Hkv, partition=Pi, kv_bits=bits)
        assert hd.page_bytes(128, Pi, bits) == h.page_bytes(c)
        for L in (1, 63, 64, 1000):
            assert hd.transfer_bytes(Hkv, 128, Pi, bits, 3, L) == h.kv_transfer_bytes(c, 3, L)


def test_shortest_queue_scheduler():
    from paper_2502_03589_b200 import dist as hd
    s = hd.DecodeScheduler([4, 5, 6, 7])
    picks = [s.assign(p, o) for p, o in ((1000, 10), (10, 10), (500, 5), (20, 20), (5, 5))]
    assert picks[:4] == [4, 5, 6, 7]          # empty queues, lowest rank first
    assert picks[4] == 5                      # 20 queued tokens is the shortest
    s.finish(4, 1000, 10)
    assert s.assign(1, 1) == 4
    with pytest.raises(ValueError):
        hd.head_shard(8, 3, 0)
    assert [hd.head_shard(8, 4, r) for r in range(4)] == [(0, 2), (2, 2), (4, 2), (6, 2)]
