"""GPU: packed-KV transfer (a10).

kv_pack -> bytes -> kv_unpack into a differently paged cache must reproduce every page
byte, the FP16 tail, seq_len and rng_id; decode on the receiver must equal decode on
the sender bit-for-bit; a corrupted header must be rejected on the device
(HACK_ERR_PROTOCOL) without touching the cache; the same through NCCL (1-rank
self-loop: ncclSend + ncclRecv in one group)."""
import numpy as np
import pytest
import torch

import hack_inputs

from .gpu_util import hk, make_cache

pytestmark = pytest.mark.gpu

LAYERS = 3
L = 200


def setup(scramble_seed):
    h = hk()
    cfgs = [h.config(num_q_heads=8, num_kv_heads=2, layer=l, out_fp32=True) for l in range(LAYERS)]
    first = make_cache(cfgs[0], max_reqs=3, max_len=L + 80, seed=scramble_seed)
    caches = [first] + [h.KVCache.allocate(cfgs[l], 3, first.block_table.shape[1], num_pages=first.pages.shape[0],
                                           shared_tables=first) for l in range(1, LAYERS)]
    return h, cfgs, caches


def prefill_all(h, cfgs, caches, slot, rng_id):
    caches[0].rng_ids[slot] = rng_id
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    sl = torch.tensor([slot], dtype=torch.int32, device="cuda")
    for l in range(LAYERS):
        q, k, v = hack_inputs.qkv(50 + l, L, 8, 2)
        out = torch.zeros((L, 8, 128), dtype=torch.float32, device="cuda")
        h.prefill_attention(cfgs[l], torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                            torch.from_numpy(v).cuda(), cu, sl, L, caches[l], out)


def request_bytes(cache, slot, L):
    np_ = (L + 63) // 64
    pg = cache.pages[cache.block_table[slot, :np_].long()].cpu().numpy()
    tail = cache.v_tail[slot, :, :L % 64].cpu().numpy()
    return pg, tail


def decode_once(h, cfgs, caches, slot):
    qd, kd, vd = hack_inputs.decode_tokens(77, 1, 1, 8, 2)
    outs = []
    sl = torch.tensor([slot], dtype=torch.int32, device="cuda")
    for l in range(LAYERS):
        out = torch.zeros((1, 8, 128), dtype=torch.float32, device="cuda")
        h.decode_attention(cfgs[l], torch.from_numpy(qd[0]).cuda(), torch.from_numpy(kd[0]).cuda(),
                           torch.from_numpy(vd[0]).cuda(), sl, L + 1, caches[l], out)
        outs.append(out.cpu().numpy())
    return outs


def check_same(src, dst, s_slot, d_slot):
    for a, b in zip(src, dst):
        pa, ta = request_bytes(a, s_slot, L)
        pb, tb = request_bytes(b, d_slot, L)
        assert np.array_equal(pa, pb) and np.array_equal(ta.view(np.uint16), tb.view(np.uint16))
    assert int(dst[0].seq_lens[d_slot]) == L and int(dst[0].rng_ids[d_slot]) == int(src[0].rng_ids[s_slot])


def test_pack_unpack_round_trip_and_decode_equivalence():
    h, cfgs, src = setup(1)
    _, _, dst = setup(2)                     # different page assignment
    prefill_all(h, cfgs, src, slot=1, rng_id=4242)
    nbytes = h.kv_transfer_bytes(cfgs[0], LAYERS, L)
    staging = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    h.kv_pack(cfgs[0], src, 1, L, first_token=31337, rng_id=4242, staging=staging)
    wire = staging.clone()                    # stand-in for the link
    from paper_2502_03589_b200 import dist as hd
    hdr = hd.WireHeader(LAYERS, 2, 128, 64, 2, L, first_token=31337, rng_id=4242, seed=cfgs[0].seed)
    assert bytes(wire[:64].cpu().numpy()) == hdr.pack()    # device header == host spec (S:350 fields)
    status = torch.full((2,), -9, dtype=torch.int32, device="cuda")
    h.kv_unpack(cfgs[0], dst, 2, L, wire, status=status)
    torch.cuda.synchronize()
    assert status.tolist() == [0, 31337]
    check_same(src, dst, 1, 2)
    o_src = decode_once(h, cfgs, src, 1)
    o_dst = decode_once(h, cfgs, dst, 2)
    for a, b in zip(o_src, o_dst):
        assert np.array_equal(a, b)
    # packed bytes vs fp16 K+V at a page-aligned prompt: <= 17% ("~15%")
    assert h.kv_transfer_bytes(cfgs[0], 1, 4096) / (4096 * 2 * 2 * 128 * 2) < 0.17


def test_corrupt_header_rejected():
    h, cfgs, src = setup(3)
    _, _, dst = setup(4)
    prefill_all(h, cfgs, src, slot=0, rng_id=7)
    nbytes = h.kv_transfer_bytes(cfgs[0], LAYERS, L)
    staging = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    h.kv_pack(cfgs[0], src, 0, L, first_token=5, rng_id=7, staging=staging)
    before = dst[0].pages.clone()
    for off in (0, 12, 16):                   # magic, partition, prompt_len fields
        bad = staging.clone()
        bad[off] ^= 0xFF
        status = torch.zeros(2, dtype=torch.int32, device="cuda")
        h.kv_unpack(cfgs[0], dst, 0, L, bad, status=status)
        torch.cuda.synchronize()
        assert int(status[0]) == h.ERR_PROTOCOL
    assert torch.equal(before, dst[0].pages) and int(dst[0].seq_lens[0]) == 0


def test_nccl_self_loop():
    h, cfgs, src = setup(5)
    _, _, dst = setup(6)
    prefill_all(h, cfgs, src, slot=2, rng_id=99)
    nbytes = h.kv_transfer_bytes(cfgs[0], LAYERS, L)
    comm = h.comm_init(1, 0, h.comm_unique_id())
    try:
        send_buf = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        recv_buf = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        h.comm_group_start()
        h.kv_send(comm, 0, cfgs[0], src, 2, L, first_token=11, rng_id=99, staging=send_buf)
        h.comm_recv_bytes(comm, 0, recv_buf, nbytes)
        h.comm_group_end()
        status = torch.zeros(2, dtype=torch.int32, device="cuda")
        h.kv_unpack(cfgs[0], dst, 1, L, recv_buf, status=status)
        torch.cuda.synchronize()
        assert status.tolist() == [0, 11]
        check_same(src, dst, 2, 1)
    finally:
        h.comm_destroy(comm)


def test_layer_pipelined_nccl_self_loop():
    """one NCCL message per layer (hack_kv_send_layer / hack_kv_recv_layer),
    each issued right after that layer's prefill on the same stream; the reassembled
    buffer equals the one-shot kv_pack bytes and unpacks to the same cache."""
    h, cfgs, src = setup(7)
    _, _, dst = setup(8)
    slot, rid, L_ = 1, 555, L
    src[0].rng_ids[slot] = rid
    nbytes = h.kv_transfer_bytes(cfgs[0], LAYERS, L_)
    comm = h.comm_init(1, 0, h.comm_unique_id())
    try:
        send_buf = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        recv_buf = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        cu = torch.tensor([0, L_], dtype=torch.int32, device="cuda")
        sl = torch.tensor([slot], dtype=torch.int32, device="cuda")
        for l in range(LAYERS):
            q, k, v = hack_inputs.qkv(50 + l, L_, 8, 2)
            out = torch.zeros((L_, 8, 128), dtype=torch.float32, device="cuda")
            h.prefill_attention(cfgs[l], torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                torch.from_numpy(v).cuda(), cu, sl, L_, src[l], out)
            h.comm_group_start()
            h.kv_send_layer(comm, 0, cfgs[0], src, l, slot, L_, first_token=3, rng_id=rid, staging=send_buf)
            h.kv_recv_layer(comm, 0, cfgs[0], LAYERS, l, L_, recv_buf)
            h.comm_group_end()
        ref = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        h.kv_pack(cfgs[0], src, slot, L_, first_token=3, rng_id=rid, staging=ref)
        torch.cuda.synchronize()
        assert torch.equal(recv_buf, ref)
        status = torch.zeros(2, dtype=torch.int32, device="cuda")
        h.kv_unpack(cfgs[0], dst, 0, L_, recv_buf, status=status)
        torch.cuda.synchronize()
        assert status.tolist() == [0, 3]
        check_same(src, dst, slot, 0)
    finally:
        h.comm_destroy(comm)


def test_kv_pull_fused_transfer():
    """hack_kv_pull copies a request cache-to-cache in one kernel, no
    staging; the result equals the pack -> unpack route byte for byte and decodes the same."""
    h, cfgs, src = setup(9)
    _, _, dst = setup(10)
    _, _, dst2 = setup(11)
    prefill_all(h, cfgs, src, slot=0, rng_id=777)
    h.kv_pull(cfgs[0], src, dst, 0, 2, L)
    nbytes = h.kv_transfer_bytes(cfgs[0], LAYERS, L)
    staging = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    h.kv_pack(cfgs[0], src, 0, L, first_token=1, rng_id=777, staging=staging)
    h.kv_unpack(cfgs[0], dst2, 2, L, staging)
    torch.cuda.synchronize()
    check_same(src, dst, 0, 2)
    check_same(dst2, dst, 2, 2)
    for a, b in zip(decode_once(h, cfgs, src, 0), decode_once(h, cfgs, dst, 2)):
        assert np.array_equal(a, b)


def test_kv_pull_cuda_ipc():
    """The pull reads another process's cache through CUDA IPC (the same mechanism maps a
    peer GPU's memory over NVLink); the pulled request equals the source bytes."""
    import torch.multiprocessing as mp
    h, cfgs, src = setup(12)
    prefill_all(h, cfgs, src, slot=1, rng_id=4321)
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q_in, q_out = ctx.Queue(), ctx.Queue()
    from . import ipc_child
    p = ctx.Process(target=ipc_child.pull_child, args=(q_in, q_out))
    p.start()
    try:
        q_in.put({"cfg": dict(num_q_heads=8, num_kv_heads=2, out_fp32=True),
                  "tensors": [(c.pages, c.v_tail, c.block_table, c.seq_lens, c.rng_ids) for c in src],
                  "L": L, "src_slot": 1, "dst_slot": 3})
        out = q_out.get(timeout=300)
        q_in.put("done")
    finally:
        p.join(timeout=120)
    assert p.exitcode == 0
    assert out["seq_len"] == L and out["rng_id"] == 4321
    for l, c in enumerate(src):
        pa, ta = request_bytes(c, 1, L)
        assert np.array_equal(pa, out["pages"][l])
        assert np.array_equal(ta.view(np.uint16), out["tails"][l].view(np.uint16))


def _wire_header_spec(layers, Hkv, d, Pi, bits, prompt_len, first_token, rng_id, head_base, seed):
    """The 64-byte header as include/hack.h documents it (S:350 fields), packed by the test
    itself: magic "HACK", version 1, num_layers, H_kv, d, Pi, b, sum bytes, prompt_len,
    tail_len, first_token, rng_id, page_bytes, head_base, payload_bytes, seed, 8 pad bytes."""
    import struct
    from oracle import pages as opages
    lay = opages.layout(d, Pi, bits)
    npages, T = (prompt_len + Pi - 1) // Pi, prompt_len % Pi
    payload = layers * (npages * Hkv * lay["page_bytes"] + Hkv * T * d * 2)
    return struct.pack("<IHHHHHBBIIiIIIQQ8x", 0x4B434148, 1, layers, Hkv, d, Pi, bits, lay["sum_bytes"], prompt_len,
                       T, first_token, rng_id, lay["page_bytes"], head_base, payload, seed)


def test_kv_pack_equals_oracle_wire_image():
    """a10 against an image built without the GPU: the staging bytes of hack_kv_pack equal a
    header packed from the documented field list, then per layer the oracle's packed pages
    (oracle.pages; undefined bytes -- the partial last page's V section, padding -- masked)
    and the oracle's FP16 tail rows (RQE)."""
    from oracle import attention as att
    from oracle import pages as opages
    h, cfgs, src = setup(13)
    slot, rid = 1, 4242
    prefill_all(h, cfgs, src, slot=slot, rng_id=rid)
    nbytes = h.kv_transfer_bytes(cfgs[0], LAYERS, L)
    staging = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    h.kv_pack(cfgs[0], src, slot, L, first_token=31337, rng_id=rid, staging=staging)
    got = staging.cpu().numpy()
    hdr = _wire_header_spec(LAYERS, 2, 128, 64, 2, L, 31337, rid, 0, cfgs[0].seed)
    assert bytes(got[:64]) == hdr
    off = 64
    for l in range(LAYERS):
        _, k, v = hack_inputs.qkv(50 + l, L, 8, 2)
        st = att.ingest_prompt(att.Config(Hq=8, Hkv=2, layer=l, seed=cfgs[0].seed), k, v, rng_id=rid)
        ref, mask = opages.pack_request(st)                       # [npages, Hkv, page_bytes]
        g = got[off:off + ref.size].reshape(ref.shape)
        bad = (g != ref) & mask
        assert not bad.any(), f"layer {l}: {bad.sum()} page bytes differ from the oracle image"
        off += ref.size
        tail = np.ascontiguousarray(st.arrays()["tail"].transpose(1, 0, 2)).view(np.uint8).reshape(-1)
        assert np.array_equal(got[off:off + tail.size], tail), f"layer {l}: FP16 tail differs"
        off += tail.size
    assert off == nbytes


def test_kv_transfer_rejects_foreign_streams():
    """The header carries the cache's rng_id, seed and head_base: a caller rng_id that does
    not match rng_ids[slot] poisons the header, and a receiver configured with another seed
    or head_base (its appends would continue different Philox streams, R3) rejects it --
    HACK_ERR_PROTOCOL on the device, cache untouched."""
    h, cfgs, src = setup(14)
    _, _, dst = setup(15)
    prefill_all(h, cfgs, src, slot=0, rng_id=7)
    nbytes = h.kv_transfer_bytes(cfgs[0], LAYERS, L)
    before = dst[0].pages.clone()

    def unpack_status(staging, cfg):
        status = torch.zeros(2, dtype=torch.int32, device="cuda")
        h.kv_unpack(cfg, dst, 0, L, staging, status=status)
        torch.cuda.synchronize()
        return int(status[0])

    bad_rid = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    h.kv_pack(cfgs[0], src, 0, L, first_token=5, rng_id=8, staging=bad_rid)
    assert unpack_status(bad_rid, cfgs[0]) == h.ERR_PROTOCOL
    good = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    h.kv_pack(cfgs[0], src, 0, L, first_token=5, rng_id=7, staging=good)
    for kw in (dict(seed=cfgs[0].seed + 1), dict(head_base=1)):
        other = h.config(num_q_heads=8, num_kv_heads=2, out_fp32=True, **kw)
        assert unpack_status(good, other) == h.ERR_PROTOCOL
    assert torch.equal(before, dst[0].pages) and int(dst[0].seq_lens[0]) == 0
    assert unpack_status(good, cfgs[0]) == h.OK
