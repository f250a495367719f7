"""Head sharding on the CUDA path (BASELINE C3: "heads sharded 1/2/4/8 GPUs"):
two processes (world_size 2, gloo for the exchange, both on cuda:0 -- gpurun boxes have one
GPU) each run the library on their KV-head shard (`head_base` = the shard's first global KV
head, so the Philox streams are the unsharded run's, R3): ingest + prefill attention, then
decode steps through hack_decode_attention.  Rank 0 gathers the shards and checks them
against the unsharded run of the same library in the same process:
  * packed pages (codes, fp16 meta, cached sums) and FP16 tails: bit-identical;
  * prefill outputs: bit-identical (a tile's arithmetic does not depend on the other heads);
  * decode outputs: the page ranges of the persistent split differ between the sharded and
    unsharded grids, so partials merge in another order -- equal within 1e-5 relative."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HQ, HKV, L, STEPS, SEED = 16, 4, 700, 5, 41


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(h, Hq, Hkv, head_base, q, k, v, qd, kd, vd):
    """Prefill one request then STEPS decode steps on KV heads [head_base, head_base + Hkv)."""
    G = HQ // HKV
    cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, out_fp32=True, seed=SEED, head_base=head_base)
    mp_ = (L + STEPS + 63) // 64
    cache = h.KVCache.allocate(cfg, max_reqs=1, max_pages_per_req=mp_, device="cuda")
    cache.rng_ids.fill_(3)
    sl = slice(head_base * G, (head_base + Hkv) * G)
    kv = slice(head_base, head_base + Hkv)
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    slots = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.zeros((L, Hq, 128), dtype=torch.float32, device="cuda")
    h.prefill_attention(cfg, q[:, sl].contiguous(), k[:, kv].contiguous(), v[:, kv].contiguous(), cu, slots, L,
                        cache, out)
    dec = []
    for s in range(STEPS):
        o = torch.zeros((1, Hq, 128), dtype=torch.float32, device="cuda")
        h.decode_attention(cfg, qd[s][:, sl].contiguous(), kd[s][:, kv].contiguous(), vd[s][:, kv].contiguous(),
                           slots, L + STEPS, cache, o)
        dec.append(o)
    torch.cuda.synchronize()
    npg = (L + STEPS + 63) // 64
    pages = cache.pages[cache.block_table[0, :npg].long()].cpu()       # [page][H_kv][bytes]
    T = (L + STEPS) % 64
    return out.cpu(), torch.stack(dec).cpu(), pages, cache.v_tail[0, :, :T].cpu()


def _worker(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", world_size=world, rank=rank)
    try:
        import hack_inputs
        from paper_2502_03589_b200 import dist as hd
        from paper_2502_03589_b200 import hack as h
        q, k, v = (torch.from_numpy(x).cuda() for x in hack_inputs.qkv(SEED, L, HQ, HKV))
        qd, kd, vd = (torch.from_numpy(x).cuda() for x in hack_inputs.decode_tokens(SEED, STEPS, 1, HQ, HKV))
        base, nloc = hd.head_shard(HKV, world, rank)
        got = _run(h, nloc * HQ // HKV, nloc, base, q, k, v, qd, kd, vd)
        gathered = [None] * world
        dist.all_gather_object(gathered, got)
        if rank == 0:
            pre, dec, pages, tail = _run(h, HQ, HKV, 0, q, k, v, qd, kd, vd)
            assert torch.equal(torch.cat([g[0] for g in gathered], 1), pre), "prefill outputs"
            assert torch.equal(torch.cat([g[2] for g in gathered], 1), pages), "pages"
            assert torch.equal(torch.cat([g[3] for g in gathered], 0), tail), "FP16 tails"
            sd = torch.cat([g[1] for g in gathered], 2)
            rel = ((sd - dec).abs().amax(-1) / dec.abs().amax(-1).clamp_min(1e-6)).max().item()
            assert rel < 1e-5, f"decode outputs: {rel}"
    finally:
        dist.destroy_process_group()


def test_head_sharded_cuda_path_matches_unsharded():
    mp.start_processes(_worker, args=(2, _free_port()), nprocs=2, join=True, start_method="spawn")
