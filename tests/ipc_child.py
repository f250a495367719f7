"""Child process of test_gpu_kv_transfer.test_kv_pull_cuda_ipc (spawned): receives a prefill
process's cache tensors through CUDA IPC (torch.multiprocessing), pulls one request into
its own differently paged cache with hack_kv_pull (the loads read the other process's
memory), and returns the pulled bytes."""


def pull_child(q_in, q_out):
    import dataclasses

    import torch

    from paper_2502_03589_b200 import hack as h
    msg = q_in.get()
    cfg_kw, layers, L, src_slot, dst_slot = msg["cfg"], msg["tensors"], msg["L"], msg["src_slot"], msg["dst_slot"]
    cfgs = [h.config(**cfg_kw, layer=l) for l in range(len(layers))]
    src = [h.KVCache(cfgs[l], *t) for l, t in enumerate(layers)]
    mp = src[0].block_table.shape[1]
    first = h.KVCache.allocate(cfgs[0], 4, mp)
    perm = torch.randperm(4 * mp, generator=torch.Generator().manual_seed(5)).to(torch.int32).reshape(4, mp)
    first.block_table.copy_(perm.cuda())
    dst = [first] + [h.KVCache.allocate(cfgs[l], 4, mp, num_pages=first.pages.shape[0], shared_tables=first)
                     for l in range(1, len(layers))]
    h.kv_pull(cfgs[0], src, dst, src_slot, dst_slot, L)
    torch.cuda.synchronize()
    npg = (L + 63) // 64
    out = {"pages": [d.pages[d.block_table[dst_slot, :npg].long()].cpu().numpy() for d in dst],
           "tails": [d.v_tail[dst_slot, :, :L % 64].cpu().numpy() for d in dst],
           "seq_len": int(first.seq_lens[dst_slot]), "rng_id": int(first.rng_ids[dst_slot])}
    q_out.put(out)
    q_in.get()  # parent's release: the shared tensors stay alive until here
    del src, dataclasses
