"""C5 (BASELINE configs[4]): the disaggregated mode on a mixed-length request trace.

    python bench.py --mode disagg --gpus N        (N even: N/2 prefill ranks, N/2 decode ranks)

What the paper's end-to-end experiment does, on B200 ranks:
  * requests arrive as a Poisson process at (about) the prefill capacity;
  * prompt / output lengths follow a 4-way mixture shaped like tab:dataset:
    IMDb, arXiv, Cocktail, HumanEval, each a lognormal fitted to the table's mean with its
    [min, max] as the ~1st / 99th percentile, clipped to [min, max];
  * a request goes to the prefill rank and to the decode rank "with the shortest updated queue
    length, defined by the number of queuing tokens";
  * the prefill rank runs hack_cache_ingest (quantization, a1-a2) and the homomorphic prefill
    attention (a3-a7) for every layer, then ships the packed KV (pages + fp16 meta + cached
    sums + FP16 tail + header, a10) to the decode rank with hack_kv_send (NCCL p2p over
    NVLink; one 2-rank communicator per prefill/decode pair);
  * each decode rank runs continuous batching: a request joins the batch when its
    hack_kv_recv completed, every iteration appends + attends one token per active request
    on every layer (a8-a9), and a request leaves after its output length.
Reported: generated tokens/s, JCT (mean / p50 / p99), the per-request phase decomposition of
fig:e2e_decompose (queue, quantization, prefill attention, KV communication, decode),
the achieved link GB/s per transfer and the wire bytes vs fp16 K+V.

Bounded for a bench run (stated in the JSON line): a few layers of a Llama-3.1-8B-shaped
attention stack (32 Q / 8 KV heads, d = 128, 2-bit, Pi = 64), prompts capped at
--c5-max-prompt, outputs at --c5-max-output, --c5-reqs requests.  Inputs are synthetic (a
pool of random q/k/v per layer, prefixes of it per request).
Schedules are computed up front from the trace so every rank knows the plan: the prefill
queue is modelled with the calibrated prefill rate (tokens/s measured on the ranks before
the trace), the decode queue by the tokens assigned so far (dist.DecodeScheduler).
"""
from __future__ import annotations

import json
import time

import numpy as np

# tab:dataset: prompt (mean, min, max), output (mean, min, max)
DATASETS = {
    "imdb": ((315, 106, 821), (37, 16, 87)),
    "arxiv": ((6300, 1600, 14100), (243, 29, 464)),
    "cocktail": ((16200, 9400, 28800), (159, 44, 246)),
    "humaneval": ((204, 75, 697), (139, 11, 552)),
}
Z99 = 2.326  # standard normal 99th percentile


def lognormal_clipped(rng, mean, lo, hi, n):
    """Lognormal with the given mean and ln-spread (ln hi - ln lo) / (2 z99), clipped."""
    sigma = (np.log(hi) - np.log(lo)) / (2 * Z99)
    mu = np.log(mean) - sigma ** 2 / 2
    return np.clip(rng.lognormal(mu, sigma, n), lo, hi).round().astype(int)


def make_trace(n, rps, seed, max_prompt, max_output, datasets=None):
    """(arrival s, prompt, output, dataset) per request; Poisson arrivals at `rps`."""
    rng = np.random.default_rng(seed)
    names = list(datasets or DATASETS)
    pick = rng.integers(0, len(names), n)
    arrivals = np.cumsum(rng.exponential(1.0 / rps, n))
    arrivals -= arrivals[0]
    reqs = []
    for i in range(n):
        (pm, plo, phi), (om, olo, ohi) = DATASETS[names[pick[i]]]
        p = int(min(lognormal_clipped(rng, pm, plo, phi, 1)[0], max_prompt))
        o = int(min(lognormal_clipped(rng, om, olo, ohi, 1)[0], max_output))
        reqs.append(dict(id=i, arrival=float(arrivals[i]), prompt=p, output=o, dataset=names[pick[i]]))
    return reqs


def schedule(reqs, n_pre, n_dec, pre_tok_s):
    """Prefill rank: shortest modelled queue at arrival (queued prompt tokens / measured rate);
    decode rank: shortest queue of assigned tokens (dist.DecodeScheduler)."""
    from paper_2502_03589_b200.dist import DecodeScheduler
    free = [0.0] * n_pre
    dec = DecodeScheduler(list(range(n_dec)))
    for r in reqs:
        p = min(range(n_pre), key=lambda x: (max(free[x], r["arrival"]), x))
        free[p] = max(free[p], r["arrival"]) + r["prompt"] / pre_tok_s
        r["pre"] = p
        r["dec"] = dec.assign(r["prompt"], r["output"])
    return reqs


def _log(rank, *a):
    import os
    import sys
    if os.environ.get("HACK_C5_VERBOSE"):
        print(f"[c5 rank {rank}]", *a, file=sys.stderr, flush=True)


def run(args, rank, local_rank, world, barrier, dev_normal):
    import torch
    import torch.distributed as dist

    from paper_2502_03589_b200 import hack as h

    if world < 2 or world % 2:
        raise SystemExit("--mode disagg needs an even number of ranks >= 2")
    dev = torch.device("cuda", local_rank)
    P = D = world // 2
    prefill = rank < P
    me = rank if prefill else rank - P
    Hq, Hkv, Pi, bits, layers = 32, 8, 64, 2, args.c5_layers
    nccl = args.dist_backend == "nccl"
    cfgs = [h.config(num_q_heads=Hq, num_kv_heads=Hkv, partition=Pi, kv_bits=bits, out_fp32=False, layer=l)
            for l in range(layers)]
    stream = torch.cuda.current_stream()

    # ---- calibration: the prefill rate (tokens/s incl. quantization) of a 4K prompt, for the
    # schedule and for Poisson arrivals at the prefill capacity
    rate = torch.zeros(1, dtype=torch.float64)
    if prefill:
        L = 4096
        cal = h.KVCache.allocate(cfgs[0], 1, L // Pi, device=dev)
        q = dev_normal((L, Hq, 128), 11, dev)
        k = dev_normal((L, Hkv, 128), 12, dev)
        v = dev_normal((L, Hkv, 128), 13, dev)
        cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
        sl = torch.zeros(1, dtype=torch.int32, device=dev)
        o = torch.empty((L, Hq, 128), dtype=torch.float16, device=dev)
        for _ in range(2):
            h.prefill_attention(cfgs[0], q, k, v, cu, sl, L, cal, o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            h.prefill_attention(cfgs[0], q, k, v, cu, sl, L, cal, o)
        e1.record(stream)
        torch.cuda.synchronize()
        rate[0] = 3 * L / (e0.elapsed_time(e1) * 1e-3) / layers  # prompt tokens/s through `layers` layers
        del cal, q, k, v, o
    rt = rate.to(dev) if dist.get_backend() == "nccl" else rate
    dist.all_reduce(rt, op=dist.ReduceOp.MAX)
    pre_tok_s = float(rt.cpu()[0])
    trace = make_trace(args.c5_reqs, 1.0, args.c5_seed, args.c5_max_prompt, args.c5_max_output)
    mean_prompt = float(np.mean([r["prompt"] for r in trace]))
    rps = args.c5_load * P * pre_tok_s / mean_prompt           # ~ the prefill capacity
    for r in trace:
        r["arrival"] /= rps                                      # unit-rate Poisson -> rate rps
    trace = schedule(trace, P, D, pre_tok_s)
    _log(rank, f"calibrated {pre_tok_s:.0f} prompt tok/s, {rps:.1f} req/s, last arrival {trace[-1]['arrival']:.4f} s")

    # ---- communicators: one 2-rank NCCL comm per (prefill p, decode d) pair
    comms = {}
    if nccl:
        for p in range(P):
            for d in range(D):
                uid = h.comm_unique_id() if rank == p else None
                box = [uid]
                dist.broadcast_object_list(box, src=p)
                if rank == p:
                    comms[d] = h.comm_init(2, 0, box[0])
                elif rank == P + d:
                    comms[p] = h.comm_init(2, 1, box[0])
    mine = [r for r in trace if (r["pre"] == me if prefill else r["dec"] == me)]
    maxL = max([r["prompt"] + r["output"] for r in mine] + [Pi]) + 1
    mp = (maxL + Pi - 1) // Pi
    nslot = max(1, len(mine))
    first = h.KVCache.allocate(cfgs[0], nslot, mp, device=dev)
    caches = [first] + [h.KVCache.allocate(cfgs[l], nslot, mp, num_pages=first.pages.shape[0], shared_tables=first,
                                           device=dev) for l in range(1, layers)]
    for i, r in enumerate(mine):
        r["slot"] = i
    first.rng_ids.copy_(torch.tensor([r["id"] for r in mine] or [0], dtype=torch.int32, device=dev)[:nslot])
    wire = {r["id"]: h.kv_transfer_bytes(cfgs[0], layers, r["prompt"]) for r in mine}
    res = []
    ev0 = torch.cuda.Event(enable_timing=True)

    def at(ev):  # a CUDA event as seconds since t0 (this rank's timeline; t0 after a common barrier)
        return ev0.elapsed_time(ev) * 1e-3

    if prefill:
        Lmax = max([r["prompt"] for r in mine] + [1])
        pool = [(dev_normal((Lmax, Hq, 128), 900 + 3 * l, dev), dev_normal((Lmax, Hkv, 128), 901 + 3 * l, dev),
                 dev_normal((Lmax, Hkv, 128), 902 + 3 * l, dev)) for l in range(layers)]
        out = torch.empty((Lmax, Hq, 128), dtype=torch.float16, device=dev)
        staging = torch.empty(max(wire.values(), default=64), dtype=torch.uint8, device=dev)
        ws_bytes = h.prefill_workspace_size(cfgs[0], 1, Lmax)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
        barrier(world)
        t0 = time.perf_counter()
        ev0.record(stream)
        _log(rank, f"prefill: {len(mine)} requests")
        for r in mine:
            while time.perf_counter() - t0 < r["arrival"]:   # Poisson arrival (host clock)
                time.sleep(2e-5)
            L, sl = r["prompt"], torch.tensor([r["slot"]], dtype=torch.int32, device=dev)
            cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * layers + 2)]
            evs[0].record(stream)
            for l in range(layers):
                q, k, v = pool[l]
                h.cache_ingest(cfgs[l], k[:L], v[:L], cu, sl, L, caches[l])        # quantization (a1, a2)
                evs[1 + 2 * l].record(stream)
                h.prefill_attention_cached(cfgs[l], q[:L], cu, sl, L, caches[l], out[:L], workspace=ws)
                evs[2 + 2 * l].record(stream)
            if nccl:
                h.kv_send(comms[r["dec"]], 1, cfgs[0], caches, r["slot"], L, first_token=r["id"], rng_id=r["id"],
                          staging=staging)
            else:  # gloo (several ranks on one GPU, tests): host-staged
                h.kv_pack(cfgs[0], caches, r["slot"], L, first_token=r["id"], rng_id=r["id"], staging=staging)
            evs[-1].record(stream)
            if not nccl:
                evs[-1].synchronize()
                dist.send(staging[:wire[r["id"]]].cpu(), dst=P + r["dec"])
            r["_ev"] = evs
            _log(rank, f"sent request {r['id']} ({L} tokens) to decode rank {r['dec']}")
        torch.cuda.synchronize()
        for r in mine:
            evs = r.pop("_ev")
            quant = sum(evs[1 + 2 * l - 1].elapsed_time(evs[1 + 2 * l]) if l else evs[0].elapsed_time(evs[1])
                        for l in range(layers)) * 1e-3
            attn = sum(evs[1 + 2 * l].elapsed_time(evs[2 + 2 * l]) for l in range(layers)) * 1e-3
            send = evs[2 * layers].elapsed_time(evs[-1]) * 1e-3
            res.append(dict(id=r["id"], arrival=r["arrival"], pre_start=at(evs[0]), quant_s=quant, attn_s=attn,
                            send_start=at(evs[2 * layers]), send_s=send, wire_bytes=wire[r["id"]],
                            prompt=r["prompt"], output=r["output"], dataset=r["dataset"]))
    else:
        # ---- decode rank: receives posted per source prefill rank (its processing order) on
        # that source's stream; continuous batching on the compute stream
        B = len(mine)
        dl = [dataclass_replace(c_, seq_lens=first.seq_lens.clone()) for c_ in caches]  # per-layer seq_lens (a8)
        qn = dev_normal((max(B, 1), Hq, 128), 700 + me, dev)
        kn = dev_normal((max(B, 1), Hkv, 128), 701 + me, dev)
        vn = dev_normal((max(B, 1), Hkv, 128), 702 + me, dev)
        dout = torch.empty((max(B, 1), Hq, 128), dtype=torch.float16, device=dev)
        ws = torch.zeros(max(h.decode_workspace_size(cfgs[0], max(B, 1), maxL), 1), dtype=torch.uint8, device=dev)
        streams = {p: torch.cuda.Stream(device=dev) for p in range(P)}
        staging = {r["id"]: torch.empty(wire[r["id"]], dtype=torch.uint8, device=dev) for r in mine}
        status = torch.zeros((max(B, 1), 2), dtype=torch.int32, device=dev)
        pend = {p: [r for r in mine if r["pre"] == p] for p in range(P)}  # in the source's order
        host = {}
        barrier(world)
        t0 = time.perf_counter()
        ev0.record(stream)
        for p in range(P):
            for r in pend[p]:
                if nccl:
                    with torch.cuda.stream(streams[p]):
                        h.kv_recv(comms[p], 0, cfgs[0], caches, r["slot"], r["prompt"], staging[r["id"]],
                                  status=status[r["slot"]], stream=streams[p])
                        r["_ev"] = torch.cuda.Event(enable_timing=True)
                        r["_ev"].record(streams[p])
                else:
                    host[r["id"]] = torch.empty(wire[r["id"]], dtype=torch.uint8)
                    r["_req"] = dist.irecv(host[r["id"]], src=p)
        active, done, gen = [], [], {}
        step_evs = []
        while len(done) < B:
            for p in range(P):  # admit requests whose KV arrived (in the source's order)
                while pend[p]:
                    r = pend[p][0]
                    if nccl:
                        if not r["_ev"].query():
                            break
                        stream.wait_event(r["_ev"])
                    else:
                        # gloo p2p Work objects only complete in wait(): block for the next
                        # request when the batch is idle (functional path for one-GPU tests)
                        if active:
                            break
                        r["_req"].wait()
                        staging[r["id"]].copy_(host[r["id"]], non_blocking=True)
                        h.kv_unpack(cfgs[0], caches, r["slot"], r["prompt"], staging[r["id"]], status=status[r["slot"]])
                    for c_ in dl:
                        c_.seq_lens[r["slot"]] = first.seq_lens[r["slot"]]
                    r["_adm"] = torch.cuda.Event(enable_timing=True)
                    r["_adm"].record(stream)
                    pend[p].pop(0)
                    active.append(r)
                    _log(rank, f"admitted request {r['id']}")
                    gen[r["id"]] = 0
            if not active:
                time.sleep(2e-5)
                continue
            slots = torch.tensor([r["slot"] for r in active], dtype=torch.int32, device=dev)
            n = len(active)
            for l in range(layers):
                h.decode_attention(cfgs[l], qn[:n], kn[:n], vn[:n], slots, maxL, dl[l], dout[:n], workspace=ws)
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            step_evs.append((n, e))
            still = []
            for r in active:
                gen[r["id"]] += 1
                if gen[r["id"]] >= r["output"]:
                    r["_fin"] = e
                    done.append(r)
                else:
                    still.append(r)
            active = still
        torch.cuda.synchronize()
        st = status.cpu().tolist()
        for r in mine:
            if st[r["slot"]][0] != 0 or st[r["slot"]][1] != r["id"]:
                raise RuntimeError(f"C5: kv_recv status {st[r['slot']]} for request {r['id']}")
            res.append(dict(id=r["id"], admit=at(r["_adm"]), finish=at(r["_fin"]), steps=r["output"]))
        res.append(dict(decode_batch_mean=float(np.mean([n for n, _ in step_evs])) if step_evs else 0.0,
                        decode_iterations=len(step_evs)))
    barrier(world)
    allr = [None] * world
    dist.all_gather_object(allr, res)
    for c_ in comms.values():
        h.comm_destroy(c_)
    if rank != 0:
        return
    pre = {x["id"]: x for rr in allr[:P] for x in rr}
    dec = {x["id"]: x for rr in allr[P:] for x in rr if "id" in x}
    dstat = [x for rr in allr[P:] for x in rr if "id" not in x]
    rows = []
    for i in sorted(pre):
        a, b = pre[i], dec[i]
        send_end = a["send_start"] + a["send_s"]
        rows.append(dict(dataset=a["dataset"], prompt=a["prompt"], output=a["output"], queue=a["pre_start"] - a["arrival"],
                         quant=a["quant_s"], prefill_attn=a["attn_s"], comm=max(b["admit"], send_end) - a["send_start"],
                         link_gbs=a["wire_bytes"] / a["send_s"] / 1e9 if nccl and a["send_s"] > 0 else None,
                         decode=b["finish"] - max(b["admit"], send_end), jct=b["finish"] - a["arrival"],
                         wire=a["wire_bytes"], fp16=layers * Hkv * a["prompt"] * 128 * 2 * 2))
    jct = np.array([r["jct"] for r in rows])
    span = max(dec[i]["finish"] for i in dec) - min(pre[i]["arrival"] for i in pre)
    tokens = sum(r["output"] for r in rows)
    mean = lambda k: float(np.mean([r[k] for r in rows]))
    line = {"metric": "C5 disaggregated trace: generated tokens/s", "value": tokens / span, "unit": "tokens/s",
            "n_gpus": world, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": f"C5: {P} prefill + {D} decode ranks, {len(rows)} requests, Poisson arrivals at "
                                   f"{args.c5_load:.2f} x the calibrated prefill capacity ({rps:.2f} req/s), "
                                   "tab:dataset-shaped 4-way length mixture (P:852-855), shortest-queue "
                                   f"assignment (P:783), {layers} layers x {Hq}/{Hkv} heads, 2-bit, Pi=64",
                       "transport": "hack_kv_send/recv (NCCL p2p)" if nccl else "kv_pack + gloo host send/irecv",
                       "max_prompt": args.c5_max_prompt, "max_output": args.c5_max_output, "seed": args.c5_seed},
            "jct_s": {"mean": float(jct.mean()), "p50": float(np.percentile(jct, 50)),
                      "p99": float(np.percentile(jct, 99))},
            "phases_mean_s": {k: mean(k) for k in ("queue", "quant", "prefill_attn", "comm", "decode")},
            "phase_share_of_jct": {k: mean(k) / float(jct.mean()) for k in ("queue", "quant", "prefill_attn", "comm",
                                                                          "decode")},
            # achieved GB/s of the NCCL send (kv_pack + ncclSend, prefill side events); None over gloo
            "link_gbs_mean": float(np.mean([r["link_gbs"] for r in rows if r["link_gbs"]])) if nccl else None,
            "wire_bytes": int(sum(r["wire"] for r in rows)),
            "wire_vs_fp16_kv": float(sum(r["wire"] for r in rows) / sum(r["fp16"] for r in rows)),
            "prefill_tokens_per_s_per_rank_calibrated": pre_tok_s,
            "decode": dstat,
            "per_dataset_jct_s": {d: float(np.mean([r["jct"] for r in rows if r["dataset"] == d]))
                                  for d in sorted({r["dataset"] for r in rows})}}
    print(json.dumps(line), flush=True)


def dataclass_replace(obj, **kw):
    import dataclasses
    return dataclasses.replace(obj, **kw)
