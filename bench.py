#!/usr/bin/env python3
"""HACK hot-path benchmark on B200 (contract: see DESIGN.md "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hack|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...    (one rank per GPU)

Workload (BASELINE.json configs[1], "C2"): Mistral-7B-shaped homomorphic prefill --
32 Q / 8 KV heads, d=128, one 4096-token prompt, 2-bit K/V, Pi=64.  One step = one
hack_prefill_attention call: the ingest (a1, a2: quantize K/V into pages + FP16 tail), then
the attention kernel (a3-a7: Q quant, Eq. 4 Q'K'^T, online softmax, P quant, Eq. 4 P'V' + FP
tail) launched as a programmatic dependent of the ingest.  The roofline times the attention
kernel alone (hack_prefill_attention_cached, separate launches).  The decode rows (a8, a9) are timed in the same run on
configs[2] ("C3": Llama-3.1-8B-shaped decode, batch 64, context 8192) and reported
under "decode".  Headline: algorithmic int8 ops (2 matmuls x 2*d*L(L+1)/2 x H_q,
causal triangle) / step time, in TOPS.  Multi-GPU: weak scaling, every rank runs its
own independent requests (no data-path collective; SURVEY e).

Timing: W warm-up steps, then K steps between barrier + synchronize, per-step CUDA
events on the launching stream, L2 flushed (512 MB write) before every prefill step
(outside the events); the C3 cache (352 MB) exceeds L2.  Max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

C2 = dict(Hq=32, Hkv=8, L=4096, Pi=64, bits=2)
C3 = dict(Hq=32, Hkv=8, B=64, ctx=8192, Pi=64, bits=2)
C4 = dict(Hq=64, Hkv=8, L=32768, B=16, Pi=64)
WORKLOAD = ("C2: Mistral-7B-shaped homomorphic prefill attention (32 Q / 8 KV heads, d=128), "
            "one 4096-token causal prompt, 2-bit K/V, Pi=64, Q/P 8-bit")
DECODE_WORKLOAD = ("C3: Llama-3.1-8B-shaped decode attention (32 Q / 8 KV heads, d=128), batch 64, "
                   "context 8192, 2-bit K/V + summation cache + FP16 last-V block, Pi=64")
METRIC = "prefill attn int8 TOPS"
BASELINE_METRIC = "decode attn tokens/s & effective KV GB/s; prefill attn int8 TOPS vs peak"


def prefill_ops(L, Hq, d=128):
    """Algorithmic int8 ops of one causal prefill: 2 matmuls x 2*d*L(L+1)/2 x H_q."""
    return 2 * 2 * d * (L * (L + 1) // 2) * Hq


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j.get("bf16_tflops_sustained"),
                    src="MEASURED_PEAKS.json (measured)", sm_max=j.get("sm_max_mhz"))
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="B200_PROFILING.md fallback", sm_max=1965.0)


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        return json.load(open(p))
    return {}


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock + throttle reasons with NVML every ~2 ms (own thread)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["nvml unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max, "reasons": names,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers

def dev_normal(shape, seed, device):
    """Seeded synthetic fp16 N(0,1) generated on the device (values never affect speed)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return torch.randn(shape, generator=g, device=device, dtype=torch.float32).to(torch.float16)


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


# ----------------------------------------------------------------------------- CPU oracle (baseline)

def oracle_sample(seconds_hint=False, L=4096, heads=1, groups=1):
    """Time the oracle (as it stands) on a bounded sample of the C2 workload: `groups` KV
    head groups (4 query heads each), of which the first `heads` query heads, over the
    full 4096-token prompt.  Returns (TOPS, seconds, ops, description)."""
    import hack_inputs
    from oracle import attention as att
    G = C2["Hq"] // C2["Hkv"]
    q, k, v = hack_inputs.qkv(hack_inputs.DATA_SEED, L, G * groups, groups)
    cfg = att.Config(Hq=G * groups, Hkv=groups, Pi=C2["Pi"], bits=C2["bits"])
    t0 = time.perf_counter()
    att.prefill(cfg, q, k, v, heads=list(range(heads)))
    dt = time.perf_counter() - t0
    ops = prefill_ops(L, heads)
    desc = (f"oracle prefill of {heads} of 32 query heads ({groups} KV head group(s)) of the C2 4096-token "
            f"prompt, incl. K/V quantization of those KV heads")
    return ops / dt / 1e12, dt, ops, desc


def cpu_threads():
    """Threads the oracle's BLAS pool actually uses (its only parallelism)."""
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_one_thread(heads=1):
    """The same oracle sample with its BLAS pool limited to one thread (SURVEY d-3)."""
    try:
        import threadpoolctl
        with threadpoolctl.threadpool_limits(1):
            return oracle_sample(heads=heads)
    except ImportError:
        return None


def cpu_record(value, desc, dt, one=None):
    rec = {"value": value, "unit": "TOPS", "cores": cpu_threads(), "kind": "oracle", "sample": f"{desc}; {dt:.1f} s wall",
           "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}
    if one is not None:
        rec["value_1thread"] = one[0]
        rec["sample_1thread"] = f"{one[3]}; {one[1]:.1f} s wall, 1 BLAS thread"
    return rec


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, rank):
    if rank != 0:
        return
    for _ in range(args.warmup):
        oracle_sample(heads=1)
    vals, secs = [], []
    for _ in range(args.steps):
        v, dt, ops, desc = oracle_sample(heads=1)
        vals.append(v)
        secs.append(dt)
    value = sum(prefill_ops(C2["L"], 1) for _ in secs) / sum(secs) / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "batch": 1, "seq_len": C2["L"],
                                            "parallelism": "cpu oracle, rank 0 only"},
            "cpu_baseline": cpu_record(value, desc + " per step", statistics.mean(secs)),
            "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- HACK arm

def run_hack(args, rank, local_rank, world):
    import torch

    from paper_2502_03589_b200 import hack as h

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    peaks = load_peaks()
    traffic = load_traffic()
    seed = 20250205 + 1000 * rank
    stream = torch.cuda.current_stream()

    # ---------------- C2 prefill setup
    L, Hq, Hkv = C2["L"], C2["Hq"], C2["Hkv"]
    cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, partition=C2["Pi"], kv_bits=C2["bits"], out_fp32=False)
    q = dev_normal((L, Hq, 128), seed + 1, dev)
    k = dev_normal((L, Hkv, 128), seed + 2, dev)
    v = dev_normal((L, Hkv, 128), seed + 3, dev)
    cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
    slots = torch.tensor([0], dtype=torch.int32, device=dev)
    cache = h.KVCache.allocate(cfg, max_reqs=1, max_pages_per_req=L // C2["Pi"], device=dev)
    cache.rng_ids.fill_(rank)
    out = torch.empty((L, Hq, 128), dtype=torch.float16, device=dev)
    ws_bytes = h.prefill_workspace_size(cfg, 1, L)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ops = prefill_ops(L, Hq)

    def prefill_step(evs=None):
        # one hack_prefill_attention call: ingest (a1, a2) + attention (a3-a7), the attention
        # kernel a programmatic dependent of the ingest (its Q quantization overlaps it)
        if evs:
            evs[0].record(stream)
        h.prefill_attention(cfg, q, k, v, cu, slots, L, cache, out, workspace=ws)
        if evs:
            evs[1].record(stream)

    def attn_only(evs):
        # the attention kernel alone (the roofline's kernel), on the ingested cache
        evs[0].record(stream)
        h.prefill_attention_cached(cfg, q, cu, slots, L, cache, out, workspace=ws)
        evs[1].record(stream)

    for _ in range(args.warmup):
        flush.fill_(1)
        prefill_step()
    barrier(world)
    n0 = h.kernel_launches()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    evk = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        barrier(world)
        for i in range(args.steps):
            flush.fill_(1)                      # L2 flush, outside the events
            prefill_step(evs[i])
        barrier(world)
        launches = h.kernel_launches() - n0
        for i in range(args.steps):
            flush.fill_(1)
            attn_only(evk[i])
        barrier(world)
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    attn_ms = [e[0].elapsed_time(e[1]) for e in evk]
    ms = max_over_ranks(sum(step_ms) / len(step_ms), world)
    attn_avg = max_over_ranks(sum(attn_ms) / len(attn_ms), world)
    value = ops * world / (ms * 1e-3) / 1e12
    int8_peak = 2.0 * peaks["bf16"]
    achieved = ops / (attn_avg * 1e-3) / 1e12
    tr = traffic.get("prefill_attention", {}).get("dram_bytes_per_launch")

    # ---------------- e2e through the C ABI with host buffers: hack_prefill_attention_host
    # stages pinned host q/k/v through device memory and pipelines the uploads, the ingest,
    # the attention per chunk of query positions (longest rows first) and the downloads of
    # the output (library streams)
    qh = q.cpu().pin_memory(); kh = k.cpu().pin_memory(); vh = v.cpu().pin_memory()
    outh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    cuh, slh = cu.cpu().pin_memory(), slots.cpu().pin_memory()
    wsh = torch.empty(h.prefill_host_workspace_size(cfg, 1, L), dtype=torch.uint8, device=dev)

    def e2e_step():
        h.prefill_attention_host(cfg, qh, kh, vh, cuh, slh, L, cache, outh, workspace=wsh)

    for _ in range(args.warmup):
        e2e_step()
    barrier(world)
    e_ms = []
    for _ in range(args.steps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        b.synchronize()
        e_ms.append(a.elapsed_time(b))
    barrier(world)
    e2e_ms = max_over_ranks(sum(e_ms) / len(e_ms), world)
    e2e_val = ops * world / (e2e_ms * 1e-3) / 1e12
    del wsh

    # ---------------- C3 decode (a8, a9)
    dec = run_decode(args, h, dev, rank, world, peaks, traffic, seed, flush)
    c4 = None if args.no_c4 else run_c4(args, h, dev, world, seed, flush)
    sweep = None if args.no_sweep or world > 1 else run_sweep(args, h, dev, seed, flush)
    xfer = None if args.no_sweep or world > 1 else run_transfer(args, h, dev, seed)

    # ---------------- CPU oracle baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v_c, dt, ops_s, desc = oracle_sample(heads=8, groups=2)  # ~10-15 s of host CPU, all BLAS threads
        cpu = cpu_record(v_c, desc, dt, oracle_one_thread(heads=1))   # + one query head on 1 thread

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch": 1, "seq_len": L, "num_q_heads": Hq, "num_kv_heads": Hkv,
                       "partition": C2["Pi"], "kv_bits": C2["bits"],
                       "parallelism": f"replicas x{world} (independent requests per GPU)",
                       "l2": "flushed (512 MB write) before every step, outside the events",
                       "baseline_metric": BASELINE_METRIC},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": int8_peak, "unit": "TOPS",
                         "frac": achieved / int8_peak, "traffic": tr,
                         "kernel": "prefill attention (hack_prefill_attention_cached)",
                         "peak_src": f"{peaks['src']} bf16 burst {peaks['bf16']} x 2 (nominal int8:bf16 4.5:2.25)",
                         "ops_per_launch": ops, "ms_per_launch": attn_avg},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "TOPS",
                    "h2d_bytes_per_step": q.nbytes + k.nbytes + v.nbytes + cuh.nbytes + slh.nbytes,
                    "d2h_bytes_per_step": out.nbytes, "ms_per_step": e2e_ms,
                    "path": "pinned host q/k/v -> hack_prefill_attention_host (K/V up + ingest, then Q up, "
                            "attention and output down per chunk of query positions, longest rows first, "
                            "pipelined) -> pinned host out"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "decode": dec,
            "c4": c4,
            "pi_bits_sweep": sweep,
            "kv_transfer": xfer,
        }
        print(json.dumps(line), flush=True)


def run_transfer(args, h, dev, seed):
    """a10 device work on this GPU: pack one C2 request (4096-token prompt, 8 KV heads, 2-bit)
    of a 32-layer model into the wire buffer (hack_kv_pack, one launch) and unpack it into
    another cache (hack_kv_unpack).  The link itself (NCCL over NVLink between two GPUs) is
    not timed on one GPU."""
    import torch
    Hq, Hkv, L, layers = C2["Hq"], C2["Hkv"], C2["L"], 32
    cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, partition=C2["Pi"], kv_bits=C2["bits"], out_fp32=False)
    mp = (L + 63) // 64
    src = [h.KVCache.allocate(cfg, 1, mp, device=dev)]
    src += [h.KVCache.allocate(cfg, 1, mp, num_pages=src[0].pages.shape[0], shared_tables=src[0], device=dev)
            for _ in range(layers - 1)]
    dst = [h.KVCache.allocate(cfg, 1, mp, device=dev)]
    dst += [h.KVCache.allocate(cfg, 1, mp, num_pages=dst[0].pages.shape[0], shared_tables=dst[0], device=dev)
            for _ in range(layers - 1)]
    k = dev_normal((L, Hkv, 128), seed + 61, dev)
    v = dev_normal((L, Hkv, 128), seed + 62, dev)
    cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
    sl = torch.zeros(1, dtype=torch.int32, device=dev)
    for c_ in src:
        h.cache_ingest(cfg, k, v, cu, sl, L, c_)
    nbytes = h.kv_transfer_bytes(cfg, layers, L)
    wire = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def timed(fn, reps=5):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / reps

    pack_ms = timed(lambda: h.kv_pack(cfg, src, 0, L, first_token=1, rng_id=0, staging=wire))
    unpack_ms = timed(lambda: h.kv_unpack(cfg, dst, 0, L, wire))
    pull_ms = timed(lambda: h.kv_pull(cfg, src, dst, 0, 0, L))
    fp16_bytes = layers * L * Hkv * 128 * 2 * 2
    del src, dst, wire
    return {"workload": f"one {L}-token request, {layers} layers x {Hkv} KV heads, 2-bit (C2 shape)",
            "wire_bytes": nbytes, "fp16_kv_bytes": fp16_bytes, "ratio_vs_fp16": nbytes / fp16_bytes,
            "pack_ms": pack_ms, "pack_gbs": 2 * nbytes / (pack_ms * 1e-3) / 1e9,
            "unpack_ms": unpack_ms, "unpack_gbs": 2 * nbytes / (unpack_ms * 1e-3) / 1e9,
            "pull_ms": pull_ms, "pull_gbs": 2 * (nbytes - 64) / (pull_ms * 1e-3) / 1e9,
            "pull": "hack_kv_pull: cache -> cache in one kernel, no staging (f1 fused transfer; across GPUs the "
                    "source is a peer cache opened through CUDA IPC and the loads cross NVLink)",
            "note": "GB/s counts read + write; repeated packs of an 88 MB request can hit the 126 MB L2; "
                    "the NVLink send/recv needs two GPUs and is not timed here"}


def run_sweep(args, h, dev, seed, flush):
    """SURVEY f (Pi/bit sweep): partition size Pi in {32, 64, 128} x K/V bits in
    {2, 4} on a reduced C2/C3 shape (32 Q / 8 KV heads): one 2048-token causal prefill (ingest +
    attention, L2 flushed) and a C3-sized decode step (batch 64 at 8K context, append + attention,
    CUDA graph).  Decode runs on the mma.sync tensor-core kernels at every Pi; prefill runs the
    tcgen05 kernel at Pi = 64 and the CUDA-core kernel at Pi = 32 and 128."""
    import torch
    Hq, Hkv, L, B, ctx = 32, 8, 2048, C3["B"], C3["ctx"]
    stream = torch.cuda.current_stream()
    q = dev_normal((L, Hq, 128), seed + 51, dev)
    k = dev_normal((L, Hkv, 128), seed + 52, dev)
    v = dev_normal((L, Hkv, 128), seed + 53, dev)
    kc_ = dev_normal((8 * ctx, Hkv, 128), seed + 54, dev)   # 8 requests per ingest call
    vc_ = dev_normal((8 * ctx, Hkv, 128), seed + 55, dev)
    cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
    cuc = torch.arange(0, 9, dtype=torch.int32, device=dev) * ctx
    out = torch.empty((L, Hq, 128), dtype=torch.float16, device=dev)
    ops = prefill_ops(L, Hq)
    n_dec = 5
    res = {"workload": f"Pi x bits sweep: {Hq} Q / {Hkv} KV heads, d=128; prefill L={L} causal; "
                       f"decode batch {B} at {ctx} context", "points": []}
    for Pi in (32, 64, 128):
        for bits in (2, 4):
            cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, partition=Pi, kv_bits=bits, out_fp32=False, layer=3)
            mp = (max(L, ctx) + n_dec + 2 + Pi - 1) // Pi + 1
            cache = h.KVCache.allocate(cfg, max_reqs=B, max_pages_per_req=mp, device=dev)
            cache.rng_ids.copy_(torch.arange(B, dtype=torch.int32, device=dev))
            sl0 = torch.zeros(1, dtype=torch.int32, device=dev)
            ms = []
            for i in range(3):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                h.cache_ingest(cfg, k, v, cu, sl0, L, cache)
                h.prefill_attention_cached(cfg, q, cu, sl0, L, cache, out)
                b.record(stream)
                b.synchronize()
                if i:
                    ms.append(a.elapsed_time(b))
            pre_ms = sum(ms) / len(ms)
            for r0 in range(0, B, 8):
                h.cache_ingest(cfg, kc_, vc_, cuc, torch.arange(r0, r0 + 8, dtype=torch.int32, device=dev), ctx, cache)
            slots = torch.arange(B, dtype=torch.int32, device=dev)
            qn = dev_normal((n_dec, B, Hq, 128), seed + 56, dev)
            kn = dev_normal((n_dec, B, Hkv, 128), seed + 57, dev)
            vn = dev_normal((n_dec, B, Hkv, 128), seed + 58, dev)
            dout = torch.empty((B, Hq, 128), dtype=torch.float16, device=dev)
            ws = torch.zeros(max(h.decode_workspace_size(cfg, B, ctx + n_dec + 2), 1), dtype=torch.uint8,
                             device=dev)
            h.decode_append(cfg, kn[0], vn[0], slots, cache)
            h.decode_attention_cached(cfg, qn[0], slots, ctx + n_dec + 2, cache, dout, workspace=ws)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(1, n_dec):
                    h.decode_append(cfg, kn[i], vn[i], slots, cache)
                    h.decode_attention_cached(cfg, qn[i], slots, ctx + n_dec + 2, cache, dout, workspace=ws)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()
            dec_ms = a.elapsed_time(b) / (n_dec - 1)
            pb = h.page_bytes(cfg)
            n = ctx + n_dec // 2 + 1
            dec_bytes = B * Hkv * (n // Pi) * pb + B * Hq * 128 * 2 * 2
            res["points"].append({
                "Pi": Pi, "bits": bits,
                "prefill_kernel": f"prefill_tc_kernel<{Pi}, {bits}> (tcgen05)",
                "decode_kernel": "decode_pair_kernel (mma.sync)" if Pi == 64 and bits == 2
                else f"decode_mma_kernel<{bits}, {Pi}> (mma.sync)",
                "prefill_tops": ops / (pre_ms * 1e-3) / 1e12, "prefill_ms": pre_ms,
                "decode_step_ms": dec_ms, "decode_kv_gbs": dec_bytes / (dec_ms * 1e-3) / 1e9,
                "bytes_per_token_head": pb / Pi})
            del cache, ws, qn, kn, vn, g
    return res


def run_c4(args, h, dev, world, seed, flush):
    """C4 (BASELINE configs[3]) on this GPU: Llama-3.1-70B-shaped attention (64 Q / 8 KV heads,
    G = 8), one 32K-token causal prefill (ingest + attention) and a batch-16 decode step at 32K
    context, 2-bit vs 4-bit K/V.  (The 8-GPU layout gives every GPU one KV head; here one GPU
    runs all eight.)  Reported beside the headline, not as it."""
    import torch
    Hq, Hkv, L, B, Pi = C4["Hq"], C4["Hkv"], C4["L"], C4["B"], C4["Pi"]
    stream = torch.cuda.current_stream()
    res = {"workload": "C4: Llama-3.1-70B-shaped (64 Q / 8 KV heads, d=128), 32K causal prefill + "
                       "batch-16 decode at 32K context, one GPU", "per_bits": {}}
    q = dev_normal((L, Hq, 128), seed + 41, dev)
    k = dev_normal((L, Hkv, 128), seed + 42, dev)
    v = dev_normal((L, Hkv, 128), seed + 43, dev)
    cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
    out = torch.empty((L, Hq, 128), dtype=torch.float16, device=dev)
    ops = prefill_ops(L, Hq)
    n_pre, n_dec = 3, 8
    for bits in (2, 4):
        cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, partition=Pi, kv_bits=bits, out_fp32=False, layer=2)
        mp = (L + n_dec + 2 + Pi - 1) // Pi + 1
        cache = h.KVCache.allocate(cfg, max_reqs=B, max_pages_per_req=mp, device=dev)
        cache.rng_ids.copy_(torch.arange(B, dtype=torch.int32, device=dev))
        sl0 = torch.zeros(1, dtype=torch.int32, device=dev)
        ms = []
        for i in range(n_pre + 1):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h.cache_ingest(cfg, k, v, cu, sl0, L, cache)
            h.prefill_attention_cached(cfg, q, cu, sl0, L, cache, out)
            b.record(stream)
            b.synchronize()
            if i:
                ms.append(a.elapsed_time(b))
        pre_ms = sum(ms) / len(ms)
        # decode: every request holds the same 32K-token prompt (values never affect speed)
        for r in range(1, B):
            h.cache_ingest(cfg, k, v, cu, torch.tensor([r], dtype=torch.int32, device=dev), L, cache)
        slots = torch.arange(B, dtype=torch.int32, device=dev)
        qn = dev_normal((n_dec, B, Hq, 128), seed + 44, dev)
        kn = dev_normal((n_dec, B, Hkv, 128), seed + 45, dev)
        vn = dev_normal((n_dec, B, Hkv, 128), seed + 46, dev)
        dout = torch.empty((B, Hq, 128), dtype=torch.float16, device=dev)
        ws = torch.zeros(max(h.decode_workspace_size(cfg, B, L + n_dec + 2), 1), dtype=torch.uint8, device=dev)
        h.decode_append(cfg, kn[0], vn[0], slots, cache)      # warm-up step
        h.decode_attention_cached(cfg, qn[0], slots, L + n_dec + 2, cache, dout, workspace=ws)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(1, n_dec):
                h.decode_append(cfg, kn[i], vn[i], slots, cache)
                h.decode_attention_cached(cfg, qn[i], slots, L + n_dec + 2, cache, dout, workspace=ws)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        b.synchronize()
        dec_ms = a.elapsed_time(b) / (n_dec - 1)
        pb = h.page_bytes(cfg)
        n = L + n_dec // 2 + 1
        dec_bytes = B * Hkv * (n // Pi) * pb + B * Hq * 128 * 2 * 2
        res["per_bits"][str(bits)] = {
            "prefill_tops": ops / (pre_ms * 1e-3) / 1e12, "prefill_ms": pre_ms,
            "decode_step_ms": dec_ms, "decode_tokens_per_s": B / (dec_ms * 1e-3),
            "decode_kv_gbs": dec_bytes / (dec_ms * 1e-3) / 1e9, "page_bytes": pb,
            "bytes_per_token_head": pb / Pi}
        del cache, ws, qn, kn, vn
    return res


def run_decode(args, h, dev, rank, world, peaks, traffic, seed, flush):
    import torch
    B, ctx, Hq, Hkv, Pi = C3["B"], C3["ctx"], C3["Hq"], C3["Hkv"], C3["Pi"]
    # C3 shards KV heads over the GPUs (BASELINE configs[2]: "heads sharded 1/2/4/8 GPUs"):
    # rank r owns KV heads [r Hkv/N, (r+1) Hkv/N) and their G query heads for all requests;
    # head_base keeps every head's Philox streams those of the unsharded run (R3).
    shard = world > 1 and Hkv % world == 0
    if shard:
        Hkv, Hq = Hkv // world, Hq // world
    cfg = h.config(num_q_heads=Hq, num_kv_heads=Hkv, partition=Pi, kv_bits=C3["bits"], out_fp32=False, layer=1,
                   head_base=rank * Hkv if shard else 0)
    nsteps = args.warmup * 2 + args.steps * 2 + 2
    max_len = ctx + nsteps + 2 * Pi     # + the two Pi-step append graphs of the RQE ablation
    mp = (max_len + Pi - 1) // Pi
    # enough layers that one pass over them exceeds 2x the 126 MB L2 (a sharded layer can be
    # L2-sized); consecutive layer-steps walk the layers as a real decode step does (SURVEY d-5)
    layer_bytes = B * Hkv * mp * h.page_bytes(cfg)
    n_layers = max(1, min(32, -(-2 * 126_000_000 // layer_bytes)))
    slots_all = torch.arange(B, dtype=torch.int32, device=dev)
    caches = []
    for _ in range(n_layers):
        c_ = h.KVCache.allocate(cfg, max_reqs=B, max_pages_per_req=mp, device=dev)
        c_.rng_ids.copy_(torch.arange(B, dtype=torch.int32, device=dev))
        caches.append(c_)
    # fill every request with an 8192-token prompt through the ingest path (chunks of 8 requests)
    for c0 in range(0, B, 8):
        kk = dev_normal((8 * ctx, Hkv, 128), seed + 100 + c0, dev)
        vv = dev_normal((8 * ctx, Hkv, 128), seed + 200 + c0, dev)
        cu = torch.arange(0, 9, dtype=torch.int32, device=dev) * ctx
        for c_ in caches:
            h.cache_ingest(cfg, kk, vv, cu, slots_all[c0:c0 + 8].contiguous(), ctx, c_)
        del kk, vv
    torch.cuda.synchronize()
    cache = caches[0]
    qn = dev_normal((nsteps, B, Hq, 128), seed + 300, dev)
    kn = dev_normal((nsteps, B, Hkv, 128), seed + 301, dev)
    vn = dev_normal((nsteps, B, Hkv, 128), seed + 302, dev)
    out = torch.empty((B, Hq, 128), dtype=torch.float16, device=dev)
    ws_bytes = h.decode_workspace_size(cfg, B, max_len)
    ws = torch.zeros(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    it = [0]

    lens = [ctx] * n_layers   # host mirror of each layer's context length
    attn_lens = []

    def step(evs=None):
        i = it[0]
        it[0] += 1
        lay = i % n_layers
        c_ = caches[lay]
        if evs:
            evs[0].record(stream)
        # one decode step through the public call: hack_decode_attention appends k/v (a8) and
        # attends (a9); for the paired kernel the append runs inside the attention launch
        h.decode_attention(cfg, qn[i % nsteps], kn[i % nsteps], vn[i % nsteps], slots_all, max_len, c_, out,
                           workspace=ws)
        lens[lay] += 1
        attn_lens.append(lens[lay])
        if evs:
            evs[1].record(stream)
            evs[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    attn_lens.clear()
    if args.no_graph:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        n0 = h.kernel_launches()
        with ClockSampler(dev.index if dev.index is not None else 0) as clk:
            barrier(world)
            for i in range(args.steps):
                step(evs[i])
            barrier(world)
        launches = h.kernel_launches() - n0
        step_ms = [e[0].elapsed_time(e[2]) for e in evs]
        attn_ms = list(step_ms)  # (the fused step has no separate attention interval)
        ms = max_over_ranks(sum(step_ms) / len(step_ms), world)
        attn_avg = max_over_ranks(sum(attn_ms) / len(attn_ms), world)
        attn_ctx = list(attn_lens)
    else:
        # One decode step per layer is a few tens of microseconds, so host launch latency
        # (ctypes + 3 launches) would be timed too: the K timed steps (append + attention,
        # each step's own inputs) are captured once as a CUDA graph and replayed (SURVEY d-5).
        # The attention kernel alone is timed the same way: a graph of K launches of
        # hack_decode_attention_cached at the context reached after the K steps.
        g_step, g_attn = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        n0 = h.kernel_launches()
        with torch.cuda.graph(g_step):
            for i in range(args.steps):
                step()
        launches = h.kernel_launches() - n0
        with torch.cuda.graph(g_attn):
            for i in range(args.steps):
                lay = (it[0] + i) % n_layers
                h.decode_attention_cached(cfg, qn[(it[0] + i) % nsteps], slots_all, max_len, caches[lay], out,
                                          workspace=ws)
        attn_ctx = [lens[(it[0] + i) % n_layers] for i in range(args.steps)]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        with ClockSampler(dev.index if dev.index is not None else 0) as clk:
            barrier(world)
            ev[0].record(stream)
            g_step.replay()
            ev[1].record(stream)
            barrier(world)
            ev[2].record(stream)
            g_attn.replay()
            ev[3].record(stream)
            barrier(world)
        torch.cuda.synchronize()
        ms = max_over_ranks(ev[0].elapsed_time(ev[1]) / args.steps, world)
        attn_avg = max_over_ranks(ev[2].elapsed_time(ev[3]) / args.steps, world)
        no_se_ms, rqe_ms = None, None
        if not args.no_ablation:
            # SURVEY f2 (HACK/SE ablation): the same attention launches with the code
            # sums recomputed from the codes every step instead of read from the summation cache
            os.environ["HACK_DECODE_NO_SE"] = "1"
            g_nose = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_nose):
                for i in range(args.steps):
                    lay = (it[0] + i) % n_layers
                    h.decode_attention_cached(cfg, qn[(it[0] + i) % nsteps], slots_all, max_len, caches[lay], out,
                                              workspace=ws)
            del os.environ["HACK_DECODE_NO_SE"]
            torch.cuda.synchronize()
            ev[2].record(stream)
            g_nose.replay()
            ev[3].record(stream)
            torch.cuda.synchronize()
            no_se_ms = max_over_ranks(ev[2].elapsed_time(ev[3]) / args.steps, world)
            # SURVEY f2 (HACK/RQE ablation): Pi consecutive appends (every tail
            # length 1..Pi once per request and layer) with the partial V block requantized at
            # every step, vs the same appends with requantization elimination
            rqe_ms = {}
            for mode in ("rqe", "no_rqe"):
                if mode == "no_rqe":
                    os.environ["HACK_DECODE_NO_RQE"] = "1"
                g_app = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_app):
                    for i in range(Pi):
                        for lay in range(n_layers):
                            h.decode_append(cfg, kn[(it[0] + i) % nsteps], vn[(it[0] + i) % nsteps], slots_all,
                                            caches[lay])
                os.environ.pop("HACK_DECODE_NO_RQE", None)
                it[0] += Pi
                torch.cuda.synchronize()
                ev[2].record(stream)
                g_app.replay()
                ev[3].record(stream)
                torch.cuda.synchronize()
                rqe_ms[mode] = max_over_ranks(ev[2].elapsed_time(ev[3]) / (Pi * n_layers), world)
                del g_app
    # algorithmic bytes of one attention launch (context n after the append): committed
    # tokens at 84 B/token/head (packed K+V, meta, sums), tail tokens at K-row bytes +
    # fp16 V, plus q in and out.
    lay = h.page_layout(cfg)
    pb = h.page_bytes(cfg)
    krow = sum(lay[x][1] for x in ("k_codes", "k_meta", "k_sums")) // Pi
    nbytes = []
    for n in attn_ctx:
        C = (n // Pi) * Pi
        T = n - C
        nbytes.append(B * Hkv * (C * pb / Pi + T * (krow + 256)) + B * Hq * 128 * 2 * 2)
    avg_bytes = sum(nbytes) / len(nbytes)
    gbs = avg_bytes / (attn_avg * 1e-3) / 1e9
    comparator = None
    if not args.no_comparator:
        # a dequantize-first system on the same pages --
        # hack_dequantize_cache expands them to dense fp16 K-hat/V-hat, then PyTorch SDPA
        # (library attention, GQA) attends; timed per layer-step like the HACK call.
        L_now = int(cache.seq_lens[0].item())
        kh = torch.empty((B, Hkv, L_now, 128), dtype=torch.float16, device=dev)
        vh = torch.empty_like(kh)
        q4 = qn[0][:, :, None, :]
        cms = []
        for i in range(args.warmup + 5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h.dequantize_cache(cfg, slots_all, L_now, cache, kh, vh)
            o4 = torch.nn.functional.scaled_dot_product_attention(q4, kh, vh, enable_gqa=True)
            b.record(stream)
            b.synchronize()
            if i >= args.warmup:
                cms.append(a.elapsed_time(b))
        c_ms = max_over_ranks(sum(cms) / len(cms), world)
        comparator = {"what": "dequantize-first: hack_dequantize_cache (packed pages -> dense fp16) + "
                              "torch SDPA (GQA) -- the KVQuant/CacheGen-style path HACK avoids",
                      "ms_per_layer_step": c_ms, "hack_attn_ms": attn_avg, "hack_speedup": c_ms / attn_avg,
                      "fp16_cache_bytes": 2 * kh.numel() * 2}
        del kh, vh, o4
    ablation = None if args.no_graph or args.no_ablation else {
        "no_summation_elimination": {"attn_ms": no_se_ms, "kv_gbs": avg_bytes / (no_se_ms * 1e-3) / 1e9,
                                     "slowdown": no_se_ms / attn_avg,
                                     "what": "code sums recomputed from the codes every step (HACK/SE, P:1036-1042)"},
        "no_requantization_elimination": {
            "append_ms": rqe_ms["no_rqe"], "append_ms_with_rqe": rqe_ms["rqe"],
            "step_ms": ms - rqe_ms["rqe"] + rqe_ms["no_rqe"],
            "slowdown": (ms - rqe_ms["rqe"] + rqe_ms["no_rqe"]) / ms,
            "what": "partial last V block requantized at every append (HACK/RQE, P:704-724, P:1040); "
                    "append averaged over Pi steps (tail lengths 1..Pi), step = measured step with that append"}}
    # strong scaling when heads are sharded (every rank serves the same B requests), weak
    # (independent replicas) otherwise
    req_factor = 1 if shard else world
    tok_s = B * req_factor / (ms * 1e-3)
    # e2e: host q/k/v in, host out back, through hack_decode_attention (append + attend)
    qh = torch.empty((B, Hq, 128), dtype=torch.float16).pin_memory()
    kh = torch.empty((B, Hkv, 128), dtype=torch.float16).pin_memory()
    vh = torch.empty((B, Hkv, 128), dtype=torch.float16).pin_memory()
    oh = torch.empty((B, Hq, 128), dtype=torch.float16).pin_memory()
    qd, kd, vd = torch.empty_like(qn[0]), torch.empty_like(kn[0]), torch.empty_like(vn[0])
    e_ms = []
    for i in range(args.steps + args.warmup):
        qh.copy_(qn[it[0] % nsteps]); kh.copy_(kn[it[0] % nsteps]); vh.copy_(vn[it[0] % nsteps])
        it[0] += 1
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        qd.copy_(qh, non_blocking=True); kd.copy_(kh, non_blocking=True); vd.copy_(vh, non_blocking=True)
        h.decode_attention(cfg, qd, kd, vd, slots_all, max_len, cache, out, workspace=ws)
        oh.copy_(out, non_blocking=True)
        b.record(stream)
        b.synchronize()
        if i >= args.warmup:
            e_ms.append(a.elapsed_time(b))
    e2e_ms = max_over_ranks(sum(e_ms) / len(e_ms), world)
    tr = traffic.get("decode_attention", {}).get("dram_bytes_per_launch")
    return {
        "metric": "decode attn tokens/s", "value": tok_s, "unit": "tokens/s (per layer)",
        "scaling": "strong (KV heads sharded over ranks)" if shard else ("weak" if world > 1 else None),
        "kv_gbs": gbs * world, "kv_gbs_per_gpu": gbs, "ms_per_step": ms, "attn_ms": attn_avg, "steps": args.steps,
        "config": {"workload": DECODE_WORKLOAD, "batch": B, "context": ctx, "num_q_heads_per_rank": Hq,
                   "num_kv_heads_per_rank": Hkv, "partition": Pi, "kv_bits": C3["bits"],
                   "layers_cycled": n_layers,
                   "step": "hack_decode_attention: append (a8) fused into the attention (a9) launch",
                   "timing": "eager launches" if args.no_graph else
                   "CUDA-graph replay of the K timed steps (each with its own inputs)",
                   "l2": f"{n_layers} layer cache(s) of {layer_bytes / 1e6:.0f} MB per rank cycled (> 2x L2)"},
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm"], "unit": "GB/s",
                     "frac": gbs / peaks["hbm"], "traffic": tr, "bytes_per_launch": avg_bytes,
                     "kernel": "decode attention (hack_decode_attention_cached)", "peak_src": peaks["src"]},
        "e2e": {"value": B * req_factor / (e2e_ms * 1e-3), "unit": "tokens/s (per layer)",
                "h2d_bytes_per_step": qh.nbytes + kh.nbytes + vh.nbytes, "d2h_bytes_per_step": oh.nbytes,
                "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "ablation": ablation,
        "comparator": comparator,
    }


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 with the same arguments; rank 0 prints the line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["hack", "reference"], default="hack")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (70B-shaped, 2- vs 4-bit) sub-benchmark")
    ap.add_argument("--no-sweep", action="store_true", help="skip the Pi x bits sweep (SURVEY f)")
    ap.add_argument("--no-comparator", action="store_true", help="skip the dequantize-first comparator (f4)")
    ap.add_argument("--no-ablation", action="store_true", help="skip the SE / RQE ablation timings (f2)")
    ap.add_argument("--no-graph", action="store_true",
                    help="decode: launch eagerly instead of replaying a CUDA graph of the K timed steps")
    ap.add_argument("--mode", default="flagship", choices=["flagship", "disagg"],
                    help="disagg: the C5 disaggregated prefill -> decode trace (needs an even N >= 2)")
    ap.add_argument("--c5-reqs", type=int, default=32, help="disagg: requests in the trace")
    ap.add_argument("--c5-layers", type=int, default=4, help="disagg: layers of the attention stack")
    ap.add_argument("--c5-load", type=float, default=0.9, help="disagg: arrival rate / calibrated prefill capacity")
    ap.add_argument("--c5-max-prompt", type=int, default=16384, help="disagg: prompt length cap")
    ap.add_argument("--c5-max-output", type=int, default=256, help="disagg: output length cap")
    ap.add_argument("--c5-seed", type=int, default=20250205)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for barriers / max-over-ranks (gloo: several ranks on one GPU, tests)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "hack" else args.warmup
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        ndev = torch.cuda.device_count()
        if ndev < world and args.dist_backend == "nccl":
            sys.exit(f"bench.py: {world} ranks need {world} GPUs, this node has {ndev}")
        local_dev = local_rank % ndev
        torch.cuda.set_device(local_dev)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_dev))
        else:
            dist.init_process_group("gloo")
        local_rank = local_dev
    try:
        if args.mode == "disagg":
            import bench_c5
            bench_c5.run(args, rank, local_rank, world, barrier, dev_normal)
        else:
            run_hack(args, rank, local_rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
