// quant_kernels.cu -- (a1) quantize K, (a2) quantize V, (a3) quantize Q, the prefill
// ingest into the paged cache, and the decode append/flush (a8).
//
// Quantizer: P:575-578 (per-partition min/max, scale = (max-min)/(2^b-1),
// stochastic rounding), exact fp32 op sequence of DESIGN.md (R1, R4, R17).
// Partition axes (fig:hoq_self_attn): K and Q along head_dim per
// token (a new token's K forms its own partitions); V along the sequence
// per channel, one partition = one Pi-token block; the ragged V tail
// stays FP16 (R10).  Sums: P:687-688 (summation elimination).
//
// K/Q rows: 16 lanes per (token, head) row of d = 128 values; each lane owns 8
// consecutive channels (one 16-byte load, two Philox blocks).  Partition min/max
// and sums reduce with xor-shuffles over the Pi/8 lanes of the partition.
// V blocks: one thread per (block, head, channel) streams the Pi tokens twice
// (min/max, then quantize + pack), one Philox block per 4 tokens.
#include <cstdlib>

#include "append.cuh"
#include "common.cuh"
#include "internal.h"

namespace hack {

// Flat K/Q quantizer (hack_quantize_pack modes K and Q).
template <int BITS, bool FP16META>
__global__ void __launch_bounds__(256) quant_rows_flat_kernel(
    const __half* __restrict__ x, int64_t rows, int heads, int64_t pos0, int head0, uint64_t seed,
    uint32_t rng_id, int layer, int tag, int Pi, int round, uint8_t* __restrict__ codes,
    void* __restrict__ meta, void* __restrict__ sums, int sum_bytes) {
  const int lane16 = threadIdx.x & 15;
  const int64_t r = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 4);  // (row, head) pair
  const int64_t nr = rows * heads;
  const bool valid = r < nr;
  const int64_t rr = valid ? r : nr - 1;
  const int64_t row = rr / heads;
  const int h = (int)(rr % heads);
  const uint4 raw = reinterpret_cast<const uint4*>(x + rr * 128)[lane16];
  uint64_t packed;
  float m, s;
  int sum;
  quant_row16<BITS, FP16META>(raw, lane16, Pi, pos0 + row, seed, rng_id,
                              stream_c3(layer, tag, head0 + h), round, packed, m, s, sum);
  if (!valid) return;
  store_lane_codes<BITS>(codes + rr * (128 * BITS / 8), lane16, packed);
  const int nb = 128 / Pi;
  if ((lane16 & (Pi / 8 - 1)) == 0) {
    const int beta = lane16 / (Pi / 8);
    const int64_t mi = rr * nb + beta;
    if (FP16META)
      reinterpret_cast<__half2*>(meta)[mi] = make_meta(m, s);
    else
      reinterpret_cast<float2*>(meta)[mi] = make_float2(m, s);
    if (sum_bytes == 1)
      reinterpret_cast<uint8_t*>(sums)[mi] = (uint8_t)sum;
    else
      reinterpret_cast<uint16_t*>(sums)[mi] = (uint16_t)sum;
  }
}

// -------------------------------------------------------------------------- V blocks
template <int BITS>
__global__ void __launch_bounds__(128) quant_v_flat_kernel(
    const __half* __restrict__ x, int64_t nblk, int heads, int64_t pos0, int head0, uint64_t seed,
    uint32_t rng_id, int layer, int Pi, int round, uint8_t* __restrict__ codes, __half2* __restrict__ meta,
    void* __restrict__ sums, int sum_bytes) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (blk, h, c)
  if (id >= nblk * heads * 128) return;
  const int c = (int)(id % 128);
  const int h = (int)((id / 128) % heads);
  const int64_t j = id / (128 * heads);
  const __half* xc = x + ((j * Pi) * heads + h) * 128 + c;
  float m, s;
  int sum;
  quant_vcol<BITS>(xc, (int64_t)heads * 128, Pi, pos0 + j * Pi, c, seed, rng_id,
                   stream_c3(layer, kTagV, head0 + h), round, codes + id * (Pi * BITS / 8), m, s, sum);
  meta[id] = make_meta(m, s);
  store_sum(reinterpret_cast<uint8_t*>(sums), (int)id, sum_bytes, sum);
}

// -------------------------------------------------------------------------- paged ingest

// K rows of every prompt token -> pages (a1).
template <int BITS>
HACK_DEV void ingest_k_body(const __half* __restrict__ k, const int32_t* __restrict__ cu_seqlens,
                            const int32_t* __restrict__ slots, const CacheView& cv, const KernelCfg& kc, int bx,
                            int b, int tid) {
  const int start = cu_seqlens[b], L = cu_seqlens[b + 1] - start;
  const int slot = slots[b];
  const int H = kc.Hkv, Hl = kc.kvh_count;  // layout heads; heads of this launch (from kc.kvh_begin)
  const int lane16 = tid & 15;
  const int r = bx * 16 + (tid >> 4);
  if (bx * 16 >= L * Hl) return;  // whole block out of range (uniform)
  const bool valid = r < L * Hl;
  const int rr = valid ? r : L * Hl - 1;
  const int t = rr / Hl, h = kc.kvh_begin + rr % Hl;
  const uint4 raw = reinterpret_cast<const uint4*>(k + ((int64_t)(start + t) * H + h) * 128)[lane16];
  uint64_t packed;
  float m, s;
  int sum;
  const uint32_t rng_id = cv.rng_ids[slot];
  quant_row16<BITS, true>(raw, lane16, kc.Pi, t, kc.seed, rng_id,
                          stream_c3(kc.layer, kTagK, kc.head_base + h), kc.kv_round, packed, m, s, sum);
  if (!valid) return;
  const PageLayout& PL = kc.pl;
  uint8_t* pg = page_ptr(cv, slot, t / kc.Pi, h);
  const int row = t % kc.Pi;
  store_lane_codes<BITS>(pg + PL.k_codes + row * (128 * BITS / 8), lane16, packed);
  const int nb = 128 / kc.Pi;
  if ((lane16 & (kc.Pi / 8 - 1)) == 0) {
    const int beta = lane16 / (kc.Pi / 8);
    reinterpret_cast<__half2*>(pg + PL.k_meta)[row * nb + beta] = make_meta(m, s);
    store_sum(pg + PL.k_sums, row * nb + beta, PL.sum_bytes, sum);
  }
}

template <int BITS>
__global__ void __launch_bounds__(256) ingest_k_kernel(const __half* __restrict__ k,
                                                       const int32_t* __restrict__ cu_seqlens,
                                                       const int32_t* __restrict__ slots, CacheView cv,
                                                       KernelCfg kc) {
  ingest_k_body<BITS>(k, cu_seqlens, slots, cv, kc, blockIdx.x, blockIdx.y, threadIdx.x);
}

// Full V blocks -> pages (a2); ragged remainder -> FP16 tail (R10); seq_lens.
template <int BITS>
__global__ void __launch_bounds__(128) ingest_v_kernel(const __half* __restrict__ v,
                                                       const int32_t* __restrict__ cu_seqlens,
                                                       const int32_t* __restrict__ slots, CacheView cv,
                                                       KernelCfg kc) {
  asm volatile("griddepcontrol.launch_dependents;");  // (prefill attention, see ingest_kv64_kernel)
  const int b = blockIdx.y;
  const int start = cu_seqlens[b], L = cu_seqlens[b + 1] - start;
  const int slot = slots[b];
  const int H = kc.Hkv, Pi = kc.Pi;
  const int nfull = L / Pi;
  const int id = blockIdx.x * blockDim.x + threadIdx.x;  // (blk, h, c), blk in [0, nfull]
  if (id == 0) cv.seq_lens[slot] = L;
  const int Hl = kc.kvh_count;  // heads of this launch (from kc.kvh_begin)
  const int c = id % 128, h = kc.kvh_begin + (id / 128) % Hl, j = id / (128 * Hl);
  if (j > nfull) return;
  const __half* xc = v + ((int64_t)(start + j * Pi) * H + h) * 128 + c;
  if (j == nfull) {  // FP16 tail rows (reading R10)
    __half* tail = reinterpret_cast<__half*>(cv.v_tail) + (((int64_t)slot * H + h) * Pi) * 128 + c;
    for (int t = 0; t < L - nfull * Pi; ++t) tail[t * 128] = xc[(int64_t)t * H * 128];
    return;
  }
  const PageLayout& PL = kc.pl;
  uint8_t* pg = page_ptr(cv, slot, j, h);
  float m, s;
  int sum;
  quant_vcol<BITS>(xc, (int64_t)H * 128, Pi, (int64_t)j * Pi, c, kc.seed, cv.rng_ids[slot],
                   stream_c3(kc.layer, kTagV, kc.head_base + h), kc.kv_round,
                   pg + PL.v_codes + c * (Pi * BITS / 8), m, s, sum);
  reinterpret_cast<__half2*>(pg + PL.v_meta)[c] = make_meta(m, s);
  store_sum(pg + PL.v_sums, c, PL.sum_bytes, sum);
}

// Full V blocks -> pages (a2) at Pi = 64, 4 threads per (block, head, channel): CTA =
// 4 warps x 32 consecutive channels of one (block, head); warp q owns tokens 16q..16q+15,
// so a warp's token loads are 64-byte coalesced rows and each thread packs exactly 16
// codes (one u32 at b = 2, one u64 at b = 4).  Partition min/max and code sums are
// combined across the 4 warps in shared memory.  Same per-element op sequence and
// Philox counters as quant_vcol (R1, R3, R4), hence the same codes.  Blocks j == nfull
// copy the ragged remainder to the FP16 tail (R10); block 0 sets seq_lens.
struct V64Red {
  float lo[4][32], hi[4][32];
  int sum[4][32];
};

// One (block, head, 32-channel group) unit on 128 threads; `bar` is the named barrier of
// those 128 threads (two units share a CTA in the fused ingest kernel).
template <int BITS>
HACK_DEV void ingest_v64_body(const __half* __restrict__ v, const int32_t* __restrict__ cu_seqlens,
                              const int32_t* __restrict__ slots, const CacheView& cv, const KernelCfg& kc, int bx,
                              int b, int tid, int bar, V64Red& red) {
  constexpr int PI = 64, qmax = (1 << BITS) - 1;
  auto sync = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory"); };
  const int start = cu_seqlens[b], L = cu_seqlens[b + 1] - start;
  const int slot = slots[b];
  const int H = kc.Hkv;
  const int nfull = L / PI;
  const int Hl = kc.kvh_count;  // heads of this launch (from kc.kvh_begin)
  const int cg = bx & 3, h = kc.kvh_begin + (bx >> 2) % Hl, j = (bx >> 2) / Hl;
  const int q = tid >> 5, lane = tid & 31;
  const int c = 32 * cg + lane;
  if (bx == 0 && tid == 0) cv.seq_lens[slot] = L;
  if (j > nfull) return;
  const __half* xc = v + ((int64_t)(start + j * PI) * H + h) * 128 + c;
  const int64_t ts = (int64_t)H * 128;
  if (j == nfull) {  // FP16 tail rows (reading R10)
    __half* tail = reinterpret_cast<__half*>(cv.v_tail) + (((int64_t)slot * H + h) * PI) * 128 + c;
    for (int t = q; t < L - nfull * PI; t += 4) tail[t * 128] = xc[(int64_t)t * ts];
    return;
  }
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = __half2float(xc[(int64_t)(16 * q + i) * ts]);
  float lo = x[0], hi = x[0];
#pragma unroll
  for (int i = 1; i < 16; ++i) {
    lo = fminf(lo, x[i]);
    hi = fmaxf(hi, x[i]);
  }
  red.lo[q][lane] = lo;
  red.hi[q][lane] = hi;
  sync();
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    lo = fminf(lo, red.lo[w][lane]);
    hi = fmaxf(hi, red.hi[w][lane]);
  }
  const QMeta qm = meta_fp16(lo, hi, qmax);
  const uint32_t rng_id = cv.rng_ids[slot];
  const uint32_t c3 = stream_c3(kc.layer, kTagV, kc.head_base + h);
  const int64_t pos = (int64_t)j * PI + 16 * q;  // absolute position of this thread's first token
  uint64_t packed = 0;
  int sum = 0;
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) {
    int cc[4];
    if (kc.kv_round == HACK_ROUND_STOCHASTIC) {
      // element (pos+t, ch): Philox block n = ((pos+t) >> 2)*d + ch, word (pos+t) & 3 (R3)
      const Philox4 r = philox_block(kc.seed, rng_id, c3, (uint64_t)((pos + 4 * k4) >> 2) * 128u + (uint64_t)c);
      cc[0] = quant_sr(x[4 * k4 + 0], qm, u24(r.x), qmax);
      cc[1] = quant_sr(x[4 * k4 + 1], qm, u24(r.y), qmax);
      cc[2] = quant_sr(x[4 * k4 + 2], qm, u24(r.z), qmax);
      cc[3] = quant_sr(x[4 * k4 + 3], qm, u24(r.w), qmax);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) cc[i] = quant_rn(x[4 * k4 + i], qm, qmax);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      packed |= (uint64_t)cc[i] << (BITS * (4 * k4 + i));
      sum += cc[i];
    }
  }
  const PageLayout& PL = kc.pl;
  uint8_t* pg = page_ptr(cv, slot, j, h);
  if (BITS == 2)
    reinterpret_cast<uint32_t*>(pg + PL.v_codes + c * 16)[q] = (uint32_t)packed;
  else
    reinterpret_cast<uint2*>(pg + PL.v_codes + c * 32)[q] = make_uint2((uint32_t)packed, (uint32_t)(packed >> 32));
  red.sum[q][lane] = sum;
  sync();
  if (q == 0) {
    const int tot = red.sum[0][lane] + red.sum[1][lane] + red.sum[2][lane] + red.sum[3][lane];
    reinterpret_cast<__half2*>(pg + PL.v_meta)[c] = make_meta(qm.m, qm.s);
    store_sum(pg + PL.v_sums, c, PL.sum_bytes, tot);
  }
}

template <int BITS>
__global__ void __launch_bounds__(128) ingest_v64_kernel(const __half* __restrict__ v,
                                                         const int32_t* __restrict__ cu_seqlens,
                                                         const int32_t* __restrict__ slots, CacheView cv,
                                                         KernelCfg kc) {
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ V64Red red;
  ingest_v64_body<BITS>(v, cu_seqlens, slots, cv, kc, blockIdx.x, blockIdx.y, threadIdx.x, 0, red);
}

// K rows and V blocks of a prompt in ONE launch (Pi = 64): blocks [0, nk) quantize K rows,
// the rest carry two V units each (threads 0-127 and 128-255), so the two ALU-bound
// quantizers overlap instead of running back to back.
template <int BITS>
__global__ void __launch_bounds__(256) ingest_kv64_kernel(const __half* __restrict__ k, const __half* __restrict__ v,
                                                          const int32_t* __restrict__ cu_seqlens,
                                                          const int32_t* __restrict__ slots, CacheView cv,
                                                          KernelCfg kc, int nk, int nv) {
  // the prefill attention kernel is launched as a programmatic dependent of the ingest
  // (hack_prefill_attention): let it start its Q quantization now; it reads the cache only
  // after griddepcontrol.wait, i.e. after this grid completed
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ V64Red red[2];
  if ((int)blockIdx.x < nk) {
    ingest_k_body<BITS>(k, cu_seqlens, slots, cv, kc, blockIdx.x, blockIdx.y, threadIdx.x);
    return;
  }
  const int half = threadIdx.x >> 7;
  const int vb = 2 * ((int)blockIdx.x - nk) + half;
  if (vb < nv) ingest_v64_body<BITS>(v, cu_seqlens, slots, cv, kc, vb, blockIdx.y, threadIdx.x & 127, 1 + half, red[half]);
}

// -------------------------------------------------------------------------- decode append (a8)
// One cluster of CL CTAs per request (grid CL x batch, CL | Hkv, CL <= 8), 128 threads
// (= d channels); CTA x serves KV heads x, x + CL, ...:
// quantize k_new into its own partitions in the current page, write v_new
// to the FP16 tail, flush the tail into the page's V section when it reaches Pi
// (P:723), then seq_lens += 1.
template <int BITS, bool RQE>
__global__ void __launch_bounds__(128) append_kernel(const __half* __restrict__ k_new,
                                                     const __half* __restrict__ v_new,
                                                     const int32_t* __restrict__ slots, CacheView cv,
                                                     KernelCfg kc) {
  const int b = blockIdx.y;
  const int slot = slots[b];
  const int H = kc.Hkv, Pi = kc.Pi;
  const int t = cv.seq_lens[slot];
  // capacity guard: a request whose next token needs a block beyond its block-table row is
  // not appended (nothing written, seq_lens unchanged) rather than spilling into the next
  // slot's row; uniform over the cluster (every CTA read the same t), so no barrier is skipped
  // by only some of them.  hack_decode_attention rejects such a call on the host.
  if (t / Pi >= cv.max_pages_per_req) return;
  for (int h = blockIdx.x; h < H; h += gridDim.x)
    append_unit<BITS, RQE, 128>(k_new, v_new, b, slot, t, h, cv, kc, threadIdx.x, [] { __syncthreads(); });
  // every thread of the request's cluster has read seq_lens before it changes
  if (gridDim.x > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cv.seq_lens[slot] = t + 1;
}

// -------------------------------------------------------------------------- launchers
cudaError_t launch_quantize_pack(const KernelCfg& kc, int mode, const void* x, int64_t rows, int heads,
                                 int64_t pos0, int head0, uint32_t rng_id, uint8_t* codes, void* meta,
                                 void* sums, cudaStream_t st) {
  const __half* xh = reinterpret_cast<const __half*>(x);
  if (mode == HACK_QMODE_V) {
    const int64_t nblk = rows / kc.Pi;
    const int64_t n = nblk * heads * 128;
    const int grid = (int)((n + 127) / 128);
    if (kc.bits == 2)
      quant_v_flat_kernel<2><<<grid, 128, 0, st>>>(xh, nblk, heads, pos0, head0, kc.seed, rng_id, kc.layer,
                                                   kc.Pi, kc.kv_round, codes, (__half2*)meta, sums,
                                                   kc.pl.sum_bytes);
    else
      quant_v_flat_kernel<4><<<grid, 128, 0, st>>>(xh, nblk, heads, pos0, head0, kc.seed, rng_id, kc.layer,
                                                   kc.Pi, kc.kv_round, codes, (__half2*)meta, sums,
                                                   kc.pl.sum_bytes);
    note_launch();
    return cudaGetLastError();
  }
  const int64_t n = rows * heads;
  const int grid = (int)((n + 15) / 16);
  if (mode == HACK_QMODE_Q)
    quant_rows_flat_kernel<8, false><<<grid, 256, 0, st>>>(xh, rows, heads, pos0, head0, kc.seed, rng_id,
                                                           kc.layer, kTagQ, kc.Pi, kc.q_round, codes, meta,
                                                           sums, 2);
  else if (kc.bits == 2)
    quant_rows_flat_kernel<2, true><<<grid, 256, 0, st>>>(xh, rows, heads, pos0, head0, kc.seed, rng_id,
                                                          kc.layer, kTagK, kc.Pi, kc.kv_round, codes, meta,
                                                          sums, kc.pl.sum_bytes);
  else
    quant_rows_flat_kernel<4, true><<<grid, 256, 0, st>>>(xh, rows, heads, pos0, head0, kc.seed, rng_id,
                                                          kc.layer, kTagK, kc.Pi, kc.kv_round, codes, meta,
                                                          sums, kc.pl.sum_bytes);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_ingest(const KernelCfg& kc, const void* k, const void* v, const int32_t* cu_seqlens,
                          const int32_t* slots, int batch, int max_seqlen, const CacheView& cv,
                          cudaStream_t st) {
  const __half* kh = reinterpret_cast<const __half*>(k);
  const __half* vh = reinterpret_cast<const __half*>(v);
  dim3 gk((max_seqlen * kc.kvh_count + 15) / 16, batch);
  dim3 gv(((max_seqlen / kc.Pi + 1) * kc.kvh_count * 128 + 127) / 128, batch);
  dim3 gv64((max_seqlen / kc.Pi + 1) * kc.kvh_count * 4, batch);  // (block, head, 32-channel group)
  const bool v64 = kc.Pi == 64;
  if (v64) {
    const int nk = gk.x, nv = gv64.x;
    dim3 g(nk + (nv + 1) / 2, batch);
    if (kc.bits == 2)
      ingest_kv64_kernel<2><<<g, 256, 0, st>>>(kh, vh, cu_seqlens, slots, cv, kc, nk, nv);
    else
      ingest_kv64_kernel<4><<<g, 256, 0, st>>>(kh, vh, cu_seqlens, slots, cv, kc, nk, nv);
    note_launch(1);
    return cudaGetLastError();
  }
  if (kc.bits == 2) {
    ingest_k_kernel<2><<<gk, 256, 0, st>>>(kh, cu_seqlens, slots, cv, kc);
    if (v64)
      ingest_v64_kernel<2><<<gv64, 128, 0, st>>>(vh, cu_seqlens, slots, cv, kc);
    else
      ingest_v_kernel<2><<<gv, 128, 0, st>>>(vh, cu_seqlens, slots, cv, kc);
  } else {
    ingest_k_kernel<4><<<gk, 256, 0, st>>>(kh, cu_seqlens, slots, cv, kc);
    if (v64)
      ingest_v64_kernel<4><<<gv64, 128, 0, st>>>(vh, cu_seqlens, slots, cv, kc);
    else
      ingest_v_kernel<4><<<gv, 128, 0, st>>>(vh, cu_seqlens, slots, cv, kc);
  }
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_append(const KernelCfg& kc, const void* k_new, const void* v_new, const int32_t* slots,
                          int batch, const CacheView& cv, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  const __half* kh = reinterpret_cast<const __half*>(k_new);
  const __half* vh = reinterpret_cast<const __half*>(v_new);
  // KV heads of one request spread over a cluster (a serial head loop in one CTA left the
  // 64-request C3 append latency-bound at ~16 us, 13 % of the decode step)
  int cl = 1;
  for (int c = 8; c > 1; --c)
    if (kc.Hkv % c == 0) { cl = c; break; }
  if (const char* e = getenv("HACK_APPEND_CL")) {  // timing knob: 1 = the serial head loop
    const int v = atoi(e);
    if (v >= 1 && v <= 8 && kc.Hkv % v == 0) cl = v;
  }
  const bool no_rqe = getenv("HACK_DECODE_NO_RQE") && kc.Pi == 64;  // f2 ablation only
  void (*kern)(const __half*, const __half*, const int32_t*, CacheView, KernelCfg) =
      kc.bits == 2 ? (no_rqe ? append_kernel<2, false> : append_kernel<2, true>)
                   : (no_rqe ? append_kernel<4, false> : append_kernel<4, true>);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cl, batch);
  lc.blockDim = dim3(128);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = cl > 1 ? 1 : 0;
  const cudaError_t err = cudaLaunchKernelEx(&lc, kern, kh, vh, slots, cv, kc);
  note_launch();
  return err != cudaSuccess ? err : cudaGetLastError();
}

}  // namespace hack
