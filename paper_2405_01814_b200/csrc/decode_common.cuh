// decode_common.cuh — parameters, KV addressing, the persistent work pipeline and the split-K
// epilogue shared by the decode kernels.
//
// Both decode kernels are persistent: gridDim.x = resident CTAs, one producer warp per CTA
// claims work items (request, kv head, q-head group, split) from a global counter and streams
// their K/V tiles into a shared-memory ring without ever draining it between items; the
// consumer warps follow the ring, reading each stage's item tag.  A CTA never ramps its
// pipeline down and up again between items, which is what a split-K grid of short-lived CTAs
// pays for on every CTA start.
//
// Semantics follow the reference's mergeable partial form
// (/root/reference/proj/core/src/attention.cpp:72-127): an item reduces a contiguous token
// range of one (request, kv head) to a max-shifted partial (acc[d], max, sum); the partials of
// one (request, q head) are merged in split order by the consumer that completes the last one
// (merge, attention.cpp:100-118, identity early-out included) and finalized to
// out = acc / sum (attention.cpp:68, 120-127).
#pragma once

#include <math.h>
#include <stdint.h>

#include "ptx.cuh"

namespace lam {

struct DecodeParams {
  const void* q;            // [B][Hq][D]
  const void* k_pool;       // see lamina_attn.h for the layouts
  const void* v_pool;
  const int32_t* page_table;  // nullptr => dense [B][Hkv][P][D]
  const int32_t* seq_lens;    // [B]
  void* out;                // [B][Hq][D], T or float
  float* lse;               // [B][Hq] or nullptr
  float* ws_acc;            // [B*Hq*S][D] split partials (unnormalised acc)
  float* ws_ml;             // [B*Hq*S][2] (max in natural-log units, sum)
  int32_t* counters;        // [B*Hkv*QG] split arrival counters (self-resetting)
  int32_t* work;            // [2] item counter, exited-producer counter (self-resetting)
  int32_t B, Hq, Hkv, G, D;
  int32_t page_size, pt_stride;
  int32_t chunk;            // tokens per split (multiple of the kernel tile)
  int32_t S;                // number of splits
  int32_t QG;               // q-head groups per kv head (G / heads per CTA)
  int32_t n_items;          // B * Hkv * QG * S
  float scale;              // softmax scale (natural units)
  float scale_log2;         // scale * log2(e)
  int32_t out_f32;
};

// Physical row of token t of (request b, kv head h) in a pool viewed as [rows][D].
// Paged: pool[page][Hkv][P][D]; dense: pool[B][Hkv][P][D] (P = row capacity).
__device__ __forceinline__ int64_t kv_row(const DecodeParams& p, int b, int h, int t) {
  const int64_t blk =
      p.page_table ? static_cast<int64_t>(__ldg(p.page_table + static_cast<int64_t>(b) * p.pt_stride +
                                                t / p.page_size))
                   : static_cast<int64_t>(b);
  return (blk * p.Hkv + h) * p.page_size + (t % p.page_size);
}

struct Item {
  int b, kvh, qg, split;
  int len, t_begin, t_end, ntiles;
};

// Work item `idx`: split fastest, then q-head group, kv head, request.
__device__ __forceinline__ Item make_item(const DecodeParams& p, int idx, int tile) {
  Item it;
  it.split = idx % p.S;
  int unit = idx / p.S;
  it.qg = unit % p.QG;
  unit /= p.QG;
  it.kvh = unit % p.Hkv;
  it.b = unit / p.Hkv;
  it.len = __ldg(p.seq_lens + it.b);
  it.t_begin = it.split * p.chunk;
  it.t_end = min(it.len, it.t_begin + p.chunk);
  it.ntiles = it.t_end > it.t_begin ? (it.t_end - it.t_begin + tile - 1) / tile : 0;
  return it;
}

// Splits of a (request, kv head, q group) unit that carry tokens (>= 1: an empty request
// still produces its zero output through split 0).
__device__ __forceinline__ int live_splits(const DecodeParams& p, int len) {
  return len > 0 ? min(p.S, (len + p.chunk - 1) / p.chunk) : 1;
}

// ---- persistent producer ---------------------------------------------------------------
// meta[s] = {item, tile index, tiles of the item, 0}; item < 0 is the end-of-work sentinel.
// `issue(s, it, j)` must arrive on full[s] with expect_tx and start the stage's TMA copies.
template <int STAGES, int TILE, class Issue>
__device__ __forceinline__ void producer_loop(const DecodeParams& p, uint64_t* full,
                                              uint64_t* empty, int4* meta, Issue issue) {
  int i = 0;
  auto acquire = [&](int k) {
    const int s = k % STAGES;
    if (k >= STAGES) mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
    return s;
  };
  for (;;) {
    const int idx = atomicAdd(p.work, 1);
    if (idx >= p.n_items) break;
    const Item it = make_item(p, idx, TILE);
    if (it.ntiles == 0) {
      if (it.split != 0 || it.len > 0) continue;  // empty split: nothing to merge
      const int s = acquire(i++);                 // empty request: zero-output marker
      meta[s] = make_int4(idx, 0, 0, 0);
      mbar_arrive(&full[s]);
      continue;
    }
    for (int j = 0; j < it.ntiles; ++j) {
      const int s = acquire(i++);
      meta[s] = make_int4(idx, j, it.ntiles, 0);
      issue(s, it, j);
    }
  }
  const int s = acquire(i);
  meta[s] = make_int4(-1, 0, 0, 0);
  mbar_arrive(&full[s]);
  // the last producer to leave resets the counters for the next launch
  if (atomicAdd(p.work + 1, 1) == static_cast<int>(gridDim.x) - 1) {
    p.work[0] = 0;
    p.work[1] = 0;
  }
}

template <typename T>
__device__ __forceinline__ void store_out(const DecodeParams& p, int64_t idx, float v) {
  if (p.out_f32)
    static_cast<float*>(p.out)[idx] = v;
  else
    static_cast<T*>(p.out)[idx] = Elem<T>::from_float(v);
}

// End of one work item, run by all NW*32 consumer threads after a consumer barrier.
// red_m/red_l/red_acc hold the NW per-warp partials for GQ q heads: red_m[w*GQ+g] (log2 units
// if kLog2, else natural), red_l[w*GQ+g], red_acc[(w*GQ+g)*D + d].  `nvalid` q heads of the
// group are real (the MMA kernel pads to 8).
template <typename T, int D, int GQ, int NW, bool kLog2>
__device__ __forceinline__ void finish_item(const DecodeParams& p, const Item& it, int nvalid,
                                            const float* red_m, const float* red_l,
                                            const float* red_acc, int* s_flag) {
  constexpr int kThreads = NW * 32;
  constexpr float kLn2 = 0.6931471805599453f;
  const int tid = threadIdx.x;
  const int b = it.b;
  const int qh0 = it.kvh * p.G + it.qg * GQ;

  // 1. merge the NW warp partials (fixed warp order => deterministic).
  float cta_m[GQ], cta_l[GQ];
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, red_m[w * GQ + g]);
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float mw = red_m[w * GQ + g];
      if (mw != -INFINITY) L += (kLog2 ? exp2f(mw - M) : expf(mw - M)) * red_l[w * GQ + g];
    }
    cta_m[g] = (M == -INFINITY) ? -INFINITY : (kLog2 ? M * kLn2 : M);  // natural units
    cta_l[g] = L;
  }
  auto merged_acc = [&](int g, int d) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, red_m[w * GQ + g]);
    float A = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float mw = red_m[w * GQ + g];
      if (mw != -INFINITY)
        A += (kLog2 ? exp2f(mw - M) : expf(mw - M)) * red_acc[(w * GQ + g) * D + d];
    }
    return A;
  };

  if (live_splits(p, it.len) == 1) {
    for (int e = tid; e < GQ * D; e += kThreads) {
      const int g = e / D, d = e % D;
      if (g >= nvalid) continue;
      const float A = merged_acc(g, d), L = cta_l[g];
      const int64_t o = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * D + d;
      store_out<T>(p, o, L > 0.f ? A / L : 0.f);
    }
    if (p.lse != nullptr && tid < GQ && tid < nvalid)
      p.lse[static_cast<int64_t>(b) * p.Hq + qh0 + tid] =
          cta_l[tid] > 0.f ? cta_m[tid] + logf(cta_l[tid]) : -INFINITY;
    return;
  }

  // 2. write this split's partial.
  for (int e = tid; e < GQ * D; e += kThreads) {
    const int g = e / D, d = e % D;
    if (g >= nvalid) continue;
    const int64_t row = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * p.S + it.split;
    p.ws_acc[row * D + d] = merged_acc(g, d);
  }
  if (tid < GQ && tid < nvalid) {
    const int64_t row = (static_cast<int64_t>(b) * p.Hq + qh0 + tid) * p.S + it.split;
    p.ws_ml[row * 2 + 0] = cta_m[tid];
    p.ws_ml[row * 2 + 1] = cta_l[tid];
  }
  __threadfence();
  named_bar_sync(1, kThreads);
  int32_t* counter = p.counters + (static_cast<int64_t>(b) * p.Hkv + it.kvh) * p.QG + it.qg;
  if (tid == 0) {
    const int prev = atomicAdd(counter, 1);
    *s_flag = (prev == live_splits(p, it.len) - 1);
  }
  named_bar_sync(1, kThreads);
  if (!*s_flag) return;
  __threadfence();

  // 3. last split of this unit: merge the live partials in split order and finalize.
  const int S_live = live_splits(p, it.len);
  for (int e = tid; e < GQ * D; e += kThreads) {
    const int g = e / D, d = e % D;
    if (g >= nvalid) continue;
    const int64_t row0 = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * p.S;
    float M = -INFINITY;
    for (int s = 0; s < S_live; ++s) M = fmaxf(M, __ldcg(p.ws_ml + (row0 + s) * 2));
    float A = 0.f, L = 0.f;
    for (int s = 0; s < S_live; ++s) {
      const float ms = __ldcg(p.ws_ml + (row0 + s) * 2);
      if (ms == -INFINITY) continue;
      const float w = expf(ms - M);
      L += w * __ldcg(p.ws_ml + (row0 + s) * 2 + 1);
      A += w * __ldcg(p.ws_acc + (row0 + s) * D + d);
    }
    const int64_t o = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * D + d;
    store_out<T>(p, o, L > 0.f ? A / L : 0.f);
    if (d == 0 && p.lse != nullptr)
      p.lse[static_cast<int64_t>(b) * p.Hq + qh0 + g] = L > 0.f ? M + logf(L) : -INFINITY;
  }
  if (tid == 0) *counter = 0;  // ready for the next launch
}

}  // namespace lam
