// decode_common.cuh — parameters, KV addressing and the split-K epilogue shared by the
// decode kernels.
//
// Semantics follow the reference's mergeable partial form
// (/root/reference/proj/core/src/attention.cpp:72-127): every CTA reduces a contiguous
// token range of one (request, kv head) to a max-shifted partial (acc[d], max, sum);
// partials of one (request, q head) are merged in split order by the last CTA to finish
// (merge, attention.cpp:100-118, identity early-out included) and finalized to
// out = acc / sum (attention.cpp:68 / 120-127).
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
  int32_t* counters;        // [B*Hkv*QG] arrival counters (self-resetting)
  int32_t B, Hq, Hkv, G, D;
  int32_t page_size, pt_stride;
  int32_t chunk;            // tokens per split (multiple of the kernel tile)
  int32_t S;                // number of splits
  int32_t QG;               // q-head groups per kv head (G / heads per CTA)
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

template <typename T>
__device__ __forceinline__ void store_out(const DecodeParams& p, int64_t idx, float v) {
  if (p.out_f32)
    static_cast<float*>(p.out)[idx] = v;
  else
    static_cast<T*>(p.out)[idx] = Elem<T>::from_float(v);
}

// Final stage of every decode CTA.  `red_m/red_l/red_acc` hold NW per-warp partials
// for GQ q heads: red_m[w*GQ+g] (log2 units if kLog2, else natural), red_l[w*GQ+g],
// red_acc[(w*GQ+g)*D + d].  Called by all NW*32 consumer threads after a consumer
// barrier.  `nvalid` q heads of the group are real (the MMA kernel pads to 8).
template <typename T, int D, int GQ, int NW, bool kLog2>
__device__ __forceinline__ void finish_cta(const DecodeParams& p, int b, int kvh, int qg,
                                           int split, int nvalid, const float* red_m,
                                           const float* red_l, const float* red_acc,
                                           int* s_flag) {
  constexpr int kThreads = NW * 32;
  constexpr float kLn2 = 0.6931471805599453f;
  const int tid = threadIdx.x;
  const int qh0 = kvh * p.G + qg * GQ;

  // 1. merge the NW warp partials of this CTA (fixed warp order => deterministic).
  //    Each thread owns (g, d) pairs.
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

  if (p.S == 1) {
    for (int e = tid; e < GQ * D; e += kThreads) {
      const int g = e / D, d = e % D;
      if (g >= nvalid) continue;
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
      const float L = cta_l[g];
      const int64_t o = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * D + d;
      store_out<T>(p, o, L > 0.f ? A / L : 0.f);
    }
    if (p.lse != nullptr && tid < GQ && tid < nvalid) {
      p.lse[static_cast<int64_t>(b) * p.Hq + qh0 + tid] =
          cta_l[tid] > 0.f ? cta_m[tid] + logf(cta_l[tid]) : -INFINITY;
    }
    return;
  }

  // 2. write this split's partial.
  for (int e = tid; e < GQ * D; e += kThreads) {
    const int g = e / D, d = e % D;
    if (g >= nvalid) continue;
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
    const int64_t row = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * p.S + split;
    p.ws_acc[row * D + d] = A;
  }
  if (tid < GQ && tid < nvalid) {
    const int64_t row = (static_cast<int64_t>(b) * p.Hq + qh0 + tid) * p.S + split;
    p.ws_ml[row * 2 + 0] = cta_m[tid];
    p.ws_ml[row * 2 + 1] = cta_l[tid];
  }
  __threadfence();
  named_bar_sync(1, kThreads);
  int32_t* counter = p.counters + (static_cast<int64_t>(b) * p.Hkv + kvh) * p.QG + qg;
  if (tid == 0) {
    const int prev = atomicAdd(counter, 1);
    *s_flag = (prev == p.S - 1);
  }
  named_bar_sync(1, kThreads);
  if (!*s_flag) return;
  __threadfence();

  // 3. last CTA of this (request, kv head, q group): merge all S partials in split
  //    order (identity partials — empty splits — contribute nothing) and finalize.
  for (int e = tid; e < GQ * D; e += kThreads) {
    const int g = e / D, d = e % D;
    if (g >= nvalid) continue;
    const int64_t row0 = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * p.S;
    float M = -INFINITY;
    for (int s = 0; s < p.S; ++s) M = fmaxf(M, __ldcg(p.ws_ml + (row0 + s) * 2));
    float A = 0.f, L = 0.f;
    for (int s = 0; s < p.S; ++s) {
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
