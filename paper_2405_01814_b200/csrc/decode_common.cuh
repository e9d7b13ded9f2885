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
  const void* q;            // request b, q head h at q + b * q_stride + h * D
  int64_t q_stride;
  const void* k_pool;       // see lamina_attn.h for the layouts
  const void* v_pool;
  const int32_t* page_table;  // nullptr => dense [B][Hkv][P][D]
  const int32_t* seq_lens;    // [B]
  void* out;                // [B][Hq][D], T or float
  float* lse;               // [B][Hq] or nullptr
  float* ws_acc;            // [B*Hq*S][D] split partials (unnormalised acc)
  float* ws_ml;             // [B*Hq*S][2] (max in natural-log units, sum)
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
  int32_t flags;            // tuning: bit2 = all-dynamic schedule, bit3 = skip epilogue (diag)
  // fused append (optional): the new token of request b (position seq_lens[b] - 1) comes from
  // k_new/v_new (request b, kv head h at + b * new_stride + h * D); the kernel attends over it
  // from shared memory and writes it into the pools for later steps.
  const void* k_new;
  const void* v_new;
  int64_t new_stride;
  void* k_pool_w;
  void* v_pool_w;
  const int32_t* order;     // optional request permutation for item enumeration (LPT)
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
  if (p.order != nullptr) it.b = __ldg(p.order + it.b);
  it.len = __ldg(p.seq_lens + it.b);
  it.t_begin = it.split * p.chunk;
  it.t_end = min(it.len, it.t_begin + p.chunk);
  it.ntiles = it.t_end > it.t_begin ? (it.t_end - it.t_begin + tile - 1) / tile : 0;
  return it;
}

// Item fields from a stage tag {idx, tile, len, t_end} without touching global memory
// (consumers must never stall on a load at an item boundary).
template <int TILE>
__device__ __forceinline__ Item item_from_tag(const DecodeParams& p, int4 tag) {
  Item it;
  it.split = tag.x % p.S;
  int unit = tag.x / p.S;
  it.qg = unit % p.QG;
  unit /= p.QG;
  it.kvh = unit % p.Hkv;
  it.b = unit / p.Hkv;
  if (p.order != nullptr) it.b = __ldg(p.order + it.b);
  it.len = tag.z;
  it.t_begin = it.split * p.chunk;
  it.t_end = tag.w;
  it.ntiles = it.t_end > it.t_begin ? (it.t_end - it.t_begin + TILE - 1) / TILE : 0;
  return it;
}

// Does tile j of this item hold the request's new token (fused append)?
template <int TILE>
__device__ __forceinline__ bool tile_has_new(const DecodeParams& p, const Item& it, int j) {
  return p.k_new != nullptr && it.t_end == it.len && it.len > 0 && j == it.ntiles - 1;
}

// Splits of a (request, kv head, q group) unit that carry tokens (>= 1: an empty request
// still produces its zero output through split 0).
__device__ __forceinline__ int live_splits(const DecodeParams& p, int len) {
  return len > 0 ? min(p.S, (len + p.chunk - 1) / p.chunk) : 1;
}

// ---- persistent producer ---------------------------------------------------------------
// meta[s] = {item, tile index, request length, item end token}; item < 0 ends the work.
// meta_row[s] = first pool row of the stage's tile (consumers write the fused new token there).
// `issue(s, it, j, row)` must arrive on full[s] with expect_tx and start the stage's TMA
// copies of tile j, whose first KV row is `row`.
//
// Schedule: hybrid static-then-dynamic.
//  * Static rounds: CTA c runs items c, c + G, c + 2G, ... for all but the last ~2 rounds.  Its
//    next item is known, so the item's length and first page-table entry are loaded while the
//    current item streams: an item boundary costs the HBM stream nothing.  (With claiming at
//    every boundary, the claim atomic -> length -> page-entry round trips idled each SM for
//    ~3 us per item, ~7 % of C2/C3.)
//  * Dynamic tail: the remaining items are claimed from a global counter, which absorbs the
//    2-3 % per-SM streaming-rate differences of the two-die part and the tail.
template <int STAGES, int TILE, class Issue>
__device__ __forceinline__ void producer_loop(const DecodeParams& p, uint64_t* full,
                                              uint64_t* empty, int4* meta, long long* meta_row,
                                              Issue issue) {
  int i = 0;
  auto acquire = [&](int k) {
    const int s = k % STAGES;
    if (k >= STAGES) mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
    return s;
  };
  // stream one item; `during` runs once, right after the stage of tile `at` is issued
  // (at < 0: after the last tile)
  auto run_item = [&](int idx, const Item& it, int64_t row0, int at, auto&& during) {
    if (it.ntiles == 0) {
      if (it.split == 0 && it.len == 0) {  // empty request: zero-output marker
        const int s = acquire(i++);
        meta[s] = make_int4(idx, 0, 0, 0);
        mbar_arrive(&full[s]);
      }                                    // (an empty split has nothing to merge)
      during();
      return;
    }
    const int when = at < 0 ? it.ntiles - 1 : min(at, it.ntiles - 1);
    for (int j = 0; j < it.ntiles; ++j) {
      const int s = acquire(i++);
      const int64_t row = j == 0 ? row0 : kv_row(p, it.b, it.kvh, it.t_begin + j * TILE);
      meta[s] = make_int4(idx, j, it.len, it.t_end);
      meta_row[s] = row;
      issue(s, it, j, row);
      if (j == when) during();
    }
  };
  auto first_row = [&](const Item& it) {
    return it.ntiles > 0 ? kv_row(p, it.b, it.kvh, it.t_begin) : int64_t{0};
  };
  const int G = static_cast<int>(gridDim.x);
  const int static_rounds = (p.flags & 4) ? 0 : max(0, p.n_items / G - 2);
  const int n_static = static_rounds * G;
  // static rounds, next item prefetched.  Round r deals items r*G .. r*G+G-1 in snake order
  // (CTA c takes c on even rounds, G-1-c on odd ones), so with longest-first item order no CTA
  // collects the longest item of every round.
  const int c = blockIdx.x;
  auto static_item = [&](int r) { return r * G + ((r & 1) ? G - 1 - c : c); };
  int r = 0;
  int idx = static_item(0);
  if (static_rounds > 0) {
    Item it = make_item(p, idx, TILE);
    int64_t row = first_row(it);
    while (r < static_rounds) {
      const int nidx = static_item(r + 1);
      Item nit{};
      int64_t nrow = 0;
      run_item(idx, it, row, 0, [&] {
        if (r + 1 < static_rounds) {
          nit = make_item(p, nidx, TILE);
          nrow = first_row(nit);
        }
      });
      ++r;
      idx = nidx;
      it = nit;
      row = nrow;
    }
  }
  // dynamic tail: the next item is claimed right after the current item's last tile is
  // issued, so the claim's round trips overlap the tiles still in the ring
  auto claim = [&](int& didx, Item& it, int64_t& row) {
    didx = n_static + atomicAdd(p.work, 1);
    if (didx < p.n_items) {
      it = make_item(p, didx, TILE);
      row = first_row(it);
    }
  };
  int didx;
  Item dit{};
  int64_t drow = 0;
  claim(didx, dit, drow);
  while (didx < p.n_items) {
    int nidx;
    Item nit{};
    int64_t nrow = 0;
    run_item(didx, dit, drow, -1, [&] { claim(nidx, nit, nrow); });
    didx = nidx;
    dit = nit;
    drow = nrow;
  }
  const int s = acquire(i);
  meta[s] = make_int4(-1, 0, 0, 0);
  mbar_arrive(&full[s]);
  // the last producer to leave resets the counters for the next launch
  if (atomicAdd(p.work + 1, 1) == G - 1) {
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

// Epilogue of one work item, run by the CTA's dedicated epilogue warp while the consumer warps
// already stream the next item: merge the warp partials and write the output (single-split
// units) or the split partial (multi-split units, merged by combine_splits_kernel afterwards).  red_m/red_l/red_acc hold the NW per-warp
// partials for GQ q heads: red_m[w*GQ+g] (log2 units if kLog2, else natural), red_l[w*GQ+g],
// red_acc[(w*GQ+g)*D + d].  `nvalid` q heads of the group are real (the MMA kernel pads to 8).
// Returns true when the item wrote a split partial (merged later by combine_splits_kernel).
template <typename T, int D, int GQ, int NW, bool kLog2, class Release>
__device__ __forceinline__ bool finish_item_warp(const DecodeParams& p, const Item& it,
                                                 int nvalid, const float* red_m,
                                                 const float* red_l, const float* red_acc,
                                                 Release release) {
  constexpr float kLn2 = 0.6931471805599453f;
  const int lane = threadIdx.x % 32;
  const int b = it.b;
  const int qh0 = it.kvh * p.G + it.qg * GQ;

  // 1. merge weights of the NW warp partials (fixed warp order => deterministic).
  float wsc[GQ][NW], cta_m[GQ], cta_l[GQ];
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, red_m[w * GQ + g]);
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float mw = red_m[w * GQ + g];
      wsc[g][w] = mw == -INFINITY ? 0.f : (kLog2 ? exp2f(mw - M) : expf(mw - M));
      L += wsc[g][w] * red_l[w * GQ + g];
    }
    cta_m[g] = (M == -INFINITY) ? -INFINITY : (kLog2 ? M * kLn2 : M);  // natural units
    cta_l[g] = L;
  }
  auto merged_acc = [&](int g, int d) {
    float A = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) A = fmaf(wsc[g][w], red_acc[(w * GQ + g) * D + d], A);
    return A;
  };

  const int S_live = live_splits(p, it.len);
  if (S_live == 1) {
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
      if (g >= nvalid) break;
      const int64_t o = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * D;
      for (int d = lane; d < D; d += 32) {
        const float L = cta_l[g];
        store_out<T>(p, o + d, L > 0.f ? merged_acc(g, d) / L : 0.f);
      }
      if (lane == 0 && p.lse != nullptr)
        p.lse[static_cast<int64_t>(b) * p.Hq + qh0 + g] =
            cta_l[g] > 0.f ? cta_m[g] + logf(cta_l[g]) : -INFINITY;
    }
    release();
    return false;
  }

  // 2. write this split's partial, then count it in.
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    if (g >= nvalid) break;
    const int64_t row = (static_cast<int64_t>(b) * p.Hq + qh0 + g) * p.S + it.split;
    for (int d = lane; d < D; d += 32) p.ws_acc[row * D + d] = merged_acc(g, d);
    if (lane == 0) {
      p.ws_ml[row * 2 + 0] = cta_m[g];
      p.ws_ml[row * 2 + 1] = cta_l[g];
    }
  }
  release();
  return true;
}

// Hand-off of per-warp partials from the consumer warps to the epilogue warp.  Single
// red buffer: red_full (count NW) fills it, red_empty (count 1) frees it.  Item index k
// counts hand-offs; the sentinel hand-off carries item -1.
struct RedPipe {
  uint64_t* full;
  uint64_t* empty;
  int* item;  // smem: {item index, request length, item end token} of the buffered partials
};

// Consumer side, per warp: wait until the epilogue warp released the buffer (k > 0).
__device__ __forceinline__ void red_acquire(const RedPipe& r, int k) {
  if (k > 0) mbar_wait(r.empty, (k - 1) & 1);
}
__device__ __forceinline__ void red_commit(const RedPipe& r) {
  __syncwarp();
  if (threadIdx.x % 32 == 0) mbar_arrive(r.full);
}

// Split-K merge, launched after a decode kernel whenever S > 1: one CTA of D threads per
// (request, q head) merges the live split partials in split order — the reference's merge with
// its identity early-out (attention.cpp:100-118) — and finalizes (attention.cpp:120-127).
// Measured on B200 this beats merging inside the persistent kernel (a last-arriver merge with
// GPU-scope fences and atomics) at every split count: C3 S=4 6386 vs 5955 GB/s, S=8 6126 vs 3436.
template <typename T>
__global__ void combine_splits_kernel(const DecodeParams p) {
  const int bh = blockIdx.x;  // b * Hq + h
  const int b = bh / p.Hq;
  const int d = threadIdx.x;
  const int len = __ldg(p.seq_lens + b);
  const int S_live = live_splits(p, len);
  const int64_t row0 = static_cast<int64_t>(bh) * p.S;
  const int64_t o = static_cast<int64_t>(bh) * p.D + d;
  if (len <= 0) {
    store_out<T>(p, o, 0.f);
    if (d == 0 && p.lse != nullptr) p.lse[bh] = -INFINITY;
    return;
  }
  if (S_live == 1) return;  // written directly by the decode kernel
  float M = -INFINITY;
  for (int s = 0; s < S_live; ++s) M = fmaxf(M, __ldg(p.ws_ml + (row0 + s) * 2));
  float A = 0.f, L = 0.f;
  for (int s = 0; s < S_live; ++s) {
    const float ms = __ldg(p.ws_ml + (row0 + s) * 2);
    if (ms == -INFINITY) continue;
    const float w = expf(ms - M);
    L += w * __ldg(p.ws_ml + (row0 + s) * 2 + 1);
    A += w * __ldg(p.ws_acc + (row0 + s) * p.D + d);
  }
  store_out<T>(p, o, L > 0.f ? A / L : 0.f);
  if (d == 0 && p.lse != nullptr) p.lse[bh] = L > 0.f ? M + logf(L) : -INFINITY;
}

// Epilogue warp main loop.
template <typename T, int D, int GQ, int NW, bool kLog2, int TILE>
__device__ __forceinline__ void epilogue_loop(const DecodeParams& p, const RedPipe& r,
                                              int nvalid, const float* red_m,
                                              const float* red_l, const float* red_acc) {
  for (int k = 0;; ++k) {
    mbar_wait(r.full, k & 1);
    const int idx = r.item[0], len = r.item[1], t_end = r.item[2];
    if (idx < 0) break;
    const Item it = item_from_tag<TILE>(p, make_int4(idx, 0, len, t_end));
    finish_item_warp<T, D, GQ, NW, kLog2>(p, it, nvalid, red_m, red_l, red_acc, [&] {
      __syncwarp();
      if (threadIdx.x % 32 == 0) mbar_arrive(r.empty);
    });
  }
}

}  // namespace lam
