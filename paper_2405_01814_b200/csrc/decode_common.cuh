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

#ifndef LAM_MAX_PEERS
#define LAM_MAX_PEERS 8
#endif

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
  int32_t* counters;        // [B*Hkv*QG] split arrival counters (self-resetting)
  // Launch slot (one of a small ring, so overlapping launches never share state): slot[0]
  // counts item claims, slot[1] finished epilogues, both monotonic.  This launch owns claims
  // [item_base, item_base + max(n_items, grid)) and arrivals [done_base, done_base + grid); it
  // starts only once the slot's previous launch has fully finished (slot[1] >= done_base).
  unsigned long long* slot;
  unsigned long long item_base, done_base;
  int32_t pdl;              // launched with programmatic dependent launch
  int32_t defer_inputs;     // KV tiles of the first item may stream before the inputs are
                            // ready; q / k_new / v_new loads wait for them: 1 = the preceding
                            // grid (overlap_prev), 2 = the peer sequence numbers (wait_flag)
  int32_t B, Hq, Hkv, G, D;
  int32_t page_size, pt_stride;
  int32_t chunk;            // tokens per split (multiple of the kernel tile)
  int32_t S;                // number of splits of a split unit
  int32_t u_head;           // leading units run whole (split tail: see item_unit)
  int32_t QG;               // q-head groups per kv head (G / heads per CTA)
  int32_t n_items;          // u_head + (B * Hkv * QG - u_head) * S
  float scale;              // softmax scale (natural units)
  float scale_log2;         // scale * log2(e)
  int32_t out_f32;
  int32_t flags;            // diagnostics: bit 4 = consumers skip the math (streaming only),
                            // bit 5 = the epilogue warp skips its work, bit 6 = the last split
                            // skips the merge (single launches only: outputs are not written)
  // fused append (optional): the new token of request b (position seq_lens[b] - 1) comes from
  // k_new/v_new (request b, kv head h at + b * new_stride + h * D); the kernel attends over it
  // from shared memory and writes it into the pools for later steps.
  const void* k_new;
  const void* v_new;
  int64_t new_stride;
  void* k_pool_w;
  void* v_pool_w;
  const int32_t* order;     // optional request permutation for item enumeration (LPT)
  // peer I/O (optional, src_rows > 0): rows come in groups of src_rows per source rank s; row
  // b = s * src_rows + i reads q at q_src[s] + i * q_stride, the new k/v rows at
  // q_src[s] + new_off[0|1] + i * new_stride, and writes its output rows [Hq][D] to
  // out_dst[s] + i * Hq * D — buffers owned by the model worker s, mapped over NVLink.
  int32_t src_rows;
  // optional row map (lam_peer_io::row_src): row b of the launch (over every micro-batch of a
  // step launch) is row row_src[b] & 0xFFFFFF of source row_src[b] >> 24
  const int32_t* row_src;
  const void* q_src[LAM_MAX_PEERS];
  void* out_dst[LAM_MAX_PEERS];
  int64_t new_off[2];
  // device-side sequence numbers (optional): the producer of every CTA waits until each
  // wait_flag[i] >= wait_value before its first load; the last CTA to finish its epilogue
  // stores done_value to every done_flag[i] after all CTAs' output stores (system scope).
  int32_t n_wait, n_done;
  uint32_t wait_value, done_value;
  const uint32_t* wait_flag[LAM_MAX_PEERS];
  uint32_t* done_flag[LAM_MAX_PEERS];
  // eager q (optional): wait_flag announces q alone, kv_wait_flag the new K / V rows, awaited
  // only before the first tile that holds a new token
  int32_t n_wait_kv;
  uint32_t kv_wait_value;
  const uint32_t* kv_wait_flag[LAM_MAX_PEERS];
  // forwarding model worker (lam_peer_io::n_relay, step launches)
  int32_t n_relay;
  uint32_t* relay_flag;
  const uint32_t* relay_wait_flag[LAM_MAX_PEERS];
  // bounded spins (see spin_expired): status word of the context and the timeout (0 = none)
  int32_t* status;
  unsigned long long spin_timeout_ns;
  // Step launch (lam_decode_step*): the items of n_lm = layers x micro-batches launches, layer
  // major, in one persistent grid.  Launch lm = layer * n_mb + mb owns attention rows
  // [mb * mb_rows, (mb + 1) * mb_rows) of page_table / seq_lens / order (order holds local
  // indices), pool rows offset by layer * layer_rows, and inputs / outputs offset by
  // lm * lm_q_stride / lm * lm_out_stride elements.  Its input sequence numbers (wait flags +
  // mb * flag_mb_stride) are awaited when a CTA first claims one of its items, and once all of
  // its units are finished (lm_done) its done flags are published; both carry epoch + layer + 1.
  // A single launch is n_lm = n_mb = 1, mb_rows = B, items_per_lm = n_items.
  int32_t n_lm, n_mb, mb_rows, items_per_lm, units_per_lm;
  int32_t pool_layers, layer0;  // pool layer of layer l: (layer0 + l) % pool_layers
  int64_t layer_rows, lm_q_stride, lm_new_stride, lm_out_stride;
  int32_t flag_mb_stride;
  uint32_t epoch;
  int32_t* lm_done;
  unsigned long long* trace;  // lam_step_layout::trace (diagnostic stamps) or null
};

// lam_ctx_status codes (include/lamina_attn.h)
constexpr int kStatusInputTimeout = 1;  // input sequence numbers never arrived
constexpr int kStatusSlotTimeout = 2;   // the launch slot's previous launch never finished

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int32_t ld_acquire_gpu_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_s32(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// A spin that has seen no progress for p.spin_timeout_ns (0 = wait forever) gives up: it records
// `code` in the context's status word (lam_ctx_status) and returns false.  The launch then
// completes normally — its outputs are unspecified and its done flags are still published, so
// no waiter on another GPU hangs — instead of trapping, which would leave a sticky error in the
// CUDA context of every attention worker.
__device__ __forceinline__ bool spin_expired(const DecodeParams& p, unsigned long long t0, int code) {
  if (p.spin_timeout_ns == 0 || globaltimer_ns() - t0 < p.spin_timeout_ns) return false;
  if (p.status != nullptr) atomicCAS(p.status, 0, code);
  return true;
}

// Wait until the previous launch on this slot has finished (normally long done).
__device__ __forceinline__ void acquire_slot(const DecodeParams& p) {
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_gpu_u64(p.slot + 1) < p.done_base) {
    __nanosleep(100);
    if (spin_expired(p, t0, kStatusSlotTimeout)) return;
  }
}

// lam_step_layout::trace: after the 4 * n_lm launch stamps, kTraceRecords claim records of
// 3 words per CTA for the first kTraceCtas CTAs
constexpr int kTraceCtas = 1024;
constexpr int kTraceRecords = 400;

// Spin until the inputs of this launch (of launch lm of a step launch) are published.
__device__ __forceinline__ void wait_inputs(const DecodeParams& p, int lm = -1) {
  if (p.n_wait <= 0) return;
  const unsigned long long t0 = globaltimer_ns();
  const int mb = lm >= 0 ? lm % p.n_mb : 0;
  const uint32_t value = lm >= 0 ? p.epoch + static_cast<uint32_t>(lm / p.n_mb) + 1u : p.wait_value;
  const int64_t moff = static_cast<int64_t>(mb) * p.flag_mb_stride;
  // forwarding model worker: this rank's inputs of layer l follow once every attention worker
  // published layer l - 1 of the micro-batch (idempotent: any waiting CTA may forward)
  bool relay = p.n_relay > 0 && lm >= p.n_mb;
  for (int i = 0; i < p.n_wait; ++i) {
    const uint32_t* f = p.wait_flag[i] + moff;
    while (static_cast<int32_t>(ld_acquire_sys(f) - value) < 0) {
      if (relay) {
        bool ready = static_cast<int32_t>(ld_acquire_sys(p.relay_flag + moff) - value) >= 0;
        if (!ready) {
          ready = true;
          for (int r = 0; r < p.n_relay && ready; ++r)
            ready = static_cast<int32_t>(ld_acquire_sys(p.relay_wait_flag[r] + moff) - (value - 1u)) >= 0;
          if (ready) st_release_sys(p.relay_flag + moff, value);
        }
        if (ready) {
          relay = false;
          continue;
        }
      }
      __nanosleep(200);
      if (spin_expired(p, t0, kStatusInputTimeout)) {
        i = p.n_wait;
        break;
      }
    }
  }
  if (p.trace != nullptr && lm >= 0) {
    atomicMin(p.trace + 4 * lm, t0);
    atomicMin(p.trace + 4 * lm + 1, globaltimer_ns());
  }
  fence_proxy_async_global();
}

// Eager q: spin until the new K / V rows of launch lm (-1: of this launch) are published.
__device__ __forceinline__ void wait_new_rows(const DecodeParams& p, int lm) {
  const unsigned long long t0 = globaltimer_ns();
  const int mb = lm >= 0 ? lm % p.n_mb : 0;
  const uint32_t value =
      lm >= 0 ? p.epoch + static_cast<uint32_t>(lm / p.n_mb) + 1u : p.kv_wait_value;
  for (int i = 0; i < p.n_wait_kv; ++i) {
    const uint32_t* f = p.kv_wait_flag[i] + static_cast<int64_t>(mb) * p.flag_mb_stride;
    while (static_cast<int32_t>(ld_acquire_sys(f) - value) < 0) {
      __nanosleep(100);
      if (spin_expired(p, t0, kStatusInputTimeout)) {
        i = p.n_wait_kv;
        break;
      }
    }
  }
  fence_proxy_async_global();
}

// Called by every CTA's epilogue warp after its last output / workspace store: count the CTA
// out of the slot; the last CTA publishes the outputs (peer transport).
__device__ __forceinline__ void finish_cta(const DecodeParams& p) {
  __syncwarp();
  if (threadIdx.x % 32 != 0) return;
  if (p.n_done > 0)
    __threadfence_system();
  else
    __threadfence();
  const unsigned long long old = atomicAdd(p.slot + 1, 1ull);
  if (p.n_done <= 0 || p.n_lm > 1 || old - p.done_base != gridDim.x - 1) return;
  fence_acq_rel_sys();
  for (int i = 0; i < p.n_done; ++i) st_relaxed_sys(p.done_flag[i], p.done_value);
}

// Physical row of token t of (request b, kv head h) of launch lm in a pool viewed as [rows][D].
// Paged: pool[page][Hkv][P][D]; dense: pool[B][Hkv][P][D] (P = row capacity); step launches add
// the layer's offset.
__device__ __forceinline__ int64_t kv_row(const DecodeParams& p, int b, int h, int t, int lm = 0) {
  const int64_t blk =
      p.page_table ? static_cast<int64_t>(__ldg(p.page_table + static_cast<int64_t>(b) * p.pt_stride +
                                                t / p.page_size))
                   : static_cast<int64_t>(b);
  return (blk * p.Hkv + h) * p.page_size + (t % p.page_size) +
         (p.n_lm > 1 ? static_cast<int64_t>((p.layer0 + lm / p.n_mb) % p.pool_layers) * p.layer_rows
                     : 0);
}

enum IssueMode { kIssueAll = 0, kIssueKV = 1, kIssueInputs = 2 };

struct Item {
  int b, kvh, qg, split;  // b: the attention row (over every micro-batch of a step launch)
  int len, t_begin, t_end, ntiles;
  int whole;  // the item is a whole unit (no split partial, no merge)
  int lm;     // launch of a step launch (layer * n_mb + micro-batch); 0 otherwise
};

// Peer I/O: source rank and row within that source's block of attention row it.b.
__device__ __forceinline__ int src_row(const DecodeParams& p, const Item& it, int& row) {
  if (p.row_src != nullptr) {
    const int v = __ldg(p.row_src + it.b);
    row = v & 0xFFFFFF;
    return v >> 24;
  }
  const int b = it.b - (it.lm % p.n_mb) * p.mb_rows;  // row within the launch
  const int s = b / p.src_rows;
  row = b - s * p.src_rows;
  return s;
}

// Start of request it.b's q rows / new k (which = 0) or v (1) rows, local or on a peer.
template <typename T>
__device__ __forceinline__ const T* q_rows(const DecodeParams& p, const Item& it) {
  const int b = it.b - (it.lm % p.n_mb) * p.mb_rows;  // row within the launch
  const int64_t lm_off = static_cast<int64_t>(it.lm) * p.lm_q_stride;
  if (p.src_rows > 0) {
    int i;
    const int s = src_row(p, it, i);
    return static_cast<const T*>(p.q_src[s]) + lm_off + static_cast<int64_t>(i) * p.q_stride;
  }
  return static_cast<const T*>(p.q) + lm_off + static_cast<int64_t>(b) * p.q_stride;
}
template <typename T>
__device__ __forceinline__ const T* new_rows(const DecodeParams& p, int which, const Item& it) {
  const int b = it.b - (it.lm % p.n_mb) * p.mb_rows;
  if (p.src_rows > 0) {  // (the new rows sit in the packed q block)
    const int64_t lm_off = static_cast<int64_t>(it.lm) * p.lm_q_stride;
    int i;
    const int s = src_row(p, it, i);
    return static_cast<const T*>(p.q_src[s]) + lm_off + p.new_off[which] +
           static_cast<int64_t>(i) * p.new_stride;
  }
  return static_cast<const T*>(which ? p.v_new : p.k_new) +
         static_cast<int64_t>(it.lm) * p.lm_new_stride + static_cast<int64_t>(b) * p.new_stride;
}

// Work item `idx` -> (unit, split).  The first u_head items are whole units; the remaining
// units are split S ways, split fastest (a split tail: the last rounds of a launch run short
// items, so the CTAs finish together).  u_head = 0 is a uniform S-way split.
__device__ __forceinline__ void item_unit(const DecodeParams& p, int idx, int& unit, int& split,
                                          int& whole) {
  if (idx < p.u_head) {
    unit = idx;
    split = 0;
    whole = 1;
  } else {
    const int j = idx - p.u_head;
    unit = p.u_head + j / p.S;
    split = j % p.S;
    whole = p.S == 1;
  }
}

// Unit of launch lm -> (request, kv head, q group): q-head group fastest, then kv head, request.
__device__ __forceinline__ void unit_coords(const DecodeParams& p, int unit, Item& it) {
  it.qg = unit % p.QG;
  unit /= p.QG;
  it.kvh = unit % p.Hkv;
  const int r0 = (it.lm % p.n_mb) * p.mb_rows;
  int b = unit / p.Hkv;
  if (p.order != nullptr) b = __ldg(p.order + r0 + b);
  it.b = r0 + b;
}

// Item index (over the whole launch) -> launch lm and the unit / split within it.
__device__ __forceinline__ void item_lm(const DecodeParams& p, int idx, int& lm, int& local) {
  lm = p.n_lm > 1 ? idx / p.items_per_lm : 0;
  local = idx - lm * p.items_per_lm;
}

__device__ __forceinline__ Item make_item(const DecodeParams& p, int idx, int tile) {
  Item it;
  int unit, local;
  item_lm(p, idx, it.lm, local);
  item_unit(p, local, unit, it.split, it.whole);
  unit_coords(p, unit, it);
  it.len = __ldg(p.seq_lens + it.b);
  it.t_begin = it.whole ? 0 : it.split * p.chunk;
  it.t_end = min(it.len, it.whole ? p.S * p.chunk : it.t_begin + p.chunk);
  it.ntiles = it.t_end > it.t_begin ? (it.t_end - it.t_begin + tile - 1) / tile : 0;
  return it;
}

// Item fields from a stage tag {idx, tile, len, t_end} without touching global memory
// (consumers must never stall on a load at an item boundary).
template <int TILE>
__device__ __forceinline__ Item item_from_tag(const DecodeParams& p, int4 tag) {
  Item it;
  int unit, local;
  item_lm(p, tag.x, it.lm, local);
  item_unit(p, local, unit, it.split, it.whole);
  unit_coords(p, unit, it);
  it.len = tag.z;
  it.t_begin = it.whole ? 0 : it.split * p.chunk;
  it.t_end = tag.w;
  it.ntiles = it.t_end > it.t_begin ? (it.t_end - it.t_begin + TILE - 1) / TILE : 0;
  return it;
}

// Does tile j of this item hold the request's new token (fused append)?
template <int TILE>
__device__ __forceinline__ bool tile_has_new(const DecodeParams& p, const Item& it, int j) {
  return p.k_new != nullptr && it.t_end == it.len && it.len > 0 && j == it.ntiles - 1;
}

// Splits of the item's unit that carry tokens (>= 1: an empty request still produces its zero
// output through split 0).
__device__ __forceinline__ int live_splits(const DecodeParams& p, const Item& it) {
  if (it.whole) return 1;
  return it.len > 0 ? min(p.S, (it.len + p.chunk - 1) / p.chunk) : 1;
}

// ---- persistent producer ---------------------------------------------------------------
// meta[s] = {item, tile index, request length, item end token}; item < 0 ends the work.
// meta_row[s] = first pool row of the stage's tile (consumers write the fused new token there).
// A tile is NSUB chunks of TILE / NSUB tokens, each contiguous in the pool (a chunk never
// crosses a page); the chunks' first pool rows are looked up together (independent loads).
// `issue(s, it, j, rows, mode)` must arrive on full[s] with expect_tx for all of the stage's
// bytes and start the stage's TMA copies of tile j, whose chunk c starts at pool row rows[c]
// (chunks past the item end are not loaded; rows[c] = -1): mode
// kIssueAll = every copy, kIssueKV = the K/V tile only, kIssueInputs = only the copies of
// request inputs (q rows, fused new K/V rows) of a stage issued before with kIssueKV.
//
// Deferred inputs (p.defer_inputs, programmatic dependent launch): the KV cache does not depend
// on the stream's preceding kernel but q / k_new / v_new may, so the producer streams the first
// item's KV tiles into the free ring (at most STAGES of them, without waiting on any stage),
// then waits for the preceding grid (griddepcontrol.wait) and issues the deferred input copies.
// The consumers cannot finish a stage before its inputs land, so the producer must not need a
// recycled stage before that: the prefetch stops at the ring size or the end of the item.
//
// Items are claimed from a global counter right after the previous item's tiles are issued.
// Measured on B200 this dynamic schedule beats a static round-robin split by 2-3 % (per-SM
// streaming rates differ across the two dies) and beats claiming one item ahead (that costs up
// to one item of tail imbalance); the stage ring covers the claim's round trips.
// META = meta slots (a multiple of STAGES; tile i's tag lives in meta[i % META]): more slots than
// stages keep a tile's tag readable after its stage has been handed back for the next load.
template <int STAGES, int TILE, int NSUB = 1, int META = STAGES, class Issue>
__device__ __forceinline__ void producer_loop(const DecodeParams& p, uint64_t* full,
                                              uint64_t* empty, int4* meta, long long* meta_row,
                                              Issue issue) {
  // The first min(grid, n_items) items go to CTAs 0, 1, ... without a claim (one global round
  // trip less before a launch's first loads); the counter hands out the rest, offset by them.
  // Claims on the counter per launch: max(n_items, grid) (capi.cu's item_base accounting).
  // Without input sequence numbers the static item's bounds (seq_lens) are read while the
  // slot is acquired: the two loads overlap.
  const int n_static = min(static_cast<int>(gridDim.x), p.n_items);
  const bool pre = p.n_wait == 0 && static_cast<int>(blockIdx.x) < n_static;
  Item it_pre{};
  if (pre) it_pre = make_item(p, static_cast<int>(blockIdx.x), TILE);
  acquire_slot(p);
  // peer transport: the inputs' sequence numbers are awaited like the preceding grid of an
  // overlap_prev launch — after the first KV tiles are in flight (p.defer_inputs = 2)
  auto inputs_ready = [&] {
    if (p.defer_inputs == 2)
      wait_inputs(p);
    else
      griddep_wait();
  };
  const bool step = p.n_lm > 1;  // inputs are awaited per launch lm, at its first claim
  if (p.defer_inputs != 2 && !step) wait_inputs(p);
  int waited_lm = -1;
  int kv_lm = p.n_wait_kv > 0 ? -2 : 0x7fffffff;  // eager q: the last launch whose new rows landed
  int i = 0;
  auto acquire = [&](int k) {
    const int s = k % STAGES;
    if (k >= STAGES) mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
    return s;
  };
  bool deferring = p.defer_inputs != 0;  // first item: KV now, inputs after griddep_wait
  // diagnostic claim records (lam_step_layout::trace): [claim time, inputs seen, item index]
  unsigned long long* rec = p.trace != nullptr && blockIdx.x < kTraceCtas
                                ? p.trace + 4 * p.n_lm + 3ull * kTraceRecords * blockIdx.x
                                : nullptr;
  int n_rec = 0;
  // (Claiming the next item ahead, ~512 tokens before the boundary, at once or one dependent
  // access per issued tile, measured 3-4% slower on B200: round 2, calls 50 and 53.)
  bool first_claim = true;
  for (;;) {
    const unsigned long long t_claim = rec != nullptr ? globaltimer_ns() : 0ull;
    const bool is_static = first_claim && static_cast<int>(blockIdx.x) < n_static;
    const long long claim =
        is_static ? static_cast<long long>(blockIdx.x)
                  : static_cast<long long>(atomicAdd(p.slot, 1ull) - p.item_base) + n_static;
    first_claim = false;
    if (claim >= p.n_items) break;
    const Item it = is_static && pre ? it_pre : make_item(p, static_cast<int>(claim), TILE);
    const int idx = static_cast<int>(claim);
    if (step && it.lm != waited_lm) {  // (claims arrive in launch order: lm only grows)
      wait_inputs(p, it.lm);
      waited_lm = it.lm;
    }
    if (rec != nullptr && n_rec < kTraceRecords) {
      rec[3 * n_rec] = t_claim;
      rec[3 * n_rec + 1] = globaltimer_ns();
      rec[3 * n_rec + 2] = static_cast<unsigned long long>(idx);
      ++n_rec;
    }
    if (it.ntiles == 0) {
      if (deferring) {  // nothing to prefetch
        inputs_ready();
        deferring = false;
      }
      if (it.split == 0 && it.len == 0) {  // empty request: zero-output marker
        const int ms = i % META;
        const int s = acquire(i++);
        meta[ms] = make_int4(idx, 0, 0, 0);
        mbar_arrive(&full[s]);
      }                                    // (an empty split has nothing to merge)
      continue;
    }
    const int i0 = i;  // first stage index of this item
    // Pool rows of the item's chunks.  The page-table entries are loaded four at a time
    // (independent loads: one L2 latency per four pages instead of a dependent load per tile),
    // and a tile's rows are looked up before its stage is acquired, so the lookup overlaps
    // the wait for a free stage.
    const int32_t* ptrow =
        p.page_table ? p.page_table + static_cast<int64_t>(it.b) * p.pt_stride : nullptr;
    const int64_t blk_rows = static_cast<int64_t>(p.Hkv) * p.page_size;
    const int64_t head_off =
        static_cast<int64_t>(it.kvh) * p.page_size +
        (p.n_lm > 1 ? static_cast<int64_t>((p.layer0 + it.lm / p.n_mb) % p.pool_layers) * p.layer_rows
                    : 0);
    int pg_first = -8;
    int32_t pg0 = 0, pg1 = 0, pg2 = 0, pg3 = 0;
    auto row_of = [&](int t) -> long long {
      const int idx = t / p.page_size;
      int64_t blk = it.b;
      if (ptrow != nullptr) {
        if (idx < pg_first || idx >= pg_first + 4) {
          pg_first = idx;
          pg0 = __ldg(ptrow + idx);
          pg1 = idx + 1 < p.pt_stride ? __ldg(ptrow + idx + 1) : 0;
          pg2 = idx + 2 < p.pt_stride ? __ldg(ptrow + idx + 2) : 0;
          pg3 = idx + 3 < p.pt_stride ? __ldg(ptrow + idx + 3) : 0;
        }
        const int o = idx - pg_first;
        blk = o == 0 ? pg0 : o == 1 ? pg1 : o == 2 ? pg2 : pg3;
      }
      return blk * blk_rows + head_off + t % p.page_size;
    };
    for (int j = 0; j < it.ntiles; ++j) {
      if (deferring && i >= STAGES) {  // ring full: the inputs must land before any reuse
        inputs_ready();
        for (int jj = 0; jj < j; ++jj)
          issue((i0 + jj) % STAGES, it, jj, &meta_row[(i0 + jj) % META], kIssueInputs);
        deferring = false;
      }
      long long rows[NSUB];
#pragma unroll
      for (int c = 0; c < NSUB; ++c) {
        const int t = it.t_begin + j * TILE + c * (TILE / NSUB);
        rows[c] = (c == 0 || t < it.t_end) ? row_of(t) : -1;
      }
      // eager q: the tile that holds the new token needs the new K / V rows
      const int want_lm = step ? it.lm : -1;
      if (kv_lm != 0x7fffffff && kv_lm < want_lm + 1 && tile_has_new<TILE>(p, it, j)) {
        wait_new_rows(p, want_lm);
        kv_lm = want_lm + 1;
      }
      const int ms = i % META;
      const int s = acquire(i++);
      meta[ms] = make_int4(idx, j, it.len, it.t_end);
      meta_row[ms] = rows[0];
      issue(s, it, j, static_cast<const long long*>(rows), deferring ? kIssueKV : kIssueAll);
    }
    if (deferring) {  // the whole (short) first item is in the ring
      inputs_ready();
      for (int jj = 0; jj < it.ntiles; ++jj)
        issue((i0 + jj) % STAGES, it, jj, &meta_row[(i0 + jj) % META], kIssueInputs);
      deferring = false;
    }
  }
  if (deferring) inputs_ready();  // no work: still order the launch after its inputs
  const int s = acquire(i);
  meta[i % META] = make_int4(-1, 0, 0, 0);
  mbar_arrive(&full[s]);
  // out of work: the next launch of the stream (programmatic dependent launch) may take this
  // SM as soon as this CTA drains
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// N contiguous floats (N = 2 or 4, 8- or 16-byte aligned) from shared / global memory.
template <int N>
__device__ __forceinline__ void ld_vec(const float* src, float (&v)[N]) {
  static_assert(N == 2 || N == 4, "vector width");
  if constexpr (N == 4) {
    const float4 x = *reinterpret_cast<const float4*>(src);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
    const float2 x = *reinterpret_cast<const float2*>(src);
    v[0] = x.x; v[1] = x.y;
  }
}
template <int N>
__device__ __forceinline__ void ldcg_vec(const float* src, float (&v)[N]) {  // L2, not L1
  if constexpr (N == 4) {
    const float4 x = __ldcg(reinterpret_cast<const float4*>(src));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
    const float2 x = __ldcg(reinterpret_cast<const float2*>(src));
    v[0] = x.x; v[1] = x.y;
  }
}
template <int N>
__device__ __forceinline__ void st_vec(float* dst, const float (&v)[N]) {
  if constexpr (N == 4)
    *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
  else
    *reinterpret_cast<float2*>(dst) = make_float2(v[0], v[1]);
}

// Elements [d, d + N) of the output of (request b, q head h), local or in the source rank's
// buffer (peer transport); fp32 or the KV type.
template <typename T, int D, int N>
__device__ __forceinline__ void store_out_vec(const DecodeParams& p, const Item& it, int h, int d,
                                              const float (&v)[N]) {
  void* base = p.out;
  int b = it.b - (it.lm % p.n_mb) * p.mb_rows;
  if (p.src_rows > 0) {
    const int s = src_row(p, it, b);
    base = p.out_dst[s];
  }
  const int64_t idx = static_cast<int64_t>(it.lm) * p.lm_out_stride +
                      (static_cast<int64_t>(b) * p.Hq + h) * D + d;
  if (sizeof(T) == 4 || p.out_f32) {
    st_vec<N>(static_cast<float*>(base) + idx, v);
  } else if constexpr (sizeof(T) == 2) {
    T* dst = static_cast<T*>(base) + idx;
    if constexpr (N == 4)
      *reinterpret_cast<uint2*>(dst) =
          make_uint2(Elem<T>::pack2(v[0], v[1]), Elem<T>::pack2(v[2], v[3]));
    else
      *reinterpret_cast<uint32_t*>(dst) = Elem<T>::pack2(v[0], v[1]);
  }
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int32_t* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
               : "memory");
  return old;
}

// A unit's outputs are all stored (step launches): count it in for its launch lm; the last unit
// publishes lm's done flags (epoch + layer + 1, micro-batch mb's flag of every model worker)
// after a system-scope fence, so a model worker that sees the number also sees the outputs.
// Flags of one micro-batch are published in layer order (lm_done[n_lm + mb] = layers published):
// in a decode step layer l + 1's inputs follow layer l's outputs, so the wait is normally empty,
// but with inputs published ahead a later layer could finish first and must not be announced
// before the earlier one.
__device__ __forceinline__ void unit_done(const DecodeParams& p, const Item& it) {
  if (p.lm_done == nullptr || p.n_done <= 0) return;  // (nothing to publish)
  __syncwarp();
  if (threadIdx.x % 32 != 0) return;
  // this unit's output stores (local or peer) precede its count (release, cumulative over the
  // warp's stores through the warp barrier); the last unit acquires every count and makes the
  // outputs visible system-wide before the flags
  if (atom_add_acq_rel_gpu(p.lm_done + it.lm, 1) != p.units_per_lm - 1) return;
  if (p.trace != nullptr) p.trace[4 * it.lm + 2] = globaltimer_ns();
  const int layer = it.lm / p.n_mb, mb = it.lm % p.n_mb;
  int32_t* published = p.lm_done + p.n_lm + mb;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_gpu_s32(published) < layer) {
    __nanosleep(100);
    if (spin_expired(p, t0, kStatusInputTimeout)) break;
  }
  const uint32_t value = p.epoch + static_cast<uint32_t>(layer) + 1u;
  const int64_t off = static_cast<int64_t>(mb) * p.flag_mb_stride;
  fence_acq_rel_sys();  // every unit's outputs (acquired through the counts) before the flags
  for (int i = 0; i < p.n_done; ++i) st_relaxed_sys(p.done_flag[i] + off, value);
  st_release_gpu_s32(published, layer + 1);
  if (p.trace != nullptr) p.trace[4 * it.lm + 3] = globaltimer_ns();
}

// Split-K epilogue of one work item, run by the CTA's dedicated epilogue warp while the
// consumer warps already stream the next item.  red_m/red_l/red_acc hold the NW per-warp
// partials for GQ q heads: red_m[w*GQ+g] (log2 units if kLog2, else natural), red_l[w*GQ+g],
// red_acc[(w*GQ+g)*RS + d] (row stride RS >= D floats, a multiple of 4).  `nvalid` q heads of
// the group are real (the MMA kernel pads to 8).
//
// Lane l owns the D/32 contiguous dims [l*D/32, (l+1)*D/32) of every head, so the warp
// partials, the split partials and the outputs all move as 8- or 16-byte vectors.  The split
// partial is published with one acq_rel atomic by lane 0 after a warp barrier (no full
// sequentially-consistent fence), and the last split of a unit merges the live partials in
// split order (merge, attention.cpp:100-118, identity early-out: an empty split weighs 0).
template <typename T, int D, int GQ, int NW, bool kLog2, int RS, class Release>
__device__ __forceinline__ void finish_item_warp(const DecodeParams& p, const Item& it,
                                                 int nvalid, const float* red_m,
                                                 const float* red_l, const float* red_acc,
                                                 Release release) {
  constexpr float kLn2 = 0.6931471805599453f;
  constexpr int DPL = D / 32;  // contiguous output dims per lane
  static_assert(RS % 4 == 0 && RS >= D, "partial row stride");
  const int lane = threadIdx.x % 32;
  const int d0 = lane * DPL;
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
  auto merged_acc = [&](int g, float (&A)[DPL]) {
#pragma unroll
    for (int e = 0; e < DPL; ++e) A[e] = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      float x[DPL];
      ld_vec<DPL>(red_acc + (w * GQ + g) * RS + d0, x);
#pragma unroll
      for (int e = 0; e < DPL; ++e) A[e] = fmaf(wsc[g][w], x[e], A[e]);
    }
  };

  const int S_live = live_splits(p, it);
  if (S_live == 1) {
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
      if (g < nvalid) {
        float A[DPL];
        merged_acc(g, A);
        const float L = cta_l[g];
        const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) A[e] *= inv;
        store_out_vec<T, D, DPL>(p, it, qh0 + g, d0, A);
        if (lane == 0 && p.lse != nullptr)
          p.lse[static_cast<int64_t>(b) * p.Hq + qh0 + g] = L > 0.f ? cta_m[g] + logf(L) : -INFINITY;
      }
    }
    release();
    unit_done(p, it);
    return;
  }

  // 2. write this split's partial, then count it in.  (Step launches keep one workspace row
  //    block per layer: bw = row over every layer.)
  const int64_t bw = b + (p.n_lm > 1 ? static_cast<int64_t>(it.lm / p.n_mb) * p.B : 0);
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    if (g < nvalid) {
      const int64_t row = (bw * p.Hq + qh0 + g) * p.S + it.split;
      float A[DPL];
      merged_acc(g, A);
      st_vec<DPL>(p.ws_acc + row * D + d0, A);
      if (lane == 0)
        *reinterpret_cast<float2*>(p.ws_ml + row * 2) = make_float2(cta_m[g], cta_l[g]);
    }
  }
  release();  // the consumers may refill red_* while this warp counts and merges splits
  __syncwarp();  // every lane's partial stores precede lane 0's release
  int32_t* counter = p.counters + (bw * p.Hkv + it.kvh) * p.QG + it.qg;
  int last = 0;
  if (lane == 0) last = (atom_add_acq_rel_gpu(counter, 1) == S_live - 1);
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  if (p.flags & 64) {  // diagnostic: the last split skips the merge (outputs are not written)
    if (lane == 0) *counter = 0;
    return;
  }

  // 3. last split of this unit: merge the live partials in split order and finalize.  Lane s
  //    holds split s's statistics; every live split's slice of a head is loaded before use.
  //    In a streaming SM a dependent global load waits behind the TMA data in flight (µs), so
  //    the loads are issued ahead: up to 4 splits, head g + 1's partials are in flight while
  //    head g is merged, and head 0's with the statistics (2 round trips instead of 9 for 8
  //    heads).
  constexpr int kPre = 4;
  float pre[2][kPre][DPL];
  auto load_head = [&](int g, float (&v)[kPre][DPL]) {
    const int64_t row0 = (bw * p.Hq + qh0 + g) * p.S;
#pragma unroll
    for (int j = 0; j < kPre; ++j) {
      if (g < nvalid && j < S_live) {
        ldcg_vec<DPL>(p.ws_acc + (row0 + j) * D + d0, v[j]);
      } else {
#pragma unroll
        for (int e = 0; e < DPL; ++e) v[j][e] = 0.f;
      }
    }
  };
  if (S_live <= kPre) load_head(0, pre[0]);
  float ms[GQ], ls[GQ];
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    ms[g] = -INFINITY;
    ls[g] = 0.f;
    if (g < nvalid && lane < S_live) {
      const float2 ml = __ldcg(reinterpret_cast<const float2*>(
          p.ws_ml + ((bw * p.Hq + qh0 + g) * p.S + lane) * 2));
      ms[g] = ml.x;
      ls[g] = ml.y;
    }
  }
  if (S_live <= kPre) {
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
      if (g + 1 < GQ) load_head(g + 1, pre[(g + 1) & 1]);
      if (g >= nvalid) continue;
      float M = ms[g];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      const float w = ms[g] == -INFINITY ? 0.f : expf(ms[g] - M);  // lanes >= S_live: 0
      float L = w * ls[g];
      float A[DPL];
#pragma unroll
      for (int e = 0; e < DPL; ++e) A[e] = 0.f;
#pragma unroll
      for (int j = 0; j < kPre; ++j) {  // split order, as the general path below
        const float wj = __shfl_sync(0xffffffffu, w, j);
#pragma unroll
        for (int e = 0; e < DPL; ++e) A[e] = fmaf(wj, pre[g & 1][j][e], A[e]);
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
      for (int e = 0; e < DPL; ++e) A[e] *= inv;
      store_out_vec<T, D, DPL>(p, it, qh0 + g, d0, A);
      if (lane == 0 && p.lse != nullptr)
        p.lse[static_cast<int64_t>(b) * p.Hq + qh0 + g] = L > 0.f ? M + logf(L) : -INFINITY;
    }
    if (lane == 0) *counter = 0;  // ready for the next launch
    unit_done(p, it);
    return;
  }
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    if (g >= nvalid) continue;
    const int64_t row0 = (bw * p.Hq + qh0 + g) * p.S;
    float M = ms[g];
    for (int s0 = 32 + lane; s0 < S_live; s0 += 32) M = fmaxf(M, __ldcg(p.ws_ml + (row0 + s0) * 2));
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    // lanes >= S_live hold -inf and weigh nothing
    const float w = ms[g] == -INFINITY ? 0.f : expf(ms[g] - M);
    float L = w * ls[g];
    float A[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) A[e] = 0.f;
    constexpr int kBatch = 8;
    if (S_live <= kBatch) {
      float v[kBatch][DPL];
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        if (j < S_live) {
          ldcg_vec<DPL>(p.ws_acc + (row0 + j) * D + d0, v[j]);
        } else {
#pragma unroll
          for (int e = 0; e < DPL; ++e) v[j][e] = 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        const float wj = __shfl_sync(0xffffffffu, w, j);
#pragma unroll
        for (int e = 0; e < DPL; ++e) A[e] = fmaf(wj, v[j][e], A[e]);
      }
    } else {
      // 9..32 splits: kBatch independent partial loads per L2 round trip, accumulated in split
      // order (an S = 16 unit: 2 round trips per head instead of 16)
      const int n = min(32, S_live);
      for (int j0 = 0; j0 < n; j0 += kBatch) {
        float v[kBatch][DPL];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
          if (j0 + j < n) {
            ldcg_vec<DPL>(p.ws_acc + (row0 + j0 + j) * D + d0, v[j]);
          } else {
#pragma unroll
            for (int e = 0; e < DPL; ++e) v[j][e] = 0.f;
          }
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
          const float wj = __shfl_sync(0xffffffffu, w, (j0 + j) & 31);
          if (j0 + j < n) {
#pragma unroll
            for (int e = 0; e < DPL; ++e) A[e] = fmaf(wj, v[j][e], A[e]);
          }
        }
      }
    }
    for (int s0 = 32; s0 < S_live; s0 += 32) {  // more than 32 splits (rare)
      float w2 = 0.f;
      if (s0 + lane < S_live) {
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml + (row0 + s0 + lane) * 2));
        w2 = ml.x == -INFINITY ? 0.f : expf(ml.x - M);
        L += w2 * ml.y;
      }
      for (int j = 0; j < min(32, S_live - s0); ++j) {
        const float wj = __shfl_sync(0xffffffffu, w2, j);
        float v[DPL];
        ldcg_vec<DPL>(p.ws_acc + (row0 + s0 + j) * D + d0, v);
#pragma unroll
        for (int e = 0; e < DPL; ++e) A[e] = fmaf(wj, v[e], A[e]);
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) A[e] *= inv;
    store_out_vec<T, D, DPL>(p, it, qh0 + g, d0, A);
    if (lane == 0 && p.lse != nullptr)
      p.lse[static_cast<int64_t>(b) * p.Hq + qh0 + g] = L > 0.f ? M + logf(L) : -INFINITY;
  }
  if (lane == 0) *counter = 0;  // ready for the next launch
  unit_done(p, it);
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

// Epilogue warp main loop.
template <typename T, int D, int GQ, int NW, bool kLog2, int TILE, int RS>
__device__ __forceinline__ void epilogue_loop(const DecodeParams& p, const RedPipe& r,
                                              int nvalid, const float* red_m,
                                              const float* red_l, const float* red_acc) {
  for (int k = 0;; ++k) {
    mbar_wait(r.full, k & 1);
    const int idx = r.item[0];
    if (idx < 0) break;
    const Item it = item_from_tag<TILE>(p, make_int4(idx, 0, r.item[1], r.item[2]));
    if (p.flags & 32) {  // diagnostic: no epilogue work (outputs are not written)
      __syncwarp();
      if (threadIdx.x % 32 == 0) mbar_arrive(r.empty);
      continue;
    }
    finish_item_warp<T, D, GQ, NW, kLog2, RS>(p, it, nvalid, red_m, red_l, red_acc, [&] {
      __syncwarp();
      if (threadIdx.x % 32 == 0) mbar_arrive(r.empty);
    });
  }
  finish_cta(p);
}

}  // namespace lam
