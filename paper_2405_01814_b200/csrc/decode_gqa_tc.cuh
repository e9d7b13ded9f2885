// decode_gqa_tc.cuh — split-K GQA decode attention on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in tensor memory).
//
// The contraction is the one of decode_gqa_mma.cuh (attention.cpp:141-162 with the G q heads
// that share a KV head as the N dimension, padded to N = 8):
//   S[128 tok x 8]   = K[128 tok x 128 d] · Q^T[128 d x 8]
//   O^T[128 d x 8]   = V^T[128 d x 128 tok] · P^T[128 tok x 8]  (one fresh accumulator per tile)
// but neither operand passes through the register file: single threads issue tcgen05.mma
// straight from the TMA rings (K K-major, V MN-major, both 128-byte swizzled) and the results
// land in TMEM.  The softmax warpgroup only touches 8 fp32 logits and 8 fp32 output values per
// thread and tile:
//
//   warp 0-3  softmax warpgroup: thread t owns token row t of S (TMEM lane t) and output row
//             d = t of O^T.  Per tile: tcgen05.ld its 8 logits (and hand the S buffer back), the
//             tile max per q head across the warpgroup, the online-softmax update, P (bf16) into
//             shared memory as the O MMA's B operand; then tcgen05.ld the previous tile's O^T row
//             and fold it into the register accumulator with that tile's rescale factor.
//   warp 4    S issuer: stages q (and the fused new K/V row) into the operand layouts and issues
//             S(i) as soon as K(i) has landed and an S buffer is free; the commit hands the K
//             slot back to the producer.
//   warp 7    O issuer: O(j) as soon as P(j) is written; the commit hands the V slot back.
//             (Two issuers, so neither stream of MMAs ever waits behind the other's inputs.)
//   warp 5    TMA producer (decode_common.cuh:producer_loop): 128-token tiles as two 64-row
//             chunks (a page each at page_size 64), K and V into separate rings.
//   warps 6, 8  epilogue (decode_common.cuh:finish_item_warp): output, LSE or split partials
//             and the last split's merge; one warp per hand-off buffer (even / odd items).
//
// S is four-buffered and O^T double-buffered in TMEM (48 of 64 allocated columns), P
// double-buffered in shared memory.  Online softmax semantics are those of the reference's
// partial form (attention.cpp:72-127): running max, exp-weights, the sum taken over the rounded
// weights fed to the MMA.
#pragma once

#include <type_traits>

#include "decode_common.cuh"

namespace lam {

// ---- tcgen05 wrappers -----------------------------------------------------------------

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrive on `bar` once every tcgen05 operation this thread issued before has completed.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] · B[smem], kind::f16 (bf16 / fp16 in, fp32 accumulate).
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 TMEM lanes x 8 consecutive 32-bit columns -> 8 registers per thread (lane = thread of the
// warp, relative to the lane base encoded in taddr).
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  // the registers are valid only after wait::ld: both in one asm statement, so no use of them
  // can be scheduled in between
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor (sm_100 layout): start >> 4 in [0,14), leading byte offset >> 4
// in [16,30), stride byte offset >> 4 in [32,46), version 1 in [46,48), layout type in [61,64)
// (0 = no swizzle, 2 = 128-byte swizzle).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) |
         (static_cast<uint64_t>(layout) << 61);
}

// Instruction descriptor, kind::f16: fp32 accumulator, A/B bf16 (1) or fp16 (0), M, N, majors
// (0 = K-major, 1 = MN-major).
template <typename T>
__host__ __device__ constexpr uint32_t tc_idesc(int M, int N, int a_mn, int b_mn) {
  constexpr uint32_t fmt = std::is_same<T, __half>::value ? 0u : 1u;  // fp16 : bf16
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

template <int KS_, int VS_>
struct TcCfg {
  static constexpr int KS = KS_;  // K slots (128 tokens each), handed back after the S MMA
  static constexpr int VS = VS_;  // V slots, handed back after the O MMA (later)
  static constexpr int NS = 4;    // S buffers in TMEM (and q buffers in shared memory)
  static constexpr int TILE = 128;  // tokens per tile = MMA M of S = MMA K of O
  static constexpr int SUB = 64;    // rows per TMA box (a page chunk)
  static constexpr int D = 128, GQ = 8, NPAD = 8;
  static constexpr int BOX_BYTES = TILE * 128;       // [128 rows][64 cols] 16-bit, swizzled
  static constexpr int MAT_BYTES = 2 * BOX_BYTES;    // one K (or V) tile, 32 KB
  static constexpr int OFF_V = KS * MAT_BYTES;
  static constexpr int QBOX = NPAD * 128;            // q rows as the S MMA's B operand: 2 boxes
  static constexpr int QBUF_BYTES = 2 * QBOX;
  static constexpr int PBUF_BYTES = TILE * 16;       // P rows (8 bf16 per token) per parity
  static constexpr int Q_BYTES = GQ * D * 2;         // an item's q rows as loaded (row-major)
  static constexpr int ROW_BYTES = D * 2;
  static constexpr int SLOT_BYTES = Q_BYTES + 2 * ROW_BYTES;  // + fused new k, v rows
  static constexpr int RS = D + 4;                   // epilogue partial row stride (floats)
  static constexpr int OFF_QBUF = OFF_V + VS * MAT_BYTES;          // [NS]
  static constexpr int OFF_PBUF = OFF_QBUF + NS * QBUF_BYTES;      // [2]
  static constexpr int OFF_SLOT = OFF_PBUF + 2 * PBUF_BYTES;       // [KS]
  static constexpr int OFF_RED = OFF_SLOT + KS * SLOT_BYTES;
  // two hand-off sets {red_m[8], red_l[8], red_lw[4][8], red_acc[8][RS]} (the warpgroup fills
  // one while the epilogue warp still finishes the other), then tmax[2][4][8]
  static constexpr int RED_SET = GQ + GQ + 4 * GQ + GQ * RS;
  static constexpr int RED_FLOATS = 2 * RED_SET + 2 * 4 * GQ;
  static constexpr int OFF_META = OFF_RED + RED_FLOATS * 4;
  static constexpr int META = 16;  // tile tags outlive their K slot (read until the O MMA)
  static constexpr int OFF_BAR = OFF_META + META * 16 + META * 8;
  // fullK, emptyK [KS]; fullV, emptyV [VS]; s, sfree [NS]; p, o, ofree [2]; hand-off full,
  // empty [2]; hand-off tags (2 x 4 ints); TMEM address
  static constexpr int N_BARS = 2 * KS + 2 * VS + 2 * NS + 16;
  static constexpr int SMEM_BYTES = OFF_BAR + N_BARS * 8 + 32 + 1024;  // + align slack
  static constexpr int THREADS = 9 * 32;
  static constexpr int TMEM_COLS = 64;  // S[4] and O[2], 8 columns each
};

template <typename T, int KS_, int VS_>
__global__ void __launch_bounds__(9 * 32, 1)
    decode_gqa_tc_kernel(const DecodeParams p, const __grid_constant__ CUtensorMap kmap,
                         const __grid_constant__ CUtensorMap vmap) {
  using C = TcCfg<KS_, VS_>;
  constexpr int KS = C::KS, VS = C::VS, NS = C::NS, TILE = C::TILE, SUB = C::SUB, D = C::D,
                GQ = C::GQ;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* vring = smem + C::OFF_V;
  uint8_t* qbuf = smem + C::OFF_QBUF;
  uint8_t* pbuf = smem + C::OFF_PBUF;
  uint8_t* qslot = smem + C::OFF_SLOT;
  // hand-off set b: red_m[8], red_l[8], red_lw[4 warps][8], red_acc[8][RS]
  float* const red0 = reinterpret_cast<float*>(smem + C::OFF_RED);
  auto red_m = [&](int b) { return red0 + b * C::RED_SET; };
  auto red_l = [&](int b) { return red0 + b * C::RED_SET + GQ; };
  auto red_lw = [&](int b) { return red0 + b * C::RED_SET + 2 * GQ; };
  auto red_acc = [&](int b) { return red0 + b * C::RED_SET + 6 * GQ; };
  float* tmax = red0 + 2 * C::RED_SET;  // [2][4 warps][8]
  int4* meta = reinterpret_cast<int4*>(smem + C::OFF_META);
  long long* meta_row = reinterpret_cast<long long*>(meta + C::META);
  // The K and V halves of a tile live in separate rings: K is handed back as soon as S has read
  // it, V only after the O MMA.  The K ring follows the tile counter i; the V ring follows the
  // count of data-carrying tiles (an empty request's marker takes a K slot but loads nothing).
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);  // K (+ q, new rows) [KS]
  uint64_t* empty = full + KS;
  uint64_t* fullv = empty + KS;      // [VS]
  uint64_t* emptyv = fullv + VS;
  uint64_t* sbar = emptyv + VS;      // S(i) in TMEM           [NS]
  uint64_t* sfree = sbar + NS;       // S(i) read out          [NS]
  uint64_t* pbar = sfree + NS;       // P(i) in smem           [2]
  uint64_t* obar = pbar + 2;         // O(i) in TMEM           [2]
  uint64_t* ofree = obar + 2;        // O(i) read out          [2]
  uint64_t* rfull = ofree + 2;   // hand-off set b filled      [2]
  uint64_t* rempty = ofree + 4;  // hand-off set b released    [2]
  int* ritem = reinterpret_cast<int*>(ofree + 6);  // [2][4]: {item, len, t_end}
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ofree + 10);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int G = p.G;  // real q heads of the group (<= 8); the MMA's other N rows are zero
  const bool nomath = p.flags & 16;  // diagnostic: no MMAs (the pipeline alone)

  if (threadIdx.x == 0) {
    for (int s = 0; s < KS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);   // tcgen05.commit after the S MMA
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(&fullv[s], 1);
      mbar_init(&emptyv[s], 1);  // tcgen05.commit after the O MMA
    }
    for (int b = 0; b < NS; ++b) {
      mbar_init(&sbar[b], 1);
      mbar_init(&sfree[b], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&pbar[b], 4);
      mbar_init(&obar[b], 1);
      mbar_init(&ofree[b], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&rfull[b], 4);
      mbar_init(&rempty[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 5 && lane == 0) {
    prefetch_tensormap(&kmap);
    prefetch_tensormap(&vmap);
  }
  if (warp == 4) {  // TMEM: S[4], O[2] (the allocating warp also frees it)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // zero the q rows G..7 of every q buffer (the MMA's padding rows)
  for (int i = threadIdx.x; i < NS * C::QBUF_BYTES / 16; i += blockDim.x)
    if ((i * 16 % C::QBOX) / 128 >= G)
      *reinterpret_cast<uint4*>(qbuf + i * 16) = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 5) {  // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int nv = 0;  // V tiles issued (data-carrying tiles so far)
      producer_loop<KS, TILE, 2, C::META>(
          p, full, empty, meta, meta_row,
          [&](int s, const Item& it, int j, const long long* rows, int mode) {
            uint8_t* kt = smem + s * C::MAT_BYTES;
            const uint32_t qb = static_cast<uint32_t>(G) * D * 2;
            const bool fused = tile_has_new<TILE>(p, it, j);
            const bool two = mode != kIssueInputs && rows[1] >= 0;
            if (mode != kIssueInputs)
              mbar_arrive_expect_tx(&full[s], (two ? 2 : 1) * 2 * SUB * 128 + (j == 0 ? qb : 0) +
                                                  (fused ? 2 * C::ROW_BYTES : 0));
            if (mode != kIssueKV && fused) {
              const int64_t off = static_cast<int64_t>(it.kvh) * D;
              uint8_t* kn = qslot + s * C::SLOT_BYTES + C::Q_BYTES;
              tma_load_1d(kn, new_rows<T>(p, 0, it) + off, C::ROW_BYTES, &full[s], pol);
              tma_load_1d(kn + C::ROW_BYTES, new_rows<T>(p, 1, it) + off, C::ROW_BYTES,
                          &full[s], pol);
            }
            if (mode != kIssueKV && j == 0)
              tma_load_1d(qslot + s * C::SLOT_BYTES,
                          q_rows<T>(p, it) + static_cast<int64_t>(it.kvh) * G * D, qb, &full[s],
                          pol);
            if (mode == kIssueInputs) return;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              if (c == 1 && !two) break;
              uint8_t* kd = kt + c * SUB * 128;
              tma_load_2d(kd, &kmap, 0, static_cast<int32_t>(rows[c]), &full[s], pol);
              tma_load_2d(kd + C::BOX_BYTES, &kmap, 64, static_cast<int32_t>(rows[c]), &full[s], pol);
            }
            // V: its slot is free once the O MMA of the tile VS data tiles back has read it
            const int v = nv++, vs = v % VS;
            if (v >= VS) mbar_wait(&emptyv[vs], ((v / VS) - 1) & 1);
            mbar_arrive_expect_tx(&fullv[vs], (two ? 2 : 1) * 2 * SUB * 128);
            uint8_t* vt = vring + vs * C::MAT_BYTES;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              if (c == 1 && !two) break;
              uint8_t* vd = vt + c * SUB * 128;
              tma_load_2d(vd, &vmap, 0, static_cast<int32_t>(rows[c]), &fullv[vs], pol);
              tma_load_2d(vd + C::BOX_BYTES, &vmap, 64, static_cast<int32_t>(rows[c]), &fullv[vs], pol);
            }
          });
    }
    return;
  }
  if (warp == 6 || warp == 8) {  // ---------------- epilogue ----------------
    // two epilogue warps, one per hand-off buffer: warp 6 finishes the even items, warp 8 the
    // odd ones, so each has two items' time for an item's split partial and the last split's
    // merge (L2 round trips that are slow under full HBM load) before its buffer is needed again
    const int b = warp == 6 ? 0 : 1;
    for (int k = 0;; ++k) {
      mbar_wait(&rfull[b], k & 1);
      const int* tg = ritem + 4 * b;
      const int idx = tg[0];
      if (idx < 0) break;
      const Item it = item_from_tag<TILE>(p, make_int4(idx, 0, tg[1], tg[2]));
      const float* lw = red_lw(b);
      if (lane < GQ)  // the four warps' partial sums of the softmax denominator
        red_l(b)[lane] = lw[lane] + lw[GQ + lane] + lw[2 * GQ + lane] + lw[3 * GQ + lane];
      __syncwarp();
      if (p.flags & 32) {  // diagnostic: no epilogue work (outputs are not written)
        if (lane == 0) mbar_arrive(&rempty[b]);
        continue;
      }
      finish_item_warp<T, D, GQ, 1, true, C::RS>(p, it, G, red_m(b), red_l(b), red_acc(b), [&] {
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[b]);
      });
    }
    named_bar_sync(5, 2 * 32);  // both epilogue warps' stores precede the CTA's count
    if (warp == 6) finish_cta(p);
    return;
  }

  constexpr uint32_t IDESC_S = tc_idesc<T>(128, C::NPAD, 0, 0);  // K-major A and B
  constexpr uint32_t IDESC_O = tc_idesc<T>(128, C::NPAD, 1, 1);  // MN-major A and B
  // TMEM columns: S(i % 4) at (i % 4) * 8, O(parity b) at 32 + b * 8
  auto s_tmem = [&](int b) { return tmem + static_cast<uint32_t>(b) * 8; };
  auto o_tmem = [&](int b) { return tmem + 32 + static_cast<uint32_t>(b) * 8; };

  if (warp == 4) {  // ---------------- S issuer ----------------
    const uint32_t kring = smem_u32(smem), qb0 = smem_u32(qbuf);
    Item it{};
    int k_item = -1, nv = 0;  // items started; data tiles so far (the V ring's counter)
    for (int i = 0;; ++i) {
      const int s = i % KS;
      mbar_wait(&full[s], (i / KS) & 1);
      const int4 mt = meta[i % C::META];
      const bool sentinel = mt.x < 0;
      const bool real = !sentinel && mt.z > 0;  // (an empty request's marker carries no data)
      // S(i) reuses the buffer of S(i - NS), which the warpgroup has read out by sfree; the q
      // buffer of item k is that of item k - NS, whose S MMAs completed before (in order)
      if (i >= NS) mbar_wait(&sfree[i % NS], ((i / NS) - 1) & 1);
      if (real) {
        const int v = nv++;
        if (mt.y == 0) {  // new item: its q rows into the S MMA's B layout (K-major, 128B swizzle)
          it = item_from_tag<TILE>(p, mt);
          ++k_item;
          uint8_t* qb = qbuf + (k_item % NS) * C::QBUF_BYTES;
          const uint8_t* src = qslot + s * C::SLOT_BYTES;
          for (int c = lane; c < G * 16; c += 32) {
            const int r = c >> 4, ch = c & 15;
            *reinterpret_cast<uint4*>(qb + (ch >> 3) * C::QBOX + r * 128 + (((ch & 7) ^ (r & 7)) << 4)) =
                *reinterpret_cast<const uint4*>(src + r * C::ROW_BYTES + ch * 16);
          }
        }
        if (tile_has_new<TILE>(p, it, mt.y)) {  // fused append: the new K / V row into the tiles and the pools
          mbar_wait(&fullv[v % VS], (v / VS) & 1);  // the V tile must have landed first
          const int r = it.len - 1 - (it.t_begin + mt.y * TILE);
          const int ch = lane & 15, is_v = lane >> 4;
          const uint4 val = *reinterpret_cast<const uint4*>(qslot + s * C::SLOT_BYTES + C::Q_BYTES +
                                                            is_v * C::ROW_BYTES + ch * 16);
          uint8_t* tile = is_v ? vring + (v % VS) * C::MAT_BYTES : smem + s * C::MAT_BYTES;
          *reinterpret_cast<uint4*>(tile + (ch >> 3) * C::BOX_BYTES + r * 128 +
                                    (((ch & 7) ^ (r & 7)) << 4)) = val;
          T* pool = static_cast<T*>(is_v ? p.v_pool_w : p.k_pool_w);
          *reinterpret_cast<uint4*>(pool + kv_row(p, it.b, it.kvh, it.len - 1, it.lm) * D + ch * 8) = val;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {  // S(i) = K(i) · Q^T
          tc_fence_after();
          if (!nomath) {
            const uint32_t kb = kring + s * C::MAT_BYTES;
            const uint32_t qb = qb0 + (k_item % NS) * C::QBUF_BYTES;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = (kk >> 2) * C::BOX_BYTES + (kk & 3) * 32;
              const uint32_t qoff = (kk >> 2) * C::QBOX + (kk & 3) * 32;
              tc_mma(s_tmem(i % NS), smem_desc(kb + off, 16, 1024, 2),
                     smem_desc(qb + qoff, 16, 1024, 2), IDESC_S, kk > 0);
            }
          }
          tc_commit(&sbar[i % NS]);
          tc_commit(&empty[s]);  // the K slot is free once S has read it
        }
      } else if (lane == 0) {
        mbar_arrive(&sbar[i % NS]);  // marker / end of work: the warpgroup reads the tag
        if (!sentinel) mbar_arrive(&empty[s]);
      }
      __syncwarp();
      if (sentinel) break;
    }
    named_bar_sync(3, 6 * 32);  // the warpgroup and the O issuer are done with TMEM
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(C::TMEM_COLS)
                 : "memory");
    return;
  }
  if (warp == 7) {  // ---------------- O issuer ----------------
    const uint32_t vring_a = smem_u32(vring), pb0 = smem_u32(pbuf);
    int nv = 0;  // data tiles so far (the V ring's counter)
    for (int j = 0;; ++j) {
      mbar_wait(&pbar[j & 1], (j >> 1) & 1);  // P(j) written (the warpgroup also passes the end)
      const int4 mt = meta[j % C::META];
      if (mt.x < 0) break;
      const bool real = mt.z > 0;
      if (j >= 2) mbar_wait(&ofree[j & 1], ((j - 2) >> 1) & 1);
      const int v = nv;
      if (real) {
        ++nv;
        mbar_wait(&fullv[v % VS], (v / VS) & 1);
      }
      if (lane == 0) {
        tc_fence_after();
        if (real) {
          const uint32_t vb = vring_a + (v % VS) * C::MAT_BYTES;
          const uint32_t pb = pb0 + (j & 1) * C::PBUF_BYTES;
          if (!nomath) {
#pragma unroll
            for (int kk = 0; kk < TILE / 16; ++kk)
              tc_mma(o_tmem(j & 1), smem_desc(vb + kk * 16 * 128, C::BOX_BYTES, 1024, 2),
                     smem_desc(pb + kk * 256, 128, 128, 0), IDESC_O, kk > 0);
          }
          tc_commit(&obar[j & 1]);
          tc_commit(&emptyv[v % VS]);
        } else {
          mbar_arrive(&obar[j & 1]);
        }
      }
      __syncwarp();
    }
    named_bar_sync(3, 6 * 32);
    return;
  }
  // ---------------- softmax warpgroup (warps 0-3) ----------------
  const int t = warp * 32 + lane;  // token row of S / dim row of O^T = TMEM lane
  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  const float sl2 = p.scale_log2;
  float m[GQ], l[GQ], o[GQ], a_prev[GQ];  // running max (log2 units), sum, output row
  int4 tag{};                             // {item, len, t_end} of the current item
  Item it{};
  bool pending = false, prev_real = false, prev_first = false;  // O(i-1) not folded yet
  int k_item = 0, bpar = 0;
  int nv = 0;  // data-carrying tiles so far (the V ring's counter)
#pragma unroll
  for (int g = 0; g < GQ; ++g) { m[g] = -INFINITY; l[g] = 0.f; o[g] = 0.f; a_prev[g] = 0.f; }
  // fold O(j) (tile j's output rows, accumulate = with its rescale factor a) into o
  auto fold = [&](int j, bool jreal, bool jfirst, const float (&a)[GQ]) {
    mbar_wait(&obar[j & 1], (j >> 1) & 1);
    tc_fence_after();
    if (jreal) {
      float ot[GQ];
      tmem_ld8(o_tmem(j & 1) + lane_base, ot);
#pragma unroll
      for (int g = 0; g < GQ; ++g) o[g] = jfirst ? ot[g] : fmaf(o[g], a[g], ot[g]);
    } else {
#pragma unroll
      for (int g = 0; g < GQ; ++g) o[g] = 0.f;  // an empty request's zero output
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&ofree[j & 1]);
  };
  for (int i = 0;; ++i) {
    mbar_wait(&sbar[i % NS], (i / NS) & 1);
    tc_fence_after();
    const int4 mt = meta[i % C::META];
    if (mt.x < 0) {  // end of work (every item was handed over at its last tile)
      __syncwarp();
      if (lane == 0) mbar_arrive(&pbar[i & 1]);  // the O issuer reads the end tag, too
      break;
    }
    float a_cur[GQ];
#pragma unroll
    for (int g = 0; g < GQ; ++g) a_cur[g] = 0.f;
    const bool first = mt.y == 0;
    if (first) {
      it = item_from_tag<TILE>(p, mt);
      tag = make_int4(mt.x, mt.z, mt.w, 0);
#pragma unroll
      for (int g = 0; g < GQ; ++g) { m[g] = -INFINITY; l[g] = 0.f; }
    }
    const bool real = mt.z > 0;
    const bool last = mt.y == max(it.ntiles, 1) - 1;
    if (real) {
      float x[GQ];
      tmem_ld8(s_tmem(i % NS) + lane_base, x);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[i % NS]);  // the S buffer may take S(i + NS)
      const int tok = it.t_begin + mt.y * TILE + t;
      const bool valid = tok < it.t_end;
#pragma unroll
      for (int g = 0; g < GQ; ++g) x[g] = valid ? x[g] * sl2 : -INFINITY;
      // warp max of the 8 columns in 9 shuffles: halve the columns per step, then reduce;
      // lanes 4g .. 4g+3 end up with column g's max
      float h4[4], h2[2], h1;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool up = lane & 16;
        const float send = up ? x[j] : x[j + 4];
        h4[j] = fmaxf(up ? x[j + 4] : x[j], __shfl_xor_sync(0xffffffffu, send, 16));
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const bool up = lane & 8;
        const float send = up ? h4[j] : h4[j + 2];
        h2[j] = fmaxf(up ? h4[j + 2] : h4[j], __shfl_xor_sync(0xffffffffu, send, 8));
      }
      {
        const bool up = lane & 4;
        const float send = up ? h2[0] : h2[1];
        h1 = fmaxf(up ? h2[1] : h2[0], __shfl_xor_sync(0xffffffffu, send, 4));
      }
      h1 = fmaxf(h1, __shfl_xor_sync(0xffffffffu, h1, 2));
      h1 = fmaxf(h1, __shfl_xor_sync(0xffffffffu, h1, 1));
      float* tm = tmax + bpar * 4 * GQ;
      if ((lane & 3) == 0) tm[warp * GQ + (lane >> 2)] = h1;
      named_bar_sync(1, 128);
      bpar ^= 1;
      uint32_t pw[GQ / 2];
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        const float mx = fmaxf(fmaxf(tm[g], tm[GQ + g]), fmaxf(tm[2 * GQ + g], tm[3 * GQ + g]));
        const float mn = fmaxf(m[g], mx);  // finite: the tile has a valid token
        a_cur[g] = m[g] == -INFINITY ? 0.f : exp2f(m[g] - mn);
        m[g] = mn;
      }
#pragma unroll
      for (int g = 0; g < GQ; g += 2) {
        pw[g / 2] = Elem<T>::pack2(exp2f(x[g] - m[g]), exp2f(x[g + 1] - m[g + 1]));
        float r0, r1;  // the sum uses the rounded weights the MMA sees
        Elem<T>::unpack2(pw[g / 2], r0, r1);
        l[g] = l[g] * a_cur[g] + r0;
        l[g + 1] = l[g + 1] * a_cur[g + 1] + r1;
      }
      *reinterpret_cast<uint4*>(pbuf + (i & 1) * C::PBUF_BYTES + t * 16) =
          make_uint4(pw[0], pw[1], pw[2], pw[3]);
      // stale rows past the end may hold non-finite values and p = 0 must meet 0: zero them,
      // once the tile's V half has landed (it is loaded after the previous O MMA read the
      // slot, so S — and this softmax — can run ahead of it)
      if (it.t_begin + mt.y * TILE + TILE > it.t_end) mbar_wait(&fullv[nv % VS], (nv / VS) & 1);
      if (!valid) {
        uint8_t* vrow = vring + (nv % VS) * C::MAT_BYTES + t * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          *reinterpret_cast<uint4*>(vrow + c * 16) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(vrow + C::BOX_BYTES + c * 16) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      fence_proxy_async_smem();
      ++nv;
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (!real) mbar_arrive(&sfree[i % NS]);  // (a marker reads no S, but owns the buffer)
      mbar_arrive(&pbar[i & 1]);
    }
    // fold the previous tile's O while this tile's O runs on the tensor core; at an item's last
    // tile fold its own O right away and hand the item over — never wait for the next item's
    // tiles (in a step launch the next item may wait for inputs that depend on this item)
    if (pending) fold(i - 1, prev_real, prev_first, a_prev);
    pending = !last;
    if (!last) {
#pragma unroll
      for (int g = 0; g < GQ; ++g) a_prev[g] = a_cur[g];
      prev_real = real;
      prev_first = first;
      continue;
    }
    fold(i, real, first, a_cur);
    float ls[GQ];  // hand the finished item to the epilogue warp
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
      float v = l[g];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      ls[g] = v;
    }
    const int rb = k_item & 1;  // set k_item % 2, free once the epilogue took item k_item - 2
    if (k_item >= 2) mbar_wait(&rempty[rb], ((k_item - 2) >> 1) & 1);
    if (lane == 0) {
      float4* lw = reinterpret_cast<float4*>(red_lw(rb) + warp * GQ);
      lw[0] = make_float4(ls[0], ls[1], ls[2], ls[3]);
      lw[1] = make_float4(ls[4], ls[5], ls[6], ls[7]);
      if (warp == 0) {
        float4* rm = reinterpret_cast<float4*>(red_m(rb));
        rm[0] = make_float4(m[0], m[1], m[2], m[3]);
        rm[1] = make_float4(m[4], m[5], m[6], m[7]);
      }
    }
    float* racc = red_acc(rb);
#pragma unroll
    for (int g = 0; g < GQ; ++g) racc[g * C::RS + t] = o[g];
    if (warp == 0 && lane == 0) {
      ritem[4 * rb] = tag.x;
      ritem[4 * rb + 1] = tag.y;
      ritem[4 * rb + 2] = tag.z;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&rfull[rb]);
    ++k_item;
  }
  for (int e = 0; e < 2; ++e) {  // end of work, to both epilogue warps
    const int k = k_item + e, rb = k & 1;
    if (k >= 2) mbar_wait(&rempty[rb], ((k - 2) >> 1) & 1);
    if (warp == 0 && lane == 0) ritem[4 * rb] = -1;
    __syncwarp();
    if (lane == 0) mbar_arrive(&rfull[rb]);
  }
  named_bar_sync(3, 6 * 32);
}

}  // namespace lam
