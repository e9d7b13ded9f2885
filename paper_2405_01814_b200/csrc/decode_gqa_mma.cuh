// decode_gqa_mma.cuh — split-K GQA decode attention on tensor cores.
//
// With grouped-query attention (attention.hpp:75-76, attention.cpp:141-150) the G query
// heads that share a KV head turn the per-token GEMV into a genuine small contraction:
//   S^T[tokens x G]  = K[tokens x d] · Q^T[d x G]
//   O^T[d x G]      += V^T[d x tokens] · P^T[tokens x G]
// Both are mma.sync m16n8k16 with N = G = 8 (fp32 accumulate), so the KV tile is read
// from HBM once for all G heads and no MMA lane is padding when G == 8.
//
// Persistent: a work item is (request, kv head, split); warp NW is the TMA producer
// (decode_common.cuh:producer_loop), warps 0..NW-1 each own 16 tokens of every tile.  K/V tiles arrive through 2-D tensor-map TMA with the
// 128-byte swizzle (two 64-column boxes per 128-wide row block), so the ldmatrix fragment
// loads are bank-conflict free.  The S^T accumulator is turned into the P^T B-operand
// in registers (exp2 -> bf16 pack -> movmatrix.trans), never touching shared memory.
#pragma once

#include "decode_common.cuh"

namespace lam {

template <int NW_, int STAGES_>
struct MmaCfg {
  static constexpr int NW = NW_;
  static constexpr int TILE = 16 * NW;  // tokens per stage, 16 per consumer warp
  static constexpr int STAGES = STAGES_;
  static constexpr int D = 128;
  static constexpr int GQ = 8;
  static constexpr int BOX_BYTES = TILE * 64 * 2;    // [TILE rows][64 cols] 16-bit
  static constexpr int MAT_BYTES = 2 * BOX_BYTES;    // one K (or V) tile
  static constexpr int STAGE_BYTES = 2 * MAT_BYTES;  // K + V
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int Q_BYTES = GQ * D * 2;        // one item's (padded) q rows
  static constexpr int ROW_BYTES = D * 2;
  static constexpr int SLOT_BYTES = Q_BYTES + 2 * ROW_BYTES;  // q rows + fused new k, v rows
  // warp partial rows padded to D + 4 floats: the fragment-layout stores of the 4 column
  // pairs of a lane quad land in distinct banks, and rows stay 16-byte aligned
  static constexpr int RS = D + 4;
  static constexpr int RED_FLOATS = NW * GQ * (RS + 2);
  static constexpr int SMEM_BYTES = RING_BYTES + STAGES * SLOT_BYTES + RED_FLOATS * 4 +
                                    STAGES * 16 + STAGES * 8 + (2 * STAGES + 4) * 8 + 16 + 64 +
                                    1024;  // +align slack
  static constexpr int THREADS = (NW + 2) * 32;  // + producer warp + epilogue warp
};

// Byte offset of 16-byte chunk `c` (0..15 across the 128-wide row) of tile row `r`
// inside one K or V tile stored as two 128B-swizzled boxes of BOX_BYTES each.
template <int BOX_BYTES>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (c >> 3) * BOX_BYTES + r * 128 + (((c & 7) ^ (r & 7)) << 4);
}

template <typename T, int NW_, int STAGES_>
__global__ void __launch_bounds__((NW_ + 2) * 32, 1)
    decode_gqa_mma_kernel(const DecodeParams p, const __grid_constant__ CUtensorMap kmap,
                          const __grid_constant__ CUtensorMap vmap) {
  using C = MmaCfg<NW_, STAGES_>;
  constexpr int NW = C::NW, TILE = C::TILE, STAGES = C::STAGES, D = C::D, GQ = C::GQ;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* qslot = smem + C::RING_BYTES;  // [STAGES][q rows 8 | new k | new v][D]
  float* red_m = reinterpret_cast<float*>(qslot + STAGES * C::SLOT_BYTES);
  float* red_l = red_m + NW * GQ;
  float* red_acc = red_l + NW * GQ;
  int4* meta = reinterpret_cast<int4*>(red_m + C::RED_FLOATS);
  long long* meta_row = reinterpret_cast<long long*>(meta + STAGES);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta_row + STAGES);
  uint64_t* empty = full + STAGES;
  RedPipe red{empty + STAGES, empty + STAGES + 1, reinterpret_cast<int*>(empty + STAGES + 2)};

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int G = p.G;  // real q heads in the group (<= 8); the rest are zero padding

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_init(red.full, NW);
    mbar_init(red.empty, 1);
    fence_barrier_init();
  }
  if (warp == NW && lane == 0) {
    prefetch_tensormap(&kmap);
    prefetch_tensormap(&vmap);
  }
  __syncthreads();

  if (warp == NW) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      producer_loop<STAGES, TILE>(p, full, empty, meta, meta_row,
                                  [&](int s, const Item& it, int j, const long long* rows, int mode) {
        const int64_t row = rows[0];
        uint8_t* st = smem + s * C::STAGE_BYTES;
        const uint32_t qb = static_cast<uint32_t>(G) * D * 2;
        const bool fused = tile_has_new<TILE>(p, it, j);
        if (mode != kIssueInputs)
          mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES + (j == 0 ? qb : 0) +
                                              (fused ? 2 * C::ROW_BYTES : 0));
        if (mode != kIssueKV && fused) {
          const int64_t off = static_cast<int64_t>(it.kvh) * D;
          uint8_t* kn = qslot + s * C::SLOT_BYTES + C::Q_BYTES;
          tma_load_1d(kn, new_rows<T>(p, 0, it) + off, C::ROW_BYTES, &full[s], pol);
          tma_load_1d(kn + C::ROW_BYTES, new_rows<T>(p, 1, it) + off, C::ROW_BYTES, &full[s],
                      pol);
        }
        if (mode != kIssueKV && j == 0)
          tma_load_1d(qslot + s * C::SLOT_BYTES,
                      q_rows<T>(p, it) + static_cast<int64_t>(it.kvh) * G * D,
                      qb, &full[s], pol);
        if (mode == kIssueInputs) return;
        const int32_t r32 = static_cast<int32_t>(row);
        tma_load_2d(st, &kmap, 0, r32, &full[s], pol);
        tma_load_2d(st + C::BOX_BYTES, &kmap, 64, r32, &full[s], pol);
        tma_load_2d(st + C::MAT_BYTES, &vmap, 0, r32, &full[s], pol);
        tma_load_2d(st + C::MAT_BYTES + C::BOX_BYTES, &vmap, 64, r32, &full[s], pol);
      });
    }
    return;
  }
  if (warp == NW + 1) {
    epilogue_loop<T, D, GQ, NW, true, TILE, C::RS>(p, red, G, red_m, red_l, red_acc);
    return;
  }

  // ---------------- consumers ----------------
  const int gr = lane >> 2;       // fragment "group" row
  const int gc = (lane & 3) * 2;  // fragment column pair
  const float sl2 = p.scale_log2;
  // per-lane ldmatrix row/chunk selectors
  const int a_row = (lane & 7) + ((lane >> 3) & 1) * 8;  // K: x4 matrices {r0-7,r8-15}x{c,c+1}
  const int a_chk = lane >> 4;
  const int v_row = (lane & 7) + (lane >> 4) * 8;        // V^T: {c,c+1}x{r0-7,r8-15}
  const int v_chk = (lane >> 3) & 1;
  const uint32_t base = smem_u32(smem);

  uint32_t qf[8][2];    // Q^T B-fragments: Q[g=gr][ks*16 + gc (+8) .. +1]
  float m0, m1;         // running max (log2 units) of columns gc, gc+1
  float l0, l1;         // this lane's share of the softmax sums
  float o[8][4];        // O^T accumulators: (d = mt*16 + gr (+8), g = gc, gc+1)
  Item it{};
  int k_item = 0;  // hand-offs to the epilogue warp
  const uint32_t q_addr = smem_u32(qslot);
  for (int i = 0;; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const int4 mt = meta[s];
    if (mt.x < 0) {
      red_acquire(red, k_item);
      if (warp == 0 && lane == 0) red.item[0] = -1;
      red_commit(red);
      break;
    }
    if (mt.y == 0) {  // first tile of a new item: its q rows arrived with this stage
      it = item_from_tag<TILE>(p, mt);
      const uint32_t qrow = q_addr + s * C::SLOT_BYTES + gr * D * 2;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t v0 = 0u, v1 = 0u;
        if (gr < G && it.ntiles > 0) {
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v0) : "r"(qrow + (ks * 16 + gc) * 2));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v1) : "r"(qrow + (ks * 16 + 8 + gc) * 2));
        }
        qf[ks][0] = v0;
        qf[ks][1] = v1;
      }
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[t][e] = 0.f;
    }
    const int tok0 = it.t_begin + mt.y * TILE + warp * 16;
    const int nval = it.ntiles > 0 ? min(16, it.t_end - tok0) : 0;
    const uint32_t kb = base + s * C::STAGE_BYTES;
    const uint32_t vb = kb + C::MAT_BYTES;
    // fused append: the warp holding the new token copies it from the slot into its K/V tile
    // rows (swizzled) and into the pools for later steps
    const int new_r = tile_has_new<TILE>(p, it, mt.y) ? it.len - 1 - (it.t_begin + mt.y * TILE)
                                                      : -1;
    const bool my_new = new_r >= warp * 16 && new_r < warp * 16 + 16;
    if (nval > 0 && !(p.flags & 16)) {  // (flags bit 4: streaming-only diagnostic)
      if (my_new) {
        const uint8_t* kn = qslot + s * C::SLOT_BYTES + C::Q_BYTES;
        const int c = lane & 15;
        const int is_v = lane >> 4;
        const uint4 val = *reinterpret_cast<const uint4*>(kn + is_v * C::ROW_BYTES + c * 16);
        *reinterpret_cast<uint4*>(smem + s * C::STAGE_BYTES + is_v * C::MAT_BYTES +
                                  swz<C::BOX_BYTES>(new_r, c)) = val;
        T* pool = static_cast<T*>(is_v ? p.v_pool_w : p.k_pool_w);
        *reinterpret_cast<uint4*>(pool + (meta_row[s] + new_r) * D + c * 8) = val;
        __syncwarp();
      }
      if (nval < 16) {
        // rows past the sequence end hold stale data: zero this warp's V rows so that
        // p = 0 never meets a non-finite value in the P·V product.
        uint8_t* vrows = smem + s * C::STAGE_BYTES + C::MAT_BYTES;
        for (int r = nval; r < 16; ++r) {
          const int tr = warp * 16 + r;
          reinterpret_cast<uint2*>(vrows + (lane >> 4) * C::BOX_BYTES + tr * 128)[lane & 15] =
              make_uint2(0u, 0u);
        }
        __syncwarp();
      }
      // S^T = K · Q^T
      float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(kb + swz<C::BOX_BYTES>(warp * 16 + a_row, ks * 2 + a_chk), a0, a1, a2, a3);
        Mma16816<T>::run(c, a0, a1, a2, a3, qf[ks][0], qf[ks][1]);
      }
      // logits (log2 units); rows gr and gr+8 of the warp's 16 tokens
      const bool ok_lo = gr < nval, ok_hi = gr + 8 < nval;
      const float x0 = ok_lo ? c[0] * sl2 : -INFINITY;
      const float x1 = ok_lo ? c[1] * sl2 : -INFINITY;
      const float x2 = ok_hi ? c[2] * sl2 : -INFINITY;
      const float x3 = ok_hi ? c[3] * sl2 : -INFINITY;
      float t0 = fmaxf(x0, x2), t1 = fmaxf(x1, x3);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, off));
        t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, off));
      }
      const float n0 = fmaxf(m0, t0), n1 = fmaxf(m1, t1);  // finite: >= 1 valid token
      const float al0 = m0 == -INFINITY ? 0.f : exp2f(m0 - n0);
      const float al1 = m1 == -INFINITY ? 0.f : exp2f(m1 - n1);
      m0 = n0;
      m1 = n1;
      const uint32_t plo = Elem<T>::pack2(exp2f(x0 - n0), exp2f(x1 - n1));
      const uint32_t phi = Elem<T>::pack2(exp2f(x2 - n0), exp2f(x3 - n1));
      // the softmax sums use the rounded weights actually fed to the MMA, so the output
      // stays an exact convex combination of the value rows.
      float r0, r1, r2, r3;
      Elem<T>::unpack2(plo, r0, r1);
      Elem<T>::unpack2(phi, r2, r3);
      l0 = l0 * al0 + (r0 + r2);
      l1 = l1 * al1 + (r1 + r3);
      const uint32_t b0 = movmatrix_trans(plo);
      const uint32_t b1 = movmatrix_trans(phi);
      // O^T = O^T * alpha + V^T · P^T.  Once the running max has settled, alpha is exactly 1
      // for the whole warp on most tiles: skipping the 32 multiplies then changes no bit and
      // saves SM issue slots (and power, which bounds the sustained step under sw_power_cap).
      if (__any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          o[t][0] *= al0;
          o[t][1] *= al1;
          o[t][2] *= al0;
          o[t][3] *= al1;
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4_trans(vb + swz<C::BOX_BYTES>(warp * 16 + v_row, t * 2 + v_chk), a0, a1, a2, a3);
        Mma16816<T>::run(o[t], a0, a1, a2, a3, b0, b1);
      }
      if (nval < 16 || my_new) fence_proxy_async_smem();  // generic stores before the next TMA
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (mt.y == max(it.ntiles, 1) - 1) {
      // end of the item: reduce the softmax sums over the 8 row groups (lanes with equal
      // lane&3), then merge the warps and the splits.
      float s0 = l0, s1 = l1;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, off);
        s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      }
      red_acquire(red, k_item);
      if (gr == 0) {
        red_m[warp * GQ + gc] = m0;
        red_m[warp * GQ + gc + 1] = m1;
        red_l[warp * GQ + gc] = s0;
        red_l[warp * GQ + gc + 1] = s1;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int d = t * 16 + gr;
        red_acc[(warp * GQ + gc) * C::RS + d] = o[t][0];
        red_acc[(warp * GQ + gc + 1) * C::RS + d] = o[t][1];
        red_acc[(warp * GQ + gc) * C::RS + d + 8] = o[t][2];
        red_acc[(warp * GQ + gc + 1) * C::RS + d + 8] = o[t][3];
      }
      if (warp == 0 && lane == 0) {
        red.item[0] = mt.x;
        red.item[1] = mt.z;
        red.item[2] = mt.w;
      }
      red_commit(red);
      ++k_item;
    }
  }
}

}  // namespace lam
