// decode_simt.cuh — persistent split-K decode attention on CUDA cores (MHA and small GQA
// groups).
//
// A work item is (request b, kv head, q-head group of GQ heads, split).  Warp NW is the
// producer: one lane claims items (decode_common.cuh:producer_loop) and streams their K/V tiles
// (TILE tokens, contiguous in the paged layout) into a STAGES-deep shared-memory ring with 1-D
// TMA bulk copies (cp.async.bulk + mbarrier complete_tx, L2 evict-first).  Warps 0..NW-1 each
// own TILE/NW tokens of every tile and run an independent online softmax over them: q·k by
// 16-byte vector FMAs reduced with warp shuffles, running max / rescale, p·v accumulated in fp32
// registers.  At the end of an item the NW warp partials, and then the split partials, are
// merged in fixed order by a dedicated epilogue warp (finish_item_warp) while the consumers
// already stream the next item; the producer also prefetches each item's q rows by TMA, so an
// item boundary costs the consumers nothing.
//
// Reference semantics: exact_attention / partial_attention
// (/root/reference/proj/core/src/attention.cpp:48-98), logits = (q·k)·scale, fp32
// accumulation.  fp32 KV uses expf/logf in natural units; 16-bit KV uses exp2f with the scale
// pre-multiplied by log2(e).
#pragma once

#include "decode_common.cuh"

namespace lam {

template <typename T, int D, int GQ, int NW_ = 8, int TILE_ = (sizeof(T) == 4 ? 32 : 64),
          int STAGES_ = 6, int NV_ = 1>
struct SimtCfg {
  static constexpr int NW = NW_;                     // consumer warps
  static constexpr int TILE = TILE_;                 // tokens per stage
  static constexpr int STAGES = STAGES_;
  static constexpr int VEC = 16 / sizeof(T);         // elements per 16-byte vector
  static constexpr int NV = NV_;                     // 16-byte vectors per lane and row
  static constexpr int EPL = VEC * NV;               // elements per lane and row
  static constexpr int LPR = D / EPL;                // lanes per K/V row
  static constexpr int RPI = 32 / LPR;               // rows per warp instruction
  static constexpr int TPW = TILE / NW;              // tokens per warp per tile
  static constexpr int ITER = TPW / RPI;
  static constexpr int TILE_BYTES = TILE * D * sizeof(T);
  static constexpr int RING_BYTES = STAGES * 2 * TILE_BYTES;
  static constexpr int Q_BYTES = GQ * D * sizeof(T);  // one item's q rows
  static constexpr int ROW_BYTES = D * sizeof(T);
  static constexpr int SLOT_BYTES = Q_BYTES + 2 * ROW_BYTES;  // q rows + fused new k, v rows
  static constexpr int RED_FLOATS = NW * GQ * (D + 2);
  static constexpr int SMEM_BYTES = RING_BYTES + STAGES * SLOT_BYTES + RED_FLOATS * 4 +
                                    STAGES * 16 + STAGES * 8 + (2 * STAGES + 4) * 8 + 16 + 64;
  static constexpr int THREADS = (NW + 2) * 32;  // + producer warp + epilogue warp
  static constexpr bool kLog2 = sizeof(T) < 4;
  static_assert(LPR >= 1 && LPR <= 32 && 32 % LPR == 0, "row must map onto a warp");
  static_assert(TPW % RPI == 0 && ITER >= 1, "warp slice must be whole instructions");
};

template <typename T, int D, int GQ, int NW, int TILE, int STAGES, int NV = 1>
__global__ void __launch_bounds__((NW + 2) * 32, 1)
    decode_simt_kernel(const DecodeParams p) {
  using C = SimtCfg<T, D, GQ, NW, TILE, STAGES, NV>;
  constexpr int VEC = C::VEC, LPR = C::LPR, RPI = C::RPI, TPW = C::TPW, ITER = C::ITER;
  constexpr int EPL = C::EPL;
  extern __shared__ __align__(128) uint8_t smem[];
  T* ring = reinterpret_cast<T*>(smem);  // [STAGES][2][TILE][D]
  uint8_t* qslot = smem + C::RING_BYTES;  // [STAGES][q rows GQ | new k | new v][D]
  float* red_m = reinterpret_cast<float*>(qslot + STAGES * C::SLOT_BYTES);
  float* red_l = red_m + NW * GQ;
  float* red_acc = red_l + NW * GQ;
  int4* meta = reinterpret_cast<int4*>(red_m + C::RED_FLOATS);
  long long* meta_row = reinterpret_cast<long long*>(meta + STAGES);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta_row + STAGES);
  uint64_t* empty = full + STAGES;
  RedPipe red{empty + STAGES, empty + STAGES + 1, reinterpret_cast<int*>(empty + STAGES + 2)};

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_init(red.full, NW);
    mbar_init(red.empty, 1);
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const T* kp = static_cast<const T*>(p.k_pool);
      const T* vp = static_cast<const T*>(p.v_pool);
      producer_loop<STAGES, TILE>(p, full, empty, meta, meta_row,
                                  [&](int s, const Item& it, int j, const long long* row0, int mode) {
        const int64_t row = row0[0];
        const int tok = it.t_begin + j * TILE;
        const int rows = min(TILE, it.t_end - tok);
        const uint32_t bytes = static_cast<uint32_t>(rows) * D * sizeof(T);
        T* ks = ring + static_cast<size_t>(s) * 2 * TILE * D;
        const bool fused = tile_has_new<TILE>(p, it, j);
        if (mode != kIssueInputs)
          mbar_arrive_expect_tx(&full[s], 2 * bytes + (j == 0 ? C::Q_BYTES : 0) +
                                              (fused ? 2 * C::ROW_BYTES : 0));
        uint8_t* slot = qslot + s * C::SLOT_BYTES;
        if (mode != kIssueKV && j == 0) {
          const T* qsrc = q_rows<T>(p, it) + static_cast<int64_t>(it.kvh * p.G + it.qg * GQ) * D;
          tma_load_1d(slot, qsrc, C::Q_BYTES, &full[s], pol);
        }
        if (mode != kIssueKV && fused) {
          const int64_t off = static_cast<int64_t>(it.kvh) * D;
          tma_load_1d(slot + C::Q_BYTES, new_rows<T>(p, 0, it) + off, C::ROW_BYTES, &full[s], pol);
          tma_load_1d(slot + C::Q_BYTES + C::ROW_BYTES, new_rows<T>(p, 1, it) + off,
                      C::ROW_BYTES, &full[s], pol);
        }
        if (mode == kIssueInputs) return;
        tma_load_1d(ks, kp + row * D, bytes, &full[s], pol);
        tma_load_1d(ks + TILE * D, vp + row * D, bytes, &full[s], pol);
      });
    }
    return;
  }
  if (warp == NW + 1) {
    epilogue_loop<T, D, GQ, NW, C::kLog2, TILE, D>(p, red, GQ, red_m, red_l, red_acc);
    return;
  }

  // ---------------- consumers ----------------
  // Lane `sub` of a row group owns the NV 16-byte vectors sub, sub + LPR, ... of each K / V row
  // (element offsets voff(v)): a quarter-warp phase of 16-byte shared loads reads 128
  // contiguous bytes of one row (no bank conflicts), and NV > 1 shortens the q·k shuffle
  // reduction to log2(LPR) steps per RPI rows.
  const int sub = lane % LPR;  // first 16-byte vector of the row owned by this lane
  const int rg = lane / LPR;   // row group within one instruction
  const float sc = C::kLog2 ? p.scale_log2 : p.scale;
  const uint32_t ring_addr = smem_u32(ring);
  const uint32_t q_addr = smem_u32(qslot);

  auto voff = [&](int v) { return (v * LPR + sub) * VEC; };  // element offset of vector v
  float q[GQ][EPL], m[GQ], l[GQ], acc[GQ][EPL];
  Item it{};
  int k_item = 0;  // hand-offs to the epilogue warp
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
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        if (it.ntiles > 0) {
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            float f[VEC];
            Elem<T>::unpack(lds128(q_addr + s * C::SLOT_BYTES + (g * D + voff(v)) * sizeof(T)), f);
#pragma unroll
            for (int e = 0; e < VEC; ++e) q[g][v * VEC + e] = f[e];
          }
        }
        m[g] = -INFINITY;
        l[g] = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[g][e] = 0.f;
      }
    }
    if (it.ntiles > 0 && !(p.flags & 16)) {  // (flags bit 4: streaming-only diagnostic)
      const int tile_tok = it.t_begin + mt.y * TILE;
      const uint32_t k_addr = ring_addr + s * 2 * C::TILE_BYTES;
      const uint32_t v_addr = k_addr + C::TILE_BYTES;
      // fused append: the request's new token is read from the slot, not from the pool
      const int new_r = tile_has_new<TILE>(p, it, mt.y) ? it.len - 1 - tile_tok : -1;
      const uint32_t kn_addr = q_addr + s * C::SLOT_BYTES + C::Q_BYTES;

      // q·k for this warp's TPW tokens.
      float logit[ITER][GQ];
      bool valid[ITER];
#pragma unroll
      for (int r8 = 0; r8 < ITER; ++r8) {
        const int r = warp * TPW + r8 * RPI + rg;  // row within the tile
        valid[r8] = tile_tok + r < it.t_end;
        float kf[EPL];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const uint32_t vb = voff(v) * sizeof(T);
          const uint4 kraw = lds128(r == new_r ? kn_addr + vb : k_addr + r * D * sizeof(T) + vb);
          if (r == new_r) {  // write the new token into the pool for later steps
            const uint4 vraw = lds128(kn_addr + C::ROW_BYTES + vb);
            const int64_t dst = (meta_row[s] + r) * D + voff(v);
            *reinterpret_cast<uint4*>(static_cast<T*>(p.k_pool_w) + dst) = kraw;
            *reinterpret_cast<uint4*>(static_cast<T*>(p.v_pool_w) + dst) = vraw;
          }
          float f[VEC];
          Elem<T>::unpack(kraw, f);
#pragma unroll
          for (int e = 0; e < VEC; ++e) kf[v * VEC + e] = f[e];
        }
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
          float d0 = 0.f;
#pragma unroll
          for (int e = 0; e < EPL; ++e) d0 = fmaf(q[g][e], kf[e], d0);
          logit[r8][g] = d0;
        }
      }
#pragma unroll
      for (int off = LPR / 2; off >= 1; off >>= 1) {
#pragma unroll
        for (int r8 = 0; r8 < ITER; ++r8)
#pragma unroll
          for (int g = 0; g < GQ; ++g)
            logit[r8][g] += __shfl_xor_sync(0xffffffffu, logit[r8][g], off);
      }

      // online softmax update (per q head, warp-uniform max).
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        float tmax = -INFINITY;
#pragma unroll
        for (int r8 = 0; r8 < ITER; ++r8) {
          logit[r8][g] = valid[r8] ? logit[r8][g] * sc : -INFINITY;
          tmax = fmaxf(tmax, logit[r8][g]);
        }
#pragma unroll
        for (int off = LPR; off < 32; off <<= 1)
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
        const float m_new = fmaxf(m[g], tmax);
        if (m_new != -INFINITY && m_new != m[g]) {
          const float alpha =
              m[g] == -INFINITY ? 0.f : (C::kLog2 ? exp2f(m[g] - m_new) : expf(m[g] - m_new));
          l[g] *= alpha;
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[g][e] *= alpha;
          m[g] = m_new;
        }
      }

      // p·v
#pragma unroll
      for (int r8 = 0; r8 < ITER; ++r8) {
        if (!valid[r8]) continue;
        const int r = warp * TPW + r8 * RPI + rg;
        float vf[EPL];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const uint32_t vb = voff(v) * sizeof(T);
          float f[VEC];
          Elem<T>::unpack(lds128(r == new_r ? kn_addr + C::ROW_BYTES + vb
                                            : v_addr + r * D * sizeof(T) + vb), f);
#pragma unroll
          for (int e = 0; e < VEC; ++e) vf[v * VEC + e] = f[e];
        }
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
          const float pr = C::kLog2 ? exp2f(logit[r8][g] - m[g]) : expf(logit[r8][g] - m[g]);
          l[g] += pr;
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[g][e] = fmaf(pr, vf[e], acc[g][e]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (mt.y == max(it.ntiles, 1) - 1) {
      // end of the item: reduce the RPI row groups of each warp (they share m) and hand the
      // warp partial to the epilogue warp.
#pragma unroll
      for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
          l[g] += __shfl_xor_sync(0xffffffffu, l[g], off);
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[g][e] += __shfl_xor_sync(0xffffffffu, acc[g][e], off);
        }
      }
      red_acquire(red, k_item);
      if (rg == 0) {
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
#pragma unroll
          for (int e = 0; e < EPL; e += 4)
            *reinterpret_cast<float4*>(red_acc + (warp * GQ + g) * D + voff(e / VEC) + e % VEC) =
                make_float4(acc[g][e], acc[g][e + 1], acc[g][e + 2], acc[g][e + 3]);
          if (sub == 0) {
            red_m[warp * GQ + g] = m[g];
            red_l[warp * GQ + g] = l[g];
          }
        }
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
