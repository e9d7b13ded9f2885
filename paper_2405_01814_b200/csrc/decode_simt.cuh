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
// merged in fixed order (finish_item).
//
// Reference semantics: exact_attention / partial_attention
// (/root/reference/proj/core/src/attention.cpp:48-98), logits = (q·k)·scale, fp32
// accumulation.  fp32 KV uses expf/logf in natural units; 16-bit KV uses exp2f with the scale
// pre-multiplied by log2(e).
#pragma once

#include "decode_common.cuh"

namespace lam {

template <typename T, int D, int GQ, int NW_ = 8, int TILE_ = (sizeof(T) == 4 ? 32 : 64),
          int STAGES_ = 6>
struct SimtCfg {
  static constexpr int NW = NW_;                     // consumer warps
  static constexpr int TILE = TILE_;                 // tokens per stage
  static constexpr int STAGES = STAGES_;
  static constexpr int VEC = 16 / sizeof(T);         // elements per 16-byte vector
  static constexpr int LPR = D / VEC;                // lanes per K/V row
  static constexpr int RPI = 32 / LPR;               // rows per warp instruction
  static constexpr int TPW = TILE / NW;              // tokens per warp per tile
  static constexpr int ITER = TPW / RPI;
  static constexpr int TILE_BYTES = TILE * D * sizeof(T);
  static constexpr int RING_BYTES = STAGES * 2 * TILE_BYTES;
  static constexpr int RED_FLOATS = NW * GQ * (D + 2);
  static constexpr int SMEM_BYTES = RING_BYTES + RED_FLOATS * 4 + STAGES * 16 + 2 * STAGES * 8 + 16;
  static constexpr bool kLog2 = sizeof(T) < 4;
  static_assert(LPR >= 1 && LPR <= 32 && 32 % LPR == 0, "row must map onto a warp");
  static_assert(TPW % RPI == 0 && ITER >= 1, "warp slice must be whole instructions");
};

template <typename T, int D, int GQ, int NW, int TILE, int STAGES>
__global__ void __launch_bounds__((NW + 1) * 32)
    decode_simt_kernel(const DecodeParams p) {
  using C = SimtCfg<T, D, GQ, NW, TILE, STAGES>;
  constexpr int VEC = C::VEC, LPR = C::LPR, RPI = C::RPI, TPW = C::TPW, ITER = C::ITER;
  extern __shared__ __align__(128) uint8_t smem[];
  T* ring = reinterpret_cast<T*>(smem);  // [STAGES][2][TILE][D]
  float* red_m = reinterpret_cast<float*>(smem + C::RING_BYTES);
  float* red_l = red_m + NW * GQ;
  float* red_acc = red_l + NW * GQ;
  int4* meta = reinterpret_cast<int4*>(red_m + C::RED_FLOATS);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + STAGES);
  uint64_t* empty = full + STAGES;
  int* s_flag = reinterpret_cast<int*>(empty + STAGES);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const T* kp = static_cast<const T*>(p.k_pool);
      const T* vp = static_cast<const T*>(p.v_pool);
      producer_loop<STAGES, TILE>(p, full, empty, meta, [&](int s, const Item& it, int j) {
        const int tok = it.t_begin + j * TILE;
        const int rows = min(TILE, it.t_end - tok);
        const uint32_t bytes = static_cast<uint32_t>(rows) * D * sizeof(T);
        const int64_t row = kv_row(p, it.b, it.kvh, tok);
        T* ks = ring + static_cast<size_t>(s) * 2 * TILE * D;
        mbar_arrive_expect_tx(&full[s], 2 * bytes);
        tma_load_1d(ks, kp + row * D, bytes, &full[s], pol);
        tma_load_1d(ks + TILE * D, vp + row * D, bytes, &full[s], pol);
      });
    }
    return;
  }

  // ---------------- consumers ----------------
  const int sub = lane % LPR;  // which 16-byte vector of the row
  const int rg = lane / LPR;   // row group within one instruction
  const float sc = C::kLog2 ? p.scale_log2 : p.scale;
  const uint32_t ring_addr = smem_u32(ring);

  float q[GQ][VEC], m[GQ], l[GQ], acc[GQ][VEC];
  Item it{};
  for (int i = 0;; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const int4 mt = meta[s];
    if (mt.x < 0) break;
    if (mt.y == 0) {  // first tile of a new item: load its q, reset the softmax state
      it = make_item(p, mt.x, TILE);
      const int qh0 = it.kvh * p.G + it.qg * GQ;
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        const T* qp = static_cast<const T*>(p.q) +
                      (static_cast<int64_t>(it.b) * p.Hq + qh0 + g) * D + sub * VEC;
        Elem<T>::unpack(*reinterpret_cast<const uint4*>(qp), q[g]);
        m[g] = -INFINITY;
        l[g] = 0.f;
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[g][e] = 0.f;
      }
    }
    if (mt.z > 0) {
      const int tile_tok = it.t_begin + mt.y * TILE;
      const uint32_t k_addr = ring_addr + s * 2 * C::TILE_BYTES;
      const uint32_t v_addr = k_addr + C::TILE_BYTES;

      // q·k for this warp's TPW tokens.
      float logit[ITER][GQ];
      bool valid[ITER];
#pragma unroll
      for (int r8 = 0; r8 < ITER; ++r8) {
        const int r = warp * TPW + r8 * RPI + rg;  // row within the tile
        valid[r8] = tile_tok + r < it.t_end;
        float kf[VEC];
        Elem<T>::unpack(lds128(k_addr + (r * D + sub * VEC) * sizeof(T)), kf);
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
          float d0 = 0.f;
#pragma unroll
          for (int e = 0; e < VEC; ++e) d0 = fmaf(q[g][e], kf[e], d0);
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
          for (int e = 0; e < VEC; ++e) acc[g][e] *= alpha;
          m[g] = m_new;
        }
      }

      // p·v
#pragma unroll
      for (int r8 = 0; r8 < ITER; ++r8) {
        if (!valid[r8]) continue;
        const int r = warp * TPW + r8 * RPI + rg;
        float vf[VEC];
        Elem<T>::unpack(lds128(v_addr + (r * D + sub * VEC) * sizeof(T)), vf);
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
          const float pr = C::kLog2 ? exp2f(logit[r8][g] - m[g]) : expf(logit[r8][g] - m[g]);
          l[g] += pr;
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[g][e] = fmaf(pr, vf[e], acc[g][e]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (mt.y == max(mt.z, 1) - 1) {
      // end of the item: reduce the RPI row groups of each warp (they share m), then the
      // warps, then the splits.
      float lr[GQ], ar[GQ][VEC];
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        lr[g] = l[g];
#pragma unroll
        for (int e = 0; e < VEC; ++e) ar[g][e] = acc[g][e];
      }
#pragma unroll
      for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
          lr[g] += __shfl_xor_sync(0xffffffffu, lr[g], off);
#pragma unroll
          for (int e = 0; e < VEC; ++e) ar[g][e] += __shfl_xor_sync(0xffffffffu, ar[g][e], off);
        }
      }
      named_bar_sync(1, NW * 32);  // the previous item's epilogue is done with red_*
      if (rg == 0) {
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) red_acc[(warp * GQ + g) * D + sub * VEC + e] = ar[g][e];
          if (sub == 0) {
            red_m[warp * GQ + g] = m[g];
            red_l[warp * GQ + g] = lr[g];
          }
        }
      }
      named_bar_sync(1, NW * 32);
      finish_item<T, D, GQ, NW, C::kLog2>(p, it, GQ, red_m, red_l, red_acc, s_flag);
    }
  }
}

}  // namespace lam
