// decode_simt.cuh — split-K decode attention on CUDA cores (MHA and small GQA groups).
//
// One CTA = one (request b, kv head, q-head group, split).  Warp NW is the producer: one
// lane streams the split's K/V tiles (TILE tokens, contiguous in the paged layout) into a
// STAGES-deep shared-memory ring with 1-D TMA bulk copies (cp.async.bulk + mbarrier
// complete_tx, L2 evict-first).  Warps 0..NW-1 each own TILE/NW tokens of every tile and
// run an independent online softmax over them: q·k by 16-byte vector FMAs reduced with
// warp shuffles, running max / rescale, p·v accumulated in fp32 registers.  The NW warp
// partials and then the S split partials are merged in fixed order (decode_common.cuh).
//
// Reference semantics: exact_attention / partial_attention
// (/root/reference/proj/core/src/attention.cpp:48-98), logits = (q·k)·scale, fp32
// accumulation.  fp32 KV uses expf/logf in natural units; 16-bit KV uses exp2f with the
// scale pre-multiplied by log2(e).
#pragma once

#include "decode_common.cuh"

namespace lam {

template <typename T, int D, int GQ>
struct SimtCfg {
  static constexpr int NW = 4;                       // consumer warps
  static constexpr int TILE = 32;                    // tokens per stage
  static constexpr int STAGES = sizeof(T) == 4 ? 3 : 4;
  static constexpr int VEC = 16 / sizeof(T);         // elements per 16-byte vector
  static constexpr int LPR = D / VEC;                // lanes per K/V row
  static constexpr int RPI = 32 / LPR;               // rows per warp instruction
  static constexpr int TPW = TILE / NW;              // tokens per warp per tile
  static constexpr int ITER = TPW / RPI;
  static constexpr int TILE_BYTES = TILE * D * sizeof(T);
  static constexpr int RING_BYTES = STAGES * 2 * TILE_BYTES;
  static constexpr int RED_BYTES = NW * GQ * (D + 2) * 4;
  static constexpr int MAIN_BYTES = RING_BYTES > RED_BYTES ? RING_BYTES : RED_BYTES;
  static constexpr int SMEM_BYTES = MAIN_BYTES + 2 * STAGES * 8 + 16;
  static constexpr bool kLog2 = sizeof(T) < 4;
  static_assert(LPR >= 1 && LPR <= 32 && 32 % LPR == 0, "row must map onto a warp");
  static_assert(TPW % RPI == 0, "warp slice must be whole instructions");
};

template <typename T, int D, int GQ>
__global__ void __launch_bounds__((SimtCfg<T, D, GQ>::NW + 1) * 32)
    decode_simt_kernel(const DecodeParams p) {
  using C = SimtCfg<T, D, GQ>;
  constexpr int NW = C::NW, TILE = C::TILE, STAGES = C::STAGES, VEC = C::VEC, LPR = C::LPR,
                RPI = C::RPI, TPW = C::TPW, ITER = C::ITER;
  extern __shared__ __align__(128) uint8_t smem[];
  T* ring = reinterpret_cast<T*>(smem);  // [STAGES][2][TILE][D]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::MAIN_BYTES);
  uint64_t* empty = full + STAGES;
  int* s_flag = reinterpret_cast<int*>(empty + STAGES);

  const int split = blockIdx.x;
  const int kvh = blockIdx.y / p.QG;
  const int qg = blockIdx.y % p.QG;
  const int b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  const int len = __ldg(p.seq_lens + b);
  const int t_begin = split * p.chunk;
  const int t_end = min(len, t_begin + p.chunk);
  const int n_tiles = t_end > t_begin ? (t_end - t_begin + TILE - 1) / TILE : 0;

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
    if (lane == 0 && n_tiles > 0) {
      const uint64_t pol = policy_evict_first();
      const T* kp = static_cast<const T*>(p.k_pool);
      const T* vp = static_cast<const T*>(p.v_pool);
      for (int i = 0; i < n_tiles; ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        const int tok = t_begin + i * TILE;
        const int rows = min(TILE, t_end - tok);
        const uint32_t bytes = static_cast<uint32_t>(rows) * D * sizeof(T);
        const int64_t row = kv_row(p, b, kvh, tok);
        T* ks = ring + static_cast<size_t>(s) * 2 * TILE * D;
        mbar_arrive_expect_tx(&full[s], 2 * bytes);
        tma_load_1d(ks, kp + row * D, bytes, &full[s], pol);
        tma_load_1d(ks + TILE * D, vp + row * D, bytes, &full[s], pol);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int sub = lane % LPR;  // which 16-byte vector of the row
  const int rg = lane / LPR;   // row group within one instruction
  const int qh0 = kvh * p.G + qg * GQ;

  float q[GQ][VEC];
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    const T* qp = static_cast<const T*>(p.q) + (static_cast<int64_t>(b) * p.Hq + qh0 + g) * D +
                  sub * VEC;
    const uint4 raw = *reinterpret_cast<const uint4*>(qp);
    Elem<T>::unpack(raw, q[g]);
  }
  const float sc = C::kLog2 ? p.scale_log2 : p.scale;

  float m[GQ], l[GQ], acc[GQ][VEC];
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[g][i] = 0.f;
  }

  const uint32_t ring_addr = smem_u32(ring);
  for (int i = 0; i < n_tiles; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const int tile_tok = t_begin + i * TILE;
    const uint32_t k_addr = ring_addr + s * 2 * C::TILE_BYTES;
    const uint32_t v_addr = k_addr + C::TILE_BYTES;

    // q·k for this warp's TPW tokens.
    float logit[ITER][GQ];
    bool valid[ITER];
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int r = warp * TPW + it * RPI + rg;  // row within the tile
      valid[it] = tile_tok + r < t_end;
      float kf[VEC];
      Elem<T>::unpack(lds128(k_addr + (r * D + sub * VEC) * sizeof(T)), kf);
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        float d0 = 0.f;
#pragma unroll
        for (int e = 0; e < VEC; ++e) d0 = fmaf(q[g][e], kf[e], d0);
        logit[it][g] = d0;
      }
    }
#pragma unroll
    for (int off = LPR / 2; off >= 1; off >>= 1) {
#pragma unroll
      for (int it = 0; it < ITER; ++it)
#pragma unroll
        for (int g = 0; g < GQ; ++g)
          logit[it][g] += __shfl_xor_sync(0xffffffffu, logit[it][g], off);
    }

    // online softmax update (per q head, warp-uniform max).
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
      float tmax = -INFINITY;
#pragma unroll
      for (int it = 0; it < ITER; ++it) {
        logit[it][g] = valid[it] ? logit[it][g] * sc : -INFINITY;
        tmax = fmaxf(tmax, logit[it][g]);
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
    for (int it = 0; it < ITER; ++it) {
      if (!valid[it]) continue;
      const int r = warp * TPW + it * RPI + rg;
      float vf[VEC];
      Elem<T>::unpack(lds128(v_addr + (r * D + sub * VEC) * sizeof(T)), vf);
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        const float pr = C::kLog2 ? exp2f(logit[it][g] - m[g]) : expf(logit[it][g] - m[g]);
        l[g] += pr;
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[g][e] = fmaf(pr, vf[e], acc[g][e]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // reduce the RPI row groups of each warp (they share m).
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
      l[g] += __shfl_xor_sync(0xffffffffu, l[g], off);
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[g][e] += __shfl_xor_sync(0xffffffffu, acc[g][e], off);
    }
  }

  // all consumers are past the ring: reuse it for the warp partials.
  named_bar_sync(1, NW * 32);
  float* red_m = reinterpret_cast<float*>(smem);
  float* red_l = red_m + NW * GQ;
  float* red_acc = red_l + NW * GQ;
  if (rg == 0) {
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) red_acc[(warp * GQ + g) * D + sub * VEC + e] = acc[g][e];
      if (sub == 0) {
        red_m[warp * GQ + g] = m[g];
        red_l[warp * GQ + g] = l[g];
      }
    }
  }
  named_bar_sync(1, NW * 32);
  finish_cta<T, D, GQ, NW, C::kLog2>(p, b, kvh, qg, split, GQ, red_m, red_l, red_acc, s_flag);
}

}  // namespace lam
