// decode.cu — instantiations and launchers of the decode kernels.
#include <atomic>
#include <cstdlib>

#include "decode_gqa_mma.cuh"
#include "decode_gqa_tc.cuh"
#include "decode_simt.cuh"
#include "lam_internal.h"

namespace lam {
namespace {

constexpr int kMaxDevices = 64;

template <typename K>
cudaError_t ensure_smem_attr(K kernel, int bytes, std::atomic<uint64_t>& done_mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev % kMaxDevices);
  if (done_mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done_mask.fetch_or(bit, std::memory_order_release);
  return e;
}

// Launch with programmatic dependent launch when p.pdl: the grid may start while the previous
// kernel of the stream is still draining (its CTAs trigger once they run out of work items).
template <typename K, typename... Args>
cudaError_t launch_k(K kernel, const DecodeParams& p, int ctas, int threads, int smem,
                     cudaStream_t stream, Args... args) {
  if (!p.pdl) {
    kernel<<<ctas, threads, smem, stream>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename T, int D, int GQ, int NW, int TILE, int STAGES, int NV = 1>
cudaError_t simt_launch(const DecodeParams& p, int ctas, cudaStream_t stream) {
  using C = SimtCfg<T, D, GQ, NW, TILE, STAGES, NV>;
  static std::atomic<uint64_t> done{0};
  auto* k = decode_simt_kernel<T, D, GQ, NW, TILE, STAGES, NV>;
  cudaError_t e = ensure_smem_attr(k, C::SMEM_BYTES, done);
  if (e != cudaSuccess) return e;
  return launch_k(k, p, ctas, C::THREADS, C::SMEM_BYTES, stream, p);
}

template <typename T, int D, int GQ, int NW, int TILE, int STAGES, int NV = 1>
int simt_occ() {
  using C = SimtCfg<T, D, GQ, NW, TILE, STAGES, NV>;
  static std::atomic<uint64_t> done{0};
  static std::atomic<int> cached{0};  // queried once per process (one device model)
  if (const int c = cached.load(std::memory_order_relaxed); c > 0) return c;
  auto* k = decode_simt_kernel<T, D, GQ, NW, TILE, STAGES, NV>;
  if (ensure_smem_attr(k, C::SMEM_BYTES, done) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, C::THREADS, C::SMEM_BYTES) !=
      cudaSuccess)
    return 0;
  cached.store(n, std::memory_order_relaxed);
  return n;
}

template <typename T, int NW, int STAGES>
cudaError_t mma_launch_v(const DecodeParams& p, const CUtensorMap& kmap, const CUtensorMap& vmap,
                         int ctas, cudaStream_t stream) {
  using C = MmaCfg<NW, STAGES>;
  static std::atomic<uint64_t> done{0};
  auto* k = decode_gqa_mma_kernel<T, NW, STAGES>;
  cudaError_t e = ensure_smem_attr(k, C::SMEM_BYTES, done);
  if (e != cudaSuccess) return e;
  return launch_k(k, p, ctas, C::THREADS, C::SMEM_BYTES, stream, p, kmap, vmap);
}

template <typename T, int NW, int STAGES>
int mma_occ_v() {
  using C = MmaCfg<NW, STAGES>;
  static std::atomic<uint64_t> done{0};
  static std::atomic<int> cached{0};  // queried once per process (one device model)
  if (const int c = cached.load(std::memory_order_relaxed); c > 0) return c;
  auto* k = decode_gqa_mma_kernel<T, NW, STAGES>;
  if (ensure_smem_attr(k, C::SMEM_BYTES, done) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, C::THREADS, C::SMEM_BYTES) !=
      cudaSuccess)
    return 0;
  cached.store(n, std::memory_order_relaxed);
  return n;
}

template <typename T, int KS, int VS>
cudaError_t tc_launch_v(const DecodeParams& p, const CUtensorMap& kmap, const CUtensorMap& vmap,
                        int ctas, cudaStream_t stream) {
  using C = TcCfg<KS, VS>;
  static std::atomic<uint64_t> done{0};
  auto* k = decode_gqa_tc_kernel<T, KS, VS>;
  cudaError_t e = ensure_smem_attr(k, C::SMEM_BYTES, done);
  if (e != cudaSuccess) return e;
  return launch_k(k, p, ctas, C::THREADS, C::SMEM_BYTES, stream, p, kmap, vmap);
}

// K / V ring slots of the tcgen05 kernel: LAM_TC_RING=33 (3 K + 3 V, default), 24, 42
int tc_ring() {
  static const int r = [] {
    const char* e = std::getenv("LAM_TC_RING");
    const int v = e ? std::atoi(e) : 33;
    return v == 24 || v == 42 ? v : 33;
  }();
  return r;
}

template <typename T>
cudaError_t tc_launch(const DecodeParams& p, const CUtensorMap& kmap, const CUtensorMap& vmap,
                      int ctas, cudaStream_t stream) {
  if (tc_ring() == 24) return tc_launch_v<T, 2, 4>(p, kmap, vmap, ctas, stream);
  if (tc_ring() == 42) return tc_launch_v<T, 4, 2>(p, kmap, vmap, ctas, stream);
  return tc_launch_v<T, 3, 3>(p, kmap, vmap, ctas, stream);
}

template <typename T, int KS, int VS>
int tc_occ_v() {
  using C = TcCfg<KS, VS>;
  static std::atomic<uint64_t> done{0};
  static std::atomic<int> cached{0};
  if (const int c = cached.load(std::memory_order_relaxed); c > 0) return c;
  auto* k = decode_gqa_tc_kernel<T, KS, VS>;
  if (ensure_smem_attr(k, C::SMEM_BYTES, done) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, C::THREADS, C::SMEM_BYTES) !=
      cudaSuccess)
    return 0;
  cached.store(n, std::memory_order_relaxed);
  return n;
}

template <typename T>
int tc_occ() {
  return tc_ring() == 24 ? tc_occ_v<T, 2, 4>() : tc_ring() == 42 ? tc_occ_v<T, 4, 2>()
                                                                   : tc_occ_v<T, 3, 3>();
}

// GQA kernel variants (consumer warps, stages): tile = 16 tokens per consumer warp.
#define LAM_MMA_VARIANTS(X) X(0, 4, 6) X(1, 4, 3) X(2, 8, 2) X(3, 2, 6) X(4, 2, 4) X(5, 4, 2) X(6, 2, 3)

template <typename T>
cudaError_t mma_launch(int variant, const DecodeParams& p, const CUtensorMap& kmap,
                       const CUtensorMap& vmap, int grid_x, cudaStream_t stream) {
#define X(id, nw, st) \
  if (variant == id) return mma_launch_v<T, nw, st>(p, kmap, vmap, grid_x, stream);
  LAM_MMA_VARIANTS(X)
#undef X
  return cudaErrorInvalidValue;
}

template <typename T>
int mma_occ(int variant) {
#define X(id, nw, st) \
  if (variant == id) return mma_occ_v<T, nw, st>();
  LAM_MMA_VARIANTS(X)
#undef X
  return 0;
}

// SIMT variants (consumer warps, tokens per stage for 32-bit / 16-bit KV, stages, 16-byte
// vectors per lane and row).  Variant 0 is the default for every (dtype, D, GQ); the others
// exist for D = 128, GQ = 1 (tuning).
#define LAM_SIMT_VARIANTS(X) \
  X(1, 8, 32, 64, 6, 1) X(2, 8, 32, 64, 3, 1) X(3, 4, 32, 32, 4, 1) X(4, 16, 32, 64, 4, 1) \
  X(5, 16, 64, 64, 3, 1) X(6, 8, 64, 64, 3, 1) X(7, 16, 64, 64, 3, 2) X(8, 8, 64, 64, 3, 2) \
  X(9, 16, 64, 128, 3, 4)

struct SimtLaunchF {
  const DecodeParams& p;
  int ctas;
  cudaStream_t s;
  template <typename T, int DD, int GG, int NW, int TILE, int ST, int NV = 1>
  cudaError_t operator()() const { return simt_launch<T, DD, GG, NW, TILE, ST, NV>(p, ctas, s); }
};
struct SimtOccF {
  template <typename T, int DD, int GG, int NW, int TILE, int ST, int NV = 1>
  int operator()() const { return simt_occ<T, DD, GG, NW, TILE, ST, NV>(); }
};
struct SimtTileF {
  template <typename T, int DD, int GG, int NW, int TILE, int ST, int NV = 1>
  int operator()() const { return TILE; }
};

template <typename T, int D, int GQ, class F>
auto simt_variant(int variant, F f) {
  constexpr bool wide = sizeof(T) == 4;
  // default: 16 consumer warps (measured best on B200 for MHA), 8 when GQ = 4 (smem)
  if (variant == 0) return f.template operator()<T, D, GQ, GQ <= 2 ? 16 : 8, wide ? 32 : 64, 6>();
  if constexpr (D == 128 && GQ == 1) {
#define X(id, nw, t32, t16, st, nv) \
    if (variant == id) return f.template operator()<T, D, GQ, nw, wide ? t32 : t16, st, nv>();
    LAM_SIMT_VARIANTS(X)
#undef X
  }
  return decltype(f.template operator()<T, D, GQ, 8, wide ? 32 : 64, 6>())();
}

template <class F>
auto simt_dispatch(int dt, int D, int GQ, int variant, F f) {
  using R = decltype(f.template operator()<float, 128, 1, 8, 32, 6>());
#define LAM_ONE(TT, DD, GG) \
  if (D == DD && GQ == GG) return simt_variant<TT, DD, GG>(variant, f);
#define LAM_ALL(TT) LAM_ONE(TT, 64, 1) LAM_ONE(TT, 64, 2) LAM_ONE(TT, 64, 4) \
                    LAM_ONE(TT, 128, 1) LAM_ONE(TT, 128, 2) LAM_ONE(TT, 128, 4)
  if (dt == 0) { LAM_ALL(float) }
  if (dt == 2) { LAM_ALL(__nv_bfloat16) }
  if (dt == 3) { LAM_ALL(__half) }
#undef LAM_ALL
#undef LAM_ONE
  return R();
}

}  // namespace

bool simt_supported(int kv_dtype, int D, int GQ) {
  return (kv_dtype == 0 || kv_dtype == 2 || kv_dtype == 3) && (D == 64 || D == 128) &&
         (GQ == 1 || GQ == 2 || GQ == 4);
}

int simt_variant_tile(int kv_dtype, int D, int GQ, int variant);

cudaError_t launch_decode_simt(int kv_dtype, int D, int GQ, int variant, const DecodeParams& p,
                               int ctas, cudaStream_t stream) {
  if (simt_variant_tile(kv_dtype, D, GQ, variant) == 0) return cudaErrorInvalidValue;
  return simt_dispatch(kv_dtype, D, GQ, variant, SimtLaunchF{p, ctas, stream});
}

int occupancy_simt(int kv_dtype, int D, int GQ, int variant) {
  return simt_dispatch(kv_dtype, D, GQ, variant, SimtOccF{});
}

int simt_variant_tile(int kv_dtype, int D, int GQ, int variant) {
  return simt_dispatch(kv_dtype, D, GQ, variant, SimtTileF{});
}

int mma_variant_tile(int variant) {
#define X(id, nw, st) \
  if (variant == id) return 16 * nw;
  LAM_MMA_VARIANTS(X)
#undef X
  return 0;
}

cudaError_t launch_decode_mma(int kv_dtype, int variant, const DecodeParams& p,
                              const CUtensorMap& kmap, const CUtensorMap& vmap, int grid_x,
                              cudaStream_t stream) {
  if (kv_dtype == 2) return mma_launch<__nv_bfloat16>(variant, p, kmap, vmap, grid_x, stream);
  if (kv_dtype == 3) return mma_launch<__half>(variant, p, kmap, vmap, grid_x, stream);
  return cudaErrorInvalidValue;
}

cudaError_t launch_decode_tc(int kv_dtype, const DecodeParams& p, const CUtensorMap& kmap,
                             const CUtensorMap& vmap, int grid_x, cudaStream_t stream) {
  if (kv_dtype == 2) return tc_launch<__nv_bfloat16>(p, kmap, vmap, grid_x, stream);
  if (kv_dtype == 3) return tc_launch<__half>(p, kmap, vmap, grid_x, stream);
  return cudaErrorInvalidValue;
}

int occupancy_tc(int kv_dtype) {
  if (kv_dtype == 2) return tc_occ<__nv_bfloat16>();
  if (kv_dtype == 3) return tc_occ<__half>();
  return 0;
}

int occupancy_mma(int kv_dtype, int variant) {
  if (kv_dtype == 2) return mma_occ<__nv_bfloat16>(variant);
  if (kv_dtype == 3) return mma_occ<__half>(variant);
  return 0;
}

}  // namespace lam
