// decode.cu — instantiations and launchers of the decode kernels.
#include <atomic>

#include "decode_gqa_mma.cuh"
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

template <typename T, int D, int GQ>
cudaError_t simt_launch(const DecodeParams& p, int grid_x, cudaStream_t stream) {
  using C = SimtCfg<T, D, GQ>;
  static std::atomic<uint64_t> done{0};
  auto* k = decode_simt_kernel<T, D, GQ>;
  cudaError_t e = ensure_smem_attr(k, C::SMEM_BYTES, done);
  if (e != cudaSuccess) return e;
  dim3 grid(grid_x, p.Hkv * p.QG, p.B);
  k<<<grid, (C::NW + 1) * 32, C::SMEM_BYTES, stream>>>(p);
  return cudaGetLastError();
}

template <typename T, int D, int GQ>
int simt_occ() {
  using C = SimtCfg<T, D, GQ>;
  static std::atomic<uint64_t> done{0};
  auto* k = decode_simt_kernel<T, D, GQ>;
  if (ensure_smem_attr(k, C::SMEM_BYTES, done) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, (C::NW + 1) * 32, C::SMEM_BYTES) !=
      cudaSuccess)
    return 0;
  return n;
}

template <typename T>
cudaError_t mma_launch(const DecodeParams& p, const CUtensorMap& kmap, const CUtensorMap& vmap,
                       int grid_x, cudaStream_t stream) {
  static std::atomic<uint64_t> done{0};
  auto* k = decode_gqa_mma_kernel<T>;
  cudaError_t e = ensure_smem_attr(k, MmaCfg::SMEM_BYTES, done);
  if (e != cudaSuccess) return e;
  dim3 grid(grid_x, p.Hkv, p.B);
  k<<<grid, (MmaCfg::NW + 1) * 32, MmaCfg::SMEM_BYTES, stream>>>(p, kmap, vmap);
  return cudaGetLastError();
}

template <typename T>
int mma_occ() {
  static std::atomic<uint64_t> done{0};
  auto* k = decode_gqa_mma_kernel<T>;
  if (ensure_smem_attr(k, MmaCfg::SMEM_BYTES, done) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, (MmaCfg::NW + 1) * 32,
                                                    MmaCfg::SMEM_BYTES) != cudaSuccess)
    return 0;
  return n;
}

// dtype codes: 0 f32, 2 bf16, 3 f16 (lamina_attn.h)
#define LAM_SIMT_DISPATCH(DT, Dv, GQv, EXPR)                          \
  do {                                                                \
    if ((DT) == 0) {                                                  \
      using T = float;                                                \
      constexpr int D_ = Dv, GQ_ = GQv;                               \
      EXPR;                                                           \
    } else if ((DT) == 2) {                                           \
      using T = __nv_bfloat16;                                        \
      constexpr int D_ = Dv, GQ_ = GQv;                               \
      EXPR;                                                           \
    } else if ((DT) == 3) {                                           \
      using T = __half;                                               \
      constexpr int D_ = Dv, GQ_ = GQv;                               \
      EXPR;                                                           \
    }                                                                 \
  } while (0)

#define LAM_SIMT_SWITCH(DT, D, GQ, EXPR)                               \
  do {                                                                 \
    if ((D) == 64 && (GQ) == 1) LAM_SIMT_DISPATCH(DT, 64, 1, EXPR);    \
    else if ((D) == 64 && (GQ) == 2) LAM_SIMT_DISPATCH(DT, 64, 2, EXPR); \
    else if ((D) == 64 && (GQ) == 4) LAM_SIMT_DISPATCH(DT, 64, 4, EXPR); \
    else if ((D) == 128 && (GQ) == 1) LAM_SIMT_DISPATCH(DT, 128, 1, EXPR); \
    else if ((D) == 128 && (GQ) == 2) LAM_SIMT_DISPATCH(DT, 128, 2, EXPR); \
    else if ((D) == 128 && (GQ) == 4) LAM_SIMT_DISPATCH(DT, 128, 4, EXPR); \
  } while (0)

}  // namespace

bool simt_supported(int kv_dtype, int D, int GQ) {
  return (kv_dtype == 0 || kv_dtype == 2 || kv_dtype == 3) && (D == 64 || D == 128) &&
         (GQ == 1 || GQ == 2 || GQ == 4);
}

cudaError_t launch_decode_simt(int kv_dtype, int D, int GQ, const DecodeParams& p, int grid_x,
                               cudaStream_t stream) {
  cudaError_t r = cudaErrorInvalidValue;
  LAM_SIMT_SWITCH(kv_dtype, D, GQ, (r = simt_launch<T, D_, GQ_>(p, grid_x, stream)));
  return r;
}

int occupancy_simt(int kv_dtype, int D, int GQ) {
  int r = 0;
  LAM_SIMT_SWITCH(kv_dtype, D, GQ, (r = simt_occ<T, D_, GQ_>()));
  return r;
}

cudaError_t launch_decode_mma(int kv_dtype, const DecodeParams& p, const CUtensorMap& kmap,
                              const CUtensorMap& vmap, int grid_x, cudaStream_t stream) {
  if (kv_dtype == 2) return mma_launch<__nv_bfloat16>(p, kmap, vmap, grid_x, stream);
  if (kv_dtype == 3) return mma_launch<__half>(p, kmap, vmap, grid_x, stream);
  return cudaErrorInvalidValue;
}

int occupancy_mma(int kv_dtype) {
  if (kv_dtype == 2) return mma_occ<__nv_bfloat16>();
  if (kv_dtype == 3) return mma_occ<__half>();
  return 0;
}

}  // namespace lam
