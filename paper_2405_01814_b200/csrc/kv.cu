// kv.cu — paged KV-cache maintenance kernels (bit-exact byte movement, no arithmetic).
//
// The reference only accounts KV bytes (KvLedger::grow, /root/reference/proj/core/src/sim.cpp:24-28,
// 279-281); this is the B200 store behind that ledger.  Layout per pool:
// [page][Hkv][P][D], so one (page, kv head) block is P*D contiguous elements and a decode
// tile is a single 1-D TMA bulk copy.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lam_internal.h"

namespace lam {
namespace {

// One warp per (request, kv head): copy the D-element K and V rows with 16-byte vectors.
__global__ void kv_append_kernel(int32_t B, int32_t Hkv, int32_t row_vecs, int32_t page_size,
                                 int32_t pt_stride, const int32_t* __restrict__ page_table,
                                 const int32_t* __restrict__ positions,
                                 const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                                 int64_t src_batch_vecs, uint4* __restrict__ k_pool,
                                 uint4* __restrict__ v_pool) {
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (wid >= static_cast<int64_t>(B) * Hkv) return;
  const int b = static_cast<int>(wid / Hkv), h = static_cast<int>(wid % Hkv);
  const int pos = positions[b];
  const int64_t blk = page_table ? page_table[static_cast<int64_t>(b) * pt_stride + pos / page_size]
                                 : static_cast<int64_t>(b);
  const int64_t dst = ((blk * Hkv + h) * page_size + pos % page_size) * row_vecs;
  const int64_t src = b * src_batch_vecs + static_cast<int64_t>(h) * row_vecs;
  for (int e = lane; e < row_vecs; e += 32) {
    k_pool[dst + e] = k_new[src + e];
    v_pool[dst + e] = v_new[src + e];
  }
}

// One CTA per (request, kv head, 32-token block): paged -> dense.
__global__ void kv_gather_kernel(int32_t Hkv, int32_t row_vecs, int32_t page_size,
                                 int32_t pt_stride, const int32_t* __restrict__ page_table,
                                 const int32_t* __restrict__ seq_lens, int32_t l_max,
                                 const uint4* __restrict__ pool, uint4* __restrict__ dense) {
  const int b = blockIdx.z, h = blockIdx.y;
  const int len = seq_lens[b];
  const int t0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * row_vecs; e += blockDim.x) {
    const int t = t0 + e / row_vecs;
    if (t >= len || t >= l_max) continue;
    const int64_t blk = page_table[static_cast<int64_t>(b) * pt_stride + t / page_size];
    const int64_t src = ((blk * Hkv + h) * page_size + t % page_size) * row_vecs + e % row_vecs;
    const int64_t dst = ((static_cast<int64_t>(b) * Hkv + h) * l_max + t) * row_vecs + e % row_vecs;
    dense[dst] = pool[src];
  }
}

}  // namespace

cudaError_t launch_kv_append(int32_t elem_bytes, int32_t B, int32_t Hkv, int32_t D,
                             int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                             const int32_t* positions, const void* k_new, const void* v_new,
                             int64_t new_stride, void* k_pool, void* v_pool, cudaStream_t stream) {
  const int32_t row_vecs = D * elem_bytes / 16;
  const int64_t warps = static_cast<int64_t>(B) * Hkv;
  if (warps == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  kv_append_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      B, Hkv, row_vecs, page_size, pt_stride, page_table, positions,
      static_cast<const uint4*>(k_new), static_cast<const uint4*>(v_new),
      new_stride * elem_bytes / 16, static_cast<uint4*>(k_pool), static_cast<uint4*>(v_pool));
  return cudaGetLastError();
}

cudaError_t launch_kv_gather(int32_t elem_bytes, int32_t B, int32_t Hkv, int32_t D,
                             int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                             const int32_t* seq_lens, int32_t l_max, const void* pool,
                             void* dense, cudaStream_t stream) {
  const int32_t row_vecs = D * elem_bytes / 16;
  if (B == 0 || Hkv == 0 || l_max == 0) return cudaSuccess;
  dim3 grid((l_max + 31) / 32, Hkv, B);
  kv_gather_kernel<<<grid, 256, 0, stream>>>(Hkv, row_vecs, page_size, pt_stride, page_table,
                                             seq_lens, l_max, static_cast<const uint4*>(pool),
                                             static_cast<uint4*>(dense));
  return cudaGetLastError();
}

}  // namespace lam
