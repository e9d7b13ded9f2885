// lam_internal.h — launchers shared between the kernel translation units and the C-ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace lam {

struct DecodeParams;

// decode.cu
// persistent launches: `ctas` resident CTAs (num_SMs x occupancy)
cudaError_t launch_decode_simt(int kv_dtype, int D, int GQ, int variant, const DecodeParams& p,
                               int ctas, cudaStream_t stream);
int simt_variant_tile(int kv_dtype, int D, int GQ, int variant);  // 0 = invalid
cudaError_t launch_decode_mma(int kv_dtype, int variant, const DecodeParams& p,
                              const CUtensorMap& kmap, const CUtensorMap& vmap, int grid_x,
                              cudaStream_t stream);
int mma_variant_tile(int variant);  // tokens per stage of a GQA kernel variant (0 = invalid)
// tcgen05 / TMEM GQA kernel: 128-token stages fed as 64-row TMA boxes
cudaError_t launch_decode_tc(int kv_dtype, const DecodeParams& p, const CUtensorMap& kmap,
                             const CUtensorMap& vmap, int grid_x, cudaStream_t stream);
int occupancy_tc(int kv_dtype);
constexpr int kTcTile = 128, kTcBoxRows = 64;
// resident CTAs per SM for an instantiation (0 if unsupported)
int occupancy_simt(int kv_dtype, int D, int GQ, int variant);
int occupancy_mma(int kv_dtype, int variant);
bool simt_supported(int kv_dtype, int D, int GQ);

// instance.cu
cudaError_t launch_instances(int dtype, int64_t n_inst, int32_t d, const void* q, const void* k,
                             const void* v, const int64_t* kv_row0, const int64_t* kv_len,
                             const int64_t* idx, const int64_t* idx_off, const void* scale,
                             void* logits, const int64_t* logit_off, void* acc, void* max_logit,
                             void* log_denom, int64_t* count, int exact, int32_t* err,
                             cudaStream_t stream);
cudaError_t launch_count_scan(int64_t n_inst, const int64_t* kv_len, const int64_t* idx_off,
                              int64_t* logit_off, cudaStream_t stream);
cudaError_t launch_merge(int dtype, int64_t n, int32_t d, const void* a_acc, const void* a_max,
                         const void* a_ld, const int64_t* a_cnt, const void* b_acc,
                         const void* b_max, const void* b_ld, const int64_t* b_cnt, void* o_acc,
                         void* o_max, void* o_ld, int64_t* o_cnt, int32_t* err,
                         cudaStream_t stream);
cudaError_t launch_finalize(int dtype, int64_t n, int32_t d, const void* acc, const void* ld,
                            const int64_t* cnt, void* out, int32_t* err, cudaStream_t stream);

// kv.cu
cudaError_t launch_kv_append(int32_t elem_bytes, int32_t B, int32_t Hkv, int32_t D,
                             int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                             const int32_t* positions, const void* k_new, const void* v_new,
                             int64_t new_stride, void* k_pool, void* v_pool, cudaStream_t stream);
cudaError_t launch_kv_gather(int32_t elem_bytes, int32_t B, int32_t Hkv, int32_t D,
                             int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                             const int32_t* seq_lens, int32_t l_max, const void* pool,
                             void* dense, cudaStream_t stream);

}  // namespace lam
