/*
 * attn_oracle.h — CPU restatement of the reference decode-attention operator.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the checker
 * or the timed CPU baseline — never as part of the product path.
 *
 * Each function restates the reference file:line it follows
 * (/root/reference/proj/core/src/attention.cpp, tests/oracles.hpp).  Parity of this port is
 * pinned against the reference itself (oracle/_ref/libref_attn.so, compiled from the
 * reference sources by oracle/Makefile) and against the committed fixtures in tests/golden/.
 */
#ifndef ATTN_ORACLE_H
#define ATTN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* exact_attention (attention.cpp:48-70).  Rows are contiguous [l][d].  Returns 1 if l == 0. */
int orc_exact_f64(int64_t d, int64_t l, const double* q, const double* k, const double* v,
                  double scale, double* out);
int orc_exact_f32(int64_t d, int64_t l, const float* q, const float* k, const float* v,
                  float scale, float* out);

/* partial_attention (attention.cpp:72-98).  Returns 2 on an out-of-range index. */
int orc_partial_f64(int64_t d, int64_t l, const double* q, const double* k, const double* v,
                    double scale, const int64_t* idx, int64_t n, double* acc, double* max_logit,
                    double* log_denom, int64_t* count);
int orc_partial_f32(int64_t d, int64_t l, const float* q, const float* k, const float* v,
                    float scale, const int64_t* idx, int64_t n, float* acc, float* max_logit,
                    float* log_denom, int64_t* count);

/* merge (attention.cpp:100-118) and finalize (120-127; returns 1 on an empty partial). */
void orc_merge_f64(int64_t d, const double* a_acc, double a_max, double a_ld, int64_t a_cnt,
                   const double* b_acc, double b_max, double b_ld, int64_t b_cnt, double* o_acc,
                   double* o_max, double* o_ld, int64_t* o_cnt);
void orc_merge_f32(int64_t d, const float* a_acc, float a_max, float a_ld, int64_t a_cnt,
                   const float* b_acc, float b_max, float b_ld, int64_t b_cnt, float* o_acc,
                   float* o_max, float* o_ld, int64_t* o_cnt);
int orc_finalize_f64(int64_t d, const double* acc, double log_denom, int64_t count, double* out);
int orc_finalize_f32(int64_t d, const float* acc, float log_denom, int64_t count, float* out);

/* long-double unstabilised oracle (tests/oracles.hpp:15-38). */
void orc_naive_ld(int64_t d, int64_t l, const double* q, const double* k, const double* v,
                  double scale, double* out);

/* head_partition (attention.cpp:164-177): 0 ok, 2 validation error. */
int orc_head_partition(int64_t num_kv_heads, int64_t num_devices, int64_t* ranges);
/* request_partition (attention.cpp:179-203). */
int orc_request_partition(const double* kv_sizes, int64_t n, int64_t num_devices,
                          int64_t* device_of, double* device_load, double* imbalance);

/* Batched decode over a dense fp32 KV layout [B][Hkv][lmax][D] with q [B][Hq][D]:
 * per (request, q head) exact_attention<float> (compute_f64 = 0) or <double> on the
 * upcast values (compute_f64 = 1), q head h reading KV head h / (Hq/Hkv)
 * (attention.cpp:141-162).  If n_pairs > 0 only the listed (b, h) pairs are computed.
 * lse (nullable) receives max + log(sum) in natural units. */
void orc_decode(int compute_f64, int32_t B, int32_t Hq, int32_t Hkv, int32_t D, int32_t lmax,
                const int32_t* lens, const float* q, const float* k, const float* v, float scale,
                int64_t n_pairs, const int32_t* pair_b, const int32_t* pair_h, float* out,
                float* lse);

/* Paged <-> dense KV movement (byte copies): pool [pages][Hkv][P][row_bytes]. */
void orc_page_scatter(int32_t row_bytes, int32_t B, int32_t Hkv, int32_t P, int32_t pt_stride,
                      const int32_t* page_table, const int32_t* lens, int32_t lmax,
                      const uint8_t* dense, uint8_t* pool);
void orc_page_gather(int32_t row_bytes, int32_t B, int32_t Hkv, int32_t P, int32_t pt_stride,
                     const int32_t* page_table, const int32_t* lens, int32_t lmax,
                     const uint8_t* pool, uint8_t* dense);

#ifdef __cplusplus
}
#endif

#endif
