/*
 * attn_oracle.c — plain-C restatement of the reference decode-attention operator.
 * TEST INFRASTRUCTURE ONLY (see attn_oracle.h): the checker for the CUDA path, never
 * part of it.  Arithmetic order follows the reference statement by statement so that,
 * compiled without fast-math, results are bitwise equal to the reference's own
 * attention.cpp built in oracle/_ref (pinned by tests/test_oracle.py).
 */
#include "attn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Generates the float and double variants of one routine. */
#define ORC_DEFINE(T, SFX, EXP, LOG, NEG_INF)                                                    \
  /* dot, attention.cpp:16-21 */                                                                 \
  static T dot_##SFX(int64_t d, const T* a, const T* b) {                                        \
    T s = 0;                                                                                     \
    for (int64_t i = 0; i < d; ++i) s += a[i] * b[i];                                            \
    return s;                                                                                    \
  }                                                                                              \
  /* exact_attention, attention.cpp:48-70 */                                                     \
  int orc_exact_##SFX(int64_t d, int64_t l, const T* q, const T* k, const T* v, T scale,         \
                      T* out) {                                                                  \
    if (l == 0) return 1;                                                                        \
    T* logits = (T*)malloc(sizeof(T) * (size_t)l);                                               \
    T max_logit = NEG_INF;                                                                       \
    for (int64_t j = 0; j < l; ++j) {                                                            \
      logits[j] = dot_##SFX(d, q, k + j * d) * scale;                                            \
      max_logit = (max_logit < logits[j]) ? logits[j] : max_logit;                               \
    }                                                                                            \
    for (int64_t i = 0; i < d; ++i) out[i] = 0;                                                  \
    T denom = 0;                                                                                 \
    for (int64_t j = 0; j < l; ++j) {                                                            \
      const T w = EXP(logits[j] - max_logit);                                                    \
      denom += w;                                                                                \
      for (int64_t i = 0; i < d; ++i) out[i] += w * v[j * d + i];                                \
    }                                                                                            \
    for (int64_t i = 0; i < d; ++i) out[i] /= denom;                                             \
    free(logits);                                                                                \
    return 0;                                                                                    \
  }                                                                                              \
  /* partial_attention, attention.cpp:72-98 */                                                   \
  int orc_partial_##SFX(int64_t d, int64_t l, const T* q, const T* k, const T* v, T scale,       \
                        const int64_t* idx, int64_t n, T* acc, T* max_out, T* ld_out,            \
                        int64_t* cnt) {                                                          \
    for (int64_t i = 0; i < d; ++i) acc[i] = 0;                                                  \
    *max_out = NEG_INF;                                                                          \
    *ld_out = NEG_INF;                                                                           \
    *cnt = 0;                                                                                    \
    if (n == 0) return 0;                                                                        \
    T max_logit = NEG_INF;                                                                       \
    T* logits = (T*)malloc(sizeof(T) * (size_t)n);                                               \
    for (int64_t t = 0; t < n; ++t) {                                                            \
      const int64_t j = idx[t];                                                                  \
      if (j < 0 || j >= l) {                                                                     \
        free(logits);                                                                            \
        return 2;                                                                                \
      }                                                                                          \
      logits[t] = dot_##SFX(d, q, k + j * d) * scale;                                            \
      max_logit = (max_logit < logits[t]) ? logits[t] : max_logit;                               \
    }                                                                                            \
    T denom = 0;                                                                                 \
    for (int64_t t = 0; t < n; ++t) {                                                            \
      const T w = EXP(logits[t] - max_logit);                                                    \
      denom += w;                                                                                \
      const T* vr = v + idx[t] * d;                                                              \
      for (int64_t i = 0; i < d; ++i) acc[i] += w * vr[i];                                       \
    }                                                                                            \
    *max_out = max_logit;                                                                        \
    *ld_out = LOG(denom);                                                                        \
    *cnt = n;                                                                                    \
    free(logits);                                                                                \
    return 0;                                                                                    \
  }                                                                                              \
  /* merge, attention.cpp:100-118 (identity early-outs copy the other side bitwise) */           \
  void orc_merge_##SFX(int64_t d, const T* a_acc, T a_max, T a_ld, int64_t a_cnt, const T* b_acc, \
                       T b_max, T b_ld, int64_t b_cnt, T* o_acc, T* o_max, T* o_ld,              \
                       int64_t* o_cnt) {                                                         \
    if (a_cnt == 0 || b_cnt == 0) {                                                              \
      const int a_empty = a_cnt == 0;                                                            \
      memmove(o_acc, a_empty ? b_acc : a_acc, sizeof(T) * (size_t)d);                            \
      *o_max = a_empty ? b_max : a_max;                                                          \
      *o_ld = a_empty ? b_ld : a_ld;                                                             \
      *o_cnt = a_empty ? b_cnt : a_cnt;                                                          \
      return;                                                                                    \
    }                                                                                            \
    const T m = (a_max < b_max) ? b_max : a_max;                                                 \
    const T wa = EXP(a_max - m);                                                                 \
    const T wb = EXP(b_max - m);                                                                 \
    for (int64_t i = 0; i < d; ++i) o_acc[i] = wa * a_acc[i] + wb * b_acc[i];                    \
    const T denom = wa * EXP(a_ld) + wb * EXP(b_ld);                                             \
    *o_max = m;                                                                                  \
    *o_ld = LOG(denom);                                                                          \
    *o_cnt = a_cnt + b_cnt;                                                                      \
  }                                                                                              \
  /* finalize, attention.cpp:120-127 */                                                          \
  int orc_finalize_##SFX(int64_t d, const T* acc, T log_denom, int64_t count, T* out) {         \
    if (count == 0) return 1;                                                                    \
    const T denom = EXP(log_denom);                                                              \
    for (int64_t i = 0; i < d; ++i) out[i] = acc[i] / denom;                                     \
    return 0;                                                                                    \
  }

ORC_DEFINE(double, f64, exp, log, -INFINITY)
ORC_DEFINE(float, f32, expf, logf, -INFINITY)

/* tests/oracles.hpp:15-38 — long double, no max shift. */
void orc_naive_ld(int64_t d, int64_t l, const double* q, const double* k, const double* v,
                  double scale, double* out) {
  long double* w = (long double*)malloc(sizeof(long double) * (size_t)(l > 0 ? l : 1));
  long double denom = 0;
  for (int64_t j = 0; j < l; ++j) {
    long double logit = 0;
    for (int64_t i = 0; i < d; ++i) logit += (long double)q[i] * (long double)k[j * d + i];
    logit *= (long double)scale;
    w[j] = expl(logit);
    denom += w[j];
  }
  for (int64_t i = 0; i < d; ++i) {
    long double acc = 0;
    for (int64_t j = 0; j < l; ++j) acc += w[j] * (long double)v[j * d + i];
    out[i] = (double)(acc / denom);
  }
  free(w);
}

/* attention.cpp:164-177 */
int orc_head_partition(int64_t num_kv_heads, int64_t num_devices, int64_t* ranges) {
  if (num_kv_heads < 1 || num_devices < 1) return 2;
  if (num_kv_heads % num_devices != 0) return 2;
  const int64_t per = num_kv_heads / num_devices;
  for (int64_t i = 0; i < num_devices; ++i) {
    ranges[2 * i] = i * per;
    ranges[2 * i + 1] = (i + 1) * per;
  }
  return 0;
}

/* attention.cpp:179-203: stable longest-first order, least-loaded device, ties low. */
int orc_request_partition(const double* kv_sizes, int64_t n, int64_t num_devices,
                          int64_t* device_of, double* device_load, double* imbalance) {
  if (num_devices < 1) return 2;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    order[i] = i;
    device_of[i] = 0;
  }
  /* stable insertion sort by descending size */
  for (int64_t i = 1; i < n; ++i) {
    const int64_t key = order[i];
    int64_t j = i - 1;
    while (j >= 0 && kv_sizes[order[j]] < kv_sizes[key]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = key;
  }
  for (int64_t d = 0; d < num_devices; ++d) device_load[d] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t r = order[i];
    int64_t t = 0;
    for (int64_t d = 1; d < num_devices; ++d)
      if (device_load[d] < device_load[t]) t = d;
    device_of[r] = t;
    device_load[t] += kv_sizes[r];
  }
  double total = 0, peak = device_load[0];
  for (int64_t d = 0; d < num_devices; ++d) {
    total += device_load[d];
    if (device_load[d] > peak) peak = device_load[d];
  }
  const double mean = total / (double)num_devices;
  *imbalance = mean > 0 ? peak / mean : 1.0;
  free(order);
  return 0;
}

/* One (request, q head) of a dense fp32 layout, exact_attention semantics. */
static void decode_one(int compute_f64, int32_t Hq, int32_t Hkv, int32_t D, int32_t lmax,
                       const int32_t* lens, const float* q, const float* k, const float* v,
                       float scale, int32_t b, int32_t h, float* out, float* lse) {
  const int32_t G = Hq / Hkv;
  const int32_t kvh = h / G;
  const int64_t l = lens[b];
  const float* qh = q + ((int64_t)b * Hq + h) * D;
  const float* kb = k + ((int64_t)b * Hkv + kvh) * lmax * D;
  const float* vb = v + ((int64_t)b * Hkv + kvh) * lmax * D;
  float* o = out + ((int64_t)b * Hq + h) * D;
  if (l == 0) {
    for (int32_t i = 0; i < D; ++i) o[i] = 0.f;
    if (lse) lse[(int64_t)b * Hq + h] = -INFINITY;
    return;
  }
  if (!compute_f64) {
    orc_exact_f32(D, l, qh, kb, vb, scale, o);
    if (lse) { /* max + log(sum exp(logit - max)), float arithmetic */
      float mx = -INFINITY;
      for (int64_t j = 0; j < l; ++j) {
        const float x = dot_f32(D, qh, kb + j * D) * scale;
        mx = (mx < x) ? x : mx;
      }
      float s = 0.f;
      for (int64_t j = 0; j < l; ++j) s += expf(dot_f32(D, qh, kb + j * D) * scale - mx);
      lse[(int64_t)b * Hq + h] = mx + logf(s);
    }
    return;
  }
  double* qd = (double*)malloc(sizeof(double) * (size_t)D);
  double* kd = (double*)malloc(sizeof(double) * (size_t)(l * D));
  double* vd = (double*)malloc(sizeof(double) * (size_t)(l * D));
  double* od = (double*)malloc(sizeof(double) * (size_t)D);
  for (int32_t i = 0; i < D; ++i) qd[i] = qh[i];
  for (int64_t i = 0; i < l * D; ++i) {
    kd[i] = kb[i];
    vd[i] = vb[i];
  }
  orc_exact_f64(D, l, qd, kd, vd, (double)scale, od);
  for (int32_t i = 0; i < D; ++i) o[i] = (float)od[i];
  if (lse) {
    double mx = -INFINITY;
    for (int64_t j = 0; j < l; ++j) {
      const double x = dot_f64(D, qd, kd + j * D) * (double)scale;
      mx = (mx < x) ? x : mx;
    }
    double s = 0.0;
    for (int64_t j = 0; j < l; ++j) s += exp(dot_f64(D, qd, kd + j * D) * (double)scale - mx);
    lse[(int64_t)b * Hq + h] = (float)(mx + log(s));
  }
  free(qd);
  free(kd);
  free(vd);
  free(od);
}

void orc_decode(int compute_f64, int32_t B, int32_t Hq, int32_t Hkv, int32_t D, int32_t lmax,
                const int32_t* lens, const float* q, const float* k, const float* v, float scale,
                int64_t n_pairs, const int32_t* pair_b, const int32_t* pair_h, float* out,
                float* lse) {
  if (n_pairs > 0) {
    for (int64_t i = 0; i < n_pairs; ++i)
      decode_one(compute_f64, Hq, Hkv, D, lmax, lens, q, k, v, scale, pair_b[i], pair_h[i], out,
                 lse);
    return;
  }
  for (int32_t b = 0; b < B; ++b)
    for (int32_t h = 0; h < Hq; ++h)
      decode_one(compute_f64, Hq, Hkv, D, lmax, lens, q, k, v, scale, b, h, out, lse);
}

void orc_page_scatter(int32_t row_bytes, int32_t B, int32_t Hkv, int32_t P, int32_t pt_stride,
                      const int32_t* page_table, const int32_t* lens, int32_t lmax,
                      const uint8_t* dense, uint8_t* pool) {
  for (int32_t b = 0; b < B; ++b)
    for (int32_t h = 0; h < Hkv; ++h)
      for (int32_t t = 0; t < lens[b] && t < lmax; ++t) {
        const int64_t page = page_table[(int64_t)b * pt_stride + t / P];
        memcpy(pool + ((page * Hkv + h) * P + t % P) * row_bytes,
               dense + (((int64_t)b * Hkv + h) * lmax + t) * row_bytes, (size_t)row_bytes);
      }
}

void orc_page_gather(int32_t row_bytes, int32_t B, int32_t Hkv, int32_t P, int32_t pt_stride,
                     const int32_t* page_table, const int32_t* lens, int32_t lmax,
                     const uint8_t* pool, uint8_t* dense) {
  for (int32_t b = 0; b < B; ++b)
    for (int32_t h = 0; h < Hkv; ++h)
      for (int32_t t = 0; t < lens[b] && t < lmax; ++t) {
        const int64_t page = page_table[(int64_t)b * pt_stride + t / P];
        memcpy(dense + (((int64_t)b * Hkv + h) * lmax + t) * row_bytes,
               pool + ((page * Hkv + h) * P + t % P) * row_bytes, (size_t)row_bytes);
      }
}
