// instance.cu — device implementation of the reference operator API on AttnInstance
// batches, for both of the reference's instantiations (float and double,
// /root/reference/proj/core/src/attention.cpp:205-230).
//
// One CTA per instance, fixed reduction trees: the result for an instance depends only on
// that instance's data, never on what else is in the batch, so head-partitioned and
// GQA-vs-replicated outputs are bitwise identical (test_attention.cpp:210-269).
//   exact_attention   attention.cpp:48-70   two passes: logits + max, weights + p·v
//   partial_attention attention.cpp:72-98   same over an index subset, index range check
//   merge             attention.cpp:100-118 identity early-outs are plain copies (bitwise)
//   finalize          attention.cpp:120-127 acc / exp(log_denom)
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "lam_internal.h"

namespace lam {
namespace {

constexpr int kThreads = 256;

template <typename T>
__device__ __forceinline__ T neg_inf();
template <>
__device__ __forceinline__ float neg_inf<float>() {
  return -INFINITY;
}
template <>
__device__ __forceinline__ double neg_inf<double>() {
  return -static_cast<double>(INFINITY);
}

__device__ __forceinline__ float dev_exp(float x) { return expf(x); }
__device__ __forceinline__ double dev_exp(double x) { return exp(x); }
__device__ __forceinline__ float dev_log(float x) { return logf(x); }
__device__ __forceinline__ double dev_log(double x) { return log(x); }

template <typename T>
__device__ T block_reduce(T v, T* scratch, bool is_max) {
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const T o = __shfl_xor_sync(0xffffffffu, v, off);
    v = is_max ? (o > v ? o : v) : v + o;
  }
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kThreads / 32 ? scratch[lane] : (is_max ? neg_inf<T>() : T(0));
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const T o = __shfl_xor_sync(0xffffffffu, v, off);
      v = is_max ? (o > v ? o : v) : v + o;
    }
    if (lane == 0) scratch[32] = v;
  }
  __syncthreads();
  const T r = scratch[32];
  __syncthreads();
  return r;
}

struct InstArgs {
  int64_t n_inst;
  int32_t d;
  const void* q;
  const void* k;
  const void* v;
  const int64_t* kv_row0;
  const int64_t* kv_len;
  const int64_t* idx;      // nullable: all tokens 0..len-1
  const int64_t* idx_off;  // [n+1] when idx != nullptr
  const void* scale;
  void* logits;            // workspace, one T per selected token
  const int64_t* logit_off;  // [n+1] prefix of selected-token counts
  void* acc;               // [n][d]
  void* max_logit;         // nullable (exact mode)
  void* log_denom;         // nullable (exact mode)
  int64_t* count;          // nullable (exact mode)
  int32_t exact;           // 1: write finalized outputs into acc
  int32_t* err;            // device error word: 1 = empty, 2 = index out of range
};

template <typename T>
__global__ void __launch_bounds__(kThreads) instance_kernel(const InstArgs a) {
  __shared__ T scratch[33];
  const int64_t i = blockIdx.x;
  const int d = a.d;
  const T* q = static_cast<const T*>(a.q) + i * d;
  const int64_t row0 = a.kv_row0[i];
  const int64_t len = a.kv_len[i];
  const T* K = static_cast<const T*>(a.k) + row0 * d;
  const T* V = static_cast<const T*>(a.v) + row0 * d;
  const int64_t n = a.idx ? a.idx_off[i + 1] - a.idx_off[i] : len;
  const int64_t* ix = a.idx ? a.idx + a.idx_off[i] : nullptr;
  T* lg = static_cast<T*>(a.logits) + a.logit_off[i];
  T* acc = static_cast<T*>(a.acc) + i * d;
  const T scale = static_cast<const T*>(a.scale)[i];

  if (n == 0) {  // identity partial / empty key set
    for (int e = threadIdx.x; e < d; e += kThreads) acc[e] = T(0);
    if (threadIdx.x == 0) {
      if (a.exact) atomicMax(a.err, 1);
      if (a.max_logit) static_cast<T*>(a.max_logit)[i] = neg_inf<T>();
      if (a.log_denom) static_cast<T*>(a.log_denom)[i] = neg_inf<T>();
      if (a.count) a.count[i] = 0;
    }
    return;
  }

  // pass 1: logits and their max — a warp per token row, lanes over d (coalesced row reads),
  // the dot (attention.cpp:16-21) summed per lane and reduced with xor shuffles
  T mx = neg_inf<T>();
  {
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    for (int64_t k = warp; k < n; k += kThreads / 32) {
      const int64_t j = ix ? ix[k] : k;
      if (j < 0 || j >= len) {
        if (lane == 0) {
          atomicMax(a.err, 2);
          lg[k] = neg_inf<T>();
        }
        continue;
      }
      const T* kr = K + j * d;
      T s = T(0);
      for (int e = lane; e < d; e += 32) s += q[e] * kr[e];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const T x = s * scale;
      if (lane == 0) lg[k] = x;
      mx = x > mx ? x : mx;
    }
  }
  __syncthreads();  // every logit stored before pass 2 reads them by another thread mapping
  mx = block_reduce<T>(mx, scratch, true);

  // pass 2: weights and their sum
  T den = T(0);
  for (int64_t k = threadIdx.x; k < n; k += kThreads) {
    const T w = dev_exp(lg[k] - mx);
    lg[k] = w;
    den += w;
  }
  __syncthreads();  // weights visible to every thread
  den = block_reduce<T>(den, scratch, false);

  // pass 3: p·v, one thread per output dimension, tokens in index order
  for (int e = threadIdx.x; e < d; e += kThreads) {
    T o = T(0);
    for (int64_t k = 0; k < n; ++k) {
      const int64_t j = ix ? ix[k] : k;
      if (j < 0 || j >= len) continue;
      o += lg[k] * V[j * d + e];
    }
    acc[e] = a.exact ? o / den : o;
  }
  if (threadIdx.x == 0 && !a.exact) {
    static_cast<T*>(a.max_logit)[i] = mx;
    static_cast<T*>(a.log_denom)[i] = dev_log(den);
    a.count[i] = n;
  }
}

template <typename T>
__global__ void merge_kernel(int64_t n, int32_t d, const T* a_acc, const T* a_max,
                             const T* a_ld, const int64_t* a_cnt, const T* b_acc,
                             const T* b_max, const T* b_ld, const int64_t* b_cnt, T* o_acc,
                             T* o_max, T* o_ld, int64_t* o_cnt, int32_t* err) {
  const int64_t i = blockIdx.x;
  const bool ae = a_cnt[i] == 0, be = b_cnt[i] == 0;
  if (ae || be) {  // identity early-outs: plain copies keep the other side bitwise
    const T* sa = ae ? b_acc : a_acc;
    const T* sm = ae ? b_max : a_max;
    const T* sl = ae ? b_ld : a_ld;
    const int64_t* sc = ae ? b_cnt : a_cnt;
    for (int e = threadIdx.x; e < d; e += blockDim.x) o_acc[i * d + e] = sa[i * d + e];
    if (threadIdx.x == 0) {
      o_max[i] = sm[i];
      o_ld[i] = sl[i];
      o_cnt[i] = sc[i];
    }
    return;
  }
  const T am = a_max[i], bm = b_max[i];
  const T m = am > bm ? am : bm;
  const T wa = dev_exp(am - m), wb = dev_exp(bm - m);
  for (int e = threadIdx.x; e < d; e += blockDim.x)
    o_acc[i * d + e] = wa * a_acc[i * d + e] + wb * b_acc[i * d + e];
  if (threadIdx.x == 0) {
    o_max[i] = m;
    o_ld[i] = dev_log(wa * dev_exp(a_ld[i]) + wb * dev_exp(b_ld[i]));
    o_cnt[i] = a_cnt[i] + b_cnt[i];
  }
}

template <typename T>
__global__ void finalize_kernel(int64_t n, int32_t d, const T* acc, const T* ld,
                                const int64_t* cnt, T* out, int32_t* err) {
  const int64_t i = blockIdx.x;
  if (cnt[i] == 0) {
    if (threadIdx.x == 0) atomicMax(err, 1);
    return;
  }
  const T den = dev_exp(ld[i]);
  for (int e = threadIdx.x; e < d; e += blockDim.x) out[i * d + e] = acc[i * d + e] / den;
}

// Exclusive prefix sum of per-instance selected-token counts (single CTA, chunked).
__global__ void __launch_bounds__(1024) count_scan_kernel(int64_t n, const int64_t* kv_len,
                                                          const int64_t* idx_off,
                                                          int64_t* off) {
  __shared__ int64_t part[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t c = i < n ? (idx_off ? idx_off[i + 1] - idx_off[i] : kv_len[i]) : 0;
    part[threadIdx.x] = c;
    __syncthreads();
    for (int s = 1; s < 1024; s <<= 1) {  // Hillis-Steele inclusive scan
      const int64_t t = threadIdx.x >= s ? part[threadIdx.x - s] : 0;
      __syncthreads();
      part[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n) off[i + 1] = carry + part[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) off[0] = 0;
}

}  // namespace

cudaError_t launch_count_scan(int64_t n_inst, const int64_t* kv_len, const int64_t* idx_off,
                              int64_t* logit_off, cudaStream_t stream) {
  count_scan_kernel<<<1, 1024, 0, stream>>>(n_inst, kv_len, idx_off, logit_off);
  return cudaGetLastError();
}

cudaError_t launch_instances(int dtype, int64_t n_inst, int32_t d, const void* q, const void* k,
                             const void* v, const int64_t* kv_row0, const int64_t* kv_len,
                             const int64_t* idx, const int64_t* idx_off, const void* scale,
                             void* logits, const int64_t* logit_off, void* acc, void* max_logit,
                             void* log_denom, int64_t* count, int exact, int32_t* err,
                             cudaStream_t stream) {
  if (n_inst == 0) return cudaSuccess;
  InstArgs a{n_inst, d,      q,        k,         v,     kv_row0,  kv_len, idx, idx_off, scale,
             logits, logit_off, acc,    max_logit, log_denom, count, exact, err};
  if (dtype == 1)
    instance_kernel<double><<<static_cast<unsigned>(n_inst), kThreads, 0, stream>>>(a);
  else
    instance_kernel<float><<<static_cast<unsigned>(n_inst), kThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_merge(int dtype, int64_t n, int32_t d, const void* a_acc, const void* a_max,
                         const void* a_ld, const int64_t* a_cnt, const void* b_acc,
                         const void* b_max, const void* b_ld, const int64_t* b_cnt, void* o_acc,
                         void* o_max, void* o_ld, int64_t* o_cnt, int32_t* err,
                         cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const unsigned threads = d >= 128 ? 128 : 32;
  if (dtype == 1)
    merge_kernel<double><<<static_cast<unsigned>(n), threads, 0, stream>>>(
        n, d, static_cast<const double*>(a_acc), static_cast<const double*>(a_max),
        static_cast<const double*>(a_ld), a_cnt, static_cast<const double*>(b_acc),
        static_cast<const double*>(b_max), static_cast<const double*>(b_ld), b_cnt,
        static_cast<double*>(o_acc), static_cast<double*>(o_max), static_cast<double*>(o_ld),
        o_cnt, err);
  else
    merge_kernel<float><<<static_cast<unsigned>(n), threads, 0, stream>>>(
        n, d, static_cast<const float*>(a_acc), static_cast<const float*>(a_max),
        static_cast<const float*>(a_ld), a_cnt, static_cast<const float*>(b_acc),
        static_cast<const float*>(b_max), static_cast<const float*>(b_ld), b_cnt,
        static_cast<float*>(o_acc), static_cast<float*>(o_max), static_cast<float*>(o_ld),
        o_cnt, err);
  return cudaGetLastError();
}

cudaError_t launch_finalize(int dtype, int64_t n, int32_t d, const void* acc, const void* ld,
                            const int64_t* cnt, void* out, int32_t* err, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const unsigned threads = d >= 128 ? 128 : 32;
  if (dtype == 1)
    finalize_kernel<double><<<static_cast<unsigned>(n), threads, 0, stream>>>(
        n, d, static_cast<const double*>(acc), static_cast<const double*>(ld), cnt,
        static_cast<double*>(out), err);
  else
    finalize_kernel<float><<<static_cast<unsigned>(n), threads, 0, stream>>>(
        n, d, static_cast<const float*>(acc), static_cast<const float*>(ld), cnt,
        static_cast<float*>(out), err);
  return cudaGetLastError();
}

}  // namespace lam
