// bench_attention_b200.cpp — the reference's attention benchmark
// (/root/reference/proj/benchmarks/bench_attention.cpp:31-47) with device-timed runs added.
//
//   BM_ExactAttention/{d,l}  and  BM_SplitMerge/{l}: the same cases and the same generator
//     (mt19937_64 seed 1, U(-1,1), bench_attention.cpp:11-27), called through the reference
//     API — i.e. the drop-in libdisagg_attention.so, GPU arithmetic, host round trip per call.
//   BM_Decode/{config}: lam_decode (C-ABI) over a device-resident paged KV cache of the
//     BASELINE.json shapes, timed with CUDA events on the launching stream, L2-proof (>= 1 GiB
//     of rotating KV), reported as attn_cost KV GB/s (perf.cpp:77-88).
//
//   BM_MultiHeadAttention/C1: BASELINE config 1 (LLaMA-7B, 32 heads, d = 128, l = 1024, fp32),
//     eight requests, multi_head_attention<float> per request through the reference API.
//
// The same source compiled with -DLAM_BENCH_REFERENCE against the reference's own
// attention.cpp (oracle/Makefile target _ref/bench_attention_ref) times the reference CPU code on
// the same cases, so the two binaries print comparable lines.
//
// google-benchmark is absent in this image (the reference skips its benchmarks then,
// proj/CMakeLists.txt:23-30), so timing is a plain best-of-N loop printing one line per case.
#ifndef LAM_BENCH_REFERENCE
#include <cuda_runtime.h>
#endif

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "disagg/attention.hpp"
#ifndef LAM_BENCH_REFERENCE
#include "lamina_attn.h"
#define LAM_WHO "drop-in, host round trip"
#else
#define LAM_WHO "reference CPU, 1 thread"
#endif

using namespace disagg;

namespace {

AttnInstance<double> make_instance(std::int64_t d_head, std::int64_t l) {
  std::mt19937_64 rng(1);
  auto uniform = [&] { return double(rng() >> 11) * 0x1p-53 * 2 - 1; };
  AttnInstance<double> inst;
  inst.scale = 1.0 / std::sqrt(double(d_head));
  inst.query.resize(size_t(d_head));
  for (auto& x : inst.query) x = uniform();
  inst.keys.resize(size_t(l));
  inst.values.resize(size_t(l));
  for (std::int64_t j = 0; j < l; ++j) {
    inst.keys[size_t(j)].resize(size_t(d_head));
    inst.values[size_t(j)].resize(size_t(d_head));
    for (auto& x : inst.keys[size_t(j)]) x = uniform();
    for (auto& x : inst.values[size_t(j)]) x = uniform();
  }
  return inst;
}

template <class F>
double best_seconds(int reps, F f) {
  double best = 1e300;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    f();
    const auto t1 = std::chrono::steady_clock::now();
    best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
  }
  return best;
}

MultiHeadInstance<float> make_mh(std::int64_t hq, std::int64_t hkv, std::int64_t d_head,
                                 std::int64_t l, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto uniform = [&] { return float(double(rng() >> 11) * 0x1p-53 * 2 - 1); };
  MultiHeadInstance<float> mh;
  mh.scale = 1.0f / std::sqrt(float(d_head));
  mh.queries.assign(size_t(hq), std::vector<float>(size_t(d_head)));
  for (auto& row : mh.queries)
    for (auto& x : row) x = uniform();
  mh.kv_keys.assign(size_t(hkv), std::vector<std::vector<float>>(size_t(l), std::vector<float>(size_t(d_head))));
  mh.kv_values = mh.kv_keys;
  for (auto* kv : {&mh.kv_keys, &mh.kv_values})
    for (auto& head : *kv)
      for (auto& row : head)
        for (auto& x : row) x = uniform();
  return mh;
}

#ifndef LAM_BENCH_REFERENCE
#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

void bench_decode(lam_ctx* ctx, const char* name, int B, int Hq, int Hkv, int L) {
  const int D = 128, P = 64;
  const int pages = B * ((L + P - 1) / P);
  const size_t pool_elems = size_t(pages) * Hkv * P * D;
  const double layer_bytes = 2.0 * pool_elems * 2;
  const int nbuf = std::max(2, int(std::ceil(1.1 * (1 << 30) / layer_bytes)));
  std::vector<void*> kp(nbuf), vp(nbuf);
  for (int i = 0; i < nbuf; ++i) {
    CK(cudaMalloc(&kp[i], pool_elems * 2));
    CK(cudaMalloc(&vp[i], pool_elems * 2));
    CK(cudaMemset(kp[i], 0x3c, pool_elems * 2));  // finite bf16 values
    CK(cudaMemset(vp[i], 0x3c, pool_elems * 2));
  }
  std::vector<int32_t> pt(static_cast<size_t>(pages)), lens(static_cast<size_t>(B), L);
  std::mt19937 rng(7);
  for (int i = 0; i < pages; ++i) pt[size_t(i)] = i;
  std::shuffle(pt.begin(), pt.end(), rng);
  int32_t *d_pt, *d_lens;
  void *d_q, *d_out;
  CK(cudaMalloc(&d_pt, pt.size() * 4));
  CK(cudaMalloc(&d_lens, lens.size() * 4));
  CK(cudaMalloc(&d_q, size_t(B) * Hq * D * 2));
  CK(cudaMalloc(&d_out, size_t(B) * Hq * D * 2));
  CK(cudaMemset(d_q, 0x3c, size_t(B) * Hq * D * 2));
  CK(cudaMemcpy(d_pt, pt.data(), pt.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_lens, lens.data(), lens.size() * 4, cudaMemcpyHostToDevice));
  lam_decode_args a{};
  a.kv_dtype = LAM_BF16;
  a.out_dtype = LAM_BF16;
  a.batch = B;
  a.num_q_heads = Hq;
  a.num_kv_heads = Hkv;
  a.head_dim = D;
  a.scale = 1.0f / std::sqrt(float(D));
  a.page_size = P;
  a.pt_stride = (L + P - 1) / P;
  a.max_len = L;
  a.num_pages = pages;
  a.q = d_q;
  a.page_table = d_pt;
  a.seq_lens = d_lens;
  a.out = d_out;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  auto launch = [&](int i) {
    a.k_pool = kp[i % nbuf];
    a.v_pool = vp[i % nbuf];
    if (lam_decode(ctx, &a, s) != LAM_OK) {
      std::fprintf(stderr, "lam_decode: %s\n", lam_last_error());
      std::exit(1);
    }
  };
  for (int i = 0; i < 5; ++i) launch(i);
  const int iters = 20;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < iters; ++i) launch(i);
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double per = ms / iters * 1e-3;
  const double kv_bytes = 2.0 * 2 * D * Hkv * double(L) * B;  // attn_cost bytes, one layer
  int32_t kernel = 0, splits = 0, chunk = 0;
  lam_decode_plan(ctx, &a, &kernel, &splits, &chunk);
  std::printf("BM_Decode/%-28s %10.1f us  %8.1f GB/s  kernel=%s splits=%d\n", name, per * 1e6,
              kv_bytes / per / 1e9,
              kernel == LAM_KERNEL_GQA_TC ? "gqa_tc" : kernel == LAM_KERNEL_GQA_MMA ? "gqa_mma" : "simt",
              splits);
  for (int i = 0; i < nbuf; ++i) {
    cudaFree(kp[i]);
    cudaFree(vp[i]);
  }
  cudaFree(d_pt);
  cudaFree(d_lens);
  cudaFree(d_q);
  cudaFree(d_out);
  cudaStreamDestroy(s);
}
#endif  // LAM_BENCH_REFERENCE

}  // namespace

int main() {
  // ---- the reference's cases, through the drop-in ----
  for (auto [d, l] : {std::pair<int, int>{64, 256}, {128, 1024}, {128, 8192}}) {
    const auto inst = make_instance(d, l);
    volatile double sink = 0;
    exact_attention(inst);  // warm
    const double t = best_seconds(20, [&] { sink = exact_attention(inst)[0]; });
    std::printf("BM_ExactAttention/%d/%-6d %10.1f us  %8.2f Mitems/s (" LAM_WHO ")\n", d, l,
                t * 1e6, l / t / 1e6);
  }
  for (int l : {256, 4096}) {
    const auto inst = make_instance(128, l);
    volatile double sink = 0;
    const double t = best_seconds(20, [&] {
      auto [prev, fresh] = split_prev_new(inst, l - 1);
      sink = finalize(merge(prev, fresh))[0];
    });
    std::printf("BM_SplitMerge/%-14d %10.1f us  %8.2f Mitems/s (" LAM_WHO ")\n", l, t * 1e6,
                l / t / 1e6);
  }
  {  // BASELINE config 1 through the reference API: 8 requests x multi_head_attention<float>
    std::vector<MultiHeadInstance<float>> reqs;
    for (int b = 0; b < 8; ++b) reqs.push_back(make_mh(32, 32, 128, 1024, 100 + b));
    volatile float sink = 0;
    for (const auto& r : reqs) sink = multi_head_attention(r)[0][0];  // warm
    const double t = best_seconds(5, [&] {
      for (const auto& r : reqs) sink = multi_head_attention(r)[0][0];
    });
    const double kv_bytes = 2.0 * 4 * 128 * 32 * 1024.0 * 8;  // attn_cost bytes, e = 4
    std::printf("BM_MultiHeadAttention/C1          %10.1f us  %8.2f GB/s KV (" LAM_WHO ")\n",
                t * 1e6, kv_bytes / t / 1e9);
  }
#ifndef LAM_BENCH_REFERENCE
  // ---- device-timed decode, BASELINE.json shapes (one layer) ----
  lam_ctx* ctx = nullptr;
  if (lam_ctx_create(0, &ctx) != LAM_OK) {
    std::fprintf(stderr, "no B200: %s\n", lam_last_error());
    return 1;
  }
  bench_decode(ctx, "c2_llama2_7b_B64_l4096", 64, 32, 32, 4096);
  bench_decode(ctx, "c3_llama2_70b_B128_l4096", 128, 64, 8, 4096);
  bench_decode(ctx, "c4_llama2_70b_B32_l32768", 32, 64, 8, 32768);
  lam_ctx_destroy(ctx);
#endif
  return 0;
}
