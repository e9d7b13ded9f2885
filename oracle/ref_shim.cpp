// ref_shim.cpp — extern "C" access to the REFERENCE implementation itself
// (/root/reference/proj/core/src/attention.cpp, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libref_attn.so).  TEST INFRASTRUCTURE ONLY: used to pin the
// C restatement (attn_oracle.c), to generate the golden fixtures in tests/golden/, and as the
// timed CPU baseline of bench.py (cpu_baseline / --impl reference).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "disagg/attention.hpp"
#include "generators.hpp"  // reference tests/generators.hpp: gen::random_instance / random_partition

using namespace disagg;

namespace {

template <typename T>
AttnInstance<T> make_inst(int64_t d, int64_t l, const T* q, const T* k, const T* v, T scale) {
  AttnInstance<T> inst;
  inst.query.assign(q, q + d);
  inst.keys.resize(static_cast<size_t>(l));
  inst.values.resize(static_cast<size_t>(l));
  for (int64_t j = 0; j < l; ++j) {
    inst.keys[j].assign(k + j * d, k + (j + 1) * d);
    inst.values[j].assign(v + j * d, v + (j + 1) * d);
  }
  inst.scale = scale;
  return inst;
}

template <typename T>
PartialAttention<T> make_partial(int64_t d, const T* acc, T mx, T ld, int64_t cnt) {
  PartialAttention<T> p;
  p.acc.assign(acc, acc + d);
  p.max_logit = mx;
  p.log_denom = ld;
  p.token_count = cnt;
  return p;
}

template <typename T>
void store_partial(const PartialAttention<T>& p, T* acc, T* mx, T* ld, int64_t* cnt) {
  std::memcpy(acc, p.acc.data(), p.acc.size() * sizeof(T));
  *mx = p.max_logit;
  *ld = p.log_denom;
  *cnt = p.token_count;
}

template <typename T>
int exact(int64_t d, int64_t l, const T* q, const T* k, const T* v, T scale, T* out) {
  try {
    auto r = exact_attention(make_inst(d, l, q, k, v, scale));
    std::memcpy(out, r.data(), r.size() * sizeof(T));
    return 0;
  } catch (const ValidationError&) {
    return 2;
  } catch (const Error&) {
    return 1;
  }
}

template <typename T>
int partial(int64_t d, int64_t l, const T* q, const T* k, const T* v, T scale, const int64_t* idx,
            int64_t n, T* acc, T* mx, T* ld, int64_t* cnt) {
  try {
    auto p = partial_attention<T>(make_inst(d, l, q, k, v, scale),
                                  std::span<const int64_t>(idx, static_cast<size_t>(n)));
    store_partial(p, acc, mx, ld, cnt);
    return 0;
  } catch (const ValidationError&) {
    return 2;
  } catch (const Error&) {
    return 1;
  }
}

template <typename T>
int multi_head(int64_t hq, int64_t hkv, int64_t l, int64_t d, const T* q, const T* k, const T* v,
               T scale, T* out) {
  MultiHeadInstance<T> inst;
  inst.scale = scale;
  for (int64_t h = 0; h < hq; ++h) inst.queries.emplace_back(q + h * d, q + (h + 1) * d);
  for (int64_t h = 0; h < hkv; ++h) {
    std::vector<std::vector<T>> kb, vb;
    for (int64_t t = 0; t < l; ++t) {
      kb.emplace_back(k + (h * l + t) * d, k + (h * l + t + 1) * d);
      vb.emplace_back(v + (h * l + t) * d, v + (h * l + t + 1) * d);
    }
    inst.kv_keys.push_back(kb);
    inst.kv_values.push_back(vb);
  }
  try {
    auto r = multi_head_attention(inst);
    for (int64_t h = 0; h < hq; ++h) std::memcpy(out + h * d, r[h].data(), d * sizeof(T));
    return 0;
  } catch (const ValidationError&) {
    return 2;
  } catch (const Error&) {
    return 1;
  }
}

// CPU baseline: one AttnInstance<float> per (request, kv head) built once, the G query
// vectors of the group swapped in (avoids multi_head_attention's per-head KV deep copy,
// attention.cpp:145-147).  Only exact_attention calls are timed.
struct Bench {
  int32_t B, Hq, Hkv, D;
  std::vector<AttnInstance<float>> units;  // (b, kvh) in unit order
  std::vector<int32_t> unit_b, unit_h;
  std::vector<float> q;                    // [B][Hq][D]
};

}  // namespace

extern "C" {

int ref_exact_f64(int64_t d, int64_t l, const double* q, const double* k, const double* v,
                  double scale, double* out) {
  return exact(d, l, q, k, v, scale, out);
}
int ref_exact_f32(int64_t d, int64_t l, const float* q, const float* k, const float* v,
                  float scale, float* out) {
  return exact(d, l, q, k, v, scale, out);
}
int ref_partial_f64(int64_t d, int64_t l, const double* q, const double* k, const double* v,
                    double scale, const int64_t* idx, int64_t n, double* acc, double* mx,
                    double* ld, int64_t* cnt) {
  return partial(d, l, q, k, v, scale, idx, n, acc, mx, ld, cnt);
}
int ref_partial_f32(int64_t d, int64_t l, const float* q, const float* k, const float* v,
                    float scale, const int64_t* idx, int64_t n, float* acc, float* mx, float* ld,
                    int64_t* cnt) {
  return partial(d, l, q, k, v, scale, idx, n, acc, mx, ld, cnt);
}
void ref_merge_f64(int64_t d, const double* a_acc, double a_mx, double a_ld, int64_t a_cnt,
                   const double* b_acc, double b_mx, double b_ld, int64_t b_cnt, double* o_acc,
                   double* o_mx, double* o_ld, int64_t* o_cnt) {
  auto o = merge(make_partial(d, a_acc, a_mx, a_ld, a_cnt), make_partial(d, b_acc, b_mx, b_ld, b_cnt));
  store_partial(o, o_acc, o_mx, o_ld, o_cnt);
}
void ref_merge_f32(int64_t d, const float* a_acc, float a_mx, float a_ld, int64_t a_cnt,
                   const float* b_acc, float b_mx, float b_ld, int64_t b_cnt, float* o_acc,
                   float* o_mx, float* o_ld, int64_t* o_cnt) {
  auto o = merge(make_partial(d, a_acc, a_mx, a_ld, a_cnt), make_partial(d, b_acc, b_mx, b_ld, b_cnt));
  store_partial(o, o_acc, o_mx, o_ld, o_cnt);
}
int ref_finalize_f64(int64_t d, const double* acc, double ld, int64_t cnt, double* out) {
  try {
    auto r = finalize(make_partial(d, acc, 0.0, ld, cnt));
    std::memcpy(out, r.data(), d * sizeof(double));
    return 0;
  } catch (const Error&) {
    return 1;
  }
}
int ref_multi_head_f64(int64_t hq, int64_t hkv, int64_t l, int64_t d, const double* q,
                       const double* k, const double* v, double scale, double* out) {
  return multi_head(hq, hkv, l, d, q, k, v, scale, out);
}
int ref_multi_head_f32(int64_t hq, int64_t hkv, int64_t l, int64_t d, const float* q,
                       const float* k, const float* v, float scale, float* out) {
  return multi_head(hq, hkv, l, d, q, k, v, scale, out);
}
int ref_head_partition(int64_t nkv, int64_t ndev, int64_t* ranges, char* msg, int64_t msg_len) {
  try {
    auto r = head_partition(nkv, ndev);
    for (size_t i = 0; i < r.size(); ++i) {
      ranges[2 * i] = r[i].begin;
      ranges[2 * i + 1] = r[i].end;
    }
    return 0;
  } catch (const ValidationError& e) {
    std::strncpy(msg, e.what(), static_cast<size_t>(msg_len - 1));
    msg[msg_len - 1] = 0;
    return 2;
  }
}
int ref_request_partition(const double* sizes, int64_t n, int64_t ndev, int64_t* device_of,
                          double* device_load, double* imbalance) {
  try {
    auto a = request_partition(std::span<const double>(sizes, static_cast<size_t>(n)), ndev);
    std::memcpy(device_of, a.device_of.data(), n * sizeof(int64_t));
    std::memcpy(device_load, a.device_load.data(), ndev * sizeof(double));
    *imbalance = a.imbalance;
    return 0;
  } catch (const ValidationError&) {
    return 2;
  }
}

// ---- the reference's own generators (tests/generators.hpp) over a persistent rng ----
void* ref_rng_create(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_destroy(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }
// q[d], k[l*d], v[l*d]
void ref_random_instance(void* r, int64_t d, int64_t l, double limit, double* q, double* k,
                         double* v, double* scale) {
  auto inst = gen::random_instance(*static_cast<std::mt19937_64*>(r), d, l, limit);
  std::memcpy(q, inst.query.data(), d * sizeof(double));
  for (int64_t j = 0; j < l; ++j) {
    std::memcpy(k + j * d, inst.keys[j].data(), d * sizeof(double));
    std::memcpy(v + j * d, inst.values[j].data(), d * sizeof(double));
  }
  *scale = inst.scale;
}
// part_of[t] = part index of token t (the partition's lists are the tokens in order)
void ref_random_partition(void* r, int64_t l, int64_t parts, int64_t* part_of) {
  auto p = gen::random_partition(*static_cast<std::mt19937_64*>(r), l, parts);
  for (size_t i = 0; i < p.size(); ++i)
    for (int64_t t : p[i]) part_of[t] = static_cast<int64_t>(i);
}

// ---- CPU baseline ----
void* ref_bench_create(int32_t B, int32_t Hq, int32_t Hkv, int32_t D, int32_t lmax,
                       const int32_t* lens, const float* q, const float* k, const float* v,
                       float scale, int64_t n_units) {
  auto* bench = new Bench{B, Hq, Hkv, D, {}, {}, {}, {}};
  bench->q.assign(q, q + static_cast<int64_t>(B) * Hq * D);
  const int64_t total = static_cast<int64_t>(B) * Hkv;
  const int64_t n = n_units > 0 && n_units < total ? n_units : total;
  for (int64_t u = 0; u < n; ++u) {
    const int32_t b = static_cast<int32_t>(u / Hkv), h = static_cast<int32_t>(u % Hkv);
    const float* kb = k + (static_cast<int64_t>(b) * Hkv + h) * lmax * D;
    const float* vb = v + (static_cast<int64_t>(b) * Hkv + h) * lmax * D;
    bench->units.push_back(make_inst<float>(D, lens[b], q, kb, vb, scale));
    bench->unit_b.push_back(b);
    bench->unit_h.push_back(h);
  }
  return bench;
}

// Runs every unit's G query heads; returns wall seconds of the compute; out may be null.
double ref_bench_run(void* handle, int32_t nthreads, float* out) {
  auto* bench = static_cast<Bench*>(handle);
  const int32_t G = bench->Hq / bench->Hkv, D = bench->D;
  if (nthreads <= 0) nthreads = static_cast<int32_t>(std::thread::hardware_concurrency());
  std::atomic<int64_t> next{0};
  const int64_t n = static_cast<int64_t>(bench->units.size());
  auto worker = [&]() {
    AttnInstance<float> inst;
    for (int64_t u; (u = next.fetch_add(1)) < n;) {
      auto& unit = bench->units[u];
      const int32_t b = bench->unit_b[u], h = bench->unit_h[u];
      for (int32_t g = 0; g < G; ++g) {
        const int32_t qh = h * G + g;
        const float* qp = bench->q.data() + (static_cast<int64_t>(b) * bench->Hq + qh) * D;
        unit.query.assign(qp, qp + D);
        auto r = exact_attention(unit);
        if (out) std::memcpy(out + (static_cast<int64_t>(b) * bench->Hq + qh) * D, r.data(), D * 4);
      }
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int32_t i = 0; i < nthreads; ++i) th.emplace_back(worker);
  for (auto& t : th) t.join();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

void ref_bench_destroy(void* handle) { delete static_cast<Bench*>(handle); }

int ref_hardware_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
