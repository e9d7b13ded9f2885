// Drop-in definitions of the reference operator API (include/disagg/attention.hpp) on top of
// the B200 C-ABI (include/lamina_attn.h).  Link this object (libdisagg_attention.so) where the
// reference links core/src/attention.cpp; callers do not change.
//
// What stays on the host is what the reference does outside the arithmetic: argument
// validation with the same exception types and messages, index-list construction
// (split_prev_new, attention.cpp:129-139) and marshalling of the nested std::vector rows
// into contiguous buffers.  Every logit, exponential, weighted sum, merge and finalize
// runs in the GPU kernels of paper_2405_01814_b200/csrc/instance.cu.
#include "disagg/attention.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <type_traits>

#include "lamina_attn.h"

namespace disagg {

namespace {

void require(bool ok, const char* what) {
  if (!ok) throw ValidationError(what);
}

// Map a C-ABI status onto the reference exception hierarchy (model.hpp:25-40).
void check(int status) {
  if (status == LAM_OK) return;
  const std::string msg = lam_last_error();
  if (status == LAM_ERR_VALIDATION) throw ValidationError(msg);
  if (status == LAM_ERR_ERROR) throw Error(msg);
  throw Error("GPU attention failed: " + msg);
}

template <typename T>
constexpr int dtype_of() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);
  return std::is_same_v<T, double> ? LAM_F64 : LAM_F32;
}

// Contiguous [rows][d] copy of vector-of-rows blocks (every row must have d entries) into
// library-owned pinned host memory (lam_host_buffer slot), so the rows cross
// PCIe at pinned speed; large blocks are copied by several threads.
template <typename T>
T* pinned_rows(int slot, const std::vector<const std::vector<std::vector<T>>*>& blocks,
               std::size_t d) {
  std::size_t rows = 0;
  for (const auto* b : blocks) {
    for (const auto& r : *b) require(r.size() == d, "key/value rows must match head dim");
    rows += b->size();
  }
  T* dst = static_cast<T*>(lam_host_buffer(slot, static_cast<int64_t>(rows * d * sizeof(T))));
  if (!dst) check(LAM_ERR_CUDA);
  std::vector<std::pair<const std::vector<T>*, T*>> jobs;
  jobs.reserve(rows);
  T* at = dst;
  for (const auto* b : blocks)
    for (const auto& r : *b) {
      jobs.emplace_back(&r, at);
      at += d;
    }
  const std::size_t bytes = rows * d * sizeof(T);
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t nt = bytes < (std::size_t{4} << 20) ? 1 : std::min<std::size_t>(hw, 16);
  auto work = [&](std::size_t t) {
    for (std::size_t i = t; i < jobs.size(); i += nt)
      std::memcpy(jobs[i].second, jobs[i].first->data(), d * sizeof(T));
  };
  std::vector<std::thread> pool;
  for (std::size_t t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return dst;
}

}  // namespace

template <typename T>
void AttnInstance<T>::validate() const {
  require(!query.empty(), "query must be non-empty");
  require(keys.size() == values.size(), "keys and values must have equal row counts");
  for (const auto& row : keys) require(row.size() == query.size(), "key rows must match head dim");
  for (const auto& row : values)
    require(row.size() == query.size(), "value rows must match head dim");
  auto finite = [](const std::vector<T>& v) {
    return std::all_of(v.begin(), v.end(), [](T x) { return std::isfinite(double(x)); });
  };
  require(finite(query), "query entries must be finite");
  for (const auto& row : keys) require(finite(row), "key entries must be finite");
  for (const auto& row : values) require(finite(row), "value entries must be finite");
}

template <typename T>
PartialAttention<T> PartialAttention<T>::identity(std::int64_t head_dim) {
  PartialAttention<T> p;
  p.acc.assign(static_cast<std::size_t>(head_dim), T(0));
  return p;
}

template <typename T>
std::vector<T> exact_attention(const AttnInstance<T>& inst) {
  if (inst.length() == 0) throw Error("exact_attention requires a non-empty key set");
  const std::size_t d = inst.query.size();
  require(d > 0, "query must be non-empty");
  require(inst.values.size() == inst.keys.size(), "keys and values must have equal row counts");
  const T* k = pinned_rows<T>(0, {&inst.keys}, d);
  const T* v = pinned_rows<T>(1, {&inst.values}, d);
  const std::int64_t row0 = 0, len = inst.length();
  std::vector<T> out(d);
  check(lam_exact_attention_host(dtype_of<T>(), 1, static_cast<int32_t>(d), inst.query.data(),
                                 len, k, v, &row0, &len, &inst.scale, out.data()));
  return out;
}

namespace {

// Partials of one instance over several index lists in a single device call.
template <typename T>
std::vector<PartialAttention<T>> partials_of(const AttnInstance<T>& inst,
                                             const std::vector<std::span<const std::int64_t>>& sets) {
  const std::size_t d = inst.query.size();
  require(d > 0, "query must be non-empty");
  require(inst.values.size() == inst.keys.size(), "keys and values must have equal row counts");
  const T* k = pinned_rows<T>(0, {&inst.keys}, d);
  const T* v = pinned_rows<T>(1, {&inst.values}, d);
  const std::size_t n = sets.size();
  std::vector<T> q, scale(n, inst.scale);
  std::vector<std::int64_t> row0(n, 0), len(n, inst.length()), idx, off{0};
  for (const auto& s : sets) {
    q.insert(q.end(), inst.query.begin(), inst.query.end());
    idx.insert(idx.end(), s.begin(), s.end());
    off.push_back(static_cast<std::int64_t>(idx.size()));
  }
  std::vector<T> acc(n * d), mx(n), ld(n);
  std::vector<std::int64_t> cnt(n);
  check(lam_partial_attention_host(dtype_of<T>(), static_cast<int64_t>(n), static_cast<int32_t>(d),
                                   q.data(), inst.length(), k, v, row0.data(),
                                   len.data(), idx.data(), off.data(), scale.data(), acc.data(),
                                   mx.data(), ld.data(), cnt.data()));
  std::vector<PartialAttention<T>> out(n);
  for (std::size_t i = 0; i < n; ++i) {
    out[i].acc.assign(acc.begin() + static_cast<std::ptrdiff_t>(i * d),
                      acc.begin() + static_cast<std::ptrdiff_t>((i + 1) * d));
    out[i].max_logit = mx[i];
    out[i].log_denom = ld[i];
    out[i].token_count = cnt[i];
  }
  return out;
}

}  // namespace

template <typename T>
PartialAttention<T> partial_attention(const AttnInstance<T>& inst,
                                      std::span<const std::int64_t> indices) {
  return partials_of(inst, {indices}).front();
}

template <typename T>
PartialAttention<T> merge(const PartialAttention<T>& a, const PartialAttention<T>& b) {
  if (!a.empty() && !b.empty())
    require(a.acc.size() == b.acc.size(), "partials must share a head dim");
  // The device kernel performs the identity early-outs (attention.cpp:104-105) as copies.
  const std::size_t d = a.empty() ? b.acc.size() : a.acc.size();
  std::vector<T> aa = a.acc, bb = b.acc;
  aa.resize(d, T(0));
  bb.resize(d, T(0));
  PartialAttention<T> o;
  o.acc.resize(d);
  check(lam_merge_host(dtype_of<T>(), 1, static_cast<int32_t>(d), aa.data(), &a.max_logit,
                       &a.log_denom, &a.token_count, bb.data(), &b.max_logit, &b.log_denom,
                       &b.token_count, o.acc.data(), &o.max_logit, &o.log_denom,
                       &o.token_count));
  return o;
}

template <typename T>
std::vector<T> finalize(const PartialAttention<T>& p) {
  if (p.empty()) throw Error("cannot finalize an empty partial");
  std::vector<T> out(p.acc.size());
  check(lam_finalize_host(dtype_of<T>(), 1, static_cast<int32_t>(p.acc.size()), p.acc.data(),
                          &p.log_denom, &p.token_count, out.data()));
  return out;
}

template <typename T>
std::pair<PartialAttention<T>, PartialAttention<T>> split_prev_new(const AttnInstance<T>& inst,
                                                                   std::int64_t boundary) {
  if (boundary < 0 || boundary > inst.length()) throw Error("split boundary out of range");
  std::vector<std::int64_t> prev(static_cast<std::size_t>(boundary));
  std::iota(prev.begin(), prev.end(), std::int64_t{0});
  std::vector<std::int64_t> fresh(static_cast<std::size_t>(inst.length() - boundary));
  std::iota(fresh.begin(), fresh.end(), boundary);
  auto parts = partials_of(inst, {std::span<const std::int64_t>(prev),
                                  std::span<const std::int64_t>(fresh)});
  return {std::move(parts[0]), std::move(parts[1])};
}

template <typename T>
AttnInstance<T> MultiHeadInstance<T>::head_instance(std::int64_t query_head) const {
  const std::int64_t group = num_query_heads() / num_kv_heads();
  AttnInstance<T> inst;
  inst.query = queries[static_cast<std::size_t>(query_head)];
  inst.keys = kv_keys[static_cast<std::size_t>(query_head / group)];
  inst.values = kv_values[static_cast<std::size_t>(query_head / group)];
  inst.scale = scale;
  return inst;
}

template <typename T>
std::vector<std::vector<T>> multi_head_attention(const MultiHeadInstance<T>& inst) {
  require(inst.num_kv_heads() > 0, "need at least one KV head");
  require(inst.num_query_heads() % inst.num_kv_heads() == 0,
          "query heads must be a multiple of KV heads");
  const std::int64_t hq = inst.num_query_heads(), hkv = inst.num_kv_heads();
  std::vector<std::vector<T>> out;
  if (hq == 0) return out;
  const std::size_t d = inst.queries[0].size();
  require(d > 0, "query must be non-empty");
  require(inst.kv_values.size() == inst.kv_keys.size(), "need one value block per KV head");
  // KV rows are laid out once per KV head; q head h points at block h / group, so the GQA
  // mapping costs no copies (the reference deep-copies per head, attention.cpp:145-147).
  std::vector<std::int64_t> block_row0(static_cast<std::size_t>(hkv)),
      block_len(static_cast<std::size_t>(hkv));
  std::vector<const std::vector<std::vector<T>>*> kblocks, vblocks;
  std::int64_t rows = 0;
  for (std::int64_t h = 0; h < hkv; ++h) {
    const auto& kb = inst.kv_keys[static_cast<std::size_t>(h)];
    const auto& vb = inst.kv_values[static_cast<std::size_t>(h)];
    require(kb.size() == vb.size(), "keys and values must have equal row counts");
    block_row0[static_cast<std::size_t>(h)] = rows;
    block_len[static_cast<std::size_t>(h)] = static_cast<std::int64_t>(kb.size());
    if (kb.empty()) throw Error("exact_attention requires a non-empty key set");
    kblocks.push_back(&kb);
    vblocks.push_back(&vb);
    rows += static_cast<std::int64_t>(kb.size());
  }
  const T* k = pinned_rows<T>(0, kblocks, d);
  const T* v = pinned_rows<T>(1, vblocks, d);
  const std::int64_t group = hq / hkv;
  std::vector<T> q, scale(static_cast<std::size_t>(hq), inst.scale);
  std::vector<std::int64_t> row0(static_cast<std::size_t>(hq)), len(static_cast<std::size_t>(hq));
  for (std::int64_t h = 0; h < hq; ++h) {
    const auto& qh = inst.queries[static_cast<std::size_t>(h)];
    require(qh.size() == d, "query heads must share a head dim");
    q.insert(q.end(), qh.begin(), qh.end());
    row0[static_cast<std::size_t>(h)] = block_row0[static_cast<std::size_t>(h / group)];
    len[static_cast<std::size_t>(h)] = block_len[static_cast<std::size_t>(h / group)];
  }
  std::vector<T> flat(static_cast<std::size_t>(hq) * d);
  check(lam_exact_attention_host(dtype_of<T>(), hq, static_cast<int32_t>(d), q.data(), rows,
                                 k, v, row0.data(), len.data(), scale.data(), flat.data()));
  out.reserve(static_cast<std::size_t>(hq));
  for (std::int64_t h = 0; h < hq; ++h)
    out.emplace_back(flat.begin() + static_cast<std::ptrdiff_t>(h * d),
                     flat.begin() + static_cast<std::ptrdiff_t>((h + 1) * d));
  return out;
}

std::vector<HeadRange> head_partition(std::int64_t num_kv_heads, std::int64_t num_devices) {
  std::vector<std::int64_t> r(static_cast<std::size_t>(std::max<std::int64_t>(num_devices, 0)) * 2);
  check(lam_head_partition(num_kv_heads, num_devices, r.data()));
  std::vector<HeadRange> out(static_cast<std::size_t>(num_devices));
  for (std::size_t i = 0; i < out.size(); ++i) out[i] = {r[2 * i], r[2 * i + 1]};
  return out;
}

RequestAssignment request_partition(std::span<const double> kv_sizes, std::int64_t num_devices) {
  RequestAssignment out;
  out.device_of.assign(kv_sizes.size(), 0);
  out.device_load.assign(static_cast<std::size_t>(std::max<std::int64_t>(num_devices, 1)), 0.0);
  check(lam_request_partition(kv_sizes.data(), static_cast<int64_t>(kv_sizes.size()), num_devices,
                              out.device_of.data(), out.device_load.data(), &out.imbalance));
  out.device_load.resize(static_cast<std::size_t>(num_devices));
  return out;
}

// The reference's shipped instantiations (attention.cpp:205-230).
template struct AttnInstance<float>;
template struct AttnInstance<double>;
template struct PartialAttention<float>;
template struct PartialAttention<double>;
template struct MultiHeadInstance<float>;
template struct MultiHeadInstance<double>;

template std::vector<float> exact_attention(const AttnInstance<float>&);
template std::vector<double> exact_attention(const AttnInstance<double>&);
template PartialAttention<float> partial_attention(const AttnInstance<float>&,
                                                   std::span<const std::int64_t>);
template PartialAttention<double> partial_attention(const AttnInstance<double>&,
                                                    std::span<const std::int64_t>);
template PartialAttention<float> merge(const PartialAttention<float>&,
                                       const PartialAttention<float>&);
template PartialAttention<double> merge(const PartialAttention<double>&,
                                        const PartialAttention<double>&);
template std::vector<float> finalize(const PartialAttention<float>&);
template std::vector<double> finalize(const PartialAttention<double>&);
template std::pair<PartialAttention<float>, PartialAttention<float>> split_prev_new(
    const AttnInstance<float>&, std::int64_t);
template std::pair<PartialAttention<double>, PartialAttention<double>> split_prev_new(
    const AttnInstance<double>&, std::int64_t);
template std::vector<std::vector<float>> multi_head_attention(const MultiHeadInstance<float>&);
template std::vector<std::vector<double>> multi_head_attention(const MultiHeadInstance<double>&);

}  // namespace disagg
