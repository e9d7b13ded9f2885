// capi.cu — the extern "C" boundary (include/lamina_attn.h): contexts, workspace, planning,
// tensor maps, status codes, and the host-buffer entry points used by the C++ drop-in.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/lamina_attn.h"
#include "decode_common.cuh"
#include "lam_internal.h"

constexpr int kSlots = 4;  // launches that may overlap (programmatic dependent launch)

struct lam_ctx {
  int device = 0;
  int num_sms = 0;
  float* ws_acc = nullptr;
  int64_t ws_acc_cap = 0;  // floats
  float* ws_ml = nullptr;
  int64_t ws_ml_cap = 0;   // floats
  int32_t* counters = nullptr;
  int64_t counters_cap = 0;
  int32_t* err = nullptr;  // device error word for the instance API
  // launch slots of the persistent decode kernels (see DecodeParams::slot): device counters
  // [kSlots][2] and the host's shadow of where each slot's next launch starts
  unsigned long long* slots = nullptr;
  uint64_t item_base[kSlots] = {};
  uint64_t done_base[kSlots] = {};
  uint64_t seq = 0;
  void* scratch = nullptr; // instance API: logits workspace
  int64_t scratch_cap = 0; // bytes
  int64_t* offs = nullptr; // instance API: logit offsets
  int64_t offs_cap = 0;
  // lam_decode_layers_host: device sequence-number flags [in_ready set 0/1, out_ready set 0/1]
  // and the monotonic layer counter that numbers them across calls
  uint32_t* host_flags = nullptr;
  uint32_t host_seq = 0;
  // step launches: finished units per launch lm, per launch slot (zeroed before each launch)
  int32_t* lm_done = nullptr;
  int64_t lm_done_cap = 0;
  // bounded device-side spins of the decode kernels (lam_ctx_status / lam_ctx_set_spin_timeout)
  int32_t* status = nullptr;
  unsigned long long spin_timeout_ns = 10ull * 1000 * 1000 * 1000;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(LAM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define LAM_CUDA(call)                                     \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);    \
  } while (0)

int elem_bytes(int dtype) {
  switch (dtype) {
    case LAM_F32: return 4;
    case LAM_F64: return 8;
    case LAM_BF16: return 2;
    case LAM_F16: return 2;
    default: return 0;
  }
}

template <typename T>
cudaError_t grow(T** ptr, int64_t* cap, int64_t need, bool zero) {
  if (need <= *cap) return cudaSuccess;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  const int64_t n = std::max<int64_t>(need, 1);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), n * sizeof(T));
  if (e != cudaSuccess) return e;
  if (zero) {
    e = cudaMemset(*ptr, 0, n * sizeof(T));
    if (e != cudaSuccess) return e;
  }
  *cap = n;
  return cudaSuccess;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// Makes `device` current for the scope of a C-ABI call and restores the caller's device after.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int device) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != device) err = cudaSetDevice(device);
    else if (err == cudaSuccess) prev = -1;  // nothing to restore
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

#define LAM_DEVICE(ctx)                                               \
  DeviceGuard device_guard_((ctx)->device);                           \
  if (device_guard_.err != cudaSuccess) return cuda_fail(device_guard_.err, "cudaSetDevice")

// ---- driver entry point for tensor maps (no -lcuda link dependency) ----
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D view [rows][D] of a 16-bit pool, 64x64 boxes, 128-byte swizzle.
int make_pool_map(CUtensorMap* map, int dtype, const void* base, int64_t rows, int D,
                  int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(LAM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt =
      dtype == LAM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  // 0 none, 1 64B, 2 128B, 3 256B.  None: the 8 KB boxes are whole 128-byte rows already; in
  // the sustained (power-capped) step it beat 256B by 0.8 % on C3, 0.2 % on C2 (call66.sh)
  static const int promo = env_int("LAM_TMAP_PROMOTION", 0);
  const CUtensorMapL2promotion pr =
      promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                 : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                              : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                           : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(LAM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return LAM_OK;
}

// Kernel variants (decode.cu LAM_MMA_VARIANTS / LAM_SIMT_VARIANTS); variant 0 is the tuned
// default, LAM_GQA_VARIANT / LAM_SIMT_VARIANT override it for tuning.
int gqa_variant() {
  static int v = env_int("LAM_GQA_VARIANT", 0);
  return v;
}
int simt_variant() {
  static int v = env_int("LAM_SIMT_VARIANT", 0);
  return v;
}

struct Plan {
  int kernel = 0;  // LAM_KERNEL_SIMT / LAM_KERNEL_GQA_MMA
  int variant = 0;
  int GQ = 1;      // q heads per CTA
  int QG = 1;      // q-head groups per kv head
  int tile = 32;
  int ctas = 0;    // persistent grid
  int chunk = 0;
  int S = 1;
  int64_t u_head = 0;  // leading units run whole; the rest split S ways (split tail)
};

// Split count and grid size for the persistent kernels, from a small model fitted on B200.
// With dynamic claiming a launch of `items` equal items on `ctas` CTAs runs
// k = ceil(items / ctas) rounds; a partial last round is not measurably faster than a full
// one.  So for a given item count the grid is the smallest one that still needs only
// k = ceil(items / max_ctas) rounds, ctas = ceil(items / k): the rounds are as even as they
// can be, and each CTA streams at min(BW_CHIP / ctas, RATE_SM) (C1: 256 items on 128 CTAs
// beat 143 CTAs by 4 %, experiments/r01/call56.sh).  Every item boundary costs ~C_ITEM; it costs the
// tensor-core kernel more (8 q heads of epilogue per item, split partial and merge round trips).
//   T(S) = k * (item_bytes / min(BW_CHIP / ctas, RATE_SM) + C_ITEM)
// The grid shrinks only by more than 5 %.  Measured choices (call46/47/54/56/57): C1 -> S = 1 on
// 128 CTAs (+3-4 %); C2, C3, C5 -> S = 1; C4 -> S = 4; the sharded GQA launches c3n8
// (512 units) -> S = 1 on 128 CTAs (+1.5 %), c4n8 (128 units) -> S = 1 on 128 CTAs.
void choose_splits(Plan& pl, int64_t units, int max_len, int max_ctas, int split_tokens,
                   double bytes_per_token) {
  static const double BW_CHIP = 7.0e12, RATE_SM = env_int("LAM_PLAN_RATE_SM", 50) * 1e9,
                      C_ITEM_SIMT = env_int("LAM_PLAN_CITEM_NS", 2000) * 1e-9,
                      C_ITEM_MMA = env_int("LAM_PLAN_CITEM_MMA_NS", 5000) * 1e-9;
  const double C_ITEM = pl.kernel == LAM_KERNEL_SIMT ? C_ITEM_SIMT : C_ITEM_MMA;
  const int tiles_total = std::max(1, (max_len + pl.tile - 1) / pl.tile);
  const int occ_per_sm = std::max(1, max_ctas / 148);
  double best = 1e300;
  int best_ct = tiles_total, best_ctas = max_ctas;
  const int s_max = split_tokens > 0 ? 1 : std::min(tiles_total, 64);
  for (int s = 1; s <= s_max; ++s) {
    const int c = split_tokens > 0 ? std::max(1, (split_tokens + pl.tile - 1) / pl.tile)
                                    : (tiles_total + s - 1) / s;
    const int s_eff = (tiles_total + c - 1) / c;
    if (split_tokens <= 0 && s_eff != s) continue;
    const double item_bytes = static_cast<double>(c) * pl.tile * bytes_per_token;
    const int64_t items = std::max<int64_t>(1, units * s_eff);
    const int64_t k = (items + max_ctas - 1) / max_ctas;
    int ctas = static_cast<int>((items + k - 1) / k);
    // shrink only when it evens the rounds out by a margin (C3: 147 CTAs lose 0.6 % to 148);
    // the SIMT kernel with 64-token fp32 tiles keeps the full grid (C1: 148 CTAs 0.878 vs 128
    // CTAs 0.874 of the copy peak, experiments/r02/call84.sh)
    if (ctas > max_ctas * 95 / 100 || (pl.kernel == LAM_KERNEL_SIMT && pl.variant == 7))
      ctas = max_ctas;
    const double rate = std::min(BW_CHIP / ctas, RATE_SM * occ_per_sm);
    const double t = static_cast<double>(k) * (item_bytes / rate + C_ITEM);
    // more splits must win by >= 1.5 % (model noise)
    if (t < best * (1 - 0.015)) {
      best = t;
      best_ct = c;
      best_ctas = ctas;
    }
  }
  pl.chunk = best_ct * pl.tile;
  pl.S = (tiles_total + best_ct - 1) / best_ct;
  pl.ctas = best_ctas;
}

int plan_decode(lam_ctx* ctx, const lam_decode_args* a, Plan* pl) {
  if (!a) return fail(LAM_ERR_VALIDATION, "null decode args");
  const int kvd = a->kv_dtype;
  if (kvd != LAM_F32 && kvd != LAM_BF16 && kvd != LAM_F16)
    return fail(LAM_ERR_VALIDATION, "kv_dtype must be f32, bf16 or f16");
  if (a->out_dtype != kvd && a->out_dtype != LAM_F32)
    return fail(LAM_ERR_VALIDATION, "out_dtype must equal kv_dtype or be f32");
  if (a->batch < 0 || a->num_q_heads < 1 || a->num_kv_heads < 1)
    return fail(LAM_ERR_VALIDATION, "need batch >= 0 and at least one q and kv head");
  if (a->num_q_heads % a->num_kv_heads != 0)
    return fail(LAM_ERR_VALIDATION, "query heads must be a multiple of KV heads");
  if (a->head_dim != 64 && a->head_dim != 128)
    return fail(LAM_ERR_VALIDATION, "head_dim must be 64 or 128 on the decode path");
  if (a->page_size < 1) return fail(LAM_ERR_VALIDATION, "page_size must be >= 1");
  if (a->max_len < 0) return fail(LAM_ERR_VALIDATION, "max_len must be >= 0");
  if (a->q_batch_stride != 0 &&
      (a->q_batch_stride < static_cast<int64_t>(a->num_q_heads) * a->head_dim ||
       (a->q_batch_stride * (kvd == LAM_F32 ? 4 : 2)) % 16 != 0))
    return fail(LAM_ERR_VALIDATION, "q_batch_stride must cover Hq*D and keep 16-byte rows");
  const int G = a->num_q_heads / a->num_kv_heads;
  const bool paged = a->page_table != nullptr;
  if (!paged && a->max_len > a->page_size)
    return fail(LAM_ERR_VALIDATION, "dense layout: max_len exceeds the row capacity page_size");

  const int variant = gqa_variant();
  const int mtile = lam::mma_variant_tile(variant);
  const bool mma_ok = (kvd == LAM_BF16 || kvd == LAM_F16) && a->head_dim == 128 && G >= 1 &&
                      G <= 8 && mtile > 0 && (!paged || a->page_size % mtile == 0);
  const bool tc_ok = (kvd == LAM_BF16 || kvd == LAM_F16) && a->head_dim == 128 && G >= 1 &&
                     G <= 8 && (!paged || a->page_size % lam::kTcBoxRows == 0);
  int kernel = a->kernel;
  // 16-bit KV with D = 128 runs on the tensor-core kernel for every group size, MHA (G = 1)
  // included: both kernels stream at the same rate when timed alone (7226 GB/s, C2), but under
  // a sustained step the SIMT kernel's FMA/shuffle load draws more SM power, the clocks drop
  // further under sw_power_cap (1736-1814 vs 1822-1886 MHz) and the step is 5 % slower
  // (experiments/r01/call49.sh).  LAM_MHA_MMA=0 restores the SIMT kernel for G = 1.
  if (kernel == LAM_KERNEL_AUTO) {
    kernel = mma_ok && (G >= 2 || env_int("LAM_MHA_MMA", 1) != 0) ? LAM_KERNEL_GQA_MMA
                                                                  : LAM_KERNEL_SIMT;
    // The tcgen05 / TMEM kernel wherever it applies.  Same box, sustained steps: C2 (MHA) 7144
    // vs 7062 GB/s per layer launch (its SMs draw less power, so the clocks hold higher under
    // sw_power_cap, experiments/r02/call12.sh); C3 (GQA) step launch 7207 vs 7098 GB/s, and at
    // N = 2 13380 vs 12845 (call22.sh).  LAM_GQA_TC=0 restores the mma.sync kernel.
    if (tc_ok && kernel == LAM_KERNEL_GQA_MMA && env_int("LAM_GQA_TC", 1) != 0)
      kernel = LAM_KERNEL_GQA_TC;
  }
  if (kernel == LAM_KERNEL_GQA_TC) {
    if (!tc_ok)
      return fail(LAM_ERR_VALIDATION,
                  "tcgen05 GQA kernel needs 16-bit KV, head_dim 128, 1 <= G <= 8 and (paged) "
                  "page_size a multiple of 64");
    pl->kernel = kernel;
    pl->variant = 0;
    pl->GQ = 8;
    pl->QG = 1;
    pl->tile = lam::kTcTile;
  } else if (kernel == LAM_KERNEL_GQA_MMA) {
    if (!mma_ok)
      return fail(LAM_ERR_VALIDATION,
                  "GQA MMA kernel needs 16-bit KV, head_dim 128, 1 <= G <= 8 and page_size a "
                  "multiple of its tile (" + std::to_string(mtile) + " tokens)");
    pl->kernel = kernel;
    pl->variant = variant;
    pl->GQ = 8;
    pl->QG = 1;
    pl->tile = mtile;
  } else if (kernel == LAM_KERNEL_SIMT) {
    pl->kernel = kernel;
    pl->GQ = G % 4 == 0 ? 4 : (G % 2 == 0 ? 2 : 1);
    pl->QG = G / pl->GQ;
    pl->variant = (a->head_dim == 128 && pl->GQ == 1) ? simt_variant() : 0;
    // fp32 MHA: 64-token tiles and two 16-byte vectors per lane and row (variant 7) — C1 0.874
    // vs 0.860 of the copy peak, same box (experiments/r02/call84.sh); needs 64-token pages
    if (pl->variant == 0 && kvd == LAM_F32 && a->head_dim == 128 && pl->GQ == 1 &&
        (!paged || a->page_size % 64 == 0))
      pl->variant = 7;
    pl->tile = lam::simt_variant_tile(kvd, a->head_dim, pl->GQ, pl->variant);
    if (pl->tile == 0) return fail(LAM_ERR_VALIDATION, "unsupported SIMT decode shape");
    if (paged && a->page_size % pl->tile != 0)
      return fail(LAM_ERR_VALIDATION, "paged layout needs page_size a multiple of " +
                                          std::to_string(pl->tile) + " tokens");
  } else {
    return fail(LAM_ERR_VALIDATION, "unknown kernel family");
  }
  const int occ = pl->kernel == LAM_KERNEL_GQA_MMA  ? lam::occupancy_mma(kvd, pl->variant)
                  : pl->kernel == LAM_KERNEL_GQA_TC ? lam::occupancy_tc(kvd)
                                                    : lam::occupancy_simt(kvd, a->head_dim, pl->GQ, pl->variant);
  if (occ <= 0) return fail(LAM_ERR_CUDA, "decode kernel cannot be resident on this device");
  const int64_t units = static_cast<int64_t>(a->batch) * a->num_kv_heads * pl->QG;
  choose_splits(*pl, units, a->max_len, occ * ctx->num_sms, a->split_tokens,
                2.0 * a->head_dim * (kvd == LAM_F32 ? 4 : 2));
  if (const int force = env_int("LAM_DECODE_CTAS", 0); force > 0)
    pl->ctas = std::min(force, occ * ctx->num_sms);
  // split tail (experiment knobs): the last `tail` units split `ts` ways
  if (const int tail = env_int("LAM_TAIL_UNITS", 0); tail > 0 && pl->S == 1 && a->split_tokens <= 0) {
    const int ts = std::max(2, env_int("LAM_TAIL_SPLITS", 4));
    const int tiles_total = std::max(1, (a->max_len + pl->tile - 1) / pl->tile);
    const int ct = (tiles_total + ts - 1) / ts;
    pl->S = (tiles_total + ct - 1) / ct;
    pl->chunk = ct * pl->tile;
    if (pl->S > 1) pl->u_head = std::max<int64_t>(0, units - tail);
  }
  if (pl->S > 65535) return fail(LAM_ERR_VALIDATION, "too many splits");
  return LAM_OK;
}

// per-thread context + staging for the host-buffer entry points
struct HostStage {
  lam_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  int32_t* err = nullptr;  // pinned: the instance kernels' error word, read after the sync
  std::vector<void*> bufs;
  std::vector<int64_t> caps;
  ~HostStage() {
    if (err) cudaFreeHost(err);
    for (void* p : bufs)
      if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
    if (ctx) lam_ctx_destroy(ctx);
  }
  int init() {
    if (ctx) return LAM_OK;
    int dev = 0;
    LAM_CUDA(cudaGetDevice(&dev));
    int rc = lam_ctx_create(dev, &ctx);
    if (rc != LAM_OK) return rc;
    LAM_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    LAM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&err), sizeof(int32_t), cudaHostAllocDefault));
    return LAM_OK;
  }
  // buffer slot i with at least `bytes`
  int get(size_t i, int64_t bytes, void** out) {
    if (bufs.size() <= i) {
      bufs.resize(i + 1, nullptr);
      caps.resize(i + 1, 0);
    }
    if (caps[i] < bytes) {
      if (bufs[i]) cudaFree(bufs[i]);
      bufs[i] = nullptr;
      caps[i] = 0;
      LAM_CUDA(cudaMalloc(&bufs[i], std::max<int64_t>(bytes, 16)));
      caps[i] = std::max<int64_t>(bytes, 16);
    }
    *out = bufs[i];
    return LAM_OK;
  }
};

// per-thread pinned host buffers (lam_host_buffer)
struct PinnedSlots {
  void* ptr[4] = {};
  int64_t cap[4] = {};
  ~PinnedSlots() {
    for (void* p : ptr)
      if (p) cudaFreeHost(p);
  }
};
thread_local PinnedSlots g_pinned;

// one staging area (and context) per device and thread: a thread that moves between devices
// stages and launches on the device that is current at each call
HostStage& host_stage() {
  thread_local std::vector<std::unique_ptr<HostStage>> stages;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  if (static_cast<size_t>(dev) >= stages.size()) stages.resize(dev + 1);
  if (!stages[dev]) stages[dev] = std::make_unique<HostStage>();
  return *stages[dev];
}

int check_err_word(lam_ctx* ctx, cudaStream_t stream, const char* empty_msg) {
  int32_t h = 0;
  LAM_CUDA(cudaMemcpyAsync(&h, ctx->err, sizeof(h), cudaMemcpyDeviceToHost, stream));
  LAM_CUDA(cudaStreamSynchronize(stream));
  if (h == 2) return fail(LAM_ERR_ERROR, "token index out of range");
  if (h == 1) return fail(LAM_ERR_ERROR, empty_msg);
  return LAM_OK;
}

// host_total >= 0: the caller knows the logit count (the host-buffer entry points sum the
// lengths on the host), so the scan's result is not read back; err_out != null: the error word
// is copied there asynchronously and the caller checks it after its own synchronisation.
// Together they leave one host synchronisation per host-buffer call instead of three.
int run_instances(lam_ctx* ctx, int dtype, int64_t n_inst, int32_t d, const void* q,
                  const void* k, const void* v, const int64_t* kv_row0, const int64_t* kv_len,
                  const int64_t* idx, const int64_t* idx_off, const void* scale, void* acc,
                  void* max_logit, void* log_denom, int64_t* count, int exact,
                  cudaStream_t stream, int64_t host_total = -1, int32_t* err_out = nullptr) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  if (dtype != LAM_F32 && dtype != LAM_F64)
    return fail(LAM_ERR_VALIDATION, "instance API supports f32 and f64");
  if (d < 1) return fail(LAM_ERR_VALIDATION, "query must be non-empty");
  if (n_inst < 0) return fail(LAM_ERR_VALIDATION, "negative instance count");
  if (n_inst == 0) return LAM_OK;
  LAM_DEVICE(ctx);
  LAM_CUDA(grow(&ctx->offs, &ctx->offs_cap, n_inst + 1, false));
  LAM_CUDA(lam::launch_count_scan(n_inst, kv_len, exact ? nullptr : idx_off, ctx->offs, stream));
  int64_t total = host_total;
  if (total < 0) {
    LAM_CUDA(cudaMemcpyAsync(&total, ctx->offs + n_inst, sizeof(total), cudaMemcpyDeviceToHost,
                             stream));
    LAM_CUDA(cudaStreamSynchronize(stream));
  }
  const int64_t need = std::max<int64_t>(total, 1) * elem_bytes(dtype);
  if (ctx->scratch_cap < need) {
    if (ctx->scratch) cudaFree(ctx->scratch);
    ctx->scratch = nullptr;
    ctx->scratch_cap = 0;
    LAM_CUDA(cudaMalloc(&ctx->scratch, need));
    ctx->scratch_cap = need;
  }
  LAM_CUDA(cudaMemsetAsync(ctx->err, 0, sizeof(int32_t), stream));
  LAM_CUDA(lam::launch_instances(dtype, n_inst, d, q, k, v, kv_row0, kv_len, exact ? nullptr : idx,
                                 exact ? nullptr : idx_off, scale, ctx->scratch, ctx->offs, acc,
                                 max_logit, log_denom, count, exact, ctx->err, stream));
  if (err_out != nullptr) {
    LAM_CUDA(cudaMemcpyAsync(err_out, ctx->err, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    return LAM_OK;
  }
  return check_err_word(ctx, stream, "exact_attention requires a non-empty key set");
}

// The deferred error word of run_instances(err_out), after the caller's synchronisation.
int deferred_err(int32_t h) {
  if (h == 2) return fail(LAM_ERR_ERROR, "token index out of range");
  if (h == 1) return fail(LAM_ERR_ERROR, "exact_attention requires a non-empty key set");
  return LAM_OK;
}

}  // namespace

extern "C" {

int lam_version(void) { return 1; }

const char* lam_last_error(void) { return g_last_error.c_str(); }

void* lam_host_buffer(int32_t slot, int64_t bytes) {
  if (slot < 0 || slot >= 4 || bytes < 0) {
    fail(LAM_ERR_VALIDATION, "lam_host_buffer: slot must be 0..3 and bytes >= 0");
    return nullptr;
  }
  if (bytes > g_pinned.cap[slot]) {
    if (g_pinned.ptr[slot]) cudaFreeHost(g_pinned.ptr[slot]);
    g_pinned.ptr[slot] = nullptr;
    g_pinned.cap[slot] = 0;
    const int64_t want = std::max<int64_t>(bytes + bytes / 4, 1 << 20);  // grow with slack
    void* p = nullptr;
    const cudaError_t e = cudaHostAlloc(&p, static_cast<size_t>(want), cudaHostAllocPortable);
    if (e != cudaSuccess) {
      cuda_fail(e, "cudaHostAlloc");
      return nullptr;
    }
    g_pinned.ptr[slot] = p;
    g_pinned.cap[slot] = want;
  }
  return g_pinned.ptr[slot];
}

int lam_ctx_create(int device, lam_ctx** out) {
  if (!out) return fail(LAM_ERR_VALIDATION, "null output pointer");
  *out = nullptr;
  int n = 0;
  LAM_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(LAM_ERR_VALIDATION, "no such CUDA device");
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  int major = 0;
  LAM_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major < 10) return fail(LAM_ERR_CUDA, "liblamina_attn is built for sm_100a (B200) only");
  auto* c = new lam_ctx();
  c->device = device;
  cudaError_t e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&c->err, sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->slots, kSlots * 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->slots, 0, kSlots * 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&c->status, sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemset(c->status, 0, sizeof(int32_t));
  if (const char* t = std::getenv("LAM_SPIN_TIMEOUT_MS"))
    c->spin_timeout_ns = static_cast<unsigned long long>(std::max(0.0, std::atof(t)) * 1e6);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "lam_ctx_create");
  }
  *out = c;
  return LAM_OK;
}

int lam_ctx_destroy(lam_ctx* c) {
  if (!c) return LAM_OK;
  DeviceGuard guard(c->device);
  cudaFree(c->status);
  cudaFree(c->ws_acc);
  cudaFree(c->ws_ml);
  cudaFree(c->counters);
  cudaFree(c->err);
  cudaFree(c->slots);
  cudaFree(c->scratch);
  cudaFree(c->offs);
  cudaFree(c->host_flags);
  cudaFree(c->lm_done);
  delete c;
  return LAM_OK;
}

int lam_ctx_num_sms(const lam_ctx* c) { return c ? c->num_sms : 0; }

int lam_ctx_set_spin_timeout(lam_ctx* c, int64_t timeout_ns) {
  if (!c || timeout_ns < 0) return fail(LAM_ERR_VALIDATION, "bad spin timeout");
  c->spin_timeout_ns = static_cast<unsigned long long>(timeout_ns);
  return LAM_OK;
}

int lam_ctx_status(lam_ctx* c, int32_t* status, int32_t clear) {
  if (!c || !status) return fail(LAM_ERR_VALIDATION, "null context or status");
  LAM_DEVICE(c);
  LAM_CUDA(cudaDeviceSynchronize());
  LAM_CUDA(cudaMemcpy(status, c->status, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (clear) LAM_CUDA(cudaMemset(c->status, 0, sizeof(int32_t)));
  return LAM_OK;
}

int lam_ctx_reserve(lam_ctx* c, int64_t partial_rows, int32_t head_dim, int64_t counters) {
  if (!c) return fail(LAM_ERR_VALIDATION, "null context");
  LAM_DEVICE(c);
  // every launch slot has its own split workspace (capacities are per slot)
  if (partial_rows * head_dim > c->ws_acc_cap) {
    int64_t cap = 0;
    LAM_CUDA(grow(&c->ws_acc, &cap, kSlots * partial_rows * head_dim, false));
    c->ws_acc_cap = partial_rows * head_dim;
  }
  if (partial_rows * 2 > c->ws_ml_cap) {
    int64_t cap = 0;
    LAM_CUDA(grow(&c->ws_ml, &cap, kSlots * partial_rows * 2, false));
    c->ws_ml_cap = partial_rows * 2;
  }
  if (counters > c->counters_cap) {
    int64_t cap = 0;
    LAM_CUDA(grow(&c->counters, &cap, kSlots * counters, true));
    c->counters_cap = counters;
  }
  return LAM_OK;
}

// ---------------- instance API (device pointers) ----------------

int lam_exact_attention(lam_ctx* ctx, int dtype, int64_t n_inst, int32_t d, const void* q,
                        const void* k_rows, const void* v_rows, const int64_t* kv_row0,
                        const int64_t* kv_len, const void* scale, void* out, void* stream) {
  return run_instances(ctx, dtype, n_inst, d, q, k_rows, v_rows, kv_row0, kv_len, nullptr,
                       nullptr, scale, out, nullptr, nullptr, nullptr, 1,
                       static_cast<cudaStream_t>(stream));
}

int lam_partial_attention(lam_ctx* ctx, int dtype, int64_t n_inst, int32_t d, const void* q,
                          const void* k_rows, const void* v_rows, const int64_t* kv_row0,
                          const int64_t* kv_len, const int64_t* idx, const int64_t* idx_off,
                          const void* scale, void* acc, void* max_logit, void* log_denom,
                          int64_t* token_count, void* stream) {
  if (!idx_off) return fail(LAM_ERR_VALIDATION, "partial_attention needs idx_off");
  return run_instances(ctx, dtype, n_inst, d, q, k_rows, v_rows, kv_row0, kv_len, idx, idx_off,
                       scale, acc, max_logit, log_denom, token_count, 0,
                       static_cast<cudaStream_t>(stream));
}

int lam_merge(lam_ctx* ctx, int dtype, int64_t n, int32_t d, const void* a_acc,
              const void* a_max, const void* a_log_denom, const int64_t* a_count,
              const void* b_acc, const void* b_max, const void* b_log_denom,
              const int64_t* b_count, void* o_acc, void* o_max, void* o_log_denom,
              int64_t* o_count, void* stream) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  if (dtype != LAM_F32 && dtype != LAM_F64)
    return fail(LAM_ERR_VALIDATION, "merge supports f32 and f64");
  if (d < 0 || n < 0) return fail(LAM_ERR_VALIDATION, "negative size");
  LAM_DEVICE(ctx);
  auto s = static_cast<cudaStream_t>(stream);
  LAM_CUDA(lam::launch_merge(dtype, n, d, a_acc, a_max, a_log_denom, a_count, b_acc, b_max,
                             b_log_denom, b_count, o_acc, o_max, o_log_denom, o_count, ctx->err,
                             s));
  return LAM_OK;
}

int lam_finalize(lam_ctx* ctx, int dtype, int64_t n, int32_t d, const void* acc,
                 const void* log_denom, const int64_t* count, void* out, void* stream) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  if (dtype != LAM_F32 && dtype != LAM_F64)
    return fail(LAM_ERR_VALIDATION, "finalize supports f32 and f64");
  LAM_DEVICE(ctx);
  auto s = static_cast<cudaStream_t>(stream);
  LAM_CUDA(cudaMemsetAsync(ctx->err, 0, sizeof(int32_t), s));
  LAM_CUDA(lam::launch_finalize(dtype, n, d, acc, log_denom, count, out, ctx->err, s));
  return check_err_word(ctx, s, "cannot finalize an empty partial");
}

// ---------------- instance API (host pointers) ----------------

namespace {
struct HostCopy {
  const void* host;
  int64_t bytes;
};
// Stage `n` host arrays into per-thread device slots starting at `slot0`.
int stage_in(int slot0, std::initializer_list<HostCopy> items, std::vector<void*>& dev) {
  int i = slot0;
  for (const auto& it : items) {
    void* d = nullptr;
    int rc = host_stage().get(i++, it.bytes, &d);
    if (rc != LAM_OK) return rc;
    if (it.host && it.bytes > 0)
      LAM_CUDA(cudaMemcpyAsync(d, it.host, it.bytes, cudaMemcpyHostToDevice, host_stage().stream));
    dev.push_back(d);
  }
  return LAM_OK;
}
}  // namespace

int lam_exact_attention_host(int dtype, int64_t n_inst, int32_t d, const void* q, int64_t n_rows,
                             const void* k_rows, const void* v_rows, const int64_t* kv_row0,
                             const int64_t* kv_len, const void* scale, void* out) {
  int rc = host_stage().init();
  if (rc != LAM_OK) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0) return fail(LAM_ERR_VALIDATION, "bad dtype");
  if (n_inst <= 0) return LAM_OK;
  std::vector<void*> dv;
  rc = stage_in(0,
                {{q, n_inst * d * e},
                 {k_rows, n_rows * d * e},
                 {v_rows, n_rows * d * e},
                 {kv_row0, n_inst * 8},
                 {kv_len, n_inst * 8},
                 {scale, n_inst * e},
                 {nullptr, n_inst * d * e}},
                dv);
  if (rc != LAM_OK) return rc;
  int64_t total = 0;  // logits the kernel stores (the host knows the lengths)
  for (int64_t i = 0; i < n_inst && total >= 0; ++i) total = kv_len[i] < 0 ? -1 : total + kv_len[i];
  HostStage& hs = host_stage();
  rc = run_instances(hs.ctx, dtype, n_inst, d, dv[0], dv[1], dv[2], static_cast<int64_t*>(dv[3]),
                     static_cast<int64_t*>(dv[4]), nullptr, nullptr, dv[5], dv[6], nullptr,
                     nullptr, nullptr, 1, hs.stream, total, hs.err);
  if (rc != LAM_OK) return rc;
  LAM_CUDA(cudaMemcpyAsync(out, dv[6], n_inst * d * e, cudaMemcpyDeviceToHost, hs.stream));
  LAM_CUDA(cudaStreamSynchronize(hs.stream));
  return deferred_err(*hs.err);
}

int lam_partial_attention_host(int dtype, int64_t n_inst, int32_t d, const void* q,
                               int64_t n_rows, const void* k_rows, const void* v_rows,
                               const int64_t* kv_row0, const int64_t* kv_len,
                               const int64_t* idx, const int64_t* idx_off, const void* scale,
                               void* acc, void* max_logit, void* log_denom,
                               int64_t* token_count) {
  int rc = host_stage().init();
  if (rc != LAM_OK) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0) return fail(LAM_ERR_VALIDATION, "bad dtype");
  if (n_inst <= 0) return LAM_OK;
  const int64_t n_idx = idx_off[n_inst];
  std::vector<void*> dv;
  rc = stage_in(0,
                {{q, n_inst * d * e},
                 {k_rows, n_rows * d * e},
                 {v_rows, n_rows * d * e},
                 {kv_row0, n_inst * 8},
                 {kv_len, n_inst * 8},
                 {idx, n_idx * 8},
                 {idx_off, (n_inst + 1) * 8},
                 {scale, n_inst * e},
                 {nullptr, n_inst * d * e},
                 {nullptr, n_inst * e},
                 {nullptr, n_inst * e},
                 {nullptr, n_inst * 8}},
                dv);
  if (rc != LAM_OK) return rc;
  int64_t total = 0;  // index entries: the logits the kernel stores
  for (int64_t i = 0; i < n_inst && total >= 0; ++i)
    total = idx_off[i + 1] < idx_off[i] ? -1 : total + (idx_off[i + 1] - idx_off[i]);
  HostStage& hs = host_stage();
  rc = run_instances(hs.ctx, dtype, n_inst, d, dv[0], dv[1], dv[2], static_cast<int64_t*>(dv[3]),
                     static_cast<int64_t*>(dv[4]), static_cast<int64_t*>(dv[5]),
                     static_cast<int64_t*>(dv[6]), dv[7], dv[8], dv[9], dv[10],
                     static_cast<int64_t*>(dv[11]), 0, hs.stream, total, hs.err);
  if (rc != LAM_OK) return rc;
  auto s = hs.stream;
  LAM_CUDA(cudaMemcpyAsync(acc, dv[8], n_inst * d * e, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaMemcpyAsync(max_logit, dv[9], n_inst * e, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaMemcpyAsync(log_denom, dv[10], n_inst * e, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaMemcpyAsync(token_count, dv[11], n_inst * 8, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaStreamSynchronize(s));
  return deferred_err(*hs.err);
}

int lam_merge_host(int dtype, int64_t n, int32_t d, const void* a_acc, const void* a_max,
                   const void* a_log_denom, const int64_t* a_count, const void* b_acc,
                   const void* b_max, const void* b_log_denom, const int64_t* b_count,
                   void* o_acc, void* o_max, void* o_log_denom, int64_t* o_count) {
  int rc = host_stage().init();
  if (rc != LAM_OK) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0) return fail(LAM_ERR_VALIDATION, "bad dtype");
  if (n <= 0) return LAM_OK;
  std::vector<void*> dv;
  rc = stage_in(0,
                {{a_acc, n * d * e},
                 {a_max, n * e},
                 {a_log_denom, n * e},
                 {a_count, n * 8},
                 {b_acc, n * d * e},
                 {b_max, n * e},
                 {b_log_denom, n * e},
                 {b_count, n * 8},
                 {nullptr, n * d * e},
                 {nullptr, n * e},
                 {nullptr, n * e},
                 {nullptr, n * 8}},
                dv);
  if (rc != LAM_OK) return rc;
  rc = lam_merge(host_stage().ctx, dtype, n, d, dv[0], dv[1], dv[2], static_cast<int64_t*>(dv[3]),
                 dv[4], dv[5], dv[6], static_cast<int64_t*>(dv[7]), dv[8], dv[9], dv[10],
                 static_cast<int64_t*>(dv[11]), host_stage().stream);
  if (rc != LAM_OK) return rc;
  auto s = host_stage().stream;
  LAM_CUDA(cudaMemcpyAsync(o_acc, dv[8], n * d * e, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaMemcpyAsync(o_max, dv[9], n * e, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaMemcpyAsync(o_log_denom, dv[10], n * e, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaMemcpyAsync(o_count, dv[11], n * 8, cudaMemcpyDeviceToHost, s));
  LAM_CUDA(cudaStreamSynchronize(s));
  return LAM_OK;
}

int lam_finalize_host(int dtype, int64_t n, int32_t d, const void* acc, const void* log_denom,
                      const int64_t* count, void* out) {
  int rc = host_stage().init();
  if (rc != LAM_OK) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0) return fail(LAM_ERR_VALIDATION, "bad dtype");
  if (n <= 0) return LAM_OK;
  std::vector<void*> dv;
  rc = stage_in(0, {{acc, n * d * e}, {log_denom, n * e}, {count, n * 8}, {nullptr, n * d * e}},
                dv);
  if (rc != LAM_OK) return rc;
  rc = lam_finalize(host_stage().ctx, dtype, n, d, dv[0], dv[1], static_cast<int64_t*>(dv[2]), dv[3],
                    host_stage().stream);
  if (rc != LAM_OK) return rc;
  LAM_CUDA(cudaMemcpyAsync(out, dv[3], n * d * e, cudaMemcpyDeviceToHost, host_stage().stream));
  LAM_CUDA(cudaStreamSynchronize(host_stage().stream));
  return LAM_OK;
}

// ---------------- partitioning (host logic) ----------------

int lam_head_partition(int64_t num_kv_heads, int64_t num_devices, int64_t* ranges) {
  if (num_kv_heads < 1) return fail(LAM_ERR_VALIDATION, "num_kv_heads must be >= 1");
  if (num_devices < 1) return fail(LAM_ERR_VALIDATION, "num_devices must be >= 1");
  if (num_kv_heads % num_devices != 0)
    return fail(LAM_ERR_VALIDATION,
                "head partition requires num_kv_heads divisible by num_devices (" +
                    std::to_string(num_kv_heads) + " % " + std::to_string(num_devices) +
                    " != 0)");
  const int64_t per = num_kv_heads / num_devices;
  for (int64_t i = 0; i < num_devices; ++i) {
    ranges[2 * i] = i * per;
    ranges[2 * i + 1] = (i + 1) * per;
  }
  return LAM_OK;
}

int lam_request_partition(const double* kv_sizes, int64_t n, int64_t num_devices,
                          int64_t* device_of, double* device_load, double* imbalance) {
  if (num_devices < 1) return fail(LAM_ERR_VALIDATION, "num_devices must be >= 1");
  for (int64_t i = 0; i < n; ++i) device_of[i] = 0;
  for (int64_t d = 0; d < num_devices; ++d) device_load[d] = 0.0;
  std::vector<int64_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return kv_sizes[a] > kv_sizes[b]; });
  for (int64_t r : order) {
    int64_t t = 0;
    for (int64_t d = 1; d < num_devices; ++d)
      if (device_load[d] < device_load[t]) t = d;
    device_of[r] = t;
    device_load[t] += kv_sizes[r];
  }
  double total = 0, peak = device_load[0];
  for (int64_t d = 0; d < num_devices; ++d) {
    total += device_load[d];
    peak = std::max(peak, device_load[d]);
  }
  const double mean = total / static_cast<double>(num_devices);
  *imbalance = mean > 0 ? peak / mean : 1.0;
  return LAM_OK;
}

// ---------------- production decode path ----------------

int lam_decode_plan(lam_ctx* ctx, const lam_decode_args* a, int32_t* kernel, int32_t* num_splits,
                    int32_t* split_tokens) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  LAM_DEVICE(ctx);
  Plan pl;
  int rc = plan_decode(ctx, a, &pl);
  if (rc != LAM_OK) return rc;
  if (kernel) *kernel = pl.kernel;
  if (num_splits) *num_splits = pl.S;
  if (split_tokens) *split_tokens = pl.chunk;
  return LAM_OK;
}

int lam_decode_plan_grid(lam_ctx* ctx, const lam_decode_args* a, int32_t* ctas) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  LAM_DEVICE(ctx);
  Plan pl;
  int rc = plan_decode(ctx, a, &pl);
  if (rc != LAM_OK) return rc;
  if (ctas) *ctas = pl.ctas;
  return LAM_OK;
}

namespace {

int decode_impl(lam_ctx* ctx, const lam_decode_args* a_in, const lam_peer_io* io,
                const lam_step_layout* st, void* stream) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  LAM_DEVICE(ctx);
  lam_decode_args a_step;
  const lam_decode_args* a = a_in;
  int n_lm = 1;
  if (st != nullptr) {  // plan one launch lm: rows_per_mb requests
    if (st->n_layers < 1 || st->n_mb < 1 || st->rows_per_mb < 1 ||
        static_cast<int64_t>(st->n_mb) * st->rows_per_mb != a_in->batch)
      return fail(LAM_ERR_VALIDATION, "step: need n_layers, n_mb, rows_per_mb >= 1 and batch == "
                                      "n_mb * rows_per_mb");
    if (st->pool_layers < 1 || st->layer0 < 0 || st->pool_layer_rows < 0)
      return fail(LAM_ERR_VALIDATION, "step: bad pool layer layout");
    if (a_in->lse != nullptr) return fail(LAM_ERR_VALIDATION, "step: lse is not supported");
    if (io != nullptr && io->row_src == nullptr && io->rows_per_src * io->n_src != st->rows_per_mb)
      return fail(LAM_ERR_VALIDATION, "step: peer io must describe one micro-batch's rows");
    a_step = *a_in;
    a_step.batch = st->rows_per_mb;
    a = &a_step;
    n_lm = st->n_layers * st->n_mb;
    if (a_in->split_tokens <= 0) {
      // Splits: without input dependencies the whole step is one pool of items and S = 1 (fewest
      // merges).  When every launch lm waits for inputs that follow the previous layer's
      // outputs, a launch's latency is its longest item, so items are capped at 8 K tokens
      // (LAM_STEP_ITEM_TOKENS; C4's 32 K-token requests -> S = 4, C5's 16 K ones -> 2).
      // Splitting further to give each launch >= 2 rounds of items on its share of the grid
      // measured slower everywhere: the tcgen05 kernel's per-item cost outweighs the rounding
      // (C3 at N = 4: 4958 vs 6106 GB/s per GPU; item caps of 4 K / 16 K tokens: C4 6667 / 5414,
      // C5 5113 / 4128 vs 6802 and 5486 at 8 K; round 2, calls 59-61).
      a_step.split_tokens = std::max(1, a_in->max_len);
      Plan p1;
      int rc1 = plan_decode(ctx, &a_step, &p1);
      if (rc1 != LAM_OK) return rc1;
      if (io != nullptr && io->n_wait > 0) {
        const int tiles = std::max(1, (a_in->max_len + p1.tile - 1) / p1.tile);
        const int max_tok = env_int("LAM_STEP_ITEM_TOKENS", 8192);
        int S = 1;
        while ((a_in->max_len + S - 1) / S > max_tok && S * 2 <= tiles) S *= 2;
        if (const int force = env_int("LAM_STEP_SPLITS", 0); force > 0) S = std::min(force, tiles);
        const int ct = (tiles + S - 1) / S;
        a_step.split_tokens = ct * p1.tile;
      }
    }
  }
  Plan pl;
  int rc = plan_decode(ctx, a, &pl);
  if (rc != LAM_OK) return rc;
  if (a->batch == 0) return LAM_OK;
  if (st != nullptr) {  // the items of every launch lm share one grid: all resident CTAs
    const int occ = pl.kernel == LAM_KERNEL_GQA_TC    ? lam::occupancy_tc(a->kv_dtype)
                    : pl.kernel == LAM_KERNEL_GQA_MMA ? lam::occupancy_mma(a->kv_dtype, pl.variant)
                                                       : lam::occupancy_simt(a->kv_dtype, a->head_dim, pl.GQ, pl.variant);
    pl.ctas = std::max(pl.ctas, occ * ctx->num_sms);
    if (const int force = env_int("LAM_DECODE_CTAS", 0); force > 0)
      pl.ctas = std::min(force, occ * ctx->num_sms);
  }
  const int G = a->num_q_heads / a->num_kv_heads;
  const int D = a->head_dim;
  lam::DecodeParams p{};
  p.n_lm = 1;
  p.n_mb = 1;
  p.pool_layers = 1;
  p.q = a->q;
  p.q_stride = a->q_batch_stride > 0 ? a->q_batch_stride
                                     : static_cast<int64_t>(a->num_q_heads) * a->head_dim;
  p.k_pool = a->k_pool;
  p.v_pool = a->v_pool;
  p.page_table = a->page_table;
  p.seq_lens = a->seq_lens;
  p.out = a->out;
  p.lse = a->lse;
  p.B = a->batch;
  p.Hq = a->num_q_heads;
  p.Hkv = a->num_kv_heads;
  p.G = G;
  p.D = D;
  p.page_size = a->page_size;
  p.pt_stride = a->pt_stride;
  p.chunk = pl.chunk;
  p.S = pl.S;
  p.QG = pl.QG;
  const int64_t units = static_cast<int64_t>(a->batch) * a->num_kv_heads * pl.QG;
  p.u_head = static_cast<int32_t>(pl.u_head);
  p.n_items = static_cast<int32_t>(pl.u_head + (units - pl.u_head) * pl.S);
  p.mb_rows = a->batch;
  p.items_per_lm = p.n_items;
  p.units_per_lm = static_cast<int32_t>(units);
  if (st != nullptr) {
    if (static_cast<int64_t>(p.n_items) * n_lm >= (int64_t{1} << 31))
      return fail(LAM_ERR_VALIDATION, "step: too many work items");
    p.B = a_in->batch;
    p.n_lm = n_lm;
    p.n_mb = st->n_mb;
    p.n_items *= n_lm;
    p.pool_layers = st->pool_layers;
    p.layer0 = st->layer0;
    p.layer_rows = st->pool_layer_rows;
    p.lm_q_stride = st->lm_q_stride;
    p.lm_new_stride = st->lm_new_stride;
    p.lm_out_stride = st->lm_out_stride;
    p.flag_mb_stride = st->flag_mb_stride;
    p.epoch = st->epoch;
    p.trace = reinterpret_cast<unsigned long long*>(st->trace);
  }
  const int slot = static_cast<int>(ctx->seq % kSlots);
  p.slot = ctx->slots + 2 * slot;
  p.item_base = ctx->item_base[slot];
  p.done_base = ctx->done_base[slot];
  p.order = a->request_order;
  p.status = ctx->status;
  p.spin_timeout_ns = ctx->spin_timeout_ns;
  if (a->k_new != nullptr) {  // fused append
    if (a->v_new == nullptr) return fail(LAM_ERR_VALIDATION, "fused append needs both k_new and v_new");
    p.k_new = a->k_new;
    p.v_new = a->v_new;
    p.new_stride = a->new_batch_stride > 0 ? a->new_batch_stride
                                           : static_cast<int64_t>(a->num_kv_heads) * D;
    p.k_pool_w = const_cast<void*>(a->k_pool);
    p.v_pool_w = const_cast<void*>(a->v_pool);
  }
  if (io != nullptr) {  // rows grouped by source, buffers local or on peers
    if (io->n_src < 1 || io->n_src > LAM_MAX_PEERS || io->rows_per_src < 1 ||
        (io->row_src == nullptr && static_cast<int64_t>(io->n_src) * io->rows_per_src != a->batch))
      return fail(LAM_ERR_VALIDATION, "peer io: need 1 <= n_src <= LAM_MAX_PEERS and batch == "
                                      "n_src * rows_per_src (or a row map)");
    if (a->lse != nullptr) return fail(LAM_ERR_VALIDATION, "peer io: lse is not supported");
    const int e = a->kv_dtype == LAM_F32 ? 4 : 2;
    if ((io->k_new_offset * e) % 16 != 0 || (io->v_new_offset * e) % 16 != 0)
      return fail(LAM_ERR_VALIDATION, "peer io: new-row offsets must keep 16-byte rows");
    for (int i = 0; i < io->n_src; ++i) {
      if (io->q_src[i] == nullptr || io->out_dst[i] == nullptr)
        return fail(LAM_ERR_VALIDATION, "peer io: null source / destination pointer");
      p.q_src[i] = io->q_src[i];
      p.out_dst[i] = io->out_dst[i];
    }
    p.src_rows = io->rows_per_src;
    p.row_src = io->row_src;
    p.new_off[0] = io->k_new_offset;
    p.new_off[1] = io->v_new_offset;
    p.q = io->q_src[0];
    p.out = io->out_dst[0];
    p.k_new = io->q_src[0];  // non-null: fused append on (addresses come from new_off)
    p.v_new = io->q_src[0];
    p.new_stride = a->new_batch_stride > 0 ? a->new_batch_stride
                                           : static_cast<int64_t>(a->num_kv_heads) * D;
    p.k_pool_w = const_cast<void*>(a->k_pool);
    p.v_pool_w = const_cast<void*>(a->v_pool);
    if (io->n_wait < 0 || io->n_wait > LAM_MAX_PEERS || io->n_done < 0 || io->n_done > LAM_MAX_PEERS)
      return fail(LAM_ERR_VALIDATION, "peer io: n_wait / n_done out of range");
    for (int i = 0; i < io->n_wait; ++i) {
      if (!io->wait_flags[i]) return fail(LAM_ERR_VALIDATION, "peer io: null wait flag");
      p.wait_flag[i] = io->wait_flags[i];
    }
    for (int i = 0; i < io->n_done; ++i) {
      if (!io->done_flags[i]) return fail(LAM_ERR_VALIDATION, "peer io: null done flag");
      p.done_flag[i] = io->done_flags[i];
    }
    p.n_wait = io->n_wait;
    p.n_done = io->n_done;
    if (io->n_wait_kv < 0 || io->n_wait_kv > LAM_MAX_PEERS)
      return fail(LAM_ERR_VALIDATION, "peer io: n_wait_kv out of range");
    for (int i = 0; i < io->n_wait_kv; ++i) {
      if (!io->kv_wait_flags[i]) return fail(LAM_ERR_VALIDATION, "peer io: null kv wait flag");
      p.kv_wait_flag[i] = io->kv_wait_flags[i];
    }
    p.n_wait_kv = io->n_wait_kv;
    p.kv_wait_value = io->kv_wait_value;
    if (io->n_relay < 0 || io->n_relay > LAM_MAX_PEERS || (io->n_relay > 0 && st == nullptr))
      return fail(LAM_ERR_VALIDATION, "peer io: n_relay out of range (step launches only)");
    if (io->n_relay > 0 && io->relay_flag == nullptr)
      return fail(LAM_ERR_VALIDATION, "peer io: null relay flag");
    for (int i = 0; i < io->n_relay; ++i) {
      if (!io->relay_wait_flags[i]) return fail(LAM_ERR_VALIDATION, "peer io: null relay wait flag");
      p.relay_wait_flag[i] = io->relay_wait_flags[i];
    }
    p.n_relay = io->n_relay;
    p.relay_flag = io->relay_flag;
    if (st != nullptr && (io->n_wait > 0 || io->n_done > 0) && st->flag_mb_stride < 0)
      return fail(LAM_ERR_VALIDATION, "step: bad flag_mb_stride");
    p.wait_value = io->wait_value;
    p.done_value = io->done_value;
    // the launch carries its own input dependencies (sequence numbers), so with overlap_prev it
    // may overlap the previous kernel's drain entirely: it never waits for that grid, which the
    // caller's overlap_prev contract allows (the preceding kernel writes none of the page table,
    // lengths, order or KV rows this launch touches)
    p.pdl = io->n_wait > 0 && a->overlap_prev != 0 && env_int("LAM_PDL", 1) != 0;
    // LAM_PEER_PREFETCH=1: stream the first KV tiles (local pool) before the inputs' sequence
    // numbers arrive.  Off by default: the inputs are normally published before the launch
    // starts, and the deferred issue cost 0.3-0.6 % at N = 2 (experiments/r01/call61.sh).
    if (io->n_wait > 0 && env_int("LAM_PEER_PREFETCH", 0) != 0) p.defer_inputs = 2;
  }
  if (st != nullptr) p.defer_inputs = 0;  // (inputs are awaited per launch lm)
  if (a->overlap_prev != 0 && io == nullptr && st == nullptr) {
    // stream the first KV tiles while the preceding kernel drains; q / k_new / v_new wait for it
    p.pdl = 1;
    p.defer_inputs = 1;
  }
  p.flags = env_int("LAM_DECODE_FLAGS", 0);
  p.scale = a->scale;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.out_f32 = a->out_dtype == LAM_F32;
  if (pl.S > 1) {
    const int64_t all_rows = st != nullptr ? static_cast<int64_t>(st->n_layers) * a_in->batch : a->batch;
    const int64_t rows = all_rows * a->num_q_heads * pl.S;
    const int64_t cnt = all_rows * a->num_kv_heads * pl.QG;
    if (rows * D > ctx->ws_acc_cap || rows * 2 > ctx->ws_ml_cap || cnt > ctx->counters_cap) {
      rc = lam_ctx_reserve(ctx, std::max<int64_t>(rows, ctx->ws_ml_cap / 2), D,
                           std::max<int64_t>(cnt, ctx->counters_cap));
      if (rc != LAM_OK) return rc;
    }
    p.ws_acc = ctx->ws_acc + slot * ctx->ws_acc_cap;
    p.ws_ml = ctx->ws_ml + slot * ctx->ws_ml_cap;
    p.counters = ctx->counters + slot * ctx->counters_cap;
  }
  auto s = static_cast<cudaStream_t>(stream);
  if (st != nullptr) {  // [n_lm] finished units, [n_mb] layers published
    const int64_t need = n_lm + st->n_mb;
    if (need > ctx->lm_done_cap) {
      LAM_CUDA(grow(&ctx->lm_done, &ctx->lm_done_cap, static_cast<int64_t>(kSlots) * need, true));
      ctx->lm_done_cap = need;
    }
    p.lm_done = ctx->lm_done + slot * ctx->lm_done_cap;
    LAM_CUDA(cudaMemsetAsync(p.lm_done, 0, need * sizeof(int32_t), s));
  }
  if (pl.kernel == LAM_KERNEL_GQA_MMA || pl.kernel == LAM_KERNEL_GQA_TC) {
    int64_t rows = a->page_table
                       ? a->num_pages * a->num_kv_heads * static_cast<int64_t>(a->page_size)
                       : static_cast<int64_t>(a_in->batch) * a->num_kv_heads * a->page_size;
    if (st != nullptr) rows = std::max(rows, st->pool_layers * st->pool_layer_rows);
    if (rows >= (int64_t{1} << 31))
      return fail(LAM_ERR_VALIDATION, "pool exceeds 2^31 rows for the tensor map");
    CUtensorMap kmap, vmap;
    const int box_rows = pl.kernel == LAM_KERNEL_GQA_TC ? lam::kTcBoxRows : pl.tile;
    rc = make_pool_map(&kmap, a->kv_dtype, a->k_pool, rows, D, box_rows);
    if (rc != LAM_OK) return rc;
    rc = make_pool_map(&vmap, a->kv_dtype, a->v_pool, rows, D, box_rows);
    if (rc != LAM_OK) return rc;
    if (pl.kernel == LAM_KERNEL_GQA_TC)
      LAM_CUDA(lam::launch_decode_tc(a->kv_dtype, p, kmap, vmap, pl.ctas, s));
    else
      LAM_CUDA(lam::launch_decode_mma(a->kv_dtype, pl.variant, p, kmap, vmap, pl.ctas, s));
  } else {
    LAM_CUDA(lam::launch_decode_simt(a->kv_dtype, D, pl.GQ, pl.variant, p, pl.ctas, s));
  }
  // the slot's next launch starts where this one ends (every CTA claims until one claim past
  // the last item, and counts itself out once)
  // (producer_loop: the first min(grid, n_items) items are assigned without a claim)
  ctx->item_base[slot] += static_cast<uint64_t>(std::max<int64_t>(p.n_items, pl.ctas));
  ctx->done_base[slot] += static_cast<uint64_t>(pl.ctas);
  ++ctx->seq;
  return LAM_OK;
}

}  // namespace

int lam_decode(lam_ctx* ctx, const lam_decode_args* a, void* stream) {
  return decode_impl(ctx, a, nullptr, nullptr, stream);
}

int lam_decode_peer(lam_ctx* ctx, const lam_decode_args* a, const lam_peer_io* io, void* stream) {
  if (!io) return fail(LAM_ERR_VALIDATION, "null peer io");
  return decode_impl(ctx, a, io, nullptr, stream);
}

int lam_decode_step(lam_ctx* ctx, const lam_decode_args* a, const lam_step_layout* step,
                    const lam_peer_io* io, void* stream) {
  if (!step) return fail(LAM_ERR_VALIDATION, "null step layout");
  return decode_impl(ctx, a, io, step, stream);
}

// ---------------- peer-memory transport ----------------

static_assert(sizeof(cudaIpcMemHandle_t) <= LAM_IPC_HANDLE_BYTES, "IPC handle size");

int lam_peer_alloc(lam_ctx* ctx, int64_t bytes, void** dptr, void* handle) {
  if (!ctx || !dptr || !handle || bytes < 1) return fail(LAM_ERR_VALIDATION, "peer_alloc: bad arguments");
  LAM_DEVICE(ctx);
  void* p = nullptr;
  LAM_CUDA(cudaMalloc(&p, static_cast<size_t>(bytes)));
  cudaError_t e = cudaMemset(p, 0, static_cast<size_t>(bytes));
  cudaIpcMemHandle_t h{};
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(LAM_ERR_CUDA, std::string("peer_alloc: ") + cudaGetErrorString(e));
  }
  std::memset(handle, 0, LAM_IPC_HANDLE_BYTES);
  std::memcpy(handle, &h, sizeof(h));
  *dptr = p;
  return LAM_OK;
}

int lam_peer_free(lam_ctx* ctx, void* dptr) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  LAM_DEVICE(ctx);
  LAM_CUDA(cudaFree(dptr));
  return LAM_OK;
}

int lam_peer_open(lam_ctx* ctx, const void* handle, void** dptr) {
  if (!ctx || !handle || !dptr) return fail(LAM_ERR_VALIDATION, "peer_open: bad arguments");
  LAM_DEVICE(ctx);
  cudaIpcMemHandle_t h{};
  std::memcpy(&h, handle, sizeof(h));
  LAM_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return LAM_OK;
}

int lam_peer_close(lam_ctx* ctx, void* dptr) {
  if (!ctx) return fail(LAM_ERR_VALIDATION, "null context");
  LAM_DEVICE(ctx);
  LAM_CUDA(cudaIpcCloseMemHandle(dptr));
  return LAM_OK;
}

namespace {

void* driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return p;
}

PFN_cuStreamWriteValue32_v11070 write_value_fn() {
  static auto fn = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(driver_fn("cuStreamWriteValue32"));
  return fn;
}
PFN_cuStreamWaitValue32_v11070 wait_value_fn() {
  static auto fn = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(driver_fn("cuStreamWaitValue32"));
  return fn;
}

}  // namespace

int lam_stream_signal(lam_ctx* ctx, void* const* addrs, int32_t n, uint32_t value, void* stream) {
  if (!ctx || (n > 0 && !addrs)) return fail(LAM_ERR_VALIDATION, "stream_signal: bad arguments");
  auto fn = write_value_fn();
  if (!fn) return fail(LAM_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  for (int32_t i = 0; i < n; ++i) {
    // default flags: a system-scope memory barrier orders the stream's prior writes (the
    // decode kernel's peer stores) before the sequence number (B200 rejects
    // CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER with CUDA_ERROR_INVALID_VALUE)
    const CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addrs[i]),
                          value, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS)
      return fail(LAM_ERR_CUDA, "cuStreamWriteValue32 failed (" + std::to_string(r) + ")");
  }
  return LAM_OK;
}

int lam_stream_wait(lam_ctx* ctx, const void* const* addrs, int32_t n, uint32_t value,
                    void* stream) {
  if (!ctx || (n > 0 && !addrs)) return fail(LAM_ERR_VALIDATION, "stream_wait: bad arguments");
  auto fn = wait_value_fn();
  if (!fn) return fail(LAM_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  for (int32_t i = 0; i < n; ++i) {
    const CUresult r = fn(static_cast<CUstream>(stream),
                          reinterpret_cast<CUdeviceptr>(const_cast<void*>(addrs[i])), value,
                          CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS)
      return fail(LAM_ERR_CUDA, "cuStreamWaitValue32 failed (" + std::to_string(r) + ")");
  }
  return LAM_OK;
}

int lam_kv_append(int32_t dtype, int32_t batch, int32_t num_kv_heads, int32_t head_dim,
                  int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                  const int32_t* positions, const void* k_new, const void* v_new,
                  int64_t new_batch_stride, void* k_pool, void* v_pool, void* stream) {
  const int e = elem_bytes(dtype);
  if (e == 0 || (head_dim * e) % 16 != 0)
    return fail(LAM_ERR_VALIDATION, "kv_append needs rows that are a multiple of 16 bytes");
  if (page_size < 1) return fail(LAM_ERR_VALIDATION, "page_size must be >= 1");
  const int64_t stride = new_batch_stride > 0 ? new_batch_stride
                                              : static_cast<int64_t>(num_kv_heads) * head_dim;
  if ((stride * e) % 16 != 0)
    return fail(LAM_ERR_VALIDATION, "kv_append batch stride must keep rows 16-byte aligned");
  LAM_CUDA(lam::launch_kv_append(e, batch, num_kv_heads, head_dim, page_size, pt_stride,
                                 page_table, positions, k_new, v_new, stride, k_pool, v_pool,
                                 static_cast<cudaStream_t>(stream)));
  return LAM_OK;
}

int lam_kv_gather(int32_t dtype, int32_t batch, int32_t num_kv_heads, int32_t head_dim,
                  int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                  const int32_t* seq_lens, int32_t l_max, const void* pool, void* dense,
                  void* stream) {
  const int e = elem_bytes(dtype);
  if (e == 0 || (head_dim * e) % 16 != 0)
    return fail(LAM_ERR_VALIDATION, "kv_gather needs rows that are a multiple of 16 bytes");
  if (!page_table) return fail(LAM_ERR_VALIDATION, "kv_gather needs a page table");
  LAM_CUDA(lam::launch_kv_gather(e, batch, num_kv_heads, head_dim, page_size, pt_stride,
                                 page_table, seq_lens, l_max, pool, dense,
                                 static_cast<cudaStream_t>(stream)));
  return LAM_OK;
}

int lam_decode_step_host(lam_ctx* ctx, const lam_decode_args* a, const void* h_q,
                         const void* h_k_new, const void* h_v_new, void* h_out, void* d_k_new,
                         void* d_v_new, const int32_t* d_positions, void* stream) {
  if (!ctx || !a) return fail(LAM_ERR_VALIDATION, "null context or args");
  auto s = static_cast<cudaStream_t>(stream);
  const int e = elem_bytes(a->kv_dtype);
  const int eo = elem_bytes(a->out_dtype);
  const int64_t qb = static_cast<int64_t>(a->batch) * a->num_q_heads * a->head_dim * e;
  const int64_t kb = static_cast<int64_t>(a->batch) * a->num_kv_heads * a->head_dim * e;
  const int64_t ob = static_cast<int64_t>(a->batch) * a->num_q_heads * a->head_dim * eo;
  LAM_CUDA(cudaMemcpyAsync(const_cast<void*>(a->q), h_q, qb, cudaMemcpyHostToDevice, s));
  LAM_CUDA(cudaMemcpyAsync(d_k_new, h_k_new, kb, cudaMemcpyHostToDevice, s));
  LAM_CUDA(cudaMemcpyAsync(d_v_new, h_v_new, kb, cudaMemcpyHostToDevice, s));
  int rc = lam_kv_append(a->kv_dtype, a->batch, a->num_kv_heads, a->head_dim, a->page_size,
                         a->pt_stride, a->page_table, d_positions, d_k_new, d_v_new, 0,
                         const_cast<void*>(a->k_pool), const_cast<void*>(a->v_pool), stream);
  if (rc != LAM_OK) return rc;
  rc = lam_decode(ctx, a, stream);
  if (rc != LAM_OK) return rc;
  LAM_CUDA(cudaMemcpyAsync(h_out, a->out, ob, cudaMemcpyDeviceToHost, s));
  return LAM_OK;
}

namespace {
struct StageLayout {
  int64_t q, kv, out, set;  // bytes of each part (256-aligned) and of one staging set
};
StageLayout stage_layout(const lam_decode_args* a) {
  auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  const int64_t e = elem_bytes(a->kv_dtype), eo = elem_bytes(a->out_dtype);
  StageLayout s;
  s.q = al(static_cast<int64_t>(a->batch) * a->num_q_heads * a->head_dim * e);
  s.kv = al(static_cast<int64_t>(a->batch) * a->num_kv_heads * a->head_dim * e);
  s.out = al(static_cast<int64_t>(a->batch) * a->num_q_heads * a->head_dim * eo);
  s.set = s.q + 2 * s.kv + s.out;
  return s;
}
}  // namespace

namespace {
// lam_decode_layers_host without events between the launches: the compute stream carries
// nothing but the decode launches, so they overlap their neighbours (programmatic dependent
// launch), and readiness travels as sequence numbers, as on the peer transport:
//  * copy stream: H2D of layer l into staging set l % 2, then writes in_ready[set] = seq(l)
//    (cuStreamWriteValue32 after a system-wide fence);
//  * decode launch of layer l (lam_decode_peer with one local source): every CTA's producer
//    polls in_ready[set] >= seq(l) before its first load; the last CTA publishes
//    out_ready[set] = seq(l) after every output store;
//  * copy stream: waits out_ready[set] >= seq(l) (cuStreamWaitValue32), D2H of layer l, then
//    the H2D of layer l + 2 into the same set (so neither the inputs nor the output of a set
//    are overwritten before they are consumed).
int decode_layers_host_flags(lam_ctx* ctx, const lam_decode_args* layer_args, int32_t n_layers,
                             const void* const* h_q, const void* const* h_k_new,
                             const void* const* h_v_new, void* const* h_out, void* d_stage,
                             const StageLayout& L, cudaStream_t cs, cudaStream_t xs) {
  auto base = [&](int set) { return static_cast<uint8_t*>(d_stage) + set * L.set; };
  if (!ctx->host_flags) {
    LAM_CUDA(cudaMalloc(&ctx->host_flags, 4 * sizeof(uint32_t)));
    LAM_CUDA(cudaMemset(ctx->host_flags, 0, 4 * sizeof(uint32_t)));
    LAM_CUDA(cudaDeviceSynchronize());
  }
  uint32_t* in_flag = ctx->host_flags;       // [2]
  uint32_t* out_flag = ctx->host_flags + 2;  // [2]
  const uint32_t seq0 = ctx->host_seq;
  ctx->host_seq += static_cast<uint32_t>(n_layers);
  auto seq = [&](int l) { return seq0 + static_cast<uint32_t>(l) + 1u; };
  cudaEvent_t start, done;
  LAM_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  LAM_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  LAM_CUDA(cudaEventRecord(start, cs));  // the copy stream starts after prior compute work
  LAM_CUDA(cudaStreamWaitEvent(xs, start, 0));
  int rc = LAM_OK;
  auto h2d = [&](int l) -> int {
    const int s = l & 1;
    uint8_t* b = base(s);
    const lam_decode_args& a = layer_args[l];
    const int64_t qb = static_cast<int64_t>(a.batch) * a.num_q_heads * a.head_dim * elem_bytes(a.kv_dtype);
    const int64_t kb = static_cast<int64_t>(a.batch) * a.num_kv_heads * a.head_dim * elem_bytes(a.kv_dtype);
    LAM_CUDA(cudaMemcpyAsync(b, h_q[l], qb, cudaMemcpyHostToDevice, xs));
    LAM_CUDA(cudaMemcpyAsync(b + L.q, h_k_new[l], kb, cudaMemcpyHostToDevice, xs));
    LAM_CUDA(cudaMemcpyAsync(b + L.q + L.kv, h_v_new[l], kb, cudaMemcpyHostToDevice, xs));
    void* f = in_flag + s;
    return lam_stream_signal(ctx, &f, 1, seq(l), xs);
  };
  auto d2h = [&](int l) -> int {
    const int s = l & 1;
    const void* f = out_flag + s;
    if ((rc = lam_stream_wait(ctx, &f, 1, seq(l), xs)) != LAM_OK) return rc;
    const lam_decode_args& a = layer_args[l];
    const int64_t ob = static_cast<int64_t>(a.batch) * a.num_q_heads * a.head_dim * elem_bytes(a.out_dtype);
    LAM_CUDA(cudaMemcpyAsync(h_out[l], base(s) + L.q + 2 * L.kv, ob, cudaMemcpyDeviceToHost, xs));
    return LAM_OK;
  };
  // copy-stream program: H2D 0, H2D 1, then per layer l: D2H l, H2D l + 2
  if ((rc = h2d(0)) != LAM_OK) return rc;
  if (n_layers > 1 && (rc = h2d(1)) != LAM_OK) return rc;
  for (int l = 0; l < n_layers; ++l) {
    const int s = l & 1;
    uint8_t* b = base(s);
    lam_decode_args a = layer_args[l];
    const int e = elem_bytes(a.kv_dtype);
    a.q_batch_stride = 0;
    a.new_batch_stride = 0;
    a.overlap_prev = l > 0;  // consecutive layers: disjoint pools (overlap_prev contract)
    lam_peer_io io{};
    io.n_src = 1;
    io.rows_per_src = a.batch;
    io.q_src[0] = b;
    io.out_dst[0] = b + L.q + 2 * L.kv;
    io.k_new_offset = L.q / e;
    io.v_new_offset = (L.q + L.kv) / e;
    io.n_wait = 1;
    io.wait_flags[0] = in_flag + s;
    io.wait_value = seq(l);
    io.n_done = 1;
    io.done_flags[0] = out_flag + s;
    io.done_value = seq(l);
    if ((rc = lam_decode_peer(ctx, &a, &io, cs)) != LAM_OK) return rc;
    if ((rc = d2h(l)) != LAM_OK) return rc;
    if (l + 2 < n_layers && (rc = h2d(l + 2)) != LAM_OK) return rc;
  }
  LAM_CUDA(cudaEventRecord(done, xs));
  LAM_CUDA(cudaStreamWaitEvent(cs, done, 0));  // `stream` completes after the last D2H
  cudaEventDestroy(start);
  cudaEventDestroy(done);
  return LAM_OK;
}
// lam_decode_layers_host with zero-copy I/O: every layer is one lam_decode_peer launch whose
// single "source" is the caller's pinned host memory (mapped into the device address space).
// The producer warps load each item's q and new K / V rows from host memory over PCIe with the
// same TMA copies that read peer memory over NVLink, hidden under the item's KV streaming, and
// the epilogue stores the outputs straight into h_out.  No staging copies, no copy-stream
// events: one launch per layer on `stream`.
bool host_mapped(const void* ptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost && at.devicePointer == ptr;
}

int decode_layers_host_mapped(lam_ctx* ctx, const lam_decode_args* layer_args, int32_t n_layers,
                              const void* const* h_q, const void* const* h_k_new,
                              const void* const* h_v_new, void* const* h_out, cudaStream_t cs) {
  for (int l = 0; l < n_layers; ++l) {
    lam_decode_args a = layer_args[l];
    const int e = elem_bytes(a.kv_dtype);
    const auto* q = static_cast<const uint8_t*>(h_q[l]);
    a.q_batch_stride = 0;     // dense [B][Hq][D] host rows
    a.new_batch_stride = 0;   // dense [B][Hkv][D]
    a.overlap_prev = 0;
    lam_peer_io io{};
    io.n_src = 1;
    io.rows_per_src = a.batch;
    io.q_src[0] = h_q[l];
    io.out_dst[0] = h_out[l];
    io.k_new_offset = (static_cast<const uint8_t*>(h_k_new[l]) - q) / e;
    io.v_new_offset = (static_cast<const uint8_t*>(h_v_new[l]) - q) / e;
    const int rc = lam_decode_peer(ctx, &a, &io, cs);
    if (rc != LAM_OK) return rc;
  }
  return LAM_OK;
}

// zero-copy applies when every host buffer is pinned, mapped and 16-byte aligned relative to q
bool host_mapped_ok(const lam_decode_args* layer_args, int32_t n_layers, const void* const* h_q,
                    const void* const* h_k_new, const void* const* h_v_new, void* const* h_out) {
  for (int l = 0; l < n_layers; ++l) {
    if (layer_args[l].lse != nullptr || layer_args[l].batch < 1) return false;
    const auto q = reinterpret_cast<uintptr_t>(h_q[l]);
    const uintptr_t ptrs[3] = {reinterpret_cast<uintptr_t>(h_k_new[l]),
                               reinterpret_cast<uintptr_t>(h_v_new[l]),
                               reinterpret_cast<uintptr_t>(h_out[l])};
    if (q % 16 != 0) return false;
    for (uintptr_t p : ptrs)
      if (p % 16 != 0) return false;
    if (!host_mapped(h_q[l]) || !host_mapped(h_k_new[l]) || !host_mapped(h_v_new[l]) ||
        !host_mapped(h_out[l]))
      return false;
  }
  return true;
}
}  // namespace

int64_t lam_decode_step_from_host_stage_bytes(const lam_decode_args* a, int32_t n_layers) {
  return a && n_layers > 0 ? n_layers * stage_layout(a).set : 0;
}

int lam_decode_step_from_host(lam_ctx* ctx, const lam_decode_args* a, const lam_step_layout* step,
                         const void* const* h_q, const void* const* h_k_new,
                         const void* const* h_v_new, void* const* h_out, void* d_stage,
                         void* stream, void* copy_stream) {
  if (!ctx || !a || !step || step->n_layers < 1 || step->n_mb != 1 || !d_stage)
    return fail(LAM_ERR_VALIDATION, "step_from_host: bad arguments (one micro-batch, >= 1 layer)");
  if (a->lse != nullptr) return fail(LAM_ERR_VALIDATION, "step_from_host: lse is not supported");
  if (a->batch == 0) return LAM_OK;
  LAM_DEVICE(ctx);
  auto cs = static_cast<cudaStream_t>(stream);
  auto xs = static_cast<cudaStream_t>(copy_stream);
  const StageLayout S = stage_layout(a);
  const int n = step->n_layers;
  const int e = elem_bytes(a->kv_dtype), eo = elem_bytes(a->out_dtype);
  const int64_t qb = static_cast<int64_t>(a->batch) * a->num_q_heads * a->head_dim * e;
  const int64_t kb = static_cast<int64_t>(a->batch) * a->num_kv_heads * a->head_dim * e;
  const int64_t ob = static_cast<int64_t>(a->batch) * a->num_q_heads * a->head_dim * eo;
  auto base = [&](int l) { return static_cast<uint8_t*>(d_stage) + l * S.set; };
  if (!ctx->host_flags) {
    LAM_CUDA(cudaMalloc(&ctx->host_flags, 4 * sizeof(uint32_t)));
    LAM_CUDA(cudaMemset(ctx->host_flags, 0, 4 * sizeof(uint32_t)));
    LAM_CUDA(cudaDeviceSynchronize());
  }
  uint32_t* in_flag = ctx->host_flags;
  uint32_t* out_flag = ctx->host_flags + 2;
  const uint32_t epoch = ctx->host_seq;
  ctx->host_seq += static_cast<uint32_t>(n);
  // the step launch: layer l's rows live in staging region l (one local "source")
  lam_decode_args la = *a;
  la.q_batch_stride = 0;
  la.new_batch_stride = 0;
  la.overlap_prev = 0;
  // layers do not wait for each other's outputs here: one pool of items, no splits
  if (la.split_tokens <= 0) la.split_tokens = std::max(1, la.max_len);
  lam_peer_io io{};
  io.n_src = 1;
  io.rows_per_src = a->batch;
  io.q_src[0] = base(0);
  io.out_dst[0] = base(0) + S.q + 2 * S.kv;
  io.k_new_offset = S.q / e;
  io.v_new_offset = (S.q + S.kv) / e;
  io.n_wait = io.n_done = 1;
  io.wait_flags[0] = in_flag;
  io.done_flags[0] = out_flag;
  // (a one-layer step is an ordinary launch: it waits for and publishes these values)
  io.wait_value = io.done_value = epoch + 1;
  lam_step_layout st = *step;
  st.n_mb = 1;
  st.rows_per_mb = a->batch;
  st.lm_q_stride = S.set / e;
  st.lm_new_stride = 0;
  st.lm_out_stride = S.set / eo;
  st.flag_mb_stride = 0;
  st.epoch = epoch;
  cudaEvent_t start, done;
  LAM_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  LAM_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  LAM_CUDA(cudaEventRecord(start, cs));  // the copies start after prior work on `stream`
  LAM_CUDA(cudaStreamWaitEvent(xs, start, 0));
  int rc = decode_impl(ctx, &la, &io, &st, stream);
  if (rc != LAM_OK) return rc;
  // copy stream: every layer's inputs go in at once, each announced by its sequence number;
  // each output comes back as soon as the launch publishes its layer
  for (int l = 0; l < n; ++l) {
    LAM_CUDA(cudaMemcpyAsync(base(l), h_q[l], qb, cudaMemcpyHostToDevice, xs));
    LAM_CUDA(cudaMemcpyAsync(base(l) + S.q, h_k_new[l], kb, cudaMemcpyHostToDevice, xs));
    LAM_CUDA(cudaMemcpyAsync(base(l) + S.q + S.kv, h_v_new[l], kb, cudaMemcpyHostToDevice, xs));
    void* f = in_flag;
    if ((rc = lam_stream_signal(ctx, &f, 1, epoch + l + 1, xs)) != LAM_OK) return rc;
  }
  for (int l = 0; l < n; ++l) {
    const void* f = out_flag;
    if ((rc = lam_stream_wait(ctx, &f, 1, epoch + l + 1, xs)) != LAM_OK) return rc;
    LAM_CUDA(cudaMemcpyAsync(h_out[l], base(l) + S.q + 2 * S.kv, ob, cudaMemcpyDeviceToHost, xs));
  }
  LAM_CUDA(cudaEventRecord(done, xs));
  LAM_CUDA(cudaStreamWaitEvent(cs, done, 0));  // `stream` completes after the last D2H
  cudaEventDestroy(start);
  cudaEventDestroy(done);
  return LAM_OK;
}

int64_t lam_decode_layers_host_stage_bytes(const lam_decode_args* a) {
  return a ? 2 * stage_layout(a).set : 0;
}

int lam_decode_layers_host(lam_ctx* ctx, const lam_decode_args* layer_args, int32_t n_layers,
                           const void* const* h_q, const void* const* h_k_new,
                           const void* const* h_v_new, void* const* h_out, void* d_stage,
                           const int32_t* d_positions, void* stream, void* copy_stream) {
  if (!ctx || !layer_args || n_layers < 0) return fail(LAM_ERR_VALIDATION, "bad arguments");
  if (n_layers == 0) return LAM_OK;
  LAM_DEVICE(ctx);
  auto cs = static_cast<cudaStream_t>(stream);
  auto xs = static_cast<cudaStream_t>(copy_stream);
  const StageLayout L = stage_layout(&layer_args[0]);
  for (int l = 1; l < n_layers; ++l) {  // both staging sets are sized from layer 0
    const StageLayout Ll = stage_layout(&layer_args[l]);
    if (Ll.q > L.q || Ll.kv > L.kv || Ll.out > L.out)
      return fail(LAM_ERR_VALIDATION, "layer " + std::to_string(l) +
                                          ": q / k_new / v_new / out larger than layer 0's staging");
  }
  // Zero-copy I/O (decode_layers_host_mapped) for a one-layer step — there the staged path's
  // H2D -> decode -> D2H chain is serial, nothing hides it — and wherever LAM_HOST_ZERO_COPY=1;
  // LAM_HOST_ZERO_COPY=0 always stages.
  const int zc = env_int("LAM_HOST_ZERO_COPY", -1);
  if ((zc == 1 || (zc < 0 && n_layers == 1)) &&
      host_mapped_ok(layer_args, n_layers, h_q, h_k_new, h_v_new, h_out))
    return decode_layers_host_mapped(ctx, layer_args, n_layers, h_q, h_k_new, h_v_new, h_out, cs);
  auto base = [&](int set) { return static_cast<uint8_t*>(d_stage) + set * L.set; };
  // LAM_HOST_FLAGS=1: launches synchronised by sequence numbers instead of events.  Measured
  // equal for C2 / C3 and slower for one-layer C1 (experiments/r01/call63.sh), so events stay default.
  const int use_flags = env_int("LAM_HOST_FLAGS", 0);
  bool flags_ok = use_flags && write_value_fn() && wait_value_fn();
  for (int l = 0; l < n_layers && flags_ok; ++l)  // (the peer-io launch has no lse output)
    flags_ok = layer_args[l].lse == nullptr && layer_args[l].batch > 0;
  if (flags_ok)
    return decode_layers_host_flags(ctx, layer_args, n_layers, h_q, h_k_new, h_v_new, h_out,
                                    d_stage, L, cs, xs);
  // in_ready[s]: H2D of staging set s landed; consumed[s]: compute done reading set s inputs;
  // out_ready[s]: output of set s written; out_free[s]: D2H of set s finished.
  cudaEvent_t in_ready[2], consumed[2], out_ready[2], out_free[2];
  for (int s = 0; s < 2; ++s) {
    LAM_CUDA(cudaEventCreateWithFlags(&in_ready[s], cudaEventDisableTiming));
    LAM_CUDA(cudaEventCreateWithFlags(&consumed[s], cudaEventDisableTiming));
    LAM_CUDA(cudaEventCreateWithFlags(&out_ready[s], cudaEventDisableTiming));
    LAM_CUDA(cudaEventCreateWithFlags(&out_free[s], cudaEventDisableTiming));
  }
  auto h2d = [&](int l) -> int {
    const int s = l & 1;
    if (l >= 2) LAM_CUDA(cudaStreamWaitEvent(xs, consumed[s], 0));
    uint8_t* b = base(s);
    const int64_t qb = static_cast<int64_t>(layer_args[l].batch) * layer_args[l].num_q_heads *
                       layer_args[l].head_dim * elem_bytes(layer_args[l].kv_dtype);
    const int64_t kb = static_cast<int64_t>(layer_args[l].batch) * layer_args[l].num_kv_heads *
                       layer_args[l].head_dim * elem_bytes(layer_args[l].kv_dtype);
    LAM_CUDA(cudaMemcpyAsync(b, h_q[l], qb, cudaMemcpyHostToDevice, xs));
    LAM_CUDA(cudaMemcpyAsync(b + L.q, h_k_new[l], kb, cudaMemcpyHostToDevice, xs));
    LAM_CUDA(cudaMemcpyAsync(b + L.q + L.kv, h_v_new[l], kb, cudaMemcpyHostToDevice, xs));
    LAM_CUDA(cudaEventRecord(in_ready[s], xs));
    return LAM_OK;
  };
  int rc = LAM_OK;
  LAM_CUDA(cudaEventRecord(consumed[0], cs));  // copy stream starts after prior compute work
  LAM_CUDA(cudaStreamWaitEvent(xs, consumed[0], 0));
  if ((rc = h2d(0)) != LAM_OK) return rc;
  for (int l = 0; l < n_layers; ++l) {
    const int s = l & 1;
    if (l + 1 < n_layers && (rc = h2d(l + 1)) != LAM_OK) return rc;
    uint8_t* b = base(s);
    lam_decode_args a = layer_args[l];
    a.q = b;
    a.q_batch_stride = 0;  // the staging set holds dense [B][Hq][D] rows
    a.out = b + L.q + 2 * L.kv;
    LAM_CUDA(cudaStreamWaitEvent(cs, in_ready[s], 0));
    if (l >= 2) LAM_CUDA(cudaStreamWaitEvent(cs, out_free[s], 0));
    // fused append: the new token (position seq_lens[b] - 1) comes from the staging set
    (void)d_positions;
    a.k_new = b + L.q;
    a.v_new = b + L.q + L.kv;
    a.new_batch_stride = 0;
    if ((rc = lam_decode(ctx, &a, stream)) != LAM_OK) return rc;
    LAM_CUDA(cudaEventRecord(consumed[s], cs));
    LAM_CUDA(cudaEventRecord(out_ready[s], cs));
    LAM_CUDA(cudaStreamWaitEvent(xs, out_ready[s], 0));
    const int64_t ob = static_cast<int64_t>(a.batch) * a.num_q_heads * a.head_dim *
                       elem_bytes(a.out_dtype);
    LAM_CUDA(cudaMemcpyAsync(h_out[l], a.out, ob, cudaMemcpyDeviceToHost, xs));
    LAM_CUDA(cudaEventRecord(out_free[s], xs));
  }
  LAM_CUDA(cudaEventRecord(out_free[0], xs));
  LAM_CUDA(cudaStreamWaitEvent(cs, out_free[0], 0));  // `stream` completes after the last D2H
  for (int s = 0; s < 2; ++s) {
    cudaEventDestroy(in_ready[s]);
    cudaEventDestroy(consumed[s]);
    cudaEventDestroy(out_ready[s]);
    cudaEventDestroy(out_free[s]);
  }
  return LAM_OK;
}

}  // extern "C"
