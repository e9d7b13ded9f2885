/*
 * lamina_attn.h — C-ABI of the B200 (sm_100a) decode-attention operator.
 *
 * This is the drop-in boundary below the reference's C++ operator API
 * (/root/reference/proj/core/include/disagg/attention.hpp:1-114).  Every entry
 * point takes plain pointers, sizes and an opaque cudaStream_t (passed as void*);
 * no C++ or torch types cross it.  The C++ wrapper that keeps the reference
 * signatures unchanged lives in paper_2405_01814_b200/dropin/attention.cpp and
 * maps the status codes below onto the reference exception hierarchy
 * (model.hpp:25-40):
 *
 *   LAM_OK               0  success
 *   LAM_ERR_ERROR        1  -> disagg::Error            (empty key set, index out of range,
 *                                                         finalize of an empty partial, bad split)
 *   LAM_ERR_VALIDATION   2  -> disagg::ValidationError  (dims, divisibility, unsupported shape)
 *   LAM_ERR_CUDA         3  CUDA runtime / driver failure (message in lam_last_error())
 *
 * Ownership: the caller owns every buffer; the library owns lam_ctx / lam_plan handles.
 * Threading: lam_ctx is not shared between concurrently running host threads; the
 * *_host entry points use a per-thread staging area and are reentrant.
 * There is no CPU fallback: every attention entry point runs on the GPU.
 */
#ifndef LAMINA_ATTN_H
#define LAMINA_ATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAM_OK 0
#define LAM_ERR_ERROR 1
#define LAM_ERR_VALIDATION 2
#define LAM_ERR_CUDA 3

/* element types */
#define LAM_F32 0
#define LAM_F64 1
#define LAM_BF16 2
#define LAM_F16 3

/* kernel families (lam_decode `kernel` argument / lam_plan_kernel result) */
#define LAM_KERNEL_AUTO 0
#define LAM_KERNEL_SIMT 1     /* warp-shuffle online softmax, CUDA cores (MHA) */
#define LAM_KERNEL_GQA_MMA 2  /* tensor-core m16n8k16 over a GQA group of 8 q heads */
#define LAM_KERNEL_GQA_TC 3   /* tcgen05.mma from the TMA ring, accumulators in TMEM */

typedef struct lam_ctx lam_ctx;

/* ---- library / context -------------------------------------------------- */

int lam_version(void);
/* Thread-local message for the last non-zero status returned on this thread. */
const char* lam_last_error(void);

/* A context binds one CUDA device and owns the split-K workspace + counters. */
int lam_ctx_create(int device, lam_ctx** out);
int lam_ctx_destroy(lam_ctx* ctx);
/* Pre-size the split-K workspace so no allocation happens inside lam_decode. */
int lam_ctx_reserve(lam_ctx* ctx, int64_t partial_rows, int32_t head_dim, int64_t counters);
/* Number of SMs of the context's device (148 on B200). */
int lam_ctx_num_sms(const lam_ctx* ctx);

/* Bounded device-side spins.  A decode launch that waits for its input sequence numbers
 * (lam_peer_io.wait_flags) or for its launch slot longer than the timeout gives up instead of
 * trapping: it records a LAM_STATUS_* code in the context's status word, completes (outputs
 * unspecified) and still publishes its done flags, so no waiter on another GPU hangs and the
 * CUDA context stays usable.  Default 10 s, or LAM_SPIN_TIMEOUT_MS at lam_ctx_create; 0 waits
 * forever.  lam_ctx_status synchronises the device and reads (and optionally clears) the word. */
#define LAM_STATUS_OK 0
#define LAM_STATUS_INPUT_TIMEOUT 1
#define LAM_STATUS_SLOT_TIMEOUT 2
int lam_ctx_set_spin_timeout(lam_ctx* ctx, int64_t timeout_ns);
int lam_ctx_status(lam_ctx* ctx, int32_t* status, int32_t clear);

/* ---- reference operator API, device pointers -----------------------------
 * One "instance" is one AttnInstance (attention.hpp:20-30): a query vector of d
 * elements and its key/value rows.  Keys/values of all instances live in two row
 * pools k_rows/v_rows of shape [rows][d]; instance i owns rows
 * [kv_row0[i], kv_row0[i] + kv_len[i]).  Several instances may share rows
 * (multi_head_attention's GQA mapping, attention.cpp:141-150) — nothing is copied.
 * dtype is LAM_F32 or LAM_F64 (the reference's two instantiations,
 * attention.cpp:205-230); scale points to n_inst values of that dtype.
 */

/* exact_attention (attention.cpp:48-70).  LAM_ERR_ERROR if any kv_len == 0. */
int lam_exact_attention(lam_ctx* ctx, int dtype, int64_t n_inst, int32_t d, const void* q,
                        const void* k_rows, const void* v_rows, const int64_t* kv_row0,
                        const int64_t* kv_len, const void* scale, void* out, void* stream);

/* partial_attention over index subsets (attention.cpp:72-98).  Instance i uses
 * indices idx[idx_off[i] .. idx_off[i+1]) into its own rows; an empty subset yields
 * the identity partial (acc = 0, max_logit = log_denom = -inf, count = 0).
 * LAM_ERR_ERROR ("token index out of range") if any index is outside [0, kv_len[i]). */
int lam_partial_attention(lam_ctx* ctx, int dtype, int64_t n_inst, int32_t d, const void* q,
                          const void* k_rows, const void* v_rows, const int64_t* kv_row0,
                          const int64_t* kv_len, const int64_t* idx, const int64_t* idx_off,
                          const void* scale, void* acc, void* max_logit, void* log_denom,
                          int64_t* token_count, void* stream);

/* merge (attention.cpp:100-118), n pairs elementwise; identity early-outs are bitwise. */
int lam_merge(lam_ctx* ctx, int dtype, int64_t n, int32_t d, const void* a_acc,
              const void* a_max, const void* a_log_denom, const int64_t* a_count,
              const void* b_acc, const void* b_max, const void* b_log_denom,
              const int64_t* b_count, void* o_acc, void* o_max, void* o_log_denom,
              int64_t* o_count, void* stream);

/* finalize (attention.cpp:120-127).  LAM_ERR_ERROR if any partial is empty. */
int lam_finalize(lam_ctx* ctx, int dtype, int64_t n, int32_t d, const void* acc,
                 const void* log_denom, const int64_t* count, void* out, void* stream);

/* ---- reference operator API, host pointers --------------------------------
 * Same semantics as above, but every array lives in host memory; the library stages
 * it through a per-thread device buffer, runs the kernel and copies results back
 * before returning.  These are what the C++ drop-in calls. */
int lam_exact_attention_host(int dtype, int64_t n_inst, int32_t d, const void* q,
                             int64_t n_rows, const void* k_rows, const void* v_rows,
                             const int64_t* kv_row0, const int64_t* kv_len, const void* scale,
                             void* out);
int lam_partial_attention_host(int dtype, int64_t n_inst, int32_t d, const void* q,
                               int64_t n_rows, const void* k_rows, const void* v_rows,
                               const int64_t* kv_row0, const int64_t* kv_len,
                               const int64_t* idx, const int64_t* idx_off, const void* scale,
                               void* acc, void* max_logit, void* log_denom,
                               int64_t* token_count);
int lam_merge_host(int dtype, int64_t n, int32_t d, const void* a_acc, const void* a_max,
                   const void* a_log_denom, const int64_t* a_count, const void* b_acc,
                   const void* b_max, const void* b_log_denom, const int64_t* b_count,
                   void* o_acc, void* o_max, void* o_log_denom, int64_t* o_count);
int lam_finalize_host(int dtype, int64_t n, int32_t d, const void* acc, const void* log_denom,
                      const int64_t* count, void* out);

/* Per-thread pinned host staging buffer `slot` (0..3) of at least `bytes` bytes, for callers of
 * the *_host entry points that marshal nested rows anyway (the C++ drop-in): rows written there
 * cross PCIe as pinned memory.  Valid until the next call with the same slot on this thread;
 * NULL on failure (lam_last_error). */
void* lam_host_buffer(int32_t slot, int64_t bytes);

/* ---- work partitioning (host logic, attention.cpp:164-203) ---------------- */

/* ranges[2*i], ranges[2*i+1] = [begin, end) of device i.  LAM_ERR_VALIDATION with a
 * message containing "divisible" unless num_kv_heads % num_devices == 0. */
int lam_head_partition(int64_t num_kv_heads, int64_t num_devices, int64_t* ranges);
/* Greedy longest-first bin packing; ties to the lower device index. */
int lam_request_partition(const double* kv_sizes, int64_t n, int64_t num_devices,
                          int64_t* device_of, double* device_load, double* imbalance);

/* ---- production decode path (paged HBM KV store) --------------------------
 * KV layout, per layer, per K and V pool:
 *   paged  (page_table != NULL): pool[num_pages][Hkv][page_size][D]; token t of request b
 *          lives in physical page page_table[b*pt_stride + t/page_size], row t%page_size.
 *   dense  (page_table == NULL): pool[B][Hkv][page_size][D], i.e. page_size is the row
 *          capacity l_max of each (request, kv head).
 * Rows are D contiguous elements (256 B for bf16 D=128): every 16-byte vector is aligned.
 * q: [B][Hq][D] in kv_dtype.  out: [B][Hq][D] in out_dtype (kv_dtype or LAM_F32).
 * lse (nullable): [B][Hq] fp32 natural-log sum-exp of the scaled logits.
 * seq_lens: [B] int32 device array; max_len is a host upper bound used for grid sizing.
 * kernel: LAM_KERNEL_AUTO picks GQA_TC (tcgen05 tensor cores, accumulators in TMEM) for 16-bit
 *         KV with D = 128 and 1 <= Hq/Hkv <= 8 — MHA included — (GQA_MMA, mma.sync, when the
 *         environment sets LAM_GQA_TC=0; SIMT for 16-bit MHA when it also sets LAM_MHA_MMA=0) and
 *         SIMT otherwise (fp32 KV, D = 64).  split_tokens: tokens per split-K chunk (0 = auto). */
typedef struct lam_decode_args {
  int32_t kv_dtype;
  int32_t out_dtype;
  int32_t batch;
  int32_t num_q_heads;
  int32_t num_kv_heads;
  int32_t head_dim;
  float scale;
  int32_t page_size;
  int32_t pt_stride;
  int32_t max_len;
  int32_t split_tokens;
  int32_t kernel;
  int64_t num_pages; /* paged: pages in the pool (tensor-map extent); dense: ignored */
  const void* q;
  const void* k_pool;
  const void* v_pool;
  const int32_t* page_table;
  const int32_t* seq_lens;
  void* out;
  float* lse;
  /* elements between consecutive requests' q blocks; 0 = num_q_heads * head_dim.  A packed QKV
   * projection output [B][Hq + 2 Hkv][D] is decoded in place with (Hq + 2 Hkv) * head_dim. */
  int64_t q_batch_stride;
  /* Fused append (optional, both or neither): k_new/v_new hold each request's new token,
   * request b / kv head h at + b * new_batch_stride + h * head_dim (0 = Hkv * head_dim).  The
   * token is position seq_lens[b] - 1: the kernel attends over it from these buffers and writes
   * it into k_pool/v_pool (which must then be writable) — lam_kv_append + lam_decode in one
   * launch. */
  const void* k_new;
  const void* v_new;
  int64_t new_batch_stride;
  /* Optional [B] int32 device permutation of the requests, longest first: work items are claimed
   * in this order (longest-processing-time-first keeps mixed-length batches balanced, in the
   * spirit of request_partition, attention.cpp:185-196).  NULL = request order. */
  const int32_t* request_order;
  /* Overlap with the preceding kernel of the stream (programmatic dependent launch): the launch
   * may start while that kernel drains and stream its first KV tiles, but it reads q, k_new and
   * v_new only after that kernel has completed (griddepcontrol.wait).  The caller guarantees the
   * preceding kernel writes neither page_table, seq_lens, request_order nor the KV rows this
   * launch reads — e.g. consecutive layers of a decode step.  0 = ordinary stream order. */
  int32_t overlap_prev;
} lam_decode_args;

int lam_decode(lam_ctx* ctx, const lam_decode_args* args, void* stream);
/* Kernel family and split count lam_decode would use for these arguments. */
int lam_decode_plan(lam_ctx* ctx, const lam_decode_args* args, int32_t* kernel,
                    int32_t* num_splits, int32_t* split_tokens);
/* Persistent grid (CTAs) lam_decode would launch for these arguments. */
int lam_decode_plan_grid(lam_ctx* ctx, const lam_decode_args* args, int32_t* ctas);

/* Write the new token of every request into the paged pools (bit-exact copy):
 *   k_pool[page_table[b][pos/P]][h][pos%P][:] = k_new[b*new_batch_stride + h*D ...], same for V,
 *   pos = positions[b].  Dense layout when page_table == NULL (pos < page_size).
 *   new_batch_stride = 0 means num_kv_heads * head_dim (dense [B][Hkv][D] inputs). */
int lam_kv_append(int32_t dtype, int32_t batch, int32_t num_kv_heads, int32_t head_dim,
                  int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                  const int32_t* positions, const void* k_new, const void* v_new,
                  int64_t new_batch_stride, void* k_pool, void* v_pool, void* stream);

/* Gather tokens [0, len_b) of every request from the paged pool into a dense
 * [B][Hkv][l_max][D] buffer (inverse of the paging; used to prove bit-exactness). */
int lam_kv_gather(int32_t dtype, int32_t batch, int32_t num_kv_heads, int32_t head_dim,
                  int32_t page_size, int32_t pt_stride, const int32_t* page_table,
                  const int32_t* seq_lens, int32_t l_max, const void* pool, void* dense,
                  void* stream);

/* Host-buffer decode step (the reference-facing end-to-end call, one layer): copies q,
 * k_new, v_new from host memory (pinned for overlap) into args->q / d_k_new / d_v_new,
 * appends the new token of request b at d_positions[b] (lam_kv_append), runs lam_decode
 * into args->out and copies it back to h_out.  Everything is enqueued on `stream`; the
 * caller synchronises.  args->k_pool / args->v_pool must be writable. */
int lam_decode_step_host(lam_ctx* ctx, const lam_decode_args* args, const void* h_q,
                         const void* h_k_new, const void* h_v_new, void* h_out, void* d_k_new,
                         void* d_v_new, const int32_t* d_positions, void* stream);

/* One decode step over n_layers layers from host buffers — the attention worker's end-to-end
 * step.  Layer l's q / k_new / v_new are copied H2D on `copy_stream` into one of two device
 * staging sets while layer l-1 appends + decodes (one fused launch, the new token at
 * seq_lens[b] - 1; d_positions is unused and may be NULL) on `stream`, and each layer's output returns
 * D2H on `copy_stream` as soon as it is ready, so the host copies hide under the HBM-bound
 * attention.  layer_args[l] describes layer l's pools (its q/out fields are ignored: the staging
 * set is used).  d_stage must hold 2 * (q + k_new + v_new + out) bytes of one layer, each part
 * 256-byte aligned (lam_decode_layers_host_stage_bytes).  Returns after enqueueing; the caller
 * synchronises `stream`.
 * Zero-copy: for a one-layer call (or any call with LAM_HOST_ZERO_COPY=1) whose host buffers are
 * all pinned, device-mapped and 16-byte aligned, each layer is a single launch that reads q /
 * k_new / v_new straight from the host buffers and stores the output into h_out (no staging
 * copies; d_stage and copy_stream are unused).  LAM_HOST_ZERO_COPY=0 always stages. */
int lam_decode_layers_host(lam_ctx* ctx, const lam_decode_args* layer_args, int32_t n_layers,
                           const void* const* h_q, const void* const* h_k_new,
                           const void* const* h_v_new, void* const* h_out, void* d_stage,
                           const int32_t* d_positions, void* stream, void* copy_stream);
int64_t lam_decode_layers_host_stage_bytes(const lam_decode_args* layer_args);

/* ---- peer-memory transport (one process per GPU, NVLink / NVSwitch) ----
 *
 * The device-initiated replacement for the scatter / gather collectives of the attention
 * offload step (reference: send-Q / send-KV / return-output, core/src/sim.cpp:310-316; the
 * paper's FHBN transport): the model worker's packed QKV rows and its output
 * rows live in its own HBM, exported to the attention workers over CUDA IPC; the attention
 * worker's decode kernel reads q / k_new / v_new straight from the model worker's memory and
 * stores each output row straight into it.  Readiness is signalled with 32-bit sequence
 * numbers written by the GPU's stream front-end (no SM time, no host round trip). */
#define LAM_MAX_PEERS 8
#define LAM_IPC_HANDLE_BYTES 64

/* cudaMalloc `bytes` (zeroed) and export it: *dptr is the local pointer, handle receives
 * LAM_IPC_HANDLE_BYTES opaque bytes for lam_peer_open in another process. */
int lam_peer_alloc(lam_ctx* ctx, int64_t bytes, void** dptr, void* handle);
int lam_peer_free(lam_ctx* ctx, void* dptr);
/* Map a peer's exported buffer into this process (NVLink peer access enabled). */
int lam_peer_open(lam_ctx* ctx, const void* handle, void** dptr);
int lam_peer_close(lam_ctx* ctx, void* dptr);
/* Stream-ordered sequence numbers: signal writes `value` to each addrs[i] (local or peer)
 * after all prior work of `stream` is visible system-wide; wait blocks `stream` until every
 * addrs[i] >= value (wrap-safe not required: values only grow). */
int lam_stream_signal(lam_ctx* ctx, void* const* addrs, int32_t n, uint32_t value, void* stream);
int lam_stream_wait(lam_ctx* ctx, const void* const* addrs, int32_t n, uint32_t value,
                    void* stream);

/* Request rows of a decode launch grouped by source: rows [s * rows_per_src, (s+1) *
 * rows_per_src) belong to model worker s; row i of source s reads its q heads at
 * q_src[s] + i * args->q_batch_stride (elements), its new k / v heads at
 * q_src[s] + k_new_offset / v_new_offset + i * args->new_batch_stride, and writes its output
 * [Hq][D] at out_dst[s] + i * Hq * D.  Pointers may be peer mappings (lam_peer_open). */
typedef struct lam_peer_io {
  int32_t n_src;
  int32_t rows_per_src;
  const void* q_src[LAM_MAX_PEERS];
  void* out_dst[LAM_MAX_PEERS];
  int64_t k_new_offset;
  int64_t v_new_offset;
  /* Optional in-kernel sequence numbers (no stream operations around the launch): every CTA
   * waits until each wait_flags[i] >= wait_value (i < n_wait) before its first load, and the
   * launch stores done_value to each done_flags[i] (i < n_done, local or peer) once all of
   * its output rows are globally visible.  n_wait = n_done = 0 disables both. */
  int32_t n_wait;
  int32_t n_done;
  uint32_t wait_value;
  uint32_t done_value;
  const uint32_t* wait_flags[LAM_MAX_PEERS];
  uint32_t* done_flags[LAM_MAX_PEERS];
  /* Eager q (optional; the reference's prev/new split, attention.cpp:129-139): with
   * n_wait_kv > 0, wait_flags announce q alone and kv_wait_flags[i] >= kv_wait_value (step
   * launches: epoch + layer + 1) the new K / V rows.  A CTA then starts attending over the cached
   * tokens as soon as q is published and waits for the new rows only when it reaches the tile
   * that holds position seq_len - 1, so the model worker's K/V projection and transfer overlap
   * the attention over the previous tokens. */
  int32_t n_wait_kv;
  uint32_t kv_wait_value;
  const uint32_t* kv_wait_flags[LAM_MAX_PEERS];
  /* Forwarding model worker (optional, step launches only): a model worker whose layer l + 1
   * inputs need nothing but layer l's outputs (a zero-compute stand-in, as in bench.py's
   * strong-scaling runs) is relayed by the launch itself.  A CTA waiting for launch
   * lm = (layer l >= 1, mb) stores epoch + l + 1 to relay_flag (+ mb * flag_mb_stride) once
   * every relay_wait_flags[i] (+ mb * flag_mb_stride, i < n_relay) >= epoch + l.  Layer 0's
   * flag is the caller's.  n_relay = 0 disables it. */
  int32_t n_relay;
  uint32_t* relay_flag;
  const uint32_t* relay_wait_flags[LAM_MAX_PEERS];
  /* Row map (optional, device memory, int32 per attention row; over every micro-batch of a
   * step launch): row b reads source row_src[b] >> 24, row row_src[b] & 0xFFFFFF of that
   * source's block (q / new rows at q_src[s] + row * q_batch_stride, outputs at out_dst[s] +
   * row * num_q_heads * head_dim).  Rows may then come from the sources in any number and
   * order — the request-level partition (attention.cpp:179-203) — and batch need not equal
   * n_src * rows_per_src.  NULL: rows grouped by source, rows_per_src each. */
  const int32_t* row_src;
} lam_peer_io;

/* lam_decode whose q / k_new / v_new / out come from lam_peer_io (args->q, k_new, v_new and out
 * are ignored; fused append is implied; args->lse must be NULL).  batch == n_src *
 * rows_per_src.  With n_wait > 0 and args->overlap_prev the launch uses programmatic dependent
 * launch and never waits for the preceding kernel of the stream: its inputs are ordered by the
 * sequence numbers alone, and the overlap_prev contract (the preceding kernel writes none of
 * page_table, seq_lens, request_order or the KV rows this launch reads or appends) orders the
 * rest.  Without overlap_prev the launch follows ordinary stream order. */
int lam_decode_peer(lam_ctx* ctx, const lam_decode_args* args, const lam_peer_io* io,
                    void* stream);

/* ---- step launch: every layer (and micro-batch) of a decode step in one persistent grid ----
 *
 * Launch lm = layer * n_mb + mb (layer major) is `args` (which describes layer 0, micro-batch 0)
 * with
 *   - rows [mb * rows_per_mb, (mb + 1) * rows_per_mb) of page_table / seq_lens / request_order
 *     (args->batch = n_mb * rows_per_mb; request_order holds indices local to the micro-batch);
 *   - KV pool rows of pool layer (layer0 + layer) % pool_layers: every layer's pool is one slice
 *     of one allocation, pool_layer_rows rows apart (pool viewed as [rows][D], i.e. num_pages *
 *     Hkv * page_size rows per layer when paged);
 *   - q / k_new / v_new / out offset by lm * lm_q_stride / lm * lm_new_stride / lm * lm_out_stride
 *     elements (with io, the per-source buffers of lam_peer_io; its new rows follow q).
 * With io, wait_flags / done_flags address micro-batch 0's sequence numbers and flag_mb_stride
 * (uint32 elements) micro-batch mb's; launch lm waits for and publishes epoch + layer + 1 — a CTA
 * waits when it first claims one of lm's items, and lm's flags are published as soon as all its
 * units are stored.  There is no launch boundary between layers: a CTA that runs out of work in
 * one layer goes on with the next, so layers run concurrently — with a fused append, layers of
 * one step must map to distinct pool layers (else the appended rows of aliased layers race).
 * The grid is every resident CTA.  split_tokens = 0 picks S = 1 unless io waits for inputs
 * (n_wait > 0: each launch then depends on the previous layer), in which case a launch is split
 * until it has two rounds of items on its share of the grid.  args->lse must be NULL. */
typedef struct lam_step_layout {
  int32_t n_layers;
  int32_t n_mb;
  int32_t rows_per_mb;
  int32_t pool_layers;
  int32_t layer0;
  int32_t flag_mb_stride;
  int64_t pool_layer_rows;
  int64_t lm_q_stride;
  int64_t lm_new_stride;
  int64_t lm_out_stride;
  uint32_t epoch;
  /* optional diagnostic (NULL: off): 4 * n_layers * n_mb globaltimer stamps (ns), launch
   * lm = layer * n_mb + mb at [4 lm ..]: first wait for its inputs, inputs seen, last unit
   * done, flags published; then per CTA (the first 1024) 400 records of its work-item claims:
   * claim time, inputs seen, item index (3 words each; 4 n_lm + 1228800 words in all).  The
   * caller fills it with 0xFF bytes before the launch. */
  uint64_t* trace;
} lam_step_layout;

int lam_decode_step(lam_ctx* ctx, const lam_decode_args* args, const lam_step_layout* step,
                    const lam_peer_io* io, void* stream);

/* The attention worker's end-to-end step from host buffers as one step launch: layer l's q /
 * k_new / v_new go H2D on copy_stream into staging region l and are announced by a sequence
 * number the launch waits for in-kernel (the first layers' attention starts while later layers'
 * inputs are still in flight), and layer l's output returns D2H as soon as the launch publishes
 * it.  `args` describes layer 0 (its q / k_new / v_new / out fields are ignored: the staging
 * regions are used; fused append at seq_lens[b] - 1); `step` gives n_layers and the pool layer
 * layout (n_mb must be 1).  d_stage holds lam_decode_step_from_host_stage_bytes(args, n_layers) bytes.
 * Returns after enqueueing; `stream` completes after the last output copy. */
int lam_decode_step_from_host(lam_ctx* ctx, const lam_decode_args* args, const lam_step_layout* step,
                         const void* const* h_q, const void* const* h_k_new,
                         const void* const* h_v_new, void* const* h_out, void* d_stage,
                         void* stream, void* copy_stream);
int64_t lam_decode_step_from_host_stage_bytes(const lam_decode_args* args, int32_t n_layers);

#ifdef __cplusplus
}
#endif

#endif /* LAMINA_ATTN_H */
