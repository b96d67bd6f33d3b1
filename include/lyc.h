/*
 * lyc.h -- C-ABI of the B200-native LycheeDecode hybrid-head decode attention.
 *
 * This is the drop-in boundary for the reference's hot path (the header-only
 * C++ library `hh` under /root/reference/proj/include).  Every entry point
 * names the reference interface it replaces.  Plain pointers and sizes only;
 * device pointers are CUDA global-memory addresses on the current device,
 * streams are cudaStream_t passed as void*.
 *
 * Error model (reference throws, we return):
 *   LYC_EINVAL  <-> std::invalid_argument   (shape / set / config violations)
 *   LYC_ESTATE  <-> std::logic_error        (engine state)
 *   LYC_ECUDA   CUDA runtime failure;  LYC_ENOTSUP unsupported shape on device
 * lyc_last_error() returns the thread-local message of the last failure.
 * Validation happens on the host before any launch; no entry point
 * synchronises the stream except where documented.
 */
#ifndef LYC_H_
#define LYC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LYC_OK 0
#define LYC_EINVAL (-1)
#define LYC_ESTATE (-2)
#define LYC_ECUDA (-3)
#define LYC_ENOTSUP (-4)
#define LYC_ENCCL (-5)

#define LYC_DTYPE_F32 0
#define LYC_DTYPE_BF16 1

/* policy.hpp:22 SparsityPolicy::Kind (TopP / Threshold are host-only) */
#define LYC_POLICY_TOPK 0
#define LYC_POLICY_TOPP 1
#define LYC_POLICY_THRESHOLD 2
#define LYC_POLICY_RATIO 3

#define LYC_SELECT_TOKENS 0 /* token-granular TokenSet (decode_engine.hpp:132) */
#define LYC_SELECT_BLOCKS 1 /* block-granular BlockIndexSet (kernel_sim.hpp:20-42) */
#define LYC_SELECT_NONE 2   /* no selection: every head dense (full-attention baseline) */

const char* lyc_last_error(void);
const char* lyc_version(void);
/* Number of CUDA kernels this thread has launched through the library. */
int64_t lyc_launch_count(void);

/* ---------------------------------------------------------------------------
 * Host planning and cost model (kernel_sim.hpp / policy.hpp).
 * ------------------------------------------------------------------------- */

/* kernel_sim.hpp:63-110 plan_splits.  head_blocks[b*H+g] = list sizes.
 * Outputs split_blocks[b*S+s], head_split_count[b*H+g] and up to max_units
 * unit records (b, s, g, begin, end, head_local_split) in emission order.
 * Returns the number of units (>= 0) or LYC_EINVAL (num_splits < 1, or a
 * batch item with zero blocks). */
int64_t lyc_plan_splits(int64_t batch, int64_t n_kv_heads, const int64_t* head_blocks,
                        int64_t num_splits, int64_t* split_blocks, int64_t* head_split_count,
                        int64_t* units, int64_t max_units);

/* kernel_sim.hpp:284-316 latency_model.  out6 = {total_blocks,
 * pooled_critical_blocks, naive_critical_blocks, bytes_per_block,
 * pooled_critical_bytes, naive_critical_bytes}; out2 = {mean_split_blocks,
 * balance_ratio}. */
int lyc_latency_model(int64_t batch, int64_t n_kv_heads, const int64_t* head_blocks,
                      int64_t num_splits, int64_t bytes_per_block, int64_t* out6, double* out2);

/* policy.hpp:57-62 fraction_budget. */
int64_t lyc_fraction_budget(double frac, int64_t n);

/* ---------------------------------------------------------------------------
 * Operator: hh::kernel::run (kernel_sim.hpp:237-279) on device memory.
 * ------------------------------------------------------------------------- */
typedef struct lyc_workload {
  int64_t batch, n_kv_heads, group_size, d_head, seq_len, block_size;
  int64_t kv_row_stride; /* rows between consecutive (b, g) slabs (>= seq_len) */
  float scale;
  int32_t dtype;         /* LYC_DTYPE_* of k, v, q and out */
  const void* k;         /* device [B*H][kv_row_stride][d] (Workload::keys)   */
  const void* v;         /* device [B*H][kv_row_stride][d] (Workload::values) */
  const void* q;         /* device [B*Hq][d]  (Workload::queries, h = g*G+j)  */
  const int64_t* blk_off;/* HOST CSR offsets [B*H+1] (BlockIndexSet::ids)     */
  const int64_t* blk_ids;/* HOST block ids, ascending per (b, g)              */
} lyc_workload;

/* Validates like Workload::validate (kernel_sim.hpp:136-145), plans like
 * plan_splits, executes every (b, split) cell as one CTA and merges like
 * combine (205-225).  out: device [B*Hq][d] (dtype).  exec_counts (optional):
 * device uint32 [B*H][n_blocks], incremented once per executed (b, g, list
 * index) -- the conservation counter of kernel_sim.hpp:192-193.  Host-side
 * copies of the plan are staged internally (not the decode hot path). */
int lyc_workload_run(const lyc_workload* w, int64_t num_splits, void* out, uint32_t* exec_counts,
                     void* stream);

/* attention.hpp:108-123 args_top_k over a device float vector: the min(k, n)
 * largest, ties to the lower index, written ascending to out (device int32).
 * Returns the count written or an error.  Uses the same cluster radix-select
 * kernel as the decode path. */
int64_t lyc_args_top_k(const float* scores, int64_t n, int64_t k, int32_t* out, void* stream);

/* ---------------------------------------------------------------------------
 * Decoder: the decode_step attention loop (decode_engine.hpp:109-151) with the
 * role mask (rolemap.hpp:33-35, layer 0 forced retrieval at :121), the TopK /
 * Ratio policy (policy.hpp:64-72) and the cross-layer per-KV-head index cache
 * sets_ (decode_engine.hpp:251).
 * ------------------------------------------------------------------------- */
typedef struct lyc_decode_config {
  int32_t n_layers, batch, n_kv_heads, group_size, d_head;
  int32_t dtype;         /* LYC_DTYPE_* */
  int64_t seq_cap;       /* KV rows allocated per (layer, b, g) slab */
  int32_t policy_kind;   /* LYC_POLICY_*: TopK / Ratio (step kernel), TopP / Threshold
                            (per-layer kernels, token selection only) */
  int32_t select_mode;   /* LYC_SELECT_TOKENS or LYC_SELECT_BLOCKS */
  int64_t top_k;         /* TopK budget in tokens (blocks mode: ceil(k / block_size) blocks) */
  double ratio;          /* Ratio theta in (0, 1); TopP p in (0, 1]; Threshold tau > 0 */
  int32_t block_size;    /* 64 (tile) */
  int32_t num_splits;    /* splits per batch item; 0 = one CTA per SM */
  float scale;           /* softmax scale; 0 -> 1/sqrt(d_head) */
  const uint8_t* roles;  /* host [n_layers][n_kv_heads]; 0 = Retrieval, 1 = Sparse */
} lyc_decode_config;

typedef struct lyc_decoder lyc_decoder;

int lyc_decoder_create(const lyc_decode_config* cfg, lyc_decoder** out);
int lyc_decoder_destroy(lyc_decoder* dec);

/* One decode step over all layers.  Device buffers:
 *   q   [n_layers][B][Hq][d]            queries of the step
 *   k,v [n_layers][B][H][seq_cap][d]    caches, rows 0..seq_len-1 valid
 *   out [n_layers][B][Hq][d]            attention outputs
 * seq_len = t+1 (current token included, decode_engine.hpp:98).  Stream
 * ordered; the index cache (sets_) is updated in place.
 * On the step kernel (lyc_decoder_is_fused) a step is two launches -- the
 * device planner (plan.cu: the split plan for this length, computed in the
 * stream) and the persistent step kernel -- with no host synchronisation,
 * no host-to-device copy and no allocation, so seq_len may change on every
 * call (token-after-token decode).  On the per-layer kernels (TopP /
 * Threshold, shard mode) a new length is planned on the host and uploaded
 * stream-ordered from pinned staging. */
int lyc_decoder_step(lyc_decoder* dec, const void* q, const void* k, const void* v,
                     int64_t seq_len, void* out, void* stream);

/* A variable-length batch: seq_lens is host [B], item b's sequence length
 * (rows 0..seq_lens[b]-1 of its slabs valid, current token included).  The
 * reference's Workload has one seq_len for the whole batch (kernel_sim.hpp:126)
 * and DecodeEngine runs one sequence (decode_engine.hpp:95-151); this is B
 * independent engines' decode_step in one call: each item's retrieval heads
 * attend its own rows, select from them with its own budget (TopK: min(k, len),
 * Ratio: ceil((1 - theta) * len)), and its sparse heads read those sets.  Equal
 * lengths run exactly as lyc_decoder_step; unequal ones run on the same step
 * kernel with every pool cut across all CTAs of the batch.  Not supported in
 * shard mode. */
int lyc_decoder_step_varlen(lyc_decoder* dec, const void* q, const void* k, const void* v,
                            const int64_t* seq_lens, void* out, void* stream);

/* The same with DEVICE-resident lengths (int64 [B], current token included),
 * read by the device planner when the step runs: a captured graph
 * (lyc_decoder_capture_dev) replays t, t+1, t+2, ... as the caller advances
 * the lengths in the stream (e.g. with lyc_kv_append_dev).  Invalid lengths
 * (< 1 or > seq_cap) make the step a no-op, reported by lyc_decoder_status.
 * Step kernel only (LYC_ENOTSUP otherwise). */
int lyc_decoder_step_dev(lyc_decoder* dec, const void* q, const void* k, const void* v,
                         const int64_t* d_seq_lens, void* out, void* stream);
/* LYC_OK, or LYC_EINVAL if the last device-planned step rejected its lengths
 * (synchronises `stream`). */
int lyc_decoder_status(lyc_decoder* dec, void* stream);

/* Single layer (decode_engine.hpp:120-143): q_l/out_l are [B][Hq][d]; k/v are
 * the full caches.  Layers must be issued in order within a step, the model's
 * own projections in between (q of layer l+1 depends on layer l's output).
 * On the step kernel this is ONE launch of the persistent step kernel over
 * [layer, layer + 1) -- attention and split-KV merge of the layer, and the
 * PREVIOUS layer's selection (deferred into this launch, LYC_TUNE_DEFER_SELECTION;
 * the last layer selects in its own launch) -- plus the device planner at
 * layer 0 (or when seq_len changes).  out_l is final when the call's work
 * completes; the layer's index sets when the next layer's does (or after
 * lyc_decoder_sync_sets). */
int lyc_decoder_layer(lyc_decoder* dec, int32_t layer, const void* q_l, const void* k,
                      const void* v, int64_t seq_len, void* out_l, void* stream);

/* Capture lyc_decoder_step into a CUDA graph for fixed pointers / seq_len,
 * then replay it.  replay returns LYC_ESTATE if nothing was captured.  The
 * graph replays the captured lengths: on the step kernel it contains the
 * device planner; on the per-layer kernels replay re-plans to the captured
 * lengths when another length was planned since (stream-ordered upload). */
int lyc_decoder_capture(lyc_decoder* dec, const void* q, const void* k, const void* v,
                        int64_t seq_len, void* out, void* stream);
/* The same for a variable-length batch (host seq_lens [B], as in
 * lyc_decoder_step_varlen); replay re-runs the captured lengths. */
int lyc_decoder_capture_varlen(lyc_decoder* dec, const void* q, const void* k, const void* v,
                               const int64_t* seq_lens, void* out, void* stream);
/* The same with device-resident lengths (lyc_decoder_step_dev): every replay
 * plans the lengths the array holds when it runs. */
int lyc_decoder_capture_dev(lyc_decoder* dec, const void* q, const void* k, const void* v,
                            const int64_t* d_seq_lens, void* out, void* stream);
int lyc_decoder_replay(lyc_decoder* dec, void* stream);

/* The device index cache: ids [B*H][k_cap] int32 (ascending token ids, or
 * block ids in blocks mode), counts [B*H] int32.  After per-layer calls the
 * selection of the last layer issued may still be pending (it runs with the
 * next layer's launch): lyc_decoder_sync_sets completes it in `stream`
 * (every other entry point does so itself). */
int lyc_decoder_sync_sets(lyc_decoder* dec, void* stream);
int lyc_decoder_index_cache(lyc_decoder* dec, int32_t** ids, int32_t** counts, int64_t* k_cap);

/* Number of kernel launches one step issues (for the bench's gpu_launches). */
int64_t lyc_decoder_launches_per_step(lyc_decoder* dec, int64_t seq_len);

/* Algorithmic HBM bytes of one step: K/V rows touched + Q
 * in + O out + index reads/writes. */
int64_t lyc_decoder_step_bytes(lyc_decoder* dec, int64_t seq_len);

/* Algorithmic HBM bytes of layer `layer`'s attention kernel (K/V rows + Q + O). */
int64_t lyc_decoder_layer_attn_bytes(lyc_decoder* dec, int32_t layer, int64_t seq_len);

/* Kernel timing: when enabled, CUDA events bracket every attention-kernel
 * launch of subsequent steps (also inside a captured graph, as event nodes).
 * lyc_decoder_attn_ms fills ms[n_layers] with the durations of the most recent
 * completed step (synchronises on the last event). */
int lyc_decoder_set_timing(lyc_decoder* dec, int enable);
int lyc_decoder_attn_ms(lyc_decoder* dec, float* ms);

/* 1 when lyc_decoder_step runs the persistent whole-step kernel (one launch:
 * attention, split-KV merge and selection of every layer), 0 when it issues
 * per-layer kernels (attention, merge, cluster top-k).  In fused mode
 * lyc_decoder_attn_ms reports the step kernel's duration in ms[0] (or one
 * duration per layer after lyc_decoder_layer calls). */
int lyc_decoder_is_fused(lyc_decoder* dec);

/* Tuning / experiment knobs (never needed for correctness):
 *   LYC_TUNE_RING_STAGES       K/V ring stages in use (0 = all that fit);
 *   LYC_TUNE_PER_LAYER_KERNELS 1 = run steps on the per-layer kernels
 *                              (attention, merge, cluster top-k), 0 = back to
 *                              the step kernel when the decoder has one;
 *   LYC_TUNE_PDL               0 = plain stream serialisation of the step's launches. */
#define LYC_TUNE_RING_STAGES 1
#define LYC_TUNE_PER_LAYER_KERNELS 2
#define LYC_TUNE_PDL 3  /* 1 (default) = programmatic dependent launch of planner / step kernels */
/* 1 (default): with per-layer calls (lyc_decoder_layer) a layer's selection
 * runs in the NEXT layer's launch, beside its attention (only the units that
 * read those sets wait for it) instead of at the tail of its own launch */
#define LYC_TUNE_DEFER_SELECTION 4
int lyc_decoder_tune(lyc_decoder* dec, int32_t what, int64_t value);

/* Step timeline (fused mode): when enabled, the step kernel stamps
 * %globaltimer (ns) for 8 events per layer per CTA: consumers begin / end,
 * epilogue sees the layer's attention done, merge done, selection barriers
 * 0-2, selection done.  lyc_decoder_trace copies [n_layers][8][n_ctas]
 * stamps into out (cap entries) and returns the count (out = NULL: size query). */
int lyc_decoder_set_trace(lyc_decoder* dec, int enable);
/* Set trace (fused mode, a debugging / parity aid): when enabled, every step
 * also records each layer's emitted index sets -- the StepTrace of
 * decode_engine.hpp:26-32, 144-147 -- so per-layer selections of the
 * whole-step kernel can be checked.  lyc_decoder_traced_sets copies
 * [n_layers][B*H][k_cap] ids and [n_layers][B*H] counts (-1: no set emitted
 * at that layer) to host buffers (synchronises) and returns k_cap
 * (ids = NULL: returns k_cap only). */
int lyc_decoder_set_trace_sets(lyc_decoder* dec, int enable);
int64_t lyc_decoder_traced_sets(lyc_decoder* dec, int32_t* ids, int32_t* counts, int64_t cap);
int64_t lyc_decoder_trace(lyc_decoder* dec, unsigned long long* out, int64_t cap);

/* ---------------------------------------------------------------------------
 * KV-sequence sharding across GPUs (the inter-GPU form of the
 * split pooling of kernel_sim.hpp:63-110 with the combine of :205-225).
 * Rank p of P holds rows [row_begin, row_begin + n_local) of every head's
 * cache, numbered locally (k, v point at local row 0 of layer 0; seq_cap is
 * the slab stride).  Per layer, in order:
 *   1. lyc_shard_layer: local attention partials -- fp32 normalized o
 *      [B][Hq][d] and base-2 LSE [B][Hq] -- and, for the layer's retrieval
 *      heads, the exact local top-k of this shard's pooled scores as
 *      (order-preserving key, GLOBAL token id) rows [B*H][k_cap], ascending,
 *      padded with key 0 / id -1.  Sparse heads read this rank's filtered
 *      index-cache rows (written by step 3 of an earlier layer).
 *   2. the caller all-gathers [part_o | part_lse | cand_key | cand_idx] of all
 *      ranks in rank order (one packed ncclAllGather).
 *   3. lyc_shard_merge: identically on every rank, the rank-ordered LSE merge
 *      into out_l (dtype) and, per retrieval (b, g), the global top-k over the
 *      gathered candidates (ties to the lower global id) -> global_sets
 *      [B*H][k_cap] (optional) and this rank's filtered index-cache row.
 * seq_total = sum of n_local over ranks (the global budget is computed on it).
 * rank_stride: distance in 4-byte words between consecutive ranks' blocks when
 * the four fields are packed per rank in that order into one gathered buffer
 * (one collective); 0 when each field was gathered into its own array.
 * Token-mode selection only (LYC_ENOTSUP for block mode). */
int lyc_shard_layer(lyc_decoder* dec, int32_t layer, const void* q_l, const void* k,
                    const void* v, int64_t n_local, int64_t row_begin, float* part_o,
                    float* part_lse, uint32_t* cand_key, int32_t* cand_idx, void* stream);
int lyc_shard_merge(lyc_decoder* dec, int32_t layer, int32_t world, const float* all_o,
                    const float* all_lse, const uint32_t* all_key, const int32_t* all_idx,
                    int64_t rank_stride, int64_t n_local, int64_t row_begin, int64_t seq_total,
                    void* out_l, int32_t* global_sets, void* stream);

/* ---------------------------------------------------------------------------
 * Device KV write path (kv_cache.hpp:14-69).  The device
 * cache is the decoder's layout [n_layers][B][H][seq_cap][d] (dtype elements),
 * one K and one V allocation.  lyc_kv_write copies n_rows rows per (b, g) of
 * one layer, from src [B][H][n_rows][d] (same dtype, contiguous) to cache rows
 * [pos, pos + n_rows):
 *   KvCache::append (23-29) + commit_row (32): n_rows = 1 at pos = length,
 *     every head of the layer at once (the caller advances the length);
 *   KvCache::overwrite (34-42): n_rows = 1 at any pos < length, or a window
 *     (cache correction rewrites the trailing W rows).
 * layer = -1 writes every layer at once (src [n_layers][B][H][n_rows][d]):
 * one launch for a decoded token's rows of the whole model.
 * LYC_EINVAL when pos + n_rows > seq_cap or the layer is out of range.
 * Stream-ordered, graph-capturable, no allocation. */
typedef struct lyc_kv_layout {
  int32_t n_layers, batch, n_kv_heads, d_head;
  int32_t dtype;         /* LYC_DTYPE_* */
  int32_t pad;
  int64_t seq_cap;
} lyc_kv_layout;
int lyc_kv_write(void* k_cache, void* v_cache, const lyc_kv_layout* layout, int32_t layer,
                 int64_t pos, int64_t n_rows, const void* k_src, const void* v_src, void* stream);
/* KvCache::append of the current token with device-resident lengths: writes
 * row d_seq_lens[b] - 1 of every (b, g) of `layer` (-1: all layers) from src
 * [(n_layers)][B][H][d]; rows outside [0, seq_cap) are skipped.  Graph-
 * capturable (the companion of lyc_decoder_step_dev). */
int lyc_kv_append_dev(void* k_cache, void* v_cache, const lyc_kv_layout* layout, int32_t layer,
                      const int64_t* d_seq_lens, const void* k_src, const void* v_src,
                      void* stream);

/* ---------------------------------------------------------------------------
 * Cache-correction attention (decode_engine.hpp:164-204):
 * after the K/V rows of the last `window` positions [start, start + window)
 * were rewritten (lyc_kv_write), window position i (p = start + i) attends
 * keys [0, p] of layer `layer` -- all window x Hq query rows of a KV head in
 * one prefill-style pass over the cache (bf16, d 64 or 128; fp32 caches with
 * d <= 128 through a simple one-warp-per-row kernel for small configs).
 *   q, out: device [B][window][Hq][d] in the cache dtype (Hq = n_kv_heads * group_size);
 *   workspace: device, >= lyc_window_workspace(...) bytes.
 * The surrounding per-position projections (compute_qkv, attn_project_residual,
 * ffn_residual) are the model's, not this library's. */
int64_t lyc_window_workspace(const lyc_kv_layout* layout, int32_t group_size, int32_t window);
int lyc_window_attention(const lyc_kv_layout* layout, int32_t layer, const void* k_cache,
                         const void* v_cache, int32_t group_size, float scale, int64_t start,
                         int32_t window, const void* q, void* out, void* workspace,
                         int64_t workspace_bytes, void* stream);

/* Index-set refresh of cache correction (decode_engine.hpp:190-197,
 * refresh_sets_on_correction): every KV head's set is re-selected from the
 * pooled query (gqa_pool_queries, attention.hpp:127-146) of the LAST window
 * position against keys [0, len) of `layer`, with the decoder's policy
 * (select_tokens on the dense-attention weights, policy.hpp:64-104), into the
 * decoder's index cache (sets_ of every (b, g)).  q_last: device [B][Hq][d],
 * that position's queries at `layer`; k: the decoder's K cache
 * [n_layers][B][H][seq_cap][d].  The reference refreshes at every layer of the
 * window pass, each layer overwriting sets_, so the state it leaves is this
 * call for its last layer.  Stream-ordered; allocates its key scratch on the
 * first call only. */
int lyc_decoder_refresh_sets(lyc_decoder* dec, int32_t layer, const void* q_last, const void* k,
                             int64_t len, void* stream);

/* ---------------------------------------------------------------------------
 * The decode operations around the attention in the reference's toy model
 * (toy_model.hpp:161-274), for an end-to-end decode step:
 * one bf16 GEMV kernel (HBM-bound at batch 1) with the vector work fused in.
 *   y = W . x,  W bf16 [M][K] (row-major per output: the transpose of the
 *   reference's Matrix [in][out], matvec_f :171-180), x fp32 (the residual
 *   stream) or bf16 [K]; with `gain` the input is rmsnorm'ed first
 *   (:161-169, eps default 1e-6).  Epilogues:
 *   STORE      y = W x (fp32 [M])                      -- output_logits (:269-274)
 *   RESIDUAL   y += W x (fp32)                         -- attn_project_residual /
 *                                                          ffn_residual adds (:245-267)
 *   SILU_BF16  yb = silu(W x) (bf16)                   -- the FFN's W1 (:259-267)
 *   QKV_ROPE   rows [0, nq*d): q (rotary, :184-194) -> q_out bf16 [nq][d];
 *              rows [nq*d, (nq+nkv)*d): the token's K rows (rotary), the rest
 *              its V rows, written to cache row `pos` of KV head g at
 *              k_cache / v_cache + g * slab_stride (bf16)  -- compute_qkv (:218-240)
 * K must be a multiple of 8 and <= 49152; W, x / xb and gain 16-B aligned. */
/* flags: the next launch in the stream is another lyc_gemv -- let it be
 * scheduled as this launch's CTAs finish (programmatic launch trigger; it
 * still waits for this launch's completion before reading its outputs).
 * Measured: a bare GEMV chain 3 % faster; the toy model's decode step, where
 * the chains are short and alternate with the attention step, 6 % slower. */
#define LYC_GEMV_FLAG_NEXT_IS_GEMV 1
#define LYC_GEMV_STORE 0
#define LYC_GEMV_RESIDUAL 1
#define LYC_GEMV_SILU_BF16 2
#define LYC_GEMV_QKV_ROPE 3
typedef struct lyc_gemv_desc {
  int64_t M, K;
  const void* w;          /* bf16 [M][K] */
  const float* x;         /* fp32 [K], or NULL */
  const void* xb;         /* bf16 [K], or NULL */
  const float* gain;      /* rmsnorm gain [K], or NULL */
  float eps;
  int32_t mode;           /* LYC_GEMV_* */
  float* y;               /* STORE / RESIDUAL: fp32 [M] */
  void* yb;               /* SILU_BF16: bf16 [M] */
  void* q_out;            /* QKV_ROPE */
  void* k_cache;
  void* v_cache;
  int64_t slab_stride;
  int32_t nq, nkv, d;
  int32_t flags;          /* LYC_GEMV_FLAG_* */
  int64_t pos;
  /* optional L2 prefetch hint: the first prefetch_bytes of the NEXT launch's
   * weights (16-B aligned, or NULL / 0).  Each warp issues its share after its
   * own rows, so the next GEMV's first loads hit L2 instead of waiting out the
   * launch boundary on HBM. */
  const void* prefetch;
  int64_t prefetch_bytes;
} lyc_gemv_desc;
int lyc_gemv(const lyc_gemv_desc* g, void* stream);

/* ---------------------------------------------------------------------------
 * Test hook: the device planner (run sequentially on the host) against the
 * host-order planner for a decoder configuration and lengths (seq_lens: host
 * [B] or NULL), every layer; LYC_OK when they agree exactly, LYC_ESTATE with
 * the first difference otherwise.  No GPU needed. */
int lyc_plan_selftest(const lyc_decode_config* cfg, int64_t seq_len, const int64_t* seq_lens,
                      int32_t n_sms);

#ifdef __cplusplus
}
#endif

#endif /* LYC_H_ */
