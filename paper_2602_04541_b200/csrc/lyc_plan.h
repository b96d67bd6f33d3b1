// lyc_plan.h -- device work descriptors shared by the host planner (capi.cu)
// and the kernels (attn_core.cuh, attn.cu, step.cu).  Plain structs, uploaded
// once per plan and read-only on the device.
//
// A "slot" is one (batch item b, KV head g) of one layer.  Its work list is a
// sequence of ITEMS; each item expands to ceil(block_size/64) TILES of <= 64
// KV rows (the kernels' unit of TMA staging):
//   ITEM_DENSE  item i -> rows [i*bs, min((i+1)*bs, seq))          retrieval head
//   ITEM_BLOCKS item i -> rows of block list[i]                     BlockIndexSet
//   ITEM_TOKENS item i -> rows list[i*64 .. min(i*64+64, list_len)) TokenSet
// The pooled plan (kernel_sim.hpp:63-110) cuts each batch item's concatenated
// item list into num_splits contiguous chunks; a chunk's per-slot pieces are
// UNITS.  One CTA executes one split (Algorithm 2).
#pragma once
#include <cuda.h>  // CUtensorMap (type only; encoded through the runtime's driver entry point)
#include <stdint.h>

#define LYC_TILE 64
#define LYC_BINS 2048
// First radix pass fused into the attention consumers (per-CTA smem histogram).
#define LYC_H1_BITS 12
#define LYC_H1_BINS (1 << LYC_H1_BITS)
// Global h1 rows carry 64 coarse bins (top 6 bits) after the fine bins.
#define LYC_H1_COARSE 64
#define LYC_H1_ROW (LYC_H1_BINS + LYC_H1_COARSE)
// Each selection row keeps LYC_H1_COPIES copies of its first-pass histogram;
// CTA c flushes into copy c % LYC_H1_COPIES (fewer same-address reductions in
// L2 -- the release that publishes a unit waits for them); readers sum them.
#define LYC_H1_COPIES 8
#define LYC_H1_STRIDE (LYC_H1_COPIES * LYC_H1_ROW)
#define LYC_TRACE_EVENTS 24  // step-timeline stamps per layer per CTA

enum { ITEM_DENSE = 0, ITEM_BLOCKS = 1, ITEM_TOKENS = 2 };

struct LycSlot {
  int64_t kv_off;        // element offset of this slot's [S_cap][d] K/V slab
  const int32_t* list;   // ITEM_BLOCKS: block ids; ITEM_TOKENS: token ids (device)
  int32_t kind;          // ITEM_*
  int32_t n_items;       // items in the work list
  int32_t list_len;      // ITEM_TOKENS: number of token ids
  int32_t first_unit;    // global index of the slot's first unit (units are consecutive)
  int32_t n_units;       // head_split_count
  int32_t q_row;         // first query/output row: b*Hq + g*G
  int32_t sel;           // selection output row (-1: none)
  int32_t dep;           // layer whose selection wrote `list` (-1: none / already complete)
  const int32_t* count;  // ITEM_TOKENS: device count of valid ids (<= list_len), or nullptr
  int32_t seq;           // rows of this slot's sequence (seq_len of its batch item)
  int32_t item;          // its batch item b
};

struct LycUnit {
  int32_t slot;
  int32_t begin;  // item range [begin, end) in the slot's work list
  int32_t end;
  int32_t hls;    // head-local split id
};

// Selection outputs written by the attention consumers for slots with sel >= 0.
enum { SEL_NONE = 0, SEL_TOKEN_KEYS = 1, SEL_BLOCK_KEYS = 2 };

// Everything one layer's attention needs except the tensor maps.
struct LycView {
  const void* k;            // [...][S_cap][d] (slot kv_off)
  const void* v;
  const void* q;            // [rows][d]
  void* out;                // [rows][d]
  const LycSlot* slots;
  const LycUnit* units;
  const LycSlot* unit_slots;// [n_units] copy of each unit's slot (one coalesced load per layer)
  const int32_t* split_off; // [B * n_splits + 1] unit ranges per (b, split)
  float* part_o;            // [n_units][G][d]  normalized partial outputs
  float* part_lse;          // [n_units][G]     base-2 log-sum-exp
  uint32_t* sel_keys;       // [n_sel][sel_stride]
  uint32_t* hist1;          // optional [n_sel][LYC_H1_ROW]: fused first radix pass (+ coarse bins)
  uint32_t* exec_counts;    // optional [n_slots][counts_stride] per item
  float* out_f32;           // optional: fp32 outputs [rows][d] instead of `out` (shard partials)
  float* out_lse;           // optional with out_f32: base-2 LSE per output row
  uint32_t* slot_ctr;       // optional [slots][16]: word 12 counts the slot's finished units
  unsigned long long* trace_l;  // optional step timeline of this layer [LYC_TRACE_EVENTS][n_ctas]
  int32_t trace_ctas;
  int64_t sel_stride;
  int32_t counts_stride;
  int32_t n_splits;         // splits per batch item (grid.x)
  int32_t seq_len;
  int32_t block_size;
  int32_t group;            // G
  int32_t sel_mode;         // SEL_*
  float scale;              // softmax scale (1/sqrt(d))
  float scale_log2;         // scale * log2(e)
  int32_t stages;           // ring stages in use (<= the kernel's capacity; 0 = all)
  int32_t early_exit;       // per-layer kernel: units may end early (device-count sets)
  const int32_t* seq_of;    // step kernel: live length of each batch item (by slot.item), or null
};

struct LycAttnParams {
  // 2D TMA views of the K and V caches: dim0 = d (elements), dim1 = all rows
  // of all slabs; box = one 128-B column panel (bf16, 128B swizzle) or the
  // whole row (fp32, no swizzle) x 64 rows.
  CUtensorMap tmap_k;
  CUtensorMap tmap_v;
  LycView v;
};

struct LycMergeTask {       // one (slot, q head j) pair needing a split-KV merge
  int32_t slot;
  int32_t j;
  int32_t first_unit;       // the slot's partials (copied from LycSlot: one load per task)
  int32_t n_units;
  int32_t q_row;
  int32_t pad;
};

struct LycMergeParams {
  const float* part_o;
  const float* part_lse;
  const LycSlot* slots;
  const LycMergeTask* tasks;
  void* out;
  float* out_f32;           // optional: fp32 outputs + base-2 LSE (shard partials)
  float* out_lse;
  int32_t n_tasks;
  int32_t group;
  int32_t chunks;           // ceil(d / 32)
  int32_t d;
};

struct LycTopkParams {
  uint32_t* keys;           // [n_sel][key_stride] order-preserving keys
  int64_t key_stride;
  int32_t n;                // candidates per selection row (seq_len or n_blocks)
  int32_t k;                // how many to keep (already min(k, n))
  int32_t* out;             // index cache base
  const int32_t* out_row;   // [n_sel] -> row in the index cache
  int64_t out_stride;       // index cache row stride (k_cap)
  int32_t* out_count;       // [cache rows] number of ids written (may be null)
  int32_t slice;            // keys per CTA of the cluster
  int32_t clear_keys;       // zero keys after use (block-max keys are atomicMax'ed)
  const int32_t* row_n;     // optional [n_sel]: candidates of each row (variable-length batch)
  const int32_t* row_k;     // optional [n_sel]: ids kept per row (<= row_n)
};

// TopP / Threshold selection (policy.cu): one CTA per selection row.
#define LYC_POLICY_KIND_TOPP 1       // = LYC_POLICY_TOPP (include/lyc.h)
#define LYC_POLICY_KIND_THRESHOLD 2  // = LYC_POLICY_THRESHOLD
struct LycPolicyParams {
  const uint32_t* keys;     // [n_sel][key_stride] order-preserving keys of sum_j q_j.k
  int64_t key_stride;
  int32_t n;                // tokens per selection row (seq_len)
  int32_t kind;             // LYC_POLICY_KIND_*
  double value;             // p (TopP) or tau (Threshold)
  float score_scale;        // key value -> the reference's scaled pooled score (bf16 keys: scale / G)
  int32_t pad;
  int32_t* out;             // index cache base
  const int32_t* out_row;   // [n_sel] -> row in the index cache
  int64_t out_stride;       // index cache row stride (k_cap)
  int32_t* out_count;       // [cache rows] size of each set
  const int32_t* row_n;     // optional [n_sel]: tokens of each row (variable-length batch)
};

// ---------------------------------------------------------------------------
// Persistent decode-step kernel (step.cu): one launch runs every layer.
struct LycLayerDesc {
  const LycSlot* slots;
  const LycUnit* units;
  const LycSlot* unit_slots;
  const int32_t* split_off;
  const LycMergeTask* merges;
  const int32_t* sel_rows;  // selection index -> index-cache row
  const int32_t* sel_n;     // optional [n_sel] (variable-length batch): keys of each row
  const int32_t* sel_k;     // optional [n_sel]: ids kept per row
  int32_t n_merges;
  int32_t n_sel;
};

// Per-layer device counters (monotonic; a step adds n_ctas to each).
enum {
  CTR_PLAN = 7,      // (layer 0 only) CTAs past the in-kernel re-plan
  CTR_ATTN = 0,      // CTAs that finished the layer's attention units
  CTR_MERGE = 1,     // CTAs that finished the layer's merge tasks (layer output final)
  CTR_SEL0 = 2,      // selection phase barriers
  CTR_SEL1 = 3,
  CTR_SEL2 = 4,
  CTR_SEL3 = 5,
  CTR_SELDONE = 6,   // CTAs that finished writing the layer's index-cache rows
  CTR_PER_LAYER = 8
};
// Counters sit 256 B apart (separate L2 lines / slices): many CTAs poll them.
#define LYC_CTR_STRIDE 64
#define LYC_CTR(base, l, e) ((base) + ((size_t)(l) * CTR_PER_LAYER + (e)) * LYC_CTR_STRIDE)
// Two counter sets, used by alternate launches (the launch parity): a launch
// counts up from zero in its own set and zeroes the other one, so no counter
// is ever reset on the host and a launch may cover any layer range.  After
// the sets: the control words (parity, then the exit count).
#define LYC_CTR_SET_WORDS(n_layers) ((size_t)(n_layers) * CTR_PER_LAYER * LYC_CTR_STRIDE)
#define LYC_CTR_WORDS(n_layers) (2 * LYC_CTR_SET_WORDS(n_layers) + 2 * LYC_CTR_STRIDE)

// ---------------------------------------------------------------------------
// Seq-parametric plan of the fused step (plan.cuh): computed on the device by
// one CTA per layer from the static role map and the step's lengths, so a
// token-after-token decode never re-plans on the host.
#define LYC_PLAN_MAX_B 160   // batch items whose lengths travel by value
#define LYC_PLAN_THREADS 256

struct LycPlanHdr {          // the last plan's lengths and the last step's status (device)
  int32_t seq_len;           // max over the batch (of the last plan)
  int32_t n_keys;            // selection keys per row (seq_len, or blocks)
  int32_t k_sel;             // ids kept per row at seq_len
  int32_t status;            // 0 ok; 1 invalid lengths (that step did nothing)
  int32_t bad_item;          // first batch item with an invalid length
  int32_t pad[3];
};
// The plan depends on the lengths only through its KEY: each item's dense
// block count nb and sparse budget kb, and the selection items per row.  A
// step whose key matches reuses the plan (a growing sequence re-plans once
// per 64 tokens); per-token values (lengths, selection sizes) are read live
// by the step kernel.  Per layer the planner keeps the key its plan was made
// for: [valid, items, nb[B], kb[B]].
#define LYC_PLAN_KEY_INTS(B) (2 + 2 * (B))

struct LycPlanIn {
  int32_t NL, B, H, G, D, S;  // layers, batch, KV heads, group, head dim, splits per item
  int32_t bs;                 // block size (64)
  int32_t select_mode;        // LYC_SELECT_* (include/lyc.h)
  int32_t policy_kind;        // LYC_POLICY_TOPK / RATIO
  int32_t item_keys;          // selection keys per epilogue item (step.cu kItemKeys)
  int64_t seq_cap, k_cap, top_k;
  double ratio;
  const uint8_t* roles;       // device [NL][H], 0 = Retrieval
  int32_t* idx;               // device index cache (values stored in token / block slots)
  LycLayerDesc* layers;       // [NL]: per-layer arrays (fixed at create); n_merges / n_sel written
  LycPlanHdr* hdr;
  int32_t* keys;              // [NL][LYC_PLAN_KEY_INTS(B)] the key of each layer's plan
  int32_t max_units;          // capacity of each layer's unit arrays
  int32_t max_merges;
  // the step's lengths: dlens (device [B], current token included) when set,
  // else lens[b] (by value) when has_lens, else seq for every item
  const int64_t* dlens;
  int64_t seq;
  int32_t has_lens;
  int32_t pad_;
  int32_t lens[LYC_PLAN_MAX_B];
};

struct LycStepParams {
  CUtensorMap tmap_k;
  CUtensorMap tmap_v;
  const void* k;
  const void* v;
  const void* q;             // [n_layers][B][Hq][d]
  void* out;                 // [n_layers][B][Hq][d]
  int64_t q_layer_stride;    // elements between consecutive layers of q / out
  const LycLayerDesc* layers;
  float* part_o;
  float* part_lse;
  uint32_t* sel_keys;        // [2 parity][max_sel][sel_stride]
  int64_t sel_stride;
  uint32_t* hist;            // [2 parity][max_sel][LYC_H1_ROW] fused first-pass histograms
  uint32_t* sel_bitmap;      // [2 parity][max_sel][bitmap_stride] selected-key bitmaps
  int64_t bitmap_stride;
  uint32_t* sel_cand;        // [2 parity][max_sel][2][sel_stride] boundary-bin candidates: keys, indices
  uint32_t* sel_ccnt;        // [2 parity][max_sel][256] per item: candidates [0,64), definite keys [64,128); row prefix [192,195)
  uint32_t* sel_csub;        // [2 parity][max_sel][64 items][256 u16] bucket starts of each item's candidates
  uint32_t* sel_rowctr;      // [2 parity][n_layers][max_sel][16]: per selection row words 0 / 8
                             // (items classified / holding copies); per SLOT word 12 (units done)
  int64_t rowctr_set;        // words of one sel_rowctr set
  uint32_t* ctr;             // LYC_CTR counters: [2 parity][n_layers][CTR_PER_LAYER], then control
  LycPlanHdr* hdr;           // the plan key; the step status
  int32_t* idx;              // index cache [B*H][idx_stride]
  int64_t idx_stride;
  int32_t* idx_count;        // [B*H]
  unsigned long long* trace; // optional [n_layers][8 events][n_ctas] %globaltimer stamps
  int32_t* set_trace;        // optional [n_layers][B*H][idx_stride]: each layer's emitted sets
  int32_t* set_trace_count;  // optional [n_layers][B*H]
  int32_t n_layers;
  int32_t l_begin, l_end;    // the layers of this launch (q / out point at layer l_begin)
  int32_t max_sel;
  int32_t n_splits;
  int32_t n_ctas;            // CTAs = n_splits * batch (grid index = b * n_splits + split)
  int32_t block_size;
  int32_t group;
  int32_t sel_mode;
  float scale;
  float scale_log2;
  int32_t stages;            // attention ring stages in use (0 = all)
  int32_t uniform;           // host lengths, every batch item plan.seq: the lengths below hold
  int32_t uni_nsel, uni_ksel;  //   selection keys / ids kept per row at plan.seq (plan_item_key)
  int32_t sel_defer_in;      // run layer l_begin - 1's selection (deferred by the previous launch)
  int32_t sel_defer_out;     // leave layer l_end - 1's selection to the next launch
  LycPlanIn plan;            // the step's lengths + the planner's input (re-plan in the kernel)
};

// Toy-model decode GEMV (model.cu, include/lyc.h lyc_gemv).
struct LycGemvParams {
  const void* w;            // bf16 [M][K]
  int64_t M, K;
  const float* x;           // fp32 input [K] (the residual stream), or null
  const void* xb;           // bf16 input [K], or null
  const float* gain;        // rmsnorm gain [K] (prologue) or null
  float eps;
  int32_t mode;             // LYC_GEMV_*
  float* y;                 // STORE: y = Wx; RESIDUAL: y += Wx (fp32 [M])
  void* yb;                 // SILU_BF16: yb = silu(Wx) (bf16)
  // QKV_ROPE: rows [0, nq*d) -> q (rotary), [nq*d, (nq+nkv)*d) -> K rows
  // (rotary), the rest -> V rows; K / V rows go to cache row `pos` of each
  // KV head's slab: k_cache + g * slab_stride + pos * d
  void* q_out;
  void* k_cache;
  void* v_cache;
  int64_t slab_stride;      // elements between consecutive KV heads' slabs
  int32_t nq, nkv, d, flags;  // flags: LYC_GEMV_FLAG_*
  int64_t pos;
  const void* pf;           // L2 prefetch of the next launch's weights [pf_bytes], or null
  int64_t pf_bytes;
};
