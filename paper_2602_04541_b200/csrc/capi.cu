// capi.cu -- host side of the C-ABI (include/lyc.h): validation with the
// reference's error semantics, the pooled split planner (kernel_sim.hpp:63-110),
// device plan upload, kernel launches and CUDA-graph capture of a decode step.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lyc.h"
#include "lyc_plan.h"
#include "plan.cuh"

#include <cudaTypedefs.h>

namespace lyc {
void plan_layer_host(const LycPlanIn& in, int l, const PlanOut& o);
cudaError_t launch_plan(const LycPlanIn& in, cudaStream_t st, bool pdl);
cudaError_t launch_attn(const LycAttnParams& p, int dtype, int d, int batch, cudaStream_t st);
int attn_stages(int dtype, int d);
cudaError_t launch_merge(const LycMergeParams& p, int dtype, cudaStream_t st);
cudaError_t launch_topk(const LycTopkParams& p, int rows, int cluster, cudaStream_t st);
cudaError_t launch_policy(const LycPolicyParams& p, int rows, cudaStream_t st);
int64_t window_workspace_bytes(int B, int H, int G, int W, int n_split);
cudaError_t launch_window_f32(const void* q, const void* k, const void* v, int layer, int B, int H,
                              int G, int d, int64_t cap, int64_t start, int W, float scale,
                              void* out, cudaStream_t st);
cudaError_t launch_window_tc(const CUtensorMap& tmap_k, const CUtensorMap& tmap_v, const void* q,
                             int layer, int B, int H, int G, int d, int64_t start, int W,
                             float scale, float* workspace, int n_split, void* out,
                             cudaStream_t st);
cudaError_t launch_gemv(const LycGemvParams& p, int n_sms, cudaStream_t st);
int topk_cluster_size(int n, int max_slice);
cudaError_t launch_refresh_scores(const void* q, const void* k_layer, int64_t cap, int B, int H,
                                  int G, int d, int dtype, int64_t len, uint32_t* keys,
                                  int64_t key_stride, int blocks, cudaStream_t st);
size_t topk_smem_bytes(int slice);
cudaError_t launch_float_keys(const float* s, uint32_t* keys, int64_t n, cudaStream_t st);
cudaError_t launch_step(const LycStepParams& p, int dtype, int d, cudaStream_t st, bool pdl);
bool step_supported(int dtype, int d);
int64_t step_max_keys();
int64_t step_ring_bytes(int dtype, int d);
cudaError_t launch_shard_candidates(const uint32_t* keys, int64_t key_stride,
                                    const int32_t* local_ids, const int32_t* cnt,
                                    const int32_t* sel_rows, int n_sel, int64_t k_cap,
                                    int64_t row_begin, uint32_t* cand_key, int32_t* cand_idx,
                                    cudaStream_t st);
cudaError_t launch_shard_merge(const float* all_o, const float* all_lse, int64_t stride_o,
                               int64_t stride_lse, int world, int rows, int d, void* out,
                               int dtype, cudaStream_t st);
cudaError_t launch_shard_gather(const uint32_t* all_key, const int32_t* all_idx, int64_t stride,
                                int world, int64_t k_cap, const int32_t* sel_rows, int n_sel,
                                uint32_t* keys, int32_t* ids, cudaStream_t st);
cudaError_t launch_shard_finalize(const int32_t* pos, int64_t pos_stride, const int32_t* ids,
                                  int64_t id_stride, int k, const int32_t* sel_rows, int n_sel,
                                  int64_t row_begin, int64_t n_local, int32_t* global_sets,
                                  int64_t global_stride, int32_t* cache, int64_t cache_stride,
                                  int32_t* cache_count, cudaStream_t st);
int64_t step_bitmap_words(int64_t n_keys);
int step_item_keys();
}  // namespace lyc

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw Error{code, m}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(LYC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int64_t guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return LYC_ECUDA;
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

int elem_bytes(int dtype) { return dtype == LYC_DTYPE_BF16 ? 2 : 4; }

bool supported_d(int dtype, int64_t d) {
  if (dtype == LYC_DTYPE_BF16) return d == 64 || d == 128 || d == 256;
  if (dtype == LYC_DTYPE_F32) return d == 16 || d == 32 || d == 64 || d == 128;
  return false;
}

// ------------------------------------------------------------- planner
// plan_splits (kernel_sim.hpp:63-110): per batch item the concatenated
// per-head item lists are cut into num_splits chunks of base + (s < rem)
// items, then mapped back to (head, begin, end, head_local_split) units.
struct HostLaunch {
  std::vector<LycSlot> slots;        // [B*H]
  std::vector<LycUnit> units;
  std::vector<int32_t> split_off;    // [B*S + 1]
  std::vector<LycMergeTask> merges;
  std::vector<int32_t> sel_rows;     // selection index -> index-cache row
  std::vector<int32_t> sel_n, sel_k; // variable-length batch: keys / ids kept per selection row
  int batch = 0, heads = 0, splits = 0;
};

void plan_launch(HostLaunch& L, int batch, int heads, int splits, int group) {
  L.batch = batch;
  L.heads = heads;
  L.splits = splits;
  L.units.clear();
  L.split_off.assign((size_t)batch * splits + 1, 0);
  L.merges.clear();
  for (int b = 0; b < batch; ++b) {
    int64_t total = 0;
    for (int g = 0; g < heads; ++g) {
      LycSlot& s = L.slots[(size_t)b * heads + g];
      s.n_units = 0;
      s.first_unit = -1;
      total += s.n_items;
    }
    if (total == 0) fail(LYC_EINVAL, "plan_splits: batch item has zero blocks");
    const int64_t base = total / splits, rem = total % splits;
    int head = 0;
    int64_t offset = 0;
    for (int s = 0; s < splits; ++s) {
      L.split_off[(size_t)b * splits + s] = (int32_t)L.units.size();
      int64_t want = base + (s < rem ? 1 : 0);
      while (want > 0) {
        while (L.slots[(size_t)b * heads + head].n_items == offset) {
          ++head;
          offset = 0;
        }
        LycSlot& sl = L.slots[(size_t)b * heads + head];
        const int64_t take = std::min<int64_t>(sl.n_items - offset, want);
        LycUnit u;
        u.slot = b * heads + head;
        u.begin = (int32_t)offset;
        u.end = (int32_t)(offset + take);
        u.hls = sl.n_units;
        if (sl.n_units == 0) sl.first_unit = (int32_t)L.units.size();
        sl.n_units++;
        L.units.push_back(u);
        offset += take;
        want -= take;
      }
    }
  }
  L.split_off[(size_t)batch * splits] = (int32_t)L.units.size();
  for (size_t i = 0; i < L.slots.size(); ++i)
    if (L.slots[i].n_units > 1)
      for (int j = 0; j < group; ++j)
        L.merges.push_back(LycMergeTask{(int32_t)i, j, L.slots[i].first_unit, L.slots[i].n_units,
                                        L.slots[i].q_row, 0});
}

// Device copy of one HostLaunch; returns the device pointers inside `blob`.
struct DevLaunch {
  LycSlot* slots = nullptr;
  LycUnit* units = nullptr;
  LycSlot* unit_slots = nullptr;
  int32_t* split_off = nullptr;
  LycMergeTask* merges = nullptr;
  int32_t* sel_rows = nullptr;
  int32_t* sel_n = nullptr;  // null unless the plan is variable-length
  int32_t* sel_k = nullptr;
  int n_units = 0, n_merges = 0, n_sel = 0;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t launch_bytes(const HostLaunch& L) {
  return align_up(L.slots.size() * sizeof(LycSlot), 256) +
         align_up(L.units.size() * sizeof(LycUnit), 256) +
         align_up(std::max<size_t>(1, L.units.size()) * sizeof(LycSlot), 256) +
         align_up(L.split_off.size() * 4, 256) +
         align_up(std::max<size_t>(1, L.merges.size()) * sizeof(LycMergeTask), 256) +
         align_up(std::max<size_t>(1, L.sel_rows.size()) * 4, 256) +
         2 * align_up(std::max<size_t>(1, L.sel_n.size()) * 4, 256);
}

// Serialise L into host staging at `off` and return device pointers relative
// to `dev_base`.
DevLaunch stage_launch(const HostLaunch& L, std::vector<uint8_t>& host, size_t& off,
                       uint8_t* dev_base) {
  DevLaunch d;
  auto put = [&](const void* src, size_t bytes, size_t reserve) -> void* {
    if (host.size() < off + reserve) host.resize(off + reserve);
    if (bytes) std::memcpy(host.data() + off, src, bytes);
    void* dp = dev_base + off;
    off += reserve;
    return dp;
  };
  d.slots = (LycSlot*)put(L.slots.data(), L.slots.size() * sizeof(LycSlot),
                          align_up(L.slots.size() * sizeof(LycSlot), 256));
  d.units = (LycUnit*)put(L.units.data(), L.units.size() * sizeof(LycUnit),
                          align_up(L.units.size() * sizeof(LycUnit), 256));
  std::vector<LycSlot> us(L.units.size());
  for (size_t u = 0; u < L.units.size(); ++u) us[u] = L.slots[(size_t)L.units[u].slot];
  d.unit_slots = (LycSlot*)put(us.data(), us.size() * sizeof(LycSlot),
                               align_up(std::max<size_t>(1, us.size()) * sizeof(LycSlot), 256));
  d.split_off = (int32_t*)put(L.split_off.data(), L.split_off.size() * 4,
                              align_up(L.split_off.size() * 4, 256));
  d.merges = (LycMergeTask*)put(L.merges.data(), L.merges.size() * sizeof(LycMergeTask),
                                align_up(std::max<size_t>(1, L.merges.size()) * sizeof(LycMergeTask), 256));
  d.sel_rows = (int32_t*)put(L.sel_rows.data(), L.sel_rows.size() * 4,
                             align_up(std::max<size_t>(1, L.sel_rows.size()) * 4, 256));
  if (!L.sel_n.empty()) {
    d.sel_n = (int32_t*)put(L.sel_n.data(), L.sel_n.size() * 4, align_up(L.sel_n.size() * 4, 256));
    d.sel_k = (int32_t*)put(L.sel_k.data(), L.sel_k.size() * 4, align_up(L.sel_k.size() * 4, 256));
  }
  d.n_units = (int)L.units.size();
  d.n_merges = (int)L.merges.size();
  d.n_sel = (int)L.sel_rows.size();
  return d;
}

// 2D TMA views of a K or V cache: dim0 = d, dim1 = every row of every slab.
// bf16: box 64 x 64 (one 128-B panel), 128B swizzle; fp32: box d x 64, no swizzle.
void encode_kv_maps(LycAttnParams& ap, const void* k, const void* v, int64_t rows, int D,
                    int dtype) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
               "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
    if (q != cudaDriverEntryPointSuccess || !fn) fail(LYC_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (rows >= ((int64_t)1 << 31)) fail(LYC_ENOTSUP, "KV cache has >= 2^31 rows");
  const bool bf16 = dtype == LYC_DTYPE_BF16;
  const int e = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * e};
  cuuint32_t box[2] = {bf16 ? 64u : (cuuint32_t)D, (cuuint32_t)LYC_TILE};
  cuuint32_t estr[2] = {1, 1};
  const void* ptrs[2] = {k, v};
  CUtensorMap* maps[2] = {&ap.tmap_k, &ap.tmap_v};
  for (int i = 0; i < 2; ++i) {
    CUresult r = encode(maps[i], bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        2, const_cast<void*>(ptrs[i]), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        bf16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(LYC_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  }
}

// 3-D TMA views of one cache for the window attention: {d, rows, slabs} with
// the row extent cut at the live length (rows past it load as zeros), box
// {64 columns, 64 rows, 1 slab}, 128B swizzle.
void encode_window_maps(CUtensorMap* mk, CUtensorMap* mv, const void* k, const void* v,
                        int64_t slabs, int64_t rows, int64_t cap, int D) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
               "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
    if (q != cudaDriverEntryPointSuccess || !fn) fail(LYC_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (rows >= ((int64_t)1 << 31) || slabs >= ((int64_t)1 << 31)) fail(LYC_ENOTSUP, "window: cache too large");
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)rows, (cuuint64_t)slabs};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)cap * D * 2};
  cuuint32_t box[3] = {64u, 64u, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  const void* ptrs[2] = {k, v};
  CUtensorMap* maps[2] = {mk, mv};
  for (int i = 0; i < 2; ++i) {
    CUresult r = encode(maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptrs[i]), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(LYC_ECUDA, "cuTensorMapEncodeTiled (window) failed (" + std::to_string((int)r) + ")");
  }
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

const char* lyc_last_error(void) { return g_err.c_str(); }
const char* lyc_version(void) { return "lyc-b200 0.1 (sm_100a)"; }
int64_t lyc_launch_count(void) { return g_launches; }

int64_t lyc_plan_splits(int64_t batch, int64_t n_kv_heads, const int64_t* head_blocks,
                        int64_t num_splits, int64_t* split_blocks, int64_t* head_split_count,
                        int64_t* units, int64_t max_units) {
  return guarded([&]() -> int64_t {
    if (num_splits < 1) fail(LYC_EINVAL, "plan_splits: num_splits must be >= 1");
    int64_t nu = 0;
    for (int64_t b = 0; b < batch; ++b) {
      int64_t total = 0;
      for (int64_t g = 0; g < n_kv_heads; ++g) total += head_blocks[b * n_kv_heads + g];
      if (total == 0) fail(LYC_EINVAL, "plan_splits: batch item has zero blocks");
      const int64_t base = total / num_splits, rem = total % num_splits;
      for (int64_t g = 0; g < n_kv_heads; ++g) head_split_count[b * n_kv_heads + g] = 0;
      int64_t head = 0, offset = 0;
      for (int64_t s = 0; s < num_splits; ++s) {
        int64_t want = base + (s < rem ? 1 : 0);
        split_blocks[b * num_splits + s] = want;
        while (want > 0) {
          while (head_blocks[b * n_kv_heads + head] == offset) {
            ++head;
            offset = 0;
          }
          const int64_t take = std::min(head_blocks[b * n_kv_heads + head] - offset, want);
          if (units && nu < max_units) {
            int64_t* u = units + nu * 6;
            u[0] = b;
            u[1] = s;
            u[2] = head;
            u[3] = offset;
            u[4] = offset + take;
            u[5] = head_split_count[b * n_kv_heads + head];
          }
          head_split_count[b * n_kv_heads + head]++;
          ++nu;
          offset += take;
          want -= take;
        }
      }
    }
    return nu;
  });
}

int lyc_latency_model(int64_t batch, int64_t n_kv_heads, const int64_t* head_blocks,
                      int64_t num_splits, int64_t bytes_per_block, int64_t* out6, double* out2) {
  return (int)guarded([&]() -> int64_t {
    std::vector<int64_t> sb((size_t)(batch * std::max<int64_t>(num_splits, 1)));
    std::vector<int64_t> hsc((size_t)(batch * n_kv_heads));
    const int64_t nu = lyc_plan_splits(batch, n_kv_heads, head_blocks, num_splits, sb.data(),
                                       hsc.data(), nullptr, 0);
    if (nu < 0) fail((int)nu, g_err);
    int64_t total = 0, pooled = 0, naive = 0, cells = 0;
    for (int64_t b = 0; b < batch; ++b) {
      for (int64_t s = 0; s < num_splits; ++s) {
        total += sb[b * num_splits + s];
        pooled = std::max(pooled, sb[b * num_splits + s]);
        ++cells;
      }
      for (int64_t g = 0; g < n_kv_heads; ++g) naive = std::max(naive, head_blocks[b * n_kv_heads + g]);
    }
    const double mean = (double)total / (double)cells;
    out6[0] = total;
    out6[1] = pooled;
    out6[2] = naive;
    out6[3] = bytes_per_block;
    out6[4] = pooled * bytes_per_block;
    out6[5] = naive * bytes_per_block;
    out2[0] = mean;
    out2[1] = mean > 0.0 ? (double)pooled / mean : 0.0;
    return LYC_OK;
  });
}

int64_t lyc_fraction_budget(double frac, int64_t n) {
  const double raw = frac * (double)n;
  const double c = std::ceil(raw - 1e-9);
  int64_t b = c < 0 ? 0 : (int64_t)c;
  b = std::max<int64_t>(b, 1);
  return std::min(b, n);
}


// ------------------------------------------------------------- kernel::run
int lyc_workload_run(const lyc_workload* w, int64_t num_splits, void* out, uint32_t* exec_counts,
                     void* stream) {
  return (int)guarded([&]() -> int64_t {
    cudaStream_t st = (cudaStream_t)stream;
    if (!w) fail(LYC_EINVAL, "Workload: null");
    if (w->batch < 1 || w->n_kv_heads < 1 || w->group_size < 1 || w->d_head < 1 ||
        w->seq_len < 1 || w->block_size < 1)
      fail(LYC_EINVAL, "Workload: all dimensions must be >= 1");
    if (num_splits < 1) fail(LYC_EINVAL, "plan_splits: num_splits must be >= 1");
    if (!supported_d(w->dtype, w->d_head)) fail(LYC_ENOTSUP, "Workload: unsupported d_head/dtype on device");
    if (w->group_size > 8) fail(LYC_ENOTSUP, "Workload: group_size > 8 not supported by the device kernel");
    if (w->kv_row_stride < w->seq_len) fail(LYC_EINVAL, "Workload: kv_row_stride < seq_len");
    const int64_t B = w->batch, H = w->n_kv_heads, G = w->group_size, D = w->d_head;
    const int64_t nb = (w->seq_len + w->block_size - 1) / w->block_size;
    // BlockIndexSet::validate (kernel_sim.hpp:27-41)
    std::vector<int32_t> ids;
    ids.reserve((size_t)w->blk_off[B * H]);
    for (int64_t s = 0; s < B * H; ++s) {
      if (w->blk_off[s + 1] < w->blk_off[s]) fail(LYC_EINVAL, "BlockIndexSet: slot count mismatch");
      for (int64_t i = w->blk_off[s]; i < w->blk_off[s + 1]; ++i) {
        const int64_t id = w->blk_ids[i];
        if (id < 0 || id >= nb) fail(LYC_EINVAL, "BlockIndexSet: block id out of range");
        if (i > w->blk_off[s] && id <= w->blk_ids[i - 1])
          fail(LYC_EINVAL, "BlockIndexSet: block ids must be strictly ascending");
        ids.push_back((int32_t)id);
      }
    }
    HostLaunch L;
    L.slots.resize((size_t)(B * H));
    for (int64_t b = 0; b < B; ++b)
      for (int64_t g = 0; g < H; ++g) {
        LycSlot& s = L.slots[(size_t)(b * H + g)];
        std::memset(&s, 0, sizeof(s));
        s.kv_off = (b * H + g) * w->kv_row_stride * D;
        s.kind = ITEM_BLOCKS;
        s.n_items = (int32_t)(w->blk_off[b * H + g + 1] - w->blk_off[b * H + g]);
        s.list_len = s.n_items;
        s.seq = (int32_t)w->seq_len;
        s.item = (int32_t)b;
        s.q_row = (int32_t)(b * H * G + g * G);
        s.sel = -1;
        s.dep = -1;
      }
    plan_launch(L, (int)B, (int)H, (int)num_splits, (int)G);
    for (auto& s : L.slots)
      if (s.n_units == 0) fail(LYC_EINVAL, "combine: head has no partials");
    // device staging: [plan | ids | part_o | part_lse]
    std::vector<uint8_t> host;
    size_t off = 0;
    const size_t plan_b = launch_bytes(L);
    const size_t ids_b = align_up(std::max<size_t>(1, ids.size()) * 4, 256);
    const size_t po_b = align_up((size_t)L.units.size() * G * D * 4, 256);
    const size_t pl_b = align_up((size_t)L.units.size() * G * 4, 256);
    uint8_t* dev = nullptr;
    cuda_check(cudaMallocAsync((void**)&dev, plan_b + ids_b + po_b + pl_b, st), "cudaMallocAsync");
    int32_t* d_ids = (int32_t*)(dev + plan_b);
    for (int64_t s = 0; s < B * H; ++s) L.slots[(size_t)s].list = d_ids + w->blk_off[s];
    DevLaunch dl = stage_launch(L, host, off, dev);
    host.resize(plan_b + ids_b);
    if (!ids.empty()) std::memcpy(host.data() + plan_b, ids.data(), ids.size() * 4);
    cuda_check(cudaMemcpyAsync(dev, host.data(), host.size(), cudaMemcpyHostToDevice, st), "H2D plan");
    LycAttnParams ap;
    std::memset(&ap, 0, sizeof(ap));
    LycView& v = ap.v;
    v.k = w->k;
    v.v = w->v;
    v.q = w->q;
    v.out = out;
    v.slots = dl.slots;
    v.units = dl.units;
    v.unit_slots = dl.unit_slots;
    v.split_off = dl.split_off;
    v.part_o = (float*)(dev + plan_b + ids_b);
    v.part_lse = (float*)(dev + plan_b + ids_b + po_b);
    v.exec_counts = exec_counts;
    v.counts_stride = (int32_t)nb;
    v.n_splits = (int32_t)num_splits;
    v.seq_len = (int32_t)w->seq_len;
    v.block_size = (int32_t)w->block_size;
    v.group = (int32_t)G;
    v.sel_mode = SEL_NONE;
    v.scale = w->scale;
    v.scale_log2 = w->scale * 1.4426950408889634f;
    encode_kv_maps(ap, w->k, w->v, B * H * w->kv_row_stride, (int)D, w->dtype);
    cuda_check(lyc::launch_attn(ap, w->dtype, (int)D, (int)B, st), "attention launch");
    ++g_launches;
    if (dl.n_merges) {
      LycMergeParams mp{};
      mp.part_o = v.part_o;
      mp.part_lse = v.part_lse;
      mp.slots = dl.slots;
      mp.tasks = dl.merges;
      mp.out = out;
      mp.n_tasks = dl.n_merges;
      mp.group = (int32_t)G;
      mp.chunks = (int32_t)((D + 31) / 32);
      mp.d = (int32_t)D;
      cuda_check(lyc::launch_merge(mp, w->dtype, st), "merge launch");
      ++g_launches;
    }
    // the pageable host staging buffer must outlive the async copy
    cuda_check(cudaStreamSynchronize(st), "sync");
    cuda_check(cudaFreeAsync(dev, st), "cudaFreeAsync");
    return LYC_OK;
  });
}

int64_t lyc_args_top_k(const float* scores, int64_t n, int64_t k, int32_t* out, void* stream) {
  return guarded([&]() -> int64_t {
    cudaStream_t st = (cudaStream_t)stream;
    if (k < 1) fail(LYC_EINVAL, "args_top_k: k must be >= 1");
    const int64_t take = std::min(k, n);
    if (take == 0) return 0;
    if (n > (int64_t)16 * 32768) fail(LYC_ENOTSUP, "args_top_k: n too large for one cluster");
    const int cluster = lyc::topk_cluster_size((int)n, 16384);
    const int slice = (int)((n + cluster - 1) / cluster);
    uint8_t* dev = nullptr;
    cuda_check(cudaMallocAsync((void**)&dev, align_up((size_t)n * 4, 256) + 256, st), "cudaMallocAsync");
    uint32_t* keys = (uint32_t*)dev;
    int32_t* row = (int32_t*)(dev + align_up((size_t)n * 4, 256));
    cuda_check(cudaMemsetAsync(row, 0, 4, st), "memset");
    cuda_check(lyc::launch_float_keys(scores, keys, n, st), "keys launch");
    LycTopkParams tp{};
    tp.keys = keys;
    tp.key_stride = n;
    tp.n = (int32_t)n;
    tp.k = (int32_t)take;
    tp.out = out;
    tp.out_row = row;
    tp.out_stride = 0;
    tp.out_count = nullptr;
    tp.slice = slice;
    tp.clear_keys = 0;
    cuda_check(lyc::launch_topk(tp, 1, cluster, st), "topk launch");
    g_launches += 2;
    cuda_check(cudaFreeAsync(dev, st), "cudaFreeAsync");
    return take;
  });
}

}  // extern "C"

// ------------------------------------------------------------- decoder
struct lyc_decoder {
  lyc_decode_config cfg{};
  std::vector<uint8_t> roles;
  int B = 0, H = 0, G = 0, Hq = 0, D = 0, NL = 0, S = 0, bs = 64;
  bool fused = false;           // the step runs on the persistent step kernel (step.cu)
  bool shard = false;           // KV-sequence shard mode (lyc_shard_layer / lyc_shard_merge)
  int32_t* shard_ids = nullptr; // [B*H][k_cap] local top-k ids
  int32_t* shard_cnt = nullptr; // [B*H]
  int32_t* shard_rows = nullptr;// [B*H] identity rows for the candidate top-k
  uint32_t* shard_ckey = nullptr;  // [B*H][world * k_cap] concatenated candidates
  int32_t* shard_cidx = nullptr;
  int32_t* shard_pos = nullptr; // [B*H][k_cap] positions of the global top-k
  int shard_world = 0;
  int64_t k_cap = 0;
  int32_t* idx = nullptr;       // [B*H][k_cap]
  int32_t* idx_count = nullptr;
  uint32_t* sel_keys = nullptr; // [2][B*H][sel_stride]
  uint32_t* refresh_keys = nullptr;  // [B*H][sel_stride] (lyc_decoder_refresh_sets, lazily)
  int32_t* ident_rows = nullptr;     // [B*H] 0..B*H-1 (lazily)
  int64_t sel_stride = 0;
  uint32_t* hist = nullptr;     // [2][B*H][LYC_H1_BINS] fused first-pass histograms
  uint32_t* sel_bitmap = nullptr;  // fused-mode pooled selection scratch (see LycStepParams)
  int64_t bitmap_stride = 0;
  uint32_t* sel_cand = nullptr;
  uint32_t* sel_ccnt = nullptr;
  uint32_t* sel_csub = nullptr;
  uint32_t* sel_rowctr = nullptr;  // [2 parity][NL][B*H][16]
  int64_t rowctr_set = 0;
  int stages = 0;               // attention ring stages in use (0 = all; lyc_decoder_tune)
  bool pdl = true;              // programmatic dependent launch of planner / step kernels
  bool defer_sel = true;        // per-layer launches: a layer's selection runs in the next launch
  int pending_sel = -1;         // layer whose selection was deferred to the next launch (-1: none)
  int64_t pending_seq = 0;      //   at this length
  uint32_t* ctr = nullptr;      // LYC_CTR_WORDS(NL)
  unsigned long long* trace = nullptr;  // optional step timeline [NL][LYC_TRACE_EVENTS][n_ctas]
  int32_t* set_trace = nullptr;        // optional per-layer sets [NL][B*H][k_cap] (fused path)
  int32_t* set_trace_count = nullptr;  // [NL][B*H], -1 where no set was emitted
  float* part_o = nullptr;      // [max_units][G][d] split partials (one layer at a time)
  float* part_lse = nullptr;
  // ---- plan storage: a fixed per-layer layout, sized at create for seq_cap
  // (no allocation afterwards).  The fused path's plan is written by the
  // device planner (plan.cu) in the stream; the per-layer-kernel path's plan
  // (TopP / Threshold, shard mode) is built on the host and uploaded
  // stream-ordered from pinned staging.
  int max_units = 0, max_merges = 0;
  size_t layer_bytes = 0;       // bytes of one layer's region in `blob`
  uint8_t* blob = nullptr;      // [NL][layer region] + descs [NL]
  size_t blob_bytes = 0;
  LycLayerDesc* d_layers = nullptr;      // device descs (pointers fixed at create)
  std::vector<LycLayerDesc> h_layers;    // host copy of the descs
  uint8_t* staging = nullptr;   // pinned host image of blob (per-layer-kernel path)
  cudaEvent_t staged = nullptr; // recorded after the last staging upload
  bool staging_busy = false;
  uint8_t* d_roles = nullptr;   // [NL][H] for the device planner
  LycPlanHdr* d_hdr = nullptr;  // the fused plan's header
  int32_t* d_keys = nullptr;    // [NL][LYC_PLAN_KEY_INTS(B)] each layer's plan key (plan.cu)
  std::vector<int32_t> host_key;  // the key of the device plan, when host lengths made it
  bool host_key_valid = false;
  std::vector<int32_t> captured_key;
  LycPlanIn pin{};              // the device planner's static input
  int64_t planned_seq = -1;     // host plan (per-layer kernels), or the last host-seq device plan
  bool planned_varlen = false;
  std::vector<int64_t> planned_lens;
  uint64_t plan_gen = 0;        // host plans uploaded so far
  int64_t captured_launches = 0;     // kernel launches in the captured graph
  uint64_t captured_gen = 0;         // host plan the captured graph reads (per-layer kernels)
  int64_t captured_seq = -1;
  std::vector<int64_t> captured_lens;
  LycAttnParams maps{};         // tensor maps for the last (k, v) pointers
  const void* map_k = nullptr;
  const void* map_v = nullptr;
  struct Layer {
    LycAttnParams ap;           // per-layer kernel path
    LycMergeParams mp;
    LycTopkParams tp;
    LycPolicyParams pp;         // TopP / Threshold selection (per-layer path)
    int n_sel = 0, cluster = 1, n_merges = 0;
  };
  std::vector<Layer> layers;
  int64_t n_keys = 0, k_sel = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool timing = false;
  bool timed_per_layer = false;  // the last timed launches were one per layer
  std::vector<cudaEvent_t> ev_pre, ev_post;  // per layer (per-layer launches) or [0] (whole step)

  int n_ctas() const { return S * B; }
  bool retrieval(int l, int g) const { return l == 0 || roles[(size_t)l * H + g] == 0; }

  int64_t budget(int64_t seq) const {  // tokens (or blocks) kept per sparse head
    if (cfg.select_mode == LYC_SELECT_BLOCKS) {
      const int64_t nb = (seq + bs - 1) / bs;
      if (cfg.policy_kind == LYC_POLICY_RATIO) return lyc_fraction_budget(1.0 - cfg.ratio, nb);
      return std::min<int64_t>((cfg.top_k + bs - 1) / bs, nb);
    }
    if (cfg.policy_kind == LYC_POLICY_RATIO) return lyc_fraction_budget(1.0 - cfg.ratio, seq);
    if (variable_sets()) return seq;  // capacity; the set size is a device count
    return std::min<int64_t>(cfg.top_k, seq);
  }
  // TopP / Threshold: data-dependent set sizes (device counts)
  bool variable_sets() const {
    return cfg.policy_kind == LYC_POLICY_TOPP || cfg.policy_kind == LYC_POLICY_THRESHOLD;
  }
};

namespace {

// The step kernel's split order: per batch item, three pools are each cut
// evenly across all splits and concatenated per split in this order --
// retrieval slots (so every CTA finishes its share of the retrieval heads
// first and their selection can start before the layer ends), sparse slots
// with an older index list, and last the sparse slots whose list the
// immediately preceding layer's selection produces (streamed while that
// selection is still running).  This is the host-order statement of the
// device planner (plan.cuh); lyc_plan_selftest checks the two agree.
void plan_step_launch(HostLaunch& L, int batch, int heads, int splits, int group, int layer,
                      int free_from, bool ragged) {
  L.batch = batch;
  L.heads = heads;
  L.splits = splits;
  L.units.clear();
  L.merges.clear();
  const int cells = batch * splits;
  L.split_off.assign((size_t)cells + 1, 0);
  std::vector<std::vector<LycUnit>> per_cell((size_t)cells);
  for (int b = 0; b < batch; ++b) {
    int64_t total = 0;
    for (int g = 0; g < heads; ++g) {
      LycSlot& s = L.slots[(size_t)b * heads + g];
      s.n_units = 0;
      total += s.n_items;
    }
    if (total == 0) fail(LYC_EINVAL, "plan_splits: batch item has zero blocks");
  }
  // Equal lengths: each batch item's pools are cut across its own `splits`
  // cells.  A variable-length batch (items differ in dense blocks or budget):
  // each pool is cut across ALL cells (every item's slots in one list), so
  // short items do not leave their SMs idle while long ones stream.
  const int groups = ragged ? 1 : batch;
  for (int grp = 0; grp < groups; ++grp)
  for (int pool = 0; pool < 3; ++pool) {
    const int b0 = ragged ? 0 : grp, b1 = ragged ? batch : grp + 1;
    const int c0 = b0 * splits, nc = (b1 - b0) * splits;  // this group's cells
    std::vector<int> hs;  // slot indices of this pool, in (b, g) order
    int64_t tot = 0;
    for (int i = b0 * heads; i < b1 * heads; ++i) {
      const LycSlot& s = L.slots[(size_t)i];
      const bool late = s.dep >= 0 && s.dep == layer - 1;
      const int my_pool = s.kind == ITEM_DENSE ? 0 : late ? 2 : 1;
      if (my_pool == pool && s.n_items > 0) {
        hs.push_back(i);
        tot += s.n_items;
      }
    }
    if (tot == 0) continue;
    // the sparse pools skip the CTAs that run this layer's selection items
    // (cells >= free_from): their epilogue classifies while the others
    // stream, without sharing issue slots with busy consumers
    int ns = nc;
    if (pool >= 1) {
      const int usable = std::min(nc, free_from - c0);
      if (usable >= (nc + 1) / 2) ns = usable;  // never squeeze a group onto a few CTAs
    }
    // even cut points, then snapped onto a slot boundary within one item:
    // a cell that would hold the end of one slot and the start of the next
    // (two units: an extra unit epilogue and signal) gets one item more or
    // less instead
    const int64_t base = tot / ns, rem = tot % ns;
    constexpr int64_t kSnap = 1;  // items (measured: 1 beats 2 and 3)
    std::vector<int64_t> cut((size_t)nc + 1);
    for (int sp = 0; sp <= nc; ++sp)
      cut[(size_t)sp] = sp <= ns ? sp * base + std::min<int64_t>(sp, rem) : tot;
    {
      int64_t hb = 0;
      for (size_t h = 0; h + 1 < hs.size(); ++h) {
        hb += L.slots[(size_t)hs[h]].n_items;
        // the cut nearest to the boundary hb
        int sp = (int)std::min<int64_t>(ns - 1, std::max<int64_t>(1, hb / std::max<int64_t>(base, 1)));
        while (sp > 1 && cut[(size_t)sp] > hb) --sp;
        while (sp < ns - 1 && cut[(size_t)sp + 1] <= hb) ++sp;
        for (int c = sp; c <= sp + 1 && c < ns; ++c)
          if (c >= 1 && std::llabs(cut[(size_t)c] - hb) <= kSnap && cut[(size_t)c - 1] < hb &&
              hb < cut[(size_t)c + 1])
            cut[(size_t)c] = hb;
      }
    }
    size_t hi = 0;
    int64_t offset = 0;
    for (int sp = 0; sp < nc; ++sp) {
      int64_t want = cut[(size_t)sp + 1] - cut[(size_t)sp];
      while (want > 0) {
        while (L.slots[(size_t)hs[hi]].n_items == offset) {
          ++hi;
          offset = 0;
        }
        LycSlot& sl = L.slots[(size_t)hs[hi]];
        const int64_t take = std::min<int64_t>(sl.n_items - offset, want);
        LycUnit u;
        u.slot = hs[hi];
        u.begin = (int32_t)offset;
        u.end = (int32_t)(offset + take);
        u.hls = sl.n_units++;
        per_cell[(size_t)(c0 + sp)].push_back(u);
        offset += take;
        want -= take;
      }
    }
  }
  for (int c = 0; c < cells; ++c) {
    L.split_off[(size_t)c] = (int32_t)L.units.size();
    for (const LycUnit& u : per_cell[(size_t)c]) L.units.push_back(u);
  }
  L.split_off[(size_t)batch * splits] = (int32_t)L.units.size();
  int32_t base = 0;  // partial-output base of every slot (units of a slot need not be adjacent)
  for (auto& s : L.slots) {
    s.first_unit = base;
    base += s.n_units;
  }
  for (size_t i = 0; i < L.slots.size(); ++i)
    if (L.slots[i].n_units > 1)
      for (int j = 0; j < group; ++j)
        L.merges.push_back(LycMergeTask{(int32_t)i, j, L.slots[i].first_unit, L.slots[i].n_units,
                                        L.slots[i].q_row, 0});
}

void free_dev(void* p) {
  if (p) cudaFree(p);
}

// ---- the fixed per-layer plan layout (both planners write into it)
struct LayerLayout {
  size_t slots, units, unit_slots, split_off, merges, sel_rows, sel_n, sel_k, bytes;
};
LayerLayout layer_layout(int BH, int cells, int max_units, int max_merges) {
  LayerLayout o{};
  size_t off = 0;
  auto put = [&](size_t bytes) {
    const size_t at = off;
    off += align_up(std::max<size_t>(bytes, 4), 256);
    return at;
  };
  o.slots = put((size_t)BH * sizeof(LycSlot));
  o.units = put((size_t)max_units * sizeof(LycUnit));
  o.unit_slots = put((size_t)max_units * sizeof(LycSlot));
  o.split_off = put((size_t)(cells + 1) * 4);
  o.merges = put((size_t)max_merges * sizeof(LycMergeTask));
  o.sel_rows = put((size_t)BH * 4);
  o.sel_n = put((size_t)BH * 4);
  o.sel_k = put((size_t)BH * 4);
  o.bytes = off;
  return o;
}

LycLayerDesc layer_desc(uint8_t* base, const LayerLayout& ll) {
  LycLayerDesc ds{};
  ds.slots = (const LycSlot*)(base + ll.slots);
  ds.units = (const LycUnit*)(base + ll.units);
  ds.unit_slots = (const LycSlot*)(base + ll.unit_slots);
  ds.split_off = (const int32_t*)(base + ll.split_off);
  ds.merges = (const LycMergeTask*)(base + ll.merges);
  ds.sel_rows = (const int32_t*)(base + ll.sel_rows);
  ds.sel_n = (const int32_t*)(base + ll.sel_n);
  ds.sel_k = (const int32_t*)(base + ll.sel_k);
  ds.n_merges = 0;
  ds.n_sel = 0;
  return ds;
}

// The slots of layer l for lengths len_of(b) (decode_engine.hpp:121-143): the
// statement both host planners start from.
void host_slots(const lyc_decoder* d, int l, const int64_t* lens, int64_t seq, bool varlen,
                std::vector<int>& last_r, HostLaunch& L) {
  const int B = d->B, H = d->H, G = d->G, D = d->D;
  const bool blocks = d->cfg.select_mode == LYC_SELECT_BLOCKS;
  const bool none = d->cfg.select_mode == LYC_SELECT_NONE;
  const int64_t kb = d->budget(seq);
  L.slots.resize((size_t)B * H);
  L.sel_rows.clear();
  L.sel_n.clear();
  L.sel_k.clear();
  for (int b = 0; b < B; ++b)
    for (int g = 0; g < H; ++g) {
      LycSlot& s = L.slots[(size_t)b * H + g];
      std::memset(&s, 0, sizeof(s));
      s.kv_off = (((int64_t)l * B + b) * H + g) * d->cfg.seq_cap * D;
      s.q_row = b * H * G + g * G;
      s.dep = -1;
      s.sel = -1;
      const int64_t seq_b = varlen ? lens[b] : seq, nb_b = (seq_b + d->bs - 1) / d->bs;
      const int64_t kb_b = varlen ? d->budget(seq_b) : kb;
      s.seq = (int32_t)seq_b;
      s.item = b;
      if (d->retrieval(l, g)) {
        s.kind = ITEM_DENSE;
        s.n_items = (int32_t)nb_b;
        if (!none) {
          s.sel = (int32_t)L.sel_rows.size();
          L.sel_rows.push_back(b * H + g);
          if (varlen) {
            L.sel_n.push_back((int32_t)(blocks ? nb_b : seq_b));
            L.sel_k.push_back((int32_t)kb_b);
          }
        }
      } else {
        s.kind = blocks ? ITEM_BLOCKS : ITEM_TOKENS;
        s.list = d->idx + (int64_t)(b * H + g) * d->k_cap;
        s.list_len = (int32_t)kb_b;
        if (d->shard || d->variable_sets())  // this rank's filtered set / a variable-size set
          s.count = d->idx_count + (b * H + g);
        s.n_items = blocks ? (int32_t)kb_b : (int32_t)((kb_b + LYC_TILE - 1) / LYC_TILE);
        s.dep = last_r[(size_t)g];
      }
    }
  for (int g = 0; g < H; ++g)
    if (d->retrieval(l, g)) last_r[(size_t)g] = l;
}

// Serialise a host plan into the layer's fixed region of the staging image.
DevLaunch stage_fixed(const HostLaunch& L, uint8_t* host_base, const LycLayerDesc& ds,
                      const uint8_t* dev_base, const LayerLayout& ll, int max_units, int max_merges) {
  if ((int)L.units.size() > max_units || (int)L.merges.size() > max_merges)
    fail(LYC_ENOTSUP, "plan exceeds the decoder's plan capacity");
  auto put = [&](size_t off, const void* src, size_t bytes) {
    if (bytes) std::memcpy(host_base + off, src, bytes);
  };
  put(ll.slots, L.slots.data(), L.slots.size() * sizeof(LycSlot));
  put(ll.units, L.units.data(), L.units.size() * sizeof(LycUnit));
  std::vector<LycSlot> us(L.units.size());
  for (size_t u = 0; u < L.units.size(); ++u) us[u] = L.slots[(size_t)L.units[u].slot];
  put(ll.unit_slots, us.data(), us.size() * sizeof(LycSlot));
  put(ll.split_off, L.split_off.data(), L.split_off.size() * 4);
  put(ll.merges, L.merges.data(), L.merges.size() * sizeof(LycMergeTask));
  put(ll.sel_rows, L.sel_rows.data(), L.sel_rows.size() * 4);
  put(ll.sel_n, L.sel_n.data(), L.sel_n.size() * 4);
  put(ll.sel_k, L.sel_k.data(), L.sel_k.size() * 4);
  (void)dev_base;
  DevLaunch dl;
  dl.slots = const_cast<LycSlot*>(ds.slots);
  dl.units = const_cast<LycUnit*>(ds.units);
  dl.unit_slots = const_cast<LycSlot*>(ds.unit_slots);
  dl.split_off = const_cast<int32_t*>(ds.split_off);
  dl.merges = const_cast<LycMergeTask*>(ds.merges);
  dl.sel_rows = const_cast<int32_t*>(ds.sel_rows);
  dl.sel_n = L.sel_n.empty() ? nullptr : const_cast<int32_t*>(ds.sel_n);
  dl.sel_k = L.sel_k.empty() ? nullptr : const_cast<int32_t*>(ds.sel_k);
  dl.n_units = (int)L.units.size();
  dl.n_merges = (int)L.merges.size();
  dl.n_sel = (int)L.sel_rows.size();
  return dl;
}

void validate_lens(const lyc_decoder* d, int64_t& seq, const int64_t*& lens) {
  if (lens) {
    bool same = true;
    for (int b = 0; b < d->B; ++b) {
      if (lens[b] < 1) fail(LYC_EINVAL, "decode_step: every seq_len must be >= 1");
      if (lens[b] > d->cfg.seq_cap) fail(LYC_EINVAL, "decode_step: seq_len exceeds seq_cap");
      same = same && lens[b] == lens[0];
    }
    if (same) {
      seq = lens[0];
      lens = nullptr;
    } else {
      if (d->shard) fail(LYC_ENOTSUP, "decode_step: variable-length batches are not sharded");
      seq = *std::max_element(lens, lens + d->B);
    }
  }
  if (seq < 1) fail(LYC_EINVAL, "decode_step: seq_len must be >= 1");
  if (seq > d->cfg.seq_cap) fail(LYC_EINVAL, "decode_step: seq_len exceeds seq_cap");
  if (!d->fused && seq > (int64_t)16 * 32768 && d->cfg.select_mode == LYC_SELECT_TOKENS)
    fail(LYC_ENOTSUP, "decode_step: token-mode selection supports seq_len <= 524288");
}

// Host plan of the per-layer-kernel path (TopP / Threshold, shard mode):
// plan_splits per batch item (kernel_sim.hpp:63-110) for every layer,
// uploaded stream-ordered (async copy from pinned staging on `st`) into the
// fixed plan layout -- a kernel still reading the previous plan on `st`
// finishes first.  lens (optional, host [B]): per-item lengths.
void decoder_plan(lyc_decoder* d, int64_t seq, const int64_t* lens, cudaStream_t st) {
  validate_lens(d, seq, lens);
  const bool varlen = lens != nullptr;
  if (!varlen && !d->planned_varlen && d->planned_seq == seq) return;
  if (varlen && d->planned_varlen && std::equal(lens, lens + d->B, d->planned_lens.begin())) return;
  const int B = d->B, H = d->H, G = d->G, D = d->D;
  const bool blocks = d->cfg.select_mode == LYC_SELECT_BLOCKS;
  const bool none = d->cfg.select_mode == LYC_SELECT_NONE;
  const int64_t kb = d->budget(seq);
  const int64_t nb = (seq + d->bs - 1) / d->bs;
  const LayerLayout ll = layer_layout(B * H, d->n_ctas(), d->max_units, d->max_merges);
  // the staging image may still feed the previous upload
  if (d->staging_busy) cuda_check(cudaEventSynchronize(d->staged), "staging event");
  d->layers.assign((size_t)d->NL, {});
  std::vector<int> last_r((size_t)H, 0);
  const int64_t sel_n = blocks ? nb : seq;
  d->n_keys = sel_n;
  d->k_sel = kb;
  const int cluster = lyc::topk_cluster_size((int)std::min<int64_t>(sel_n, 1 << 30), 16384);
  std::vector<LycLayerDesc> descs = d->h_layers;
  for (int l = 0; l < d->NL; ++l) {
    HostLaunch L;
    host_slots(d, l, lens, seq, varlen, last_r, L);
    plan_launch(L, B, H, d->S, G);
    const LycLayerDesc& ds = d->h_layers[(size_t)l];
    DevLaunch dl = stage_fixed(L, d->staging + (size_t)l * d->layer_bytes, ds,
                               d->blob + (size_t)l * d->layer_bytes, ll, d->max_units, d->max_merges);
    lyc_decoder::Layer& ly = d->layers[(size_t)l];
    std::memset(&ly.ap, 0, sizeof(ly.ap));
    LycView& v = ly.ap.v;
    v.slots = dl.slots;
    v.units = dl.units;
    v.unit_slots = dl.unit_slots;
    v.split_off = dl.split_off;
    v.part_o = d->part_o;
    v.part_lse = d->part_lse;
    v.sel_keys = d->sel_keys;
    v.sel_stride = d->sel_stride;
    v.n_splits = d->S;
    v.seq_len = (int32_t)seq;
    v.block_size = d->bs;
    v.group = G;
    v.sel_mode = none ? SEL_NONE : blocks ? SEL_BLOCK_KEYS : SEL_TOKEN_KEYS;
    v.scale = d->cfg.scale;
    v.scale_log2 = d->cfg.scale * 1.4426950408889634f;
    v.stages = d->stages;
    v.early_exit = (d->variable_sets() || d->shard) ? 1 : 0;
    LycMergeParams& mp = ly.mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.part_o = d->part_o;
    mp.part_lse = d->part_lse;
    mp.slots = dl.slots;
    mp.tasks = dl.merges;
    mp.n_tasks = dl.n_merges;
    mp.group = G;
    mp.chunks = (D + 31) / 32;
    mp.d = D;
    ly.n_merges = dl.n_merges;
    LycTopkParams& tp = ly.tp;
    std::memset(&tp, 0, sizeof(tp));
    tp.keys = d->sel_keys;
    tp.key_stride = d->sel_stride;
    tp.n = (int32_t)sel_n;
    tp.k = (int32_t)kb;
    tp.out = d->idx;
    tp.out_row = dl.sel_rows;
    tp.out_stride = d->k_cap;
    tp.out_count = d->idx_count;
    tp.slice = (int32_t)((sel_n + cluster - 1) / cluster);
    tp.clear_keys = blocks ? 1 : 0;
    tp.row_n = dl.sel_n;
    tp.row_k = dl.sel_k;
    LycPolicyParams& pp = ly.pp;
    std::memset(&pp, 0, sizeof(pp));
    pp.keys = d->sel_keys;
    pp.key_stride = d->sel_stride;
    pp.n = (int32_t)sel_n;
    pp.kind = d->cfg.policy_kind;
    pp.value = d->cfg.ratio;
    // the consumers' key value: bf16 sum_j q_j.k (= G * pooled_q.k), fp32 pooled_q.k
    pp.score_scale = d->cfg.dtype == LYC_DTYPE_BF16 ? d->cfg.scale / (float)G : d->cfg.scale;
    pp.out = d->idx;
    pp.out_row = dl.sel_rows;
    pp.out_stride = d->k_cap;
    pp.out_count = d->idx_count;
    pp.row_n = dl.sel_n;
    ly.n_sel = dl.n_sel;
    ly.cluster = cluster;
    descs[(size_t)l].n_merges = dl.n_merges;
    descs[(size_t)l].n_sel = dl.n_sel;
  }
  uint8_t* desc_host = d->staging + (size_t)d->NL * d->layer_bytes;
  std::memcpy(desc_host, descs.data(), sizeof(LycLayerDesc) * d->NL);
  cuda_check(cudaMemcpyAsync(d->blob, d->staging, d->blob_bytes, cudaMemcpyHostToDevice, st),
             "H2D plan");
  cuda_check(cudaEventRecord(d->staged, st), "staging event");
  d->staging_busy = true;
  ++d->plan_gen;
  d->planned_seq = varlen ? -1 : seq;
  d->planned_varlen = varlen;
  if (varlen) d->planned_lens.assign(lens, lens + d->B);
}

void ensure_maps(lyc_decoder* d, const void* k, const void* v) {
  if (k != d->map_k || v != d->map_v) {
    encode_kv_maps(d->maps, k, v, (int64_t)d->NL * d->B * d->H * d->cfg.seq_cap, d->D,
                   d->cfg.dtype);
    d->map_k = k;
    d->map_v = v;
  }
}

void record(lyc_decoder* d, std::vector<cudaEvent_t>& ev, size_t i, cudaStream_t st) {
  // External records become event nodes when the stream is being captured.
  if (d->timing)
    cuda_check(cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal), "event record");
}

void decoder_layer(lyc_decoder* d, int l, const void* q_l, const void* k, const void* v,
                   void* out_l, cudaStream_t st) {
  lyc_decoder::Layer& ly = d->layers[(size_t)l];
  ensure_maps(d, k, v);
  ly.ap.tmap_k = d->maps.tmap_k;
  ly.ap.tmap_v = d->maps.tmap_v;
  ly.ap.v.k = k;
  ly.ap.v.v = v;
  ly.ap.v.q = q_l;
  ly.ap.v.out = out_l;
  ly.ap.v.out_f32 = nullptr;
  ly.ap.v.out_lse = nullptr;
  ly.mp.out_f32 = nullptr;
  ly.mp.out_lse = nullptr;
  record(d, d->ev_pre, (size_t)l, st);
  cuda_check(lyc::launch_attn(ly.ap, d->cfg.dtype, d->D, d->B, st), "attention launch");
  record(d, d->ev_post, (size_t)l, st);
  ++g_launches;
  if (ly.n_merges) {
    ly.mp.out = out_l;
    cuda_check(lyc::launch_merge(ly.mp, d->cfg.dtype, st), "merge launch");
    ++g_launches;
  }
  if (ly.n_sel) {
    if (d->variable_sets())
      cuda_check(lyc::launch_policy(ly.pp, ly.n_sel, st), "policy launch");
    else
      cuda_check(lyc::launch_topk(ly.tp, ly.n_sel, ly.cluster, st), "topk launch");
    ++g_launches;
  }
}

// The plan key of host lengths (plan.cuh): items per row, then every item's
// dense blocks and sparse budget.
std::vector<int32_t> host_plan_key(const lyc_decoder* d, int64_t seq, const int64_t* lens) {
  std::vector<int32_t> k((size_t)1 + 2 * d->B);
  int64_t mx = 0;
  for (int b = 0; b < d->B; ++b) {
    const int64_t v = lens ? lens[b] : seq;
    mx = std::max(mx, v);
    int32_t nb, kb;
    lyc::plan_item_key(d->pin, v, nb, kb);
    k[(size_t)1 + b] = nb;
    k[(size_t)1 + d->B + b] = kb;
  }
  k[0] = lyc::plan_items(d->pin, mx);
  return k;
}

// Fused path: make the device plan fit the step's lengths.  Host lengths: the
// planner runs only when their key changes (once per 64 tokens of a growing
// sequence).  Device lengths: the planner runs every step, and each layer
// returns at once when its stored key matches (plan.cu).
void ensure_plan(lyc_decoder* d, int64_t seq, const int64_t* lens, const int64_t* dlens,
                 cudaStream_t st) {
  LycPlanIn in = d->pin;
  in.seq = seq;
  in.dlens = dlens;
  in.has_lens = lens ? 1 : 0;
  if (lens)
    for (int b = 0; b < d->B; ++b) in.lens[b] = (int32_t)lens[b];
  if (!dlens) {
    std::vector<int32_t> key = host_plan_key(d, seq, lens);
    if (d->host_key_valid && key == d->host_key) return;
    d->host_key = std::move(key);
    d->host_key_valid = true;
  } else {
    d->host_key_valid = false;
  }
  cuda_check(lyc::launch_plan(in, st, d->pdl), "plan launch");
  ++g_launches;
}

// One launch of the step kernel over layers [l0, l1): q / out point at layer
// l0's [B][Hq][d] block (consecutive layers follow at B*Hq*d elements).  The
// step's lengths travel by value (host seq / lens) or as a device array
// (dlens); the kernel re-plans itself when they change its plan key.
void launch_step_range(lyc_decoder* d, int l0, int l1, const void* q, const void* k,
                       const void* v, void* out, cudaStream_t st, int64_t seq,
                       const int64_t* lens, const int64_t* dlens, bool defer_in = false,
                       bool defer_out = false) {
  ensure_maps(d, k, v);
  LycStepParams p;
  std::memset(&p, 0, sizeof(p));
  p.tmap_k = d->maps.tmap_k;
  p.tmap_v = d->maps.tmap_v;
  p.k = k;
  p.v = v;
  p.q = q;
  p.out = out;
  p.q_layer_stride = (int64_t)d->B * d->Hq * d->D;
  p.layers = d->d_layers;
  p.part_o = d->part_o;
  p.part_lse = d->part_lse;
  p.sel_keys = d->sel_keys;
  p.sel_stride = d->sel_stride;
  p.hist = d->hist;
  p.sel_bitmap = d->sel_bitmap;
  p.bitmap_stride = d->bitmap_stride;
  p.sel_cand = d->sel_cand;
  p.sel_ccnt = d->sel_ccnt;
  p.sel_csub = d->sel_csub;
  p.sel_rowctr = d->sel_rowctr;
  p.rowctr_set = d->rowctr_set;
  p.ctr = d->ctr;
  p.hdr = d->d_hdr;
  p.idx = d->idx;
  p.idx_stride = d->k_cap;
  p.idx_count = d->idx_count;
  p.trace = d->trace;
  p.set_trace = d->set_trace;
  p.set_trace_count = d->set_trace_count;
  p.n_layers = d->NL;
  p.l_begin = l0;
  p.l_end = l1;
  p.max_sel = d->B * d->H;
  p.n_splits = d->S;
  p.n_ctas = d->n_ctas();
  p.block_size = d->bs;
  p.group = d->G;
  p.sel_mode = d->cfg.select_mode == LYC_SELECT_NONE    ? SEL_NONE
               : d->cfg.select_mode == LYC_SELECT_BLOCKS ? SEL_BLOCK_KEYS
                                                         : SEL_TOKEN_KEYS;
  p.scale = d->cfg.scale;
  p.scale_log2 = d->cfg.scale * 1.4426950408889634f;
  p.stages = d->stages;
  p.sel_defer_in = defer_in ? 1 : 0;
  p.sel_defer_out = defer_out ? 1 : 0;
  p.plan = d->pin;
  p.plan.seq = seq;
  p.plan.dlens = dlens;
  p.plan.has_lens = lens ? 1 : 0;
  if (!lens && !dlens) {  // one validated host length: the kernel's lengths prologue is skipped
    int32_t nb = 0, kb = 0;
    lyc::plan_item_key(d->pin, seq, nb, kb);
    p.uniform = 1;
    p.uni_nsel = d->cfg.select_mode == LYC_SELECT_BLOCKS ? nb : (int32_t)seq;
    p.uni_ksel = kb;
  }
  if (lens)
    for (int b = 0; b < d->B; ++b) p.plan.lens[b] = (int32_t)lens[b];
  const bool per_layer = d->NL > 1 && l1 - l0 == 1;
  const size_t ev = per_layer ? (size_t)l0 : 0;
  if (d->timing && l1 > l0) d->timed_per_layer = per_layer;
  if (l1 > l0) record(d, d->ev_pre, ev, st);
  cuda_check(lyc::launch_step(p, d->cfg.dtype, d->D, st, d->pdl), "step launch");
  if (l1 > l0) record(d, d->ev_post, ev, st);
  ++g_launches;
}

bool layer_selects(const lyc_decoder* d, int l) {
  if (d->cfg.select_mode == LYC_SELECT_NONE) return false;
  for (int g = 0; g < d->H; ++g)
    if (d->retrieval(l, g)) return true;
  return false;
}

// Completes a selection deferred by the last per-layer launch: a launch over
// no layers that runs only that selection (at the length it was made for).
void flush_pending(lyc_decoder* d, cudaStream_t st) {
  if (d->pending_sel < 0) return;
  const int l = d->pending_sel + 1;
  d->pending_sel = -1;
  launch_step_range(d, l, l, nullptr, d->map_k, d->map_v, nullptr, st, d->pending_seq, nullptr,
                    nullptr, true, false);
}

void decoder_step(lyc_decoder* d, const void* q, const void* k, const void* v, int64_t seq,
                  void* out, cudaStream_t st, const int64_t* lens = nullptr,
                  const int64_t* dlens = nullptr) {
  flush_pending(d, st);
  if (d->fused) {
    if (!dlens) validate_lens(d, seq, lens);
    ensure_plan(d, seq, lens, dlens, st);
    launch_step_range(d, 0, d->NL, q, k, v, out, st, seq, lens, dlens);
    return;
  }
  if (dlens) fail(LYC_ENOTSUP, "decode_step: device-resident lengths need the fused step kernel");
  decoder_plan(d, seq, lens, st);
  const int esz = elem_bytes(d->cfg.dtype);
  const size_t qstride = (size_t)d->B * d->Hq * d->D;
  for (int l = 0; l < d->NL; ++l)
    decoder_layer(d, l, (const uint8_t*)q + l * qstride * esz, k, v,
                  (uint8_t*)out + l * qstride * esz, st);
}

}  // namespace

extern "C" {

int lyc_decoder_create(const lyc_decode_config* cfg, lyc_decoder** out) {
  return (int)guarded([&]() -> int64_t {
    if (!cfg || !out) fail(LYC_EINVAL, "decoder: null argument");
    const lyc_decode_config& c = *cfg;
    if (c.n_layers < 1 || c.batch < 1 || c.n_kv_heads < 1 || c.group_size < 1 || c.d_head < 1 ||
        c.seq_cap < 1)
      fail(LYC_EINVAL, "ModelConfig: all dimensions must be >= 1");
    if (!supported_d(c.dtype, c.d_head)) fail(LYC_ENOTSUP, "decoder: unsupported d_head/dtype");
    if (c.group_size > 8) fail(LYC_ENOTSUP, "decoder: group_size > 8 not supported by the device kernel");
    if ((int64_t)c.batch * c.n_kv_heads > 2048)
      fail(LYC_ENOTSUP, "decoder: batch * n_kv_heads > 2048 not supported");
    if (c.policy_kind == LYC_POLICY_TOPK) {
      if (c.top_k < 1) fail(LYC_EINVAL, "top_k: k must be >= 1");
    } else if (c.policy_kind == LYC_POLICY_RATIO) {
      if (!(c.ratio > 0.0 && c.ratio < 1.0)) fail(LYC_EINVAL, "ratio: theta must lie in (0,1)");
    } else if (c.policy_kind == LYC_POLICY_TOPP) {
      if (!(c.ratio > 0.0 && c.ratio <= 1.0)) fail(LYC_EINVAL, "top_p: p must lie in (0,1]");
      if (c.select_mode != LYC_SELECT_TOKENS) fail(LYC_ENOTSUP, "decoder: TopP selects tokens only");
    } else if (c.policy_kind == LYC_POLICY_THRESHOLD) {
      if (!(c.ratio > 0.0)) fail(LYC_EINVAL, "threshold: tau must be positive");
      if (c.select_mode != LYC_SELECT_TOKENS) fail(LYC_ENOTSUP, "decoder: Threshold selects tokens only");
    } else {
      fail(LYC_EINVAL, "decoder: unknown policy");
    }
    if (c.select_mode != LYC_SELECT_TOKENS && c.select_mode != LYC_SELECT_BLOCKS &&
        c.select_mode != LYC_SELECT_NONE)
      fail(LYC_EINVAL, "decoder: unknown select mode");
    if (c.block_size != 0 && c.block_size != 64) fail(LYC_ENOTSUP, "decoder: block_size must be 64");
    if (!c.roles) fail(LYC_EINVAL, "RoleMap: null roles");
    for (int g = 0; g < c.n_kv_heads; ++g)
      if (c.roles[g] != 0) fail(LYC_EINVAL, "RoleMap: layer 0 heads must all be Retrieval");
    if (c.select_mode == LYC_SELECT_NONE)
      for (int64_t i = 0; i < (int64_t)c.n_layers * c.n_kv_heads; ++i)
        if (c.roles[i] != 0) fail(LYC_EINVAL, "decoder: sparse heads need a selection mode");
    auto* d = new lyc_decoder();
    d->cfg = c;
    d->roles.assign(c.roles, c.roles + (size_t)c.n_layers * c.n_kv_heads);
    d->cfg.roles = nullptr;
    if (d->cfg.scale == 0.f) d->cfg.scale = (float)(1.0 / std::sqrt((double)c.d_head));
    d->B = c.batch;
    d->H = c.n_kv_heads;
    d->G = c.group_size;
    d->Hq = d->H * d->G;
    d->D = c.d_head;
    d->NL = c.n_layers;
    d->bs = 64;
    const int sms = num_sms();
    d->S = c.num_splits > 0 ? c.num_splits : std::max(1, sms / d->B);
    // The persistent step kernel needs every CTA co-resident: 1 CTA per SM,
    // S*B <= #SMs; its selection handles up to 64 items of 8192 keys per row
    // (block mode: one item); TopP / Threshold run on the per-layer kernels.
    const int64_t nb_cap = (c.seq_cap + d->bs - 1) / d->bs;
    d->fused = lyc::step_supported(c.dtype, c.d_head) && !d->variable_sets() &&
               d->S * d->B <= sms && d->B <= LYC_PLAN_MAX_B && c.seq_cap <= lyc::step_max_keys() &&
               !(c.select_mode == LYC_SELECT_BLOCKS && nb_cap > lyc::step_item_keys()) &&
               (int64_t)lyc::plan_scratch_ints(d->B, d->H, d->S, d->NL) * 4 <= 150 * 1024;
    if (c.select_mode == LYC_SELECT_BLOCKS) {
      d->k_cap = c.policy_kind == LYC_POLICY_RATIO ? nb_cap
                                                   : std::min<int64_t>((c.top_k + 63) / 64, nb_cap);
      d->sel_stride = (nb_cap + 3) & ~(int64_t)3;  // 16-B aligned key rows
    } else {
      d->k_cap = (c.policy_kind == LYC_POLICY_RATIO || d->variable_sets())
                     ? c.seq_cap
                     : std::min<int64_t>(c.top_k, c.seq_cap);
      d->sel_stride = (c.seq_cap + 3) & ~(int64_t)3;
    }
    try {
      const size_t rows = (size_t)d->B * d->H;
      cuda_check(cudaMalloc(&d->idx, rows * d->k_cap * 4), "cudaMalloc index cache");
      cuda_check(cudaMalloc(&d->idx_count, rows * 4), "cudaMalloc index counts");
      cuda_check(cudaMemset(d->idx, 0, rows * d->k_cap * 4), "memset");
      cuda_check(cudaMemset(d->idx_count, 0, rows * 4), "memset");
      cuda_check(cudaMalloc(&d->sel_keys, 2 * rows * d->sel_stride * 4), "cudaMalloc keys");
      cuda_check(cudaMemset(d->sel_keys, 0, 2 * rows * d->sel_stride * 4), "memset");
      cuda_check(cudaMalloc(&d->hist, 2 * rows * LYC_H1_STRIDE * 4), "cudaMalloc hist");
      cuda_check(cudaMemset(d->hist, 0, 2 * rows * LYC_H1_STRIDE * 4), "memset");
      // plan capacity: a pool cut over a group's cells adds at most one unit
      // per cut, so units <= slots + 3 * cells per layer (both planners)
      const int cells = d->n_ctas();
      d->max_units = (int)rows + 3 * cells + 3;
      d->max_merges = (int)rows * d->G;
      const LayerLayout ll = layer_layout((int)rows, cells, d->max_units, d->max_merges);
      d->layer_bytes = ll.bytes;
      d->blob_bytes = (size_t)d->NL * ll.bytes + align_up(sizeof(LycLayerDesc) * d->NL, 256);
      cuda_check(cudaMalloc(&d->blob, d->blob_bytes), "cudaMalloc plan");
      cuda_check(cudaMemset(d->blob, 0, d->blob_bytes), "memset plan");
      d->d_layers = (LycLayerDesc*)(d->blob + (size_t)d->NL * ll.bytes);
      d->h_layers.resize((size_t)d->NL);
      for (int l = 0; l < d->NL; ++l) d->h_layers[(size_t)l] = layer_desc(d->blob + (size_t)l * ll.bytes, ll);
      cuda_check(cudaMemcpy(d->d_layers, d->h_layers.data(), sizeof(LycLayerDesc) * d->NL,
                            cudaMemcpyHostToDevice),
                 "H2D descs");
      cuda_check(cudaMalloc(&d->part_o, (size_t)d->max_units * d->G * d->D * 4), "cudaMalloc part_o");
      cuda_check(cudaMalloc(&d->part_lse, (size_t)d->max_units * d->G * 4), "cudaMalloc part_lse");
      cuda_check(cudaEventCreateWithFlags(&d->staged, cudaEventDisableTiming), "event");
      if (!d->fused) {  // host plans: pinned staging image of the plan blob
        cuda_check(cudaHostAlloc((void**)&d->staging, d->blob_bytes, cudaHostAllocDefault),
                   "cudaHostAlloc staging");
        std::memset(d->staging, 0, d->blob_bytes);
      }
      if (d->fused && c.select_mode != LYC_SELECT_NONE) {  // pooled-selection scratch
        d->bitmap_stride = (lyc::step_bitmap_words(d->sel_stride) + 3) & ~(int64_t)3;
        cuda_check(cudaMalloc(&d->sel_bitmap, 2 * rows * d->bitmap_stride * 4), "cudaMalloc bitmap");
        cuda_check(cudaMalloc(&d->sel_cand, 2 * rows * 2 * d->sel_stride * 4), "cudaMalloc cand");
        cuda_check(cudaMalloc(&d->sel_ccnt, 2 * rows * 256 * 4), "cudaMalloc ccnt");
        // per row: 64 selection items x 256 u16 bucket starts
        cuda_check(cudaMalloc(&d->sel_csub, 2 * rows * 64 * 128 * 4), "cudaMalloc csub");
        cuda_check(cudaMemset(d->sel_csub, 0, 2 * rows * 64 * 128 * 4), "memset");
      }
      if (d->fused) {  // step-kernel counters (two launch-parity sets), planner inputs
        d->rowctr_set = (int64_t)d->NL * (int64_t)rows * 16;
        cuda_check(cudaMalloc(&d->sel_rowctr, 2 * (size_t)d->rowctr_set * 4), "cudaMalloc rowctr");
        cuda_check(cudaMemset(d->sel_rowctr, 0, 2 * (size_t)d->rowctr_set * 4), "memset");
        cuda_check(cudaMalloc(&d->ctr, LYC_CTR_WORDS(d->NL) * 4), "cudaMalloc ctr");
        cuda_check(cudaMemset(d->ctr, 0, LYC_CTR_WORDS(d->NL) * 4), "memset");
        cuda_check(cudaMalloc(&d->d_roles, d->roles.size()), "cudaMalloc roles");
        cuda_check(cudaMemcpy(d->d_roles, d->roles.data(), d->roles.size(), cudaMemcpyHostToDevice),
                   "H2D roles");
        cuda_check(cudaMalloc(&d->d_hdr, sizeof(LycPlanHdr)), "cudaMalloc plan header");
        cuda_check(cudaMemset(d->d_hdr, 0, sizeof(LycPlanHdr)), "memset");
        const size_t key_bytes = (size_t)d->NL * LYC_PLAN_KEY_INTS(d->B) * 4;
        cuda_check(cudaMalloc(&d->d_keys, key_bytes), "cudaMalloc plan keys");
        cuda_check(cudaMemset(d->d_keys, 0, key_bytes), "memset");
        LycPlanIn& in = d->pin;
        std::memset(&in, 0, sizeof(in));
        in.NL = d->NL;
        in.B = d->B;
        in.H = d->H;
        in.G = d->G;
        in.D = d->D;
        in.S = d->S;
        in.bs = d->bs;
        in.select_mode = c.select_mode;
        in.policy_kind = c.policy_kind;
        in.item_keys = lyc::step_item_keys();
        in.seq_cap = c.seq_cap;
        in.k_cap = d->k_cap;
        in.top_k = c.top_k;
        in.ratio = c.ratio;
        in.roles = d->d_roles;
        in.idx = d->idx;
        in.layers = d->d_layers;
        in.hdr = d->d_hdr;
        in.keys = d->d_keys;
        in.max_units = d->max_units;
        in.max_merges = d->max_merges;
      }
      cuda_check(cudaDeviceSynchronize(), "sync");  // creation only: buffers initialised
    } catch (...) {
      lyc_decoder_destroy(d);
      throw;
    }
    *out = d;
    return LYC_OK;
  });
}

int lyc_decoder_destroy(lyc_decoder* d) {
  if (!d) return LYC_OK;
  if (d->exec) cudaGraphExecDestroy(d->exec);
  if (d->graph) cudaGraphDestroy(d->graph);
  for (auto e : d->ev_pre) cudaEventDestroy(e);
  for (auto e : d->ev_post) cudaEventDestroy(e);
  if (d->staged) cudaEventDestroy(d->staged);
  if (d->staging) cudaFreeHost(d->staging);
  free_dev(d->idx);
  free_dev(d->idx_count);
  free_dev(d->sel_keys);
  free_dev(d->refresh_keys);
  free_dev(d->ident_rows);
  free_dev(d->hist);
  free_dev(d->sel_bitmap);
  free_dev(d->sel_cand);
  free_dev(d->sel_ccnt);
  free_dev(d->sel_csub);
  free_dev(d->sel_rowctr);
  free_dev(d->ctr);
  free_dev(d->d_roles);
  free_dev(d->d_hdr);
  free_dev(d->d_keys);
  free_dev(d->trace);
  free_dev(d->set_trace);
  free_dev(d->set_trace_count);
  free_dev(d->part_o);
  free_dev(d->part_lse);
  free_dev(d->blob);
  free_dev(d->shard_ids);
  free_dev(d->shard_cnt);
  free_dev(d->shard_rows);
  free_dev(d->shard_ckey);
  free_dev(d->shard_cidx);
  free_dev(d->shard_pos);
  delete d;
  return LYC_OK;
}

int lyc_decoder_step(lyc_decoder* d, const void* q, const void* k, const void* v, int64_t seq_len,
                     void* out, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    decoder_step(d, q, k, v, seq_len, out, (cudaStream_t)stream);
    return LYC_OK;
  });
}

int lyc_decoder_step_varlen(lyc_decoder* d, const void* q, const void* k, const void* v,
                            const int64_t* seq_lens, void* out, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (!seq_lens) fail(LYC_EINVAL, "decode_step: seq_lens is null");
    decoder_step(d, q, k, v, 0, out, (cudaStream_t)stream, seq_lens);
    return LYC_OK;
  });
}

int lyc_decoder_step_dev(lyc_decoder* d, const void* q, const void* k, const void* v,
                         const int64_t* d_seq_lens, void* out, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (!d_seq_lens) fail(LYC_EINVAL, "decode_step: d_seq_lens is null");
    decoder_step(d, q, k, v, 0, out, (cudaStream_t)stream, nullptr, d_seq_lens);
    return LYC_OK;
  });
}

int lyc_decoder_layer(lyc_decoder* d, int32_t layer, const void* q_l, const void* k, const void* v,
                      int64_t seq_len, void* out_l, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (layer < 0 || layer >= d->NL) fail(LYC_EINVAL, "decoder: layer out of range");
    cudaStream_t st = (cudaStream_t)stream;
    if (d->fused) {
      // the step kernel over [layer, layer + 1): attention, merge and the
      // layer's selection in one launch (re-planning itself when the length
      // leaves the planned 64-row block)
      int64_t seq = seq_len;
      const int64_t* lens = nullptr;
      validate_lens(d, seq, lens);
      // a selection deferred by the previous launch runs in this one when this
      // is the next layer at the same length; otherwise it is completed first
      if (d->pending_sel >= 0 && (d->pending_sel != layer - 1 || d->pending_seq != seq))
        flush_pending(d, st);
      const bool defer_in = d->pending_sel >= 0;
      const bool defer_out = d->defer_sel && layer + 1 < d->NL && layer_selects(d, layer);
      ensure_plan(d, seq, nullptr, nullptr, st);
      launch_step_range(d, layer, layer + 1, q_l, k, v, out_l, st, seq, nullptr, nullptr, defer_in,
                        defer_out);
      d->pending_sel = defer_out ? layer : -1;
      d->pending_seq = seq;
      return LYC_OK;
    }
    decoder_plan(d, seq_len, nullptr, st);
    decoder_layer(d, layer, q_l, k, v, out_l, st);
    return LYC_OK;
  });
}

// Status of the last device-planned step (device lengths are validated by the
// planner): LYC_OK, or LYC_EINVAL when a length was < 1 or > seq_cap (that
// step did nothing).  Synchronises the stream.
int lyc_decoder_status(lyc_decoder* d, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (!d->fused) return LYC_OK;
    LycPlanHdr h{};
    cuda_check(cudaMemcpyAsync(&h, d->d_hdr, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream),
               "D2H plan header");
    cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "sync");
    if (h.status != 0)
      fail(LYC_EINVAL, "decode_step: seq_len of batch item " + std::to_string(h.bad_item) +
                           " is < 1 or exceeds seq_cap");
    return LYC_OK;
  });
}

// ------------------------------------------------------------ shard mode
namespace {
void shard_enter(lyc_decoder* d) {
  if (d->cfg.select_mode == LYC_SELECT_BLOCKS)
    fail(LYC_ENOTSUP, "shard: sequence sharding supports token-mode selection only");
  if (d->variable_sets())
    fail(LYC_ENOTSUP, "shard: sequence sharding supports TopK / Ratio selection only");
  if (d->fused || !d->shard) {
    d->fused = false;  // per-layer kernels: the collective sits between layers
    d->shard = true;   // sparse slots read device counts of the filtered sets
    d->planned_seq = -1;
  }
  if (!d->staging) {
    cuda_check(cudaHostAlloc((void**)&d->staging, d->blob_bytes, cudaHostAllocDefault),
               "cudaHostAlloc staging");
    std::memset(d->staging, 0, d->blob_bytes);
  }
  const size_t rows = (size_t)d->B * d->H;
  if (!d->shard_ids) {
    cuda_check(cudaMalloc(&d->shard_ids, rows * d->k_cap * 4), "cudaMalloc shard ids");
    cuda_check(cudaMalloc(&d->shard_cnt, rows * 4), "cudaMalloc shard cnt");
    cuda_check(cudaMalloc(&d->shard_rows, rows * 4), "cudaMalloc shard rows");
    cuda_check(cudaMalloc(&d->shard_pos, rows * d->k_cap * 4), "cudaMalloc shard pos");
    std::vector<int32_t> iota(rows);
    for (size_t i = 0; i < rows; ++i) iota[i] = (int32_t)i;
    cuda_check(cudaMemcpy(d->shard_rows, iota.data(), rows * 4, cudaMemcpyHostToDevice), "H2D");
  }
}
}  // namespace

int lyc_shard_layer(lyc_decoder* d, int32_t layer, const void* q_l, const void* k, const void* v,
                    int64_t n_local, int64_t row_begin, float* part_o, float* part_lse,
                    uint32_t* cand_key, int32_t* cand_idx, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (layer < 0 || layer >= d->NL) fail(LYC_EINVAL, "decoder: layer out of range");
    if (!part_o || !part_lse || !cand_key || !cand_idx) fail(LYC_EINVAL, "shard: null output");
    if (row_begin < 0) fail(LYC_EINVAL, "shard: row_begin must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    shard_enter(d);
    decoder_plan(d, n_local, nullptr, st);
    lyc_decoder::Layer& ly = d->layers[(size_t)layer];
    ensure_maps(d, k, v);
    ly.ap.tmap_k = d->maps.tmap_k;
    ly.ap.tmap_v = d->maps.tmap_v;
    ly.ap.v.k = k;
    ly.ap.v.v = v;
    ly.ap.v.q = q_l;
    ly.ap.v.out = nullptr;
    ly.ap.v.out_f32 = part_o;
    ly.ap.v.out_lse = part_lse;
    cuda_check(lyc::launch_attn(ly.ap, d->cfg.dtype, d->D, d->B, st), "attention launch");
    ++g_launches;
    if (ly.n_merges) {
      ly.mp.out = nullptr;
      ly.mp.out_f32 = part_o;
      ly.mp.out_lse = part_lse;
      cuda_check(lyc::launch_merge(ly.mp, d->cfg.dtype, st), "merge launch");
      ++g_launches;
    }
    if (ly.n_sel) {  // local top-k of this shard's pooled scores -> (key, global id)
      LycTopkParams tp = ly.tp;
      tp.out = d->shard_ids;
      tp.out_count = d->shard_cnt;
      cuda_check(lyc::launch_topk(tp, ly.n_sel, ly.cluster, st), "topk launch");
      cuda_check(lyc::launch_shard_candidates(tp.keys, tp.key_stride, d->shard_ids, d->shard_cnt,
                                              tp.out_row, ly.n_sel, d->k_cap, row_begin, cand_key,
                                              cand_idx, st),
                 "shard candidates");
      g_launches += 2;
    }
    return LYC_OK;
  });
}

int lyc_shard_merge(lyc_decoder* d, int32_t layer, int32_t world, const float* all_o,
                    const float* all_lse, const uint32_t* all_key, const int32_t* all_idx,
                    int64_t rank_stride, int64_t n_local, int64_t row_begin, int64_t seq_total,
                    void* out_l, int32_t* global_sets, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (layer < 0 || layer >= d->NL) fail(LYC_EINVAL, "decoder: layer out of range");
    if (world < 1) fail(LYC_EINVAL, "shard: world must be >= 1");
    if (seq_total < n_local) fail(LYC_EINVAL, "shard: seq_total < n_local");
    cudaStream_t st = (cudaStream_t)stream;
    shard_enter(d);
    decoder_plan(d, n_local, nullptr, st);
    lyc_decoder::Layer& ly = d->layers[(size_t)layer];
    const int rows = d->B * d->Hq;
    const size_t brows0 = (size_t)d->B * d->H;
    // per-rank strides in 4-byte words: one packed block per rank, or the
    // natural stride of each separately gathered array
    const int64_t so = rank_stride ? rank_stride : (int64_t)rows * d->D;
    const int64_t sl = rank_stride ? rank_stride : (int64_t)rows;
    const int64_t sc = rank_stride ? rank_stride : (int64_t)brows0 * d->k_cap;
    cuda_check(lyc::launch_shard_merge(all_o, all_lse, so, sl, world, rows, d->D, out_l,
                                       d->cfg.dtype, st),
               "shard merge");
    ++g_launches;
    if (ly.n_sel) {
      const int64_t kg = d->budget(seq_total);  // global budget (TopK / Ratio on the full length)
      if (kg > d->k_cap) fail(LYC_ENOTSUP, "shard: global budget exceeds the index-cache capacity");
      const size_t brows = (size_t)d->B * d->H;
      const int64_t n = (int64_t)world * d->k_cap;
      if (world > d->shard_world) {
        free_dev(d->shard_ckey);
        free_dev(d->shard_cidx);
        d->shard_ckey = nullptr;
        d->shard_cidx = nullptr;
        cuda_check(cudaMalloc(&d->shard_ckey, brows * n * 4), "cudaMalloc shard cand");
        cuda_check(cudaMalloc(&d->shard_cidx, brows * n * 4), "cudaMalloc shard cand");
        d->shard_world = world;
      }
      cuda_check(lyc::launch_shard_gather(all_key, all_idx, sc, world, d->k_cap, ly.tp.out_row,
                                          ly.n_sel, d->shard_ckey, d->shard_cidx, st),
                 "shard gather");
      LycTopkParams tp;
      std::memset(&tp, 0, sizeof(tp));
      tp.keys = d->shard_ckey;
      tp.key_stride = n;
      tp.n = (int32_t)n;
      tp.k = (int32_t)kg;
      tp.out = d->shard_pos;
      tp.out_row = d->shard_rows;
      tp.out_stride = d->k_cap;
      tp.out_count = nullptr;
      const int cluster = lyc::topk_cluster_size((int)n, 16384);
      tp.slice = (int32_t)((n + cluster - 1) / cluster);
      tp.clear_keys = 0;
      cuda_check(lyc::launch_topk(tp, ly.n_sel, cluster, st), "shard topk");
      cuda_check(lyc::launch_shard_finalize(d->shard_pos, d->k_cap, d->shard_cidx, n, (int)kg,
                                            ly.tp.out_row, ly.n_sel, row_begin, n_local,
                                            global_sets, d->k_cap, d->idx, d->k_cap, d->idx_count,
                                            st),
                 "shard finalize");
      g_launches += 3;
    }
    return LYC_OK;
  });
}

namespace {
int64_t decoder_capture(lyc_decoder* d, const void* q, const void* k, const void* v,
                        int64_t seq_len, const int64_t* lens, const int64_t* dlens, void* out,
                        void* stream) {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    cudaStream_t st = (cudaStream_t)stream;
    if (dlens && !d->fused) fail(LYC_ENOTSUP, "capture: device-resident lengths need the fused step kernel");
    int64_t seq = seq_len;
    const int64_t* vl = lens;
    if (!dlens) validate_lens(d, seq, vl);
    // per-layer-kernel path: host plan + upload outside the capture (the
    // graph reads the fixed plan layout; replay re-plans to these lengths if
    // another length was planned since).  Fused path: the graph holds the
    // device planner, so every replay plans its own lengths.
    flush_pending(d, st);  // outside the graph
    if (!d->fused) decoder_plan(d, seq_len, lens, st);
    else if (!dlens) ensure_plan(d, seq, vl, nullptr, st);  // outside the graph
    ensure_maps(d, k, v);
    if (d->exec) {
      cudaGraphExecDestroy(d->exec);
      d->exec = nullptr;
    }
    if (d->graph) {
      cudaGraphDestroy(d->graph);
      d->graph = nullptr;
    }
    const int64_t before = g_launches;
    cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      decoder_step(d, q, k, v, seq_len, out, st, lens, dlens);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    d->captured_launches = g_launches - before;
    g_launches = before;  // captured launches execute on replay
    cuda_check(cudaStreamEndCapture(st, &d->graph), "end capture");
    cuda_check(cudaGraphInstantiate(&d->exec, d->graph, 0), "graph instantiate");
    d->captured_gen = d->plan_gen;
    d->captured_key = d->fused && !dlens ? d->host_key : std::vector<int32_t>();
    d->captured_seq = seq_len;
    d->captured_lens.assign(lens ? lens : &seq_len, lens ? lens + d->B : &seq_len + 1);
    return LYC_OK;
}
}  // namespace

int lyc_decoder_capture(lyc_decoder* d, const void* q, const void* k, const void* v,
                        int64_t seq_len, void* out, void* stream) {
  return (int)guarded([&]() -> int64_t {
    return decoder_capture(d, q, k, v, seq_len, nullptr, nullptr, out, stream);
  });
}

int lyc_decoder_capture_varlen(lyc_decoder* d, const void* q, const void* k, const void* v,
                               const int64_t* seq_lens, void* out, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!seq_lens) fail(LYC_EINVAL, "decode_step: seq_lens is null");
    return decoder_capture(d, q, k, v, 0, seq_lens, nullptr, out, stream);
  });
}

int lyc_decoder_capture_dev(lyc_decoder* d, const void* q, const void* k, const void* v,
                            const int64_t* d_seq_lens, void* out, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d_seq_lens) fail(LYC_EINVAL, "decode_step: d_seq_lens is null");
    return decoder_capture(d, q, k, v, 0, nullptr, d_seq_lens, out, stream);
  });
}

int lyc_decoder_replay(lyc_decoder* d, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d || !d->exec) fail(LYC_ESTATE, "decoder: no captured step");
    cudaStream_t st = (cudaStream_t)stream;
    flush_pending(d, st);
    const bool varlen = d->captured_lens.size() == (size_t)d->B && d->captured_seq == 0;
    if (!d->fused && d->plan_gen != d->captured_gen) {
      // another length was planned since the capture: restore the captured plan
      decoder_plan(d, d->captured_seq, varlen ? d->captured_lens.data() : nullptr, st);
      d->captured_gen = d->plan_gen;
    }
    if (d->fused && !d->captured_key.empty() &&
        (!d->host_key_valid || d->host_key != d->captured_key)) {
      // the plan was remade for other lengths since the capture: remake it
      int64_t seq = d->captured_seq;
      const int64_t* lens = varlen ? d->captured_lens.data() : nullptr;
      validate_lens(d, seq, lens);
      ensure_plan(d, seq, lens, nullptr, st);
    }
    cuda_check(cudaGraphLaunch(d->exec, st), "graph launch");
    g_launches += d->captured_launches;
    return LYC_OK;
  });
}

int lyc_decoder_sync_sets(lyc_decoder* d, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    flush_pending(d, (cudaStream_t)stream);
    return LYC_OK;
  });
}

int lyc_decoder_index_cache(lyc_decoder* d, int32_t** ids, int32_t** counts, int64_t* k_cap) {
  if (!d) return LYC_EINVAL;
  if (ids) *ids = d->idx;
  if (counts) *counts = d->idx_count;
  if (k_cap) *k_cap = d->k_cap;
  return LYC_OK;
}

int64_t lyc_decoder_launches_per_step(lyc_decoder* d, int64_t seq_len) {
  return guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (d->fused) return 1;  // the step kernel (+ the planner once per plan key)
    // per-layer kernels: attention, merge (split slots), selection (retrieval layers)
    int64_t seq = seq_len;
    const int64_t* lens = nullptr;
    validate_lens(d, seq, lens);
    std::vector<int> last_r((size_t)d->H, 0);
    int64_t n = 0;
    for (int l = 0; l < d->NL; ++l) {
      HostLaunch L;
      host_slots(d, l, nullptr, seq, false, last_r, L);
      plan_launch(L, d->B, d->H, d->S, d->G);
      n += 1 + (L.merges.empty() ? 0 : 1) + (L.sel_rows.empty() ? 0 : 1);
    }
    return n;
  });
}

int64_t lyc_decoder_step_bytes(lyc_decoder* d, int64_t seq) {
  return guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    int64_t bytes = 0;
    for (int l = 0; l < d->NL; ++l) bytes += lyc_decoder_layer_attn_bytes(d, l, seq);
    return bytes;
  });
}

int64_t lyc_decoder_layer_attn_bytes(lyc_decoder* d, int32_t layer, int64_t seq) {
  return guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (layer < 0 || layer >= d->NL) fail(LYC_EINVAL, "decoder: layer out of range");
    const int64_t e = elem_bytes(d->cfg.dtype), D = d->D;
    const int64_t kb = d->cfg.select_mode == LYC_SELECT_NONE ? seq : d->budget(seq);
    const bool blocks = d->cfg.select_mode == LYC_SELECT_BLOCKS;
    const int64_t sparse_rows = blocks ? std::min<int64_t>(kb * d->bs, seq) : kb;
    int64_t bytes = 0;
    for (int g = 0; g < d->H; ++g) {
      const bool r = d->retrieval(layer, g);
      bytes += (int64_t)d->B * ((r ? seq : sparse_rows) * 2 * D * e + (r ? 0 : 4 * kb));
    }
    bytes += (int64_t)d->B * d->Hq * D * e * 2;  // Q in, O out
    return bytes;
  });
}

int lyc_decoder_set_timing(lyc_decoder* d, int enable) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (enable && d->ev_pre.empty()) {
      d->ev_pre.resize((size_t)d->NL);
      d->ev_post.resize((size_t)d->NL);
      for (int l = 0; l < d->NL; ++l) {
        cuda_check(cudaEventCreate(&d->ev_pre[(size_t)l]), "event create");
        cuda_check(cudaEventCreate(&d->ev_post[(size_t)l]), "event create");
      }
    }
    d->timing = enable != 0;
    return LYC_OK;
  });
}

int lyc_decoder_attn_ms(lyc_decoder* d, float* ms) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (d->ev_pre.empty()) fail(LYC_ESTATE, "decoder: timing was never enabled");
    const int n = d->fused && !d->timed_per_layer ? 1 : d->NL;
    cuda_check(cudaEventSynchronize(d->ev_post[(size_t)n - 1]), "event sync");
    for (int l = 0; l < d->NL; ++l) ms[l] = 0.f;
    for (int l = 0; l < n; ++l)
      cuda_check(cudaEventElapsedTime(&ms[l], d->ev_pre[(size_t)l], d->ev_post[(size_t)l]),
                 "event elapsed");
    return LYC_OK;
  });
}

int lyc_decoder_is_fused(lyc_decoder* d) { return d && d->fused ? 1 : 0; }

int lyc_decoder_tune(lyc_decoder* d, int32_t what, int64_t value) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    switch (what) {
      case LYC_TUNE_RING_STAGES:
        if (value < 0) fail(LYC_EINVAL, "tune: stages must be >= 0");
        d->stages = (int)value;
        d->planned_seq = -1;  // the per-layer path bakes stages into its views
        d->planned_varlen = false;
        return LYC_OK;
      case LYC_TUNE_PER_LAYER_KERNELS:
        if (value) {
          if (!d->staging) {
            cuda_check(cudaHostAlloc((void**)&d->staging, d->blob_bytes, cudaHostAllocDefault),
                       "cudaHostAlloc staging");
            std::memset(d->staging, 0, d->blob_bytes);
          }
          d->fused = false;
          d->planned_seq = -1;
          d->planned_varlen = false;
        } else if (!d->ctr) {
          fail(LYC_ENOTSUP, "tune: this decoder was not created for the step kernel");
        } else if (!d->shard) {
          d->fused = true;
        }
        return LYC_OK;
      case LYC_TUNE_PDL:
        d->pdl = value != 0;
        return LYC_OK;
      case LYC_TUNE_DEFER_SELECTION:
        d->defer_sel = value != 0;
        return LYC_OK;
      default:
        fail(LYC_EINVAL, "tune: unknown knob");
    }
    return LYC_OK;
  });
}

int lyc_decoder_set_trace(lyc_decoder* d, int enable) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (enable && !d->trace) {
      cuda_check(cudaMalloc(&d->trace, (size_t)d->NL * LYC_TRACE_EVENTS * d->n_ctas() * 8), "cudaMalloc trace");
      cuda_check(cudaMemset(d->trace, 0, (size_t)d->NL * LYC_TRACE_EVENTS * d->n_ctas() * 8), "memset trace");
    }
    if (!enable) {
      free_dev(d->trace);
      d->trace = nullptr;
    }
    return LYC_OK;
  });
}

int lyc_decoder_set_trace_sets(lyc_decoder* d, int enable) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    const size_t rows = (size_t)d->NL * d->B * d->H;
    if (enable && !d->set_trace) {
      cuda_check(cudaMalloc(&d->set_trace, rows * d->k_cap * 4), "cudaMalloc set trace");
      cuda_check(cudaMalloc(&d->set_trace_count, rows * 4), "cudaMalloc set trace");
      cuda_check(cudaMemset(d->set_trace_count, 0xff, rows * 4), "memset set trace");
    }
    if (!enable) {
      free_dev(d->set_trace);
      free_dev(d->set_trace_count);
      d->set_trace = d->set_trace_count = nullptr;
    }
    return LYC_OK;
  });
}

int64_t lyc_decoder_traced_sets(lyc_decoder* d, int32_t* ids, int32_t* counts, int64_t cap) {
  return guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (!d->set_trace) fail(LYC_ESTATE, "decoder: set tracing is off");
    const int64_t rows = (int64_t)d->NL * d->B * d->H;
    if (!ids) return d->k_cap;  // size query: ids hold [rows][k_cap]
    if (cap < rows * d->k_cap) fail(LYC_EINVAL, "decoder: set trace buffer too small");
    cuda_check(cudaDeviceSynchronize(), "sync");
    if (d->pending_sel >= 0) {  // a deferred selection (per-layer launches) completes first
      flush_pending(d, nullptr);
      cuda_check(cudaDeviceSynchronize(), "sync");
    }
    cuda_check(cudaMemcpy(ids, d->set_trace, (size_t)rows * d->k_cap * 4, cudaMemcpyDeviceToHost),
               "D2H set trace");
    if (counts)
      cuda_check(cudaMemcpy(counts, d->set_trace_count, (size_t)rows * 4, cudaMemcpyDeviceToHost),
                 "D2H set trace");
    return d->k_cap;
  });
}

int64_t lyc_decoder_trace(lyc_decoder* d, unsigned long long* out, int64_t cap) {
  return guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "decoder: null");
    if (!d->trace) fail(LYC_ESTATE, "decoder: tracing is off");
    const int64_t n = (int64_t)d->NL * LYC_TRACE_EVENTS * d->n_ctas();
    if (!out) return n;  // size query
    if (cap < n) fail(LYC_EINVAL, "decoder: trace buffer too small");
    cuda_check(cudaMemcpy(out, d->trace, (size_t)n * 8, cudaMemcpyDeviceToHost), "D2H trace");
    return n;
  });
}

}  // extern "C"

// ------------------------------------------------------------ KV write path
namespace {
// One 16-B chunk per thread: (b, g, row, chunk) flattened; src rows are
// contiguous per (b, g), cache rows are contiguous per slab.
__global__ void kv_write_kernel(uint4* __restrict__ kc, uint4* __restrict__ vc,
                                const uint4* __restrict__ ks, const uint4* __restrict__ vs,
                                int64_t slabs, int64_t n_rows, int64_t chunks, int64_t slab_chunks,
                                int64_t dst0) {
  const int64_t total = slabs * n_rows * chunks;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % chunks, rs = i / chunks;
    const int64_t r = rs % n_rows, sl = rs / n_rows;
    const int64_t dst = dst0 + sl * slab_chunks + r * chunks + c;
    kc[dst] = ks[i];
    vc[dst] = vs[i];
  }
}
}  // namespace

int lyc_kv_write(void* k_cache, void* v_cache, const lyc_kv_layout* lay, int32_t layer,
                 int64_t pos, int64_t n_rows, const void* k_src, const void* v_src, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!lay) fail(LYC_EINVAL, "KvCache: null layout");
    if (!k_cache || !v_cache || !k_src || !v_src) fail(LYC_EINVAL, "KvCache: null buffer");
    if (lay->n_layers < 1 || lay->batch < 1 || lay->n_kv_heads < 1 || lay->d_head < 1 ||
        lay->seq_cap < 1)
      fail(LYC_EINVAL, "KvCache: all dimensions must be >= 1");
    if (lay->dtype != LYC_DTYPE_F32 && lay->dtype != LYC_DTYPE_BF16) fail(LYC_EINVAL, "KvCache: dtype");
    if (layer < -1 || layer >= lay->n_layers) fail(LYC_EINVAL, "KvCache: layer out of range");
    if (pos < 0 || n_rows < 0 || pos + n_rows > lay->seq_cap)
      fail(LYC_EINVAL, "KvCache: rows beyond seq_cap");
    const bool all = layer == -1;  // every layer: src [n_layers][B][H][n_rows][d]
    const int64_t row_bytes = (int64_t)lay->d_head * (lay->dtype == LYC_DTYPE_BF16 ? 2 : 4);
    if (row_bytes % 16) fail(LYC_ENOTSUP, "KvCache: rows must be a multiple of 16 bytes");
    if (n_rows == 0) return LYC_OK;
    const int64_t chunks = row_bytes / 16;
    const int64_t slabs = (int64_t)lay->batch * lay->n_kv_heads * (all ? lay->n_layers : 1);
    const int64_t slab_chunks = lay->seq_cap * chunks;
    const int64_t dst0 = ((int64_t)(all ? 0 : layer) * lay->batch * lay->n_kv_heads) * slab_chunks +
                         pos * chunks;
    const int64_t total = slabs * n_rows * chunks;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
    kv_write_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        static_cast<uint4*>(k_cache), static_cast<uint4*>(v_cache),
        static_cast<const uint4*>(k_src), static_cast<const uint4*>(v_src), slabs, n_rows, chunks,
        slab_chunks, dst0);
    cuda_check(cudaGetLastError(), "kv write launch");
    ++g_launches;
    return LYC_OK;
  });
}

// ------------------------------------------------------------ cache correction
namespace {
// key splits per (b, g, 128-row block): about one CTA per SM (the tensor-core
// kernel holds a whole SM); clamped to the key tiles at launch
int window_splits(const lyc_kv_layout* lay, int32_t group_size, int32_t window) {
  const int rows = window * group_size, rb = (rows + 127) / 128;
  const int ctas = lay->batch * lay->n_kv_heads * rb;
  return std::max(1, num_sms() / ctas);
}
void window_validate(const lyc_kv_layout* lay, int32_t group_size, int32_t window) {
  if (!lay) fail(LYC_EINVAL, "window: null layout");
  if (lay->n_layers < 1 || lay->batch < 1 || lay->n_kv_heads < 1 || lay->seq_cap < 1)
    fail(LYC_EINVAL, "window: all dimensions must be >= 1");
  if (group_size < 1 || window < 1) fail(LYC_EINVAL, "window: group_size and window must be >= 1");
  if (lay->dtype == LYC_DTYPE_BF16 ? (lay->d_head != 64 && lay->d_head != 128)
                                    : (lay->dtype != LYC_DTYPE_F32 || lay->d_head > 128))
    fail(LYC_ENOTSUP, "window: bf16 caches with d_head 64 or 128, or fp32 with d_head <= 128");
}
}  // namespace

int64_t lyc_window_workspace(const lyc_kv_layout* lay, int32_t group_size, int32_t window) {
  return guarded([&]() -> int64_t {
    window_validate(lay, group_size, window);
    return lyc::window_workspace_bytes(lay->batch, lay->n_kv_heads, group_size, window,
                                       window_splits(lay, group_size, window));
  });
}

int lyc_window_attention(const lyc_kv_layout* lay, int32_t layer, const void* k_cache,
                         const void* v_cache, int32_t group_size, float scale, int64_t start,
                         int32_t window, const void* q, void* out, void* workspace,
                         int64_t workspace_bytes, void* stream) {
  return (int)guarded([&]() -> int64_t {
    window_validate(lay, group_size, window);
    if (layer < 0 || layer >= lay->n_layers) fail(LYC_EINVAL, "window: layer out of range");
    if (start < 0 || start + window > lay->seq_cap) fail(LYC_EINVAL, "window: rows beyond seq_cap");
    if (!k_cache || !v_cache || !q || !out || !workspace) fail(LYC_EINVAL, "window: null buffer");
    const int ns = window_splits(lay, group_size, window);
    if (workspace_bytes < lyc::window_workspace_bytes(lay->batch, lay->n_kv_heads, group_size,
                                                       window, ns))
      fail(LYC_EINVAL, "window: workspace too small");
    const float sc = scale != 0.f ? scale : (float)(1.0 / std::sqrt((double)lay->d_head));
    if (lay->dtype == LYC_DTYPE_F32) {
      cuda_check(lyc::launch_window_f32(q, k_cache, v_cache, layer, lay->batch, lay->n_kv_heads,
                                        group_size, lay->d_head, lay->seq_cap, start, window, sc,
                                        out, (cudaStream_t)stream),
                 "window launch");
      ++g_launches;
      return LYC_OK;
    }
    CUtensorMap mk, mv;
    encode_window_maps(&mk, &mv, k_cache, v_cache, (int64_t)lay->n_layers * lay->batch * lay->n_kv_heads,
                       start + window, lay->seq_cap, lay->d_head);
    cuda_check(lyc::launch_window_tc(mk, mv, q, layer, lay->batch, lay->n_kv_heads, group_size,
                                     lay->d_head, start, window, sc, static_cast<float*>(workspace),
                                     ns, out, (cudaStream_t)stream),
               "window launch");
    g_launches += 2;
    return LYC_OK;
  });
}

// ------------------------------------------------------------ toy-model decode ops

int lyc_gemv(const lyc_gemv_desc* g, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!g || !g->w) fail(LYC_EINVAL, "gemv: null descriptor or weights");
    if (g->M < 1 || g->K < 8 || g->K % 8) fail(LYC_EINVAL, "gemv: M >= 1 and K a multiple of 8");
    if (g->K > 49152) fail(LYC_ENOTSUP, "gemv: K > 49152 (the input vector lives in shared memory)");
    if ((g->x == nullptr) == (g->xb == nullptr)) fail(LYC_EINVAL, "gemv: exactly one of x (fp32) / xb (bf16)");
    if ((uintptr_t)g->w % 16) fail(LYC_EINVAL, "gemv: weights must be 16-B aligned");
    if ((uintptr_t)g->x % 16 || (uintptr_t)g->xb % 16 || (uintptr_t)g->gain % 16)
      fail(LYC_EINVAL, "gemv: x / xb / gain must be 16-B aligned");
    LycGemvParams p{};
    p.w = g->w;
    p.M = g->M;
    p.K = g->K;
    p.x = g->x;
    p.xb = g->xb;
    p.gain = g->gain;
    p.eps = g->eps > 0.f ? g->eps : 1e-6f;
    p.mode = g->mode;
    if (g->flags & ~LYC_GEMV_FLAG_NEXT_IS_GEMV) fail(LYC_EINVAL, "gemv: unknown flags");
    p.flags = g->flags;
    switch (g->mode) {
      case LYC_GEMV_STORE:
      case LYC_GEMV_RESIDUAL:
        if (!g->y) fail(LYC_EINVAL, "gemv: y is null");
        p.y = g->y;
        break;
      case LYC_GEMV_SILU_BF16:
        if (!g->yb) fail(LYC_EINVAL, "gemv: yb is null");
        p.yb = g->yb;
        break;
      case LYC_GEMV_QKV_ROPE:
        if (!g->q_out || !g->k_cache || !g->v_cache) fail(LYC_EINVAL, "gemv: q / k / v outputs are null");
        if (g->d < 2 || g->d % 2 || g->nq < 1 || g->nkv < 1 || g->pos < 0)
          fail(LYC_EINVAL, "gemv: qkv shapes");
        if (g->M != (int64_t)(g->nq + 2 * g->nkv) * g->d) fail(LYC_EINVAL, "gemv: M != (nq + 2 nkv) d");
        p.q_out = g->q_out;
        p.k_cache = g->k_cache;
        p.v_cache = g->v_cache;
        p.slab_stride = g->slab_stride;
        p.nq = g->nq;
        p.nkv = g->nkv;
        p.d = g->d;
        p.pos = g->pos;
        break;
      default:
        fail(LYC_EINVAL, "gemv: unknown mode");
    }
    if (g->prefetch && g->prefetch_bytes > 0) {
      if ((uintptr_t)g->prefetch % 16) fail(LYC_EINVAL, "gemv: prefetch must be 16-B aligned");
      p.pf = g->prefetch;
      p.pf_bytes = g->prefetch_bytes & ~(int64_t)15;
    }
    cuda_check(lyc::launch_gemv(p, num_sms(), (cudaStream_t)stream), "gemv launch");
    ++g_launches;
    return LYC_OK;
  });
}

// ------------------------------------------------------------ set refresh
int lyc_decoder_refresh_sets(lyc_decoder* d, int32_t layer, const void* q_last, const void* k,
                             int64_t len, void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!d) fail(LYC_EINVAL, "refresh: null decoder");
    if (layer < 0 || layer >= d->NL) fail(LYC_EINVAL, "refresh: layer out of range");
    if (!q_last || !k) fail(LYC_EINVAL, "refresh: null buffer");
    if (len < 1 || len > d->cfg.seq_cap) fail(LYC_EINVAL, "refresh: len must be in [1, seq_cap]");
    if (d->cfg.select_mode == LYC_SELECT_NONE) fail(LYC_ESTATE, "refresh: the decoder selects nothing");
    if (d->shard) fail(LYC_ENOTSUP, "refresh: not in sequence-shard mode");
    cudaStream_t st = (cudaStream_t)stream;
    flush_pending(d, st);
    const size_t rows = (size_t)d->B * d->H;
    if (!d->refresh_keys) {
      cuda_check(cudaMalloc(&d->refresh_keys, rows * d->sel_stride * 4), "cudaMalloc refresh keys");
      cuda_check(cudaMalloc(&d->ident_rows, rows * 4), "cudaMalloc rows");
      std::vector<int32_t> id(rows);
      for (size_t i = 0; i < rows; ++i) id[i] = (int32_t)i;
      cuda_check(cudaMemcpy(d->ident_rows, id.data(), rows * 4, cudaMemcpyHostToDevice), "H2D rows");
    }
    const bool blocks = d->cfg.select_mode == LYC_SELECT_BLOCKS;
    const int64_t n = blocks ? (len + d->bs - 1) / d->bs : len;
    if (blocks) cuda_check(cudaMemsetAsync(d->refresh_keys, 0, rows * d->sel_stride * 4, st), "memset keys");
    const int esz = d->cfg.dtype == LYC_DTYPE_BF16 ? 2 : 4;
    const char* k_layer = static_cast<const char*>(k) + (size_t)layer * rows * d->cfg.seq_cap * d->D * esz;
    cuda_check(lyc::launch_refresh_scores(q_last, k_layer, d->cfg.seq_cap, d->B, d->H, d->G, d->D,
                                          d->cfg.dtype == LYC_DTYPE_BF16 ? 1 : 0, len,
                                          d->refresh_keys, d->sel_stride, blocks ? 1 : 0, st),
               "refresh launch");
    ++g_launches;
    if (d->variable_sets()) {  // TopP / Threshold (policy.hpp:73-101)
      LycPolicyParams pp{};
      pp.keys = d->refresh_keys;
      pp.key_stride = d->sel_stride;
      pp.n = (int32_t)n;
      pp.kind = d->cfg.policy_kind == LYC_POLICY_TOPP ? LYC_POLICY_KIND_TOPP : LYC_POLICY_KIND_THRESHOLD;
      pp.value = d->cfg.ratio;
      pp.score_scale = d->cfg.scale;  // keys are pooled-mean scores
      pp.out = d->idx;
      pp.out_row = d->ident_rows;
      pp.out_stride = d->k_cap;
      pp.out_count = d->idx_count;
      pp.row_n = nullptr;
      cuda_check(lyc::launch_policy(pp, (int)rows, st), "policy launch");
    } else {  // TopK / Ratio (policy.hpp:57-72)
      const int cluster = lyc::topk_cluster_size((int)n, 16384);
      LycTopkParams tp{};
      tp.keys = d->refresh_keys;
      tp.key_stride = d->sel_stride;
      tp.n = (int32_t)n;
      tp.k = (int32_t)d->budget(len);
      tp.out = d->idx;
      tp.out_row = d->ident_rows;
      tp.out_stride = d->k_cap;
      tp.out_count = d->idx_count;
      tp.slice = (int32_t)((n + cluster - 1) / cluster);
      tp.clear_keys = 0;
      tp.row_n = nullptr;
      tp.row_k = nullptr;
      cuda_check(lyc::launch_topk(tp, (int)rows, cluster, st), "topk launch");
    }
    ++g_launches;
    return LYC_OK;
  });
}

// ------------------------------------------------------------ planner self-test
// The device planner (plan.cuh, run here sequentially) against the host-order
// planner (plan_step_launch) on identical inputs, every layer: slots, units,
// split offsets, merge tasks and selection rows must agree exactly.
int lyc_plan_selftest(const lyc_decode_config* cfg, int64_t seq_len, const int64_t* seq_lens,
                      int32_t n_sms) {
  return (int)guarded([&]() -> int64_t {
    if (!cfg || !cfg->roles) fail(LYC_EINVAL, "selftest: null config");
    lyc_decoder dd;
    lyc_decoder* d = &dd;
    d->cfg = *cfg;
    d->roles.assign(cfg->roles, cfg->roles + (size_t)cfg->n_layers * cfg->n_kv_heads);
    d->B = cfg->batch;
    d->H = cfg->n_kv_heads;
    d->G = cfg->group_size;
    d->Hq = d->H * d->G;
    d->D = cfg->d_head;
    d->NL = cfg->n_layers;
    d->S = cfg->num_splits > 0 ? cfg->num_splits : std::max(1, n_sms / d->B);
    d->fused = true;
    if (d->B > LYC_PLAN_MAX_B || d->S * d->B > n_sms) fail(LYC_ENOTSUP, "selftest: not a fused shape");
    const int64_t nb_cap = (cfg->seq_cap + 63) / 64;
    d->k_cap = cfg->select_mode == LYC_SELECT_BLOCKS
                   ? (cfg->policy_kind == LYC_POLICY_RATIO ? nb_cap : std::min<int64_t>((cfg->top_k + 63) / 64, nb_cap))
                   : (cfg->policy_kind == LYC_POLICY_RATIO ? cfg->seq_cap : std::min<int64_t>(cfg->top_k, cfg->seq_cap));
    d->idx = reinterpret_cast<int32_t*>(uintptr_t{0x7f0000000000});  // a device address value only
    int64_t seq = seq_len;
    const int64_t* lens = seq_lens;
    validate_lens(d, seq, lens);
    const bool varlen = lens != nullptr;
    const int B = d->B, H = d->H, G = d->G, cells = d->n_ctas(), BH = B * H;
    const int max_units = BH + 3 * cells + 3, max_merges = BH * G;
    LycPlanIn in{};
    in.NL = d->NL; in.B = B; in.H = H; in.G = G; in.D = d->D; in.S = d->S; in.bs = 64;
    in.select_mode = cfg->select_mode; in.policy_kind = cfg->policy_kind;
    in.item_keys = lyc::step_item_keys(); in.seq_cap = cfg->seq_cap; in.k_cap = d->k_cap;
    in.top_k = cfg->top_k; in.ratio = cfg->ratio; in.roles = d->roles.data(); in.idx = d->idx;
    in.max_units = max_units; in.max_merges = max_merges; in.seq = seq;
    LycPlanHdr hdr{};
    in.hdr = &hdr;
    if (seq_lens) {
      in.has_lens = 1;
      for (int b = 0; b < B; ++b) in.lens[b] = (int32_t)seq_lens[b];
    }
    const bool blocks = cfg->select_mode == LYC_SELECT_BLOCKS;
    const bool none = cfg->select_mode == LYC_SELECT_NONE;
    std::vector<int> last_r((size_t)H, 0);
    auto mismatch = [&](int l, const std::string& what) {
      fail(LYC_ESTATE, "selftest: layer " + std::to_string(l) + ": " + what);
    };
    for (int l = 0; l < d->NL; ++l) {
      HostLaunch L;
      host_slots(d, l, lens, seq, varlen, last_r, L);
      int free_from = cells;
      if (!none) {
        const int64_t nk = blocks ? (seq + 63) / 64 : seq;
        const int64_t items = (nk + lyc::step_item_keys() - 1) / lyc::step_item_keys();
        const int64_t n_items = (int64_t)L.sel_rows.size() * items;
        if (n_items > 0 && 2 * n_items <= cells) free_from = cells - (int)n_items;
      }
      bool ragged = false;
      for (int b = 1; b < B; ++b) {
        const int64_t lb = varlen ? lens[b] : seq, l0 = varlen ? lens[0] : seq;
        ragged = ragged || (lb + 63) / 64 != (l0 + 63) / 64 || d->budget(lb) != d->budget(l0);
      }
      plan_step_launch(L, B, H, d->S, G, l, free_from, ragged);
      std::vector<LycSlot> slots((size_t)BH), uslots((size_t)max_units);
      std::vector<LycUnit> units((size_t)max_units);
      std::vector<LycMergeTask> merges((size_t)max_merges);
      std::vector<int32_t> split((size_t)cells + 1), srow((size_t)BH), sn((size_t)BH), sk((size_t)BH);
      int32_t n_merges = -1, n_sel = -1, n_units = -1;
      lyc::PlanOut o{slots.data(), units.data(), uslots.data(), split.data(), merges.data(),
                     srow.data(), sn.data(), sk.data(), &n_merges, &n_sel, &n_units};
      lyc::plan_layer_host(in, l, o);
      if (hdr.status) mismatch(l, "planner flagged the lengths");
      if (n_units != (int)L.units.size()) mismatch(l, "unit count " + std::to_string(n_units) + " vs " + std::to_string(L.units.size()));
      if (n_merges != (int)L.merges.size()) mismatch(l, "merge count");
      if (n_sel != (int)L.sel_rows.size()) mismatch(l, "selection rows");
      for (int i = 0; i < BH; ++i)
        if (std::memcmp(&slots[(size_t)i], &L.slots[(size_t)i], sizeof(LycSlot)))
          mismatch(l, "slot " + std::to_string(i));
      for (int u = 0; u < n_units; ++u) {
        const LycUnit &a = units[(size_t)u], &b = L.units[(size_t)u];
        if (a.slot != b.slot || a.begin != b.begin || a.end != b.end || a.hls != b.hls)
          mismatch(l, "unit " + std::to_string(u));
        if (std::memcmp(&uslots[(size_t)u], &L.slots[(size_t)b.slot], sizeof(LycSlot)))
          mismatch(l, "unit slot " + std::to_string(u));
      }
      for (int c = 0; c <= cells; ++c)
        if (split[(size_t)c] != L.split_off[(size_t)c]) mismatch(l, "split offset " + std::to_string(c));
      for (int m = 0; m < n_merges; ++m)
        if (std::memcmp(&merges[(size_t)m], &L.merges[(size_t)m], sizeof(LycMergeTask)))
          mismatch(l, "merge task " + std::to_string(m));
      for (int r = 0; r < n_sel; ++r) {
        if (srow[(size_t)r] != L.sel_rows[(size_t)r]) mismatch(l, "selection row " + std::to_string(r));
        const int b = L.sel_rows[(size_t)r] / H;
        const int64_t len_b = varlen ? lens[b] : seq;
        const int64_t want_n = varlen ? L.sel_n[(size_t)r] : (blocks ? (len_b + 63) / 64 : len_b);
        const int64_t want_k = varlen ? L.sel_k[(size_t)r] : d->budget(len_b);
        if (sn[(size_t)r] != want_n || sk[(size_t)r] != want_k) mismatch(l, "selection budget " + std::to_string(r));
      }
    }
    const int64_t mx = varlen ? *std::max_element(lens, lens + B) : seq;
    if (hdr.seq_len != mx || hdr.n_keys != (blocks ? (mx + 63) / 64 : mx) || hdr.k_sel != d->budget(mx))
      fail(LYC_ESTATE, "selftest: plan header");
    return LYC_OK;
  });
}

// KvCache::append of the current token for device-resident lengths: row
// d_seq_lens[b] - 1 of every (b, g) of layer `layer` (-1: every layer) from
// src [n_layers?][B][H][d] -- the graph-capturable companion of
// lyc_decoder_step_dev / lyc_decoder_capture_dev.
namespace {
__global__ void kv_append_kernel(uint4* __restrict__ kc, uint4* __restrict__ vc,
                                 const uint4* __restrict__ ks, const uint4* __restrict__ vs,
                                 const int64_t* __restrict__ lens, int64_t slabs, int64_t BH,
                                 int64_t H, int64_t chunks, int64_t slab_chunks, int64_t slab0,
                                 int64_t seq_cap) {
  const int64_t total = slabs * chunks;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % chunks, sl = i / chunks;
    const int64_t b = (sl % BH) / H;
    const int64_t pos = lens[b] - 1;
    if (pos < 0 || pos >= seq_cap) continue;  // invalid length: the planner rejects the step
    const int64_t dst = (slab0 + sl) * slab_chunks + pos * chunks + c;
    kc[dst] = ks[i];
    vc[dst] = vs[i];
  }
}
}  // namespace

int lyc_kv_append_dev(void* k_cache, void* v_cache, const lyc_kv_layout* lay, int32_t layer,
                      const int64_t* d_seq_lens, const void* k_src, const void* v_src,
                      void* stream) {
  return (int)guarded([&]() -> int64_t {
    if (!lay) fail(LYC_EINVAL, "KvCache: null layout");
    if (!k_cache || !v_cache || !k_src || !v_src || !d_seq_lens) fail(LYC_EINVAL, "KvCache: null buffer");
    if (lay->n_layers < 1 || lay->batch < 1 || lay->n_kv_heads < 1 || lay->d_head < 1 ||
        lay->seq_cap < 1)
      fail(LYC_EINVAL, "KvCache: all dimensions must be >= 1");
    if (lay->dtype != LYC_DTYPE_F32 && lay->dtype != LYC_DTYPE_BF16) fail(LYC_EINVAL, "KvCache: dtype");
    if (layer < -1 || layer >= lay->n_layers) fail(LYC_EINVAL, "KvCache: layer out of range");
    const int64_t row_bytes = (int64_t)lay->d_head * (lay->dtype == LYC_DTYPE_BF16 ? 2 : 4);
    if (row_bytes % 16) fail(LYC_ENOTSUP, "KvCache: rows must be a multiple of 16 bytes");
    const bool all = layer == -1;
    const int64_t chunks = row_bytes / 16, BH = (int64_t)lay->batch * lay->n_kv_heads;
    const int64_t slabs = BH * (all ? lay->n_layers : 1);
    const int64_t total = slabs * chunks;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
    kv_append_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        static_cast<uint4*>(k_cache), static_cast<uint4*>(v_cache),
        static_cast<const uint4*>(k_src), static_cast<const uint4*>(v_src), d_seq_lens, slabs, BH,
        lay->n_kv_heads, chunks, lay->seq_cap * chunks, (all ? 0 : (int64_t)layer) * BH,
        lay->seq_cap);
    cuda_check(cudaGetLastError(), "kv append launch");
    ++g_launches;
    return LYC_OK;
  });
}
