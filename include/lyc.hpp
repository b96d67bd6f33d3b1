// lyc.hpp -- C++20 host API of the B200-native LycheeDecode hybrid-head decode
// attention, the drop-in for the reference's header-only C++ library `hh`
// (/root/reference/proj/include/hh).  Header-only, on top of the C-ABI in
// lyc.h (link liblyc.so and libcudart).
//
// Mirrors, with the same names, argument meaning and exception types:
//   hh::kernel::BlockIndexSet / WorkUnit / SplitSchedule  kernel_sim.hpp:20-61
//   hh::kernel::plan_splits                               kernel_sim.hpp:63-110
//   hh::kernel::Workload / RunResult / run                kernel_sim.hpp:120-146, 227-279
//   hh::kernel::CostReport / latency_model                kernel_sim.hpp:284-316
//   hh::args_top_k                                        attention.hpp:108-123
//   hh::SparsityPolicy / fraction_budget / select_tokens  policy.hpp:20-104 (TopK, Ratio)
//   hh::DecodeEngine::decode_step attention loop          decode_engine.hpp:109-151
//     (role mask rolemap.hpp:33-35, layer 0 forced retrieval :121, per-KV-head
//      index cache sets_ :251)  -> lyc::HybridDecoder
//
// Error model: the C-ABI status codes come back as the reference's exception
// types -- std::invalid_argument (LYC_EINVAL), std::logic_error (LYC_ESTATE);
// lyc::cuda_error / lyc::not_supported (std::runtime_error) for device
// failures and shapes the device kernels do not cover.
//
// `run` is generic over the workload type: it accepts lyc::kernel::Workload<T>
// or the reference's hh::kernel::Workload<T> itself (same members), and
// `run_as<R>` fills any result type with the reference's RunResult members,
// so reference call sites switch with a one-line change:
//     auto r = hh::kernel::run(w, splits, workers);                       // CPU
//     auto r = lyc::kernel::run_as<hh::kernel::RunResult<float>>(w, splits); // B200
// The device computes in fp32 (float / double workloads: inputs are converted
// to fp32 on upload) or bf16 (HybridDecoder).
#ifndef LYC_HPP_
#define LYC_HPP_

#include <cuda_runtime.h>

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "lyc.h"

namespace lyc {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct not_supported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Status code -> the reference's exception type.
inline int64_t check(int64_t rc) {
  if (rc >= 0) return rc;
  const std::string msg = lyc_last_error();
  switch (rc) {
    case LYC_EINVAL: throw std::invalid_argument(msg);
    case LYC_ESTATE: throw std::logic_error(msg);
    case LYC_ENOTSUP: throw not_supported(msg);
    default: throw cuda_error(msg);
  }
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device buffer (RAII).
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t bytes) : bytes_(bytes) {
    if (bytes) cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc");
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), bytes_(o.bytes_) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    return *this;
  }
  void* get() const { return p_; }
  template <typename U>
  U* as() const {
    return static_cast<U*>(p_);
  }
  std::size_t bytes() const { return bytes_; }
  void upload(const void* src, std::size_t n) {
    cuda_check(cudaMemcpy(p_, src, n, cudaMemcpyHostToDevice), "H2D");
  }
  void download(void* dst, std::size_t n) const {
    cuda_check(cudaMemcpy(dst, p_, n, cudaMemcpyDeviceToHost), "D2H");
  }

 private:
  void* p_ = nullptr;
  std::size_t bytes_ = 0;
};

namespace kernel {

// kernel_sim.hpp:20-42
struct BlockIndexSet {
  std::size_t batch = 0;
  std::size_t n_kv_heads = 0;
  std::vector<std::vector<std::uint32_t>> ids;  // [b * n_kv_heads + g]

  std::size_t slot(std::size_t b, std::size_t g) const { return b * n_kv_heads + g; }
};

// kernel_sim.hpp:45-50
struct WorkUnit {
  std::size_t kv_head = 0;
  std::size_t begin = 0;
  std::size_t end = 0;
  std::size_t head_local_split = 0;
};

// kernel_sim.hpp:54-61
struct SplitSchedule {
  std::size_t batch = 0;
  std::size_t num_splits = 0;
  std::vector<std::vector<std::vector<WorkUnit>>> units;  // [b][split]
  std::vector<std::vector<std::size_t>> split_blocks;     // [b][split]
  std::vector<std::vector<std::size_t>> head_blocks;      // [b][kv head]
  std::vector<std::vector<std::size_t>> head_split_count; // [b][kv head]
};

// kernel_sim.hpp:63-110, through the library's planner (lyc_plan_splits) --
// the same plan the device kernels execute.  Any BlockIndexSet-like type.
template <class Blocks>
SplitSchedule plan_splits(const Blocks& blocks, std::size_t num_splits) {
  const std::size_t B = blocks.batch, H = blocks.n_kv_heads;
  if (blocks.ids.size() != B * H) throw std::invalid_argument("BlockIndexSet: slot count mismatch");
  std::vector<int64_t> hb(B * H);
  std::size_t total = 0;
  for (std::size_t i = 0; i < B * H; ++i) total += (hb[i] = (int64_t)blocks.ids[i].size());
  const std::size_t S = num_splits < 1 ? 1 : num_splits;
  (void)total;
  std::vector<int64_t> sb(B * S), hsc(B * H);
  const int64_t n = check(lyc_plan_splits((int64_t)B, (int64_t)H, hb.data(), (int64_t)num_splits,
                                          sb.data(), hsc.data(), nullptr, 0));  // count
  std::vector<int64_t> units((std::size_t)n * 6);
  check(lyc_plan_splits((int64_t)B, (int64_t)H, hb.data(), (int64_t)num_splits, sb.data(),
                        hsc.data(), units.data(), n));
  SplitSchedule s;
  s.batch = B;
  s.num_splits = num_splits;
  s.units.assign(B, std::vector<std::vector<WorkUnit>>(num_splits));
  s.split_blocks.assign(B, std::vector<std::size_t>(num_splits));
  s.head_blocks.assign(B, std::vector<std::size_t>(H));
  s.head_split_count.assign(B, std::vector<std::size_t>(H));
  for (std::size_t b = 0; b < B; ++b) {
    for (std::size_t sp = 0; sp < num_splits; ++sp) s.split_blocks[b][sp] = (std::size_t)sb[b * S + sp];
    for (std::size_t g = 0; g < H; ++g) {
      s.head_blocks[b][g] = (std::size_t)hb[b * H + g];
      s.head_split_count[b][g] = (std::size_t)hsc[b * H + g];
    }
  }
  for (int64_t u = 0; u < n; ++u) {  // records (b, s, g, begin, end, head_local_split)
    const int64_t* r = units.data() + 6 * u;
    s.units[(std::size_t)r[0]][(std::size_t)r[1]].push_back(
        WorkUnit{(std::size_t)r[2], (std::size_t)r[3], (std::size_t)r[4], (std::size_t)r[5]});
  }
  return s;
}

// kernel_sim.hpp:284-316
struct CostReport {
  std::size_t total_blocks = 0;
  std::size_t pooled_critical_blocks = 0;
  std::size_t naive_critical_blocks = 0;
  double mean_split_blocks = 0.0;
  double balance_ratio = 0.0;
  std::size_t bytes_per_block = 0;
  std::size_t pooled_critical_bytes = 0;
  std::size_t naive_critical_bytes = 0;
};

template <class Schedule>
CostReport latency_model(const Schedule& sched, std::size_t bytes_per_block) {
  const std::size_t B = sched.batch;
  const std::size_t H = B ? sched.head_blocks[0].size() : 0;
  std::vector<int64_t> hb;
  for (std::size_t b = 0; b < B; ++b)
    for (std::size_t g = 0; g < H; ++g) hb.push_back((int64_t)sched.head_blocks[b][g]);
  int64_t o6[6];
  double o2[2];
  check(lyc_latency_model((int64_t)B, (int64_t)H, hb.data(), (int64_t)sched.num_splits,
                          (int64_t)bytes_per_block, o6, o2));
  CostReport r;
  r.total_blocks = (std::size_t)o6[0];
  r.pooled_critical_blocks = (std::size_t)o6[1];
  r.naive_critical_blocks = (std::size_t)o6[2];
  r.bytes_per_block = (std::size_t)o6[3];
  r.pooled_critical_bytes = (std::size_t)o6[4];
  r.naive_critical_bytes = (std::size_t)o6[5];
  r.mean_split_blocks = o2[0];
  r.balance_ratio = o2[1];
  return r;
}

// mat.hpp:12-30 (row-major, `data` holds rows*cols values)
template <typename T>
struct Matrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<T> data;
  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, T(0)) {}
  T* row(std::size_t r) { return data.data() + r * cols; }
  const T* row(std::size_t r) const { return data.data() + r * cols; }
};

// kernel_sim.hpp:120-146
template <typename T>
struct Workload {
  std::size_t batch = 0;
  std::size_t n_kv_heads = 0;
  std::size_t group_size = 1;
  std::size_t d_head = 0;
  std::size_t seq_len = 0;
  std::size_t block_size = 64;
  T scale = T(1);
  std::vector<Matrix<T>> keys, values;  // [b * n_kv_heads + g], seq x d
  std::vector<std::vector<T>> queries;  // [b * n_q_heads + h], d
  BlockIndexSet blocks;

  std::size_t n_q_heads() const { return n_kv_heads * group_size; }
  std::size_t n_blocks() const { return (seq_len + block_size - 1) / block_size; }
};

// kernel_sim.hpp:227-232
template <typename T>
struct RunResult {
  std::vector<std::vector<T>> outputs;  // [b * n_q_heads + h]
  SplitSchedule schedule;
  std::vector<std::uint32_t> block_exec_counts;
};

namespace detail {
template <class W>
using value_t = std::remove_cvref_t<decltype(std::declval<const W&>().scale)>;

// Host validation with the reference's messages (kernel_sim.hpp:27-41, 136-145).
template <class W>
void validate(const W& w) {
  if (w.batch < 1 || w.n_kv_heads < 1 || w.group_size < 1 || w.d_head < 1 || w.seq_len < 1 ||
      w.block_size < 1)
    throw std::invalid_argument("Workload: all dimensions must be >= 1");
  if (w.keys.size() != w.batch * w.n_kv_heads || w.values.size() != w.keys.size())
    throw std::invalid_argument("Workload: KV slot count mismatch");
  if (w.queries.size() != w.batch * w.n_kv_heads * w.group_size)
    throw std::invalid_argument("Workload: query slot count mismatch");
  if (w.blocks.ids.size() != w.batch * w.n_kv_heads)
    throw std::invalid_argument("BlockIndexSet: slot count mismatch");
  const std::size_t nb = (w.seq_len + w.block_size - 1) / w.block_size;
  for (const auto& list : w.blocks.ids) {
    bool first = true;
    std::uint32_t prev = 0;
    for (std::uint32_t id : list) {
      if (id >= nb) throw std::invalid_argument("BlockIndexSet: block id out of range");
      if (!first && id <= prev)
        throw std::invalid_argument("BlockIndexSet: block ids must be strictly ascending");
      prev = id;
      first = false;
    }
  }
  for (std::size_t i = 0; i < w.keys.size(); ++i)
    if (w.keys[i].rows < w.seq_len || w.keys[i].cols != w.d_head || w.values[i].rows < w.seq_len ||
        w.values[i].cols != w.d_head)
      throw std::invalid_argument("Workload: K/V matrix shape mismatch");
  for (const auto& q : w.queries)
    if (q.size() != w.d_head) throw std::invalid_argument("Workload: query length mismatch");
}

// Member-wise copy of our schedule into any SplitSchedule-like type.
template <class S>
S convert_schedule(const SplitSchedule& s) {
  if constexpr (std::is_same_v<S, SplitSchedule>) {
    return s;
  } else {
    S o;
    o.batch = s.batch;
    o.num_splits = s.num_splits;
    o.split_blocks = s.split_blocks;
    o.head_blocks = s.head_blocks;
    o.head_split_count = s.head_split_count;
    o.units.resize(s.units.size());
    for (std::size_t b = 0; b < s.units.size(); ++b) {
      o.units[b].resize(s.units[b].size());
      for (std::size_t sp = 0; sp < s.units[b].size(); ++sp)
        for (const WorkUnit& u : s.units[b][sp]) {
          typename std::remove_cvref_t<decltype(o.units[b][sp])>::value_type x;
          x.kv_head = u.kv_head;
          x.begin = u.begin;
          x.end = u.end;
          x.head_local_split = u.head_local_split;
          o.units[b][sp].push_back(x);
        }
    }
    return o;
  }
}
}  // namespace detail

// kernel_sim.hpp:237-279 on the B200: validate on the host, stage the
// workload to device memory (fp32), execute every (b, split) cell as one CTA
// (lyc_workload_run), copy outputs and the per-(b, g, list index) execution
// counters back.  n_workers is accepted for signature compatibility (the
// device result is independent of it, like the reference's).  Fills any
// result type R with the reference's RunResult members.
template <class R, class W>
R run_as(const W& w, std::size_t num_splits, std::size_t n_workers = 1, void* stream = nullptr) {
  (void)n_workers;
  using T = detail::value_t<W>;
  static_assert(std::is_floating_point_v<T>, "Workload element type must be float or double");
  detail::validate(w);
  if (num_splits < 1) throw std::invalid_argument("plan_splits: num_splits must be >= 1");
  const std::size_t B = w.batch, H = w.n_kv_heads, G = w.group_size, D = w.d_head, L = w.seq_len;
  const std::size_t slots = B * H, nq = B * H * G;
  std::vector<float> kv((std::size_t)2 * slots * L * D), q(nq * D);
  for (std::size_t i = 0; i < slots; ++i)
    for (std::size_t r = 0; r < L; ++r)
      for (std::size_t c = 0; c < D; ++c) {
        kv[(i * L + r) * D + c] = (float)w.keys[i].data[r * w.keys[i].cols + c];
        kv[((slots + i) * L + r) * D + c] = (float)w.values[i].data[r * w.values[i].cols + c];
      }
  for (std::size_t h = 0; h < nq; ++h)
    for (std::size_t c = 0; c < D; ++c) q[h * D + c] = (float)w.queries[h][c];
  std::vector<int64_t> off(slots + 1, 0), ids;
  for (std::size_t i = 0; i < slots; ++i) {
    for (std::uint32_t id : w.blocks.ids[i]) ids.push_back((int64_t)id);
    off[i + 1] = (int64_t)ids.size();
  }
  const std::size_t nb = (L + w.block_size - 1) / w.block_size;
  DeviceBuffer d_kv(kv.size() * 4), d_q(q.size() * 4), d_out(nq * D * 4), d_cnt(slots * nb * 4);
  d_kv.upload(kv.data(), kv.size() * 4);
  d_q.upload(q.data(), q.size() * 4);
  cuda_check(cudaMemset(d_cnt.get(), 0, slots * nb * 4), "memset");
  lyc_workload lw{};
  lw.batch = (int64_t)B;
  lw.n_kv_heads = (int64_t)H;
  lw.group_size = (int64_t)G;
  lw.d_head = (int64_t)D;
  lw.seq_len = (int64_t)L;
  lw.block_size = (int64_t)w.block_size;
  lw.kv_row_stride = (int64_t)L;
  lw.scale = (float)w.scale;
  lw.dtype = LYC_DTYPE_F32;
  lw.k = d_kv.get();
  lw.v = d_kv.as<float>() + slots * L * D;
  lw.q = d_q.get();
  lw.blk_off = off.data();
  lw.blk_ids = ids.data();
  check(lyc_workload_run(&lw, (int64_t)num_splits, d_out.get(), d_cnt.as<uint32_t>(), stream));
  cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "workload run");
  std::vector<float> out(nq * D);
  std::vector<std::uint32_t> cnt(slots * nb);
  d_out.download(out.data(), out.size() * 4);
  d_cnt.download(cnt.data(), cnt.size() * 4);
  R res;
  res.outputs.assign(nq, {});
  for (std::size_t h = 0; h < nq; ++h) res.outputs[h].assign(out.begin() + h * D, out.begin() + (h + 1) * D);
  for (std::size_t i = 0; i < slots; ++i)  // (b, g, index) order, kernel_sim.hpp:266-275
    for (std::size_t j = 0; j < w.blocks.ids[i].size(); ++j) res.block_exec_counts.push_back(cnt[i * nb + j]);
  res.schedule = detail::convert_schedule<std::remove_cvref_t<decltype(res.schedule)>>(
      lyc::kernel::plan_splits(w.blocks, num_splits));
  return res;
}

template <class W>
RunResult<detail::value_t<W>> run(const W& w, std::size_t num_splits, std::size_t n_workers = 1) {
  return run_as<RunResult<detail::value_t<W>>>(w, num_splits, n_workers);
}

}  // namespace kernel

// attention.hpp:17-33
struct TokenSet {
  std::vector<std::size_t> indices;
  std::size_t size() const { return indices.size(); }
  bool empty() const { return indices.empty(); }
  void validate(std::size_t seq_len) const {
    std::size_t prev = 0;
    bool first = true;
    for (std::size_t i : indices) {
      if (i >= seq_len) throw std::invalid_argument("TokenSet: index out of range");
      if (!first && i <= prev) throw std::invalid_argument("TokenSet: indices must be strictly ascending");
      prev = i;
      first = false;
    }
  }
};

// attention.hpp:108-123: the min(k, n) largest, ties to the lower index,
// ascending.  Runs the device radix select on fp32 scores (fp64 inputs are
// ranked after conversion to fp32; see DESIGN.md for the tie band).
template <typename T>
TokenSet args_top_k(std::span<const T> scores, std::size_t k) {
  if (k < 1) throw std::invalid_argument("args_top_k: k must be >= 1");
  std::vector<float> s(scores.begin(), scores.end());
  const std::size_t n = s.size();
  if (n == 0) return {};
  DeviceBuffer d_s(n * 4), d_o(std::min(n, k) * 4);
  d_s.upload(s.data(), n * 4);
  const int64_t m = check(lyc_args_top_k(d_s.as<float>(), (int64_t)n, (int64_t)k, d_o.as<int32_t>(), nullptr));
  cuda_check(cudaDeviceSynchronize(), "args_top_k");
  std::vector<int32_t> o((std::size_t)m);
  d_o.download(o.data(), o.size() * 4);
  return TokenSet{std::vector<std::size_t>(o.begin(), o.end())};
}

// policy.hpp:57-62
inline std::size_t fraction_budget(double frac, std::size_t n) {
  return (std::size_t)lyc_fraction_budget(frac, (int64_t)n);
}

// policy.hpp:20-53.  All four kinds run on the device: TopK and Ratio in the
// persistent step kernel, TopP and Threshold (data-dependent set sizes) with
// per-layer kernels (csrc/policy.cu).
struct SparsityPolicy {
  enum class Kind { TopK, TopP, Threshold, Ratio };
  Kind kind = Kind::TopK;
  std::size_t k = 0;
  double value = 0.0;

  static SparsityPolicy top_k(std::size_t k) {
    if (k < 1) throw std::invalid_argument("top_k: k must be >= 1");
    return {Kind::TopK, k, 0.0};
  }
  static SparsityPolicy ratio(double theta) {
    if (!(theta > 0.0 && theta < 1.0)) throw std::invalid_argument("ratio: theta must lie in (0,1)");
    return {Kind::Ratio, 0, theta};
  }
  static SparsityPolicy top_p(double p) {
    if (!(p > 0.0 && p <= 1.0)) throw std::invalid_argument("top_p: p must lie in (0,1]");
    return {Kind::TopP, 0, p};
  }
  static SparsityPolicy threshold(double tau) {
    if (!(tau > 0.0)) throw std::invalid_argument("threshold: tau must be positive");
    return {Kind::Threshold, 0, tau};
  }
};

enum class Dtype { F32 = LYC_DTYPE_F32, BF16 = LYC_DTYPE_BF16 };
enum class Select { Tokens = LYC_SELECT_TOKENS, Blocks = LYC_SELECT_BLOCKS, None = LYC_SELECT_NONE };

// The toy model's decode operations around the attention (toy_model.hpp:218-274)
// on device buffers through lyc_gemv: weights bf16 [out][in] (the transpose of
// the reference's Matrix<float> [in][out]: the same sums, coalesced per output
// row), the residual stream x fp32 [d_model].  Each call is one launch.
namespace model {

inline lyc_gemv_desc gemv_desc(const void* w, int64_t M, int64_t K, int32_t mode) {
  lyc_gemv_desc g{};
  g.w = w;
  g.M = M;
  g.K = K;
  g.mode = mode;
  return g;
}

// compute_qkv (toy_model.hpp:218-241): h = rmsnorm(x, attn_norm); q = W_q h,
// k = W_k h, v = W_v h (W_qkv = [W_q; W_k; W_v]); rotary on q and k; q -> q_out
// bf16 [nq][d]; the K / V rows of every KV head g -> row `pos` of
// k_cache / v_cache + g * slab_stride (the layer's [H][S_cap][d] slabs, bf16).
inline void compute_qkv(const void* w_qkv, int64_t d_model, const float* x, const float* attn_norm,
                        int nq, int nkv, int d, int64_t pos, void* q_out, void* k_cache,
                        void* v_cache, int64_t slab_stride, void* stream = nullptr) {
  lyc_gemv_desc g = gemv_desc(w_qkv, (int64_t)(nq + 2 * nkv) * d, d_model, LYC_GEMV_QKV_ROPE);
  g.x = x;
  g.gain = attn_norm;
  g.nq = nq;
  g.nkv = nkv;
  g.d = d;
  g.pos = pos;
  g.q_out = q_out;
  g.k_cache = k_cache;
  g.v_cache = v_cache;
  g.slab_stride = slab_stride;
  check(lyc_gemv(&g, stream));
}

// attn_project_residual (toy_model.hpp:243-255): x += W_o concat(head_outputs)
// (head outputs bf16 [Hq * d], the attention's output layout).
inline void attn_project_residual(const void* w_o, int64_t d_model, const void* head_outputs,
                                  int64_t hq_d, float* x, void* stream = nullptr) {
  lyc_gemv_desc g = gemv_desc(w_o, d_model, hq_d, LYC_GEMV_RESIDUAL);
  g.xb = head_outputs;
  g.y = x;
  check(lyc_gemv(&g, stream));
}

// ffn_residual (toy_model.hpp:257-267): x += W_2 silu(W_1 rmsnorm(x, ffn_norm)),
// two launches; mid bf16 [d_ff] holds silu(W_1 h) between them.
inline void ffn_residual(const void* w1, const void* w2, int64_t d_model, int64_t d_ff,
                         const float* ffn_norm, float* x, void* mid, void* stream = nullptr) {
  lyc_gemv_desc g1 = gemv_desc(w1, d_ff, d_model, LYC_GEMV_SILU_BF16);
  g1.x = x;
  g1.gain = ffn_norm;
  g1.yb = mid;
  check(lyc_gemv(&g1, stream));
  lyc_gemv_desc g2 = gemv_desc(w2, d_model, d_ff, LYC_GEMV_RESIDUAL);
  g2.xb = mid;
  g2.y = x;
  check(lyc_gemv(&g2, stream));
}

// output_logits (toy_model.hpp:269-274): logits = W_lm rmsnorm(x, final_norm).
inline void output_logits(const void* w_lm, int64_t vocab, int64_t d_model, const float* x,
                          const float* final_norm, float* logits, void* stream = nullptr) {
  lyc_gemv_desc g = gemv_desc(w_lm, vocab, d_model, LYC_GEMV_STORE);
  g.x = x;
  g.gain = final_norm;
  g.y = logits;
  check(lyc_gemv(&g, stream));
}

}  // namespace model

// Device KV cache write path (kv_cache.hpp:14-69) over caller-owned device
// caches in the decoder layout [n_layers][B][H][seq_cap][d]: append writes one
// row per (b, g) of a layer at length() (KvCache::append, 23-29), commit_row
// advances the shared length (32), overwrite rewrites rows below it (34-42;
// n_rows > 1 for the cache-correction window).  Rows are [B][H][n_rows][d] in
// the cache dtype.
class KvCache {
 public:
  KvCache(int n_layers, int batch, int n_kv_heads, int d_head, std::size_t seq_cap, Dtype dtype,
          void* k_cache, void* v_cache)
      : k_(k_cache), v_(v_cache) {
    lay_.n_layers = n_layers;
    lay_.batch = batch;
    lay_.n_kv_heads = n_kv_heads;
    lay_.d_head = d_head;
    lay_.dtype = (int32_t)dtype;
    lay_.pad = 0;
    lay_.seq_cap = (int64_t)seq_cap;
  }
  std::size_t length() const { return length_; }
  void append(int layer, const void* k_rows, const void* v_rows, void* stream = nullptr) {
    check(lyc_kv_write(k_, v_, &lay_, layer, (int64_t)length_, 1, k_rows, v_rows, stream));
  }
  void commit_row() { ++length_; }
  void overwrite(int layer, std::size_t pos, std::size_t n_rows, const void* k_rows,
                 const void* v_rows, void* stream = nullptr) {
    if (pos + n_rows > length_) throw std::invalid_argument("KvCache: overwrite beyond the committed length");
    check(lyc_kv_write(k_, v_, &lay_, layer, (int64_t)pos, (int64_t)n_rows, k_rows, v_rows, stream));
  }

 private:
  void* k_;
  void* v_;
  lyc_kv_layout lay_{};
  std::size_t length_ = 0;
};

// The decode-step attention loop of DecodeEngine (decode_engine.hpp:109-151)
// over device-resident caches: per layer, retrieval heads (layer 0, or role
// Retrieval in the role map; rolemap.hpp:33-35) run dense split-KV attention
// and refresh the per-KV-head index cache from the pooled-query scores
// (decode_engine.hpp:129-132); sparse heads attend to the set of the nearest
// earlier retrieval layer of the same head index (:133-143).  Device layouts:
//   q, out [n_layers][B][Hq][d]     k, v [n_layers][B][H][seq_cap][d]
class HybridDecoder {
 public:
  struct Config {
    int n_layers = 1, batch = 1, n_kv_heads = 1, group_size = 1, d_head = 64;
    Dtype dtype = Dtype::BF16;
    std::size_t seq_cap = 0;
    SparsityPolicy policy = SparsityPolicy::top_k(1);
    Select select = Select::Tokens;
    int num_splits = 0;  // 0: one CTA per SM
    float scale = 0.f;   // 0: 1/sqrt(d_head)
  };

  // roles: [n_layers][n_kv_heads], 0 = Retrieval, 1 = Sparse (RoleMap::role)
  HybridDecoder(const Config& c, std::span<const std::uint8_t> roles) : cfg_(c) {
    if (roles.size() != (std::size_t)c.n_layers * c.n_kv_heads)
      throw std::invalid_argument("RoleMap: role count mismatch");
    lyc_decode_config lc{};
    lc.n_layers = c.n_layers;
    lc.batch = c.batch;
    lc.n_kv_heads = c.n_kv_heads;
    lc.group_size = c.group_size;
    lc.d_head = c.d_head;
    lc.dtype = (int32_t)c.dtype;
    lc.seq_cap = (int64_t)c.seq_cap;
    switch (c.policy.kind) {
      case SparsityPolicy::Kind::TopK: lc.policy_kind = LYC_POLICY_TOPK; break;
      case SparsityPolicy::Kind::TopP: lc.policy_kind = LYC_POLICY_TOPP; break;
      case SparsityPolicy::Kind::Threshold: lc.policy_kind = LYC_POLICY_THRESHOLD; break;
      case SparsityPolicy::Kind::Ratio: lc.policy_kind = LYC_POLICY_RATIO; break;
    }
    lc.select_mode = (int32_t)c.select;
    lc.top_k = (int64_t)c.policy.k;
    lc.ratio = c.policy.value;
    lc.block_size = 64;
    lc.num_splits = c.num_splits;
    lc.scale = c.scale;
    lc.roles = roles.data();
    check(lyc_decoder_create(&lc, &d_));
  }
  ~HybridDecoder() {
    if (d_) lyc_decoder_destroy(d_);
  }
  HybridDecoder(const HybridDecoder&) = delete;
  HybridDecoder& operator=(const HybridDecoder&) = delete;

  // One decode step over all layers (seq_len = t + 1, the current token's
  // K/V row already appended).  Stream ordered.
  void decode_step(const void* q, const void* k, const void* v, std::size_t seq_len, void* out,
                   cudaStream_t st = nullptr) {
    check(lyc_decoder_step(d_, q, k, v, (int64_t)seq_len, out, st));
  }
  // A variable-length batch: seq_lens[b] for batch item b (B independent
  // sequences; lyc_decoder_step_varlen).
  void decode_step(const void* q, const void* k, const void* v, const std::vector<std::size_t>& seq_lens,
                   void* out, cudaStream_t st = nullptr) {
    check(lyc_decoder_step_varlen(d_, q, k, v, lens_of(seq_lens).data(), out, st));
  }
  // One layer (layers issued in order within a step).
  void decode_layer(int layer, const void* q_l, const void* k, const void* v, std::size_t seq_len,
                    void* out_l, cudaStream_t st = nullptr) {
    check(lyc_decoder_layer(d_, layer, q_l, k, v, (int64_t)seq_len, out_l, st));
  }
  // cache_correction's set refresh (decode_engine.hpp:190-197): every KV head's
  // set re-selected from the last window position's pooled query at `layer`.
  void refresh_sets(int layer, const void* q_last, const void* k, std::size_t len,
                    cudaStream_t st = nullptr) {
    check(lyc_decoder_refresh_sets(d_, layer, q_last, k, (int64_t)len, st));
  }
  // CUDA-graph capture of decode_step for fixed pointers / seq_len, then replay.
  void capture(const void* q, const void* k, const void* v, std::size_t seq_len, void* out,
               cudaStream_t st) {
    check(lyc_decoder_capture(d_, q, k, v, (int64_t)seq_len, out, st));
  }
  // The same for a variable-length batch (one length per batch item).
  void capture(const void* q, const void* k, const void* v, const std::vector<std::size_t>& seq_lens,
               void* out, cudaStream_t st) {
    check(lyc_decoder_capture_varlen(d_, q, k, v, lens_of(seq_lens).data(), out, st));
  }
  void replay(cudaStream_t st) { check(lyc_decoder_replay(d_, st)); }

  // DecodeEngine::token_sets(): the per-(b, KV head) index cache, ascending
  // (token ids, or block ids in Select::Blocks).  Synchronises.
  std::vector<std::vector<std::int32_t>> token_sets() const {
    int32_t *ids = nullptr, *counts = nullptr;
    int64_t kcap = 0;
    check(lyc_decoder_index_cache(d_, &ids, &counts, &kcap));
    cuda_check(cudaDeviceSynchronize(), "sync");
    check(lyc_decoder_sync_sets(d_, nullptr));  // a selection deferred by decode_layer
    cuda_check(cudaDeviceSynchronize(), "sync");
    const std::size_t rows = (std::size_t)cfg_.batch * cfg_.n_kv_heads;
    std::vector<int32_t> n(rows), all(rows * (std::size_t)kcap);
    cuda_check(cudaMemcpy(n.data(), counts, rows * 4, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(all.data(), ids, all.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    std::vector<std::vector<int32_t>> sets(rows);
    for (std::size_t r = 0; r < rows; ++r)
      sets[r].assign(all.begin() + r * kcap, all.begin() + r * kcap + n[r]);
    return sets;
  }

  bool fused() const { return lyc_decoder_is_fused(d_) != 0; }
  int64_t launches_per_step(std::size_t seq_len) { return lyc_decoder_launches_per_step(d_, (int64_t)seq_len); }
  int64_t step_bytes(std::size_t seq_len) { return lyc_decoder_step_bytes(d_, (int64_t)seq_len); }
  lyc_decoder* handle() const { return d_; }

 private:
  std::vector<int64_t> lens_of(const std::vector<std::size_t>& seq_lens) const {
    if (seq_lens.size() != (std::size_t)cfg_.batch)
      throw std::invalid_argument("decode_step: one seq_len per batch item");
    return std::vector<int64_t>(seq_lens.begin(), seq_lens.end());
  }

  Config cfg_;
  lyc_decoder* d_ = nullptr;
};

// KV-sequence sharding across GPUs (lyc_shard_layer / lyc_shard_merge): this
// rank holds rows [row_begin, row_begin + n_local) of every head's cache.
// Per layer: local partials + local top-k candidates into this rank's packed
// block, the caller's all-gather of every rank's block (rank order; e.g. one
// ncclAllGather), then the identical rank-ordered merge + global top-k.
class ShardedDecoder {
 public:
  // exchange(send, recv, words): gather `words` 4-byte words from every rank
  // into recv[rank * words ...] (device pointers, stream ordered)
  using Exchange = std::function<void(const float* send, float* recv, std::size_t words)>;

  ShardedDecoder(const HybridDecoder::Config& c, std::span<const std::uint8_t> roles, int world,
                 int rank, Exchange exchange)
      : dec_(c, roles), cfg_(c), world_(world), rank_(rank), exchange_(std::move(exchange)) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("shard: bad world/rank");
    int32_t *ids = nullptr, *counts = nullptr;
    check(lyc_decoder_index_cache(dec_.handle(), &ids, &counts, &k_cap_));
    rows_ = (std::size_t)c.batch * c.n_kv_heads * c.group_size;
    bh_ = (std::size_t)c.batch * c.n_kv_heads;
    off_lse_ = rows_ * c.d_head;
    off_key_ = off_lse_ + rows_;
    off_idx_ = off_key_ + bh_ * (std::size_t)k_cap_;
    words_ = (off_idx_ + bh_ * (std::size_t)k_cap_ + 3) / 4 * 4;
    send_ = DeviceBuffer(words_ * 4);
    recv_ = DeviceBuffer(words_ * 4 * (std::size_t)world);
  }

  // Step 1 of a layer: this rank's partials + local top-k candidates into its
  // packed send block (send(), block_words() 4-byte words).
  void layer_local(int l, const void* q_l, const void* k, const void* v, std::size_t n_local,
                   std::size_t row_begin, cudaStream_t st = nullptr) {
    float* sb = send_.as<float>();
    check(lyc_shard_layer(dec_.handle(), l, q_l, k, v, (int64_t)n_local, (int64_t)row_begin, sb,
                          sb + off_lse_, reinterpret_cast<uint32_t*>(sb + off_key_),
                          reinterpret_cast<int32_t*>(sb + off_idx_), st));
  }
  // Step 3 of a layer (after the all-gather of every rank's block into
  // `gathered`, rank order): identical on every rank.
  void layer_combine(int l, const float* gathered, std::size_t n_local, std::size_t row_begin,
                     std::size_t seq_total, void* out_l, int32_t* global_sets = nullptr,
                     cudaStream_t st = nullptr) {
    check(lyc_shard_merge(dec_.handle(), l, world_, gathered, gathered + off_lse_,
                          reinterpret_cast<const uint32_t*>(gathered + off_key_),
                          reinterpret_cast<const int32_t*>(gathered + off_idx_), (int64_t)words_,
                          (int64_t)n_local, (int64_t)row_begin, (int64_t)seq_total, out_l,
                          global_sets, st));
  }

  // One decode step: q/out [L][B][Hq][d] (identical q on every rank), k/v this
  // rank's [L][B][H][seq_cap][d] with local row 0 = global row row_begin.
  void decode_step(const void* q, const void* k, const void* v, std::size_t n_local,
                   std::size_t row_begin, std::size_t seq_total, void* out, cudaStream_t st = nullptr) {
    const std::size_t esz = cfg_.dtype == Dtype::BF16 ? 2 : 4;
    const std::size_t qstride = rows_ * cfg_.d_head * esz;
    for (int l = 0; l < cfg_.n_layers; ++l) {
      layer_local(l, static_cast<const char*>(q) + l * qstride, k, v, n_local, row_begin, st);
      exchange_(send_.as<float>(), recv_.as<float>(), words_);
      layer_combine(l, recv_.as<float>(), n_local, row_begin, seq_total,
                    static_cast<char*>(out) + l * qstride, nullptr, st);
    }
  }

  const float* send() const { return send_.as<float>(); }
  HybridDecoder& local() { return dec_; }
  std::size_t block_words() const { return words_; }

 private:
  HybridDecoder dec_;
  HybridDecoder::Config cfg_;
  int world_, rank_;
  Exchange exchange_;
  int64_t k_cap_ = 0;
  std::size_t rows_ = 0, bh_ = 0, off_lse_ = 0, off_key_ = 0, off_idx_ = 0, words_ = 0;
  DeviceBuffer send_, recv_;
};

}  // namespace lyc

#endif  // LYC_HPP_
