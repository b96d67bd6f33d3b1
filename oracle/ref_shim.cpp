// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference headers, compiled in place
// from /root/reference/proj/include (never copied) by oracle/Makefile into
// oracle/_ref/libhh_ref.so.  It exposes the reference's own implementation
// of the hot path with the same C signatures as oracle/hh_oracle.c (prefix
// ref_ instead of orc_), so tests can pin the C restatement against the real
// reference and bench.py can time the reference CPU path (kind "reference").
//
// Exceptions map to codes: std::invalid_argument -> -1, std::logic_error -> -2.
#include <cstdint>
#include <chrono>
#include <cstring>
#include <optional>
#include <numeric>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "hh/rng.hpp"  // kernel_sim.hpp does not include it itself
#include "hh/attention.hpp"
#include "hh/kernel_sim.hpp"
#include "hh/policy.hpp"

namespace {

template <typename F>
int64_t guard(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::logic_error&) {
    return -2;
  }
}

template <typename T>
hh::kernel::Workload<T> make_workload(int64_t batch, int64_t n_kv, int64_t group, int64_t d,
                                      int64_t seq_len, int64_t block_size, T scale, const T* K,
                                      const T* V, const T* Q, const int64_t* blk_off,
                                      const int64_t* blk_ids) {
  hh::kernel::Workload<T> w;
  w.batch = batch;
  w.n_kv_heads = n_kv;
  w.group_size = group;
  w.d_head = d;
  w.seq_len = seq_len;
  w.block_size = block_size;
  w.scale = scale;
  w.keys.resize(batch * n_kv);
  w.values.resize(batch * n_kv);
  for (int64_t s = 0; s < batch * n_kv; ++s) {
    w.keys[s] = hh::Matrix<T>(seq_len, d);
    w.values[s] = hh::Matrix<T>(seq_len, d);
    std::memcpy(w.keys[s].data.data(), K + s * seq_len * d, sizeof(T) * seq_len * d);
    std::memcpy(w.values[s].data.data(), V + s * seq_len * d, sizeof(T) * seq_len * d);
  }
  const int64_t hq = n_kv * group;
  w.queries.resize(batch * hq);
  for (int64_t h = 0; h < batch * hq; ++h) w.queries[h].assign(Q + h * d, Q + (h + 1) * d);
  w.blocks.batch = batch;
  w.blocks.n_kv_heads = n_kv;
  w.blocks.ids.resize(batch * n_kv);
  for (int64_t s = 0; s < batch * n_kv; ++s)
    for (int64_t i = blk_off[s]; i < blk_off[s + 1]; ++i)
      w.blocks.ids[s].push_back(static_cast<std::uint32_t>(blk_ids[i]));
  return w;
}

}  // namespace

extern "C" {

int ref_dense_attention_f64(const double* q, const double* K, const double* V, int64_t n,
                            int64_t d, double scale, double* out, double* weights) {
  return (int)guard([&]() -> int64_t {
    hh::AttnInput<double> in{std::span<const double>(q, d), hh::MatView<double>(K, n, d),
                             hh::MatView<double>(V, n, d), scale};
    auto r = hh::dense_attention(in);
    std::memcpy(out, r.out.data(), sizeof(double) * d);
    if (weights) std::memcpy(weights, r.weights.data(), sizeof(double) * n);
    return 0;
  });
}

int ref_sparse_attention_f64(const double* q, const double* K, const double* V, int64_t n,
                             int64_t d, double scale, const int64_t* idx, int64_t k,
                             double* out) {
  return (int)guard([&]() -> int64_t {
    hh::AttnInput<double> in{std::span<const double>(q, d), hh::MatView<double>(K, n, d),
                             hh::MatView<double>(V, n, d), scale};
    hh::TokenSet s;
    s.indices.assign(idx, idx + k);
    auto r = hh::sparse_attention(in, s);
    std::memcpy(out, r.data(), sizeof(double) * d);
    return 0;
  });
}

int64_t ref_args_top_k_f64(const double* w, int64_t n, int64_t k, int64_t* out) {
  return guard([&]() -> int64_t {
    auto s = hh::args_top_k<double>(std::span<const double>(w, n), k);
    for (std::size_t i = 0; i < s.size(); ++i) out[i] = (int64_t)s.indices[i];
    return (int64_t)s.size();
  });
}

int64_t ref_args_top_k_f32(const float* w, int64_t n, int64_t k, int64_t* out) {
  return guard([&]() -> int64_t {
    auto s = hh::args_top_k<float>(std::span<const float>(w, n), k);
    for (std::size_t i = 0; i < s.size(); ++i) out[i] = (int64_t)s.indices[i];
    return (int64_t)s.size();
  });
}

int ref_gqa_pool_queries_f64(const double* q, int64_t n_heads, int64_t d, int64_t group,
                             double* out) {
  return (int)guard([&]() -> int64_t {
    std::vector<std::vector<double>> qs(n_heads);
    for (int64_t h = 0; h < n_heads; ++h) qs[h].assign(q + h * d, q + (h + 1) * d);
    auto p = hh::gqa_pool_queries(qs, group);
    for (std::size_t g = 0; g < p.size(); ++g)
      std::memcpy(out + g * d, p[g].data(), sizeof(double) * d);
    return 0;
  });
}

int64_t ref_fraction_budget(double frac, int64_t n) { return (int64_t)hh::fraction_budget(frac, n); }

int64_t ref_select_tokens(int kind, int64_t k, double value, const double* w, int64_t n,
                          int64_t* out) {
  return guard([&]() -> int64_t {
    hh::SparsityPolicy p;
    switch (kind) {
      case 0: p = hh::SparsityPolicy::top_k(k); break;
      case 1: p = hh::SparsityPolicy::top_p(value); break;
      case 2: p = hh::SparsityPolicy::threshold(value); break;
      case 3: p = hh::SparsityPolicy::ratio(value); break;
      default: throw std::invalid_argument("kind");
    }
    auto s = hh::select_tokens(p, std::span<const double>(w, n), n);
    for (std::size_t i = 0; i < s.size(); ++i) out[i] = (int64_t)s.indices[i];
    return (int64_t)s.size();
  });
}

int64_t ref_plan_splits(int64_t batch, int64_t n_kv, const int64_t* head_blocks,
                        int64_t num_splits, int64_t* split_blocks, int64_t* head_split_count,
                        int64_t* units, int64_t max_units) {
  return guard([&]() -> int64_t {
    hh::kernel::BlockIndexSet b;
    b.batch = batch;
    b.n_kv_heads = n_kv;
    b.ids.resize(batch * n_kv);
    for (int64_t s = 0; s < batch * n_kv; ++s) {
      b.ids[s].resize(head_blocks[s]);
      std::iota(b.ids[s].begin(), b.ids[s].end(), 0u);
    }
    auto sched = hh::kernel::plan_splits(b, num_splits);
    int64_t nu = 0;
    for (int64_t bi = 0; bi < batch; ++bi) {
      for (int64_t s = 0; s < num_splits; ++s) {
        split_blocks[bi * num_splits + s] = sched.split_blocks[bi][s];
        for (const auto& u : sched.units[bi][s]) {
          if (nu < max_units) {
            int64_t* r = units + nu * 6;
            r[0] = bi; r[1] = s; r[2] = u.kv_head; r[3] = u.begin; r[4] = u.end;
            r[5] = u.head_local_split;
          }
          ++nu;
        }
      }
      for (int64_t g = 0; g < n_kv; ++g)
        head_split_count[bi * n_kv + g] = sched.head_split_count[bi][g];
    }
    return nu;
  });
}

#define REF_RUN(T, SFX)                                                                      \
  int ref_kernel_run_##SFX(int64_t batch, int64_t n_kv, int64_t group, int64_t d,            \
                           int64_t seq_len, int64_t block_size, T scale, const T* K,         \
                           const T* V, const T* Q, const int64_t* blk_off,                   \
                           const int64_t* blk_ids, int64_t num_splits, T* out,               \
                           int64_t* exec_counts, int64_t n_workers) {                        \
    return (int)guard([&]() -> int64_t {                                                     \
      auto w = make_workload<T>(batch, n_kv, group, d, seq_len, block_size, scale, K, V, Q,  \
                                blk_off, blk_ids);                                           \
      auto r = hh::kernel::run(w, num_splits, n_workers < 1 ? 1 : n_workers);                \
      for (std::size_t h = 0; h < r.outputs.size(); ++h)                                     \
        std::memcpy(out + h * d, r.outputs[h].data(), sizeof(T) * d);                        \
      if (exec_counts) {                                                                     \
        /* reference flattens counts in (b, g, list index) order (:267-275); scatter to */   \
        /* the [b][g][nb] grid used by the C restatement.                               */   \
        const int64_t nb = (seq_len + block_size - 1) / block_size;                          \
        std::size_t c = 0;                                                                   \
        for (int64_t i = 0; i < batch * n_kv * nb; ++i) exec_counts[i] = 0;                  \
        for (int64_t s = 0; s < batch * n_kv; ++s)                                           \
          for (int64_t i = 0; i < blk_off[s + 1] - blk_off[s]; ++i)                          \
            exec_counts[s * nb + i] = r.block_exec_counts[c++];                              \
      }                                                                                      \
      return 0;                                                                              \
    });                                                                                      \
  }
REF_RUN(float, f32)
REF_RUN(double, f64)

// Time-only entry for the CPU baseline: builds the Workload once from
// caller-owned buffers, then runs hh::kernel::run `reps` times and returns the
// best wall time in seconds through *best_s.
#define REF_TIME(T, SFX)                                                                     \
  int ref_kernel_run_time_##SFX(int64_t batch, int64_t n_kv, int64_t group, int64_t d,       \
                                int64_t seq_len, int64_t block_size, T scale, const T* K,    \
                                const T* V, const T* Q, const int64_t* blk_off,              \
                                const int64_t* blk_ids, int64_t num_splits, int64_t n_workers,\
                                int64_t reps, T* out, double* best_s) {                      \
    return (int)guard([&]() -> int64_t {                                                     \
      auto w = make_workload<T>(batch, n_kv, group, d, seq_len, block_size, scale, K, V, Q,  \
                                blk_off, blk_ids);                                           \
      double best = 1e30;                                                                    \
      for (int64_t r = 0; r < reps; ++r) {                                                   \
        auto t0 = std::chrono::steady_clock::now();                                          \
        auto res = hh::kernel::run(w, num_splits, n_workers < 1 ? 1 : n_workers);            \
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)     \
                        .count();                                                            \
        if (dt < best) best = dt;                                                            \
        if (r == 0 && out)                                                                   \
          for (std::size_t h = 0; h < res.outputs.size(); ++h)                               \
            std::memcpy(out + h * d, res.outputs[h].data(), sizeof(T) * d);                  \
      }                                                                                      \
      *best_s = best;                                                                        \
      return 0;                                                                              \
    });                                                                                      \
  }
REF_TIME(float, f32)

int ref_latency_model(int64_t batch, int64_t n_kv, const int64_t* head_blocks, int64_t num_splits,
                      int64_t bytes_per_block, int64_t* out, double* dout) {
  return (int)guard([&]() -> int64_t {
    hh::kernel::BlockIndexSet b;
    b.batch = batch;
    b.n_kv_heads = n_kv;
    b.ids.resize(batch * n_kv);
    for (int64_t s = 0; s < batch * n_kv; ++s) {
      b.ids[s].resize(head_blocks[s]);
      std::iota(b.ids[s].begin(), b.ids[s].end(), 0u);
    }
    auto c = hh::kernel::latency_model(hh::kernel::plan_splits(b, num_splits), bytes_per_block);
    out[0] = c.total_blocks; out[1] = c.pooled_critical_blocks; out[2] = c.naive_critical_blocks;
    out[3] = c.bytes_per_block; out[4] = c.pooled_critical_bytes; out[5] = c.naive_critical_bytes;
    dout[0] = c.mean_split_blocks;
    dout[1] = c.balance_ratio;
    return 0;
  });
}

// decode_engine.hpp:109-151 attention loop over synthetic q/K/V, calling the
// reference primitives unchanged (dense_attention, gqa_pool_queries,
// select_tokens, sparse_attention).  Same signature as orc_decode_step_f64.
int ref_decode_step_f64(int64_t n_layers, int64_t n_kv, int64_t group, int64_t d, int64_t seq,
                        int64_t seq_cap, double scale, const double* q, const double* K,
                        const double* V, const uint8_t* roles, int kind, int64_t k, double value,
                        int64_t* sets, int64_t* set_len, int64_t set_cap, double* out,
                        int64_t* trace_sets, int64_t* trace_len) {
  return (int)guard([&]() -> int64_t {
    hh::SparsityPolicy p;
    switch (kind) {
      case 0: p = hh::SparsityPolicy::top_k(k); break;
      case 1: p = hh::SparsityPolicy::top_p(value); break;
      case 2: p = hh::SparsityPolicy::threshold(value); break;
      case 3: p = hh::SparsityPolicy::ratio(value); break;
      default: throw std::invalid_argument("kind");
    }
    const int64_t hq = n_kv * group;
    std::vector<hh::TokenSet> sets_(n_kv);
    for (int64_t g = 0; g < n_kv; ++g)
      sets_[g].indices.assign(sets + g * set_cap, sets + g * set_cap + set_len[g]);
    for (int64_t l = 0; l < n_layers; ++l) {
      std::vector<std::vector<double>> qh(hq);
      for (int64_t h = 0; h < hq; ++h)
        qh[h].assign(q + (l * hq + h) * d, q + (l * hq + h + 1) * d);
      std::optional<std::vector<std::vector<double>>> pooled;
      for (int64_t g = 0; g < n_kv; ++g) {
        const double* Kg = K + (l * n_kv + g) * seq_cap * d;
        const double* Vg = V + (l * n_kv + g) * seq_cap * d;
        hh::MatView<double> kv(Kg, seq, d), vv(Vg, seq, d);
        const bool retrieval = l == 0 || roles[l * n_kv + g] == 0;
        if (retrieval) {
          for (int64_t j = 0; j < group; ++j) {
            const int64_t hd = g * group + j;
            hh::AttnInput<double> in{qh[hd], kv, vv, scale};
            auto o = hh::dense_attention(in).out;
            std::memcpy(out + (l * hq + hd) * d, o.data(), sizeof(double) * d);
          }
          if (!pooled) pooled = hh::gqa_pool_queries(qh, group);
          hh::AttnInput<double> sel{(*pooled)[g], kv, vv, scale};
          sets_[g] = hh::select_tokens(p, hh::dense_attention(sel).weights, seq);
        } else {
          const hh::TokenSet& s = sets_[g];
          if (s.empty()) throw std::logic_error("decode_step: sparse head with empty token set");
          for (int64_t j = 0; j < group; ++j) {
            const int64_t hd = g * group + j;
            hh::AttnInput<double> in{qh[hd], kv, vv, scale};
            auto o = hh::sparse_attention(in, s);
            std::memcpy(out + (l * hq + hd) * d, o.data(), sizeof(double) * d);
          }
        }
        if (trace_sets) {
          for (std::size_t i = 0; i < sets_[g].size(); ++i)
            trace_sets[(l * n_kv + g) * set_cap + i] = (int64_t)sets_[g].indices[i];
          trace_len[l * n_kv + g] = (int64_t)sets_[g].size();
        }
      }
    }
    for (int64_t g = 0; g < n_kv; ++g) {
      if ((int64_t)sets_[g].size() > set_cap) throw std::invalid_argument("set_cap");
      for (std::size_t i = 0; i < sets_[g].size(); ++i) sets[g * set_cap + i] = (int64_t)sets_[g].indices[i];
      set_len[g] = (int64_t)sets_[g].size();
    }
    return 0;
  });
}

// ---------------------------------------------------------------------------
// Timed CPU decode step for bench.py's reference arm (BASELINE metric, whole
// step, every layer executed).  Per layer, as the reference does it:
//   * the layer's attention through the reference's own multi-threaded
//     operator hh::kernel::run<float> (kernel_sim.hpp:237-279): retrieval heads
//     list every block, sparse heads a ceil(k/64)-block subset -- the
//     BlockIndexSet form of their k-token sets (same rows touched);
//   * the selection pass of every retrieval head (decode_engine.hpp:129-132):
//     gqa_pool_queries, dense_attention<double> weights over the head's seq
//     rows, select_tokens(TopK) -- serial f64, as DecodeEngine runs it.
// One Workload (K/V of H heads, batch 1) is built once and reused for every
// layer (CPU time does not depend on the values); only the block lists
// change per layer.  The f64 selection pass reuses one head's upcast K/V.
struct RefStepCtx {
  hh::kernel::Workload<float> w;
  std::vector<double> k64, v64;
  int64_t H = 0, G = 0, d = 0, L = 0;
  float scale = 1.f;
};

void* ref_step_ctx_create(int64_t n_kv, int64_t group, int64_t d, int64_t seq, float scale,
                          const float* K, const float* V, const float* Q) {
  auto* c = new RefStepCtx();
  const int64_t off0 = 0;
  std::vector<int64_t> off(n_kv + 1, 0);
  c->w = make_workload<float>(1, n_kv, group, d, seq, 64, scale, K, V, Q, off.data(), &off0);
  c->H = n_kv;
  c->G = group;
  c->d = d;
  c->L = seq;
  c->scale = scale;
  c->k64.assign(K, K + seq * d);
  c->v64.assign(V, V + seq * d);
  return c;
}

void ref_step_ctx_destroy(void* ctx) { delete static_cast<RefStepCtx*>(ctx); }

// roles [n_layers][H] (0 = Retrieval); blocks: per layer per head CSR
// (blk_off [n_layers][H + 1] offsets into blk_ids).  Returns seconds of the
// step in *seconds and the attention / selection parts in parts[2].
int ref_step_run(void* ctx, int64_t n_layers, const uint8_t* roles, const int64_t* blk_off,
                 const int64_t* blk_ids, int64_t num_splits, int64_t n_workers, int64_t top_k,
                 double* seconds, double* parts) {
  return (int)guard([&]() -> int64_t {
    auto* c = static_cast<RefStepCtx*>(ctx);
    const auto clk = [] { return std::chrono::steady_clock::now(); };
    double t_attn = 0, t_sel = 0;
    const auto t0 = clk();
    for (int64_t l = 0; l < n_layers; ++l) {
      const int64_t* off = blk_off + l * (c->H + 1);
      for (int64_t g = 0; g < c->H; ++g) {
        auto& ids = c->w.blocks.ids[g];
        ids.clear();
        for (int64_t i = off[g]; i < off[g + 1]; ++i) ids.push_back((std::uint32_t)blk_ids[i]);
      }
      const auto ta = clk();
      auto res = hh::kernel::run(c->w, num_splits, n_workers < 1 ? 1 : n_workers);
      const auto tb = clk();
      t_attn += std::chrono::duration<double>(tb - ta).count();
      std::vector<std::vector<double>> qh(c->H * c->G);
      std::optional<std::vector<std::vector<double>>> pooled;
      for (int64_t g = 0; g < c->H; ++g) {
        if (!(l == 0 || roles[l * c->H + g] == 0)) continue;
        if (!pooled) {
          for (int64_t h = 0; h < c->H * c->G; ++h)
            qh[h].assign(c->w.queries[h].begin(), c->w.queries[h].end());
          pooled = hh::gqa_pool_queries(qh, c->G);
        }
        hh::MatView<double> kv(c->k64.data(), c->L, c->d), vv(c->v64.data(), c->L, c->d);
        hh::AttnInput<double> sel{(*pooled)[g], kv, vv, (double)c->scale};
        auto set = hh::select_tokens(hh::SparsityPolicy::top_k(top_k),
                                     hh::dense_attention(sel).weights, c->L);
        if (set.empty()) throw std::logic_error("empty selection");
      }
      t_sel += std::chrono::duration<double>(clk() - tb).count();
      if (res.outputs.empty()) throw std::logic_error("no outputs");
    }
    *seconds = std::chrono::duration<double>(clk() - t0).count();
    parts[0] = t_attn;
    parts[1] = t_sel;
    return 0;
  });
}

}  // extern "C"
