// test_dropin.cpp -- TEST INFRASTRUCTURE (links the reference as the checker).
//
// The drop-in demonstration: the reference's own types and CPU operator
// (hh::kernel::Workload / run / plan_splits / latency_model, hh::args_top_k;
// the UNMODIFIED headers, compiled in place from $(HH_REF_INCLUDE)) side by
// side with lyc:: on the SAME hh:: objects.  Reference call site
//     auto r = hh::kernel::run(w, splits, workers);
// becomes
//     auto r = lyc::kernel::run_as<hh::kernel::RunResult<float>>(w, splits);
// Built by tests/cpp/Makefile into oracle/_ref/ only where the reference is
// present (this container); the binary travels to the GPU box.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "hh/rng.hpp"  // kernel_sim.hpp does not include it itself
#include "hh/attention.hpp"
#include "hh/kernel_sim.hpp"
#include "lyc.hpp"

static int g_fail = 0;
#define CHECK(c)                                                             \
  do {                                                                       \
    if (!(c)) {                                                              \
      ++g_fail;                                                              \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);             \
    }                                                                        \
  } while (0)

static hh::kernel::Workload<float> make(std::mt19937_64& rng, int B, int H, int G, int d, int L) {
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  hh::kernel::Workload<float> w;
  w.batch = B;
  w.n_kv_heads = H;
  w.group_size = G;
  w.d_head = d;
  w.seq_len = L;
  w.block_size = 64;
  w.scale = 1.f / std::sqrt((float)d);
  for (int i = 0; i < B * H; ++i) {
    hh::Matrix<float> k(L, d), v(L, d);
    for (auto& x : k.data) x = U(rng);
    for (auto& x : v.data) x = U(rng);
    w.keys.push_back(std::move(k));
    w.values.push_back(std::move(v));
  }
  for (int h = 0; h < B * H * G; ++h) {
    std::vector<float> q(d);
    for (auto& x : q) x = U(rng);
    w.queries.push_back(std::move(q));
  }
  w.blocks.batch = B;
  w.blocks.n_kv_heads = H;
  const int nb = (L + 63) / 64;
  for (int i = 0; i < B * H; ++i) {
    std::vector<uint32_t> ids;
    for (int b = 0; b < nb; ++b)
      if (i % 3 == 0 || std::uniform_real_distribution<double>(0, 1)(rng) < 0.1) ids.push_back(b);
    if (ids.empty()) ids.push_back(nb - 1);
    w.blocks.ids.push_back(ids);
  }
  return w;
}

int main() {
  std::mt19937_64 rng(2602);
  double worst = 0;
  for (int trial = 0; trial < 8; ++trial) {
    const int B = 1 + trial % 4, H = 1 + trial % 8, G = 1 + trial % 4;
    const int L = 257 + 500 * trial;
    auto w = make(rng, B, H, G, trial % 2 ? 64 : 16, L);
    const size_t splits = 1 + trial;
    auto ref = hh::kernel::run(w, splits, 2);
    auto got = lyc::kernel::run_as<hh::kernel::RunResult<float>>(w, splits);
    CHECK(got.outputs.size() == ref.outputs.size());
    for (size_t h = 0; h < ref.outputs.size(); ++h)
      for (size_t c = 0; c < w.d_head; ++c)
        worst = std::max(worst, (double)std::abs(got.outputs[h][c] - ref.outputs[h][c]));
    CHECK(got.block_exec_counts == ref.block_exec_counts);
    CHECK(got.schedule.split_blocks == ref.schedule.split_blocks);
    CHECK(got.schedule.head_split_count == ref.schedule.head_split_count);
    for (size_t b = 0; b < w.batch; ++b)
      for (size_t s = 0; s < splits; ++s) {
        CHECK(got.schedule.units[b][s].size() == ref.schedule.units[b][s].size());
        for (size_t u = 0; u < ref.schedule.units[b][s].size(); ++u) {
          CHECK(got.schedule.units[b][s][u].kv_head == ref.schedule.units[b][s][u].kv_head);
          CHECK(got.schedule.units[b][s][u].begin == ref.schedule.units[b][s][u].begin);
          CHECK(got.schedule.units[b][s][u].end == ref.schedule.units[b][s][u].end);
          CHECK(got.schedule.units[b][s][u].head_local_split ==
                ref.schedule.units[b][s][u].head_local_split);
        }
      }
    auto cr = hh::kernel::latency_model(ref.schedule, 16384);
    auto cg = lyc::kernel::latency_model(ref.schedule, 16384);
    CHECK(cr.pooled_critical_blocks == cg.pooled_critical_blocks);
    CHECK(cr.naive_critical_blocks == cg.naive_critical_blocks);
    CHECK(cr.total_blocks == cg.total_blocks);
    CHECK(std::abs(cr.balance_ratio - cg.balance_ratio) < 1e-12);
  }
  std::printf("kernel::run  max |lyc - hh| = %.3g over 8 workloads (bar 1e-5)\n", worst);
  CHECK(worst < 1e-5);
  // args_top_k on the same scores (attention.hpp:108-123)
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  for (int n : {7, 1000, 32768, 131072}) {
    std::vector<float> s(n);
    for (auto& x : s) x = U(rng);
    for (size_t k : {1, 3, 256, 4096}) {
      auto r = hh::args_top_k<float>(std::span<const float>(s), k);
      auto g = lyc::args_top_k<float>(s, k);
      CHECK(r.indices == g.indices);
    }
  }
  // the reference's exception types come back unchanged
  auto w = make(rng, 1, 2, 2, 16, 300);
  w.blocks.ids[1] = {3, 2};
  bool ok = false;
  try {
    lyc::kernel::run_as<hh::kernel::RunResult<float>>(w, 2);
  } catch (const std::invalid_argument&) {
    ok = true;
  }
  CHECK(ok);
  std::printf("%s\n", g_fail ? "DROP-IN FAILED" : "drop-in OK: lyc::kernel::run_as == hh::kernel::run");
  return g_fail ? 1 : 0;
}
