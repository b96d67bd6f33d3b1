// test_lyc.cpp -- C++ parity tests of the drop-in host API (include/lyc.hpp)
// on the B200, written like the reference's own GTest suites
// (tests/kernel_sim_test.cpp, attention_test.cpp, decode_engine_test.cpp;
// GTest is not in this image, so a minimal CHECK harness).  The expected
// values come from plain-loop oracles in this file (the reference's
// test_util.hpp style: two-pass softmax in double), never from the library.
//
//   make -C tests/cpp && build/cpp/test_lyc            (needs a GPU)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "lyc.hpp"

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                      \
  } while (0)
#define CHECK_THROWS(stmt, Exc)                                            \
  do {                                                                     \
    bool thrown_ = false;                                                  \
    try {                                                                  \
      stmt;                                                                \
    } catch (const Exc&) {                                                 \
      thrown_ = true;                                                      \
    } catch (...) {                                                        \
    }                                                                      \
    CHECK(thrown_ && #Exc);                                                \
  } while (0)

using lyc::kernel::BlockIndexSet;
using lyc::kernel::Workload;

// ---------------------------------------------------------------- oracles
// test_util.hpp naive_attention: two-pass softmax over the listed rows, f64.
static std::vector<double> naive_attention(const float* q, const float* K, const float* V, int d,
                                           const std::vector<int>& rows, double scale) {
  std::vector<double> s(rows.size());
  double m = -INFINITY;
  for (size_t i = 0; i < rows.size(); ++i) {
    double acc = 0;
    for (int c = 0; c < d; ++c) acc += (double)q[c] * K[(size_t)rows[i] * d + c];
    s[i] = acc * scale;
    m = std::max(m, s[i]);
  }
  double l = 0;
  for (double& x : s) l += (x = std::exp(x - m));
  std::vector<double> o(d, 0.0);
  for (size_t i = 0; i < rows.size(); ++i)
    for (int c = 0; c < d; ++c) o[c] += s[i] / l * V[(size_t)rows[i] * d + c];
  return o;
}

// attention.hpp:108-123: k largest, ties to the lower index, ascending.
static std::vector<int> top_k(const std::vector<double>& w, size_t k) {
  std::vector<int> idx(w.size());
  std::iota(idx.begin(), idx.end(), 0);
  const size_t kk = std::min(k, w.size());
  std::partial_sort(idx.begin(), idx.begin() + kk, idx.end(),
                    [&](int a, int b) { return w[a] > w[b] || (w[a] == w[b] && a < b); });
  idx.resize(kk);
  std::sort(idx.begin(), idx.end());
  return idx;
}

static Workload<float> random_workload(std::mt19937_64& rng, int B, int H, int G, int d, int L,
                                       double sparse_frac) {
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  Workload<float> w;
  w.batch = B;
  w.n_kv_heads = H;
  w.group_size = G;
  w.d_head = d;
  w.seq_len = L;
  w.block_size = 64;
  w.scale = 1.f / std::sqrt((float)d);
  const int nb = (L + 63) / 64;
  for (int i = 0; i < B * H; ++i) {
    lyc::kernel::Matrix<float> k(L, d), v(L, d);
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
  for (int i = 0; i < B * H; ++i) {
    std::vector<uint32_t> ids;
    for (int b = 0; b < nb; ++b)
      if (i % 2 == 0 || std::uniform_real_distribution<double>(0, 1)(rng) < sparse_frac) ids.push_back(b);
    if (ids.empty()) ids.push_back(0);
    w.blocks.ids.push_back(ids);
  }
  return w;
}

// kernel_sim_test.cpp:69-88 reference_outputs: sparse attention over the
// expanded token set of every slot.
static std::vector<std::vector<double>> expected_outputs(const Workload<float>& w) {
  std::vector<std::vector<double>> out;
  for (size_t b = 0; b < w.batch; ++b)
    for (size_t g = 0; g < w.n_kv_heads; ++g) {
      const size_t slot = b * w.n_kv_heads + g;
      std::vector<int> rows;
      for (uint32_t blk : w.blocks.ids[slot])
        for (size_t r = blk * 64; r < std::min<size_t>((blk + 1) * 64, w.seq_len); ++r) rows.push_back((int)r);
      for (size_t j = 0; j < w.group_size; ++j)
        out.push_back(naive_attention(w.queries[(b * w.n_kv_heads + g) * w.group_size + j].data(),
                                      w.keys[slot].data.data(), w.values[slot].data.data(),
                                      (int)w.d_head, rows, w.scale));
    }
  return out;
}

// ---------------------------------------------------------------- tests
static void test_plan_splits_known() {  // kernel_sim_test.cpp:113-138
  BlockIndexSet a{1, 1, {{0, 1, 2, 3, 4, 5, 6, 7}}};
  auto s = lyc::kernel::plan_splits(a, 2);
  CHECK(s.split_blocks[0] == (std::vector<size_t>{4, 4}));
  CHECK(s.units[0][0].size() == 1 && s.units[0][1][0].head_local_split == 1);
  BlockIndexSet b{1, 3, {{}, {}, {}}};
  for (uint32_t i = 0; i < 16; ++i) b.ids[0].push_back(i);
  b.ids[1] = {0, 1};
  b.ids[2] = {0, 1};
  auto t = lyc::kernel::plan_splits(b, 4);
  CHECK(t.split_blocks[0] == (std::vector<size_t>{5, 5, 5, 5}));
  CHECK(t.head_split_count[0] == (std::vector<size_t>{4, 1, 1}));
  auto r = lyc::kernel::latency_model(t, 1024);
  CHECK(r.pooled_critical_blocks == 5 && r.naive_critical_blocks == 16 && r.total_blocks == 20);
  CHECK(r.pooled_critical_bytes == 5 * 1024);
  CHECK_THROWS(lyc::kernel::plan_splits(a, 0), std::invalid_argument);
  BlockIndexSet z{1, 2, {{}, {}}};
  CHECK_THROWS(lyc::kernel::plan_splits(z, 2), std::invalid_argument);
}

static void test_run_exactness_sweep() {  // acceptance_test.cpp:269-345, kernel_sim_test.cpp:219-239
  std::mt19937_64 rng(2602);
  double worst = 0;
  for (int trial = 0; trial < 6; ++trial) {
    const int B = 1 + trial % 3, H = 1 + trial % 4, G = 1 + trial % 4, d = trial % 2 ? 64 : 128;
    const int L = 300 + 700 * trial;
    auto w = random_workload(rng, B, H, G, d, L, 0.1);
    auto want = expected_outputs(w);
    for (size_t splits : {1, 3, 8}) {
      auto res = lyc::kernel::run(w, splits, 2);
      CHECK(res.outputs.size() == want.size());
      for (size_t h = 0; h < want.size(); ++h)
        for (size_t c = 0; c < w.d_head; ++c)
          worst = std::max(worst, std::abs((double)res.outputs[h][c] - want[h][c]));
      // conservation (kernel_sim_test.cpp:241-248): every listed block once
      CHECK(std::all_of(res.block_exec_counts.begin(), res.block_exec_counts.end(),
                        [](uint32_t c) { return c == 1; }));
      size_t listed = 0;
      for (auto& l : w.blocks.ids) listed += l.size();
      CHECK(res.block_exec_counts.size() == listed);
      CHECK(res.schedule.num_splits == splits);
    }
  }
  std::printf("  run: max |gpu - f64 oracle| = %.3g (bar 1e-5)\n", worst);
  CHECK(worst < 1e-5);
}

static void test_run_determinism() {  // kernel_sim_test.cpp:250-264
  std::mt19937_64 rng(7);
  auto w = random_workload(rng, 2, 4, 4, 64, 2000, 0.3);
  auto a = lyc::kernel::run(w, 16, 1);
  auto b = lyc::kernel::run(w, 16, 8);
  CHECK(a.outputs == b.outputs);
}

static void test_run_errors() {
  std::mt19937_64 rng(3);
  auto w = random_workload(rng, 1, 2, 2, 64, 256, 0.5);
  auto bad = w;
  bad.blocks.ids[0] = {2, 1};
  CHECK_THROWS(lyc::kernel::run(bad, 2), std::invalid_argument);
  bad = w;
  bad.blocks.ids[0] = {99};
  CHECK_THROWS(lyc::kernel::run(bad, 2), std::invalid_argument);
  bad = w;
  bad.queries.pop_back();
  CHECK_THROWS(lyc::kernel::run(bad, 2), std::invalid_argument);
  CHECK_THROWS(lyc::kernel::run(w, 0), std::invalid_argument);
}

static void test_args_top_k() {  // attention_test.cpp:110-135
  std::vector<float> a{0.4f, 0.1f, 0.3f, 0.2f};
  CHECK(lyc::args_top_k<float>(a, 2).indices == (std::vector<size_t>{0, 2}));
  std::vector<float> e(5, 1.f);
  CHECK(lyc::args_top_k<float>(e, 3).indices == (std::vector<size_t>{0, 1, 2}));
  CHECK(lyc::args_top_k<float>(a, 9).size() == 4);
  CHECK_THROWS(lyc::args_top_k<float>(a, 0), std::invalid_argument);
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> s(32768);
  for (auto& x : s) x = U(rng);
  std::vector<double> sd(s.begin(), s.end());
  auto got = lyc::args_top_k<float>(s, 2048).indices;
  auto want = top_k(sd, 2048);
  CHECK(std::equal(got.begin(), got.end(), want.begin(), want.end()));
}

// decode_engine.hpp:109-151 restated on host in f64 for one step.
static void test_hybrid_decoder_tiny() {
  const int NL = 4, H = 2, G = 4, d = 64, L = 4096, K = 256;
  std::vector<uint8_t> roles(NL * H, 1);
  roles[0] = roles[1] = 0;  // layer 0 all retrieval
  roles[2 * H + 1] = 0;     // one retrieval head above
  std::mt19937_64 rng(1234);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> q((size_t)NL * H * G * d), k((size_t)NL * H * L * d), v(k.size());
  for (auto* vec : {&q, &k, &v})
    for (auto& x : *vec) x = U(rng);
  lyc::DeviceBuffer dq(q.size() * 4), dk(k.size() * 4), dv(v.size() * 4), dout(q.size() * 4);
  dq.upload(q.data(), q.size() * 4);
  dk.upload(k.data(), k.size() * 4);
  dv.upload(v.data(), v.size() * 4);
  lyc::HybridDecoder::Config c;
  c.n_layers = NL;
  c.batch = 1;
  c.n_kv_heads = H;
  c.group_size = G;
  c.d_head = d;
  c.dtype = lyc::Dtype::F32;
  c.seq_cap = L;
  c.policy = lyc::SparsityPolicy::top_k(K);
  lyc::HybridDecoder dec(c, roles);
  dec.decode_step(dq.get(), dk.get(), dv.get(), L, dout.get());
  std::vector<float> out(q.size());
  cudaDeviceSynchronize();
  dout.download(out.data(), out.size() * 4);
  auto sets = dec.token_sets();
  // host restatement
  const double scale = 1.0 / std::sqrt((double)d);
  std::vector<std::vector<int>> sets_ref(H);
  double worst = 0, ref_max = 0;
  std::vector<int> all(L);
  std::iota(all.begin(), all.end(), 0);
  for (int l = 0; l < NL; ++l)
    for (int g = 0; g < H; ++g) {
      const float* Kl = k.data() + ((size_t)l * H + g) * L * d;
      const float* Vl = v.data() + ((size_t)l * H + g) * L * d;
      const bool retrieval = l == 0 || roles[l * H + g] == 0;
      const std::vector<int>& rows = retrieval ? all : sets_ref[g];
      for (int j = 0; j < G; ++j) {
        const float* qh = q.data() + (((size_t)l * H + g) * G + j) * d;
        auto o = naive_attention(qh, Kl, Vl, d, rows, scale);
        for (int cc = 0; cc < d; ++cc) {
          worst = std::max(worst, std::abs((double)out[(((size_t)l * H + g) * G + j) * d + cc] - o[cc]));
          ref_max = std::max(ref_max, std::abs(o[cc]));
        }
      }
      if (retrieval) {  // pooled-query selection (gqa_pool_queries + dense weights)
        std::vector<double> pooled(d, 0.0), w(L);
        for (int j = 0; j < G; ++j)
          for (int cc = 0; cc < d; ++cc) pooled[cc] += q[(((size_t)l * H + g) * G + j) * d + cc];
        for (auto& x : pooled) x /= G;
        for (int t = 0; t < L; ++t) {
          double acc = 0;
          for (int cc = 0; cc < d; ++cc) acc += pooled[cc] * Kl[(size_t)t * d + cc];
          w[t] = acc * scale;
        }
        sets_ref[g] = top_k(w, K);
      }
    }
  const double rel = worst / std::max(ref_max, 1e-3);
  std::printf("  decoder: rel err %.3g (bar 1e-5), sets %s\n", rel,
              sets[0] == std::vector<int32_t>(sets_ref[0].begin(), sets_ref[0].end()) ? "equal" : "DIFFER");
  CHECK(rel < 1e-5);
  for (int g = 0; g < H; ++g) CHECK(sets[g] == std::vector<int32_t>(sets_ref[g].begin(), sets_ref[g].end()));
}

static void test_hybrid_decoder_errors() {
  lyc::HybridDecoder::Config c;
  c.n_layers = 2;
  c.n_kv_heads = 2;
  c.group_size = 4;
  c.d_head = 64;
  c.seq_cap = 1024;
  c.policy = lyc::SparsityPolicy::top_k(16);
  std::vector<uint8_t> bad{1, 0, 0, 0};  // layer 0 must be all retrieval
  CHECK_THROWS(lyc::HybridDecoder(c, bad), std::invalid_argument);
  std::vector<uint8_t> ok{0, 0, 1, 1};
  c.policy = lyc::SparsityPolicy::top_p(0.9);
  c.select = lyc::Select::Blocks;  // TopP selects tokens only
  CHECK_THROWS(lyc::HybridDecoder(c, ok), lyc::not_supported);
  c.select = lyc::Select::Tokens;
  CHECK_THROWS(lyc::SparsityPolicy::threshold(0.0), std::invalid_argument);
  CHECK_THROWS(lyc::SparsityPolicy::top_k(0), std::invalid_argument);
  CHECK_THROWS(lyc::SparsityPolicy::ratio(1.5), std::invalid_argument);
  CHECK(lyc::fraction_budget(0.1, 100) == 10);
}

// Sequence sharding over P = 2 ranks emulated on one GPU: each rank's
// exchange copies its block into a shared gathered buffer; the step runs rank
// by rank per layer (local work of both ranks, then both combines), so the
// result must equal the unsharded decoder.
static void test_sharded_decoder_two_ranks() {
  const int NL = 2, H = 2, G = 4, d = 64, L = 3000, K = 128, P = 2;
  std::vector<uint8_t> roles{0, 0, 1, 0};
  std::mt19937_64 rng(99);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> q((size_t)NL * H * G * d), k((size_t)NL * H * L * d), v(k.size());
  for (auto* vec : {&q, &k, &v})
    for (auto& x : *vec) x = U(rng);
  lyc::DeviceBuffer dq(q.size() * 4), dk(k.size() * 4), dv(v.size() * 4), dref(q.size() * 4);
  dq.upload(q.data(), q.size() * 4);
  dk.upload(k.data(), k.size() * 4);
  dv.upload(v.data(), v.size() * 4);
  lyc::HybridDecoder::Config c;
  c.n_layers = NL;
  c.n_kv_heads = H;
  c.group_size = G;
  c.d_head = d;
  c.dtype = lyc::Dtype::F32;
  c.seq_cap = L;
  c.policy = lyc::SparsityPolicy::top_k(K);
  lyc::HybridDecoder full(c, roles);
  full.decode_step(dq.get(), dk.get(), dv.get(), L, dref.get());
  std::vector<float> ref(q.size());
  cudaDeviceSynchronize();
  dref.download(ref.data(), ref.size() * 4);
  // two ranks, rows [0, 1500) and [1500, 3000): their caches are views of the
  // full cache at the same slab stride (seq_cap = L); one shared gathered
  // buffer stands in for the all-gather
  const size_t half = L / 2;
  std::vector<std::unique_ptr<lyc::ShardedDecoder>> ranks;
  for (int r = 0; r < P; ++r)
    ranks.push_back(std::make_unique<lyc::ShardedDecoder>(c, roles, P, r, nullptr));
  const size_t words = ranks[0]->block_words();
  lyc::DeviceBuffer gathered(words * 4 * P), d0(q.size() * 4), d1(q.size() * 4);
  const size_t qstride = (size_t)H * G * d;
  for (int l = 0; l < NL; ++l) {
    for (int r = 0; r < P; ++r) {
      const float* kr = dk.as<float>() + r * half * d;
      const float* vr = dv.as<float>() + r * half * d;
      ranks[r]->layer_local(l, dq.as<float>() + l * qstride, kr, vr, half, r * half);
      cudaMemcpy(gathered.as<float>() + r * words, ranks[r]->send(), words * 4, cudaMemcpyDeviceToDevice);
    }
    for (int r = 0; r < P; ++r)
      ranks[r]->layer_combine(l, gathered.as<float>(), half, r * half, L,
                              (r ? d1 : d0).as<float>() + l * qstride);
  }
  std::vector<float> o0(q.size()), o1(q.size());
  cudaDeviceSynchronize();
  d0.download(o0.data(), o0.size() * 4);
  d1.download(o1.data(), o1.size() * 4);
  double worst = 0, mx = 0;
  for (size_t i = 0; i < ref.size(); ++i) {
    worst = std::max(worst, (double)std::abs(o0[i] - ref[i]));
    mx = std::max(mx, (double)std::abs(ref[i]));
  }
  std::printf("  sharded x2: rel err vs unsharded %.3g (bar 1e-5), ranks bitwise equal: %s\n",
              worst / std::max(mx, 1e-3), o0 == o1 ? "yes" : "NO");
  CHECK(worst / std::max(mx, 1e-3) < 1e-5);
  CHECK(o0 == o1);
}

// kv_cache.hpp:23-42 through lyc::KvCache, then the cache-correction
// attention (decode_engine.hpp:164-204) against a host two-pass softmax loop.
static void test_kv_cache_and_correction() {
  const int L = 2, B = 1, H = 2, G = 2, d = 32, cap = 300, T = 200, W = 8;
  const std::size_t slab = (std::size_t)cap * d, n = (std::size_t)L * B * H * slab;
  lyc::DeviceBuffer kc(n * 4), vc(n * 4);
  cudaMemset(kc.get(), 0, n * 4);
  cudaMemset(vc.get(), 0, n * 4);
  lyc::KvCache kv(L, B, H, d, cap, lyc::Dtype::F32, kc.get(), vc.get());
  std::mt19937 rng(5);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> hk(n, 0.f), hv(n, 0.f), rowk((std::size_t)B * H * d), rowv(rowk.size());
  lyc::DeviceBuffer dk(rowk.size() * 4), dv(rowv.size() * 4);
  for (int t = 0; t < T; ++t) {
    for (int l = 0; l < L; ++l) {
      for (std::size_t i = 0; i < rowk.size(); ++i) {
        rowk[i] = U(rng);
        rowv[i] = U(rng);
      }
      dk.upload(rowk.data(), rowk.size() * 4);
      dv.upload(rowv.data(), rowv.size() * 4);
      kv.append(l, dk.get(), dv.get());
      for (int g = 0; g < H; ++g)
        for (int c = 0; c < d; ++c) {
          hk[((std::size_t)l * H + g) * slab + (std::size_t)t * d + c] = rowk[(std::size_t)g * d + c];
          hv[((std::size_t)l * H + g) * slab + (std::size_t)t * d + c] = rowv[(std::size_t)g * d + c];
        }
    }
    kv.commit_row();
  }
  CHECK(kv.length() == (std::size_t)T);
  // rewrite the trailing window of layer 1 (overwrite, n_rows = W)
  std::vector<float> wk((std::size_t)H * W * d), wv(wk.size());
  for (std::size_t i = 0; i < wk.size(); ++i) {
    wk[i] = U(rng);
    wv[i] = U(rng);
  }
  lyc::DeviceBuffer dwk(wk.size() * 4), dwv(wv.size() * 4);
  dwk.upload(wk.data(), wk.size() * 4);
  dwv.upload(wv.data(), wv.size() * 4);
  const int start = T - W;
  kv.overwrite(1, start, W, dwk.get(), dwv.get());
  for (int g = 0; g < H; ++g)
    for (int i = 0; i < W; ++i)
      for (int c = 0; c < d; ++c) {
        hk[((std::size_t)1 * H + g) * slab + (std::size_t)(start + i) * d + c] = wk[((std::size_t)g * W + i) * d + c];
        hv[((std::size_t)1 * H + g) * slab + (std::size_t)(start + i) * d + c] = wv[((std::size_t)g * W + i) * d + c];
      }
  std::vector<float> gk(n), gv(n);
  kc.download(gk.data(), n * 4);
  vc.download(gv.data(), n * 4);
  CHECK(gk == hk && gv == hv);
  CHECK_THROWS(kv.overwrite(0, T - 2, W, dwk.get(), dwv.get()), std::invalid_argument);
  // correction attention of layer 1: window position i attends keys [0, start + i]
  const int Hq = H * G;
  std::vector<float> q((std::size_t)B * W * Hq * d);
  for (auto& x : q) x = U(rng);
  lyc::DeviceBuffer dq(q.size() * 4), dout(q.size() * 4);
  dq.upload(q.data(), q.size() * 4);
  lyc_kv_layout lay{L, B, H, d, LYC_DTYPE_F32, 0, cap};
  const int64_t ws = lyc::check(lyc_window_workspace(&lay, G, W));
  lyc::DeviceBuffer dws((std::size_t)std::max<int64_t>(ws, 16));
  lyc::check(lyc_window_attention(&lay, 1, kc.get(), vc.get(), G, 0.f, start, W, dq.get(), dout.get(),
                                  dws.get(), ws, nullptr));
  std::vector<float> got(q.size());
  dout.download(got.data(), got.size() * 4);
  const double scale = 1.0 / std::sqrt((double)d);
  double worst = 0.0;
  for (int i = 0; i < W; ++i)
    for (int hq = 0; hq < Hq; ++hq) {
      const int g = hq / G, p = start + i;
      const float* qr = &q[((std::size_t)i * Hq + hq) * d];
      const float* K = &hk[((std::size_t)1 * H + g) * slab];
      const float* V = &hv[((std::size_t)1 * H + g) * slab];
      std::vector<double> w(p + 1);
      double m = -1e300, den = 0.0;
      for (int t = 0; t <= p; ++t) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += (double)qr[c] * K[(std::size_t)t * d + c];
        w[t] = acc * scale;
        m = std::max(m, w[t]);
      }
      for (int t = 0; t <= p; ++t) den += (w[t] = std::exp(w[t] - m));
      for (int c = 0; c < d; ++c) {
        double o = 0.0;
        for (int t = 0; t <= p; ++t) o += w[t] / den * V[(std::size_t)t * d + c];
        worst = std::max(worst, std::abs(o - got[((std::size_t)i * Hq + hq) * d + c]));
      }
    }
  CHECK(worst < 1e-5);
}

// A variable-length batch (lyc_decoder_step_varlen) equals batch-1 decoders
// each run at its own item's length (DecodeEngine is one sequence,
// decode_engine.hpp:95-151).
static void test_decoder_varlen() {
  const int NL = 3, B = 2, H = 2, G = 2, d = 64, cap = 4096, K = 128;
  const std::vector<std::size_t> lens = {3000, 1100};
  std::vector<uint8_t> roles(NL * H, 1);
  roles[0] = roles[1] = 0;
  roles[1 * H + 1] = 0;
  std::mt19937_64 rng(77);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  const std::size_t qi = (std::size_t)H * G * d, ki = (std::size_t)H * cap * d;
  std::vector<float> q((size_t)NL * B * qi), k((size_t)NL * B * ki), v(k.size());
  for (auto* vec : {&q, &k, &v})
    for (auto& x : *vec) x = U(rng);
  lyc::HybridDecoder::Config c;
  c.n_layers = NL;
  c.batch = B;
  c.n_kv_heads = H;
  c.group_size = G;
  c.d_head = d;
  c.dtype = lyc::Dtype::F32;
  c.seq_cap = cap;
  c.policy = lyc::SparsityPolicy::top_k(K);
  lyc::DeviceBuffer dq(q.size() * 4), dk(k.size() * 4), dv(v.size() * 4), dout(q.size() * 4);
  dq.upload(q.data(), q.size() * 4);
  dk.upload(k.data(), k.size() * 4);
  dv.upload(v.data(), v.size() * 4);
  lyc::HybridDecoder dec(c, roles);
  dec.decode_step(dq.get(), dk.get(), dv.get(), lens, dout.get());
  cudaDeviceSynchronize();
  std::vector<float> out(q.size());
  dout.download(out.data(), out.size() * 4);
  const auto sets = dec.token_sets();
  c.batch = 1;
  double worst = 0.0;
  bool sets_equal = true;
  for (int b = 0; b < B; ++b) {
    std::vector<float> q1((size_t)NL * qi), k1((size_t)NL * ki), v1(k1.size());
    for (int l = 0; l < NL; ++l) {
      std::copy_n(q.begin() + ((size_t)l * B + b) * qi, qi, q1.begin() + (size_t)l * qi);
      std::copy_n(k.begin() + ((size_t)l * B + b) * ki, ki, k1.begin() + (size_t)l * ki);
      std::copy_n(v.begin() + ((size_t)l * B + b) * ki, ki, v1.begin() + (size_t)l * ki);
    }
    lyc::DeviceBuffer eq(q1.size() * 4), ek(k1.size() * 4), ev(v1.size() * 4), eo(q1.size() * 4);
    eq.upload(q1.data(), q1.size() * 4);
    ek.upload(k1.data(), k1.size() * 4);
    ev.upload(v1.data(), v1.size() * 4);
    lyc::HybridDecoder one(c, roles);
    one.decode_step(eq.get(), ek.get(), ev.get(), lens[(size_t)b], eo.get());
    cudaDeviceSynchronize();
    std::vector<float> o1(q1.size());
    eo.download(o1.data(), o1.size() * 4);
    for (int l = 0; l < NL; ++l)
      for (std::size_t i = 0; i < qi; ++i)
        worst = std::max(worst, (double)std::abs(out[((size_t)l * B + b) * qi + i] - o1[(size_t)l * qi + i]));
    const auto s1 = one.token_sets();
    for (int g = 0; g < H; ++g) sets_equal = sets_equal && sets[(size_t)b * H + g] == s1[(size_t)g];
  }
  std::printf("  varlen: max |diff| vs batch-1 decoders %.2e, sets equal: %s\n", worst,
              sets_equal ? "yes" : "no");
  CHECK(worst < 1e-5);
  CHECK(sets_equal);
  CHECK(sets[1].size() == (std::size_t)K && sets[1].back() < 3000);
  CHECK_THROWS(dec.decode_step(dq.get(), dk.get(), dv.get(), std::vector<std::size_t>{10, 0}, dout.get()),
               std::invalid_argument);
}


// toy_model.hpp:161-274 decode operations (lyc::model, through lyc_gemv)
// against plain double loops of the reference's own formulas on the same
// bf16-rounded weights.
static uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
static double rel_err(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 1e-3;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a[i] - b[i]));
    den = std::max(den, std::abs(b[i]));
  }
  return num / den;
}

static void test_model_ops() {
  const int D = 256, nq = 4, nkv = 2, d = 32, dff = 512, vocab = 300, cap = 8, pos = 5;
  const int Mqkv = (nq + 2 * nkv) * d, hqd = nq * d;
  std::mt19937_64 rng(91);
  std::normal_distribution<float> N(0.f, 1.f);
  auto weights = [&](int M, int K, std::vector<uint16_t>& hb, std::vector<double>& hd) {
    hb.resize((size_t)M * K);
    hd.resize(hb.size());
    for (size_t i = 0; i < hb.size(); ++i) {
      hb[i] = to_bf16(N(rng) / std::sqrt((float)K));
      hd[i] = from_bf16(hb[i]);
    }
  };
  std::vector<uint16_t> bqkv, bo, b1, b2, blm;
  std::vector<double> wqkv, wo, w1, w2, wlm;
  weights(Mqkv, D, bqkv, wqkv);
  weights(D, hqd, bo, wo);
  weights(dff, D, b1, w1);
  weights(D, dff, b2, w2);
  weights(vocab, D, blm, wlm);
  std::vector<float> x(D), g(D), o(hqd);
  for (auto& v : x) v = N(rng);
  for (auto& v : g) v = 1.f + 0.1f * N(rng);
  std::vector<uint16_t> ob(hqd);
  for (int i = 0; i < hqd; ++i) ob[i] = to_bf16(N(rng) * 0.5f);
  auto up = [](const void* src, std::size_t bytes) {
    lyc::DeviceBuffer b(bytes);
    b.upload(src, bytes);
    return b;
  };
  lyc::DeviceBuffer dwqkv = up(bqkv.data(), bqkv.size() * 2), dwo = up(bo.data(), bo.size() * 2),
                    dw1 = up(b1.data(), b1.size() * 2), dw2 = up(b2.data(), b2.size() * 2),
                    dwlm = up(blm.data(), blm.size() * 2), dx = up(x.data(), D * 4),
                    dg = up(g.data(), D * 4), dob = up(ob.data(), hqd * 2);
  lyc::DeviceBuffer dq(hqd * 2), dk((size_t)nkv * cap * d * 2), dv((size_t)nkv * cap * d * 2),
      dmid((size_t)dff * 2), dlog((size_t)vocab * 4);
  cudaMemset(dk.get(), 0, dk.bytes());
  cudaMemset(dv.get(), 0, dv.bytes());
  // host references (toy_model.hpp formulas, double)
  auto rms = [&](const std::vector<double>& v) {
    double ss = 0.0;
    for (double e : v) ss += e * e;
    const double inv = 1.0 / std::sqrt(ss / (double)v.size() + 1e-6);
    std::vector<double> y(v.size());
    for (size_t i = 0; i < v.size(); ++i) y[i] = v[i] * inv * (double)g[i];
    return y;
  };
  auto matvec = [](const std::vector<double>& w, int M, int K, const std::vector<double>& in) {
    std::vector<double> y((size_t)M, 0.0);
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < K; ++c) y[(size_t)r] += w[(size_t)r * K + c] * in[(size_t)c];
    return y;
  };
  auto rope = [&](double* h) {
    for (int i = 0; i + 1 < d; i += 2) {
      const double f = std::pow(10000.0, -(double)i / (double)d), a = pos * f;
      const double c = std::cos(a), sn = std::sin(a), u = h[i], w = h[i + 1];
      h[i] = u * c - w * sn;
      h[i + 1] = u * sn + w * c;
    }
  };
  std::vector<double> xd(x.begin(), x.end());
  // compute_qkv
  lyc::model::compute_qkv(dwqkv.get(), D, dx.as<float>(), dg.as<float>(), nq, nkv, d, pos, dq.get(),
                          dk.get(), dv.get(), (int64_t)cap * d);
  std::vector<double> y = matvec(wqkv, Mqkv, D, rms(xd));
  for (int h = 0; h < nq + nkv; ++h) rope(&y[(size_t)h * d]);
  std::vector<uint16_t> qh(hqd), kh((size_t)nkv * cap * d), vh(kh.size());
  dq.download(qh.data(), qh.size() * 2);
  dk.download(kh.data(), kh.size() * 2);
  dv.download(vh.data(), vh.size() * 2);
  std::vector<double> got(Mqkv), want(y);
  for (int i = 0; i < hqd; ++i) got[(size_t)i] = from_bf16(qh[(size_t)i]);
  for (int gk = 0; gk < nkv; ++gk)
    for (int i = 0; i < d; ++i) {
      got[(size_t)hqd + gk * d + i] = from_bf16(kh[((size_t)gk * cap + pos) * d + i]);
      got[(size_t)hqd + nkv * d + gk * d + i] = from_bf16(vh[((size_t)gk * cap + pos) * d + i]);
    }
  CHECK(rel_err(got, want) < 1e-2);
  CHECK(from_bf16(kh[((size_t)0 * cap + pos - 1) * d]) == 0.f);  // only row `pos` written
  // attn_project_residual: x += W_o o
  lyc::model::attn_project_residual(dwo.get(), D, dob.get(), hqd, dx.as<float>());
  std::vector<double> od(hqd);
  for (int i = 0; i < hqd; ++i) od[(size_t)i] = from_bf16(ob[(size_t)i]);
  const std::vector<double> pr = matvec(wo, D, hqd, od);
  for (int i = 0; i < D; ++i) xd[(size_t)i] += pr[(size_t)i];
  std::vector<float> xh(D);
  dx.download(xh.data(), D * 4);
  CHECK(rel_err(std::vector<double>(xh.begin(), xh.end()), xd) < 1e-4);
  // ffn_residual: x += W2 silu(W1 rmsnorm(x))   (mid rounded to bf16 on the device)
  lyc::model::ffn_residual(dw1.get(), dw2.get(), D, dff, dg.as<float>(), dx.as<float>(), dmid.get());
  std::vector<double> mid = matvec(w1, dff, D, rms(xd));
  for (auto& v : mid) v = (double)from_bf16(to_bf16((float)(v / (1.0 + std::exp(-v)))));
  const std::vector<double> f2 = matvec(w2, D, dff, mid);
  for (int i = 0; i < D; ++i) xd[(size_t)i] += f2[(size_t)i];
  dx.download(xh.data(), D * 4);
  CHECK(rel_err(std::vector<double>(xh.begin(), xh.end()), xd) < 2e-3);
  // output_logits
  lyc::model::output_logits(dwlm.get(), vocab, D, dx.as<float>(), dg.as<float>(), dlog.as<float>());
  const std::vector<double> lg = matvec(wlm, vocab, D, rms(xd));
  std::vector<float> lh(vocab);
  cudaDeviceSynchronize();
  dlog.download(lh.data(), lh.size() * 4);
  CHECK(rel_err(std::vector<double>(lh.begin(), lh.end()), lg) < 2e-3);
  std::printf("  model ops: qkv / o-proj / ffn / logits match the double loops\n");
  // errors as the reference's: shape violations throw std::invalid_argument
  CHECK_THROWS(lyc::model::compute_qkv(dwqkv.get(), D, dx.as<float>(), dg.as<float>(), nq, nkv, d + 1,
                                       pos, dq.get(), dk.get(), dv.get(), (int64_t)cap * d),
               std::invalid_argument);
  CHECK_THROWS(lyc::model::output_logits(dwlm.get(), vocab, D - 4, dx.as<float>(), dg.as<float>(),
                                         dlog.as<float>()),
               std::invalid_argument);
}

int main() {
  const std::pair<const char*, std::function<void()>> tests[] = {
      {"PlanSplits.KnownAnswersAndErrors", test_plan_splits_known},
      {"Run.ExactnessSweepF32", test_run_exactness_sweep},
      {"Run.DeterministicAcrossWorkers", test_run_determinism},
      {"Run.Errors", test_run_errors},
      {"ArgsTopK.KnownCasesTiesAndSort", test_args_top_k},
      {"HybridDecoder.TinyStepMatchesHostLoop", test_hybrid_decoder_tiny},
      {"HybridDecoder.Errors", test_hybrid_decoder_errors},
      {"ShardedDecoder.TwoRanksEqualUnsharded", test_sharded_decoder_two_ranks},
      {"KvCache.AppendOverwriteAndCorrectionAttention", test_kv_cache_and_correction},
      {"HybridDecoder.VariableLengthBatch", test_decoder_varlen},
      {"Model.DecodeOpsMatchDoubleLoops", test_model_ops},
  };
  for (const auto& [name, fn] : tests) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  FAIL uncaught %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "  OK  " : " FAIL ", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
