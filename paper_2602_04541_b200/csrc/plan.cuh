// plan.cuh -- the seq-parametric plan of the fused decode step (Algorithm 2's
// pooled split plan, kernel_sim.hpp:63-110, in the step kernel's three-pool
// order), computed from the static role map (rolemap.hpp:33-35) and the
// step's sequence lengths.
//
// The same code runs
//   * on the device, one CTA per layer (plan_kernel in plan.cu): a decode
//     loop re-plans every token inside the stream / CUDA graph, with no host
//     work, no host synchronisation and no allocation;
//   * on the host, sequentially (HostX below): the planner self-test compares
//     it with the host-order planner of capi.cu (lyc_plan_selftest).
// Every phase is a "for i in [0, n)" over independent items (threads on the
// device, a loop on the host) separated by barriers; an item reads only what
// earlier phases wrote.
//
// Per layer l (B batch items, H KV heads, S splits per item):
//   slot (b, g): retrieval (l == 0 or role R) -> dense items ceil(len_b / bs)
//     and selection row sel = b * n_ret + rank(g); sparse -> token tiles
//     ceil(k_b / 64) (or k_b blocks) of the index-cache row b*H+g, inheriting
//     the set of the nearest earlier retrieval layer of head g (dep);
//   pools: 0 = retrieval slots, 1 = sparse slots with an older set, 2 = sparse
//     slots whose set the previous layer selects (streamed last);
//   each (group, pool) list is cut evenly over the group's cells (the sparse
//     pools over the cells not running selection items when those fit in
//     half the grid), cut points snapped onto slot boundaries within one
//     item; a cell's units are pool 0, 1, 2 in order.
#pragma once
#include <stdint.h>

#include "../../include/lyc.h"
#include "lyc_plan.h"

#if defined(__CUDACC__)
#define LYC_HD __host__ __device__
#else
#define LYC_HD
#endif
#ifndef LYC_PLAN_STAMP
#define LYC_PLAN_STAMP(k)  // profiling hook (scripts/micro/plan_profile.cu)
#endif

namespace lyc {

// Write targets of one layer's plan (device arrays, or host staging in the
// emulation).  Pointer VALUES stored inside records (a slot's index-cache
// row) are device addresses in both cases.
struct PlanOut {
  LycSlot* slots;
  LycUnit* units;
  LycSlot* unit_slots;
  int32_t* split_off;
  LycMergeTask* merges;
  int32_t* sel_rows;
  int32_t* sel_n;
  int32_t* sel_k;
  int32_t* n_merges;   // -> LycLayerDesc::n_merges
  int32_t* n_sel;      // -> LycLayerDesc::n_sel
  int32_t* n_units;    // optional: units of the layer (self-test)
};

// Scratch of one layer (shared memory on the device).
struct PlanScratch {
  int32_t *items, *pool, *start, *nunits, *first_sp, *first_unit, *mrg, *list;  // [BH] ([3BH] list)
  int32_t *seqs, *dep, *rank;               // [B], [H], [H]
  int32_t *roles;                           // [NL * H] the role map (staged once)
  int32_t *cb_n, *cb_tot, *cb_ns;           // [3 * groups]
  int32_t *cuts;                            // [3 * (cells + groups)]
  int32_t *ccount, *coff;                   // [cells], [cells + 1]
  int32_t *misc;                            // [64]: scan scratch + layer scalars
};

enum { PM_RAGGED = 40, PM_NRET, PM_SEQMAX, PM_FREE, PM_BAD, PM_BADITEM, PM_NMERGE, PM_NUNITS };

inline LYC_HD int plan_scratch_ints(int B, int H, int S, int NL) {
  const int BH = B * H, cells = B * S, groups = B;
  return 7 * BH + 3 * BH + B + 2 * H + NL * H + 3 * 3 * groups + 3 * (cells + groups) + cells +
         cells + 1 + 64;
}

inline LYC_HD PlanScratch plan_carve(int32_t* base, int B, int H, int S, int NL) {
  const int BH = B * H, cells = B * S, groups = B;
  PlanScratch s;
  int32_t* p = base;
  auto take = [&](int n) { int32_t* r = p; p += n; return r; };
  s.items = take(BH);
  s.pool = take(BH);
  s.start = take(BH);
  s.nunits = take(BH);
  s.first_sp = take(BH);
  s.first_unit = take(BH);
  s.mrg = take(BH);
  s.list = take(3 * BH);
  s.seqs = take(B);
  s.dep = take(H);
  s.rank = take(H);
  s.roles = take(NL * H);
  s.cb_n = take(3 * groups);
  s.cb_tot = take(3 * groups);
  s.cb_ns = take(3 * groups);
  s.cuts = take(3 * (cells + groups));
  s.ccount = take(cells);
  s.coff = take(cells + 1);
  s.misc = take(64);
  return s;
}

// policy.hpp:57-62 fraction_budget (the same double arithmetic as the host)
inline LYC_HD int64_t plan_fraction_budget(double frac, int64_t n) {
  const double raw = frac * (double)n;
  const double c = ceil(raw - 1e-9);
  int64_t b = c < 0 ? 0 : (int64_t)c;
  b = b < 1 ? 1 : b;
  return b < n ? b : n;
}

// Tokens (or blocks) kept per sparse head at length seq (lyc_decoder::budget).
inline LYC_HD int64_t plan_budget(const LycPlanIn& in, int64_t seq) {
  if (in.select_mode == LYC_SELECT_BLOCKS) {
    const int64_t nb = (seq + in.bs - 1) / in.bs;
    if (in.policy_kind == LYC_POLICY_RATIO) return plan_fraction_budget(1.0 - in.ratio, nb);
    const int64_t kb = (in.top_k + in.bs - 1) / in.bs;
    return kb < nb ? kb : nb;
  }
  if (in.policy_kind == LYC_POLICY_RATIO) return plan_fraction_budget(1.0 - in.ratio, seq);
  return in.top_k < seq ? in.top_k : seq;
}

// The slot record of (b, g) = slot i of layer l (every field from the scratch
// arrays: no global reads).
inline LYC_HD LycSlot plan_slot(const LycPlanIn& in, int l, int i, const PlanScratch& s, int nret,
                                bool none, bool blocks) {
  const int H = in.H, b = i / H, g = i - b * H;
  const int64_t seq_b = s.seqs[b];
  const int64_t kb_b = plan_budget(in, seq_b);
  LycSlot sl;
  sl.kv_off = (((int64_t)l * in.B + b) * H + g) * in.seq_cap * in.D;
  sl.list = nullptr;
  sl.count = nullptr;
  sl.list_len = 0;
  sl.first_unit = s.first_unit[i];
  sl.n_units = s.nunits[i];
  sl.q_row = b * H * in.G + g * in.G;
  sl.sel = -1;
  sl.dep = -1;
  sl.seq = (int32_t)seq_b;
  sl.item = b;
  sl.n_items = s.items[i];
  if (s.rank[g] >= 0) {
    sl.kind = ITEM_DENSE;
    if (!none) sl.sel = b * nret + s.rank[g];
  } else {
    sl.kind = blocks ? ITEM_BLOCKS : ITEM_TOKENS;
    sl.list = in.idx + (int64_t)i * in.k_cap;
    sl.list_len = (int32_t)kb_b;
    sl.dep = s.dep[g];
  }
  return sl;
}

// The plan key of one batch item: dense blocks and sparse budget at length seq.
inline LYC_HD void plan_item_key(const LycPlanIn& in, int64_t seq, int32_t& nb, int32_t& kb) {
  nb = (int32_t)((seq + in.bs - 1) / in.bs);
  kb = (int32_t)plan_budget(in, seq);
}

// Selection items per row (step.cu kItemKeys keys each) at maximum length mx.
inline LYC_HD int32_t plan_items(const LycPlanIn& in, int64_t mx) {
  if (in.select_mode == LYC_SELECT_NONE) return 0;
  const int64_t nk = in.select_mode == LYC_SELECT_BLOCKS ? (mx + in.bs - 1) / in.bs : mx;
  return (int32_t)((nk + in.item_keys - 1) / in.item_keys);
}

// Combo cb = (group, pool): its cells [c0, c0 + nc) and slots [s0, s0 + ns).
struct Combo {
  int grp, pool, c0, nc, s0, nslots;
};
inline LYC_HD Combo plan_combo(int cb, bool ragged, int B, int H, int S) {
  Combo c;
  c.grp = cb / 3;
  c.pool = cb % 3;
  const int b0 = ragged ? 0 : c.grp, b1 = ragged ? B : c.grp + 1;
  c.c0 = b0 * S;
  c.nc = (b1 - b0) * S;
  c.s0 = b0 * H;
  c.nslots = (b1 - b0) * H;
  return c;
}
inline LYC_HD int32_t* plan_cuts(const PlanScratch& s, int cb, bool ragged, int B, int S) {
  // combo cb's nc + 1 cut points; groups are B (uniform) or 1 (ragged)
  const int nc = ragged ? B * S : S;
  return s.cuts + cb * (nc + 1);
}
inline LYC_HD int32_t* plan_list(const PlanScratch& s, int cb, bool ragged, int B, int H) {
  const Combo c = plan_combo(cb, ragged, B, H, 1);
  return s.list + 3 * c.s0 + c.pool * c.nslots;
}

// Largest sp in [0, nc] with cut[sp] <= x (x < cut[nc]): the cell holding item x.
inline LYC_HD int plan_cell_of(const int32_t* cut, int nc, int32_t x) {
  int lo = 0, hi = nc;  // cut[lo] <= x < cut[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cut[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Exclusive scan of a[0, n) in place; returns the total.  X provides the
// parallel primitive (device: block scan; host: a loop).
template <class X>
LYC_HD int32_t plan_scan(X& x, int32_t* a, int n, int32_t* tmp) {
  return x.scan(a, n, tmp);
}

template <class X>
LYC_HD void plan_layer(X& x, const LycPlanIn& in, int l, const PlanScratch& s, const PlanOut& o) {
  const int B = in.B, H = in.H, G = in.G, S = in.S, BH = B * H, cells = B * S;
  const bool blocks = in.select_mode == LYC_SELECT_BLOCKS;
  const bool none = in.select_mode == LYC_SELECT_NONE;
  int32_t* misc = s.misc;
  LYC_PLAN_STAMP(0);
  // ---- phase 0: lengths, the role map on chip, per-head role facts
  for (int i = x.tid(); i < in.NL * H; i += x.nthreads()) s.roles[i] = in.roles[i];
  for (int b = x.tid(); b < B; b += x.nthreads()) {
    const int64_t v = in.dlens ? in.dlens[b] : in.has_lens ? (int64_t)in.lens[b] : in.seq;
    s.seqs[b] = (int32_t)(v < 1 ? 0 : v > in.seq_cap ? -1 : v);
  }
  x.sync();
  for (int g = x.tid(); g < H; g += x.nthreads()) {
    const bool R = l == 0 || s.roles[l * H + g] == 0;
    int dep = -1;
    if (!R)
      for (int j = l - 1; j >= 0; --j)
        if (j == 0 || s.roles[j * H + g] == 0) {
          dep = j;
          break;
        }
    s.dep[g] = dep;
    int rk = -1;
    if (R) {
      rk = 0;
      for (int h = 0; h < g; ++h) rk += (l == 0 || s.roles[l * H + h] == 0) ? 1 : 0;
    }
    s.rank[g] = rk;
  }
  x.sync();
  if (x.tid() == 0) {
    int nret = 0;
    for (int g = 0; g < H; ++g) nret += s.rank[g] >= 0 ? 1 : 0;
    int ragged = 0, bad = 0, bad_item = -1;
    int32_t mx = 0, nb0 = 0, kb0 = 0;
    if (s.seqs[0] > 0) plan_item_key(in, s.seqs[0], nb0, kb0);
    for (int b = 0; b < B; ++b) {
      if (s.seqs[b] <= 0 && !bad) {
        bad = 1;
        bad_item = b;
      }
      if (s.seqs[b] > 0) {  // ragged: the items' plan keys differ (a pool per batch or one pool)
        int32_t nb, kb;
        plan_item_key(in, s.seqs[b], nb, kb);
        ragged |= nb != nb0 || kb != kb0;
      }
      mx = s.seqs[b] > mx ? s.seqs[b] : mx;
    }
    misc[PM_NRET] = nret;
    misc[PM_RAGGED] = ragged;
    misc[PM_SEQMAX] = mx;
    misc[PM_BAD] = bad;
    misc[PM_BADITEM] = bad_item;
    // this layer's selection items run on the last n_items CTAs when they fit
    // in half the grid (step.cu split roles); the sparse pools skip them
    int free_from = cells;
    if (!none && !bad) {
      const int64_t n_items = (int64_t)B * nret * plan_items(in, mx);
      if (n_items > 0 && 2 * n_items <= cells) free_from = cells - (int)n_items;
    }
    misc[PM_FREE] = free_from;
  }
  x.sync();
  if (misc[PM_BAD]) {  // invalid lengths: an empty plan, flagged in the header
    if (x.tid() == 0) {
      *o.n_merges = 0;
      *o.n_sel = 0;
      for (int c = 0; c <= cells; ++c) o.split_off[c] = 0;
      if (l == 0) {
        in.hdr->status = 1;
        in.hdr->bad_item = misc[PM_BADITEM];
      }
    }
    return;
  }
  const bool ragged = misc[PM_RAGGED] != 0;
  const int nret = misc[PM_NRET];
  LYC_PLAN_STAMP(1);
  // ---- phase 1: items and pool of every slot, the selection rows
  for (int i = x.tid(); i < BH; i += x.nthreads()) {
    const int b = i / H, g = i - b * H;
    const int64_t seq_b = s.seqs[b];
    const int64_t nb_b = (seq_b + in.bs - 1) / in.bs;
    const int64_t kb_b = plan_budget(in, seq_b);
    if (s.rank[g] >= 0) {
      s.items[i] = (int32_t)nb_b;
      if (!none) {
        const int sel = b * nret + s.rank[g];
        o.sel_rows[sel] = i;
        o.sel_n[sel] = (int32_t)(blocks ? nb_b : seq_b);
        o.sel_k[sel] = (int32_t)kb_b;
      }
      s.pool[i] = 0;
    } else {
      s.items[i] = blocks ? (int32_t)kb_b : (int32_t)((kb_b + LYC_TILE - 1) / LYC_TILE);
      s.pool[i] = s.dep[g] == l - 1 ? 2 : 1;
    }
  }
  x.sync();
  LYC_PLAN_STAMP(2);
  // ---- phase 2: per (group, pool): the slot list, item offsets, cut points
  const int groups = ragged ? 1 : B;
  const int free_from = misc[PM_FREE];
  for (int cb = x.tid(); cb < 3 * groups; cb += x.nthreads()) {
    const Combo c = plan_combo(cb, ragged, B, H, S);
    int32_t* lst = plan_list(s, cb, ragged, B, H);
    int n = 0;
    int32_t tot = 0;
    for (int i = c.s0; i < c.s0 + c.nslots; ++i)
      if (s.pool[i] == c.pool && s.items[i] > 0) {
        lst[n++] = i;
        s.start[i] = tot;
        tot += s.items[i];
      }
    s.cb_n[cb] = n;
    s.cb_tot[cb] = tot;
    const int nc = c.nc;
    int ns = nc;
    if (c.pool >= 1) {
      const int usable = nc < free_from - c.c0 ? nc : free_from - c.c0;
      if (usable >= (nc + 1) / 2) ns = usable;  // never squeeze a group onto a few CTAs
    }
    s.cb_ns[cb] = ns;
  }
  x.sync();
  {  // even cut points of every combo, in parallel
    const int nc1 = (ragged ? B * S : S) + 1;
    for (int e = x.tid(); e < 3 * groups * nc1; e += x.nthreads()) {
      const int cb = e / nc1, sp = e - cb * nc1;
      const int32_t tot = s.cb_tot[cb], ns = s.cb_ns[cb];
      int32_t v = 0;
      if (tot > 0) {
        const int32_t base = tot / ns, rem = tot % ns;
        v = sp <= ns ? sp * base + (sp < rem ? sp : rem) : tot;
      }
      s.cuts[e] = v;
    }
  }
  x.sync();
  for (int cb = x.tid(); cb < 3 * groups; cb += x.nthreads()) {
    const int32_t tot = s.cb_tot[cb], ns = s.cb_ns[cb];
    if (tot == 0) continue;
    const int32_t* lst = plan_list(s, cb, ragged, B, H);
    const int n = s.cb_n[cb];
    int32_t* cut = plan_cuts(s, cb, ragged, B, S);
    const int32_t base = tot / ns;
    // snap a cut within one item of a slot boundary onto it
    int32_t hb = 0;
    for (int h = 0; h + 1 < n; ++h) {
      hb += s.items[lst[h]];
      int sp = hb / (base > 1 ? base : 1);
      sp = sp < 1 ? 1 : sp;
      sp = sp > ns - 1 ? ns - 1 : sp;
      while (sp > 1 && cut[sp] > hb) --sp;
      while (sp < ns - 1 && cut[sp + 1] <= hb) ++sp;
      for (int cc = sp; cc <= sp + 1 && cc < ns; ++cc) {
        const int32_t dlt = cut[cc] > hb ? cut[cc] - hb : hb - cut[cc];
        if (cc >= 1 && dlt <= 1 && cut[cc - 1] < hb && hb < cut[cc + 1]) cut[cc] = hb;
      }
    }
  }
  x.sync();
  LYC_PLAN_STAMP(3);
  // ---- phase 3: cells of each slot; units per cell
  for (int i = x.tid(); i < BH; i += x.nthreads()) {
    s.nunits[i] = 0;
    s.first_sp[i] = 0;
    if (s.items[i] <= 0) continue;
    const int grp = ragged ? 0 : i / H;
    const int cb = grp * 3 + s.pool[i];
    const int nc = plan_combo(cb, ragged, B, H, S).nc;
    const int32_t* cut = plan_cuts(s, cb, ragged, B, S);
    const int f = plan_cell_of(cut, nc, s.start[i]);
    const int e = plan_cell_of(cut, nc, s.start[i] + s.items[i] - 1);
    s.first_sp[i] = f;
    s.nunits[i] = e - f + 1;
  }
  for (int c = x.tid(); c < cells; c += x.nthreads()) {
    const int grp = ragged ? 0 : c / S;
    int cnt = 0;
    for (int pool = 0; pool < 3; ++pool) {
      const int cb = grp * 3 + pool;
      const Combo cm = plan_combo(cb, ragged, B, H, S);
      const int sp = c - cm.c0;
      const int32_t* cut = plan_cuts(s, cb, ragged, B, S);
      if (s.cb_tot[cb] == 0 || cut[sp] >= cut[sp + 1]) continue;
      const int32_t* lst = plan_list(s, cb, ragged, B, H);
      for (int j = 0; j < s.cb_n[cb]; ++j) {
        const int32_t a = s.start[lst[j]], z = a + s.items[lst[j]];
        if (z > cut[sp] && a < cut[sp + 1]) ++cnt;
      }
    }
    s.ccount[c] = cnt;
  }
  x.sync();
  for (int i = x.tid(); i < BH; i += x.nthreads()) {
    s.first_unit[i] = s.nunits[i];
    s.mrg[i] = s.nunits[i] > 1 ? G : 0;
  }
  for (int c = x.tid(); c < cells; c += x.nthreads()) s.coff[c] = s.ccount[c];
  x.sync();
  LYC_PLAN_STAMP(5);
  const int32_t n_parts = plan_scan(x, s.first_unit, BH, misc);
  const int32_t n_merge = plan_scan(x, s.mrg, BH, misc);
  const int32_t n_units = plan_scan(x, s.coff, cells, misc);
  (void)n_parts;
  LYC_PLAN_STAMP(4);
  // ---- phase 4: slots, units, unit_slots, split_off, merges
  for (int i = x.tid(); i < BH; i += x.nthreads()) o.slots[i] = plan_slot(in, l, i, s, nret, none, blocks);
  for (int c = x.tid(); c < cells; c += x.nthreads()) {
    const int grp = ragged ? 0 : c / S;
    int u = s.coff[c];
    o.split_off[c] = u;
    for (int pool = 0; pool < 3; ++pool) {
      const int cb = grp * 3 + pool;
      const Combo cm = plan_combo(cb, ragged, B, H, S);
      const int sp = c - cm.c0;
      const int32_t* cut = plan_cuts(s, cb, ragged, B, S);
      if (s.cb_tot[cb] == 0 || cut[sp] >= cut[sp + 1]) continue;
      const int32_t* lst = plan_list(s, cb, ragged, B, H);
      for (int j = 0; j < s.cb_n[cb]; ++j) {
        const int i = lst[j];
        const int32_t a = s.start[i], z = a + s.items[i];
        if (!(z > cut[sp] && a < cut[sp + 1])) continue;
        LycUnit un;
        un.slot = i;
        un.begin = (cut[sp] > a ? cut[sp] : a) - a;
        un.end = (cut[sp + 1] < z ? cut[sp + 1] : z) - a;
        un.hls = sp - s.first_sp[i];
        o.units[u] = un;
        o.unit_slots[u] = plan_slot(in, l, i, s, nret, none, blocks);
        ++u;
      }
    }
  }
  for (int i = x.tid(); i < BH; i += x.nthreads())
    if (s.nunits[i] > 1)
      for (int j = 0; j < G; ++j) {
        LycMergeTask t;
        t.slot = i;
        t.j = j;
        t.first_unit = s.first_unit[i];
        t.n_units = s.nunits[i];
        t.q_row = (i / H) * H * G + (i % H) * G;
        t.pad = 0;
        o.merges[s.mrg[i] + j] = t;
      }
  LYC_PLAN_STAMP(6);
  if (x.tid() == 0) {
    o.split_off[cells] = n_units;
    *o.n_merges = n_merge;
    *o.n_sel = none ? 0 : B * nret;
    if (o.n_units) *o.n_units = n_units;
    if (l == 0) {
      const int32_t mx = misc[PM_SEQMAX];
      in.hdr->seq_len = mx;
      in.hdr->n_keys = blocks ? (mx + in.bs - 1) / in.bs : mx;
      in.hdr->k_sel = (int32_t)plan_budget(in, mx);
      in.hdr->status = 0;
      in.hdr->bad_item = -1;
    }
  }
}

#if defined(__CUDACC__)
// One CTA executes plan_layer (the step kernel's in-kernel re-plan).
struct DevX {
  __device__ int tid() const { return threadIdx.x; }
  __device__ int nthreads() const { return blockDim.x; }
  __device__ void sync() const { __syncthreads(); }
  // block-wide exclusive scan of a[0, n) in place (tmp: >= 33 ints of smem)
  __device__ int32_t scan(int32_t* a, int n, int32_t* tmp) const {
    const int T = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int per = (n + T - 1) / T;
    const int lo = min(n, t * per), hi = min(n, lo + per);
    int32_t sum = 0;
    for (int i = lo; i < hi; ++i) sum += a[i];
    int32_t v = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v += y;
    }
    if (lane == 31) tmp[w] = v;
    __syncthreads();
    if (t == 0) {
      int32_t run = 0;
      for (int i = 0; i < T / 32; ++i) {
        const int32_t x = tmp[i];
        tmp[i] = run;
        run += x;
      }
      tmp[32] = run;
    }
    __syncthreads();
    int32_t run = tmp[w] + v - sum;
    for (int i = lo; i < hi; ++i) {
      const int32_t x = a[i];
      a[i] = run;
      run += x;
    }
    const int32_t total = tmp[32];
    __syncthreads();
    return total;
  }
};

// The writable outputs of layer l from its (fixed) descriptor.
__device__ __forceinline__ PlanOut plan_out_of(LycLayerDesc* d) {
  PlanOut o;
  o.slots = const_cast<LycSlot*>(d->slots);
  o.units = const_cast<LycUnit*>(d->units);
  o.unit_slots = const_cast<LycSlot*>(d->unit_slots);
  o.split_off = const_cast<int32_t*>(d->split_off);
  o.merges = const_cast<LycMergeTask*>(d->merges);
  o.sel_rows = const_cast<int32_t*>(d->sel_rows);
  o.sel_n = const_cast<int32_t*>(d->sel_n);
  o.sel_k = const_cast<int32_t*>(d->sel_k);
  o.n_merges = &d->n_merges;
  o.n_sel = &d->n_sel;
  o.n_units = nullptr;
  return o;
}
#endif

// Sequential host execution of plan_layer (the planner self-test).
struct HostX {
  LYC_HD int tid() const { return 0; }
  LYC_HD int nthreads() const { return 1; }
  LYC_HD void sync() const {}
  LYC_HD int32_t scan(int32_t* a, int n, int32_t*) const {
    int32_t run = 0;
    for (int i = 0; i < n; ++i) {
      const int32_t v = a[i];
      a[i] = run;
      run += v;
    }
    return run;
  }
};

}  // namespace lyc
