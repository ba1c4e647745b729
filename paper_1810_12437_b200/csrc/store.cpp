// Host-side builder of the pattern-only tiled store (see store.h).
//
// Reference semantics kept: the CSR invariants checked here are those of
// SparseDesignMatrix._validate (pkg/src/priorcg/sparse.py:94-117); the dense
// intercept column is the one hstack_dense_columns prepends (sparse.py:314-341).
#include "store.h"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

namespace pcgs {

namespace {

// Layout of the pass streams: grouped (default) or the flat stream with
// per-block segment masks (PCGS_LAYOUT=flat), see store.h.
bool layout_grouped() {
#if PCGS_FLAT_WALK
  const char* e = getenv("PCGS_LAYOUT");
  return !(e && std::string(e) == "flat");
#else
  return true;
#endif
}

// CSC pieces: at most this many vectors (load balance); PCGS_PIECE_MAX overrides (tuning)
int64_t piece_max_vec() {
  const char* e = getenv("PCGS_PIECE_MAX");
  return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)256;
}

std::vector<int64_t> make_slabs(int64_t len, int64_t slab_max) {
  std::vector<int64_t> lo;
  int64_t ns = len <= 0 ? 1 : (len + slab_max - 1) / slab_max;
  int64_t per = (len + ns - 1) / ns;
  per = (per + 15) / 16 * 16;  // keep slab starts 128-byte aligned in doubles
  if (per > slab_max) per = slab_max;
  for (int64_t s = 0; s <= ns; ++s) lo.push_back(std::min<int64_t>(s * per, std::max<int64_t>(len, 0)));
  while (lo.size() > 2 && lo[lo.size() - 2] == lo.back()) lo.pop_back();
  return lo;
}

struct Seg {
  uint32_t id;
  uint64_t off;  // into the slab buffer
  uint32_t len;  // real indices
  uint32_t nv;   // vectors (>= 1)
};

struct SlabSegs {
  std::vector<uint16_t> buf;
  std::vector<Seg> segs;
  uint16_t sentinel = 0;
  std::vector<uint16_t> rep_of;  // slab index -> its replica's index (0xffff: none), grouped layout
  void add(uint32_t id, const uint16_t* d, uint32_t len) {
    Seg s{id, buf.size(), len, len == 0 ? 1u : (len + kVecIdx - 1) / kVecIdx};
    buf.insert(buf.end(), d, d + len);
    segs.push_back(s);
  }
};

// Indices of one segment still to be placed, bucketed by shared-memory bank pair.
//
// A 64-bit LDS costs, per half-warp, the largest number of distinct addresses
// sharing a bank pair (index mod 16) -- measured on B200 with
// tools/microbench/bank_rule.cu.  Taking the fullest buckets first is close to
// the bound for a segment that fills whole half-warps: its most popular pair
// holds max_b c_b indices but each group takes it once, so max_b c_b - groups
// extra wavefronts are unavoidable (~20 % for an 800-index row).
struct Pool {
  std::array<std::vector<uint16_t>, 16> b;  // entries with one address, by bank pair
  // entries with a replica: two addresses (store.h, REPLICAS); each id sits in
  // the lists of both its bank pairs and is removed lazily
  std::vector<std::array<uint16_t, 2>> flex;
  std::vector<uint8_t> taken;
  std::array<std::vector<uint32_t>, 16> fl;
  std::array<uint32_t, 16> nfl{};
  uint32_t remaining = 0;
  void load(const uint16_t* d, uint32_t len, const std::vector<uint16_t>* rep_of = nullptr) {
    for (auto& v : b) v.clear();
    for (auto& v : fl) v.clear();
    flex.clear();
    taken.clear();
    nfl.fill(0);
    for (uint32_t t = 0; t < len; ++t) {
      const uint16_t ix = d[t];
      const uint16_t rp = rep_of && !rep_of->empty() ? (*rep_of)[ix] : (uint16_t)0xffff;
      if (rp == 0xffff || ((rp ^ ix) & 15) == 0) {
        b[ix & 15].push_back(ix);
      } else {
        const uint32_t id = (uint32_t)flex.size();
        flex.push_back({ix, rp});
        taken.push_back(0);
        fl[ix & 15].push_back(id);
        fl[rp & 15].push_back(id);
        ++nfl[ix & 15];
        ++nfl[rp & 15];
      }
    }
    remaining = len;
  }
  int take(int k) {
    --remaining;
    if (!b[k].empty()) {
      const int v = b[k].back();
      b[k].pop_back();
      return v;
    }
    auto& L = fl[k];
    while (taken[L.back()]) L.pop_back();
    const uint32_t id = L.back();
    L.pop_back();
    taken[id] = 1;
    --nfl[flex[id][0] & 15];
    --nfl[flex[id][1] & 15];
    return (flex[id][0] & 15) == k ? flex[id][0] : flex[id][1];
  }
  // an index whose bank pair has the lowest multiplicity in the group so far;
  // among those a single-address entry (largest bucket) before a two-address
  // one (they stay free to fill the gaps later); -1 when empty
  int pick(const uint8_t* mult) {
    if (remaining == 0) return -1;
    int best = -1;
    uint64_t best_key = 0;
    for (int k = 0; k < 16; ++k) {
      const bool fixed = !b[k].empty();
      if (!fixed && nfl[k] == 0) continue;
      // smaller is better: multiplicity, then fixed before flexible, then the fuller bucket
      const uint64_t key = ((uint64_t)mult[k] << 40) | ((uint64_t)(fixed ? 0 : 1) << 32) |
                           (uint64_t)(0xffffffffu - (fixed ? (uint32_t)b[k].size() : nfl[k]));
      if (best < 0 || key < best_key) {
        best = k;
        best_key = key;
      }
    }
    return take(best);
  }
};

// Wavefronts one (slot, half-warp) group costs beyond the first: the largest
// number of distinct addresses sharing a bank pair, minus one.
int group_extra(const uint16_t* ix, int n) {
  int mult[16] = {};
  int worst = 0;
  for (int i = 0; i < n; ++i) {
    bool seen = false;
    for (int j = 0; j < i; ++j) seen |= ix[j] == ix[i];
    if (!seen) worst = std::max(worst, ++mult[ix[i] & 15]);
  }
  return worst > 0 ? worst - 1 : 0;
}

// Appends one warp range (segments [s0, s1) of slab S) to the pass.
void emit_warp(PassHost& P, const SlabSegs& S, size_t s0, size_t s1, std::vector<Pool>& pools) {
  WarpRange R{};
  R.v0 = (uint32_t)(P.idx.size() / kVecIdx);
  R.blk0 = (uint32_t)P.blocks.size();
  uint64_t nvec = 0;
  for (size_t s = s0; s < s1; ++s) nvec += S.segs[s].nv;
  R.nvec = (uint32_t)nvec;
  P.warps.push_back(R);
  if (nvec == 0) return;
  P.idx.resize(P.idx.size() + nvec * kVecIdx, S.sentinel);
  uint16_t* out = P.idx.data() + (size_t)R.v0 * kVecIdx;
  const uint64_t nb = (nvec + 31) / 32;
  // per-lane segment for the current block; pools keyed by lane-segment slot
  size_t seg = s0;
  uint32_t in_seg = 0;  // vectors of `seg` already laid out
  int lane_seg[32];
  int lane_pool[32];
  int next_pool = 0;
  int seg_pool = -1;
  for (uint64_t k = 0; k < nb; ++k) {
    uint32_t mask = 0;
    uint32_t first_id = 0;
    bool have_first = false;
    // assign lanes
    for (int l = 0; l < 32; ++l) {
      const uint64_t v = k * 32 + l;
      if (v >= nvec) { lane_seg[l] = -1; lane_pool[l] = -1; continue; }
      while (in_seg >= S.segs[seg].nv) { ++seg; in_seg = 0; seg_pool = -1; }
      if (in_seg == 0) {
        mask |= 1u << l;
        if (!have_first) { first_id = S.segs[seg].id; have_first = true; }
      }
      if (seg_pool < 0) {
        seg_pool = next_pool;
        next_pool = (next_pool + 1) % (int)pools.size();
        pools[seg_pool].load(S.buf.data() + S.segs[seg].off, S.segs[seg].len);
      }
      lane_seg[l] = (int)seg;
      lane_pool[l] = seg_pool;
      ++in_seg;
    }
    P.blocks.push_back(BlockDesc{first_id, mask});
    // bank-balanced placement: group = (slot, half-warp)
    for (int slot = 0; slot < kVecIdx; ++slot) {
      for (int h = 0; h < 2; ++h) {
        const int l0 = h * 16;
        bool any = false;
        for (int l = l0; l < l0 + 16; ++l) any |= lane_seg[l] >= 0;
        if (!any) continue;
        uint16_t g[16];
        int ng = 0;
        {
          uint8_t mult[16] = {};
          bool pad_seen = false;
          for (int l = l0; l < l0 + 16; ++l) {
            if (lane_seg[l] < 0) continue;
            const int ix = pools[lane_pool[l]].pick(mult);
            if (ix < 0) {  // pad: the sentinel is already in place (one broadcast address)
              if (!pad_seen) { pad_seen = true; ++mult[S.sentinel & 15]; g[ng++] = S.sentinel; }
              continue;
            }
            ++mult[ix & 15];
            out[(k * 32 + l) * kVecIdx + slot] = (uint16_t)ix;
            g[ng++] = (uint16_t)ix;
          }
        }
        ++P.lds_groups;
        P.lds_conflict_excess += group_extra(g, ng);
      }
    }
  }
}


// ---------------------------------------------------------------------------
// Grouped layout (store.h): width classes, slices, warp dealing, placement.
// ---------------------------------------------------------------------------
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// log2 of the lane-group width of a segment of nv vectors: wide groups for
// long segments (the round-up to W vectors stays a few percent), one lane for
// the shortest ones.
int width_log(uint32_t nv) {
  // swept on the config-2 PCG iteration (tools/gpu_ab_grouped.sh): 80/40/12
  // with 128-vector pieces 73.3 us, 128/64/16 71.5, with 256-vector pieces 70.8
  static const int w8 = env_int("PCGS_GW8", 128), w4 = env_int("PCGS_GW4", 64), w2 = env_int("PCGS_GW2", 16);
  return nv >= (uint32_t)w8 ? 3 : nv >= (uint32_t)w4 ? 2 : nv >= (uint32_t)w2 ? 1 : 0;
}

// vector slots a segment occupies in its slice, in 1/16 vector units, plus its
// share of the slice close
uint64_t group_cost16(uint32_t nv) {
  static const int close = env_int("PCGS_G_CLOSE16", 16);
  const uint32_t W = 1u << width_log(nv);
  return 16ull * ((nv + W - 1) / W * W) + (uint64_t)close;
}

long long g_hist[6 * 20];
long long* g_dbg_hist = nullptr;  // PCGS_STORE_STATS: [lw][decile of the slice]{gathers, excess}

struct Slice {
  uint32_t first, count;  // items [first, first + count)
  uint32_t T;             // steps
  uint8_t lw;
};

// Lays out segments [s0, s1) of slab S as one CTA task: P.nranges warp ranges.
void emit_task_grouped(PassHost& P, const SlabSegs& S, size_t s0, size_t s1, std::vector<Pool>& pools) {
  const int NR = P.nranges;
  struct Item {
    uint32_t seg, nv;
    uint8_t lw;
  };
  std::vector<Item> items;
  items.reserve(s1 - s0);
  for (size_t s = s0; s < s1; ++s) items.push_back(Item{(uint32_t)s, S.segs[s].nv, (uint8_t)width_log(S.segs[s].nv)});
  // a task with fewer slices than warps (small designs, many CTAs) widens its
  // groups, up to the whole warp, while a segment still fills its lanes
  for (int round = 0; round < 5; ++round) {
    size_t nslices = 0;
    uint32_t cnt[6] = {};
    for (const Item& it : items) ++cnt[it.lw];
    for (int lw = 0; lw < 6; ++lw) nslices += (cnt[lw] + (32u >> lw) - 1) / (32u >> lw);
    if (nslices >= (size_t)NR) break;
    bool any = false;
    for (Item& it : items)
      if (it.lw < 5 && (2u << it.lw) <= it.nv) {
        ++it.lw;
        any = true;
      }
    if (!any) break;
  }
  std::stable_sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    return a.lw != b.lw ? a.lw > b.lw : a.nv > b.nv;
  });
  std::vector<Slice> slices;
  for (size_t i = 0; i < items.size();) {
    const uint8_t lw = items[i].lw;
    const uint32_t NG = 32u >> lw, W = 1u << lw;
    size_t j = i;
    while (j < items.size() && items[j].lw == lw && j - i < NG) ++j;
    slices.push_back(Slice{(uint32_t)i, (uint32_t)(j - i), (items[i].nv + W - 1) / W, lw});
    i = j;
  }
  // deal slices to warps, longest first, each to the least loaded warp
  std::vector<uint32_t> order(slices.size());
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return slices[a].T > slices[b].T; });
  std::vector<std::vector<uint32_t>> mine(NR);
  {
    static const int close = env_int("PCGS_G_SLICE_COST", 1);
    uint64_t load[kWarps] = {};  // NR <= kWarps
    for (uint32_t q : order) {
      int w = 0;
      for (int c = 1; c < NR; ++c)
        if (load[c] < load[w]) w = c;
      mine[w].push_back(q);
      load[w] += slices[q].T + (uint64_t)close;
    }
  }
  for (int w = 0; w < NR; ++w) {
    WarpRange R{};
    R.v0 = (uint32_t)(P.idx.size() / kVecIdx);
    R.blk0 = (uint32_t)P.blocks.size();
    R.pad = (uint32_t)mine[w].size();
    uint64_t nvec = 0;
    for (uint32_t q : mine[w]) nvec += 32ull * slices[q].T;
    R.nvec = (uint32_t)nvec;
    P.warps.push_back(R);
    if (nvec == 0) continue;
    P.idx.resize(P.idx.size() + nvec * kVecIdx, S.sentinel);
    uint16_t* out = P.idx.data() + (size_t)R.v0 * kVecIdx;
    for (uint32_t q : mine[w]) {
      const Slice& L = slices[q];
      const uint32_t NG = 32u >> L.lw, W = 1u << L.lw;
      P.blocks.push_back(BlockDesc{(uint32_t)P.ids.size(), L.T | ((uint32_t)L.lw << 24)});
      uint64_t real_vec = 0;
      for (uint32_t g = 0; g < NG; ++g) {
        if (g < L.count) {
          const Seg& sg = S.segs[items[L.first + g].seg];
          P.ids.push_back(sg.id);
          pools[g].load(S.buf.data() + sg.off, sg.len, &S.rep_of);
          real_vec += sg.nv;
        } else {
          P.ids.push_back(0xffffffffu);
          pools[g].load(nullptr, 0);
        }
      }
      P.pad_vectors += 32ll * L.T - (int64_t)real_vec;
      // bank-balanced placement: one LDS.64 per (step, slot); group = half-warp
      for (uint32_t t = 0; t < L.T; ++t) {
        for (int slot = 0; slot < kVecIdx; ++slot) {
          for (int h = 0; h < 2; ++h) {
            uint16_t g16[16];
            int ng = 0;
            uint8_t mult[16] = {};
            bool pad_seen = false;
            // the half-warp's groups pick in turn (one lane of each per
            // round, the starting group rotating), so no group is left the
            // residues the others did not want
            const int ngh = L.lw >= 4 ? 1 : 16 >> L.lw;  // groups per half-warp
            const int rot = (int)((t * kVecIdx + slot) % ngh);
            for (int r = 0; r < 16; ++r) {
              const int gi = (r + rot) % ngh, ki = r / ngh;
              const int l = 16 * h + (L.lw >= 4 ? r : gi * (int)W + ki);
              const int ix = pools[l >> L.lw].pick(mult);
              if (ix < 0) {  // the sentinel is already in place (one broadcast address)
                if (!pad_seen) {
                  pad_seen = true;
                  ++mult[S.sentinel & 15];
                  g16[ng++] = S.sentinel;
                }
                continue;
              }
              ++mult[ix & 15];
              out[((size_t)t * 32 + l) * kVecIdx + slot] = (uint16_t)ix;
              g16[ng++] = (uint16_t)ix;
            }
            ++P.lds_groups;
            const int ex = group_extra(g16, ng);
            P.lds_conflict_excess += ex;
            if (g_dbg_hist) {
              const int dec = (int)((t * kVecIdx + slot) * 10 / (L.T * kVecIdx));
              g_dbg_hist[L.lw * 20 + dec * 2] += 1;
              g_dbg_hist[L.lw * 20 + dec * 2 + 1] += ex;
            }
          }
        }
      }
      out += (size_t)L.T * 32 * kVecIdx;
    }
  }
}


// REPLICAS (store.h): the shared-memory area behind a slab's sentinel holds
// second copies of the slab's most gathered entries at a different bank pair,
// so the placement below can move an occurrence off an over-subscribed bank
// pair.  Fills `rep_of` of every slab and the pass's rep_ptr / rep_src.
void choose_replicas(PassHost& P, std::vector<SlabSegs>& slabs, int64_t area, bool grouped) {
  P.rep_ptr.assign(1, 0);
  // off by default: measured at config 2 the replicas cut the predicted (and
  // ncu-counted) bank conflicts from 16 % to 2 % of the gather wavefronts and
  // the PCG iteration not at all (71.3 vs 71.0 us) -- the passes are bound by
  // the LSU's 16 lanes per cycle, not by the data banks
  const int on = env_int("PCGS_REPLICAS", 0);
  for (SlabSegs& S : slabs) {
    const int64_t len = S.sentinel;
    int64_t K = std::min<int64_t>(area - (len + 1), 65535 - (len + 1));
    K = std::min<int64_t>(K, len);
    if (!grouped || !on || K < 16) {
      P.rep_ptr.push_back((int32_t)P.rep_src.size());
      continue;
    }
    std::vector<uint32_t> cnt((size_t)len, 0);
    for (uint16_t ix : S.buf) ++cnt[ix];
    std::vector<uint32_t> order((size_t)len);
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cnt[a] > cnt[b]; });
    std::array<std::vector<uint32_t>, 16> free_;
    for (int64_t k = K - 1; k >= 0; --k) free_[(len + 1 + k) & 15].push_back((uint32_t)k);
    S.rep_of.assign((size_t)len, (uint16_t)0xffff);
    std::vector<uint16_t> src((size_t)K, (uint16_t)len);  // unused slots copy the sentinel's zero
    int64_t placed = 0;
    for (int64_t q = 0; q < len && placed < K; ++q) {
      const uint32_t j = order[q];
      if (cnt[j] == 0) break;
      // the replica's bank pair: a pseudo-random offset from the original's, so
      // the two-address entries link all 16 pairs (a fixed offset would only
      // trade occurrences inside 8 rigid pair classes)
      const uint32_t h = (j * 2654435761u) >> 16;
      for (int d = 0; d < 16; ++d) {
        const int r = (int)((j + 1 + h % 15 + d) & 15);
        if (r == (int)(j & 15) || free_[r].empty()) continue;
        const uint32_t slot = free_[r].back();
        free_[r].pop_back();
        S.rep_of[j] = (uint16_t)(len + 1 + slot);
        src[slot] = (uint16_t)j;
        ++placed;
        break;
      }
    }
    P.rep_src.insert(P.rep_src.end(), src.begin(), src.end());
    P.rep_ptr.push_back((int32_t)P.rep_src.size());
  }
}

// Balanced cut of segments [a, b) into `parts` ranges by vector count.
void cut(const std::vector<uint64_t>& pre, size_t a, size_t b, int parts, std::vector<size_t>& outv) {
  outv.clear();
  outv.push_back(a);
  const uint64_t w0 = pre[a], W = pre[b] - pre[a];
  for (int q = 1; q < parts; ++q) {
    const uint64_t target = w0 + (W * q + parts / 2) / parts;
    size_t s = std::lower_bound(pre.begin() + a, pre.begin() + b + 1, target) - pre.begin();
    // choose the closer of s-1 / s
    if (s > a && s <= b && target - pre[s - 1] < pre[s] - target) --s;
    s = std::max(s, outv.back());
    s = std::min(s, b);
    outv.push_back(s);
  }
  outv.push_back(b);
}

// Balancing cost model, in 1/16 vector units: one unit per vector, plus a
// charge per segment for its close (the warp reduction that ends it and its
// epilogue).  Reductions are paid per 32-vector block that contains segment
// starts, so short segments sharing a block share that cost: the charge is
// emit + block * min(len, 32) / 32.  Defaults from sweeps of the PCG iteration
// time at config 2 (tools/segw_sweep.sh); PCGS_SEG_WEIGHT (CSR),
// PCGS_SEG_WEIGHT_CSC / PCGS_SEG_EMIT override them for tuning experiments.
double env_or(const char* name, double dflt) {
  const char* e = getenv(name);
  return e ? atof(e) : dflt;
}

uint64_t seg_charge16(uint32_t nv, bool csc) {
  // CSR 40, CSC 64: swept on the PCG iteration after the 2-op gather change
  // (24/24 82.4 us, 32/48 82.0, 40/64 81.6, 32/96 82.1)
  static const double block = env_or("PCGS_SEG_WEIGHT", 40.0);
  static const double block_csc = env_or("PCGS_SEG_WEIGHT_CSC", 64.0);
  static const double emit = env_or("PCGS_SEG_EMIT", 0.0);
  const double frac = nv >= 32 ? 1.0 : (double)nv / 32.0;
  return (uint64_t)((emit + (csc ? block_csc : block) * frac) * 16.0 + 0.5);
}

void plan_and_emit(PassHost& P, std::vector<SlabSegs>& slabs, int G, bool csc, int64_t area) {
  const int ns = (int)slabs.size();
  P.cta_task_ptr.assign(G + 1, 0);
  std::vector<Pool> pools(40);
  const bool grouped = layout_grouped();
  P.grouped = grouped ? 1 : 0;
  choose_replicas(P, slabs, area, grouped);
  std::vector<std::vector<uint64_t>> pre(ns);
  std::vector<uint64_t> sw(ns);
  uint64_t W = 0;
  for (int s = 0; s < ns; ++s) {
    auto& pr = pre[s];
    pr.assign(slabs[s].segs.size() + 1, 0);
    // cost model for balancing: a vector plus a per-segment charge (segment
    // closes: reductions, epilogue), in 1/16 vector units
    for (size_t q = 0; q < slabs[s].segs.size(); ++q)
      pr[q + 1] = pr[q] + (grouped ? group_cost16(slabs[s].segs[q].nv)
                                   : 16u * slabs[s].segs[q].nv + seg_charge16(slabs[s].segs[q].nv, csc));
    sw[s] = pr.back();
    W += sw[s];
  }
  auto emit_task = [&](int s, size_t a, size_t b) {
    Task t{s, (int32_t)P.warps.size()};
    if (grouped) {
      emit_task_grouped(P, slabs[s], a, b, pools);
    } else {
      std::vector<size_t> wc;
      cut(pre[s], a, b, P.nranges, wc);
      for (int w = 0; w < P.nranges; ++w) emit_warp(P, slabs[s], wc[w], wc[w + 1], pools);
    }
    P.tasks.push_back(t);
  };
  if (ns <= G) {
    std::vector<int> cnt(ns, 1);
    int left = G - ns;
    std::vector<std::pair<double, int>> rem;
    for (int s = 0; s < ns; ++s) {
      const double ideal = W ? (double)sw[s] / (double)W * G - 1.0 : 0.0;
      int add = std::min(std::max(0, (int)ideal), left);
      cnt[s] += add;
      left -= add;
      rem.push_back({ideal - add, s});
    }
    std::sort(rem.begin(), rem.end(), [](auto& x, auto& y) { return x.first > y.first; });
    for (size_t q = 0; left > 0; q = (q + 1) % rem.size(), --left) cnt[rem[q].second]++;
    int c = 0;
    for (int s = 0; s < ns; ++s) {
      std::vector<size_t> cb;
      cut(pre[s], 0, slabs[s].segs.size(), cnt[s], cb);
      for (int q = 0; q < cnt[s]; ++q, ++c) {
        P.cta_task_ptr[c] = (int32_t)P.tasks.size();
        emit_task(s, cb[q], cb[q + 1]);
        P.cta_task_ptr[c + 1] = (int32_t)P.tasks.size();
      }
      std::vector<uint16_t>().swap(slabs[s].buf);
    }
  } else {
    // more slabs than CTAs: contiguous groups of slabs per CTA
    for (int c = 0; c < G; ++c) {
      P.cta_task_ptr[c] = (int32_t)P.tasks.size();
      const int a = (int)((int64_t)ns * c / G), b = (int)((int64_t)ns * (c + 1) / G);
      for (int s = a; s < b; ++s) {
        emit_task(s, 0, slabs[s].segs.size());
        std::vector<uint16_t>().swap(slabs[s].buf);
      }
      P.cta_task_ptr[c + 1] = (int32_t)P.tasks.size();
    }
  }
}

}  // namespace

std::string validate_csr(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx) {
  if (n < 1) return "design must have at least one row";
  if (p < 0) return "negative column count";
  if (row_ptr[0] != 0) return "row_ptr endpoints must be 0 and nnz";
  for (int64_t i = 0; i < n; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return "row_ptr must be nondecreasing";
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      if (col_idx[k] < 0 || col_idx[k] >= p) return "col_idx entry out of range";
      if (k > row_ptr[i] && col_idx[k] <= col_idx[k - 1])
        return "col_idx must be strictly increasing within each row";
    }
  }
  return "";
}

std::string build_design(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx,
                         int intercept, int slab_max, int G, DesignHost& D, int q_dense, int nranges) {
  if (nranges < 1 || nranges > kWarps) return "warp ranges per task must be in [1, 32]";
  D.csr.nranges = D.csc.nranges = nranges;
  if (q_dense < 0 || (q_dense > 0 && intercept)) return "dense columns replace the intercept flag";
  g_dbg_hist = getenv("PCGS_STORE_STATS") ? g_hist : nullptr;
  if (g_dbg_hist) memset(g_hist, 0, sizeof(g_hist));
  {
    std::string err = validate_csr(n, p, row_ptr, col_idx);
    if (!err.empty()) return err;
  }
  const int64_t nnz = row_ptr[n];
  const int64_t hard_max = 22528 - 16;  // doubles per slab (+ sentinel): 176 KB, leaves room for PCG state
  int64_t smax = slab_max > 0 ? std::min<int64_t>(slab_max, hard_max) : hard_max;
  if (smax < 16) smax = 16;
  D.n = n;
  D.p = p;
  D.intercept = intercept ? 1 : 0;
  D.q_dense = q_dense;
  D.p_total = p + D.intercept + q_dense;
  D.nnz = nnz;
  D.slab_max = (int)smax;
  {
    // shared-memory area of the slab vector: the longest slab plus its
    // sentinel, grown by the replica region to what one CTA has left next to
    // the persistent kernels' own-slice state and piece pointers
    const char* cs = getenv("PCGS_CSC_SLAB_MAX");
    const int64_t csc_max = cs ? std::max<int64_t>(16, std::min<int64_t>(smax, atoll(cs))) : smax;
    const std::vector<int64_t> a = make_slabs(p, smax), b = make_slabs(n, csc_max);
    int64_t maxlen = 0;
    for (size_t q = 0; q + 1 < a.size(); ++q) maxlen = std::max(maxlen, a[q + 1] - a[q]);
    for (size_t q = 0; q + 1 < b.size(); ++q) maxlen = std::max(maxlen, b[q + 1] - b[q]);
    const int64_t base = (maxlen + 1 + 15) / 16 * 16;
    const int64_t chunk = (D.p_total + G - 1) / G;
    const int64_t budget =
        (227 * 1024 - 4096 - chunk * 64 - (int64_t)(b.size() - 1) * (chunk + 1) * 4) / 8 / 16 * 16;
    D.slab_area = (int)(env_int("PCGS_REPLICAS", 0) ? std::max(base, std::min<int64_t>(budget, 65520)) : base);
  }

  // ---------------- CSR pass: segments = (column slab, row) ----------------
  {
    PassHost& P = D.csr;
    P.slab_lo = make_slabs(p, smax);
    P.nslab = (int)P.slab_lo.size() - 1;
    P.nseg = (int64_t)P.nslab * n;
    std::vector<int64_t> cursor(row_ptr, row_ptr + n);
    std::vector<SlabSegs> slabs(P.nslab);
    std::vector<uint16_t> tmp;
    for (int s = 0; s < P.nslab; ++s) {
      const int64_t lo = P.slab_lo[s], hi = P.slab_lo[s + 1];
      SlabSegs& S = slabs[s];
      S.sentinel = (uint16_t)(hi - lo);
      for (int64_t i = 0; i < n; ++i) {
        tmp.clear();
        int64_t k = cursor[i];
        while (k < row_ptr[i + 1] && col_idx[k] < hi) tmp.push_back((uint16_t)(col_idx[k++] - lo));
        cursor[i] = k;
        S.add((uint32_t)(s * n + i), tmp.data(), (uint32_t)tmp.size());
      }
    }
    plan_and_emit(P, slabs, G, false, D.slab_area);
  }

  // ------------- CSC pass: segments = pieces of (row slab, column) -------------
  {
    PassHost& P = D.csc;
    const int64_t pt = D.p_total;  // internal column layout: shrunk 0..p-1, intercept p
    std::vector<int64_t> col_ptr(p + 1, 0);
    for (int64_t k = 0; k < nnz; ++k) col_ptr[col_idx[k] + 1]++;
    for (int64_t j = 0; j < p; ++j) col_ptr[j + 1] += col_ptr[j];
    std::vector<int32_t> row_idx(nnz);
    {
      std::vector<int64_t> fill(col_ptr.begin(), col_ptr.end() - 1);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) row_idx[fill[col_idx[k]]++] = (int32_t)i;
    }
    // PCGS_CSC_SLAB_MAX caps the row slabs separately (tuning experiments)
    const char* cs = getenv("PCGS_CSC_SLAB_MAX");
    P.slab_lo = make_slabs(n, cs ? std::max<int64_t>(16, std::min<int64_t>(smax, atoll(cs))) : smax);
    P.nslab = (int)P.slab_lo.size() - 1;
    P.piece_ptr.assign((size_t)P.nslab * (pt + 1), 0);
    std::vector<int64_t> cursor(col_ptr.begin(), col_ptr.end() - 1);
    std::vector<SlabSegs> slabs(P.nslab);
    std::vector<uint16_t> tmp;
    uint32_t piece = 0;
    for (int s = 0; s < P.nslab; ++s) {
      const int64_t lo = P.slab_lo[s], hi = P.slab_lo[s + 1];
      SlabSegs& S = slabs[s];
      S.sentinel = (uint16_t)(hi - lo);
      for (int64_t j = 0; j < pt; ++j) {
        P.piece_ptr[(size_t)s * (pt + 1) + j] = (int32_t)piece;
        tmp.clear();
        if (j < p) {
          int64_t k = cursor[j];
          while (k < col_ptr[j + 1] && row_idx[k] < hi) tmp.push_back((uint16_t)(row_idx[k++] - lo));
          cursor[j] = k;
        } else if (j < p + D.intercept) {
          for (int64_t i = lo; i < hi; ++i) tmp.push_back((uint16_t)(i - lo));
        }  // dense columns (j >= p + intercept): no pattern pieces
        const int64_t len = (int64_t)tmp.size();
        for (int64_t a = 0; a < len; a += piece_max_vec() * kVecIdx) {
          const int64_t m = std::min<int64_t>(piece_max_vec() * kVecIdx, len - a);
          S.add(piece++, tmp.data() + a, (uint32_t)m);
        }
      }
      P.piece_ptr[(size_t)s * (pt + 1) + pt] = (int32_t)piece;
    }
    P.nseg = piece;
    {
      // column-major slots: column j's pieces of slab 0, then slab 1, ...
      P.col_piece_ptr.assign((size_t)pt + 1, 0);
      for (int s = 0; s < P.nslab; ++s)
        for (int64_t j = 0; j < pt; ++j)
          P.col_piece_ptr[j + 1] += P.piece_ptr[(size_t)s * (pt + 1) + j + 1] - P.piece_ptr[(size_t)s * (pt + 1) + j];
      for (int64_t j = 0; j < pt; ++j) P.col_piece_ptr[j + 1] += P.col_piece_ptr[j];
      P.piece_perm.assign((size_t)piece, 0);
      std::vector<int32_t> next(P.col_piece_ptr.begin(), P.col_piece_ptr.end() - 1);
      for (int s = 0; s < P.nslab; ++s)
        for (int64_t j = 0; j < pt; ++j)
          for (int32_t q = P.piece_ptr[(size_t)s * (pt + 1) + j]; q < P.piece_ptr[(size_t)s * (pt + 1) + j + 1]; ++q)
            P.piece_perm[q] = next[j]++;
    }
    plan_and_emit(P, slabs, G, true, D.slab_area);
  }
  const long long* hist = g_hist;
  if (getenv("PCGS_STORE_STATS")) {
    for (int lw = 0; lw < 6; ++lw) {
      long long tot = 0;
      for (int d = 0; d < 10; ++d) tot += hist[lw * 20 + 2 * d];
      if (!tot) continue;
      fprintf(stderr, "  W=%d excess per gather by slice decile:", 1 << lw);
      for (int d = 0; d < 10; ++d)
        fprintf(stderr, " %.2f", (double)hist[lw * 20 + 2 * d + 1] / (double)std::max(1ll, hist[lw * 20 + 2 * d]));
      fprintf(stderr, "  (%lld gathers)\n", tot);
    }
  }
  if (getenv("PCGS_STORE_STATS"))
    for (const PassHost* P : {&D.csr, &D.csc})
      fprintf(stderr, "pcgs store: %s vectors %zu pad %lld slices/blocks %zu replicas %zu half-warp gathers %lld excess %lld (%.3f)\n",
              P == &D.csr ? "csr" : "csc", P->idx.size() / kVecIdx, (long long)P->pad_vectors, P->blocks.size(),
              P->rep_src.size(),
              (long long)P->lds_groups, (long long)P->lds_conflict_excess,
              (double)P->lds_conflict_excess / (double)std::max<int64_t>(1, P->lds_groups));
  return "";
}

// Rebuilds the pattern from the tiled passes and compares it with the input
// CSR (host-only; used by the CPU test-suite through pcgs_store_selftest).
std::string verify_design(const DesignHost& D, const int64_t* row_ptr, const int32_t* col_idx) {
  const int64_t n = D.n, p = D.p, pt = D.p_total;
  // walk every warp range of a pass, calling f(segment id, index) per real index
  auto walk = [](const PassHost& P, auto&& f) -> std::string {
    for (size_t t = 0; t < P.tasks.size(); ++t) {
      const Task& T = P.tasks[t];
      const int64_t lo = P.slab_lo[T.slab], hi = P.slab_lo[T.slab + 1];
      const uint16_t sent = (uint16_t)(hi - lo);
      for (int w = 0; w < P.nranges; ++w) {
        const WarpRange& R = P.warps[T.warp0 + w];
        if (R.nvec == 0) continue;
        if (P.grouped) {
          if (R.nvec % 32) return std::string("grouped range is not whole blocks");
          uint64_t v = R.v0;
          for (uint32_t q = 0; q < R.pad; ++q) {
            const BlockDesc& B = P.blocks[R.blk0 + q];
            const uint32_t steps = B.mask & 0xffffffu, lw = B.mask >> 24;
            if (lw > 5 || steps == 0) return std::string("bad slice descriptor");
            for (uint32_t t = 0; t < steps; ++t)
              for (int l = 0; l < 32; ++l, ++v) {
                const uint32_t id = P.ids[B.first_id + (l >> lw)];
                for (int e = 0; e < kVecIdx; ++e) {
                  uint16_t ix = P.idx[v * kVecIdx + e];
                  if (ix == sent) continue;
                  if (ix > sent) {  // a replica: back to the entry it copies
                    const int64_t k = (int64_t)ix - sent - 1, r0 = P.rep_ptr[T.slab], r1 = P.rep_ptr[T.slab + 1];
                    if (k >= r1 - r0) return std::string("index beyond slab and replicas");
                    ix = P.rep_src[r0 + k];
                    if (ix >= sent) return std::string("replica of nothing gathered");
                  }
                  if (id == 0xffffffffu) return std::string("index in an empty group");
                  f(T.slab, (int64_t)id, lo + ix);
                }
              }
          }
          if (v != (uint64_t)R.v0 + R.nvec) return std::string("slices do not cover the warp range");
          continue;
        }
        const uint32_t nb = (R.nvec + 31) / 32;
        int64_t seg = -1;
        for (uint32_t k = 0; k < nb; ++k) {
          const BlockDesc& B = P.blocks[R.blk0 + k];
          if (k == 0 && !(B.mask & 1u)) return std::string("warp range does not start a segment");
          int rank = 0;
          for (int l = 0; l < 32; ++l) {
            const uint64_t v = (uint64_t)k * 32 + l;
            if (v >= R.nvec) {
              if (B.mask >> l & 1u) return std::string("segment start beyond range");
              continue;
            }
            if (B.mask >> l & 1u) seg = (int64_t)B.first_id + rank++;
            for (int e = 0; e < kVecIdx; ++e) {
              const uint16_t ix = P.idx[((size_t)R.v0 + v) * kVecIdx + e];
              if (ix == sent) continue;
              if (ix > sent) return std::string("index beyond slab");
              f(T.slab, seg, lo + ix);
            }
          }
        }
      }
    }
    return std::string();
  };
  // grouped layout: every segment id is emitted by exactly one slice group
  for (const PassHost* P : {&D.csr, &D.csc}) {
    if (!P->grouped) continue;
    std::vector<uint8_t> seen((size_t)P->nseg, 0);
    for (uint32_t id : P->ids) {
      if (id == 0xffffffffu) continue;
      if ((int64_t)id >= P->nseg || seen[id]) return std::string("segment id emitted twice or out of range");
      seen[id] = 1;
    }
    for (uint8_t b : seen)
      if (!b) return std::string("segment never emitted");
  }
  // CSR: segment (s, i) -> column set of row i within slab s
  std::vector<std::vector<int32_t>> got_rows(n);
  std::string err = walk(D.csr, [&](int s, int64_t seg, int64_t col) {
    const int64_t i = seg - (int64_t)s * n;
    if (i >= 0 && i < n) got_rows[i].push_back((int32_t)col);
  });
  if (!err.empty()) return "csr: " + err;
  for (int64_t i = 0; i < n; ++i) {
    std::vector<int32_t>& g = got_rows[i];
    std::sort(g.begin(), g.end());
    if ((int64_t)g.size() != row_ptr[i + 1] - row_ptr[i] ||
        !std::equal(g.begin(), g.end(), col_idx + row_ptr[i]))
      return "csr: row " + std::to_string(i) + " differs";
  }
  // CSC: pieces -> column via piece_ptr
  const PassHost& C = D.csc;
  std::vector<int32_t> piece_col(C.nseg, -1);
  for (int s = 0; s < C.nslab; ++s)
    for (int64_t j = 0; j < pt; ++j)
      for (int q = C.piece_ptr[(size_t)s * (pt + 1) + j]; q < C.piece_ptr[(size_t)s * (pt + 1) + j + 1]; ++q)
        piece_col[q] = (int32_t)j;
  {
    std::vector<uint8_t> hit((size_t)C.nseg, 0);
    for (int64_t q = 0; q < C.nseg; ++q) {
      const int32_t slot = C.piece_perm[q];
      if (slot < 0 || slot >= C.nseg || hit[slot]) return "csc: piece_perm is not a permutation";
      hit[slot] = 1;
      const int32_t j = piece_col[q];
      if (j < 0 || slot < C.col_piece_ptr[j] || slot >= C.col_piece_ptr[j + 1])
        return "csc: piece_perm leaves its column's slots";
    }
  }
  std::vector<std::vector<int32_t>> got_cols(pt);
  err = walk(C, [&](int, int64_t seg, int64_t row) {
    if (seg >= 0 && seg < C.nseg && piece_col[seg] >= 0) got_cols[piece_col[seg]].push_back((int32_t)row);
  });
  if (!err.empty()) return "csc: " + err;
  std::vector<std::vector<int32_t>> want(pt);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) want[col_idx[k]].push_back((int32_t)i);
    if (D.intercept) want[p].push_back((int32_t)i);
  }
  for (int64_t j = 0; j < pt; ++j) {
    std::sort(got_cols[j].begin(), got_cols[j].end());
    if (got_cols[j] != want[j]) return "csc: column " + std::to_string(j) + " differs";
  }
  return "";
}

}  // namespace pcgs

// ---------------------------------------------------------------------------
// Native synthetic generator for the large BASELINE configurations (config 5:
// 1.09e9 nonzeros).  Same recipe as synth.binary_design (log-uniform column
// rates, Binomial(n, rate) distinct rows per column) with a xoshiro256** stream
// instead of numpy's PCG64, and a counting-sort transpose straight into CSR.
// Bench/test infrastructure; not on the sampling path.
// ---------------------------------------------------------------------------
#include <cmath>
#include <random>
#include <unordered_set>

namespace pcgs {

namespace {
struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull;
    for (int i = 0; i < 4; ++i) {
      z += 0x9E3779B97F4A7C15ull;
      uint64_t x = z;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
      s[i] = x ^ (x >> 31);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  uint64_t below(uint64_t m) { return (uint64_t)(((__uint128_t)next() * m) >> 64); }
};
}  // namespace

int64_t synth_binary_design(int64_t n, int64_t p, double rate_lo, double rate_hi, uint64_t seed,
                            std::vector<int64_t>& row_ptr, std::vector<int32_t>& col_idx) {
  Xoshiro rng(seed);
  std::mt19937_64 eng(seed ^ 0x5DEECE66Dull);
  std::vector<int64_t> counts(p);
  const double la = std::log(rate_lo), lb = std::log(rate_hi);
  for (int64_t j = 0; j < p; ++j) {
    const double rate = std::exp(la + (lb - la) * rng.uniform());
    std::binomial_distribution<int64_t> bin(n, rate);
    counts[j] = bin(eng);
  }
  int64_t nnz = 0;
  for (int64_t j = 0; j < p; ++j) nnz += counts[j];
  // per-column distinct rows (Floyd's algorithm for sparse columns, a Bernoulli
  // scan with exact count correction for dense ones), counted per row
  std::vector<int32_t> rows_of_col;
  rows_of_col.reserve((size_t)nnz);
  std::vector<int64_t> col_start(p + 1, 0);
  std::vector<uint8_t> mark;
  std::vector<uint64_t> bits;
  for (int64_t j = 0; j < p; ++j) {
    const int64_t k = counts[j];
    col_start[j] = (int64_t)rows_of_col.size();
    if (k == 0) continue;
    if (k * 16 < n) {  // Floyd's algorithm on a reusable bitmap
      if (bits.empty()) bits.assign((size_t)(n + 63) / 64, 0ull);
      const size_t first = rows_of_col.size();
      for (int64_t t = n - k; t < n; ++t) {
        int64_t r = (int64_t)rng.below((uint64_t)t + 1);
        if (bits[r >> 6] >> (r & 63) & 1ull) r = t;
        bits[r >> 6] |= 1ull << (r & 63);
        rows_of_col.push_back((int32_t)r);
      }
      for (size_t q = first; q < rows_of_col.size(); ++q) bits[rows_of_col[q] >> 6] = 0ull;
    } else {
      mark.assign((size_t)n, 0);
      int64_t left = k;
      for (int64_t i = 0; i < n && left > 0; ++i) {  // selection sampling (Knuth S)
        if (rng.uniform() * (double)(n - i) < (double)left) {
          mark[i] = 1;
          --left;
        }
      }
      for (int64_t i = 0; i < n; ++i)
        if (mark[i]) rows_of_col.push_back((int32_t)i);
    }
  }
  col_start[p] = (int64_t)rows_of_col.size();
  row_ptr.assign((size_t)n + 1, 0);
  for (int32_t r : rows_of_col) row_ptr[(size_t)r + 1]++;
  for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
  col_idx.assign((size_t)nnz, 0);
  std::vector<int64_t> fill(row_ptr.begin(), row_ptr.end() - 1);
  for (int64_t j = 0; j < p; ++j)  // columns in order -> rows' columns ascending
    for (int64_t q = col_start[j]; q < col_start[j + 1]; ++q) col_idx[fill[rows_of_col[q]]++] = (int32_t)j;
  return nnz;
}

}  // namespace pcgs
