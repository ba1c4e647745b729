// Host-side builder of the sliced store for batched chains (see sliced.h).
//
// Reference semantics kept: the CSR invariants are SparseDesignMatrix._validate
// (pkg/src/priorcg/sparse.py:94-117); the products are those of
// PrecisionOperator.apply (sampler.py:53-58) per chain.
#include "sliced.h"

#include <algorithm>
#include <array>
#include <numeric>

namespace pcgs {

int sliced_slab_max(int R) {
  // 28,600 doubles (223 KB) of shared memory for the slab + sentinel row,
  // leaving room for the batched PCG kernel's static shared memory
  const int elems = 28600 / R - 1;
  return elems / 16 * 16;
}

namespace {

struct Piece {
  uint32_t out;     // output row / column
  uint32_t id;      // global piece id (output-major)
  uint64_t off;     // into the slab buffer
  uint32_t len;     // indices
  uint32_t nv;      // vectors
};

struct SlabPieces {
  std::vector<uint16_t> buf;
  std::vector<Piece> pieces;
  uint16_t sentinel = 0;
};

// Indices of one piece still to be placed, bucketed by bank group (index mod H).
struct Pool {
  std::array<std::vector<uint16_t>, 16> b;
  int H = 1;
  uint32_t remaining = 0;
  void load(const uint16_t* d, uint32_t len, int h) {
    H = h;
    for (auto& v : b) v.clear();
    for (uint32_t t = 0; t < len; ++t) b[d[t] % H].push_back(d[t]);
    remaining = len;
  }
  // an index whose group is least used in this half-warp so far (largest bucket on ties)
  int pick(const int* mult) {
    if (remaining == 0) return -1;
    int best = -1;
    for (int k = 0; k < H; ++k) {
      if (b[k].empty()) continue;
      if (best < 0 || mult[k] < mult[best] || (mult[k] == mult[best] && b[k].size() > b[best].size())) best = k;
    }
    const int v = b[best].back();
    b[best].pop_back();
    --remaining;
    return v;
  }
};

// extra wavefronts of one half-warp LDS.64: the largest number of distinct
// indices sharing a bank group (index mod H), minus one
int half_extra(const int* ix, int n, int H) {
  int mult[16] = {};
  int worst = 0;
  for (int i = 0; i < n; ++i) {
    bool seen = false;
    for (int j = 0; j < i; ++j) seen |= ix[j] == ix[i];
    if (!seen) worst = std::max(worst, ++mult[ix[i] % H]);
  }
  return worst > 0 ? worst - 1 : 0;
}

// The slots of each shared-memory wavefront group (see sliced.h): slots whose
// lanes read the same chunk of their rows at one instruction.
std::vector<std::vector<int>> slot_groups(int R) {
  const int C = sliced_cpl(R), LS = sliced_lanes_per_slot(R), NS = sliced_slots(R);
  std::vector<std::vector<int>> g;
  if (C == 1) {  // 64-bit loads: half-warps of 16 / R consecutive slots
    for (int h = 0; h < 2; ++h) {
      g.emplace_back();
      for (int s = h * NS / 2; s < (h + 1) * NS / 2; ++s) g.back().push_back(s);
    }
    return g;
  }
  const int spq = 8 / LS, classes = C / 2;  // slots per quarter-warp, chunk classes
  for (int q = 0; q < 4; ++q)
    for (int b = 0; b < classes; ++b) {
      g.emplace_back();
      for (int m = b; m < spq; m += classes) g.back().push_back(q * spq + m);
    }
  return g;
}

// Lays out slices [a, b) of a slab (pieces already sorted) into the pass.
void emit_slices(SPassHost& P, SlabPieces& S, const std::vector<uint32_t>& sl_first, size_t a, size_t b, int R) {
  const int NS = sliced_slots(R), H = 16 / R;
  const std::vector<std::vector<int>> groups = slot_groups(R);
  std::vector<Pool> pools(NS);
  for (size_t q = a; q < b; ++q) {
    const uint32_t p0 = sl_first[q], p1 = sl_first[q + 1];
    const uint32_t L = S.pieces[p0].nv;
    SliceDesc D{(uint32_t)(P.idx.size() / kVecIdx), L};
    P.slices.push_back(D);
    for (int s = 0; s < NS; ++s) {
      const uint32_t pi = p0 + (uint32_t)s;
      if (pi < p1) {
        const Piece& pc = S.pieces[pi];
        P.piece.push_back(pc.id);
        pools[s].load(S.buf.data() + pc.off, pc.len, H);
        P.pad_vectors += L - pc.nv;
      } else {
        P.piece.push_back(0xffffffffu);
        pools[s].load(nullptr, 0, H);
        P.pad_vectors += L;
      }
    }
    P.idx.resize(P.idx.size() + (size_t)L * NS * kVecIdx, S.sentinel);
    uint16_t* out = P.idx.data() + (size_t)D.v0 * kVecIdx;
    for (uint32_t t = 0; t < L; ++t) {
      for (int k = 0; k < kVecIdx; ++k) {
        for (const auto& grp : groups) {
          int mult[16] = {};
          int g[16];
          int ng = 0;
          bool pad_seen = false, any = false;
          for (const int s : grp) {
            const int ix = pools[s].pick(mult);
            if (ix < 0) {  // the sentinel is in place (one broadcast address)
              if (!pad_seen) {
                pad_seen = true;
                ++mult[S.sentinel % H];
                g[ng++] = S.sentinel;
              }
              continue;
            }
            any = true;
            ++mult[ix % H];
            out[((size_t)t * NS + s) * kVecIdx + k] = (uint16_t)ix;
            g[ng++] = ix;
          }
          if (!any) continue;
          ++P.lds_groups;
          P.lds_excess += half_extra(g, ng, H);
        }
      }
    }
  }
}

// Balanced cut of items [a, b) with prefix costs `pre` into `parts` ranges.
void cut_ranges(const std::vector<uint64_t>& pre, size_t a, size_t b, int parts, std::vector<size_t>& outv) {
  outv.clear();
  outv.push_back(a);
  const uint64_t w0 = pre[a], W = pre[b] - pre[a];
  for (int q = 1; q < parts; ++q) {
    const uint64_t target = w0 + (W * q + parts / 2) / parts;
    size_t s = std::lower_bound(pre.begin() + a, pre.begin() + b + 1, target) - pre.begin();
    if (s > a && s <= b && target - pre[s - 1] < pre[s] - target) --s;
    s = std::max(s, outv.back());
    s = std::min(s, b);
    outv.push_back(s);
  }
  outv.push_back(b);
}

// Builds one pass from its per-slab pieces: sort, slice, plan over G CTAs, place.
void plan_pass(SPassHost& P, std::vector<SlabPieces>& slabs, int R, int G) {
  const int NS = sliced_slots(R);
  const int ns = (int)slabs.size();
  // cost of a slice: its vectors plus a per-piece epilogue charge (in vectors)
  constexpr uint64_t kEpi = 2;
  std::vector<std::vector<uint32_t>> first(ns);
  std::vector<std::vector<uint64_t>> pre(ns);
  std::vector<uint64_t> sw(ns);
  uint64_t W = 0;
  for (int s = 0; s < ns; ++s) {
    auto& pcs = slabs[s].pieces;
    std::stable_sort(pcs.begin(), pcs.end(), [](const Piece& x, const Piece& y) { return x.nv > y.nv; });
    auto& f = first[s];
    for (size_t i = 0; i < pcs.size(); i += NS) f.push_back((uint32_t)i);
    const size_t nsl = f.size();
    f.push_back((uint32_t)pcs.size());
    auto& pr = pre[s];
    pr.assign(nsl + 1, 0);
    for (size_t q = 0; q < nsl; ++q)
      pr[q + 1] = pr[q] + (uint64_t)pcs[f[q]].nv * NS + kEpi * (f[q + 1] - f[q]);
    sw[s] = pr.back();
    W += sw[s];
  }
  P.cta_task_ptr.assign(G + 1, 0);
  auto emit_task = [&](int s, size_t a, size_t b) {
    Task t{s, (int32_t)(P.warp_slices.size() / 2)};
    std::vector<size_t> wc;
    cut_ranges(pre[s], a, b, kSWarps, wc);
    for (int w = 0; w < kSWarps; ++w) {
      const uint32_t s0 = (uint32_t)P.slices.size();
      emit_slices(P, slabs[s], first[s], wc[w], wc[w + 1], R);
      P.warp_slices.push_back(s0);
      P.warp_slices.push_back((uint32_t)P.slices.size());
    }
    P.tasks.push_back(t);
  };
  if (ns <= G) {
    std::vector<int> cnt(ns, 1);
    int left = G - ns;
    std::vector<std::pair<double, int>> rem;
    for (int s = 0; s < ns; ++s) {
      const double ideal = W ? (double)sw[s] / (double)W * G - 1.0 : 0.0;
      const int add = std::min(std::max(0, (int)ideal), left);
      cnt[s] += add;
      left -= add;
      rem.push_back({ideal - add, s});
    }
    std::sort(rem.begin(), rem.end(), [](auto& x, auto& y) { return x.first > y.first; });
    for (size_t q = 0; left > 0; q = (q + 1) % rem.size(), --left) cnt[rem[q].second]++;
    int c = 0;
    for (int s = 0; s < ns; ++s) {
      std::vector<size_t> cb;
      cut_ranges(pre[s], 0, first[s].size() - 1, cnt[s], cb);
      for (int q = 0; q < cnt[s]; ++q, ++c) {
        P.cta_task_ptr[c] = (int32_t)P.tasks.size();
        emit_task(s, cb[q], cb[q + 1]);
        P.cta_task_ptr[c + 1] = (int32_t)P.tasks.size();
      }
      std::vector<uint16_t>().swap(slabs[s].buf);
    }
  } else {
    for (int c = 0; c < G; ++c) {
      P.cta_task_ptr[c] = (int32_t)P.tasks.size();
      const int a = (int)((int64_t)ns * c / G), b = (int)((int64_t)ns * (c + 1) / G);
      for (int s = a; s < b; ++s) {
        emit_task(s, 0, first[s].size() - 1);
        std::vector<uint16_t>().swap(slabs[s].buf);
      }
      P.cta_task_ptr[c + 1] = (int32_t)P.tasks.size();
    }
  }
}

std::vector<int64_t> slab_bounds(int64_t len, int64_t smax) {
  std::vector<int64_t> lo;
  const int64_t ns = len <= 0 ? 1 : (len + smax - 1) / smax;
  int64_t per = (len + ns - 1) / ns;
  per = std::min<int64_t>((per + 15) / 16 * 16, smax);
  for (int64_t s = 0; s <= ns; ++s) lo.push_back(std::min<int64_t>(s * per, std::max<int64_t>(len, 0)));
  while (lo.size() > 2 && lo[lo.size() - 2] == lo.back()) lo.pop_back();
  return lo;
}

// Generic pass: outputs 0..n_out-1, gathered coordinates 0..n_in-1 cut into
// slabs; `entries(o, fn)` calls fn(g) for the gathered coordinates of output o
// in increasing order.
template <class Entries>
void build_pass(SPassHost& P, int64_t n_out, int64_t n_in, int64_t smax, int R, int G, Entries&& entries) {
  P.slab_lo = slab_bounds(n_in, smax);
  P.nslab = (int)P.slab_lo.size() - 1;
  const int64_t PMI = (int64_t)kSlicedPieceMax * kVecIdx;
  // pieces per (output, slab), output-major numbering
  std::vector<SlabPieces> slabs(P.nslab);
  for (int s = 0; s < P.nslab; ++s) slabs[s].sentinel = (uint16_t)(P.slab_lo[s + 1] - P.slab_lo[s]);
  P.out_ptr.assign((size_t)n_out + 1, 0);
  std::vector<uint16_t> tmp;
  uint32_t id = 0;
  for (int64_t o = 0; o < n_out; ++o) {
    P.out_ptr[o] = id;
    int s = 0;
    tmp.clear();
    auto flush = [&]() {
      for (int64_t a = 0; a < (int64_t)tmp.size(); a += PMI) {
        const int64_t m = std::min<int64_t>(PMI, (int64_t)tmp.size() - a);
        SlabPieces& S = slabs[s];
        Piece pc{(uint32_t)o, id++, S.buf.size(), (uint32_t)m, (uint32_t)((m + kVecIdx - 1) / kVecIdx)};
        S.buf.insert(S.buf.end(), tmp.begin() + a, tmp.begin() + a + m);
        S.pieces.push_back(pc);
      }
      tmp.clear();
    };
    entries(o, [&](int64_t g) {
      while (g >= P.slab_lo[s + 1]) {
        flush();
        ++s;
      }
      tmp.push_back((uint16_t)(g - P.slab_lo[s]));
    });
    flush();
  }
  P.out_ptr[n_out] = id;
  P.npiece = id;
  plan_pass(P, slabs, R, G);
}

}  // namespace

std::string build_sliced(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx, int intercept,
                         int R, int slab_max, int G, SlicedHost& H) {
  if (R != 1 && R != 2 && R != 4 && R != 8) return "nchains must be 1, 2, 4 or 8";
  {
    std::string err = validate_csr(n, p, row_ptr, col_idx);
    if (!err.empty()) return err;
  }
  const int64_t hard = sliced_slab_max(R);
  int64_t smax = slab_max > 0 ? std::min<int64_t>(slab_max, hard) : hard;
  if (smax < 16) smax = 16;
  H.n = n;
  H.p = p;
  H.intercept = intercept ? 1 : 0;
  H.p_total = p + H.intercept;
  H.nnz = row_ptr[n];
  H.R = R;
  H.slab_max = (int)smax;
  // CSR: outputs = rows, gathered = shrunk columns (the intercept is added in the row combine)
  build_pass(H.csr, n, p, smax, R, G, [&](int64_t i, auto&& fn) {
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) fn(col_idx[k]);
  });
  // CSC: outputs = internal columns (shrunk 0..p-1, intercept p = every row), gathered = rows
  {
    std::vector<int64_t> col_ptr(p + 1, 0);
    for (int64_t k = 0; k < H.nnz; ++k) col_ptr[col_idx[k] + 1]++;
    for (int64_t j = 0; j < p; ++j) col_ptr[j + 1] += col_ptr[j];
    std::vector<int32_t> row_idx(H.nnz);
    {
      std::vector<int64_t> fill(col_ptr.begin(), col_ptr.end() - 1);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) row_idx[fill[col_idx[k]]++] = (int32_t)i;
    }
    build_pass(H.csc, H.p_total, n, smax, R, G, [&](int64_t j, auto&& fn) {
      if (j < p) {
        for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k) fn(row_idx[k]);
      } else {
        for (int64_t i = 0; i < n; ++i) fn(i);
      }
    });
  }
  return "";
}

std::string verify_sliced(const SlicedHost& H, const int64_t* row_ptr, const int32_t* col_idx) {
  const int NS = sliced_slots(H.R);
  auto walk = [&](const SPassHost& P, int64_t n_out, std::vector<std::vector<int32_t>>& got) -> std::string {
    std::vector<int32_t> owner((size_t)P.npiece, -1);
    for (int64_t o = 0; o < n_out; ++o)
      for (int64_t q = P.out_ptr[o]; q < P.out_ptr[o + 1]; ++q) owner[q] = (int32_t)o;
    std::vector<uint8_t> seen((size_t)P.npiece, 0);
    for (size_t t = 0; t < P.tasks.size(); ++t) {
      const Task& T = P.tasks[t];
      const int64_t lo = P.slab_lo[T.slab], hi = P.slab_lo[T.slab + 1];
      const uint16_t sent = (uint16_t)(hi - lo);
      for (int w = 0; w < kSWarps; ++w) {
        const uint32_t s0 = P.warp_slices[2 * (T.warp0 + w)], s1 = P.warp_slices[2 * (T.warp0 + w) + 1];
        for (uint32_t q = s0; q < s1; ++q) {
          const SliceDesc& D = P.slices[q];
          for (int s = 0; s < NS; ++s) {
            const uint32_t pid = P.piece[(size_t)q * NS + s];
            for (uint32_t v = 0; v < D.len; ++v)
              for (int e = 0; e < kVecIdx; ++e) {
                const uint16_t ix = P.idx[((size_t)D.v0 + (size_t)v * NS + s) * kVecIdx + e];
                if (ix == sent) continue;
                if (ix > sent) return "index beyond slab";
                if (pid == 0xffffffffu) return "index in an idle slot";
                if (pid >= (uint32_t)P.npiece || owner[pid] < 0) return "bad piece id";
                got[owner[pid]].push_back((int32_t)(lo + ix));
              }
            if (pid != 0xffffffffu) {
              if (seen[pid]) return "piece walked twice";
              seen[pid] = 1;
            }
          }
        }
      }
    }
    for (int64_t q = 0; q < P.npiece; ++q)
      if (!seen[q]) return "piece " + std::to_string(q) + " never walked";
    return "";
  };
  const int64_t n = H.n, p = H.p, pt = H.p_total;
  std::vector<std::vector<int32_t>> rows(n), cols(pt);
  std::string err = walk(H.csr, n, rows);
  if (!err.empty()) return "csr: " + err;
  for (int64_t i = 0; i < n; ++i) {
    std::sort(rows[i].begin(), rows[i].end());
    if ((int64_t)rows[i].size() != row_ptr[i + 1] - row_ptr[i] || !std::equal(rows[i].begin(), rows[i].end(), col_idx + row_ptr[i]))
      return "csr: row " + std::to_string(i) + " differs";
  }
  err = walk(H.csc, pt, cols);
  if (!err.empty()) return "csc: " + err;
  std::vector<std::vector<int32_t>> want(pt);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) want[col_idx[k]].push_back((int32_t)i);
    if (H.intercept) want[p].push_back((int32_t)i);
  }
  for (int64_t j = 0; j < pt; ++j) {
    std::sort(cols[j].begin(), cols[j].end());
    if (cols[j] != want[j]) return "csc: column " + std::to_string(j) + " differs";
  }
  return "";
}

}  // namespace pcgs
