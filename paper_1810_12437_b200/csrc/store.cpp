// Host-side builder of the pattern-only tiled store (see store.h).
//
// Reference semantics kept: the CSR invariants checked here are those of
// SparseDesignMatrix._validate (pkg/src/priorcg/sparse.py:94-117); the dense
// intercept column is the one hstack_dense_columns prepends (sparse.py:314-341).
#include "store.h"

#include <algorithm>
#include <array>
#include <cstring>
#include <numeric>
#include <string>

namespace pcgs {

namespace {

constexpr int64_t kPieceMaxVec = 256;  // CSC pieces: at most 8 warp iterations

std::vector<int64_t> make_slabs(int64_t len, int64_t slab_max) {
  std::vector<int64_t> lo;
  int64_t ns = len <= 0 ? 1 : (len + slab_max - 1) / slab_max;
  int64_t per = (len + ns - 1) / ns;
  per = (per + 15) / 16 * 16;  // keep slab starts 128-byte aligned in doubles
  if (per > slab_max) per = slab_max;
  for (int64_t s = 0; s <= ns; ++s) lo.push_back(std::min<int64_t>(s * per, std::max<int64_t>(len, 0)));
  // drop empty trailing slabs (possible after rounding)
  while (lo.size() > 2 && lo[lo.size() - 2] == lo.back()) lo.pop_back();
  return lo;
}

// Writes segments of one slab into a pass, packing them into bundles and
// permuting indices for bank balance.
class Emitter {
 public:
  Emitter(PassHost& P, uint16_t sentinel) : P_(P), sent_(sentinel) {}
  ~Emitter() { flush(); }

  void add(uint32_t seg, const uint16_t* d, int64_t len) {
    int64_t nv = len == 0 ? 1 : (len + kVecIdx - 1) / kVecIdx;
    if (!pend_.empty() && (seg != last_seg_ + 1 || pend_vec_ + nv > 32)) flush();
    last_seg_ = seg;
    if (nv > 32) {
      flush();
      emit_long(seg, d, len, nv);
      return;
    }
    pend_.push_back({seg, std::vector<uint16_t>(d, d + len), (int)nv});
    pend_vec_ += (int)nv;
    if (pend_vec_ == 32) flush();
  }

  void flush() {
    if (pend_.empty()) return;
    const uint32_t off = (uint32_t)(P_.idx.size() / kVecIdx);
    const int nvec = pend_vec_;
    P_.idx.resize(P_.idx.size() + (size_t)nvec * kVecIdx, sent_);
    uint16_t* out = P_.idx.data() + (size_t)off * kVecIdx;
    uint32_t mask = 0;
    int lane = 0;
    // counts[slot][half][bank pair]
    std::array<std::array<std::array<uint16_t, 16>, 2>, 8> cnt{};
    for (auto& s : pend_) {
      mask |= 1u << lane;
      // deal the segment's indices round-robin over its lanes, bank-sorted,
      // so each lane gets a spread of banks
      std::vector<uint16_t>& v = s.idx;
      std::stable_sort(v.begin(), v.end(), [](uint16_t a, uint16_t b) { return (a & 15) < (b & 15); });
      std::vector<std::vector<uint16_t>> per(s.nv);
      for (size_t t = 0; t < v.size(); ++t) per[t % s.nv].push_back(v[t]);
      for (int q = 0; q < s.nv; ++q, ++lane) {
        const int h = lane >> 4;
        bool used[8] = {false, false, false, false, false, false, false, false};
        for (uint16_t ix : per[q]) {
          const int b = ix & 15;
          int best = -1;
          for (int k = 0; k < 8; ++k)
            if (!used[k] && (best < 0 || cnt[k][h][b] < cnt[best][h][b])) best = k;
          used[best] = true;
          cnt[best][h][b]++;
          out[lane * kVecIdx + best] = ix;
        }
      }
    }
    Bundle B{off, pend_.front().seg, mask, (uint32_t)nvec};
    P_.bundles.push_back(B);
    pend_.clear();
    pend_vec_ = 0;
  }

 private:
  struct Pend {
    uint32_t seg;
    std::vector<uint16_t> idx;
    int nv;
  };

  void emit_long(uint32_t seg, const uint16_t* d, int64_t len, int64_t nv) {
    const uint32_t off = (uint32_t)(P_.idx.size() / kVecIdx);
    P_.idx.resize(P_.idx.size() + (size_t)nv * kVecIdx, sent_);
    uint16_t* out = P_.idx.data() + (size_t)off * kVecIdx;
    std::array<std::vector<uint16_t>, 16> bucket;
    for (int64_t t = 0; t < len; ++t) bucket[d[t] & 15].push_back(d[t]);
    int64_t remaining = len;
    const int64_t iters = (nv + 31) / 32;
    std::array<int, 16> order;
    for (int64_t it = 0; it < iters && remaining > 0; ++it) {
      for (int k = 0; k < kVecIdx && remaining > 0; ++k) {
        for (int h = 0; h < 2 && remaining > 0; ++h) {
          // lanes of this half-warp group that own a vector
          int64_t v0 = it * 32 + h * 16;
          int m = (int)std::max<int64_t>(0, std::min<int64_t>(16, nv - v0));
          if (m == 0) continue;
          std::iota(order.begin(), order.end(), 0);
          std::sort(order.begin(), order.end(),
                    [&](int a, int b) { return bucket[a].size() > bucket[b].size(); });
          int take = (int)std::min<int64_t>(m, remaining);
          for (int q = 0; q < take; ++q) {
            int b = order[q % 16];
            if (bucket[b].empty()) {  // fewer non-empty buckets than lanes: reuse the largest
              for (int r = 0; r < 16; ++r)
                if (!bucket[order[r]].empty()) { b = order[r]; break; }
            }
            out[(v0 + q) * kVecIdx + k] = bucket[b].back();
            bucket[b].pop_back();
            --remaining;
          }
        }
      }
    }
    Bundle B{off, seg, 0u, (uint32_t)nv | kLongFlag};
    P_.bundles.push_back(B);
  }

  PassHost& P_;
  uint16_t sent_;
  std::vector<Pend> pend_;
  int pend_vec_ = 0;
  uint32_t last_seg_ = 0xffffffffu;
};

inline int64_t bundle_weight(const Bundle& b) { return (int64_t)(b.nvec & ~kLongFlag) + 2; }

// Static CTA/warp plan (deterministic: every output is produced by exactly one
// warp and every partial sum is reduced in a fixed order).
void plan_pass(PassHost& P, const std::vector<int64_t>& slab_b, int G) {
  const int ns = P.nslab;
  std::vector<int64_t> pre(P.bundles.size() + 1, 0);
  for (size_t b = 0; b < P.bundles.size(); ++b) pre[b + 1] = pre[b] + bundle_weight(P.bundles[b]);
  auto cut = [&](int64_t b0, int64_t b1, int parts, std::vector<int32_t>& outv) {
    // boundaries of `parts` ranges over [b0, b1) with balanced weight
    const int64_t w0 = pre[b0], W = pre[b1] - pre[b0];
    outv.push_back((int32_t)b0);
    for (int q = 1; q < parts; ++q) {
      int64_t target = w0 + (W * q + parts - 1) / parts;
      int64_t b = std::lower_bound(pre.begin() + b0, pre.begin() + b1 + 1, target) - pre.begin();
      b = std::max<int64_t>(b, outv.back());
      b = std::min<int64_t>(b, b1);
      outv.push_back((int32_t)b);
    }
    outv.push_back((int32_t)b1);
  };
  P.tasks.clear();
  P.warp_split.clear();
  P.cta_task_ptr.assign(G + 1, 0);
  auto add_task = [&](int slab, int32_t b0, int32_t b1) {
    Task t{slab, b0, b1, (int32_t)P.warp_split.size()};
    std::vector<int32_t> ws;
    cut(b0, b1, kWarps, ws);
    P.warp_split.insert(P.warp_split.end(), ws.begin(), ws.end());
    P.tasks.push_back(t);
  };
  if (ns <= G) {
    // proportional CTA allocation per slab (largest remainder, at least one each)
    std::vector<int64_t> sw(ns);
    int64_t W = 0;
    for (int s = 0; s < ns; ++s) { sw[s] = pre[slab_b[s + 1]] - pre[slab_b[s]] + 1; W += sw[s]; }
    std::vector<int> cnt(ns, 1);
    int left = G - ns;
    std::vector<std::pair<double, int>> rem;
    for (int s = 0; s < ns; ++s) {
      double ideal = (double)sw[s] / (double)W * G - 1.0;
      int add = std::max(0, (int)ideal);
      add = std::min(add, left);
      cnt[s] += add;
      left -= add;
      rem.push_back({ideal - add, s});
    }
    std::sort(rem.begin(), rem.end(), [](auto& a, auto& b) { return a.first > b.first; });
    for (size_t q = 0; left > 0; q = (q + 1) % rem.size(), --left) cnt[rem[q].second]++;
    int c = 0;
    for (int s = 0; s < ns; ++s) {
      std::vector<int32_t> cb;
      cut(slab_b[s], slab_b[s + 1], cnt[s], cb);
      for (int q = 0; q < cnt[s]; ++q, ++c) {
        P.cta_task_ptr[c] = (int32_t)P.tasks.size();
        add_task(s, cb[q], cb[q + 1]);
        P.cta_task_ptr[c + 1] = (int32_t)P.tasks.size();
      }
    }
  } else {
    std::vector<int32_t> cb;
    cut(0, (int64_t)P.bundles.size(), G, cb);
    for (int c = 0; c < G; ++c) {
      P.cta_task_ptr[c] = (int32_t)P.tasks.size();
      for (int s = 0; s < ns; ++s) {
        int64_t a = std::max<int64_t>(cb[c], slab_b[s]), b = std::min<int64_t>(cb[c + 1], slab_b[s + 1]);
        if (a < b) add_task(s, (int32_t)a, (int32_t)b);
      }
      P.cta_task_ptr[c + 1] = (int32_t)P.tasks.size();
    }
  }
}

}  // namespace

std::string build_design(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx,
                         int intercept, int slab_max, int G, DesignHost& D) {
  if (n < 1) return "design must have at least one row";
  if (p < 0) return "negative column count";
  if (row_ptr[0] != 0) return "row_ptr endpoints must be 0 and nnz";
  for (int64_t i = 0; i < n; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return "row_ptr must be nondecreasing";
  const int64_t nnz = row_ptr[n];
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      if (col_idx[k] < 0 || col_idx[k] >= p) return "col_idx entry out of range";
      if (k > row_ptr[i] && col_idx[k] <= col_idx[k - 1])
        return "col_idx must be strictly increasing within each row";
    }
  }
  const int64_t hard_max = 28672 - 16;  // doubles of shared memory per slab (+ sentinel)
  int64_t smax = slab_max > 0 ? std::min<int64_t>(slab_max, hard_max) : hard_max;
  if (smax < 16) smax = 16;
  D.n = n;
  D.p = p;
  D.intercept = intercept ? 1 : 0;
  D.p_total = p + D.intercept;
  D.nnz = nnz;
  D.slab_max = (int)smax;

  // ---------------- CSR pass: segments = (column slab, row) ----------------
  {
    PassHost& P = D.csr;
    P.slab_lo = make_slabs(p, smax);
    P.nslab = (int)P.slab_lo.size() - 1;
    P.nseg = (int64_t)P.nslab * n;
    std::vector<int64_t> cursor(row_ptr, row_ptr + n);
    std::vector<int64_t> slab_b(P.nslab + 1, 0);
    std::vector<uint16_t> buf;
    for (int s = 0; s < P.nslab; ++s) {
      slab_b[s] = (int64_t)P.bundles.size();
      const int64_t lo = P.slab_lo[s], hi = P.slab_lo[s + 1];
      Emitter E(P, (uint16_t)(hi - lo));
      for (int64_t i = 0; i < n; ++i) {
        buf.clear();
        int64_t k = cursor[i];
        while (k < row_ptr[i + 1] && col_idx[k] < hi) buf.push_back((uint16_t)(col_idx[k++] - lo));
        cursor[i] = k;
        E.add((uint32_t)(s * n + i), buf.data(), (int64_t)buf.size());
      }
      E.flush();
    }
    slab_b[P.nslab] = (int64_t)P.bundles.size();
    plan_pass(P, slab_b, G);
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
    P.slab_lo = make_slabs(n, smax);
    P.nslab = (int)P.slab_lo.size() - 1;
    P.piece_ptr.assign((size_t)P.nslab * (pt + 1), 0);
    std::vector<int64_t> cursor(col_ptr.begin(), col_ptr.end() - 1);
    std::vector<int64_t> slab_b(P.nslab + 1, 0);
    std::vector<uint16_t> buf;
    uint32_t piece = 0;
    for (int s = 0; s < P.nslab; ++s) {
      slab_b[s] = (int64_t)P.bundles.size();
      const int64_t lo = P.slab_lo[s], hi = P.slab_lo[s + 1];
      Emitter E(P, (uint16_t)(hi - lo));
      for (int64_t j = 0; j < pt; ++j) {
        P.piece_ptr[(size_t)s * (pt + 1) + j] = (int32_t)piece;
        buf.clear();
        if (j < p) {
          int64_t k = cursor[j];
          while (k < col_ptr[j + 1] && row_idx[k] < hi) buf.push_back((uint16_t)(row_idx[k++] - lo));
          cursor[j] = k;
        } else {
          for (int64_t i = lo; i < hi; ++i) buf.push_back((uint16_t)(i - lo));
        }
        const int64_t len = (int64_t)buf.size();
        for (int64_t a = 0; a < len; a += kPieceMaxVec * kVecIdx) {
          int64_t m = std::min<int64_t>(kPieceMaxVec * kVecIdx, len - a);
          E.add(piece++, buf.data() + a, m);
        }
      }
      P.piece_ptr[(size_t)s * (pt + 1) + pt] = (int32_t)piece;
      E.flush();
    }
    slab_b[P.nslab] = (int64_t)P.bundles.size();
    P.nseg = piece;
    plan_pass(P, slab_b, G);
  }
  return "";
}

}  // namespace pcgs
