// Streaming Matrix Market reader/writer for binary designs (see mtx.h).
//
// Restates the file contract scipy.io.mmread/mmwrite implement for the
// reference (matrixio.py:35-58): banner "%%MatrixMarket matrix <format>
// <field> <symmetry>", '%' comment lines, a size line, then 1-based
// coordinate entries (or column-major array values).
#include "mtx.h"

#include <zlib.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <charconv>
#include <cstdlib>
#include <cstring>

namespace pcgs {

namespace {

constexpr size_t kChunk = 8u << 20;

std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

// Line source over a zlib stream (transparent for uncompressed files).
class LineReader {
 public:
  explicit LineReader(gzFile f) : f_(f), buf_(kChunk + 1) {}
  // next line without the newline; false at end of file
  bool next(const char*& b, const char*& e) {
    for (;;) {
      const char* nl = (const char*)memchr(buf_.data() + pos_, '\n', len_ - pos_);
      if (nl) {
        b = buf_.data() + pos_;
        e = nl;
        pos_ = (size_t)(nl - buf_.data()) + 1;
        ++line_;
        if (e > b && e[-1] == '\r') --e;
        return true;
      }
      if (eof_) {
        if (pos_ >= len_) return false;
        b = buf_.data() + pos_;
        e = buf_.data() + len_;
        pos_ = len_;
        ++line_;
        if (e > b && e[-1] == '\r') --e;
        return true;
      }
      // move the partial line to the front and refill
      const size_t rest = len_ - pos_;
      if (rest == buf_.size() - 1) buf_.resize(buf_.size() * 2);  // very long line
      memmove(buf_.data(), buf_.data() + pos_, rest);
      pos_ = 0;
      len_ = rest;
      const int got = gzread(f_, buf_.data() + len_, (unsigned)(buf_.size() - 1 - len_));
      if (got < 0) { error_ = true; eof_ = true; continue; }
      if (got == 0) eof_ = true;
      len_ += (size_t)got;
    }
  }
  int64_t line() const { return line_; }
  bool error() const { return error_; }

 private:
  gzFile f_;
  std::vector<char> buf_;
  size_t pos_ = 0, len_ = 0;
  bool eof_ = false, error_ = false;
  int64_t line_ = 0;
};

inline const char* skip_ws(const char* p, const char* e) {
  while (p < e && (*p == ' ' || *p == '\t')) ++p;
  return p;
}

inline bool parse_i64(const char*& p, const char* e, int64_t& v) {
  p = skip_ws(p, e);
  auto r = std::from_chars(p, e, v);
  if (r.ec != std::errc() || r.ptr == p) return false;
  p = r.ptr;
  return true;
}

// value token -> 0, 1, or -1 (anything else); `bad` gets the token
inline int parse_binary_value(const char*& p, const char* e, std::string& bad) {
  p = skip_ws(p, e);
  const char* t = p;
  while (p < e && *p != ' ' && *p != '\t') ++p;
  if (p == t) return -2;  // missing
  if (p - t == 1 && *t == '1') return 1;
  if (p - t == 1 && *t == '0') return 0;
  std::string tok(t, p);
  char* end = nullptr;
  const double v = strtod(tok.c_str(), &end);
  if (end != tok.c_str() + tok.size()) { bad = tok; return -1; }
  if (v == 1.0) return 1;
  if (v == 0.0) return 0;
  bad = tok;
  return -1;
}

inline bool blank(const char* b, const char* e) { return skip_ws(b, e) == e; }

struct GzCloser {
  gzFile f;
  ~GzCloser() { if (f) gzclose(f); }
};

}  // namespace

int mtx_load(const char* path, MtxPattern& out, std::string& msg) {
  gzFile f = gzopen(path, "rb");
  if (!f) { msg = std::string(path) + ": cannot open (" + strerror(errno) + ")"; return kMtxIo; }
  GzCloser closer{f};
  gzbuffer(f, 1u << 20);
  LineReader L(f);
  const char *b, *e;
  auto where = [&]() { return std::string(path) + ":" + std::to_string(L.line()) + ": "; };
  if (!L.next(b, e)) { msg = std::string(path) + ": empty file"; return kMtxFormat; }
  {
    std::string banner(b, e);
    char w[5][64] = {};
    const int got = sscanf(banner.c_str(), "%63s %63s %63s %63s %63s", w[0], w[1], w[2], w[3], w[4]);
    if (got != 5 || lower(w[0]) != "%%matrixmarket" || lower(w[1]) != "matrix") {
      msg = where() + "not a Matrix Market matrix banner";
      return kMtxFormat;
    }
    const std::string fmt = lower(w[2]), field = lower(w[3]), sym = lower(w[4]);
    if (fmt == "coordinate") out.format = kMtxCoordinate;
    else if (fmt == "array") out.format = kMtxArray;
    else { msg = where() + "unknown format '" + fmt + "'"; return kMtxFormat; }
    if (field == "pattern") out.field = kMtxPattern;
    else if (field == "real" || field == "double") out.field = kMtxReal;
    else if (field == "integer") out.field = kMtxInteger;
    else if (field == "complex") { msg = where() + "complex values: the store is pattern-only"; return kMtxUnsupported; }
    else { msg = where() + "unknown field '" + field + "'"; return kMtxFormat; }
    if (sym == "general") out.symmetry = kMtxGeneral;
    else if (sym == "symmetric") out.symmetry = kMtxSymmetric;
    else if (sym == "skew-symmetric" || sym == "hermitian") {
      msg = where() + sym + " matrices cannot be binary designs";
      return kMtxUnsupported;
    } else { msg = where() + "unknown symmetry '" + sym + "'"; return kMtxFormat; }
    if (out.format == kMtxArray && out.field == kMtxPattern) { msg = where() + "array format needs values"; return kMtxFormat; }
    if (out.format == kMtxArray && out.symmetry != kMtxGeneral) {
      msg = where() + "symmetric array files are not supported";
      return kMtxUnsupported;
    }
  }
  // size line (after comments / blank lines)
  int64_t n = -1, p = -1, ent = -1;
  for (;;) {
    if (!L.next(b, e)) { msg = std::string(path) + ": missing size line"; return kMtxFormat; }
    if (blank(b, e) || *skip_ws(b, e) == '%') continue;
    const char* q = b;
    bool ok = parse_i64(q, e, n) && parse_i64(q, e, p);
    if (ok && out.format == kMtxCoordinate) ok = parse_i64(q, e, ent);
    if (ok && out.format == kMtxArray) ent = n * p;
    if (!ok || !blank(q, e) || n < 0 || p < 0 || ent < 0) { msg = where() + "bad size line"; return kMtxFormat; }
    break;
  }
  if (n > INT32_MAX || p > INT32_MAX) { msg = where() + "dimensions exceed the int32 index range"; return kMtxUnsupported; }
  if (out.symmetry == kMtxSymmetric && n != p) { msg = where() + "symmetric matrix must be square"; return kMtxFormat; }
  out.n = n;
  out.p = p;
  out.entries = ent;
  std::vector<uint64_t> pairs;  // (row << 32) | col, 0-based
  pairs.reserve((size_t)std::min<int64_t>(ent, int64_t(1) << 32) * (out.symmetry == kMtxSymmetric ? 2 : 1));
  std::string bad;
  int64_t seen = 0;
  while (L.next(b, e)) {
    if (blank(b, e) || *skip_ws(b, e) == '%') continue;
    if (seen >= ent) { msg = where() + "more entries than the size line declares (" + std::to_string(ent) + ")"; return kMtxFormat; }
    const char* q = b;
    int64_t i, j;
    int v = 1;
    if (out.format == kMtxCoordinate) {
      if (!parse_i64(q, e, i) || !parse_i64(q, e, j)) { msg = where() + "bad coordinate entry"; return kMtxFormat; }
      if (i < 1 || i > n || j < 1 || j > p) {
        msg = where() + "entry (" + std::to_string(i) + ", " + std::to_string(j) + ") outside " +
              std::to_string(n) + " x " + std::to_string(p);
        return kMtxFormat;
      }
      --i;
      --j;
    } else {
      i = seen % (n ? n : 1);
      j = seen / (n ? n : 1);
    }
    if (out.field != kMtxPattern) {
      v = parse_binary_value(q, e, bad);
      if (v == -2) { msg = where() + "missing value"; return kMtxFormat; }
      if (v == -1) {
        msg = where() + "value '" + bad + "' is not 0/1: the device store is pattern-only (binary designs)";
        return kMtxUnsupported;
      }
    }
    if (!blank(q, e)) { msg = where() + "trailing characters in entry"; return kMtxFormat; }
    ++seen;
    if (v == 0) { ++out.zeros_dropped; continue; }
    pairs.push_back(((uint64_t)i << 32) | (uint64_t)j);
    if (out.symmetry == kMtxSymmetric && i != j) pairs.push_back(((uint64_t)j << 32) | (uint64_t)i);
  }
  if (L.error()) { msg = std::string(path) + ": read error (corrupt gzip stream?)"; return kMtxIo; }
  if (seen != ent) {
    msg = std::string(path) + ": truncated: " + std::to_string(seen) + " of " + std::to_string(ent) + " entries";
    return kMtxFormat;
  }
  // counting sort by row, then sort each row's columns and reject duplicates
  out.row_ptr.assign((size_t)n + 1, 0);
  for (uint64_t x : pairs) ++out.row_ptr[(x >> 32) + 1];
  for (int64_t r = 0; r < n; ++r) out.row_ptr[r + 1] += out.row_ptr[r];
  out.col_idx.resize(pairs.size());
  {
    std::vector<int64_t> cur(out.row_ptr.begin(), out.row_ptr.end() - 1);
    for (uint64_t x : pairs) out.col_idx[cur[x >> 32]++] = (int32_t)(x & 0xffffffffu);
  }
  std::vector<uint64_t>().swap(pairs);
  for (int64_t r = 0; r < n; ++r) {
    int32_t* a = out.col_idx.data() + out.row_ptr[r];
    int32_t* z = out.col_idx.data() + out.row_ptr[r + 1];
    if (!std::is_sorted(a, z)) std::sort(a, z);
    for (int32_t* t = a; t + 1 < z; ++t)
      if (t[0] == t[1]) {
        msg = std::string(path) + ": duplicate entry (" + std::to_string(r + 1) + ", " + std::to_string(t[0] + 1) +
              ")";
        return kMtxFormat;
      }
  }
  return kMtxOk;
}

int mtx_write(const char* path, int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx, int field,
              int gz, std::string& msg) {
  gzFile f = gzopen(path, gz ? "wb6" : "wbT");
  if (!f) { msg = std::string(path) + ": cannot open for writing (" + strerror(errno) + ")"; return kMtxIo; }
  GzCloser closer{f};
  std::string buf;
  buf.reserve(kChunk + 256);
  const int64_t nnz = row_ptr[n] - row_ptr[0];
  buf += field ? "%%MatrixMarket matrix coordinate real general\n" : "%%MatrixMarket matrix coordinate pattern general\n";
  buf += "% binary design (pattern store), 1-based row col" + std::string(field ? " value" : "") + "\n";
  buf += std::to_string(n) + " " + std::to_string(p) + " " + std::to_string(nnz) + "\n";
  char num[32];
  auto flush = [&]() -> bool {
    if (buf.empty()) return true;
    if (gzwrite(f, buf.data(), (unsigned)buf.size()) != (int)buf.size()) return false;
    buf.clear();
    return true;
  };
  for (int64_t r = 0; r < n; ++r) {
    auto rr = std::to_chars(num, num + sizeof num, r + 1);
    const std::string rs(num, rr.ptr);
    for (int64_t t = row_ptr[r]; t < row_ptr[r + 1]; ++t) {
      buf += rs;
      buf += ' ';
      auto cr = std::to_chars(num, num + sizeof num, (int64_t)col_idx[t] + 1);
      buf.append(num, cr.ptr);
      buf += field ? " 1\n" : "\n";
    }
    if (buf.size() >= kChunk && !flush()) { msg = std::string(path) + ": write failed"; return kMtxIo; }
  }
  if (!flush()) { msg = std::string(path) + ": write failed"; return kMtxIo; }
  if (gzclose(closer.f) != Z_OK) {
    closer.f = nullptr;
    msg = std::string(path) + ": close failed";
    return kMtxIo;
  }
  closer.f = nullptr;
  return kMtxOk;
}

}  // namespace pcgs
