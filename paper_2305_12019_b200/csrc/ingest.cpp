// LIBSVM text parser (reference ingest.py:102-182, parse_libsvm) -- native,
// multi-threaded, with the reference's grammar, label handling and errors.
//
// The text is split into line-aligned chunks, one per thread; each thread
// tokenises its lines into per-sample (index, value) runs, recording the
// first error it meets.  Because chunks are ordered, the earliest failing
// chunk's first error is the error the reference's single pass reports.
// Samples are then numbered across chunks (prefix sums) and laid out as CSC
// (samples are columns, entries in strictly increasing feature order, exact
// zeros dropped -- ingest.py:163-167).
//
// Grammar follows Python's: str.split() whitespace, universal newlines
// (\n, \r\n, \r), '#' comments, labels via float() (sign, digits with single
// underscores, '.', exponent, inf/infinity/nan -- no hex), indices via int()
// (decimal, leading zeros and single underscores allowed).  Non-ASCII
// digits / whitespace, which Python also accepts, are not recognised here.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

namespace {

bool is_ws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}

// Python repr of an ASCII token: single quotes unless the token contains a
// single quote and no double quote.
std::string py_repr(const char* b, const char* e) {
  std::string s(b, e);
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char c : s) {
    if (c == '\\') out += "\\\\";
    else if (c == (unsigned char)q) { out += '\\'; out += (char)c; }
    else if (c == '\t') out += "\\t";
    else if (c < 0x20 || c == 0x7f) {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", c);
      out += buf;
    } else out += (char)c;
  }
  out += q;
  return out;
}

// digits with single underscores between digits (Python numeric literal rule)
bool digit_run(const char*& p, const char* e, std::string& out) {
  if (p >= e || !(*p >= '0' && *p <= '9')) return false;
  while (p < e) {
    if (*p >= '0' && *p <= '9') {
      out += *p++;
    } else if (*p == '_' && p + 1 < e && p[1] >= '0' && p[1] <= '9' && !out.empty()) {
      ++p;
    } else {
      break;
    }
  }
  return true;
}

bool ieq(const char* b, const char* e, const char* w) {
  const size_t n = strlen(w);
  if ((size_t)(e - b) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if (tolower((unsigned char)b[i]) != w[i]) return false;
  return true;
}

// Python float() of a whitespace-free token
bool py_float(const char* b, const char* e, double& v) {
  const char* p = b;
  std::string s;
  if (p < e && (*p == '+' || *p == '-')) s += *p++;
  if (ieq(p, e, "inf") || ieq(p, e, "infinity")) {
    v = (s == "-") ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(p, e, "nan")) {
    v = NAN;
    return true;
  }
  bool mant = false;
  if (p < e && *p >= '0' && *p <= '9') mant = digit_run(p, e, s);
  if (p < e && *p == '.') {
    s += *p++;
    if (p < e && *p >= '0' && *p <= '9') mant = digit_run(p, e, s) || mant;
  }
  if (!mant) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    s += *p++;
    if (p < e && (*p == '+' || *p == '-')) s += *p++;
    if (!digit_run(p, e, s)) return false;
  }
  if (p != e) return false;
  v = strtod(s.c_str(), nullptr);  // correctly rounded, like Python
  return true;
}

// Python int() of a whitespace-free token (base 10); false on overflow of int64
bool py_int(const char* b, const char* e, int64_t& v, bool& big) {
  const char* p = b;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  std::string s;
  if (!digit_run(p, e, s) || p != e) return false;
  size_t i = 0;
  while (i + 1 < s.size() && s[i] == '0') ++i;
  s = s.substr(i);
  big = s.size() > 18;
  v = 0;
  if (!big)
    for (char c : s) v = v * 10 + (c - '0');
  if (neg) v = -v;
  return true;
}

struct Chunk {
  // samples of this chunk
  std::vector<int64_t> cnt;     // entries per sample
  std::vector<int64_t> rows;    // 0-based feature index
  std::vector<double> vals;
  std::vector<double> labels;   // NaN when unlabeled
  std::vector<int64_t> lines;   // line (chunk-relative, 1-based) of each sample
  int64_t lines_total = 0;
  int64_t dmax = 0;
  bool unlabeled = false;
  // first error
  int64_t err_line = 0;  // chunk-relative, 0 = none
  std::string err;
};

void parse_chunk(const char* b, const char* e, bool require_labels, Chunk& c) {
  const char* p = b;
  int64_t line = 0;
  while (p < e) {
    const char* ls = p;
    while (p < e && *p != '\n' && *p != '\r') ++p;
    const char* le = p;
    if (p < e) {
      if (*p == '\r' && p + 1 < e && p[1] == '\n') p += 2;
      else ++p;
    }
    ++line;
    const char* hash = (const char*)memchr(ls, '#', le - ls);
    if (hash) le = hash;
    // tokens
    const char* t = ls;
    while (t < le && is_ws((unsigned char)*t)) ++t;
    if (t >= le) continue;
    auto next_tok = [&](const char*& tb, const char*& te) -> bool {
      while (t < le && is_ws((unsigned char)*t)) ++t;
      if (t >= le) return false;
      tb = t;
      while (t < le && !is_ws((unsigned char)*t)) ++t;
      te = t;
      return true;
    };
    const char *tb, *te;
    next_tok(tb, te);
    auto fail = [&](const std::string& msg) {
      c.err_line = line;
      c.err = msg;
    };
    double label = NAN;
    const bool first_has_colon = memchr(tb, ':', te - tb) != nullptr;
    bool consumed_first = false;
    if (first_has_colon) {
      if (require_labels) {
        fail("expected a label, got " + py_repr(tb, te));
        return;
      }
      c.unlabeled = true;
    } else {
      if (!py_float(tb, te, label)) {
        fail("bad label token " + py_repr(tb, te));
        return;
      }
      if (!std::isfinite(label)) {
        fail("non-finite label " + py_repr(tb, te));
        return;
      }
      consumed_first = true;
    }
    int64_t prev = 0, k = 0;
    bool have = !consumed_first;  // the first token is a feature when unlabeled
    while (true) {
      if (!have && !next_tok(tb, te)) break;
      have = false;
      const char* colon = (const char*)memchr(tb, ':', te - tb);
      if (!colon) {
        fail("bad feature token " + py_repr(tb, te));
        return;
      }
      int64_t idx = 0;
      bool big = false;
      double val = 0.0;
      if (!py_int(tb, colon, idx, big) || !py_float(colon + 1, te, val)) {
        fail("bad feature token " + py_repr(tb, te));
        return;
      }
      if (big) {  // beyond int64: a positive one is not increasing-checkable here
        fail("feature index " + std::string(tb, colon) + " is too large");
        return;
      }
      if (idx < 1) {
        fail("feature index " + std::to_string(idx) + " is not positive");
        return;
      }
      if (idx <= prev) {
        fail("feature index " + std::to_string(idx) + " not increasing (after " + std::to_string(prev) + ")");
        return;
      }
      if (!std::isfinite(val)) {
        fail("non-finite value in token " + py_repr(tb, te));
        return;
      }
      prev = idx;
      if (val != 0.0) {
        c.rows.push_back(idx - 1);
        c.vals.push_back(val);
        ++k;
      }
      c.dmax = std::max(c.dmax, idx);
    }
    c.cnt.push_back(k);
    c.labels.push_back(label);
    c.lines.push_back(line);
  }
  c.lines_total = line;
}

}  // namespace

struct gdwd_libsvm {
  int64_t n = 0, d = 0, nnz = 0;
  bool unlabeled = false;
  std::vector<int64_t> colptr, rowidx, label_lines;
  std::vector<double> values, labels;
};

extern "C" {

int gdwd_libsvm_parse(const char* path, const char* text, int64_t text_len, int32_t require_labels,
                      int32_t threads, gdwd_libsvm** out, int64_t* err_line, char* err_msg, int64_t err_cap) {
  if (!out) return 2;
  *out = nullptr;
  if (err_line) *err_line = 0;
  auto set_msg = [&](const std::string& m) {
    if (err_msg && err_cap > 0) {
      const size_t k = std::min<size_t>(m.size(), (size_t)err_cap - 1);
      memcpy(err_msg, m.data(), k);
      err_msg[k] = 0;
    }
  };
  std::string owned;
  if (path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) {
      set_msg(std::string("cannot open ") + path);
      return 7;
    }
    std::ostringstream ss;
    ss << f.rdbuf();
    owned = ss.str();
    text = owned.data();
    text_len = (int64_t)owned.size();
  }
  if (!text && text_len > 0) return 2;
  const char* b = text;
  const char* e = text + text_len;
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  T = (int)std::min<int64_t>(T, std::max<int64_t>(1, text_len / (1 << 16)));
  // line-aligned chunk boundaries (after a '\n', or after a lone '\r')
  std::vector<const char*> cut{b};
  for (int t = 1; t < T; ++t) {
    const char* p = b + (text_len * t) / T;
    if (p <= cut.back()) continue;
    while (p < e && !(p[-1] == '\n' || (p[-1] == '\r' && *p != '\n'))) ++p;
    if (p < e && p > cut.back()) cut.push_back(p);
  }
  cut.push_back(e);
  const int C = (int)cut.size() - 1;
  std::vector<Chunk> ch(C);
  std::vector<std::thread> th;
  for (int c = 1; c < C; ++c) th.emplace_back(parse_chunk, cut[c], cut[c + 1], require_labels != 0, std::ref(ch[c]));
  if (C > 0) parse_chunk(cut[0], cut[1], require_labels != 0, ch[0]);
  for (auto& t : th) t.join();
  // the earliest error wins (chunks are in file order)
  int64_t line_off = 0;
  for (int c = 0; c < C; ++c) {
    if (ch[c].err_line) {
      if (err_line) *err_line = line_off + ch[c].err_line;
      set_msg(ch[c].err);
      return 2;
    }
    line_off += ch[c].lines_total;
  }
  auto* r = new gdwd_libsvm();
  int64_t n = 0, nnz = 0, d = 0;
  for (auto& c : ch) {
    n += (int64_t)c.cnt.size();
    nnz += (int64_t)c.rows.size();
    d = std::max(d, c.dmax);
    r->unlabeled = r->unlabeled || c.unlabeled;
  }
  if (n == 0) {
    delete r;
    if (err_line) *err_line = 0;
    set_msg("no samples in input");
    return 2;
  }
  r->n = n;
  r->d = d;
  r->nnz = nnz;
  r->colptr.resize(n + 1);
  r->rowidx.resize(nnz);
  r->values.resize(nnz);
  r->labels.resize(n);
  r->label_lines.resize(n);
  int64_t s = 0, z = 0;
  line_off = 0;
  r->colptr[0] = 0;
  for (auto& c : ch) {
    for (size_t i = 0; i < c.cnt.size(); ++i) {
      r->colptr[s + 1] = r->colptr[s] + c.cnt[i];
      r->labels[s] = c.labels[i];
      r->label_lines[s] = line_off + c.lines[i];
      ++s;
    }
    std::copy(c.rows.begin(), c.rows.end(), r->rowidx.begin() + z);
    std::copy(c.vals.begin(), c.vals.end(), r->values.begin() + z);
    z += (int64_t)c.rows.size();
    line_off += c.lines_total;
  }
  *out = r;
  return 0;
}

int gdwd_libsvm_sizes(const gdwd_libsvm* p, int64_t* n, int64_t* d, int64_t* nnz, int32_t* unlabeled) {
  if (!p) return 2;
  if (n) *n = p->n;
  if (d) *d = p->d;
  if (nnz) *nnz = p->nnz;
  if (unlabeled) *unlabeled = p->unlabeled ? 1 : 0;
  return 0;
}

int gdwd_libsvm_copy(const gdwd_libsvm* p, int64_t* colptr, int64_t* rowidx, double* values, double* labels,
                     int64_t* label_lines) {
  if (!p) return 2;
  if (colptr) memcpy(colptr, p->colptr.data(), p->colptr.size() * sizeof(int64_t));
  if (rowidx) memcpy(rowidx, p->rowidx.data(), p->rowidx.size() * sizeof(int64_t));
  if (values) memcpy(values, p->values.data(), p->values.size() * sizeof(double));
  if (labels) memcpy(labels, p->labels.data(), p->labels.size() * sizeof(double));
  if (label_lines) memcpy(label_lines, p->label_lines.data(), p->label_lines.size() * sizeof(int64_t));
  return 0;
}

void gdwd_libsvm_free(gdwd_libsvm* p) { delete p; }

// preprocess (ingest.py:185-211): per-feature max-abs, drop all-zero
// features, divide each kept feature by its max-abs, prune entries that the
// division took to zero (csc_from_scipy's eliminate_zeros), renumber rows.
// Multi-threaded over columns; bit-identical to the numpy version (max is
// order-free, the quotient is one IEEE division).  Returns 2 with
// *kept_count = 0 when every feature is zero, 2 on a non-finite value.
int gdwd_preprocess_csc(int64_t d, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                        int32_t threads, int64_t* kept_count, int64_t* kept_ids, double* scales, int64_t* new_colptr,
                        int64_t* new_rowidx, double* new_values, int64_t* new_nnz) {
  if (d < 0 || n < 0 || !colptr || !kept_count || !kept_ids || !scales || !new_colptr || !new_nnz) return 2;
  const int64_t nnz = colptr[n];
  for (int64_t k = 0; k < nnz; ++k)
    if (!std::isfinite(values[k]) || rowidx[k] < 0 || rowidx[k] >= d) return 2;
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  T = (int)std::max<int64_t>(1, std::min<int64_t>(T, nnz / (1 << 15)));
  while (T > 1 && (double)T * d * 8.0 > 512e6) --T;  // per-thread max arrays
  // 1. max-abs per feature: per-thread partial maxima over column ranges
  std::vector<std::vector<double>> part(T, std::vector<double>());
  auto colrange = [&](int t, int64_t& c0, int64_t& c1) {
    c0 = n * t / T;
    c1 = n * (t + 1) / T;
  };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        std::vector<double>& m = part[t];
        m.assign(d, 0.0);
        int64_t c0, c1;
        colrange(t, c0, c1);
        for (int64_t k = colptr[c0]; k < colptr[c1]; ++k) m[rowidx[k]] = std::max(m[rowidx[k]], std::fabs(values[k]));
      });
    for (auto& x : th) x.join();
  }
  std::vector<double>& mx = part[0];
  for (int t = 1; t < T; ++t)
    for (int64_t j = 0; j < d; ++j) mx[j] = std::max(mx[j], part[t][j]);
  // 2. kept features and their ranks
  std::vector<int64_t> rank(d, -1);
  int64_t kc = 0;
  for (int64_t j = 0; j < d; ++j)
    if (mx[j] > 0.0) {
      kept_ids[kc] = j;
      scales[kc] = mx[j];
      rank[j] = kc++;
    }
  *kept_count = kc;
  if (kc == 0) return 2;
  // 3. scaled entries, zero quotients pruned, rows renumbered (column counts,
  //    then a prefix sum, then the fill -- each pass threaded over columns)
  std::vector<int64_t> cnt(n, 0);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        int64_t c0, c1;
        colrange(t, c0, c1);
        for (int64_t c = c0; c < c1; ++c)
          for (int64_t k = colptr[c]; k < colptr[c + 1]; ++k) cnt[c] += (values[k] / mx[rowidx[k]] != 0.0) ? 1 : 0;
      });
    for (auto& x : th) x.join();
  }
  new_colptr[0] = 0;
  for (int64_t c = 0; c < n; ++c) new_colptr[c + 1] = new_colptr[c] + cnt[c];
  *new_nnz = new_colptr[n];
  if (new_rowidx && new_values) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        int64_t c0, c1;
        colrange(t, c0, c1);
        for (int64_t c = c0; c < c1; ++c) {
          int64_t o = new_colptr[c];
          for (int64_t k = colptr[c]; k < colptr[c + 1]; ++k) {
            const double v = values[k] / mx[rowidx[k]];
            if (v != 0.0) {
              new_rowidx[o] = rank[rowidx[k]];
              new_values[o++] = v;
            }
          }
        }
      });
    for (auto& x : th) x.join();
  }
  return 0;
}

}  // extern "C"
