// mmio.cu -- SURVEY 8f-3: Matrix Market coordinate I/O (io.py:33-132),
// host side, multi-threaded; the parsed triplets feed the GPU build.
//
// Parse: the header / size lines are read sequentially with the reference's
// rules (io.py:70-93); the entry region is cut into one chunk per thread at
// line boundaries, each thread parses its lines into (row, col, value) with
// std::from_chars (correctly rounded, like Python's float()), recording its
// first malformed line; a sequential pass over the chunk summaries then
// reports exactly the error the reference's in-order loop would raise first
// (malformed entry, too many entries, out-of-range coordinate, count
// mismatch) with its line number.  Format: `%d %d %.17g` per entry in
// column-major order (io.py:44-51), chunks formatted in parallel.
//
// Numeric tokens: Python's int() / float() also accept a leading '+',
// underscores between digits and inf/nan spellings; those are normalised
// before from_chars so the accepted set matches.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "capi_util.cuh"

namespace as {
namespace mm {

struct Span {
  const char* b;
  const char* e;
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

inline Span strip(const char* b, const char* e) {
  while (b < e && is_space(*b)) b++;
  while (e > b && is_space(e[-1])) e--;
  return {b, e};
}

// split a stripped line into whitespace-separated tokens (at most 4 kept)
inline int tokens(Span s, Span* out, int cap) {
  int n = 0;
  const char* p = s.b;
  while (p < s.e) {
    while (p < s.e && is_space(*p)) p++;
    if (p >= s.e) break;
    const char* q = p;
    while (q < s.e && !is_space(*q)) q++;
    if (n < cap) out[n] = {p, q};
    n++;
    p = q;
  }
  return n;
}

// Python-int-like: [+-]digits with single underscores between digits
inline bool parse_int(Span t, long long* v) {
  char buf[64];
  int n = 0;
  const char* p = t.b;
  bool neg = false;
  if (p < t.e && (*p == '+' || *p == '-')) {
    neg = *p == '-';
    p++;
  }
  if (p >= t.e) return false;
  bool prev_digit = false;
  for (; p < t.e; p++) {
    if (*p == '_') {
      if (!prev_digit || p + 1 >= t.e || !(p[1] >= '0' && p[1] <= '9')) return false;
      prev_digit = false;
      continue;
    }
    if (!(*p >= '0' && *p <= '9') || n >= 40) return false;
    buf[n++] = *p;
    prev_digit = true;
  }
  long long x = 0;
  auto r = std::from_chars(buf, buf + n, x);
  if (r.ec != std::errc() || r.ptr != buf + n) return false;
  *v = neg ? -x : x;
  return true;
}

// Python-float-like: decimal / exponent forms, '+' sign, underscores between
// digits, inf / infinity / nan (any case)
inline bool parse_float(Span t, double* v) {
  char buf[400];
  int n = 0;
  const char* p = t.b;
  bool neg = false;
  if (p < t.e && (*p == '+' || *p == '-')) {
    neg = *p == '-';
    p++;
  }
  const size_t len = (size_t)(t.e - p);
  auto ieq = [&](const char* w) {
    const size_t wl = strlen(w);
    if (len != wl) return false;
    for (size_t i = 0; i < wl; i++)
      if ((p[i] | 0x20) != w[i]) return false;
    return true;
  };
  if (ieq("inf") || ieq("infinity")) {
    *v = neg ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (ieq("nan")) {
    *v = neg ? -NAN : NAN;
    return true;
  }
  auto digit = [](char c) { return c >= '0' && c <= '9'; };
  for (const char* q = p; q < t.e; q++) {
    if (*q == '_') {
      if (q == p || !digit(q[-1]) || q + 1 >= t.e || !digit(q[1])) return false;
      continue;
    }
    if (n >= (int)sizeof(buf) - 1) return false;
    buf[n++] = *q;
  }
  if (n == 0 || buf[0] == '+' || buf[0] == '-') return false;
  double x = 0.0;
  auto r = std::from_chars(buf, buf + n, x, std::chars_format::general);
  if (r.ec == std::errc::result_out_of_range) {
    // from_chars reports under/overflow; Python returns 0.0 / inf
    x = strtod(std::string(buf, n).c_str(), nullptr);
  } else if (r.ec != std::errc() || r.ptr != buf + n) {
    return false;
  }
  *v = neg ? -x : x;
  return true;
}

enum Err { kNone = 0, kMalformedLine = 1, kMalformedEntry = 2 };

struct Chunk {
  const char* b;
  const char* e;
  long long first_line;  // 1-based line number of the chunk's first line
  long long n_entries = 0;
  long long n_lines = 0;
  int err = kNone;        // first malformed line in the chunk
  long long err_line = 0;
  long long err_entry = 0;  // entries before it in the chunk
  long long bad_line = 0;   // first out-of-range entry (line), entry index in chunk
  long long bad_entry = -1;
  long long bad_r = 0, bad_c = 0;
  std::vector<long long> rows, cols;
  std::vector<double> vals;
};

void parse_chunk(Chunk& ch, long long n_rows, long long n_cols) {
  const char* p = ch.b;
  long long line = ch.first_line;
  while (p < ch.e) {
    const char* q = (const char*)memchr(p, '\n', (size_t)(ch.e - p));
    const char* le = q ? q : ch.e;
    const Span s = strip(p, le);
    if (s.b < s.e && *s.b != '%') {
      Span tk[4];
      const int nt = tokens(s, tk, 4);
      long long r, c;
      double v;
      if (nt != 3) {
        ch.err = kMalformedLine;
        ch.err_line = line;
        ch.err_entry = ch.n_entries;
        ch.n_lines = line - ch.first_line + 1;
        return;
      }
      if (!parse_int(tk[0], &r) || !parse_int(tk[1], &c) || !parse_float(tk[2], &v)) {
        ch.err = kMalformedEntry;
        ch.err_line = line;
        ch.err_entry = ch.n_entries;
        ch.n_lines = line - ch.first_line + 1;
        return;
      }
      if (ch.bad_entry < 0 && !(1 <= r && r <= n_rows && 1 <= c && c <= n_cols)) {
        ch.bad_entry = ch.n_entries;
        ch.bad_line = line;
        ch.bad_r = r;
        ch.bad_c = c;
      }
      ch.rows.push_back(r - 1);
      ch.cols.push_back(c - 1);
      ch.vals.push_back(v);
      ch.n_entries++;
    }
    line++;
    p = q ? q + 1 : ch.e;
  }
  ch.n_lines = line - ch.first_line;
}

}  // namespace mm
}  // namespace as

using namespace as;
using namespace as::mm;

extern "C" {

// Header + size line (io.py:65-93).  Outputs the dimensions, the declared
// nnz, the byte offset and 1-based line number where entries start and the
// total line count.  Status AS_ERR_ARG with *err_line set (0 = none) and
// the message in as_last_error() on a MatrixMarketError.
int as_mm_header(const char* buf, int64_t len, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, int64_t* entries_off,
                 int64_t* entries_line, int64_t* err_line) {
  *err_line = 0;
  const char* end = buf + len;
  const char* p = buf;
  long long line = 1;
  auto next_line = [&](Span* out) -> bool {
    if (p >= end) return false;
    const char* q = (const char*)memchr(p, '\n', (size_t)(end - p));
    const char* le = q ? q : end;
    *out = {p, le};
    p = q ? q + 1 : end;
    return true;
  };
  Span ln;
  // Python's splitlines() on an empty string gives no lines
  if (len == 0 || !next_line(&ln)) {
    *err_line = 1;
    set_error("empty input");
    return AS_ERR_ARG;
  }
  {
    Span tk[6];
    const int nt = tokens(strip(ln.b, ln.e), tk, 6);
    static const char* want[5] = {"%%MatrixMarket", "matrix", "coordinate", "real", "general"};
    bool ok = nt == 5;
    for (int i = 0; ok && i < 5; i++)
      ok = (size_t)(tk[i].e - tk[i].b) == strlen(want[i]) && memcmp(tk[i].b, want[i], strlen(want[i])) == 0;
    if (!ok) {
      *err_line = 1;
      set_error("header must be exactly '%%%%MatrixMarket matrix coordinate real general'");
      return AS_ERR_ARG;
    }
  }
  long long total_lines = 1;
  while (next_line(&ln)) {
    line++;
    total_lines = line;
    const Span s = strip(ln.b, ln.e);
    if (s.b >= s.e || *s.b == '%') continue;
    Span tk[4];
    const int nt = tokens(s, tk, 4);
    *entries_off = (int64_t)(p - buf);
    *entries_line = line + 1;
    if (nt != 3) {  // the reference reports the size line's own number (io.py:87-93)
      *err_line = line;
      set_error("size line needs 'rows cols nnz'");
      return AS_ERR_ARG;
    }
    long long v[3];
    for (int i = 0; i < 3; i++)
      if (!parse_int(tk[i], &v[i])) {
        *err_line = line;
        set_error("size line needs three integers");
        return AS_ERR_ARG;
      }
    *n_rows = v[0];
    *n_cols = v[1];
    *nnz = v[2];
    return AS_OK;
  }
  *err_line = total_lines;
  set_error("missing size line");
  return AS_ERR_ARG;
}

// Entries (io.py:95-126): rows / cols (0-based int64) and values, nnz of
// each.  Status AS_OK, or AS_ERR_ARG (MatrixMarketError, *err_line set) or
// AS_ERR_CORRUPT (CorruptionError, *err_line set) with the reference's
// message in as_last_error().
int as_mm_entries(const char* buf, int64_t len, int64_t entries_off, int64_t entries_line, int64_t n_rows,
                  int64_t n_cols, int64_t nnz, int64_t* rows, int64_t* cols, double* vals, int n_threads,
                  int64_t* err_line) {
  *err_line = 0;
  const char* b = buf + entries_off;
  const char* e = buf + len;
  // the line count of the whole input (for the final count-mismatch error,
  // which the reference reports at len(lines))
  int T = std::max(1, std::min(n_threads, 256));
  if (e - b < (1 << 20)) T = 1;
  std::vector<Chunk> ch(T);
  {
    const char* cur = b;
    for (int t = 0; t < T; t++) {
      const char* stop = t == T - 1 ? e : b + (e - b) * (t + 1) / T;
      if (stop < cur) stop = cur;
      if (t < T - 1) {
        const char* nl = (const char*)memchr(stop, '\n', (size_t)(e - stop));
        stop = nl ? nl + 1 : e;
      }
      ch[t].b = cur;
      ch[t].e = stop;
      cur = stop;
    }
  }
  // line numbers of the chunk starts need the newline counts before them
  std::vector<long long> nl_count(T, 0);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++)
      th.emplace_back([&, t] {
        long long c = 0;
        for (const char* p = ch[t].b; p < ch[t].e; p++) c += *p == '\n';
        nl_count[t] = c;
      });
    for (auto& x : th) x.join();
  }
  long long ln = entries_line;
  for (int t = 0; t < T; t++) {
    ch[t].first_line = ln;
    ln += nl_count[t];
  }
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++) th.emplace_back([&, t] { parse_chunk(ch[t], n_rows, n_cols); });
    for (auto& x : th) x.join();
  }
  // replay the reference's in-order checks over the chunk summaries
  long long k = 0;
  for (int t = 0; t < T; t++) {
    Chunk& c = ch[t];
    const long long upto = c.err ? c.err_entry : c.n_entries;
    // too many entries: the (nnz+1)-th entry line, unless an earlier error
    if (k + upto > nnz) {
      // the (nnz - k)-th entry of this chunk is the last allowed; find the next entry's line
      const long long idx = nnz - k;  // index in chunk of the first excess entry
      if (c.bad_entry >= 0 && c.bad_entry < idx) {
        *err_line = c.bad_line;
        set_error("(%lld, %lld)", c.bad_r, c.bad_c);
        return AS_ERR_CORRUPT;
      }
      // locate its line by re-walking the chunk
      const char* p = c.b;
      long long line = c.first_line, seen = 0;
      while (p < c.e) {
        const char* q = (const char*)memchr(p, '\n', (size_t)(c.e - p));
        const char* le = q ? q : c.e;
        const Span s = strip(p, le);
        if (s.b < s.e && *s.b != '%') {
          if (seen == idx) break;
          seen++;
        }
        line++;
        p = q ? q + 1 : c.e;
      }
      *err_line = line;
      set_error("more entries than the size line declares");
      return AS_ERR_ARG;
    }
    if (c.bad_entry >= 0 && c.bad_entry < upto) {
      *err_line = c.bad_line;
      set_error("(%lld, %lld)", c.bad_r, c.bad_c);
      return AS_ERR_CORRUPT;
    }
    if (c.err) {
      *err_line = c.err_line;
      if (c.err == kMalformedLine) {
        // the token count is checked before the entry count (io.py:103-106)
        set_error("entry needs 'row col value'");
      } else if (k + c.err_entry >= nnz) {
        set_error("more entries than the size line declares");
      } else {
        set_error("malformed entry");
      }
      return AS_ERR_ARG;
    }
    k += c.n_entries;
  }
  if (k != nnz) {  // reported at len(lines) (io.py:121-124)
    if (e == b) *err_line = entries_line - 1;
    else *err_line = ln - (buf[len - 1] == '\n' ? 1 : 0);
    set_error("size line declares %lld entries, found %lld", (long long)nnz, k);
    return AS_ERR_ARG;
  }
  long long off = 0;
  for (int t = 0; t < T; t++) {
    const long long n = ch[t].n_entries;
    if (n) {
      memcpy(rows + off, ch[t].rows.data(), n * sizeof(long long));
      memcpy(cols + off, ch[t].cols.data(), n * sizeof(long long));
      memcpy(vals + off, ch[t].vals.data(), n * sizeof(double));
    }
    off += n;
  }
  return AS_OK;
}

// Format (io.py:44-51): header, size line, "%d %d %.17g" per entry (1-based,
// column-major order as given).  Returns the byte count, or -1 if cap is too
// small (cap >= 64 + 72 * nnz always suffices).
int64_t as_mm_format(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows, const int64_t* cols,
                     const double* vals, char* out, int64_t cap, int n_threads) {
  int hn = snprintf(out, (size_t)cap, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n",
                    (long long)n_rows, (long long)n_cols, (long long)nnz);
  if (hn < 0 || hn >= cap) return -1;
  int T = std::max(1, std::min(n_threads, 256));
  if (nnz < 100000) T = 1;
  std::vector<std::string> parts(T);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++)
      th.emplace_back([&, t] {
        const long long lo = nnz * t / T, hi = nnz * (t + 1) / T;
        std::string& s = parts[t];
        s.reserve((size_t)(hi - lo) * 32);
        char line[96];
        for (long long k = lo; k < hi; k++) {
          // std::to_chars with a precision is specified to print exactly like
          // printf("%.17g") (and is several times faster than snprintf)
          char* q = line;
          q = std::to_chars(q, line + sizeof(line), (long long)rows[k] + 1).ptr;
          *q++ = ' ';
          q = std::to_chars(q, line + sizeof(line), (long long)cols[k] + 1).ptr;
          *q++ = ' ';
          q = std::to_chars(q, line + sizeof(line), vals[k], std::chars_format::general, 17).ptr;
          *q++ = '\n';
          s.append(line, (size_t)(q - line));
        }
      });
    for (auto& x : th) x.join();
  }
  int64_t off = hn;
  for (auto& s : parts) {
    if (off + (int64_t)s.size() > cap) return -1;
    memcpy(out + off, s.data(), s.size());
    off += (int64_t)s.size();
  }
  return off;
}

}  // extern "C"
