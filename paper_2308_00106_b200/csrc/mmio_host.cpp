// mmio_host.cpp — native, multithreaded Matrix Market coordinate body parser and
// writer (host code).  Restates the entry loop of the
// reference's parse_matrix_market (matio.py:196-239) and the line format of
// _write_mm (matio.py:270-274); the banner and size line (a few bytes) stay in
// Python (matio.py).
//
// Parse = two passes over the body split into per-thread byte ranges at line
// boundaries: (1) count lines and entry lines per range, (2) exclusive scan, then
// every range parses its entries straight into its slice of the outputs.  The
// first error in LINE ORDER wins, as in the reference's sequential loop: the
// "more than the declared entries" error belongs to the line of entry number
// `declared`, and only parse errors on earlier lines can precede it.
//
// Token rules follow Python's int() / float() on str.split() fields for ASCII
// input: optional sign + decimal digits for indices and integer values (an
// integer value converts with correct rounding, -0 gives +0.0 like
// float(int("-0"))), decimal / inf / infinity / nan (any case, optional sign)
// for real values, converted with std::from_chars (correctly rounded, locale
// free).  Anything else on an entry line — including non-ASCII bytes and the
// digit-group underscores Python would accept — is reported as an error on that
// line; the Python wrapper then re-checks that one line with the reference's
// rules to word the exception exactly (or names the unsupported literal).
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <charconv>
#include <thread>
#include <vector>

#include "../../include/sme.h"

#define SME_API extern "C" __attribute__((visibility("default")))

namespace sme {
void set_error(const char* fmt, ...);
}

namespace {

inline bool is_ws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f) || c == '\n';
}

struct Token {
  const char* p;
  size_t n;
};

// split [a, b) on whitespace into at most 4 tokens; returns the token count (4 = "more than 3")
inline int split(const char* a, const char* b, Token* t) {
  int k = 0;
  while (a < b) {
    while (a < b && is_ws((unsigned char)*a)) ++a;
    if (a >= b) break;
    const char* s = a;
    while (a < b && !is_ws((unsigned char)*a)) ++a;
    if (k < 4) t[k] = Token{s, (size_t)(a - s)};
    ++k;
    if (k >= 4) return 4;
  }
  return k;
}

// Python int(token) for [+-]?[0-9]+; false on anything else.  ovf: |v| >= 2^62.
inline bool parse_int(const Token& t, int64_t* v, bool* ovf) {
  const char* p = t.p;
  const char* e = t.p + t.n;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= e) return false;
  int64_t acc = 0;
  *ovf = false;
  for (; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    if (acc < ((int64_t)1 << 58)) acc = acc * 10 + (*p - '0');
    else *ovf = true;
  }
  *v = neg ? -acc : acc;
  return true;
}

inline bool ieq(const char* p, size_t n, const char* lit) {
  if (strlen(lit) != n) return false;
  for (size_t i = 0; i < n; ++i) {
    char c = p[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != lit[i]) return false;
  }
  return true;
}

// Python float(token) for decimal / inf / infinity / nan literals
inline bool parse_real(const Token& t, double* v) {
  const char* p = t.p;
  const char* e = t.p + t.n;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= e) return false;
  const size_t n = (size_t)(e - p);
  if (ieq(p, n, "inf") || ieq(p, n, "infinity")) {
    *v = neg ? -__builtin_inf() : __builtin_inf();
    return true;
  }
  if (ieq(p, n, "nan")) {
    *v = neg ? -__builtin_nan("") : __builtin_nan("");
    return true;
  }
  // decimal only: digits, one '.', exponent [eE][+-]?digits (from_chars alone would
  // also take "nan(...)", which Python rejects)
  bool digit = false;
  const char* q = p;
  while (q < e && *q >= '0' && *q <= '9') ++q, digit = true;
  if (q < e && *q == '.') {
    ++q;
    while (q < e && *q >= '0' && *q <= '9') ++q, digit = true;
  }
  if (!digit) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    const char* d0 = q;
    while (q < e && *q >= '0' && *q <= '9') ++q;
    if (q == d0) return false;
  }
  if (q != e) return false;
  double d = 0.0;
  const auto r = std::from_chars(p, e, d, std::chars_format::general);
  if (r.ec != std::errc() && r.ec != std::errc::result_out_of_range) return false;
  if (r.ec == std::errc::result_out_of_range) {
    // from_chars leaves d unset: Python gives +-inf on overflow, +-0.0 on underflow.
    // Decimal magnitude = (integer digits - leading zeros) + exponent.
    int64_t intd = 0, lead = -1, pos = 0, ex = 0;
    bool frac = false;
    const char* x = p;
    for (; x < e && *x != 'e' && *x != 'E'; ++x) {
      if (*x == '.') {
        frac = true;
        continue;
      }
      if (!frac) ++intd;
      if (lead < 0 && *x != '0') lead = pos;
      ++pos;
    }
    if (x < e) {
      ++x;
      const bool eneg = *x == '-';
      if (*x == '+' || *x == '-') ++x;
      for (; x < e; ++x) ex = std::min<int64_t>(ex * 10 + (*x - '0'), (int64_t)1 << 40);
      if (eneg) ex = -ex;
    }
    d = (lead >= 0 && intd - lead + ex > 0) ? __builtin_inf() : 0.0;
  }
  *v = neg ? -d : d;
  return true;
}

// an integer value: float(int(token)), correctly rounded, -0 -> +0.0
inline bool parse_int_value(const Token& t, double* v) {
  const char* p = t.p;
  const char* e = t.p + t.n;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= e) return false;
  bool nonzero = false;
  for (const char* q = p; q < e; ++q) {
    if (*q < '0' || *q > '9') return false;
    nonzero |= *q != '0';
  }
  if (!nonzero) {
    *v = 0.0;
    return true;
  }
  double d = 0.0;
  const auto r = std::from_chars(p, e, d, std::chars_format::fixed);
  if (r.ec == std::errc::result_out_of_range) return false;  // > DBL_MAX: Python raises OverflowError
  if (r.ec != std::errc() || r.ptr != e) return false;
  *v = neg ? -d : d;
  return true;
}

enum Err : int64_t {
  E_OK = 0,
  E_TOO_MANY = 1,
  E_FIELDS = 2,
  E_INDEX = 3,
  E_ROW_RANGE = 4,
  E_COL_RANGE = 5,
  E_INT_VALUE = 6,
  E_REAL_VALUE = 7,
  E_NON_ASCII = 8,
};

// [a, b) holds whole lines.  Line ends: '\n', and with cr_newline also '\r' alone or "\r\n".
template <typename F>
inline void for_lines(const char* a, const char* b, bool cr_newline, F&& f) {
  const char* s = a;
  while (s < b) {
    const char* e = s;
    while (e < b && *e != '\n' && !(cr_newline && *e == '\r')) ++e;
    f(s, e);
    if (e >= b) break;
    if (cr_newline && *e == '\r' && e + 1 < b && e[1] == '\n') ++e;
    s = e + 1;
  }
}

inline bool entry_line(const char* s, const char* e) {
  while (s < e && is_ws((unsigned char)*s)) ++s;
  return s < e && *s != '%';
}

struct RangeStats {
  int64_t lines = 0, entries = 0;
};

}  // namespace

// Parse the entry lines of a coordinate body.
//   buf/len          the bytes after the size line (the line after it starts at first_line_no)
//   field            0 real, 1 integer, 2 pattern;  symmetric mirroring is done by the caller
//   declared         entries promised by the size line; outputs hold `declared` entries
//   rows/cols        int32[declared] 0-based (n_rows, n_cols < 2^31); vals f64[declared]
//   cr_newline       1: '\r' and "\r\n" also end lines (text-file reading), 0: only '\n'
//   status[4]        out: {error code, error line (1-based) or 0, entries found, byte offset of the error line}
// Returns SME_OK also when the content is malformed (status[0] != 0 says what and where);
// SME_EINVAL only for bad arguments.
SME_API int sme_host_mm_parse(const char* buf, int64_t len, int field, int64_t n_rows, int64_t n_cols,
                              int64_t declared, int64_t first_line_no, int cr_newline, int threads, int32_t* rows,
                              int32_t* cols, double* vals, int64_t* status) {
  if (!status || len < 0 || (len > 0 && !buf) || field < 0 || field > 2 || n_rows < 1 || n_cols < 1 ||
      n_rows > INT32_MAX || n_cols > INT32_MAX || declared < 0 || (declared > 0 && (!rows || !cols || !vals))) {
    sme::set_error("sme_host_mm_parse: bad arguments");
    return SME_EINVAL;
  }
  status[0] = status[1] = status[2] = status[3] = 0;
  const bool crnl = cr_newline != 0;
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  T = (int)std::min<int64_t>(T, std::max<int64_t>(1, len >> 20));  // >= 1 MiB per range
  // range starts at line boundaries
  std::vector<int64_t> cut(T + 1, len);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    int64_t c = std::max(cut[t - 1], len * t / T);
    while (c < len && c > 0 && buf[c - 1] != '\n' && !(crnl && buf[c - 1] == '\r' && buf[c] != '\n')) ++c;
    cut[t] = c;
  }
  std::vector<RangeStats> st(T);
  auto run = [&](auto&& body) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(body, t);
    body(0);
    for (auto& x : th) x.join();
  };
  run([&](int t) {
    RangeStats s;
    for_lines(buf + cut[t], buf + cut[t + 1], crnl, [&](const char* a, const char* b) {
      ++s.lines;
      s.entries += entry_line(a, b);
    });
    // a range that ends exactly after a line terminator holds no extra empty line
    st[t] = s;
  });
  std::vector<int64_t> line0(T + 1, 0), ent0(T + 1, 0);
  for (int t = 0; t < T; ++t) {
    line0[t + 1] = line0[t] + st[t].lines;
    ent0[t + 1] = ent0[t] + st[t].entries;
  }
  const int64_t want = field == 2 ? 2 : 3;
  struct FirstErr {
    int64_t line = INT64_MAX, code = 0, off = 0;
  };
  std::vector<FirstErr> fe(T);
  run([&](int t) {
    int64_t line = first_line_no + line0[t], k = ent0[t];
    FirstErr f;
    for_lines(buf + cut[t], buf + cut[t + 1], crnl, [&](const char* a, const char* b) {
      const int64_t ln = line++;
      if (f.code != 0 || !entry_line(a, b)) return;
      const int64_t idx = k++;
      auto fail = [&](int64_t code) {
        f.line = ln;
        f.code = code;
        f.off = a - buf;
      };
      if (idx >= declared) return fail(E_TOO_MANY);
      for (const char* q = a; q < b; ++q)
        if ((unsigned char)*q >= 0x80) return fail(E_NON_ASCII);
      Token tk[4];
      const int nt = split(a, b, tk);
      if (nt != want) return fail(E_FIELDS);
      int64_t i = 0, j = 0;
      bool oi = false, oj = false;
      if (!parse_int(tk[0], &i, &oi) || !parse_int(tk[1], &j, &oj)) return fail(E_INDEX);
      if (oi || i < 1 || i > n_rows) return fail(E_ROW_RANGE);
      if (oj || j < 1 || j > n_cols) return fail(E_COL_RANGE);
      double v = 1.0;
      if (field == 1 && !parse_int_value(tk[2], &v)) return fail(E_INT_VALUE);
      if (field == 0 && !parse_real(tk[2], &v)) return fail(E_REAL_VALUE);
      rows[idx] = (int32_t)(i - 1);
      cols[idx] = (int32_t)(j - 1);
      vals[idx] = v;
    });
    fe[t] = f;
  });
  for (int t = 0; t < T; ++t) {
    if (fe[t].code != 0) {  // ranges are in line order: the first range with an error has the first error
      status[0] = fe[t].code;
      status[1] = fe[t].line;
      status[3] = fe[t].off;
      break;
    }
  }
  status[2] = ent0[T];
  return SME_OK;
}

// Format n entries as Matrix Market lines "i+1 j+1 v\n" with v in %.17g (matio.py:270-274,
// f"{v:.17g}"; NaN prints as "nan" whatever its sign, like Python).  out has cap bytes
// (72 per entry always suffices); *out_len receives the bytes written.  Multithreaded:
// ranges are formatted in parallel into per-range buffers and then concatenated.
SME_API int sme_host_mm_format(const int64_t* rows, const int64_t* cols, const double* vals, int64_t n, char* out,
                               int64_t cap, int threads, int64_t* out_len) {
  if (!out_len || n < 0 || (n > 0 && (!rows || !cols || !vals || !out)) || cap < 0) {
    sme::set_error("sme_host_mm_format: bad arguments");
    return SME_EINVAL;
  }
  if (cap < n * 72) {
    sme::set_error("sme_host_mm_format: capacity %lld < 72 bytes per entry", (long long)cap);
    return SME_ENOSPACE;
  }
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  T = (int)std::min<int64_t>(T, std::max<int64_t>(1, n >> 16));
  std::vector<int64_t> used(T, 0);
  auto body = [&](int t) {
    const int64_t a = n * t / T, b = n * (t + 1) / T;
    char* o = out + a * 72;
    for (int64_t k = a; k < b; ++k) {
      const double v = vals[k];
      int w;
      if (v != v)
        w = snprintf(o, 72, "%lld %lld nan\n", (long long)(rows[k] + 1), (long long)(cols[k] + 1));
      else
        w = snprintf(o, 72, "%lld %lld %.17g\n", (long long)(rows[k] + 1), (long long)(cols[k] + 1), v);
      o += w;
    }
    used[t] = o - (out + a * 72);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(body, t);
  body(0);
  for (auto& x : th) x.join();
  int64_t pos = used[0];
  for (int t = 1; t < T; ++t) {
    const int64_t a = n * t / T;
    memmove(out + pos, out + a * 72, (size_t)used[t]);
    pos += used[t];
  }
  *out_len = pos;
  return SME_OK;
}
