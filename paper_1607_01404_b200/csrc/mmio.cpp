// Matrix Market ingestion and output (host side of the device CSR build).
//
// Restates the reference reader / writers (pkg/src/itersvd/matio.py:158-276)
// as a native single-pass parser: the file is read once into memory, split
// into lines with Python's universal-newline rules, and every token is
// checked with the same acceptance rules as Python's int() / float(), so a
// file the reference rejects is rejected here with the same message and
// line number (MatrixMarketError).  The triplets it returns go straight to
// the device assembly (svdsb_csr_create_coo_device), which sums duplicates
// in input order exactly like SparseMatrixCsr.from_coo.
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "svdsb.h"

namespace svdsb {
void set_error(const char *fmt, ...);
}

namespace {

using svdsb::set_error;

// Python's str.isspace() for the ASCII range (the reference decodes with
// errors="replace", so nothing above 0x7f is whitespace)
inline bool is_ws(unsigned char c) {
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

struct Line {
  const char *b, *e;  // stripped content [b, e)
};

bool slurp(const char *path, std::string &buf) {
  FILE *f = fopen(path, "rb");
  if (!f) {
    set_error("cannot open %s: %s", path, strerror(errno));
    return false;
  }
  char tmp[1 << 16];
  size_t got;
  while ((got = fread(tmp, 1, sizeof(tmp), f)) > 0) buf.append(tmp, got);
  bool err = ferror(f) != 0;
  fclose(f);
  if (err) {
    set_error("cannot read %s", path);
    return false;
  }
  return true;
}

// readlines() with universal newlines: "\r\n", "\r" and "\n" all end a line
void split_lines(const std::string &buf, std::vector<Line> &out) {
  const char *p = buf.data(), *end = p + buf.size();
  while (p < end) {
    const char *q = p;
    while (q < end && *q != '\n' && *q != '\r') ++q;
    const char *b = p, *e = q;
    while (b < e && is_ws((unsigned char)*b)) ++b;
    while (e > b && is_ws((unsigned char)e[-1])) --e;
    out.push_back({b, e});
    if (q < end && *q == '\r' && q + 1 < end && q[1] == '\n') ++q;
    p = q + 1;
  }
}

void tokens(const Line &l, std::vector<std::string> &out) {
  out.clear();
  const char *p = l.b;
  while (p < l.e) {
    while (p < l.e && is_ws((unsigned char)*p)) ++p;
    const char *q = p;
    while (q < l.e && !is_ws((unsigned char)*q)) ++q;
    if (q > p) out.emplace_back(p, q);
    p = q;
  }
}

// digits with single underscores strictly between digits (PEP 515);
// appends the digits to `clean`
bool digit_run(const std::string &s, size_t &i, std::string &clean) {
  size_t start = i;
  bool prev_digit = false;
  while (i < s.size()) {
    char c = s[i];
    if (c >= '0' && c <= '9') {
      clean.push_back(c);
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < s.size() && s[i + 1] >= '0' && s[i + 1] <= '9') {
      prev_digit = false;
    } else {
      break;
    }
    ++i;
  }
  return i > start && s[i - 1] != '_';
}

// Python int(token): [+-] digits (underscores allowed between digits).
// Values beyond +-2^62 saturate (they only ever feed range checks).
bool parse_int(const std::string &s, int64_t &v) {
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  std::string d;
  if (!digit_run(s, i, d) || i != s.size()) return false;
  const int64_t cap = (int64_t)1 << 62;
  int64_t x = 0;
  for (char c : d) {
    x = x * 10 + (c - '0');
    if (x > cap) {
      x = cap;
      break;
    }
  }
  v = neg ? -x : x;
  return true;
}

bool ieq(const std::string &s, size_t i, const char *word) {
  size_t n = strlen(word);
  if (s.size() - i != n) return false;
  for (size_t k = 0; k < n; ++k)
    if ((s[i + k] | 0x20) != word[k]) return false;
  return true;
}

// Python float(token): [+-] (inf | infinity | nan | decimal[exp]),
// case-insensitive words, underscores between digits, no hex
bool parse_float(const std::string &s, double &v) {
  size_t i = 0;
  std::string clean;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) clean.push_back(s[i++]);
  if (i < s.size() && !(s[i] >= '0' && s[i] <= '9') && s[i] != '.') {
    if (ieq(s, i, "inf") || ieq(s, i, "infinity") || ieq(s, i, "nan")) {
      clean.append(s, i, std::string::npos);
      v = strtod(clean.c_str(), nullptr);
      return true;
    }
    return false;
  }
  bool mant = false;
  if (i < s.size() && s[i] >= '0' && s[i] <= '9') {
    if (!digit_run(s, i, clean)) return false;
    mant = true;
  }
  if (i < s.size() && s[i] == '.') {
    clean.push_back('.');
    ++i;
    if (i < s.size() && s[i] >= '0' && s[i] <= '9') {
      if (!digit_run(s, i, clean)) return false;
      mant = true;
    }
  }
  if (!mant) return false;
  if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
    clean.push_back('e');
    ++i;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) clean.push_back(s[i++]);
    if (!digit_run(s, i, clean)) return false;
  }
  if (i != s.size()) return false;
  v = strtod(clean.c_str(), nullptr);  // correctly rounded, like CPython
  return true;
}

struct Header {
  int64_t m = 0, n = 0, entries = 0;
  int is_array = 0, symmetric = 0;
  size_t body = 0;  // index of the first entry line candidate
};

// returns SVDSB_OK, or SVDSB_ERR_FORMAT with *err_line set
int parse_header(const std::vector<Line> &lines, Header &h, int64_t *err_line) {
  auto fail = [&](int64_t line, const char *fmt, const char *arg) {
    if (arg)
      set_error(fmt, arg);
    else
      set_error("%s", fmt);
    *err_line = line;
    return SVDSB_ERR_FORMAT;
  };
  if (lines.empty()) return fail(1, "empty file", nullptr);
  std::string ban(lines[0].b, lines[0].e);
  for (auto &c : ban) c = (char)((c >= 'A' && c <= 'Z') ? c + 32 : c);
  std::vector<std::string> t;
  tokens({ban.data(), ban.data() + ban.size()}, t);
  if (t.size() < 4 || t[0] != "%%matrixmarket") return fail(1, "missing %%MatrixMarket banner", nullptr);
  if (t[1] != "matrix") return fail(1, "unsupported object '%s'", t[1].c_str());
  const std::string &fmt = t[2], &field = t[3];
  std::string sym = t.size() > 4 ? t[4] : "general";
  if (fmt != "coordinate" && fmt != "array") return fail(1, "unsupported format '%s'", fmt.c_str());
  if (field == "pattern") return fail(1, "pattern matrices carry no values", nullptr);
  if (field != "real" && field != "integer" && field != "double")
    return fail(1, "unsupported field '%s'", field.c_str());
  if (sym != "general" && sym != "symmetric") return fail(1, "unsupported symmetry '%s'", sym.c_str());
  h.is_array = fmt == "array";
  h.symmetric = sym == "symmetric";
  if (h.is_array && h.symmetric) return fail(1, "array storage is supported for general symmetry only", nullptr);
  size_t i = 1;
  for (; i < lines.size(); ++i)
    if (lines[i].e > lines[i].b && *lines[i].b != '%') break;
  if (i >= lines.size()) return fail((int64_t)lines.size(), "missing size line", nullptr);
  int64_t lineno = (int64_t)i + 1;
  std::string body(lines[i].b, lines[i].e);
  tokens(lines[i], t);
  bool ok = true;
  if (!h.is_array) {
    ok = t.size() == 3 && parse_int(t[0], h.m) && parse_int(t[1], h.n) && parse_int(t[2], h.entries);
  } else {
    ok = t.size() == 2 && parse_int(t[0], h.m) && parse_int(t[1], h.n);
    if (ok) {
      // m * n in Python integers: only the sign and the sanity cap matter
      if (h.m > 0 && h.n > 0 && h.m > ((int64_t)1 << 62) / h.n)
        h.entries = (int64_t)1 << 62;
      else
        h.entries = h.m * h.n;
      if ((h.m < 0) != (h.n < 0) && h.m != 0 && h.n != 0) h.entries = -1;
    }
  }
  if (!ok) return fail(lineno, "malformed size line '%s'", body.c_str());
  if (h.m < 0 || h.n < 0 || h.entries < 0) return fail(lineno, "negative size", nullptr);
  if (h.is_array && h.entries > ((int64_t)1 << 27))
    return fail(lineno, "array dimensions overflow sane limits", nullptr);
  h.body = i + 1;
  return SVDSB_OK;
}

}  // namespace

extern "C" {

int svdsb_mm_read_header(const char *path, int64_t *m, int64_t *n, int64_t *entries, int *is_array,
                         int *symmetric, int64_t *err_line) {
  if (!path || !m || !n || !entries || !is_array || !symmetric || !err_line) {
    set_error("svdsb_mm_read_header: NULL argument");
    return SVDSB_ERR_ARG;
  }
  *err_line = 0;
  std::string buf;
  if (!slurp(path, buf)) return SVDSB_ERR_IO;
  std::vector<Line> lines;
  split_lines(buf, lines);
  Header h;
  int rc = parse_header(lines, h, err_line);
  if (rc) return rc;
  *m = h.m;
  *n = h.n;
  *entries = h.entries;
  *is_array = h.is_array;
  *symmetric = h.symmetric;
  return SVDSB_OK;
}

int svdsb_mm_read_entries(const char *path, int64_t entries, int64_t *rows_host, int64_t *cols_host,
                          double *vals_host, int64_t *err_line) {
  if (!path || !err_line || entries < 0 || (entries > 0 && (!rows_host || !cols_host || !vals_host))) {
    set_error("svdsb_mm_read_entries: bad argument");
    return SVDSB_ERR_ARG;
  }
  *err_line = 0;
  std::string buf;
  if (!slurp(path, buf)) return SVDSB_ERR_IO;
  std::vector<Line> lines;
  split_lines(buf, lines);
  Header h;
  int rc = parse_header(lines, h, err_line);
  if (rc) return rc;
  if (h.entries != entries) {
    set_error("svdsb_mm_read_entries: entry count %lld does not match the header (%lld)", (long long)entries,
              (long long)h.entries);
    return SVDSB_ERR_ARG;
  }
  std::vector<std::string> t;
  int64_t k = 0;
  for (size_t i = h.body; i < lines.size(); ++i) {
    const Line &l = lines[i];
    if (l.e == l.b || *l.b == '%') continue;
    std::string text(l.b, l.e);
    if (k >= entries) {
      set_error("more entries than declared");
      *err_line = (int64_t)i + 1;
      return SVDSB_ERR_FORMAT;
    }
    tokens(l, t);
    int64_t r, c;
    double v;
    bool ok;
    if (!h.is_array) {
      ok = t.size() == 3 && parse_int(t[0], r) && parse_int(t[1], c) && parse_float(t[2], v);
      r -= 1;
      c -= 1;
    } else {
      ok = t.size() == 1 && parse_float(t[0], v);
      r = h.m ? k % h.m : 0;
      c = h.m ? k / h.m : 0;  // column major
    }
    if (!ok) {
      set_error("malformed entry '%s'", text.c_str());
      *err_line = (int64_t)i + 1;
      return SVDSB_ERR_FORMAT;
    }
    if (!(r >= 0 && r < h.m && c >= 0 && c < h.n)) {
      set_error("index out of bounds in '%s'", text.c_str());
      *err_line = (int64_t)i + 1;
      return SVDSB_ERR_FORMAT;
    }
    rows_host[k] = r;
    cols_host[k] = c;
    vals_host[k] = v;
    ++k;
  }
  if (k != entries) {
    set_error("expected %lld entries, found %lld", (long long)entries, (long long)k);
    *err_line = (int64_t)lines.size();
    return SVDSB_ERR_FORMAT;
  }
  if (h.symmetric && h.m != h.n) {
    set_error("symmetric matrix must be square");
    *err_line = 1;
    return SVDSB_ERR_FORMAT;
  }
  return SVDSB_OK;
}

// "%.17g" as Python formats it: inf / -inf / nan (never "-nan")
static void put_double(std::string &out, double v) {
  char tmp[40];
  if (v != v) {
    out += "nan";
    return;
  }
  snprintf(tmp, sizeof(tmp), "%.17g", v);
  out += tmp;
}

static int flush_file(const char *path, const std::string &s) {
  FILE *f = fopen(path, "wb");
  if (!f) {
    set_error("cannot open %s for writing: %s", path, strerror(errno));
    return SVDSB_ERR_IO;
  }
  bool ok = fwrite(s.data(), 1, s.size(), f) == s.size();
  ok = (fclose(f) == 0) && ok;
  if (!ok) {
    set_error("cannot write %s", path);
    return SVDSB_ERR_IO;
  }
  return SVDSB_OK;
}

int svdsb_mm_write_coo(const char *path, int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr_host,
                       const int64_t *col_host, const double *vals_host) {
  if (!path || m < 0 || n < 0 || nnz < 0 || !row_ptr_host || (nnz > 0 && (!col_host || !vals_host))) {
    set_error("svdsb_mm_write_coo: bad argument");
    return SVDSB_ERR_ARG;
  }
  std::string s = "%%MatrixMarket matrix coordinate real general\n";
  char tmp[64];
  snprintf(tmp, sizeof(tmp), "%lld %lld %lld\n", (long long)m, (long long)n, (long long)nnz);
  s += tmp;
  s.reserve(s.size() + (size_t)nnz * 40);
  for (int64_t r = 0; r < m; ++r)
    for (int64_t k = row_ptr_host[r]; k < row_ptr_host[r + 1]; ++k) {
      snprintf(tmp, sizeof(tmp), "%lld %lld ", (long long)(r + 1), (long long)(col_host[k] + 1));
      s += tmp;
      put_double(s, vals_host[k]);
      s += '\n';
    }
  return flush_file(path, s);
}

int svdsb_mm_write_array(const char *path, int64_t m, int64_t n, const double *a_host, int64_t lda) {
  if (!path || m < 0 || n < 0 || (m * n > 0 && (!a_host || lda < m))) {
    set_error("svdsb_mm_write_array: bad argument");
    return SVDSB_ERR_ARG;
  }
  std::string s = "%%MatrixMarket matrix array real general\n";
  char tmp[64];
  snprintf(tmp, sizeof(tmp), "%lld %lld\n", (long long)m, (long long)n);
  s += tmp;
  s.reserve(s.size() + (size_t)(m * n) * 26);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      put_double(s, a_host[i + j * lda]);
      s += '\n';
    }
  return flush_file(path, s);
}

}  // extern "C"
