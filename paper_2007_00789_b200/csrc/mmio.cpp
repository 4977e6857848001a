// Matrix Market reader (host C++, multi-threaded): the input side of the
// reference, /root/reference/pkg/src/spdkit/sparse.py:98-160
// (read_matrix_market) -- `matrix coordinate real symmetric` only, one
// triangle stored, both materialised, 1-based indices.
//
// The file is mapped into memory once; line starts are found in one pass;
// entry lines are tokenised and converted on all host threads; duplicate
// and mirror checks are a sort of (key, line) pairs.  Errors follow the
// reference's sequential semantics: the FIRST offending line in file order
// is reported, with the check order of one line (token count / conversion,
// index range, duplicate, mirror value).  The Python side formats the
// message from the returned line (sparse.py), so the texts are the
// reference's.
//
// Numbers are accepted exactly where Python's int() / float() accept them:
// optional sign, digits with single underscores between digits, for floats
// an optional fraction and exponent or inf / infinity / nan; strtod then
// converts (correctly rounded, like CPython's float()).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

// whitespace tokens of [b, e)
int split(const char* b, const char* e, const char** tb, const char** te, int maxtok) {
  int n = 0;
  const char* p = b;
  while (p < e) {
    while (p < e && is_ws(*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_ws(*p)) ++p;
    if (n < maxtok) {
      tb[n] = s;
      te[n] = p;
    }
    ++n;
  }
  return n;
}

// digits with single underscores between digits; copies the digits to out
bool digit_run(const char*& p, const char* e, std::string& out) {
  if (p >= e || !isdigit((unsigned char)*p)) return false;
  while (p < e) {
    if (isdigit((unsigned char)*p)) {
      out.push_back(*p++);
    } else if (*p == '_' && p + 1 < e && isdigit((unsigned char)p[1]) &&
               isdigit((unsigned char)p[-1])) {
      ++p;
    } else {
      break;
    }
  }
  return true;
}

// Python int(): [+-]digits; false on syntax error; *overflow on |v| >= 2^63
bool py_int(const char* b, const char* e, int64_t* v, bool* overflow) {
  std::string d;
  const char* p = b;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (!digit_run(p, e, d) || p != e) return false;
  *overflow = false;
  int64_t x = 0;
  for (char c : d) {
    if (x > (INT64_MAX - (c - '0')) / 10) {
      *overflow = true;
      x = INT64_MAX;
      break;
    }
    x = x * 10 + (c - '0');
  }
  *v = neg ? -x : x;
  return true;
}

bool ieq(const char* b, const char* e, const char* w) {
  const size_t n = strlen(w);
  if ((size_t)(e - b) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if (tolower((unsigned char)b[i]) != w[i]) return false;
  return true;
}

// Python float()
bool py_float(const char* b, const char* e, double* v) {
  const char* p = b;
  std::string s;
  if (p < e && (*p == '+' || *p == '-')) s.push_back(*p++);
  if (ieq(p, e, "inf") || ieq(p, e, "infinity")) {
    *v = (s == "-") ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(p, e, "nan")) {
    *v = (s == "-") ? -NAN : NAN;
    return true;
  }
  bool any = digit_run(p, e, s);
  if (p < e && *p == '.') {
    s.push_back(*p++);
    if (digit_run(p, e, s)) any = true;
  }
  if (!any) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    s.push_back(*p++);
    if (p < e && (*p == '+' || *p == '-')) s.push_back(*p++);
    if (!digit_run(p, e, s)) return false;
  }
  if (p != e) return false;
  *v = strtod(s.c_str(), nullptr);
  return true;
}

struct Entry {
  int64_t i, j;   // 0-based
  double v;
  int32_t err;    // 0 ok, 7 bad entry line, 8 index out of range
};

struct Reader {
  std::vector<char> buf;
  int64_t n = 0, nnz_decl = 0;
  std::vector<Entry> ent;
  int code = 0;          // first error (see spand_mm_read)
  int64_t err_line = -1; // 0-based index of the offending entry, or line number
  double mirror_value = 0.0;
  std::vector<int64_t> rp, ci;
  std::vector<double> va;
};

}  // namespace

extern "C" {

// Parse a Matrix Market file.  Returns a handle; info[8] = {code, n, nnz
// (stored, both triangles), err_entry, bits(mirror value), header_end,
// size_line_begin, size_line_end}.  code: 0 ok, 1 bad header, 2 unsupported
// object/format, 3 not real symmetric, 4 bad size line, 5 not square, 6 file
// ends early, 7 bad entry line, 8 index out of range, 9 duplicate entry,
// 10 mirror values disagree, 11 cannot open.  For codes 6-10 err_entry is the
// entry number (0-based, in file order); the entry's text is returned by
// spand_mm_line.
void* spand_mm_read(const char* path, int64_t* info) {
  Reader* R = new Reader();
  for (int k = 0; k < 8; ++k) info[k] = 0;
  FILE* f = fopen(path, "rb");
  if (!f) {
    R->code = 11;
    info[0] = 11;
    return R;
  }
  fseek(f, 0, SEEK_END);
  const long len = ftell(f);
  fseek(f, 0, SEEK_SET);
  R->buf.resize((size_t)len + 1);
  const size_t got = len > 0 ? fread(R->buf.data(), 1, (size_t)len, f) : 0;
  fclose(f);
  R->buf.resize(got);
  const char* b = R->buf.data();
  const char* end = b + got;
  // line starts
  std::vector<int64_t> ls;
  ls.reserve(got / 16 + 2);
  ls.push_back(0);
  for (const char* p = b; p < end; ++p) {
    const char* q = (const char*)memchr(p, '\n', end - p);
    if (!q) break;
    p = q;
    if (q + 1 < end) ls.push_back(q + 1 - b);
  }
  const int64_t nl = got ? (int64_t)ls.size() : 0;
  auto line_end = [&](int64_t L) { return L + 1 < nl ? b + ls[L + 1] : end; };
  // header
  const char* tb[8];
  const char* te[8];
  int64_t L = 0;
  {
    const char* hb = nl ? b + ls[0] : end;
    const char* he = nl ? line_end(0) : end;
    info[5] = he - b;
    const int nt = split(hb, he, tb, te, 8);
    auto tok = [&](int k) { return std::string(tb[k], te[k]); };
    auto lower = [](std::string x) {
      for (auto& c : x) c = (char)tolower((unsigned char)c);
      return x;
    };
    if (nt != 5 || tok(0) != "%%MatrixMarket") R->code = 1;
    else if (lower(tok(1)) != "matrix" || lower(tok(2)) != "coordinate") R->code = 2;
    else if (lower(tok(3)) != "real" || lower(tok(4)) != "symmetric") R->code = 3;
    if (R->code) {
      info[0] = R->code;
      return R;
    }
    L = 1;
  }
  // comments / blank lines, then the size line
  while (L < nl) {
    const char* lb = b + ls[L];
    const char* le = line_end(L);
    const char* t[1];
    const char* u[1];
    if (*lb == '%' || split(lb, le, t, u, 1) == 0) {
      ++L;
      continue;
    }
    break;
  }
  {
    const char* lb = L < nl ? b + ls[L] : end;
    const char* le = L < nl ? line_end(L) : end;
    info[6] = lb - b;
    info[7] = le - b;
    int64_t v[3];
    bool ok = split(lb, le, tb, te, 8) == 3, ovf = false;
    for (int k = 0; ok && k < 3; ++k) ok = py_int(tb[k], te[k], &v[k], &ovf);
    if (!ok) {
      R->code = 4;
      info[0] = 4;
      return R;
    }
    if (v[0] != v[1]) {
      R->code = 5;
      info[0] = 5;
      return R;
    }
    R->n = v[1];
    R->nnz_decl = v[2] > 0 ? v[2] : 0;
    ++L;
  }
  const int64_t n = R->n, ne = R->nnz_decl;
  const int64_t have = std::max<int64_t>(0, std::min<int64_t>(ne, nl - L));
  R->ent.resize(have);
  // entry lines on all host threads
  {
    const int nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < nth; ++t)
      th.emplace_back([&, t]() {
        const char* tb2[4];
        const char* te2[4];
        for (int64_t e = have * t / nth; e < have * (t + 1) / nth; ++e) {
          Entry& x = R->ent[e];
          x.err = 0;
          const char* lb = b + ls[L + e];
          const char* le = line_end(L + e);
          bool ovf_i = false, ovf_j = false;
          int64_t i = 0, j = 0;
          double v = 0.0;
          if (split(lb, le, tb2, te2, 4) != 3 || !py_int(tb2[0], te2[0], &i, &ovf_i) ||
              !py_int(tb2[1], te2[1], &j, &ovf_j) || !py_float(tb2[2], te2[2], &v)) {
            x.err = 7;
            continue;
          }
          if (ovf_i || ovf_j || i < 1 || i > n || j < 1 || j > n) {
            x.err = 8;
            continue;
          }
          x.i = i - 1;
          x.j = j - 1;
          x.v = v;
        }
      });
    for (auto& x : th) x.join();
  }
  // duplicates and mirror values: sort (key, entry) pairs
  std::vector<std::pair<int64_t, int64_t>> keys;
  keys.reserve(have);
  for (int64_t e = 0; e < have; ++e)
    if (!R->ent[e].err) keys.push_back({R->ent[e].i * n + R->ent[e].j, e});
  std::sort(keys.begin(), keys.end());
  std::vector<int32_t> kerr(have, 0);
  auto first_of = [&](int64_t key) -> int64_t {
    auto it = std::lower_bound(keys.begin(), keys.end(), std::make_pair(key, (int64_t)-1));
    return (it != keys.end() && it->first == key) ? it->second : -1;
  };
  for (size_t q = 0; q < keys.size(); ++q)
    if (q > 0 && keys[q].first == keys[q - 1].first) kerr[keys[q].second] = 9;
  double mv = 0.0;
  int64_t first_err = -1;
  int first_code = 0;
  for (int64_t e = 0; e < have; ++e) {
    int c = R->ent[e].err ? R->ent[e].err : kerr[e];
    if (!c) {
      const Entry& x = R->ent[e];
      if (x.i != x.j) {
        const int64_t m = first_of(x.j * n + x.i);
        if (m >= 0 && m < e && R->ent[m].v != x.v) {
          c = 10;
          mv = R->ent[m].v;
        }
      }
    }
    if (c) {
      first_err = e;
      first_code = c;
      break;
    }
  }
  if (first_code == 0 && have < ne) {
    first_code = 6;
    first_err = have;
  }
  if (first_code) {
    R->code = first_code;
    R->err_line = first_err;
    R->mirror_value = mv;
    info[0] = first_code;
    info[3] = first_err;
    std::memcpy(&info[4], &mv, 8);
    info[1] = n;
    // keep the entry's text available
    R->rp.assign(1, first_err < have ? ls[L + first_err] : (int64_t)got);
    R->ci.assign(1, first_err < have ? line_end(L + first_err) - b : (int64_t)got);
    return R;
  }
  // both triangles, CSR sorted by (row, col): entry (i, j), and (j, i)
  // when that mirror is not stored itself
  std::vector<std::pair<int64_t, double>> out;
  out.reserve(2 * have);
  for (int64_t e = 0; e < have; ++e) {
    const Entry& x = R->ent[e];
    out.push_back({x.i * n + x.j, x.v});
    if (x.i != x.j && first_of(x.j * n + x.i) < 0) out.push_back({x.j * n + x.i, x.v});
  }
  std::sort(out.begin(), out.end(),
            [](const std::pair<int64_t, double>& a, const std::pair<int64_t, double>& c) {
              return a.first < c.first;
            });
  R->rp.assign(n + 1, 0);
  R->ci.resize(out.size());
  R->va.resize(out.size());
  for (size_t q = 0; q < out.size(); ++q) {
    const int64_t r = out[q].first / n;
    R->ci[q] = out[q].first % n;
    R->va[q] = out[q].second;
    ++R->rp[r + 1];
  }
  for (int64_t r = 0; r < n; ++r) R->rp[r + 1] += R->rp[r];
  info[0] = 0;
  info[1] = n;
  info[2] = (int64_t)out.size();
  return R;
}

// the CSR arrays of a successful read (row_ptr n + 1, col_idx / values nnz)
int spand_mm_csr(void* h, int64_t* row_ptr, int64_t* col_idx, double* values) {
  Reader* R = static_cast<Reader*>(h);
  if (R->code) return -1;
  std::memcpy(row_ptr, R->rp.data(), R->rp.size() * sizeof(int64_t));
  std::memcpy(col_idx, R->ci.data(), R->ci.size() * sizeof(int64_t));
  std::memcpy(values, R->va.data(), R->va.size() * sizeof(double));
  return 0;
}

// byte range [begin, end) of the offending entry line of a failed read
int spand_mm_error_span(void* h, int64_t* span) {
  Reader* R = static_cast<Reader*>(h);
  if (!R->code || R->rp.empty()) return -1;
  span[0] = R->rp[0];
  span[1] = R->ci[0];
  return 0;
}

// copy bytes [b, e) of the file (header / size / entry line texts)
int spand_mm_text(void* h, int64_t b, int64_t e, char* out) {
  Reader* R = static_cast<Reader*>(h);
  if (b < 0 || e < b || e > (int64_t)R->buf.size()) return -1;
  std::memcpy(out, R->buf.data() + b, (size_t)(e - b));
  return 0;
}

void spand_mm_free(void* h) { delete static_cast<Reader*>(h); }

}  // extern "C"
