// MULTICUT text format: native parser and
// serializer for parse_instance / serialize_instance (graph.py:160-313).
//
// Host code only (no device work; the caller canonicalises the parsed COO
// on the GPU with rama_canonicalize).  The text is split into line-aligned
// chunks parsed by a thread pool with std::from_chars.  Acceptance and
// errors follow the reference exactly:
//   * header: the first non-blank, non-'#' line must read exactly MULTICUT;
//     an optional 'NODES <n>' line follows;
//   * edge block, fast path (np.loadtxt, graph.py:266-297): '#' starts a
//     comment anywhere, each remaining line has three numbers, ids integral;
//   * if anything is off, the line-by-line path (graph.py:160-201) decides
//     and its first failing line gives the ParseError message.
#include "../../include/rama_b200.h"
#include "internal.h"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fcntl.h>
#include <string>
#include <sys/mman.h>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>

namespace rama {
namespace {

// Python's str.splitlines() breaks (ASCII subset); \r\n counts as one
inline bool is_break(char ch) {
  return ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f' || ch == '\x1c' || ch == '\x1d' || ch == '\x1e';
}
// Python's str.split() / str.strip() whitespace (ASCII subset)
inline bool is_ws(char ch) {
  return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f' ||
         (ch >= '\x1c' && ch <= '\x1f');
}

struct Line {
  const char* b;
  const char* e;  // [b, e) without the break
};

// all lines of [p, q) (q ends at a break or at the end of the text)
void split_lines(const char* p, const char* q, std::vector<Line>& out) {
  while (p < q) {
    const char* e = p;
    while (e < q && !is_break(*e)) e++;
    out.push_back(Line{p, e});
    if (e < q) {
      if (*e == '\r' && e + 1 < q && e[1] == '\n') e++;
      e++;
    }
    p = e;
  }
}

inline void strip(const char*& b, const char*& e) {
  while (b < e && is_ws(*b)) b++;
  while (e > b && is_ws(e[-1])) e--;
}

int split_tokens(const char* b, const char* e, Line* tok, int max_tok) {
  int k = 0;
  while (b < e) {
    while (b < e && is_ws(*b)) b++;
    if (b == e) break;
    const char* s = b;
    while (b < e && !is_ws(*b)) b++;
    if (k < max_tok) tok[k] = Line{s, b};
    k++;
  }
  return k;
}

inline bool ieq(const char* b, const char* e, const char* lit) {
  size_t n = strlen(lit);
  if ((size_t)(e - b) != n) return false;
  for (size_t i = 0; i < n; i++)
    if (tolower((unsigned char)b[i]) != lit[i]) return false;
  return true;
}

// float token (numpy / Python float syntax without underscores)
bool parse_double(const char* b, const char* e, double* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    b++;
  }
  if (b == e) return false;
  if (ieq(b, e, "inf") || ieq(b, e, "infinity")) {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(b, e, "nan")) {
    *out = NAN;
    return true;
  }
  if (*b == '+' || *b == '-') return false;
  double x = 0.0;
  auto r = std::from_chars(b, e, x, std::chars_format::general);
  if (r.ec != std::errc() || r.ptr != e) {
    if (r.ec == std::errc::result_out_of_range && r.ptr == e) {  // overflow -> inf, underflow -> 0 (like strtod)
      x = std::strtod(std::string(b, e).c_str(), nullptr);
    } else {
      return false;
    }
  }
  *out = neg ? -x : x;
  return true;
}

// Python float(): also accepts single underscores between digits
bool parse_py_float(const char* b, const char* e, double* out) {
  std::string t;
  for (const char* p = b; p < e; p++) {
    if (*p == '_') {
      if (p == b || p + 1 == e || !isdigit((unsigned char)p[-1]) || !isdigit((unsigned char)p[1])) return false;
      continue;
    }
    t.push_back(*p);
  }
  return parse_double(t.data(), t.data() + t.size(), out);
}

// Python int(): optional sign, decimal digits, single underscores between digits
bool parse_py_int(const char* b, const char* e, int64_t* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    b++;
  }
  if (b == e || !isdigit((unsigned char)*b) || !isdigit((unsigned char)e[-1])) return false;
  __int128 x = 0;
  for (const char* p = b; p < e; p++) {
    if (*p == '_') {
      if (!isdigit((unsigned char)p[-1]) || !isdigit((unsigned char)p[1])) return false;
      continue;
    }
    if (!isdigit((unsigned char)*p)) return false;
    x = x * 10 + (*p - '0');
    if (x > ((__int128)1 << 62)) x = ((__int128)1 << 62);  // saturate: any such id is out of range anyway
  }
  *out = (int64_t)(neg ? -x : x);
  return true;
}

// Python repr() of an ASCII str (quotes, escapes)
std::string py_repr(const char* b, const char* e) {
  bool has_sq = std::find(b, e, '\'') != e, has_dq = std::find(b, e, '"') != e;
  char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string s(1, q);
  for (const char* p = b; p < e; p++) {
    unsigned char ch = (unsigned char)*p;
    if (ch == (unsigned char)q || ch == '\\') {
      s.push_back('\\');
      s.push_back((char)ch);
    } else if (ch == '\t') {
      s += "\\t";
    } else if (ch == '\n') {
      s += "\\n";
    } else if (ch == '\r') {
      s += "\\r";
    } else if (ch < 0x20 || ch == 0x7f) {
      char buf[8];
      snprintf(buf, sizeof(buf), "\\x%02x", ch);
      s += buf;
    } else {
      s.push_back((char)ch);
    }
  }
  s.push_back(q);
  return s;
}

struct Parsed {
  std::vector<int64_t> u, v;
  std::vector<double> c;
};

// graph.py:160-201, line by line; throws the reference's ParseError text
void parse_slow(const std::vector<Line>& lines, size_t start, int64_t declared, Parsed& out) {
  Line tok[4];
  for (size_t i = start; i < lines.size(); i++) {
    const int64_t lineno = (int64_t)i + 1;
    const char *b = lines[i].b, *e = lines[i].e;
    strip(b, e);
    if (b == e || *b == '#') continue;
    char msg[256];
    if (split_tokens(b, e, tok, 4) != 3) {
      std::string r = py_repr(lines[i].b, lines[i].e);
      throw Error(kInvalid, "line " + std::to_string(lineno) + ": expected '<u> <v> <cost>', got " + r);
    }
    int64_t a = 0, bb = 0;
    if (!parse_py_int(tok[0].b, tok[0].e, &a) || !parse_py_int(tok[1].b, tok[1].e, &bb)) {
      snprintf(msg, sizeof(msg), "line %lld: node ids must be decimal integers", (long long)lineno);
      throw Error(kInvalid, msg);
    }
    double w = 0.0;
    if (!parse_py_float(tok[2].b, tok[2].e, &w))
      throw Error(kInvalid, "line " + std::to_string(lineno) + ": malformed cost " + py_repr(tok[2].b, tok[2].e));
    if (!std::isfinite(w)) {
      snprintf(msg, sizeof(msg), "line %lld: cost must be finite", (long long)lineno);
      throw Error(kInvalid, msg);
    }
    if (a < 0 || bb < 0) {
      snprintf(msg, sizeof(msg), "line %lld: negative node id", (long long)lineno);
      throw Error(kInvalid, msg);
    }
    if (a == bb) {
      snprintf(msg, sizeof(msg), "line %lld: self-loop edge (%lld, %lld)", (long long)lineno, (long long)a,
               (long long)bb);
      throw Error(kInvalid, msg);
    }
    if (declared >= 0 && (a >= declared || bb >= declared)) {
      snprintf(msg, sizeof(msg), "line %lld: node id exceeds declared NODES %lld", (long long)lineno,
               (long long)declared);
      throw Error(kInvalid, msg);
    }
    out.u.push_back(a);
    out.v.push_back(bb);
    out.c.push_back(w);
  }
}

// np.loadtxt fast path (graph.py:266-297) for lines [lo, hi): false if any
// line is off (the caller then runs the line-by-line path)
bool parse_fast(const std::vector<Line>& lines, size_t lo, size_t hi, int64_t declared, Parsed& out) {
  Line tok[4];
  for (size_t i = lo; i < hi; i++) {
    const char *b = lines[i].b, *e = lines[i].e;
    const char* hash = (const char*)memchr(b, '#', e - b);
    if (hash) e = hash;
    strip(b, e);
    if (b == e) continue;
    if (split_tokens(b, e, tok, 4) != 3) return false;
    double x[3];
    for (int k = 0; k < 3; k++)
      if (!parse_double(tok[k].b, tok[k].e, &x[k]) || !std::isfinite(x[k])) return false;
    if (x[0] != std::floor(x[0]) || x[1] != std::floor(x[1]) || x[0] < 0 || x[1] < 0 || x[0] == x[1]) return false;
    if (x[0] > 9.0e15 || x[1] > 9.0e15) return false;
    if (declared >= 0 && (x[0] >= (double)declared || x[1] >= (double)declared)) return false;
    out.u.push_back((int64_t)x[0]);
    out.v.push_back((int64_t)x[1]);
    out.c.push_back(x[2]);
  }
  return true;
}

int pool_size(int32_t threads) {
  int t = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  return t < 1 ? 1 : (t > 64 ? 64 : t);
}

void parse_text(const char* text, int64_t len, int32_t threads, int64_t* n_out, Parsed& out) {
  std::vector<Line> lines;
  // line split in parallel over break-aligned byte chunks
  const int T = len > (1 << 20) ? pool_size(threads) : 1;
  std::vector<int64_t> cut(T + 1);
  cut[0] = 0;
  cut[T] = len;
  for (int t = 1; t < T; t++) {
    int64_t p = std::max(cut[t - 1], len * t / T);
    while (p < len && !is_break(text[p])) p++;
    if (p < len) {
      if (text[p] == '\r' && p + 1 < len && text[p + 1] == '\n') p++;
      p++;
    }
    cut[t] = p;
  }
  {
    std::vector<std::vector<Line>> part(T);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; t++)
      pool.emplace_back([&, t] { split_lines(text + cut[t], text + cut[t + 1], part[t]); });
    for (auto& th : pool) th.join();
    for (auto& p : part) lines.insert(lines.end(), p.begin(), p.end());
  }
  // header (graph.py:214-231)
  size_t idx = 0;
  bool header = false;
  while (idx < lines.size()) {
    const char *b = lines[idx].b, *e = lines[idx].e;
    strip(b, e);
    if (b == e || *b == '#') {
      idx++;
      continue;
    }
    if (!(lines[idx].e - lines[idx].b == 8 && memcmp(lines[idx].b, "MULTICUT", 8) == 0))
      throw Error(kInvalid, "line " + std::to_string(idx + 1) + ": expected MULTICUT header, got " +
                                py_repr(lines[idx].b, lines[idx].e));
    header = true;
    idx++;
    break;
  }
  if (!header) throw Error(kInvalid, "missing MULTICUT header");
  // optional NODES line (graph.py:233-249)
  int64_t declared = -1;
  for (size_t probe = idx; probe < lines.size(); probe++) {
    const char *b = lines[probe].b, *e = lines[probe].e;
    strip(b, e);
    if (b == e || *b == '#') continue;
    Line tok[3];
    int k = split_tokens(b, e, tok, 3);
    if (tok[0].e - tok[0].b == 5 && memcmp(tok[0].b, "NODES", 5) == 0) {
      std::string ln = std::to_string(probe + 1);
      if (k != 2) throw Error(kInvalid, "line " + ln + ": expected 'NODES <n>'");
      int64_t d = 0;
      if (!parse_py_int(tok[1].b, tok[1].e, &d)) throw Error(kInvalid, "line " + ln + ": NODES count must be an integer");
      if (d < 0) throw Error(kInvalid, "line " + ln + ": NODES count must be non-negative");
      declared = d;
      idx = probe + 1;
    }
    break;
  }
  // edge block: fast path in parallel, line-by-line path on any doubt
  const size_t nl = lines.size() - idx;
  const int P = nl > 65536 ? pool_size(threads) : 1;
  std::vector<Parsed> part(P);
  std::vector<char> ok(P, 1);
  {
    std::vector<std::thread> pool;
    for (int t = 0; t < P; t++)
      pool.emplace_back([&, t] {
        size_t lo = idx + nl * t / P, hi = idx + nl * (t + 1) / P;
        ok[t] = parse_fast(lines, lo, hi, declared, part[t]);
      });
    for (auto& th : pool) th.join();
  }
  bool fast = std::all_of(ok.begin(), ok.end(), [](char x) { return x != 0; });
  bool any = false;
  for (auto& p : part) any |= !p.u.empty();
  if (fast && any) {
    size_t m = 0;
    for (auto& p : part) m += p.u.size();
    out.u.reserve(m);
    out.v.reserve(m);
    out.c.reserve(m);
    for (auto& p : part) {
      out.u.insert(out.u.end(), p.u.begin(), p.u.end());
      out.v.insert(out.v.end(), p.v.begin(), p.v.end());
      out.c.insert(out.c.end(), p.c.begin(), p.c.end());
    }
  } else {
    parse_slow(lines, idx, declared, out);
  }
  int64_t n = 0;
  if (declared >= 0) {
    n = declared;
  } else if (!out.u.empty()) {
    n = std::max(*std::max_element(out.u.begin(), out.u.end()), *std::max_element(out.v.begin(), out.v.end())) + 1;
  }
  *n_out = n;
}

// Python repr(float): shortest round-trip digits, fixed notation for
// -4 <= exponent < 16 (always with a fractional part), else d.ddde+XX
int py_float_repr(double x, char* buf) {
  if (std::isnan(x)) return sprintf(buf, "nan");
  if (std::isinf(x)) return sprintf(buf, x < 0 ? "-inf" : "inf");
  if (x == 0.0) return sprintf(buf, std::signbit(x) ? "-0.0" : "0.0");
  char sci[64];
  auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
  *r.ptr = 0;
  // sci: [-]d[.ddd]e[+-]XX
  const char* p = sci;
  bool neg = *p == '-';
  if (neg) p++;
  char digits[32];
  int nd = 0;
  const char* q = p;
  for (; *q && *q != 'e'; q++)
    if (*q != '.') digits[nd++] = *q;
  int exp10 = atoi(q + 1);
  char* o = buf;
  if (neg) *o++ = '-';
  if (exp10 >= -4 && exp10 < 16) {
    if (exp10 < 0) {
      *o++ = '0';
      *o++ = '.';
      for (int k = 0; k < -exp10 - 1; k++) *o++ = '0';
      for (int k = 0; k < nd; k++) *o++ = digits[k];
    } else {
      for (int k = 0; k <= exp10; k++) *o++ = k < nd ? digits[k] : '0';
      *o++ = '.';
      if (nd > exp10 + 1) {
        for (int k = exp10 + 1; k < nd; k++) *o++ = digits[k];
      } else {
        *o++ = '0';
      }
    }
  } else {
    *o++ = digits[0];
    if (nd > 1) {
      *o++ = '.';
      for (int k = 1; k < nd; k++) *o++ = digits[k];
    }
    o += sprintf(o, "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
  }
  *o = 0;
  return (int)(o - buf);
}

}  // namespace
}  // namespace rama

using namespace rama;

namespace {
thread_local std::string g_io_err;

template <class F>
int guarded_host(F&& f) {
  g_io_err.clear();
  try {
    f();
    return RAMA_OK;
  } catch (const Error& e) {
    g_io_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_io_err = e.what();
    return RAMA_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

const char* rama_io_last_error(void) { return g_io_err.c_str(); }

int rama_parse_multicut(const char* text, int64_t len, const char* path, int64_t* n, int64_t* m, int64_t* u,
                        int64_t* v, double* c, int64_t cap, int32_t threads) {
  return guarded_host([&] {
    const char* data = text;
    int64_t size = len;
    void* map = nullptr;
    int fd = -1;
    if (path) {
      fd = open(path, O_RDONLY);
      if (fd < 0) throw Error(kInvalid, std::string("cannot open ") + path);
      struct stat st;
      if (fstat(fd, &st) != 0) {
        close(fd);
        throw Error(kInvalid, std::string("cannot stat ") + path);
      }
      size = st.st_size;
      if (size > 0) {
        map = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
        if (map == MAP_FAILED) {
          close(fd);
          throw Error(kInvalid, std::string("cannot map ") + path);
        }
        madvise(map, size, MADV_SEQUENTIAL);
      }
      data = (const char*)map;
    }
    struct Unmap {
      void* p;
      int64_t s;
      int fd;
      ~Unmap() {
        if (p) munmap(p, s);
        if (fd >= 0) close(fd);
      }
    } guard{map, size, fd};
    Parsed out;
    int64_t nn = 0;
    if (size > 0) {
      parse_text(data, size, threads, &nn, out);
    } else {
      throw Error(kInvalid, "missing MULTICUT header");
    }
    *n = nn;
    *m = (int64_t)out.u.size();
    if ((int64_t)out.u.size() > cap) return;  // caller retries with *m capacity
    memcpy(u, out.u.data(), out.u.size() * sizeof(int64_t));
    memcpy(v, out.v.data(), out.v.size() * sizeof(int64_t));
    memcpy(c, out.c.data(), out.c.size() * sizeof(double));
  });
}

int rama_serialize_multicut(int64_t n, const int64_t* u, const int64_t* v, const double* c, int64_t m, char* out,
                            int64_t cap, int64_t* len, int32_t threads) {
  return guarded_host([&] {
    char head[64];
    int hl = snprintf(head, sizeof(head), "MULTICUT\nNODES %lld\n", (long long)n);
    const int T = m > (1 << 16) ? pool_size(threads) : 1;
    std::vector<std::string> part(T);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; t++)
      pool.emplace_back([&, t] {
        int64_t lo = m * t / T, hi = m * (t + 1) / T;
        std::string& s = part[t];
        s.reserve((size_t)(hi - lo) * 32);
        char buf[96];
        for (int64_t i = lo; i < hi; i++) {
          int k = snprintf(buf, sizeof(buf), "%lld %lld ", (long long)u[i], (long long)v[i]);
          k += py_float_repr(c[i], buf + k);
          buf[k++] = '\n';
          s.append(buf, k);
        }
      });
    for (auto& th : pool) th.join();
    int64_t total = hl;
    for (auto& s : part) total += (int64_t)s.size();
    *len = total;
    if (!out || cap < total) return;
    memcpy(out, head, hl);
    int64_t at = hl;
    for (auto& s : part) {
      memcpy(out + at, s.data(), s.size());
      at += (int64_t)s.size();
    }
  });
}

}  // extern "C"
