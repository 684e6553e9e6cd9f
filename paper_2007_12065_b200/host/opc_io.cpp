// libopcfe_io.so: organized point-cloud ingestion (include/opcfe_io.h).
//
// Host-side, parallel and allocation-free on the data path: the caller owns the output
// buffer (typically pinned host memory that the front end's H2D copy reads), text bodies
// are split at line boundaries and parsed by all cores, and binary PLY whose vertex record
// is three little-endian doubles is read straight into that buffer with pread().
//
// Reference semantics followed (file:line in /root/reference/pkg/src/flatpoly/io.py):
//   * _parse_floats (:31-37): >= 3 tokens, the first 3 parsed with Python float();
//   * load_xyz / load_grid (:40-78): blank lines and lines whose first token starts with
//     '#' are skipped; the grid header is the first such line, two ints "M N"; errors
//     "grid header must be two integers 'M N'", "missing or invalid grid header",
//     "expected {M*N} rows, got {k}" (reported at the last line), parse errors first;
//   * PLY (:97-184): "ply" magic, format ascii | binary_little_endian, "comment grid M N",
//     element / property (list) declarations, "end_header"; the vertex element's x, y, z
//     of any numeric type as float64; ascii reads exactly `count` lines;
//   * write_ply (:187-212) and load_cloud (:238-266).
#include "../../include/opcfe_io.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_line = 0;

int fail(int code, const std::string& path, int64_t line, const std::string& what) {
  g_err = path + ":" + std::to_string(line) + ": " + what;
  g_err_line = line;
  return code;
}
int fail_os(const std::string& path, const char* what) {
  g_err = path + ": " + what + ": " + std::strerror(errno);
  g_err_line = 0;
  return OPCFE_IO_ERR_OS;
}

// Python str.split() whitespace for the ASCII range
inline bool is_ws(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

// Text files are read the way the reference's text-mode open() sees them (io.py:43, :55):
// universal newlines (\n, \r\n and a lone \r each end a line) and str.split()'s Unicode
// whitespace in the UTF-8 decoding (U+0085, U+00A0, U+1680, U+2000-U+200A, U+2028,
// U+2029, U+202F, U+205F, U+3000).  Files without any \r / non-ASCII byte (the usual
// case, checked once) take the plain byte paths.
struct TextMode {
  bool cr = false;    // a '\r' somewhere: universal newlines
  bool utf8 = false;  // a byte >= 0x80 somewhere: multi-byte whitespace
};
TextMode g_text_plain;  // PLY bodies / headers: bytes, '\n' lines (binary-mode readline)

// length of the Unicode whitespace sequence at p (0 if none)
inline int ws_len(const char* p, const char* e, const TextMode& m) {
  const unsigned char c = (unsigned char)*p;
  if (c < 0x80) return is_ws(c) ? 1 : 0;
  if (!m.utf8) return 0;
  const unsigned char* u = reinterpret_cast<const unsigned char*>(p);
  const ptrdiff_t n = e - p;
  if (c == 0xC2 && n >= 2 && (u[1] == 0x85 || u[1] == 0xA0)) return 2;
  if (c == 0xE1 && n >= 3 && u[1] == 0x9A && u[2] == 0x80) return 3;
  if (c == 0xE2 && n >= 3 && u[1] == 0x80 &&
      (u[2] <= 0x8A || u[2] == 0xA8 || u[2] == 0xA9 || u[2] == 0xAF))
    return 3;
  if (c == 0xE2 && n >= 3 && u[1] == 0x81 && u[2] == 0x9F) return 3;
  if (c == 0xE3 && n >= 3 && u[1] == 0x80 && u[2] == 0x80) return 3;
  return 0;
}

// ---------------------------------------------------------------- Python float()
// Accepts exactly what CPython's float(str) accepts for an ASCII token: optional sign,
// then inf / infinity / nan (any case) or a decimal literal whose digit groups may be
// separated by single underscores.  The value is strtod's (correctly rounded, as
// CPython's dtoa).  Returns false (and leaves *out) for anything float() rejects.
bool py_float(const char* b, const char* e, double* out) {
  char buf[128];
  const size_t n = (size_t)(e - b);
  if (n == 0 || n >= sizeof(buf)) {
    if (n == 0) return false;
    std::string s(b, e);  // long literal: same rules, heap buffer
    std::string t;
    for (size_t i = 0; i < s.size(); ++i) {
      if (s[i] == '_') {
        if (i == 0 || i + 1 >= s.size() || !isdigit((unsigned char)s[i - 1]) ||
            !isdigit((unsigned char)s[i + 1]))
          return false;
        continue;
      }
      t.push_back(s[i]);
    }
    return py_float(t.data(), t.data() + t.size(), out);
  }
  // strip digit-separating underscores
  size_t m = 0;
  for (size_t i = 0; i < n; ++i) {
    const char c = b[i];
    if (c == '_') {
      if (i == 0 || i + 1 >= n || !isdigit((unsigned char)b[i - 1]) ||
          !isdigit((unsigned char)b[i + 1]))
        return false;
      continue;
    }
    buf[m++] = c;
  }
  buf[m] = 0;
  const char* p = buf;
  if (*p == '+' || *p == '-') ++p;
  auto ieq = [](const char* a, const char* lit) {
    for (; *lit; ++a, ++lit)
      if (std::tolower((unsigned char)*a) != *lit) return false;
    return *a == 0;
  };
  if (ieq(p, "inf") || ieq(p, "infinity") || ieq(p, "nan")) {
    *out = std::strtod(buf, nullptr);
    return true;
  }
  // decimal literal: digits [. digits] [e [sign] digits], at least one mantissa digit
  const char* q = p;
  int mant = 0;
  while (isdigit((unsigned char)*q)) ++q, ++mant;
  if (*q == '.') {
    ++q;
    while (isdigit((unsigned char)*q)) ++q, ++mant;
  }
  if (mant == 0) return false;
  if (*q == 'e' || *q == 'E') {
    ++q;
    if (*q == '+' || *q == '-') ++q;
    if (!isdigit((unsigned char)*q)) return false;
    while (isdigit((unsigned char)*q)) ++q;
  }
  if (*q != 0) return false;
  *out = std::strtod(buf, nullptr);
  return true;
}

// Python int(str) for the grid header (sign, digits, single underscores between digits)
bool py_int(const char* b, const char* e, int64_t* out) {
  std::string t;
  size_t n = (size_t)(e - b);
  for (size_t i = 0; i < n; ++i) {
    const char c = b[i];
    if (c == '_') {
      if (i == 0 || i + 1 >= n || !isdigit((unsigned char)b[i - 1]) ||
          !isdigit((unsigned char)b[i + 1]))
        return false;
      continue;
    }
    t.push_back(c);
  }
  const char* p = t.c_str();
  if (*p == '+' || *p == '-') ++p;
  if (!*p) return false;
  for (const char* q = p; *q; ++q)
    if (!isdigit((unsigned char)*q)) return false;
  errno = 0;
  const long long v = std::strtoll(t.c_str(), nullptr, 10);
  if (errno == ERANGE) return false;
  *out = v;
  return true;
}

// ------------------------------------------------------------------ mapped file
struct Mapped {
  int fd = -1;
  const char* p = nullptr;
  size_t n = 0;
  ~Mapped() {
    if (p && n) munmap(const_cast<char*>(p), n);
    if (fd >= 0) close(fd);
  }
  int open_(const std::string& path) {
    fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) return fail_os(path, "cannot open");
    struct stat st;
    if (fstat(fd, &st) != 0) return fail_os(path, "cannot stat");
    n = (size_t)st.st_size;
    if (n == 0) {
      p = "";
      return OPCFE_IO_OK;
    }
    void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) return fail_os(path, "cannot map");
    madvise(m, n, MADV_SEQUENTIAL);
    p = static_cast<const char*>(m);
    return OPCFE_IO_OK;
  }
};

struct Tok {
  const char* b;
  const char* e;
};

// split [b, e) (one line, no line terminator) into up to `cap` tokens; returns the count
int split(const char* b, const char* e, Tok* t, int cap, const TextMode& m = g_text_plain) {
  int k = 0;
  if (!m.utf8) {
    while (b < e) {
      while (b < e && is_ws((unsigned char)*b)) ++b;
      if (b >= e) break;
      const char* s = b;
      while (b < e && !is_ws((unsigned char)*b)) ++b;
      if (k < cap) t[k] = Tok{s, b};
      ++k;
    }
    return k;
  }
  while (b < e) {
    int w;
    while (b < e && (w = ws_len(b, e, m)) > 0) b += w;
    if (b >= e) break;
    const char* s = b;
    while (b < e && ws_len(b, e, m) == 0) ++b;
    if (k < cap) t[k] = Tok{s, b};
    ++k;
  }
  return k;
}

// end of the line starting at b: the first '\n' (or, universal newlines, '\r')
inline const char* line_end(const char* b, const char* e, const TextMode& m = g_text_plain) {
  if (!m.cr) {
    const void* q = memchr(b, '\n', (size_t)(e - b));
    return q ? static_cast<const char*>(q) : e;
  }
  while (b < e && *b != '\n' && *b != '\r') ++b;
  return b;
}
// start of the next line after the terminator at le ("\r\n" is one terminator)
inline const char* next_line(const char* le, const char* e, const TextMode& m = g_text_plain) {
  if (le >= e) return e;
  if (m.cr && *le == '\r' && le + 1 < e && le[1] == '\n') return le + 2;
  return le + 1;
}
TextMode text_mode(const char* b, const char* e) {
  TextMode m;
  m.cr = memchr(b, '\r', (size_t)(e - b)) != nullptr;
  for (const char* p = b; p < e; ++p)
    if ((unsigned char)*p >= 0x80) {
      m.utf8 = true;
      break;
    }
  return m;
}

// A text body parsed in parallel.  Mode kRows: skip blank / '#' lines, every other line
// is a data row with >= 3 float tokens (xyz, grid).  Mode kPly: exactly `count` lines,
// tokens at fixed indices (PLY ascii vertex element).
enum Mode { kRows, kPly };

struct ChunkStat {
  const char* b;
  const char* e;
  int64_t lines = 0, rows = 0;    // pass 1
  int64_t line0 = 0, row0 = 0;    // prefix
  int64_t err_line = 0;           // pass 2: first error in the chunk
  int err_code = 0;
  std::string err;
};

int nthreads(int want, size_t bytes) {
  int hw = (int)std::thread::hardware_concurrency();
  if (hw < 1) hw = 1;
  int t = want > 0 ? want : hw;
  const int by_size = (int)std::max<size_t>(1, bytes / (1u << 20));  // >= 1 MiB per thread
  return std::max(1, std::min(t, by_size));
}

template <typename F>
void parallel(int T, F fn) {
  if (T == 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (int i = 0; i < T; ++i) th.emplace_back(fn, i);
  for (auto& t : th) t.join();
}

std::vector<ChunkStat> chunk(const char* b, const char* e, int T, const TextMode& m) {
  std::vector<ChunkStat> c(T);
  const size_t n = (size_t)(e - b);
  const char* s = b;
  for (int i = 0; i < T; ++i) {
    const char* x = (i == T - 1) ? e : b + n * (size_t)(i + 1) / (size_t)T;
    if (x < s) x = s;
    if (x < e) {  // end the chunk after a line terminator (never inside "\r\n")
      if (m.cr && x > b && x[-1] == '\r' && *x == '\n') ++x;
      else {
        const char* nl = line_end(x, e, m);
        x = next_line(nl, e, m);
      }
    }
    c[i].b = s;
    c[i].e = x;
    s = x;
  }
  return c;
}

inline bool skip_line(const Tok* t, int k) { return k == 0 || t[0].b[0] == '#'; }

// count lines and data rows of each chunk (pass 1)
void count_pass(std::vector<ChunkStat>& cs, Mode mode, int T, const TextMode& m) {
  parallel(T, [&](int i) {
    ChunkStat& c = cs[i];
    for (const char* p = c.b; p < c.e;) {
      const char* le = line_end(p, c.e, m);
      ++c.lines;
      if (mode == kRows) {
        Tok t[1];
        if (!skip_line(t, split(p, le, t, 1, m))) ++c.rows;
      } else {
        ++c.rows;
      }
      p = next_line(le, c.e, m);
    }
  });
  int64_t l = 0, r = 0;
  for (auto& c : cs) {
    c.line0 = l;
    c.row0 = r;
    l += c.lines;
    r += c.rows;
  }
}

std::string not_float_msg(const Tok& t) {
  return "could not convert string to float: '" + std::string(t.b, t.e) + "'";
}

// parse rows (pass 2); dst == nullptr validates only.  Rows beyond `max_rows` are
// validated but not stored.  line_base = line number of the body's first line.
void parse_pass(std::vector<ChunkStat>& cs, Mode mode, int T, double* dst, int64_t max_rows,
                int64_t line_base, const int* idx, int max_idx, const TextMode& m) {
  parallel(T, [&](int i) {
    ChunkStat& c = cs[i];
    int64_t line = line_base + c.line0, row = c.row0;
    for (const char* p = c.b; p < c.e; ++line) {
      const char* le = line_end(p, c.e, m);
      Tok t[64];
      const int k = split(p, le, t, 64, m);
      p = next_line(le, c.e, m);
      if (mode == kRows && skip_line(t, k)) continue;
      double v[3];
      if (mode == kRows) {
        if (k < 3) {
          c.err_line = line;
          c.err = "expected 3 values, got " + std::to_string(k);
          c.err_code = OPCFE_IO_ERR_PARSE;
          return;
        }
        for (int j = 0; j < 3; ++j)
          if (!py_float(t[j].b, t[j].e, &v[j])) {
            c.err_line = line;
            c.err = not_float_msg(t[j]);
            c.err_code = OPCFE_IO_ERR_PARSE;
            return;
          }
      } else {
        if (k <= max_idx || max_idx >= 64) {
          c.err_line = line;
          c.err = "vertex row has " + std::to_string(k) + " values";
          c.err_code = OPCFE_IO_ERR_PARSE;
          return;
        }
        for (int j = 0; j < 3; ++j)
          if (!py_float(t[idx[j]].b, t[idx[j]].e, &v[j])) {
            c.err_line = line;
            c.err = not_float_msg(t[idx[j]]);
            c.err_code = OPCFE_IO_ERR_PARSE;
            return;
          }
      }
      if (dst && row < max_rows) {
        dst[3 * row] = v[0];
        dst[3 * row + 1] = v[1];
        dst[3 * row + 2] = v[2];
      }
      ++row;
    }
  });
}

int first_error(const std::vector<ChunkStat>& cs, const std::string& path) {
  for (const auto& c : cs)
    if (c.err_code) return fail(c.err_code, path, c.err_line, c.err);
  return OPCFE_IO_OK;
}

// ------------------------------------------------------------------------ PLY
int type_size(const std::string& t, char* code) {
  struct E {
    const char* n;
    char c;
    int s;
  };
  static const E tab[] = {{"float", 'f', 4}, {"float32", 'f', 4}, {"double", 'd', 8},
                          {"float64", 'd', 8}, {"char", 'b', 1},  {"int8", 'b', 1},
                          {"uchar", 'B', 1},   {"uint8", 'B', 1},  {"short", 'h', 2},
                          {"int16", 'h', 2},   {"ushort", 'H', 2}, {"uint16", 'H', 2},
                          {"int", 'i', 4},     {"int32", 'i', 4},  {"uint", 'I', 4},
                          {"uint32", 'I', 4}};
  for (const auto& e : tab)
    if (t == e.n) {
      *code = e.c;
      return e.s;
    }
  return 0;
}

inline double load_le(const char* p, int code) {
  switch (code) {
    case 'f': { float v; memcpy(&v, p, 4); return v; }
    case 'd': { double v; memcpy(&v, p, 8); return v; }
    case 'b': return (double)(int8_t)p[0];
    case 'B': return (double)(uint8_t)p[0];
    case 'h': { int16_t v; memcpy(&v, p, 2); return v; }
    case 'H': { uint16_t v; memcpy(&v, p, 2); return v; }
    case 'i': { int32_t v; memcpy(&v, p, 4); return v; }
    default: { uint32_t v; memcpy(&v, p, 4); return v; }
  }
}

int probe_ply(const Mapped& m, const std::string& path, opcfe_cloud_info* info) {
  const char* p = m.p;
  const char* e = m.p + m.n;
  int64_t line_no = 1;
  const char* le = line_end(p, e);
  {
    Tok t[2];
    const int k = split(p, le, t, 2);
    if (!(k == 1 && t[0].e - t[0].b == 3 && memcmp(t[0].b, "ply", 3) == 0))
      return fail(OPCFE_IO_ERR_PARSE, path, 1, "not a PLY file");
  }
  p = le < e ? le + 1 : e;
  std::string fmt;
  struct Elem {
    std::string name;
    int64_t count;
    std::vector<std::pair<std::string, std::string>> props;  // (name, type) or ("list", ...)
    bool has_list = false;
    std::string list_count_t, list_item_t;  // the first list property's types (faces)
  };
  std::vector<Elem> els;
  int64_t gm = -1, gn = -1;
  while (true) {
    if (p >= e) return fail(OPCFE_IO_ERR_PARSE, path, line_no + 1, "unexpected end of header");
    le = line_end(p, e);
    ++line_no;
    Tok t[8];
    const int k = split(p, le, t, 8);
    const char* next = le < e ? le + 1 : e;
    if (k == 0) {
      p = next;
      continue;
    }
    const std::string w0(t[0].b, t[0].e);
    if (w0 == "format") {
      fmt = k > 1 ? std::string(t[1].b, t[1].e) : "";
    } else if (w0 == "comment") {
      if (k == 4 && std::string(t[1].b, t[1].e) == "grid") {
        if (!py_int(t[2].b, t[2].e, &gm) || !py_int(t[3].b, t[3].e, &gn))
          return fail(OPCFE_IO_ERR_PARSE, path, line_no, "invalid grid comment");
      }
    } else if (w0 == "element") {
      int64_t cnt = 0;
      if (k < 3 || !py_int(t[2].b, t[2].e, &cnt))
        return fail(OPCFE_IO_ERR_PARSE, path, line_no, "invalid element line");
      els.push_back(Elem{std::string(t[1].b, t[1].e), cnt, {}, false, "", ""});
    } else if (w0 == "property") {
      if (els.empty()) return fail(OPCFE_IO_ERR_PARSE, path, line_no, "property before element");
      if (k >= 2 && std::string(t[1].b, t[1].e) == "list") {
        if (!els.back().has_list && k >= 4) {
          els.back().list_count_t = std::string(t[2].b, t[2].e);
          els.back().list_item_t = std::string(t[3].b, t[3].e);
        }
        els.back().has_list = true;
        els.back().props.emplace_back("list", k >= 5 ? std::string(t[4].b, t[4].e) : "");
      } else if (k >= 3) {
        els.back().props.emplace_back(std::string(t[2].b, t[2].e), std::string(t[1].b, t[1].e));
      } else {
        return fail(OPCFE_IO_ERR_PARSE, path, line_no, "invalid property line");
      }
    } else if (w0 == "end_header") {
      p = next;
      break;
    }
    p = next;
  }
  if (fmt != "ascii" && fmt != "binary_little_endian")
    return fail(OPCFE_IO_ERR_PARSE, path, line_no, "unsupported PLY format '" + fmt + "'");
  const bool bin = fmt == "binary_little_endian";
  int vi = -1;
  for (size_t i = 0; i < els.size(); ++i)
    if (els[i].name == "vertex") {
      vi = (int)i;
      break;
    }
  if (vi < 0) return fail(OPCFE_IO_ERR_PARSE, path, line_no, "no vertex element");
  // elements before the vertex element are read past as the reference reads them
  // (io.py:139-181): ascii -- `count` lines each, face rows must be triangles; binary --
  // face records (count + 3 indices, triangles only), any other element is an error
  for (int i = 0; i < vi; ++i) {
    const Elem& el = els[i];
    const bool face = el.name == "face";
    if (!bin) {
      const int64_t first = line_no + 1;
      for (int64_t r = 0; r < el.count; ++r) {
        ++line_no;
        const char* le2 = line_end(p, e);
        if (face) {
          Tok t[2];
          int64_t nv = 0;
          if (split(p, le2, t, 2) < 1 || !py_int(t[0].b, t[0].e, &nv))
            return fail(OPCFE_IO_ERR_PARSE, path, line_no, "invalid face row");
          if (nv != 3) {  // the reference checks after reading the element's rows
            line_no = first + el.count - 1;
            return fail(OPCFE_IO_ERR_PARSE, path, line_no, "only triangular faces are supported");
          }
        }
        p = le2 < e ? le2 + 1 : e;
      }
    } else {
      if (!face)
        return fail(OPCFE_IO_ERR_PARSE, path, line_no,
                    "cannot skip binary element '" + el.name + "'");
      char cc = 0, ic = 0;
      const int cs = type_size(el.list_count_t, &cc), is = type_size(el.list_item_t, &ic);
      if (cs == 0 || is == 0)
        return fail(OPCFE_IO_ERR_PARSE, path, line_no, "face element without a list property");
      for (int64_t r = 0; r < el.count; ++r) {
        if (e - p < cs + 3 * is) return fail(OPCFE_IO_ERR_PARSE, path, 0, "face data truncated");
        if (load_le(p, cc) != 3.0)
          return fail(OPCFE_IO_ERR_PARSE, path, 0, "only triangular faces are supported");
        p += cs + 3 * is;
      }
    }
  }
  const Elem& v = els[vi];
  info->format = OPCFE_FMT_PLY;
  info->ply_binary = bin ? 1 : 0;
  info->rows = gm;
  info->cols = gn;
  info->count = v.count;
  info->data_offset = (int64_t)(p - m.p);
  info->first_line = line_no + 1;
  int ix = -1, iy = -1, iz = -1, off = 0, offs[3] = {0, 0, 0};
  char codes[3] = {0, 0, 0};
  for (size_t j = 0; j < v.props.size(); ++j) {
    const auto& pr = v.props[j];
    if (pr.first == "list" && bin)
      return fail(OPCFE_IO_ERR_PARSE, path, line_no, "list property on vertex element");
    char c = 0;
    const int sz = bin ? type_size(pr.second, &c) : 1;
    if (bin && sz == 0)
      return fail(OPCFE_IO_ERR_PARSE, path, line_no, "unknown property type '" + pr.second + "'");
    const int pos = bin ? off : (int)j;
    int slot = pr.first == "x" ? 0 : pr.first == "y" ? 1 : pr.first == "z" ? 2 : -1;
    if (slot >= 0 && ((slot == 0 && ix < 0) || (slot == 1 && iy < 0) || (slot == 2 && iz < 0))) {
      (slot == 0 ? ix : slot == 1 ? iy : iz) = (int)j;
      offs[slot] = pos;
      codes[slot] = c;
    }
    off += sz;
  }
  if (ix < 0 || iy < 0 || iz < 0)
    return fail(OPCFE_IO_ERR_PARSE, path, line_no, "vertex element lacks x/y/z");
  info->vertex_stride = bin ? off : 0;
  info->x_off = offs[0];
  info->y_off = offs[1];
  info->z_off = offs[2];
  info->x_type = codes[0];
  info->y_type = codes[1];
  info->z_type = codes[2];
  info->direct = bin && off == 24 && codes[0] == 'd' && codes[1] == 'd' && codes[2] == 'd' &&
                 offs[0] == 0 && offs[1] == 8 && offs[2] == 16;
  return OPCFE_IO_OK;
}

// grid / xyz header + body row count
int probe_text(const Mapped& m, const std::string& path, int format, opcfe_cloud_info* info,
               int threads) {
  const char* p = m.p;
  const char* e = m.p + m.n;
  int64_t line_no = 0, M = -1, N = -1;
  const TextMode tm = text_mode(p, e);
  if (format == OPCFE_FMT_GRID) {
    bool found = false;
    while (p < e) {
      const char* le = line_end(p, e, tm);
      ++line_no;
      Tok t[3];
      const int k = split(p, le, t, 3, tm);
      p = next_line(le, e, tm);
      if (skip_line(t, k)) continue;
      if (k < 2 || !py_int(t[0].b, t[0].e, &M) || !py_int(t[1].b, t[1].e, &N))
        return fail(OPCFE_IO_ERR_PARSE, path, line_no, "grid header must be two integers 'M N'");
      found = true;
      break;
    }
    if (!found || M < 1 || N < 1)
      return fail(OPCFE_IO_ERR_PARSE, path, found ? line_no : 1, "missing or invalid grid header");
  }
  info->format = format;
  info->ply_binary = 0;
  info->rows = M;
  info->cols = N;
  info->data_offset = (int64_t)(p - m.p);
  info->first_line = line_no + 1;
  const int T = nthreads(threads, (size_t)(e - p));
  auto cs = chunk(p, e, T, tm);
  count_pass(cs, kRows, T, tm);
  info->count = cs.empty() ? 0 : cs.back().row0 + cs.back().rows;
  info->vertex_stride = 0;
  info->direct = 0;
  return OPCFE_IO_OK;
}

int64_t total_lines(const Mapped& m, const TextMode& tm) {
  // Python readlines(): a final line without a terminator still counts
  int64_t n = 0;
  for (const char* p = m.p; p < m.p + m.n;) {
    const char* le = line_end(p, m.p + m.n, tm);
    ++n;
    p = next_line(le, m.p + m.n, tm);
  }
  return n;
}

}  // namespace

extern "C" {

const char* opcfe_io_last_error(void) { return g_err.c_str(); }
int64_t opcfe_io_error_line(void) { return g_err_line; }

int opcfe_io_probe(const char* path, int format, opcfe_cloud_info* info) {
  if (!path || !info) return OPCFE_IO_ERR_ARG;
  std::memset(info, 0, sizeof(*info));
  Mapped m;
  if (int rc = m.open_(path)) return rc;
  if (format == OPCFE_FMT_PLY) return probe_ply(m, path, info);
  if (format == OPCFE_FMT_GRID || format == OPCFE_FMT_XYZ)
    return probe_text(m, path, format, info, 0);
  g_err = std::string(path) + ": unknown format";
  return OPCFE_IO_ERR_ARG;
}

int opcfe_io_read(const char* path, const opcfe_cloud_info* info, double* dst, int threads) {
  if (!path || !info || (!dst && info->count > 0)) return OPCFE_IO_ERR_ARG;
  const std::string P(path);
  if (info->format == OPCFE_FMT_PLY && info->ply_binary) {
    const int64_t need = info->count * (int64_t)info->vertex_stride;
    if (info->direct) {  // the record IS (x, y, z) float64: read into dst as is
      int fd = ::open(path, O_RDONLY);
      if (fd < 0) return fail_os(P, "cannot open");
      char* out = reinterpret_cast<char*>(dst);
      int64_t done = 0;
      while (done < need) {
        const ssize_t r = pread(fd, out + done, (size_t)std::min<int64_t>(need - done, 1 << 30),
                                (off_t)(info->data_offset + done));
        if (r < 0) {
          close(fd);
          return fail_os(P, "read failed");
        }
        if (r == 0) break;
        done += r;
      }
      close(fd);
      if (done < need)
        return fail(OPCFE_IO_ERR_PARSE, P, info->first_line, "vertex data truncated");
      return OPCFE_IO_OK;
    }
    Mapped m;
    if (int rc = m.open_(P)) return rc;
    if ((int64_t)m.n < info->data_offset + need)
      return fail(OPCFE_IO_ERR_PARSE, P, info->first_line, "vertex data truncated");
    const char* base = m.p + info->data_offset;
    const int T = nthreads(threads, (size_t)need);
    parallel(T, [&](int t) {
      const int64_t b = info->count * t / T, e = info->count * (t + 1) / T;
      for (int64_t i = b; i < e; ++i) {
        const char* r = base + i * info->vertex_stride;
        dst[3 * i] = load_le(r + info->x_off, info->x_type);
        dst[3 * i + 1] = load_le(r + info->y_off, info->y_type);
        dst[3 * i + 2] = load_le(r + info->z_off, info->z_type);
      }
    });
    return OPCFE_IO_OK;
  }
  Mapped m;
  if (int rc = m.open_(P)) return rc;
  const char* b = m.p + info->data_offset;
  const char* e = m.p + m.n;
  if (info->format == OPCFE_FMT_PLY) {  // ascii: exactly `count` lines
    const char* q = b;
    int64_t got = 0;
    while (got < info->count && q < e) {
      const char* le = line_end(q, e);
      q = le < e ? le + 1 : e;
      ++got;
    }
    if (got < info->count)
      return fail(OPCFE_IO_ERR_PARSE, P, info->first_line + got, "unexpected end of vertex data");
    const int idx[3] = {info->x_off, info->y_off, info->z_off};
    const int T = nthreads(threads, (size_t)(q - b));
    auto cs = chunk(b, q, T, g_text_plain);
    count_pass(cs, kPly, T, g_text_plain);
    parse_pass(cs, kPly, T, dst, info->count, info->first_line, idx,
               std::max(idx[0], std::max(idx[1], idx[2])), g_text_plain);
    return first_error(cs, P);
  }
  // grid / xyz text: parse errors first (in line order), then the row count
  const TextMode tm = text_mode(m.p, e);
  const int T = nthreads(threads, (size_t)(e - b));
  auto cs = chunk(b, e, T, tm);
  count_pass(cs, kRows, T, tm);
  const int64_t rows = cs.empty() ? 0 : cs.back().row0 + cs.back().rows;
  const bool fits = rows == info->count;
  parse_pass(cs, kRows, T, fits ? dst : nullptr, info->count, info->first_line, nullptr, 0, tm);
  if (int rc = first_error(cs, P)) return rc;
  if (info->format == OPCFE_FMT_GRID && rows != info->rows * info->cols)
    return fail(OPCFE_IO_ERR_PARSE, P, total_lines(m, tm),
                "expected " + std::to_string(info->rows * info->cols) + " rows, got " +
                    std::to_string(rows));
  if (!fits)
    return fail(OPCFE_IO_ERR_PARSE, P, total_lines(m, tm), "file changed while reading");
  return OPCFE_IO_OK;
}

int opcfe_io_write_ply(const char* path, const double* v, int64_t n, int binary,
                       int64_t grid_rows, int64_t grid_cols) {
  if (!path || (n > 0 && !v) || n < 0) return OPCFE_IO_ERR_ARG;
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail_os(path, "cannot open for writing");
  std::string h = "ply\n";
  h += binary ? "format binary_little_endian 1.0\n" : "format ascii 1.0\n";
  if (grid_rows > 0 && grid_cols > 0)
    h += "comment grid " + std::to_string(grid_rows) + " " + std::to_string(grid_cols) + "\n";
  h += "element vertex " + std::to_string(n) + "\n";
  h += "property double x\nproperty double y\nproperty double z\nend_header\n";
  bool ok = std::fwrite(h.data(), 1, h.size(), f) == h.size();
  if (binary) {
    ok = ok && std::fwrite(v, sizeof(double), (size_t)(3 * n), f) == (size_t)(3 * n);
  } else {
    char line[96];
    auto g17 = [](char* o, double x) {  // Python format(x, '.17g')
      if (std::isnan(x)) return std::snprintf(o, 8, "nan");
      return std::snprintf(o, 32, "%.17g", x);
    };
    for (int64_t i = 0; ok && i < n; ++i) {
      int k = g17(line, v[3 * i]);
      line[k++] = ' ';
      k += g17(line + k, v[3 * i + 1]);
      line[k++] = ' ';
      k += g17(line + k, v[3 * i + 2]);
      line[k++] = '\n';
      ok = std::fwrite(line, 1, (size_t)k, f) == (size_t)k;
    }
  }
  if (std::fclose(f) != 0) ok = false;
  if (!ok) return fail_os(path, "write failed");
  return OPCFE_IO_OK;
}

}  // extern "C"
