// mm_ingest.cpp -- native Matrix Market coordinate reader (reference
// io.py:37-104 load_matrix_market): header / size line validation, entries
// parsed in parallel (the file is mmapped and split at line boundaries, one
// thread per chunk: count pass, prefix sum, parse pass into the caller's
// arrays in file order), 1-based -> 0-based, index range checks, symmetric
// storage expanded exactly as the reference does (original entries, then the
// off-diagonal ones mirrored, in file order).  Errors carry the reference's
// "path:line: reason" text.  Canonicalisation (sort, duplicate sum, zero drop)
// runs on the GPU (coo_csr.cu).  Values are parsed with strtod (correctly
// rounded, like Python's float()).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sketch_b200.h"

namespace skt {
void set_error(const std::string &msg);
}

namespace {

struct Mapped {
  const char *p = nullptr;
  size_t n = 0;
  int fd = -1;
  ~Mapped() {
    if (p && n) munmap((void *)p, n);
    if (fd >= 0) close(fd);
  }
};

skt_status err(const std::string &m) {
  skt::set_error(m);
  return SKT_EINVAL;
}

bool map_file(const char *path, Mapped &m, std::string &why) {
  m.fd = open(path, O_RDONLY);
  if (m.fd < 0) {
    why = std::string(path) + ": " + strerror(errno);
    return false;
  }
  struct stat st;
  if (fstat(m.fd, &st) != 0) {
    why = std::string(path) + ": " + strerror(errno);
    return false;
  }
  m.n = (size_t)st.st_size;
  if (m.n == 0) return true;
  void *q = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
  if (q == MAP_FAILED) {
    why = std::string(path) + ": mmap failed";
    m.n = 0;
    return false;
  }
  m.p = (const char *)q;
  return true;
}

std::string lower_trim(const char *b, const char *e) {
  while (b < e && isspace((unsigned char)*b)) ++b;
  while (e > b && isspace((unsigned char)e[-1])) --e;
  std::string s(b, e);
  for (auto &c : s) c = (char)tolower((unsigned char)c);
  return s;
}

std::vector<std::string> split_ws(const std::string &s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && isspace((unsigned char)s[i])) ++i;
    size_t j = i;
    while (j < s.size() && !isspace((unsigned char)s[j])) ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

struct Header {
  int field = 0;  // 0 real, 1 integer, 2 pattern
  int symmetric = 0;
  int64_t n_rows = 0, n_cols = 0, n_entries = 0;
  size_t body = 0;      // byte offset of the first line after the size line
  int64_t body_line = 0;  // line number of the size line
};

// header + size line (io.py:25-35, 40-62)
skt_status parse_header(const char *path, const Mapped &m, Header &h) {
  const char *p = m.p, *e = m.p + m.n;
  const char *nl = p ? (const char *)memchr(p, '\n', (size_t)(e - p)) : nullptr;
  const char *l1e = nl ? nl : e;
  const std::string raw(p ? p : "", p ? (size_t)(l1e - p) : 0);
  const std::string hdr = lower_trim(raw.data(), raw.data() + raw.size());
  auto parts = split_ws(hdr);
  std::string shown = lower_trim(raw.data(), raw.data() + raw.size());
  {
    // the reference shows the stripped original line (not lower-cased)
    const char *b = raw.data(), *x = raw.data() + raw.size();
    while (b < x && isspace((unsigned char)*b)) ++b;
    while (x > b && isspace((unsigned char)x[-1])) --x;
    shown.assign(b, x);
  }
  if (parts.size() != 5 || parts[0] != "%%matrixmarket" || parts[1] != "matrix")
    return err(std::string(path) + ":1: bad MatrixMarket header: '" + shown + "'");
  const std::string &layout = parts[2], &field = parts[3], &sym = parts[4];
  if (field != "real" && field != "integer" && field != "pattern")
    return err(std::string(path) + ":1: unsupported field type '" + field + "'");
  if (sym != "general" && sym != "symmetric")
    return err(std::string(path) + ":1: unsupported symmetry '" + sym + "'");
  if (layout != "coordinate") return err(std::string(path) + ":1: expected coordinate layout, got '" + layout + "'");
  h.field = field == "real" ? 0 : field == "integer" ? 1 : 2;
  h.symmetric = sym == "symmetric";
  int64_t lineno = 1;
  const char *q = nl ? nl + 1 : e;
  while (q < e) {
    const char *le = (const char *)memchr(q, '\n', (size_t)(e - q));
    if (!le) le = e;
    ++lineno;
    const std::string s = lower_trim(q, le);
    const char *next = le < e ? le + 1 : e;
    if (s.empty() || s[0] == '%') {
      q = next;
      continue;
    }
    auto tok = split_ws(s);
    char *end1 = nullptr;
    bool ok = tok.size() == 3;
    int64_t v[3] = {0, 0, 0};
    for (int i = 0; ok && i < 3; ++i) {
      errno = 0;
      v[i] = strtoll(tok[i].c_str(), &end1, 10);
      ok = errno == 0 && end1 && *end1 == '\0';
    }
    if (!ok) {
      const char *b = q, *x = le;
      while (b < x && isspace((unsigned char)*b)) ++b;
      while (x > b && isspace((unsigned char)x[-1])) --x;
      return err(std::string(path) + ":" + std::to_string(lineno) + ": bad size line '" + std::string(b, x) + "'");
    }
    h.n_rows = v[0];
    h.n_cols = v[1];
    h.n_entries = v[2];
    h.body = (size_t)(next - m.p);
    h.body_line = lineno;
    return SKT_OK;
  }
  return err(std::string(path) + ":" + std::to_string(lineno) + ": missing size line");
}

struct Chunk {
  size_t b = 0, e = 0;
  int64_t lines = 0, entries = 0;  // count pass
  int64_t line0 = 0, entry0 = 0;   // prefix sums
  std::string error;
  int64_t error_line = -1;
};

// parse one line into (i, j, v); returns false if malformed
bool parse_entry(const char *b, const char *e, int field, int64_t &i, int64_t &j, double &v) {
  auto skip = [&](const char *&p) {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
  };
  auto token = [&](const char *&p, std::string &out) -> bool {
    skip(p);
    const char *s = p;
    while (p < e && !isspace((unsigned char)*p)) ++p;
    if (p == s) return false;
    out.assign(s, p);
    return true;
  };
  const char *p = b;
  std::string t0, t1, t2;
  if (!token(p, t0) || !token(p, t1)) return false;
  char *end = nullptr;
  errno = 0;
  i = strtoll(t0.c_str(), &end, 10);
  if (errno || *end) return false;
  j = strtoll(t1.c_str(), &end, 10);
  if (errno || *end) return false;
  if (field == 2) {
    v = 1.0;
    return true;
  }
  if (!token(p, t2)) return false;
  v = strtod(t2.c_str(), &end);
  return *end == '\0';
}

}  // namespace

extern "C" skt_status skt_mm_probe(const char *path, skt_mm_info *info) {
  if (!path || !info) return err("skt_mm_probe: NULL argument");
  Mapped m;
  std::string why;
  if (!map_file(path, m, why)) return err(why);
  Header h;
  const skt_status st = parse_header(path, m, h);
  if (st != SKT_OK) return st;
  info->n_rows = h.n_rows;
  info->n_cols = h.n_cols;
  info->n_entries = h.n_entries;
  info->field = h.field;
  info->symmetric = h.symmetric;
  return SKT_OK;
}

extern "C" skt_status skt_mm_read_coo(const char *path, int64_t capacity, int64_t *rows, int64_t *cols, double *vals,
                                      int64_t *count, int32_t n_threads) {
  if (!path || !count) return err("skt_mm_read_coo: NULL argument");
  Mapped m;
  std::string why;
  if (!map_file(path, m, why)) return err(why);
  Header h;
  skt_status st = parse_header(path, m, h);
  if (st != SKT_OK) return st;
  const int64_t need = h.symmetric ? 2 * h.n_entries : h.n_entries;
  if (capacity < need || (need > 0 && (!rows || !cols || !vals)))
    return err("skt_mm_read_coo: capacity below the declared entries (x2 for symmetric)");
  // ---- split the body at line boundaries
  const size_t body = h.body, total = m.n;
  int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)((total - body) / (1 << 16)) + 1));
  std::vector<Chunk> ch(nt);
  size_t pos = body;
  for (int c = 0; c < nt; ++c) {
    ch[c].b = pos;
    size_t e = c == nt - 1 ? total : std::max(pos, body + (total - body) * (size_t)(c + 1) / nt);
    if (e < total) {
      const char *nl = (const char *)memchr(m.p + e, '\n', total - e);
      e = nl ? (size_t)(nl - m.p) + 1 : total;
    }
    ch[c].e = e;
    pos = e;
  }
  // ---- pass 1: lines and entries per chunk
  auto count_pass = [&](Chunk &k) {
    const char *p = m.p + k.b, *e = m.p + k.e;
    while (p < e) {
      const char *le = (const char *)memchr(p, '\n', (size_t)(e - p));
      if (!le) le = e;
      ++k.lines;
      const char *q = p;
      while (q < le && isspace((unsigned char)*q)) ++q;
      if (q < le && *q != '%') ++k.entries;
      p = le < e ? le + 1 : e;
    }
  };
  {
    std::vector<std::thread> th;
    for (int c = 1; c < nt; ++c) th.emplace_back(count_pass, std::ref(ch[c]));
    count_pass(ch[0]);
    for (auto &t : th) t.join();
  }
  int64_t line = h.body_line, entry = 0;
  for (auto &k : ch) {
    k.line0 = line;
    k.entry0 = entry;
    line += k.lines;
    entry += k.entries;
  }
  const int64_t found = entry;
  // ---- pass 2: parse into place (entries beyond the declared count are an error)
  auto parse_pass = [&](Chunk &k) {
    const char *p = m.p + k.b, *e = m.p + k.e;
    int64_t ln = k.line0, idx = k.entry0;
    while (p < e) {
      const char *le = (const char *)memchr(p, '\n', (size_t)(e - p));
      if (!le) le = e;
      ++ln;
      const char *q = p, *x = le;
      while (q < x && isspace((unsigned char)*q)) ++q;
      while (x > q && isspace((unsigned char)x[-1])) --x;
      if (q < x && *q != '%') {
        if (idx >= h.n_entries) {
          k.error = std::string(path) + ":" + std::to_string(ln) + ": more entries than declared";
          k.error_line = ln;
          return;
        }
        int64_t i, j;
        double v;
        if (!parse_entry(q, x, h.field, i, j, v)) {
          k.error = std::string(path) + ":" + std::to_string(ln) + ": bad entry '" + std::string(q, x) + "'";
          k.error_line = ln;
          return;
        }
        if (!(1 <= i && i <= h.n_rows && 1 <= j && j <= h.n_cols)) {
          k.error = std::string(path) + ":" + std::to_string(ln) + ": index out of range";
          k.error_line = ln;
          return;
        }
        rows[idx] = i - 1;
        cols[idx] = j - 1;
        vals[idx] = v;
        ++idx;
      }
      p = le < e ? le + 1 : e;
    }
  };
  {
    std::vector<std::thread> th;
    for (int c = 1; c < nt; ++c) th.emplace_back(parse_pass, std::ref(ch[c]));
    parse_pass(ch[0]);
    for (auto &t : th) t.join();
  }
  for (auto &k : ch)  // the first error in file order, as the sequential reader reports it
    if (!k.error.empty()) return err(k.error);
  if (found != h.n_entries)
    return err(std::string(path) + ":" + std::to_string(line) + ": expected " + std::to_string(h.n_entries) +
               " entries, found " + std::to_string(found));
  int64_t nn = h.n_entries;
  if (h.symmetric) {  // io.py:94-100: off-diagonal entries mirrored, appended in file order
    for (int64_t e = 0; e < h.n_entries; ++e)
      if (rows[e] != cols[e]) {
        rows[nn] = cols[e];
        cols[nn] = rows[e];
        vals[nn] = vals[e];
        ++nn;
      }
  }
  *count = nn;
  return SKT_OK;
}
