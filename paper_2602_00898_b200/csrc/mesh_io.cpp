// On-disk formats: the host text I/O around the device
// path -- OFF / OBJ meshes, MatrixMarket coordinate patterns, patch files,
// permutation and etree files -- with the reference's accepted syntax, error
// texts and written bytes (core/src/io.cpp, core/include/meshperm/io.hpp).
//
// Design: a file is read with fread into memory and walked by a Scanner that
// hands out lines and whitespace-separated tokens as string_views, so a
// 10M-vertex mesh costs one pass over its bytes instead of a stream and a
// string per line.  Numbers go through strtoll / strtod on a NUL-terminated
// copy of the token, with the acceptance rules of std::stoll / std::stod (the
// whole token must be consumed; ERANGE is an error).  The reference's
// std::runtime_error becomes MP_EIO; validate_mesh's std::invalid_argument
// (types.cpp:20-33) stays MP_EINVAL.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "mp_internal.h"

namespace mp {
namespace {

struct IoError {
  std::string msg;
};

[[noreturn]] void raise_at(const std::string& path, int line, const std::string& what) {
  throw IoError{path + ":" + std::to_string(line) + ": " + what};
}

bool is_space(char c) {  // the C-locale isspace set operator>> splits on
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

std::string lower(std::string_view s) {
  std::string r(s);
  for (char& c : r)
    if (c >= 'A' && c <= 'Z') c = static_cast<char>(c - 'A' + 'a');
  return r;
}

class Scanner {
 public:
  explicit Scanner(const std::string& path) : path_(path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError{"cannot open " + path};
    char chunk[1 << 16];
    for (std::size_t got; (got = std::fread(chunk, 1, sizeof chunk, f)) > 0;) buf_.append(chunk, got);
    std::fclose(f);
  }

  int line_no() const { return line_; }

  // The next raw line (without '\n'); false at end of input.  A final line
  // without a newline still counts, an empty tail after the last '\n' not.
  bool raw_line(std::string_view& out) {
    if (pos_ >= buf_.size()) return false;
    const char* b = buf_.data() + pos_;
    const void* nl = std::memchr(b, '\n', buf_.size() - pos_);
    const std::size_t len = nl ? static_cast<std::size_t>(static_cast<const char*>(nl) - b) : buf_.size() - pos_;
    out = std::string_view(b, len);
    pos_ += len + (nl ? 1 : 0);
    ++line_;
    return true;
  }

  // The next line holding anything besides blanks once a '#' comment is cut.
  bool data_line(std::string_view& out) {
    while (raw_line(out)) {
      out = out.substr(0, out.find('#'));
      if (out.find_first_not_of(" \t\r\n") != std::string_view::npos) return true;
    }
    return false;
  }

  [[noreturn]] void fail(const std::string& what) const { raise_at(path_, line_, what); }

 private:
  std::string path_;
  std::string buf_;
  std::size_t pos_ = 0;
  int line_ = 0;
};

// Splits into `toks` (reused across lines to keep the hot loop allocation-free).
void tokens(std::string_view line, std::vector<std::string_view>& toks) {
  toks.clear();
  std::size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_space(line[i])) ++i;
    const std::size_t b = i;
    while (i < line.size() && !is_space(line[i])) ++i;
    if (i > b) toks.push_back(line.substr(b, i - b));
  }
}

// strtoll / strtod need a terminator; short tokens stay on the stack.
template <class Fn>
auto with_cstr(std::string_view tok, Fn&& fn) {
  char small[64];
  if (tok.size() < sizeof small) {
    std::memcpy(small, tok.data(), tok.size());
    small[tok.size()] = '\0';
    return fn(static_cast<const char*>(small));
  }
  std::string big(tok);
  return fn(big.c_str());
}

long long integer(const Scanner& s, std::string_view tok, const char* what) {
  bool ok = false;
  const long long v = with_cstr(tok, [&](const char* c) {
    char* end = nullptr;
    errno = 0;
    const long long r = std::strtoll(c, &end, 10);
    ok = end != c && errno != ERANGE && *end == '\0';
    return r;
  });
  if (!ok) s.fail(std::string(what) + " is not an integer: '" + std::string(tok) + "'");
  return v;
}

void real(const Scanner& s, std::string_view tok, const char* what) {  // value discarded, as in the reference
  const bool ok = with_cstr(tok, [&](const char* c) {
    char* end = nullptr;
    errno = 0;
    (void)std::strtod(c, &end);
    return end != c && errno != ERANGE && *end == '\0';
  });
  if (!ok) s.fail(std::string(what) + " is not a number: '" + std::string(tok) + "'");
}

struct Mesh {
  int32_t nv = 0;
  std::vector<int32_t> tri;  // 3 per triangle

  void add_polygon(const int32_t* c, std::size_t k) {  // fan from the first corner
    for (std::size_t j = 1; j + 1 < k; ++j) tri.insert(tri.end(), {c[0], c[j], c[j + 1]});
  }

  void validate() const {  // types.cpp:20-33
    const std::size_t nt = tri.size() / 3;
    for (std::size_t t = 0; t < nt; ++t) {
      const int32_t* c = &tri[3 * t];
      for (int k = 0; k < 3; ++k)
        if (c[k] < 0 || c[k] >= nv)
          throw Error(MP_EINVAL, "triangle " + std::to_string(t) + " references vertex " + std::to_string(c[k]) +
                                     " outside [0, " + std::to_string(nv) + ")");
      if (c[0] == c[1] || c[1] == c[2] || c[0] == c[2])
        throw Error(MP_EINVAL, "triangle " + std::to_string(t) + " has repeated corners");
    }
  }
};

// io.cpp:88-139.  Header "OFF [nv nf [ne]]", else the counts on the next data
// line; vertex lines need three numbers; face lines "k c0 .. c(k-1)", k >= 3.
Mesh read_off(const std::string& path) {
  Scanner s(path);
  std::string_view ln;
  std::vector<std::string_view> tk;
  if (!s.data_line(ln)) s.fail("empty file");
  tokens(ln, tk);
  if (tk.empty() || tk[0] != "OFF") s.fail("expected OFF header");
  std::size_t at = 1;
  if (tk.size() < 3) {
    if (!s.data_line(ln)) s.fail("missing count line");
    tokens(ln, tk);
    if (tk.size() < 2) s.fail("count line needs nv nf [ne]");
    at = 0;
  }
  const long long nv = integer(s, tk[at], "vertex count");
  const long long nf = integer(s, tk[at + 1], "face count");
  if (nv < 0 || nf < 0) s.fail("negative count");
  Mesh m;
  m.nv = static_cast<int32_t>(nv);
  for (long long v = 0; v < nv; ++v) {
    if (!s.data_line(ln)) s.fail("unexpected end of file in vertex list");
    tokens(ln, tk);
    if (tk.size() < 3) s.fail("vertex needs 3 coordinates");
    for (int c = 0; c < 3; ++c) real(s, tk[c], "coordinate");
  }
  m.tri.reserve(static_cast<std::size_t>(std::min<long long>(nf, 1 << 26)) * 3);
  std::vector<int32_t> poly;
  for (long long f = 0; f < nf; ++f) {
    if (!s.data_line(ln)) s.fail("unexpected end of file in face list");
    tokens(ln, tk);
    if (tk.empty()) s.fail("empty face record");
    const long long k = integer(s, tk[0], "corner count");
    if (k < 3) s.fail("face needs at least 3 corners");
    if (tk.size() < static_cast<std::size_t>(k) + 1) s.fail("truncated face record");
    poly.clear();
    for (long long c = 1; c <= k; ++c) {
      const long long v = integer(s, tk[c], "face corner");
      if (v < 0 || v >= nv) s.fail("face corner out of range");
      poly.push_back(static_cast<int32_t>(v));
    }
    m.add_polygon(poly.data(), poly.size());
  }
  m.validate();
  return m;
}

// io.cpp:141-176.  Only "v" and "f" records matter; "f" corners are 1-based
// with any "/vt/vn" suffix dropped, and are range-checked after the whole file
// (a face may precede its vertices) against the line the face was on.
Mesh read_obj(const std::string& path) {
  Scanner s(path);
  std::string_view ln;
  std::vector<std::string_view> tk;
  Mesh m;
  std::vector<long long> corner;                  // all face corners, file order
  std::vector<std::pair<int, std::size_t>> face;  // (line, end offset into corner)
  while (s.raw_line(ln)) {
    tokens(ln.substr(0, ln.find('#')), tk);
    if (tk.empty()) continue;
    if (tk[0] == "v") {
      if (tk.size() < 4) s.fail("vertex needs 3 coordinates");
      for (int c = 1; c <= 3; ++c) real(s, tk[c], "coordinate");
      ++m.nv;
    } else if (tk[0] == "f") {
      if (tk.size() < 4) s.fail("face needs at least 3 corners");
      for (std::size_t c = 1; c < tk.size(); ++c)
        corner.push_back(integer(s, tk[c].substr(0, tk[c].find('/')), "face corner"));
      face.emplace_back(s.line_no(), corner.size());
    }
  }
  std::vector<int32_t> poly;
  std::size_t b = 0;
  for (const auto& [line, e] : face) {
    poly.clear();
    for (std::size_t c = b; c < e; ++c) {
      if (corner[c] < 1 || corner[c] > m.nv) raise_at(path, line, "face corner out of range");
      poly.push_back(static_cast<int32_t>(corner[c] - 1));
    }
    m.add_polygon(poly.data(), poly.size());
    b = e;
  }
  m.validate();
  return m;
}

// io.cpp:178-184
Mesh read_mesh_by_extension(const std::string& path, int32_t format) {
  if (format == 1) return read_off(path);
  if (format == 2) return read_obj(path);
  const auto dot = path.rfind('.');
  const std::string ext = dot == std::string::npos ? "" : lower(std::string_view(path).substr(dot));
  if (ext == ".off") return read_off(path);
  if (ext == ".obj") return read_obj(path);
  throw IoError{"unsupported mesh format: " + path};
}

// io.cpp:186-240 + SparsePattern::symmetrize (types.cpp:9-18).  Entries are
// packed as (row << 32 | col) keys so mirroring, sorting and deduplication run
// on one uint64 array.
std::vector<uint64_t> read_mm(const std::string& path, int32_t& n) {
  Scanner s(path);
  std::string_view ln;
  std::vector<std::string_view> tk;
  if (!s.raw_line(ln)) raise_at(path, 1, "empty file");
  tokens(ln, tk);
  if (tk.size() < 5 || lower(tk[0]) != "%%matrixmarket") s.fail("expected MatrixMarket banner");
  if (lower(tk[1]) != "matrix" || lower(tk[2]) != "coordinate") s.fail("only coordinate matrices are supported");
  const std::string field = lower(tk[3]), symmetry = lower(tk[4]);
  if (field != "real" && field != "integer" && field != "pattern")
    s.fail("unsupported field type: " + std::string(tk[3]));
  if (symmetry != "symmetric" && symmetry != "general") s.fail("unsupported symmetry: " + std::string(tk[4]));
  // blank lines and '%' comment lines are skipped ('#' has no meaning here)
  auto entry_line = [&]() {
    while (s.raw_line(ln)) {
      if (ln.find_first_not_of(" \t\r\n") == std::string_view::npos) continue;
      if (ln[ln.find_first_not_of(" \t")] == '%') continue;
      return true;
    }
    return false;
  };
  if (!entry_line()) s.fail("missing size line");
  tokens(ln, tk);
  if (tk.size() != 3) s.fail("size line needs rows cols nnz");
  const long long rows = integer(s, tk[0], "row count");
  const long long cols = integer(s, tk[1], "column count");
  const long long nnz = integer(s, tk[2], "entry count");
  if (rows != cols) s.fail("matrix is not square");
  if (rows < 0 || nnz < 0) s.fail("negative size");
  std::vector<uint64_t> key;
  key.reserve(static_cast<std::size_t>(std::min<long long>(nnz, 1 << 28)) * 2);
  for (long long k = 0; k < nnz; ++k) {
    if (!entry_line()) s.fail("unexpected end of file in entry list");
    tokens(ln, tk);
    if (tk.size() < 2) s.fail("entry needs row and column");
    const long long i = integer(s, tk[0], "row index");
    const long long j = integer(s, tk[1], "column index");
    if (i < 1 || i > rows || j < 1 || j > rows) s.fail("entry index out of range");
    const uint64_t r = static_cast<uint64_t>(i - 1), c = static_cast<uint64_t>(j - 1);
    key.push_back(r << 32 | c);
    if (r != c) key.push_back(c << 32 | r);
  }
  std::sort(key.begin(), key.end());
  key.erase(std::unique(key.begin(), key.end()), key.end());
  n = static_cast<int32_t>(rows);
  return key;
}

// Every whitespace-separated integer of every data line, in order.
template <class Check>
std::vector<int32_t> read_int_list(const std::string& path, const char* what, Check&& check) {
  Scanner s(path);
  std::string_view ln;
  std::vector<std::string_view> tk;
  std::vector<int32_t> out;
  while (s.data_line(ln)) {
    tokens(ln, tk);
    for (auto t : tk) {
      const long long v = integer(s, t, what);
      check(s, v);
      out.push_back(static_cast<int32_t>(v));
    }
  }
  return out;
}

// Buffered decimal writer; opened before anything is formatted so an
// unwritable path fails first.
class Writer {
 public:
  explicit Writer(const std::string& path) : path_(path), f_(std::fopen(path.c_str(), "wb")) {
    if (!f_) throw IoError{"cannot open " + path + " for writing"};
    buf_.reserve(1 << 20);
  }
  ~Writer() {
    if (f_) std::fclose(f_);
  }
  Writer& num(long long v) {
    char t[24];
    const int k = std::snprintf(t, sizeof t, "%lld", v);
    buf_.append(t, static_cast<std::size_t>(k));
    return *this;
  }
  Writer& ch(char c) {
    buf_.push_back(c);
    if (buf_.size() >= (1u << 20)) flush();
    return *this;
  }
  void finish() {
    flush();
    const bool closed = std::fclose(f_) == 0;
    f_ = nullptr;
    if (!ok_ || !closed) throw IoError{"write failed: " + path_};
  }

 private:
  void flush() {
    if (!buf_.empty() && std::fwrite(buf_.data(), 1, buf_.size(), f_) != buf_.size()) ok_ = false;
    buf_.clear();
  }
  std::string path_;
  FILE* f_;
  std::string buf_;
  bool ok_ = true;
};

template <class F>
int io_guarded(F&& f) {
  return guarded([&] {
    try {
      f();
    } catch (const IoError& e) {
      throw Error(MP_EIO, e.msg);
    }
  });
}

}  // namespace
}  // namespace mp

using namespace mp;

extern "C" {

// parse_mesh / parse_off / parse_obj (io.hpp:15-22).  format 0 = by extension,
// 1 = OFF, 2 = OBJ.  tris NULL returns the counts only.
int mp_read_mesh(const char* path, int32_t format, int32_t* vertex_count, int64_t* triangle_count, int32_t* tris) {
  return io_guarded([&] {
    if (!path || !vertex_count || !triangle_count) throw Error(MP_EINVAL, "null argument");
    if (format < 0 || format > 2) throw Error(MP_EINVAL, "unknown mesh format code");
    const Mesh m = read_mesh_by_extension(path, format);
    *vertex_count = m.nv;
    *triangle_count = static_cast<int64_t>(m.tri.size() / 3);
    if (tris && !m.tri.empty()) std::memcpy(tris, m.tri.data(), sizeof(int32_t) * m.tri.size());
  });
}

// parse_matrix_market (io.hpp:27): symmetrised, sorted, unique 0-based entries.
int mp_read_matrix_market(const char* path, int32_t* n, int64_t* nnz, int32_t* rows, int32_t* cols) {
  return io_guarded([&] {
    if (!path || !n || !nnz) throw Error(MP_EINVAL, "null argument");
    const auto key = read_mm(path, *n);
    *nnz = static_cast<int64_t>(key.size());
    if (rows && cols)
      for (std::size_t k = 0; k < key.size(); ++k) {
        rows[k] = static_cast<int32_t>(key[k] >> 32);
        cols[k] = static_cast<int32_t>(key[k] & 0xffffffffu);
      }
  });
}

// read_patch_file (io.hpp:30): exactly n nonnegative ids, patch_count = max + 1.
int mp_read_patch_file(const char* path, int32_t n, int32_t* assignment, int32_t* patch_count) {
  return io_guarded([&] {
    if (!path || (n > 0 && !assignment) || !patch_count) throw Error(MP_EINVAL, "null argument");
    const auto ids = read_int_list(path, "patch id", [](const Scanner& s, long long v) {
      if (v < 0) s.fail("patch id must be nonnegative");
    });
    if (ids.size() != static_cast<std::size_t>(n))
      throw IoError{std::string(path) + ": expected " + std::to_string(n) + " patch ids, found " +
                    std::to_string(ids.size())};
    int32_t pc = 0;
    for (int32_t p : ids) pc = std::max(pc, p + 1);
    std::copy(ids.begin(), ids.end(), assignment);
    *patch_count = pc;
  });
}

// write_permutation (io.hpp:33): perm[k] per line.
int mp_write_permutation(const char* path, int32_t n, const int32_t* perm) {
  return io_guarded([&] {
    if (!path || (n > 0 && !perm)) throw Error(MP_EINVAL, "null argument");
    Writer w(path);
    for (int32_t k = 0; k < n; ++k) w.num(perm[k]).ch('\n');
    w.finish();
  });
}

// read_permutation (io.hpp:34): every integer, no range check.  perm NULL
// returns the count only.
int mp_read_permutation(const char* path, int32_t* n, int32_t* perm) {
  return io_guarded([&] {
    if (!path || !n) throw Error(MP_EINVAL, "null argument");
    const auto p = read_int_list(path, "index", [](const Scanner&, long long) {});
    *n = static_cast<int32_t>(p.size());
    if (perm) std::copy(p.begin(), p.end(), perm);
  });
}

// write_etree (io.hpp:37): "idx level count v..." for the 2^(L+1)-1 nodes in
// heap order; the level of node i is floor(log2(i + 1)).
int mp_write_etree(const char* path, int32_t nd_level, const int32_t* node_offsets, const int32_t* node_vertices) {
  return io_guarded([&] {
    if (!path || !node_offsets) throw Error(MP_EINVAL, "null argument");
    if (nd_level < 0 || nd_level > 24) throw Error(MP_EINVAL, "nd_level out of range");
    Writer w(path);
    const int32_t nodes = (2 << nd_level) - 1;
    for (int32_t i = 0; i < nodes; ++i) {
      const int32_t b = node_offsets[i], e = node_offsets[i + 1];
      w.num(i).ch(' ').num(31 - __builtin_clz(static_cast<uint32_t>(i) + 1)).ch(' ').num(e - b);
      for (int32_t k = b; k < e; ++k) w.ch(' ').num(node_vertices[k]);
      w.ch('\n');
    }
    w.finish();
  });
}

}  // extern "C"

// ---- benchmark CSV (pipeline.cpp:188-205 csv_header / write_csv) ----------
extern "C" const char* mp_csv_header(void) {
  return "input,n,nnz_A,method,patch_size,nd_level,t_patch_ms,t_quotient_ms,"
         "t_etree_ms,t_local_ms,t_assemble_ms,nnz_L,fill_ratio,cost";
}

extern "C" int mp_write_csv(const char* path, const mp_bench_row* rows, int32_t count) {
  return io_guarded([&] {
    if (!path || (count > 0 && !rows)) throw Error(MP_EINVAL, "null argument");
    std::string text = std::string(mp_csv_header()) + "\n";
    char buf[192];
    for (int32_t i = 0; i < count; ++i) {
      const mp_bench_row& r = rows[i];
      std::snprintf(buf, sizeof buf, "%lld,%lld,", static_cast<long long>(r.n), static_cast<long long>(r.nnz_A));
      text += std::string(r.input ? r.input : "") + "," + buf + (r.method ? r.method : "") + ",";
      std::snprintf(buf, sizeof buf, "%d,%d,%.3f,%.3f,%.3f,%.3f,%.3f,%lld,%.6f,%lld\n", r.patch_size, r.nd_level,
                    r.t_patch_ms, r.t_quotient_ms, r.t_etree_ms, r.t_local_ms, r.t_assemble_ms,
                    static_cast<long long>(r.nnz_L), r.fill_ratio, static_cast<long long>(r.cost));
      text += buf;
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) throw IoError{std::string("cannot open ") + path + " for writing"};
    const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
    if (std::fclose(f) != 0 || !ok) throw IoError{std::string("write failed: ") + path};
  });
}
