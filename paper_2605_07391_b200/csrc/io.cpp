// io.cpp -- the host side of the MERBIT path's on-disk formats (SURVEY 8f,
// row f3).  Byte layouts are the reference's, so files cross between the
// two implementations; the readers are written here from the layouts:
//
//   MBTL  TILE cache      (tile.cpp:161-234)  "MBTL" | u32 version 1 | u32 omega
//                         | u32 sigma | u64 nnz | u64 n_rows | u8 f64-flag
//                         | u32 tile_x[tiles+1] | u32 tile_y[tiles+1]
//                         | u32 lane_desc[lanes]
//   MBMX  matrix cache    (matrix_market.cpp:178-225)  "MBMX" | u32 1
//                         | i64 n_rows | i64 n_cols | i64 count
//                         | count x {i64 row, i64 col, f64 value}
//   Matrix Market text    (matrix_market.cpp:47-133)  coordinate real /
//                         integer / pattern, general / symmetric (mirrored
//                         off-diagonals), 1-based, '%' comments, CRLF
//
// Design: every reader pulls the whole file into memory once and walks it
// with a cursor (MM: a line scanner + token splitter; binaries: one header
// record and bulk array copies), so no per-field stream calls.  Errors keep
// the reference's classes -- io_error (open / write), parse_error (MM syntax
// as "origin:line: message", bad magic / version), corruption_error (short
// files, impossible headers, out-of-range cache entries) -- with this file's
// own messages.  Device-side ingest (COO -> CSR, TILE upload) is ingest.cu.
#include <algorithm>
#include <bit>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <system_error>
#include <vector>

#include "mbx_internal.h"

static_assert(std::endian::native == std::endian::little,
              "MBTL / MBMX are little-endian raw layouts");

namespace mbx {
namespace {

constexpr uint32_t kFormatVersion = 1;

// ---- whole-file I/O ---------------------------------------------------------
std::string slurp(const std::string& path, bool binary) {
  std::FILE* f = std::fopen(path.c_str(), binary ? "rb" : "r");
  if (!f) fail(MBX_IO_ERROR, "cannot open '" + path + "'");
  std::string data;
  char chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) data.append(chunk, got);
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  if (bad) fail(MBX_IO_ERROR, "read error on '" + path + "'");
  return data;
}

class Sink {  // buffered binary / text writer with one error check at the end
 public:
  Sink(const std::string& path, bool binary) : path_(path) {
    f_ = std::fopen(path.c_str(), binary ? "wb" : "w");
    if (!f_) fail(MBX_IO_ERROR, "cannot write '" + path + "'");
  }
  ~Sink() {
    if (f_) std::fclose(f_);
  }
  void bytes(const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f_) != n) ok_ = false;
  }
  template <typename V>
  void pod(const V& v) {
    bytes(&v, sizeof(V));
  }
  void text(std::string_view s) { bytes(s.data(), s.size()); }
  void close() {
    const bool closed = std::fclose(f_) == 0;
    f_ = nullptr;
    if (!ok_ || !closed) fail(MBX_IO_ERROR, "write to '" + path_ + "' failed");
  }

 private:
  std::FILE* f_ = nullptr;
  std::string path_;
  bool ok_ = true;
};

// ---- binary cursor ----------------------------------------------------------
class Reader {
 public:
  Reader(const std::string& data, std::string path, const char* kind)
      : d_(data), path_(std::move(path)), kind_(kind) {}
  template <typename V>
  V pod() {
    V v;
    need(sizeof(V));
    std::memcpy(&v, d_.data() + at_, sizeof(V));
    at_ += sizeof(V);
    return v;
  }
  template <typename V>
  void array(V* out, int64_t n) {
    if (n <= 0) return;
    need(size_t(n) * sizeof(V));
    std::memcpy(out, d_.data() + at_, size_t(n) * sizeof(V));
    at_ += size_t(n) * sizeof(V);
  }
  bool magic(const char (&m)[5]) const {
    return d_.size() >= 4 && std::memcmp(d_.data(), m, 4) == 0;
  }
  void skip(size_t n) { at_ += n; }

 private:
  void need(size_t n) const {
    if (d_.size() - at_ < n)
      fail(MBX_CORRUPTION_ERROR, std::string(kind_) + " '" + path_ + "' ends early (" +
                                     std::to_string(d_.size()) + " bytes)");
  }
  const std::string& d_;
  std::string path_;
  const char* kind_;
  size_t at_ = 0;
};

template <typename V>
V* malloc_array(int64_t n) {
  void* p = std::malloc(sizeof(V) * size_t(std::max<int64_t>(n, 1)));
  if (!p) fail(MBX_ERROR, "host allocation failed");
  return static_cast<V*>(p);
}

struct HostCoo {
  int64_t n_rows = 0, n_cols = 0;
  std::vector<int64_t> r, c;
  std::vector<double> v;
  void add(int64_t row, int64_t col, double val) {
    r.push_back(row);
    c.push_back(col);
    v.push_back(val);
  }
};

void hand_over(HostCoo&& h, mbx_coo* out) {
  const int64_t n = int64_t(h.r.size());
  mbx_coo o{};
  o.n_rows = h.n_rows;
  o.n_cols = h.n_cols;
  o.nnz = n;
  o.rows = malloc_array<int64_t>(n);
  o.cols = malloc_array<int64_t>(n);
  o.vals = malloc_array<double>(n);
  std::copy(h.r.begin(), h.r.end(), o.rows);
  std::copy(h.c.begin(), h.c.end(), o.cols);
  std::copy(h.v.begin(), h.v.end(), o.vals);
  *out = o;
}

// ---- Matrix Market ----------------------------------------------------------
class MmText {
 public:
  MmText(std::string_view text, std::string origin) : t_(text), origin_(std::move(origin)) {}

  // the next physical line (CR stripped); false at the end
  bool raw_line(std::string_view& line) {
    if (pos_ >= t_.size() && !(pos_ == 0 && !t_.empty())) return false;
    const size_t nl = t_.find('\n', pos_);
    const size_t end = nl == std::string_view::npos ? t_.size() : nl;
    line = t_.substr(pos_, end - pos_);
    pos_ = nl == std::string_view::npos ? t_.size() + 1 : nl + 1;
    ++line_no_;
    if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
    return true;
  }
  // the next line carrying data: not blank, not a '%' comment
  bool data_line(std::string_view& line) {
    while (raw_line(line)) {
      const size_t k = line.find_first_not_of(" \t");
      if (k != std::string_view::npos && line[k] != '%') return true;
    }
    return false;
  }
  [[noreturn]] void error(const std::string& msg) const {
    fail(MBX_PARSE_ERROR, origin_ + ":" + std::to_string(line_no_) + ": " + msg);
  }
  size_t line_no() const { return line_no_; }

 private:
  std::string_view t_;
  std::string origin_;
  size_t pos_ = 0;
  size_t line_no_ = 0;
};

// whitespace-separated tokens of one line, at most N
template <int N>
int split(std::string_view line, std::string_view (&tok)[N]) {
  int k = 0;
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && (line[i] == ' ' || line[i] == '\t')) ++i;
    if (i >= line.size()) break;
    size_t j = i;
    while (j < line.size() && line[j] != ' ' && line[j] != '\t') ++j;
    if (k == N) return N + 1;  // more tokens than the caller accepts
    tok[k++] = line.substr(i, j - i);
    i = j;
  }
  return k;
}

bool to_int(std::string_view s, int64_t& v) {
  if (!s.empty() && s.front() == '+') s.remove_prefix(1);
  const auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  return ec == std::errc{} && p == s.data() + s.size();
}

bool to_real(std::string_view s, double& v) {
  // decimal notation only (no nan / inf / hex spellings)
  if (s.empty() || s.find_first_not_of("0123456789+-.eE") != std::string_view::npos) return false;
  if (s.front() == '+') s.remove_prefix(1);
  const auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  return ec == std::errc{} && p == s.data() + s.size();
}

bool same_word(std::string_view a, const char* b) {
  const size_t n = std::strlen(b);
  if (a.size() != n) return false;
  for (size_t i = 0; i < n; ++i)
    if (char(std::tolower(static_cast<unsigned char>(a[i]))) != b[i]) return false;
  return true;
}

enum class Field { real, integer, pattern };

HostCoo read_mm(std::string_view text, const std::string& origin) {
  MmText mm(text, origin);
  std::string_view line;
  if (!mm.raw_line(line) || (text.empty())) fail(MBX_PARSE_ERROR, origin + ": no content");
  // banner: %%MatrixMarket <object> <format> <field> <symmetry>
  std::string_view b[6];
  const int nb = split(line, b);
  if (nb < 1 || b[0] != "%%MatrixMarket") mm.error("first line is not a %%MatrixMarket header");
  if (nb < 5) mm.error("header needs object, format, field and symmetry");
  if (!same_word(b[1], "matrix")) mm.error("object '" + std::string(b[1]) + "' is not a matrix");
  if (!same_word(b[2], "coordinate"))
    mm.error("format '" + std::string(b[2]) + "' is not coordinate (dense arrays unsupported)");
  Field field;
  if (same_word(b[3], "real"))
    field = Field::real;
  else if (same_word(b[3], "integer"))
    field = Field::integer;
  else if (same_word(b[3], "pattern"))
    field = Field::pattern;
  else
    mm.error("field '" + std::string(b[3]) + "' is not real, integer or pattern");
  bool mirror;
  if (same_word(b[4], "general"))
    mirror = false;
  else if (same_word(b[4], "symmetric"))
    mirror = true;
  else
    mm.error("symmetry '" + std::string(b[4]) + "' is not general or symmetric");

  // size line: rows cols entries
  if (!mm.data_line(line)) mm.error("no size line after the header");
  std::string_view s[3];
  const int ns = split(line, s);
  HostCoo coo;
  int64_t count = 0;
  if (ns > 3) mm.error("size line has more than three numbers");
  if (ns != 3 || !to_int(s[0], coo.n_rows) || !to_int(s[1], coo.n_cols) || !to_int(s[2], count))
    mm.error("size line is not three integers");
  if (coo.n_rows < 0 || coo.n_cols < 0 || count < 0) mm.error("size line has a negative number");
  const size_t reserve = size_t(count) * (mirror ? 2 : 1);
  coo.r.reserve(reserve);
  coo.c.reserve(reserve);
  coo.v.reserve(reserve);

  const int want = field == Field::pattern ? 2 : 3;
  for (int64_t k = 0; k < count; ++k) {
    if (!mm.data_line(line))
      mm.error("file ends after " + std::to_string(k) + " of " + std::to_string(count) +
               " entries");
    std::string_view e[3];
    const int ne = split(line, e);
    if (ne > want) mm.error("entry has more than " + std::to_string(want) + " fields");
    int64_t i = 0, j = 0;
    if (ne < 2 || !to_int(e[0], i) || !to_int(e[1], j)) mm.error("entry indices are not integers");
    double val = 1.0;  // pattern entries count as 1
    if (want == 3 && (ne < 3 || !to_real(e[2], val))) mm.error("entry has no numeric value");
    if (i < 1 || i > coo.n_rows || j < 1 || j > coo.n_cols)
      mm.error("entry (" + std::to_string(i) + ", " + std::to_string(j) + ") is outside the " +
               std::to_string(coo.n_rows) + "x" + std::to_string(coo.n_cols) + " matrix");
    coo.add(i - 1, j - 1, val);
    if (mirror && i != j) coo.add(j - 1, i - 1, val);
  }
  if (mm.data_line(line)) mm.error("more entries than the size line declares");
  return coo;
}

void write_mm(const std::string& path, const mbx_coo& c) {
  Sink out(path, false);
  out.text("%%MatrixMarket matrix coordinate real general\n");
  out.text(std::to_string(c.n_rows) + " " + std::to_string(c.n_cols) + " " +
           std::to_string(c.nnz) + "\n");
  char buf[96];
  for (int64_t k = 0; k < c.nnz; ++k) {
    char* p = std::to_chars(buf, buf + 24, c.rows[k] + 1).ptr;
    *p++ = ' ';
    p = std::to_chars(p, p + 24, c.cols[k] + 1).ptr;
    *p++ = ' ';
    const auto r = std::to_chars(p, buf + sizeof(buf) - 1, c.vals[k]);  // shortest round trip
    if (r.ec != std::errc{}) fail(MBX_IO_ERROR, "cannot format a matrix value");
    *r.ptr = '\n';
    out.bytes(buf, size_t(r.ptr + 1 - buf));
  }
  out.close();
}

// ---- MBMX ---------------------------------------------------------------------
struct MbmxHeader {
  char magic[4];
  uint32_t version;
  int64_t n_rows, n_cols, count;
};
static_assert(sizeof(MbmxHeader) == 32, "MBMX header is 32 bytes");
struct MbmxEntry {
  int64_t row, col;
  double val;
};
static_assert(sizeof(MbmxEntry) == 24, "MBMX entries are 24 bytes");

HostCoo read_mbmx(const std::string& path) {
  const std::string data = slurp(path, true);
  Reader rd(data, path, "matrix cache");
  if (!rd.magic("MBMX")) fail(MBX_PARSE_ERROR, "'" + path + "' has no MBMX signature");
  rd.skip(4);
  const uint32_t version = rd.pod<uint32_t>();
  if (version != kFormatVersion)
    fail(MBX_PARSE_ERROR, "matrix cache '" + path + "' has version " + std::to_string(version) +
                              ", expected " + std::to_string(kFormatVersion));
  HostCoo coo;
  coo.n_rows = rd.pod<int64_t>();
  coo.n_cols = rd.pod<int64_t>();
  const int64_t count = rd.pod<int64_t>();
  if (coo.n_rows < 0 || coo.n_cols < 0 || count < 0)
    fail(MBX_CORRUPTION_ERROR, "matrix cache '" + path + "' declares a negative size");
  std::vector<MbmxEntry> e(static_cast<size_t>(count));
  rd.array(e.data(), count);
  coo.r.resize(e.size());
  coo.c.resize(e.size());
  coo.v.resize(e.size());
  for (size_t k = 0; k < e.size(); ++k) {
    if (e[k].row < 0 || e[k].row >= coo.n_rows || e[k].col < 0 || e[k].col >= coo.n_cols)
      fail(MBX_CORRUPTION_ERROR, "matrix cache '" + path + "' entry " + std::to_string(k) +
                                     " lies outside its " + std::to_string(coo.n_rows) + "x" +
                                     std::to_string(coo.n_cols) + " bounds");
    coo.r[k] = e[k].row;
    coo.c[k] = e[k].col;
    coo.v[k] = e[k].val;
  }
  return coo;
}

void write_mbmx(const std::string& path, const mbx_coo& c) {
  Sink out(path, true);
  MbmxHeader h;
  std::memcpy(h.magic, "MBMX", 4);
  h.version = kFormatVersion;
  h.n_rows = c.n_rows;
  h.n_cols = c.n_cols;
  h.count = c.nnz;
  out.pod(h);
  std::vector<MbmxEntry> buf;
  constexpr int64_t kBatch = 1 << 16;
  for (int64_t k0 = 0; k0 < c.nnz; k0 += kBatch) {
    const int64_t k1 = std::min(c.nnz, k0 + kBatch);
    buf.resize(size_t(k1 - k0));
    for (int64_t k = k0; k < k1; ++k) buf[size_t(k - k0)] = {c.rows[k], c.cols[k], c.vals[k]};
    out.bytes(buf.data(), buf.size() * sizeof(MbmxEntry));
  }
  out.close();
}

template <typename F>
int io_guard(F&& f) {
  try {
    f();
    return MBX_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MBX_ERROR;
  }
}

}  // namespace

// ---- MBTL (also used by ingest.cu for device TILEs) --------------------------
#pragma pack(push, 1)
struct MbtlHeader {
  char magic[4];
  uint32_t version, omega, sigma;
  uint64_t nnz, n_rows;
  uint8_t f64;
};
#pragma pack(pop)
static_assert(sizeof(MbtlHeader) == 33, "MBTL header is 33 bytes");

void write_tile_cache_host(const std::string& path, const mbx_tile_info& info,
                           const uint32_t* tx, const uint32_t* ty, const uint32_t* ld,
                           int precision) {
  Sink out(path, true);
  MbtlHeader h;
  std::memcpy(h.magic, "MBTL", 4);
  h.version = kFormatVersion;
  h.omega = uint32_t(info.omega);
  h.sigma = uint32_t(info.sigma);
  h.nnz = uint64_t(info.nnz);
  h.n_rows = uint64_t(info.n_rows);
  h.f64 = precision == MBX_F64 ? 1 : 0;
  out.pod(h);
  out.bytes(tx, size_t(info.tile_num + 1) * 4);
  out.bytes(ty, size_t(info.tile_num + 1) * 4);
  out.bytes(ld, size_t(info.lane_num) * 4);
  out.close();
}

void read_tile_cache_host(const std::string& path, mbx_tile_info* info, uint32_t** tx,
                          uint32_t** ty, uint32_t** ld, int* precision) {
  const std::string data = slurp(path, true);
  Reader rd(data, path, "tile cache");
  if (!rd.magic("MBTL")) fail(MBX_PARSE_ERROR, "'" + path + "' has no MBTL signature");
  const MbtlHeader h = rd.pod<MbtlHeader>();
  if (h.version != kFormatVersion)
    fail(MBX_PARSE_ERROR, "tile cache '" + path + "' has version " + std::to_string(h.version) +
                              ", expected " + std::to_string(kFormatVersion));
  mbx_tile_info t{};
  t.omega = int32_t(h.omega);
  t.sigma = int32_t(h.sigma);
  t.nnz = int64_t(h.nnz);
  t.n_rows = int64_t(h.n_rows);
  if (t.omega < 1 || t.sigma < 1 || t.nnz < 0 || t.n_rows < 0)
    fail(MBX_CORRUPTION_ERROR, "tile cache '" + path + "' has an impossible header");
  // the array lengths follow from the header, as generate_tile sizes them
  const int64_t steps = t.nnz + t.n_rows;
  const int64_t lanes = steps == 0 ? 0 : (steps + t.sigma - 1) / t.sigma;
  const int64_t tiles = steps == 0 ? 0 : (steps + int64_t(t.omega) * t.sigma - 1) /
                                             (int64_t(t.omega) * t.sigma);
  t.tile_num = tiles;
  t.lane_num = lanes;
  std::unique_ptr<uint32_t, void (*)(void*)> x(malloc_array<uint32_t>(tiles + 1), std::free);
  std::unique_ptr<uint32_t, void (*)(void*)> y(malloc_array<uint32_t>(tiles + 1), std::free);
  std::unique_ptr<uint32_t, void (*)(void*)> d(malloc_array<uint32_t>(lanes), std::free);
  rd.array(x.get(), tiles + 1);
  rd.array(y.get(), tiles + 1);
  rd.array(d.get(), lanes);
  *info = t;
  *tx = x.release();
  *ty = y.release();
  *ld = d.release();
  if (precision) *precision = h.f64 ? MBX_F64 : MBX_F32;
}

}  // namespace mbx

extern "C" {

MBX_API void mbx_free(void* p) { std::free(p); }

MBX_API void mbx_coo_free(mbx_coo* c) {
  if (!c) return;
  std::free(c->rows);
  std::free(c->cols);
  std::free(c->vals);
  c->rows = c->cols = nullptr;
  c->vals = nullptr;
  c->nnz = 0;
}

MBX_API int mbx_tile_cache_write_host(const char* path, const mbx_tile_info* info,
                                      const uint32_t* tile_x, const uint32_t* tile_y,
                                      const uint32_t* lane_desc, int precision) {
  return mbx::io_guard(
      [&] { mbx::write_tile_cache_host(path, *info, tile_x, tile_y, lane_desc, precision); });
}

MBX_API int mbx_tile_cache_read_host(const char* path, mbx_tile_info* info, uint32_t** tile_x,
                                     uint32_t** tile_y, uint32_t** lane_desc, int* precision) {
  return mbx::io_guard(
      [&] { mbx::read_tile_cache_host(path, info, tile_x, tile_y, lane_desc, precision); });
}

MBX_API int mbx_mm_read(const char* path, mbx_coo* out) {
  return mbx::io_guard([&] {
    const std::string text = mbx::slurp(path, false);
    mbx::hand_over(mbx::read_mm(text, path), out);
  });
}

MBX_API int mbx_mm_parse(const char* text, int64_t len, const char* origin, mbx_coo* out) {
  return mbx::io_guard([&] {
    mbx::hand_over(mbx::read_mm(std::string_view(text, size_t(len)), origin ? origin : "<memory>"),
                   out);
  });
}

MBX_API int mbx_mm_write(const char* path, const mbx_coo* c) {
  return mbx::io_guard([&] { mbx::write_mm(path, *c); });
}

MBX_API int mbx_matrix_cache_write(const char* path, const mbx_coo* c) {
  return mbx::io_guard([&] { mbx::write_mbmx(path, *c); });
}

MBX_API int mbx_matrix_cache_read(const char* path, mbx_coo* out) {
  return mbx::io_guard([&] { mbx::hand_over(mbx::read_mbmx(path), out); });
}

MBX_API int mbx_matrix_load_any(const char* path, mbx_coo* out) {
  return mbx::io_guard([&] {
    // the binary cache announces itself with its signature; anything else
    // is read as Matrix Market text
    std::FILE* f = std::fopen(path, "rb");
    if (!f) mbx::fail(MBX_IO_ERROR, std::string("cannot open '") + path + "'");
    char head[4] = {0, 0, 0, 0};
    const size_t got = std::fread(head, 1, 4, f);
    std::fclose(f);
    if (got == 4 && std::memcmp(head, "MBMX", 4) == 0) {
      mbx::hand_over(mbx::read_mbmx(path), out);
    } else {
      const std::string text = mbx::slurp(path, false);
      mbx::hand_over(mbx::read_mm(text, path), out);
    }
  });
}

}  // extern "C"
