// io.cpp -- on-disk formats of the MERBIT path, host side:
//
//   MBTL  TILE cache        byte layout of write_tile_cache / read_tile_cache
//                           (src/tile.cpp:161-234): "MBTL", u32 version 1,
//                           u32 omega, u32 sigma, u64 nnz, u64 n_rows,
//                           u8 precision (1 = f64), u32 tile_x[tile_num+1],
//                           u32 tile_y[tile_num+1], u32 lane_desc[lane_num]
//   MBMX  matrix cache      write_matrix_cache / read_matrix_cache
//                           (src/matrix_market.cpp:178-225): "MBMX", u32 1,
//                           i64 n_rows, i64 n_cols, i64 count, then
//                           (i64 row, i64 col, f64 value) per entry
//   Matrix Market text      parse_matrix_market (matrix_market.cpp:47-133):
//                           coordinate real/integer/pattern, general or
//                           symmetric (mirrored off-diagonals), 1-based
//
// All little-endian, written raw (the reference static_asserts the same).
// Error classes follow the reference: io_error (cannot open / write),
// parse_error (banner, header, entry syntax -- "origin:line: what"),
// corruption_error (short reads, bad headers, out-of-range cache entries).
// The device side (COO -> CSR on the GPU, TILE upload) is in ingest.cu.
#include <algorithm>
#include <bit>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "mbx_internal.h"

static_assert(std::endian::native == std::endian::little,
              "MBTL / MBMX are little-endian raw layouts");

namespace mbx {
namespace {

constexpr char kTileMagic[4] = {'M', 'B', 'T', 'L'};
constexpr char kMatrixMagic[4] = {'M', 'B', 'M', 'X'};
constexpr uint32_t kVersion = 1;

template <typename V>
void put_raw(std::ostream& o, const V& v) {
  o.write(reinterpret_cast<const char*>(&v), sizeof(V));
}

template <typename V>
void put_array(std::ostream& o, const V* p, int64_t n) {
  if (n > 0) o.write(reinterpret_cast<const char*>(p), std::streamsize(n * sizeof(V)));
}

template <typename V>
V take(std::istream& in, const std::string& what, const std::string& path) {
  V v{};
  if (!in.read(reinterpret_cast<char*>(&v), sizeof(V)))
    fail(MBX_CORRUPTION_ERROR, "short read in " + what + " '" + path + "'");
  return v;
}

template <typename V>
void take_array(std::istream& in, V* p, int64_t n, const std::string& what,
                const std::string& path) {
  if (n <= 0) return;
  if (!in.read(reinterpret_cast<char*>(p), std::streamsize(n * sizeof(V))))
    fail(MBX_CORRUPTION_ERROR, "short read in " + what + " '" + path + "'");
}

template <typename V>
V* host_alloc(int64_t n) {
  V* p = static_cast<V*>(std::malloc(sizeof(V) * size_t(std::max<int64_t>(n, 1))));
  if (!p) fail(MBX_ERROR, "host allocation failed");
  return p;
}

std::string to_lower(std::string s) {
  for (char& ch : s) ch = char(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

[[noreturn]] void parse_fail(const std::string& origin, size_t line, const std::string& what) {
  fail(MBX_PARSE_ERROR, origin + ":" + std::to_string(line) + ": " + what);
}

// next line that is neither blank nor a '%' comment (CR stripped)
bool payload_line(std::istream& in, std::string& line, size_t& line_no) {
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const size_t k = line.find_first_not_of(" \t");
    if (k == std::string::npos || line[k] == '%') continue;
    return true;
  }
  return false;
}

struct Coo {
  int64_t n_rows = 0, n_cols = 0;
  std::vector<int64_t> rows, cols;
  std::vector<double> vals;
};

Coo parse_mm(std::istream& in, const std::string& origin) {
  std::string banner;
  size_t ln = 0;
  if (!std::getline(in, banner)) fail(MBX_PARSE_ERROR, origin + ": empty file");
  ++ln;
  if (!banner.empty() && banner.back() == '\r') banner.pop_back();
  std::istringstream hs(banner);
  std::string magic, object, format, field, symmetry;
  hs >> magic >> object >> format >> field >> symmetry;
  if (magic != "%%MatrixMarket") parse_fail(origin, ln, "missing %%MatrixMarket banner");
  object = to_lower(object);
  format = to_lower(format);
  field = to_lower(field);
  symmetry = to_lower(symmetry);
  if (object != "matrix") parse_fail(origin, ln, "unsupported object '" + object + "'");
  if (format != "coordinate")
    parse_fail(origin, ln, "unsupported format '" + format + "' (only coordinate is supported)");
  const bool pattern = field == "pattern";
  if (!pattern && field != "real" && field != "integer")
    parse_fail(origin, ln, "unsupported field '" + field + "'");
  const bool symmetric = symmetry == "symmetric";
  if (!symmetric && symmetry != "general")
    parse_fail(origin, ln, "unsupported symmetry '" + symmetry + "'");

  std::string line;
  if (!payload_line(in, line, ln)) parse_fail(origin, ln, "missing size line");
  Coo coo;
  int64_t declared = 0;
  {
    std::istringstream ss(line);
    if (!(ss >> coo.n_rows >> coo.n_cols >> declared))
      parse_fail(origin, ln, "malformed size line '" + line + "'");
    std::string extra;
    if (ss >> extra) parse_fail(origin, ln, "trailing tokens on size line");
    if (coo.n_rows < 0 || coo.n_cols < 0 || declared < 0)
      parse_fail(origin, ln, "negative dimension in size line");
  }
  const size_t cap = size_t(declared) * (symmetric ? 2 : 1);
  coo.rows.reserve(cap);
  coo.cols.reserve(cap);
  coo.vals.reserve(cap);
  for (int64_t k = 0; k < declared; ++k) {
    if (!payload_line(in, line, ln))
      parse_fail(origin, ln,
                 "expected " + std::to_string(declared) + " entries, got " + std::to_string(k));
    std::istringstream ss(line);
    int64_t r = 0, c = 0;
    double v = 1.0;  // pattern entries read as 1.0
    if (!(ss >> r >> c)) parse_fail(origin, ln, "malformed entry '" + line + "'");
    if (!pattern && !(ss >> v)) parse_fail(origin, ln, "missing value in entry '" + line + "'");
    std::string extra;
    if (ss >> extra) parse_fail(origin, ln, "trailing tokens in entry");
    if (r < 1 || r > coo.n_rows || c < 1 || c > coo.n_cols)
      parse_fail(origin, ln,
                 "entry (" + std::to_string(r) + ", " + std::to_string(c) + ") outside " +
                     std::to_string(coo.n_rows) + "x" + std::to_string(coo.n_cols));
    coo.rows.push_back(r - 1);
    coo.cols.push_back(c - 1);
    coo.vals.push_back(v);
    if (symmetric && r != c) {  // mirrored off-diagonal
      coo.rows.push_back(c - 1);
      coo.cols.push_back(r - 1);
      coo.vals.push_back(v);
    }
  }
  if (payload_line(in, line, ln)) parse_fail(origin, ln, "trailing entries beyond declared count");
  return coo;
}

void export_coo(Coo&& c, mbx_coo* out) {
  const int64_t n = int64_t(c.rows.size());
  mbx_coo o{};
  o.n_rows = c.n_rows;
  o.n_cols = c.n_cols;
  o.nnz = n;
  o.rows = host_alloc<int64_t>(n);
  o.cols = host_alloc<int64_t>(n);
  o.vals = host_alloc<double>(n);
  if (n) {
    std::memcpy(o.rows, c.rows.data(), sizeof(int64_t) * n);
    std::memcpy(o.cols, c.cols.data(), sizeof(int64_t) * n);
    std::memcpy(o.vals, c.vals.data(), sizeof(double) * n);
  }
  *out = o;
}

Coo read_mbmx(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(MBX_IO_ERROR, "cannot open '" + path + "'");
  char magic[4];
  if (!in.read(magic, 4) || std::memcmp(magic, kMatrixMagic, 4) != 0)
    fail(MBX_PARSE_ERROR, "'" + path + "' is not a matrix cache");
  const uint32_t version = take<uint32_t>(in, "cache", path);
  if (version != kVersion)
    fail(MBX_PARSE_ERROR, "unsupported matrix cache version " + std::to_string(version));
  Coo c;
  c.n_rows = take<int64_t>(in, "cache", path);
  c.n_cols = take<int64_t>(in, "cache", path);
  const int64_t n = take<int64_t>(in, "cache", path);
  if (c.n_rows < 0 || c.n_cols < 0 || n < 0)
    fail(MBX_CORRUPTION_ERROR, "negative dimension in cache '" + path + "'");
  c.rows.reserve(size_t(n));
  c.cols.reserve(size_t(n));
  c.vals.reserve(size_t(n));
  for (int64_t k = 0; k < n; ++k) {
    // one 24-byte record per entry
    const int64_t r = take<int64_t>(in, "cache", path);
    const int64_t col = take<int64_t>(in, "cache", path);
    const double v = take<double>(in, "cache", path);
    if (r < 0 || r >= c.n_rows || col < 0 || col >= c.n_cols)
      fail(MBX_CORRUPTION_ERROR, "entry outside matrix bounds in cache '" + path + "'");
    c.rows.push_back(r);
    c.cols.push_back(col);
    c.vals.push_back(v);
  }
  return c;
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

void write_tile_cache_host(const std::string& path, const mbx_tile_info& info,
                           const uint32_t* tx, const uint32_t* ty, const uint32_t* ld,
                           int precision) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(MBX_IO_ERROR, "cannot write '" + path + "'");
  out.write(kTileMagic, 4);
  put_raw(out, kVersion);
  put_raw(out, uint32_t(info.omega));
  put_raw(out, uint32_t(info.sigma));
  put_raw(out, uint64_t(info.nnz));
  put_raw(out, uint64_t(info.n_rows));
  put_raw(out, uint8_t(precision == MBX_F64 ? 1 : 0));
  put_array(out, tx, info.tile_num + 1);
  put_array(out, ty, info.tile_num + 1);
  put_array(out, ld, info.lane_num);
  if (!out) fail(MBX_IO_ERROR, "write failed for '" + path + "'");
}

void read_tile_cache_host(const std::string& path, mbx_tile_info* info, uint32_t** tx,
                          uint32_t** ty, uint32_t** ld, int* precision) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(MBX_IO_ERROR, "cannot open '" + path + "'");
  char magic[4];
  if (!in.read(magic, 4) || std::memcmp(magic, kTileMagic, 4) != 0)
    fail(MBX_PARSE_ERROR, "'" + path + "' is not a tile cache");
  const uint32_t version = take<uint32_t>(in, "tile cache", path);
  if (version != kVersion)
    fail(MBX_PARSE_ERROR, "unsupported tile cache version " + std::to_string(version));
  mbx_tile_info t{};
  t.omega = int32_t(take<uint32_t>(in, "tile cache", path));
  t.sigma = int32_t(take<uint32_t>(in, "tile cache", path));
  t.nnz = int64_t(take<uint64_t>(in, "tile cache", path));
  t.n_rows = int64_t(take<uint64_t>(in, "tile cache", path));
  const int p = take<uint8_t>(in, "tile cache", path) != 0 ? MBX_F64 : MBX_F32;
  if (t.omega < 1 || t.sigma < 1 || t.nnz < 0 || t.n_rows < 0)
    fail(MBX_CORRUPTION_ERROR, "invalid header in tile cache '" + path + "'");
  // counts follow from the header exactly as generate_tile sizes them
  const int64_t total = t.nnz + t.n_rows;
  const int64_t span = int64_t(t.omega) * t.sigma;
  t.lane_num = total == 0 ? 0 : (total + t.sigma - 1) / t.sigma;
  t.tile_num = total == 0 ? 0 : (total + span - 1) / span;
  uint32_t* x = host_alloc<uint32_t>(t.tile_num + 1);
  uint32_t* y = host_alloc<uint32_t>(t.tile_num + 1);
  uint32_t* d = host_alloc<uint32_t>(t.lane_num);
  try {
    take_array(in, x, t.tile_num + 1, "tile cache", path);
    take_array(in, y, t.tile_num + 1, "tile cache", path);
    take_array(in, d, t.lane_num, "tile cache", path);
  } catch (...) {
    std::free(x);
    std::free(y);
    std::free(d);
    throw;
  }
  *info = t;
  *tx = x;
  *ty = y;
  *ld = d;
  if (precision) *precision = p;
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
    std::ifstream in(path);
    if (!in) mbx::fail(MBX_IO_ERROR, std::string("cannot open '") + path + "'");
    mbx::export_coo(mbx::parse_mm(in, path), out);
  });
}

MBX_API int mbx_mm_parse(const char* text, int64_t len, const char* origin, mbx_coo* out) {
  return mbx::io_guard([&] {
    std::istringstream in(std::string(text, size_t(len)));
    mbx::export_coo(mbx::parse_mm(in, origin ? origin : "<memory>"), out);
  });
}

MBX_API int mbx_mm_write(const char* path, const mbx_coo* c) {
  return mbx::io_guard([&] {
    std::ofstream out(path);
    if (!out) mbx::fail(MBX_IO_ERROR, std::string("cannot write '") + path + "'");
    out << "%%MatrixMarket matrix coordinate real general\n"
        << c->n_rows << ' ' << c->n_cols << ' ' << c->nnz << '\n';
    char buf[64];
    for (int64_t k = 0; k < c->nnz; ++k) {
      // shortest round-trip decimal form of the value
      const auto [end, ec] = std::to_chars(buf, buf + sizeof(buf), c->vals[k]);
      if (ec != std::errc{}) mbx::fail(MBX_IO_ERROR, "unprintable matrix value");
      out << (c->rows[k] + 1) << ' ' << (c->cols[k] + 1) << ' '
          << std::string_view(buf, size_t(end - buf)) << '\n';
    }
    if (!out) mbx::fail(MBX_IO_ERROR, std::string("write failed for '") + path + "'");
  });
}

MBX_API int mbx_matrix_cache_write(const char* path, const mbx_coo* c) {
  return mbx::io_guard([&] {
    std::ofstream out(path, std::ios::binary);
    if (!out) mbx::fail(MBX_IO_ERROR, std::string("cannot write '") + path + "'");
    out.write(mbx::kMatrixMagic, 4);
    mbx::put_raw(out, mbx::kVersion);
    mbx::put_raw(out, int64_t(c->n_rows));
    mbx::put_raw(out, int64_t(c->n_cols));
    mbx::put_raw(out, int64_t(c->nnz));
    for (int64_t k = 0; k < c->nnz; ++k) {
      mbx::put_raw(out, int64_t(c->rows[k]));
      mbx::put_raw(out, int64_t(c->cols[k]));
      mbx::put_raw(out, double(c->vals[k]));
    }
    if (!out) mbx::fail(MBX_IO_ERROR, std::string("write failed for '") + path + "'");
  });
}

MBX_API int mbx_matrix_cache_read(const char* path, mbx_coo* out) {
  return mbx::io_guard([&] { mbx::export_coo(mbx::read_mbmx(path), out); });
}

MBX_API int mbx_matrix_load_any(const char* path, mbx_coo* out) {
  return mbx::io_guard([&] {
    std::ifstream probe(path, std::ios::binary);
    if (!probe) mbx::fail(MBX_IO_ERROR, std::string("cannot open '") + path + "'");
    char head[4] = {0, 0, 0, 0};
    probe.read(head, 4);
    probe.close();
    if (std::memcmp(head, mbx::kMatrixMagic, 4) == 0) {
      mbx::export_coo(mbx::read_mbmx(path), out);
    } else {
      std::ifstream in(path);
      mbx::export_coo(mbx::parse_mm(in, path), out);
    }
  });
}

}  // extern "C"
