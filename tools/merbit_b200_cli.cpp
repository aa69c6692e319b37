// merbit_b200 -- command-line harness over libmerbit_b200.so (SURVEY 8f row
// f4), verb for verb the reference's tools/merbit_cli.cpp: ingest, validate,
// benchmark, sigma sweeps, and the two iterative workloads, with BenchRecord
// schema-v1 CSV/JSON output so rows compare with the reference tooling.
// Every multiply, TILE, COO normalisation and solver runs on the GPU; this
// program only parses arguments, moves host arrays and prints.
//
//   merbit_b200 validate    <matrix> [--tile cache] [config options]
//   merbit_b200 bench       <matrix> [--kernels coo,csr,merge,merge-cub,merbit]
//                           [--iters N] [--warmup N] [--format csv|json] [--out f]
//   merbit_b200 sigma-sweep <matrix> [--sigmas 4,7,14|1-20] [--iters --warmup
//                           --format --out]
//   merbit_b200 pagerank    <adjacency> [--damping --err-tol --max-iters
//                           --reference-iters --out]
//   merbit_b200 bicgstab    <matrix> [--tol --max-iters --out]
//   merbit_b200 convert     <matrix> --out cache.mbmx [--tile cache.mbtl]
//   merbit_b200 gen         <walkthrough|laplacian|ring|dense-row|singular>
//                           --out f.mtx [--grid --nodes --chords --width --seed]
//   config options: --precision f32|f64 (default f64) --omega 32 --sigma S
//                   --block-size B (default 4*omega) --seed 1
//
// Exit codes (merbit_cli.cpp:1-6, 770-791): 0 success; 2 validation failure;
// 3 I/O or malformed input; 4 infeasible or invalid configuration; 5 solver
// breakdown; 1 anything else; 64 usage error.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "merbit_b200.h"
#include "merbit_b200/bench_record.hpp"
#include "merbit_b200/merbit.hpp"

namespace {

using namespace merbit_b200;

constexpr int kExitValidation = 2;
constexpr int kExitInput = 3;
constexpr int kExitConfig = 4;
constexpr int kExitBreakdown = 5;
constexpr int kExitUsage = 64;

struct usage_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- arguments --------------------------------------------------------------
struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  double num(const std::string& k, double d) const {
    if (!has(k)) return d;
    try {
      size_t used = 0;
      const double v = std::stod(opt.at(k), &used);
      if (used != opt.at(k).size()) throw std::invalid_argument(k);
      return v;
    } catch (const std::exception&) {
      throw usage_error("--" + k + " expects a number, got '" + opt.at(k) + "'");
    }
  }
  int64_t integer(const std::string& k, int64_t d) const {
    const double v = num(k, double(d));
    if (v != std::floor(v)) throw usage_error("--" + k + " expects an integer");
    return int64_t(v);
  }
};

Args parse_args(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) == 0) {
      std::string key = s.substr(2), val;
      const auto eq = key.find('=');
      if (eq != std::string::npos) {
        val = key.substr(eq + 1);
        key = key.substr(0, eq);
      } else {
        if (i + 1 >= argc) throw usage_error("option --" + key + " needs a value");
        val = argv[++i];
      }
      a.opt[key] = val;
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

std::string dataset_id(const std::string& path) {
  return std::filesystem::path(path).stem().string();
}

struct Sink {
  explicit Sink(const std::string& path) {
    if (!path.empty()) {
      f.open(path);
      if (!f) throw io_error("cannot write '" + path + "'");
      out = &f;
    }
  }
  std::ofstream f;
  std::ostream* out = &std::cout;
};

// a flat JSON object with sorted keys and two-space indentation (the layout
// of the reference's nlohmann reports)
using Fields = std::vector<std::pair<std::string, std::string>>;
std::string json_object(Fields f, const std::string& indent = "") {
  std::sort(f.begin(), f.end());
  std::string o = indent + "{\n";
  for (size_t i = 0; i < f.size(); ++i)
    o += indent + "  " + json_string(f[i].first) + ": " + f[i].second + (i + 1 < f.size() ? ",\n" : "\n");
  return o + indent + "}";
}

// ---- config -------------------------------------------------------------------
struct Kernel {
  int precision = MBX_F64;
  int omega = 32;
  std::optional<int> sigma, block;
  uint64_t seed = 1;
  const char* pname() const { return precision == MBX_F32 ? "f32" : "f64"; }
  size_t vs() const { return precision == MBX_F32 ? 4 : 8; }
  mbx_simt_config config(std::optional<int> s = {}) const {
    const int sg = mbx_select_sigma(precision, s.value_or(sigma.value_or(0)));
    mbx_simt_config c{};
    check(mbx_config_make(omega, sg, block.value_or(4 * omega), &c));
    return c;
  }
};

Kernel kernel_options(const Args& a) {
  Kernel k;
  const std::string p = a.get("precision", "f64");
  if (p != "f32" && p != "f64")
    throw config_error("unknown precision '" + p + "' (expected f32 or f64)");
  k.precision = p == "f32" ? MBX_F32 : MBX_F64;
  k.omega = int(a.integer("omega", 32));
  if (a.has("sigma")) k.sigma = int(a.integer("sigma", 0));
  if (a.has("block-size")) k.block = int(a.integer("block-size", 0));
  k.seed = uint64_t(a.integer("seed", 1));
  return k;
}

// ---- host helpers (inputs only) -------------------------------------------------
// seed_test_vector (random.hpp:23-31): mt19937_64, top 53 bits -> [lo, hi)
std::vector<double> seed_vector(int64_t n, double lo, double hi, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<double> v(size_t(std::max<int64_t>(n, 0)));
  for (double& e : v) e = lo + (hi - lo) * (double(rng() >> 11) * 0x1.0p-53);
  return v;
}

std::vector<char> as_precision(const std::vector<double>& v, int precision) {
  std::vector<char> out(v.size() * (precision == MBX_F32 ? 4 : 8));
  if (precision == MBX_F32)
    for (size_t i = 0; i < v.size(); ++i) reinterpret_cast<float*>(out.data())[i] = float(v[i]);
  else
    std::memcpy(out.data(), v.data(), v.size() * 8);
  return out;
}

struct Coo {
  mbx_coo c{};
  ~Coo() { mbx_coo_free(&c); }
};

struct Matrix {
  mbx_matrix* h = nullptr;
  ~Matrix() {
    if (h) mbx_matrix_destroy(h);
  }
};
struct Tile {
  mbx_tile* h = nullptr;
  ~Tile() {
    if (h) mbx_tile_destroy(h);
  }
};

struct Loaded {
  Coo raw;
  Matrix a;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
};

void load(mbx_context* ctx, const std::string& path, int precision, Loaded& L) {
  check(mbx_matrix_load_any(path.c_str(), &L.raw.c));
  check(mbx_matrix_from_coo(ctx, precision, &L.raw.c, &L.a.h));  // coo_to_csr<T> on the GPU
  int p = 0;
  check(mbx_matrix_info(L.a.h, &p, &L.n_rows, &L.n_cols, &L.nnz));
}

struct HostCsr {
  std::vector<int64_t> ro;
  std::vector<int32_t> cols;
  std::vector<char> vals;
};

HostCsr download(const Loaded& L, size_t vs) {
  HostCsr h;
  h.ro.resize(L.n_rows + 1);
  h.cols.resize(std::max<int64_t>(L.nnz, 1));
  h.vals.resize(std::max<int64_t>(L.nnz, 1) * vs);
  check(mbx_matrix_download(L.a.h, h.ro.data(), h.cols.data(), h.vals.data()));
  return h;
}

double long_row_fraction(const mbx_tile_info& info, const std::vector<uint32_t>& ty) {
  if (info.tile_num == 0) return 0.0;
  int64_t marked = 0;
  for (int64_t i = 0; i < info.tile_num; ++i) marked += (ty[i] & 0x80000000u) ? 1 : 0;
  return double(marked) / double(info.tile_num);
}

struct TileHost {
  mbx_tile_info info{};
  std::vector<uint32_t> tx, ty, ld;
};

TileHost download_tile(const mbx_tile* t) {
  TileHost h;
  check(mbx_tile_get_info(t, &h.info));
  h.tx.resize(h.info.tile_num + 1);
  h.ty.resize(h.info.tile_num + 1);
  h.ld.resize(std::max<int64_t>(h.info.lane_num, 1));
  check(mbx_tile_download(t, h.tx.data(), h.ty.data(), h.ld.data()));
  return h;
}

// reconstruct_path (tile.cpp:86-133) on the decoded descriptors vs the
// one-step-at-a-time walk of row_offsets: true iff they agree everywhere
bool path_matches(const mbx_tile_info& t, int ob, const uint32_t* tx, const uint32_t* ty,
                  const uint32_t* ld, const std::vector<int64_t>& ro, int64_t n, int64_t m) {
  if (t.n_rows != n || t.nnz != m) return false;
  const uint32_t mask = (1u << ob) - 1u;
  int64_t x = 0, y = 0, wx = 0, wy = 0;
  const int64_t total = n + m;
  for (int64_t j = 0; j < t.lane_num; ++j) {
    const int64_t tile = j / t.omega;
    const uint32_t d = ld[j];
    if (int64_t(tx[tile]) + (d & mask) != x ||
        int64_t(ty[tile] & 0x7FFFFFFFu) + ((d >> ob) & mask) != y)
      return false;
    const int64_t steps = std::min<int64_t>(t.sigma, total - j * t.sigma);
    const uint32_t fl = d >> (2 * ob);
    for (int64_t k = 0; k < steps; ++k) {
      const bool down_walk = !(wy < n && wx < ro[wy + 1]);
      if (down_walk) ++wy; else ++wx;
      if ((fl >> k) & 1u) ++y; else ++x;
      if (x != wx || y != wy) return false;
    }
  }
  return x == m && y == n;
}

// ToleranceBound-style componentwise check (reference.hpp:51-67):
// |got - want| <= 4 eps len max|A| max|x| per row
bool within_bound(const HostCsr& h, int precision, const std::vector<double>& x,
                  const std::vector<double>& want, const std::vector<double>& got) {
  const bool f32 = precision == MBX_F32;
  const double eps = f32 ? 1.1920928955078125e-07 : 2.220446049250313e-16;
  double max_a = 0.0, max_x = 0.0;
  const int64_t m = h.ro.back();
  for (int64_t k = 0; k < m; ++k) {
    const double v = f32 ? double(reinterpret_cast<const float*>(h.vals.data())[k])
                         : reinterpret_cast<const double*>(h.vals.data())[k];
    max_a = std::max(max_a, std::abs(v));
  }
  for (double v : x) max_x = std::max(max_x, std::abs(v));
  for (size_t r = 0; r + 1 < h.ro.size(); ++r) {
    const double bound = 4.0 * eps * double(h.ro[r + 1] - h.ro[r]) * max_a * max_x;
    if (!(std::abs(got[r] - want[r]) <= bound)) return false;
  }
  return true;
}

std::vector<double> to_double(const std::vector<char>& v, int precision, int64_t n) {
  std::vector<double> o(size_t(std::max<int64_t>(n, 0)));
  for (int64_t i = 0; i < n; ++i)
    o[i] = precision == MBX_F32 ? double(reinterpret_cast<const float*>(v.data())[i])
                                : reinterpret_cast<const double*>(v.data())[i];
  return o;
}

// y = A x through the C ABI's host-facing spmv_merbit (H2D x, K2+K3, D2H y)
std::vector<double> multiply(mbx_context* ctx, const Loaded& L, const mbx_tile* t,
                             const mbx_simt_config& c, int precision, const std::vector<char>& x) {
  std::vector<char> y(std::max<int64_t>(L.n_rows, 1) * (precision == MBX_F32 ? 4 : 8));
  check(mbx_spmv(ctx, L.a.h, t, &c, x.data(), y.data(), nullptr));
  return to_double(y, precision, L.n_rows);
}

std::vector<double> host_reference(const HostCsr& h, int precision, const std::vector<double>& xs,
                                   int64_t n_rows) {
  const bool f32 = precision == MBX_F32;
  std::vector<double> want(size_t(std::max<int64_t>(n_rows, 0)));
  for (int64_t r = 0; r < n_rows; ++r) {
    long double s = 0.0L;
    for (int64_t q = h.ro[r]; q < h.ro[r + 1]; ++q) {
      const double v = f32 ? double(reinterpret_cast<const float*>(h.vals.data())[q])
                           : reinterpret_cast<const double*>(h.vals.data())[q];
      const double xv = f32 ? double(float(xs[h.cols[q]])) : xs[h.cols[q]];
      s += (long double)v * (long double)xv;
    }
    want[r] = double(s);
  }
  return want;
}

// ---- verbs ----------------------------------------------------------------------
int cmd_validate(mbx_context* ctx, const Args& a) {
  if (a.pos.size() != 1) throw usage_error("validate needs exactly one matrix path");
  const std::string path = a.pos[0];
  const bool explicit_cfg = a.has("omega") || a.has("sigma") || a.has("block-size");
  std::vector<int> precs;
  if (a.has("precision") || explicit_cfg)
    precs.push_back(kernel_options(a).precision);
  else
    precs = {MBX_F32, MBX_F64};
  bool ok = true;
  for (int p : precs) {
    Args ap = a;
    ap.opt["precision"] = p == MBX_F32 ? "f32" : "f64";
    const Kernel k = kernel_options(ap);
    std::vector<mbx_simt_config> cfgs;
    if (explicit_cfg) {
      cfgs.push_back(k.config());
    } else {
      for (auto [w, s, b] : {std::tuple{32, 14, 128}, std::tuple{32, 7, 128}, std::tuple{4, 4, 16}}) {
        mbx_simt_config c{};
        check(mbx_config_make(w, s, b, &c));
        cfgs.push_back(c);
      }
    }
    Loaded L;
    load(ctx, path, p, L);
    const HostCsr h = download(L, k.vs());
    const auto xs = seed_vector(L.n_cols, -1.0, 1.0, k.seed);
    const auto x = as_precision(xs, p);
    // reference product for the bound check: the CSR sum in long double (a
    // validation checker on the downloaded matrix, not a compute path)
    const std::vector<double> want = host_reference(h, p, xs, L.n_rows);
    for (const mbx_simt_config& c : cfgs) {
      const std::string tag = std::string("(") + (p == MBX_F32 ? "f32" : "f64") +
                              ", omega=" + std::to_string(c.omega) +
                              ", sigma=" + std::to_string(c.sigma) + ") ";
      auto report = [&](bool pass, const std::string& what) {
        std::cout << (pass ? "[ok]   " : "[FAIL] ") << tag << what << '\n';
        ok = ok && pass;
      };
      Tile t;
      check(mbx_matrix_generate_tile(ctx, L.a.h, &c, &t.h));
      const TileHost th = download_tile(t.h);
      report(path_matches(th.info, c.offset_bits, th.tx.data(), th.ty.data(), th.ld.data(), h.ro,
                          L.n_rows, L.nnz),
             "path reconstruction matches sequential walk");
      bool rt = true;
      const uint32_t mask = (1u << c.offset_bits) - 1u;
      for (int64_t j = 0; j < th.info.lane_num; ++j) {
        const uint32_t w = th.ld[j];
        const uint32_t xo = w & mask, yo = (w >> c.offset_bits) & mask, fl = w >> (2 * c.offset_bits);
        rt = rt && (fl >> c.sigma) == 0 &&
             ((fl << (2 * c.offset_bits)) | (yo << c.offset_bits) | xo) == w;
      }
      report(rt, "lane descriptors round-trip");
      const auto got = multiply(ctx, L, t.h, c, p, x);
      report(within_bound(h, p, xs, want, got), "descriptor product within error bound");
    }
  }
  if (a.has("tile")) {
    const std::string tp = a.get("tile");
    mbx_tile_info info{};
    uint32_t *tx = nullptr, *ty = nullptr, *ld = nullptr;
    int prec = 0;
    check(mbx_tile_cache_read_host(tp.c_str(), &info, &tx, &ty, &ld, &prec));
    Loaded L;
    load(ctx, path, MBX_F64, L);
    const HostCsr h = download(L, 8);
    mbx_simt_config c{};
    check(mbx_config_make(info.omega, info.sigma, 4 * info.omega, &c));
    const bool pass = path_matches(info, c.offset_bits, tx, ty, ld, h.ro, L.n_rows, L.nnz);
    mbx_free(tx);
    mbx_free(ty);
    mbx_free(ld);
    std::cout << (pass ? "[ok]   " : "[FAIL] ") << "tile cache '" << tp
              << "' reproduces the merge path\n";
    ok = ok && pass;
  }
  std::cout << (ok ? "validation passed" : "validation FAILED") << " for " << dataset_id(path)
            << '\n';
  return ok ? 0 : kExitValidation;
}

int kind_of(const std::string& name) {
  if (name == "coo") return 1;
  if (name == "csr") return 0;
  if (name == "merge") return 2;
  if (name == "merge-cub") return 3;
  if (name == "merbit") return -1;
  throw config_error("unknown kernel id '" + name + "'");
}

std::vector<std::string> split(const std::string& s, char d) {
  std::vector<std::string> out;
  std::string cell;
  std::istringstream in(s);
  while (std::getline(in, cell, d))
    if (!cell.empty()) out.push_back(cell);
  return out;
}

struct Timed {
  double mean = 0.0, preprocess = 0.0, r_f = 0.0;
};

Timed time_kernel(mbx_context* ctx, Loaded& L, const mbx_simt_config& c, int kind, int iters,
                  int warmup, const std::vector<char>& x) {
  Timed out;
  Tile t;
  if (kind == -1) {
    check(mbx_matrix_generate_tile(ctx, L.a.h, &c, &t.h));
    double xc = 0.0;
    check(mbx_matrix_build_xcache(ctx, L.a.h, -1, &xc));
    mbx_tile_info info{};
    check(mbx_tile_get_info(t.h, &info));
    out.preprocess = info.preprocess_seconds + xc;
    const TileHost th = download_tile(t.h);
    out.r_f = long_row_fraction(th.info, th.ty);
  }
  check(mbx_bench_spmv(ctx, L.a.h, t.h, &c, kind, iters, warmup, x.data(), &out.mean));
  if (kind == -1) {
    int64_t slots = 0;
    double ss = 0.0;
    check(mbx_matrix_slot_info(L.a.h, &slots, &ss));
    out.preprocess += ss;  // the slot copy built by the first multiply
  }
  return out;
}

int cmd_bench(mbx_context* ctx, const Args& a) {
  if (a.pos.size() != 1) throw usage_error("bench needs exactly one matrix path");
  const std::string path = a.pos[0];
  const Kernel k = kernel_options(a);
  const int iters = int(a.integer("iters", 400)), warmup = int(a.integer("warmup", 10));
  if (iters < 1) throw config_error("--iters must be at least 1");
  const std::string format = a.get("format", "csv");
  if (format != "csv" && format != "json") throw usage_error("--format csv|json");
  const auto kernels = split(a.get("kernels", "coo,csr,merge,merbit"), ',');
  for (const auto& kn : kernels) kind_of(kn);
  const mbx_simt_config c = k.config();
  Loaded L;
  load(ctx, path, k.precision, L);
  const auto x = as_precision(seed_vector(L.n_cols, -1.0, 1.0, k.seed), k.precision);
  mbx_degree_stats degrees{};  // degree_stats(a, select_sigma(p)) (merbit_cli.cpp:270)
  check(mbx_matrix_degree_stats(ctx, L.a.h, mbx_select_sigma(k.precision, 0), &degrees));
  const bool low = degrees.low_degree != 0;
  // the COO baseline is always measured in-process (every speedup refers to it)
  const double coo = time_kernel(ctx, L, c, 1, iters, warmup, x).mean;
  std::vector<BenchRecord> rows;
  for (const auto& kn : kernels) {
    const int kind = kind_of(kn);
    const Timed t = kind == 1 ? Timed{coo, 0.0, 0.0} : time_kernel(ctx, L, c, kind, iters, warmup, x);
    BenchRecord r;
    r.dataset = dataset_id(path);
    r.kernel = kn;
    r.precision = k.pname();
    if (kind == -1 || kind == 2) {
      r.omega = c.omega;
      r.sigma = c.sigma;
      r.block_size = c.block_size;
    }
    r.iterations = iters;
    r.nnz = L.nnz;
    r.mean_seconds = t.mean;
    r.baseline_seconds = coo;
    r.ct = computational_throughput(L.nnz, t.mean);
    r.speedup = speedup(coo, t.mean);
    r.preprocess_seconds = t.preprocess;
    r.degree_group = low ? "G-L" : "G-H";
    if (kind == -1) {
      r.long_row_fraction = t.r_f;
      r.metadata_bytes = mbx_metadata_footprint(L.nnz, L.n_rows, &c, t.r_f);
      std::cerr << "note: merbit preprocessing cost = "
                << (t.mean > 0 ? t.preprocess / t.mean : 0.0)
                << "x one multiply (informational reference point: 1.29)\n";
    }
    rows.push_back(r);
  }
  Sink sink(a.get("out"));
  if (format == "json") {
    *sink.out << emit_json_array(rows) << '\n';
  } else {
    *sink.out << bench_csv_header() << '\n';
    for (const auto& r : rows) *sink.out << emit_csv(r) << '\n';
  }
  return 0;
}

std::vector<int> parse_sigmas(const std::string& text) {
  std::vector<int> out;
  for (const auto& tok : split(text, ',')) {
    const auto dash = tok.find('-', 1);
    try {
      if (dash == std::string::npos) {
        out.push_back(std::stoi(tok));
      } else {
        const int lo = std::stoi(tok.substr(0, dash)), hi = std::stoi(tok.substr(dash + 1));
        if (hi < lo) throw config_error("empty sigma range '" + tok + "'");
        for (int s = lo; s <= hi; ++s) out.push_back(s);
      }
    } catch (const std::logic_error&) {
      throw config_error("bad sigma list entry '" + tok + "'");
    }
  }
  if (out.empty()) throw config_error("empty sigma list");
  return out;
}

int cmd_sigma_sweep(mbx_context* ctx, const Args& a) {
  if (a.pos.size() != 1) throw usage_error("sigma-sweep needs exactly one matrix path");
  const std::string path = a.pos[0];
  const Kernel k = kernel_options(a);
  const int iters = int(a.integer("iters", 100)), warmup = int(a.integer("warmup", 5));
  if (iters < 1) throw config_error("--iters must be at least 1");
  const std::string format = a.get("format", "csv");
  Loaded L;
  load(ctx, path, k.precision, L);
  const HostCsr h = download(L, k.vs());
  const auto xs = seed_vector(L.n_cols, -1.0, 1.0, k.seed);
  const auto x = as_precision(xs, k.precision);
  const std::vector<double> want = host_reference(h, k.precision, xs, L.n_rows);
  mbx_simt_config c0 = k.config();
  const double coo = time_kernel(ctx, L, c0, 1, iters, warmup, x).mean;
  bool any = false, all_ok = true;
  std::ostringstream body;
  std::vector<std::string> json_rows;
  for (int s : parse_sigmas(a.get("sigmas", "4,7,14"))) {
    mbx_simt_config c{};
    const int rc = mbx_config_make(k.omega, s, k.block.value_or(4 * k.omega), &c);
    std::string note;
    bool feasible = rc == MBX_OK, validated = false;
    Timed t;
    double meta = 0.0, smem = 0.0;
    if (!feasible) {
      note = mbx_last_error();
      std::cerr << "sigma=" << s << " rejected: " << note << '\n';
    } else {
      any = true;
      Tile tt;
      check(mbx_matrix_generate_tile(ctx, L.a.h, &c, &tt.h));
      validated = within_bound(h, k.precision, xs, want, multiply(ctx, L, tt.h, c, k.precision, x));
      all_ok = all_ok && validated;
      t = time_kernel(ctx, L, c, -1, iters, warmup, x);
      meta = mbx_metadata_footprint(L.nnz, L.n_rows, &c, t.r_f);
      smem = double(c.block_size + 1) * c.sigma * double(k.vs());  // config.hpp:44-47
    }
    const double sp = feasible ? speedup(coo, t.mean) : 0.0;
    if (note.find_first_of(",\n") != std::string::npos) std::replace(note.begin(), note.end(), ',', ';');
    body << s << ',' << (feasible ? 1 : 0) << ',' << (validated ? 1 : 0) << ','
         << exact_double(sp) << ',' << exact_double(t.r_f) << ',' << exact_double(meta) << ','
         << exact_double(smem) << ',' << exact_double(t.mean) << ','
         << exact_double(t.preprocess) << ',' << note << '\n';
    std::ostringstream j;
    j << json_object({{"sigma", std::to_string(s)},
                      {"feasible", feasible ? "true" : "false"},
                      {"validated", validated ? "true" : "false"},
                      {"speedup_vs_coo", json_double(sp)},
                      {"r_f", json_double(t.r_f)},
                      {"metadata_bytes", json_double(meta)},
                      {"smem_bytes", json_double(smem)},
                      {"mean_seconds", json_double(t.mean)},
                      {"preprocess_seconds", json_double(t.preprocess)},
                      {"note", json_string(note)}},
                     "  ");
    json_rows.push_back(j.str());
  }
  Sink sink(a.get("out"));
  if (format == "json") {
    *sink.out << "[\n";
    for (size_t i = 0; i < json_rows.size(); ++i)
      *sink.out << json_rows[i] << (i + 1 < json_rows.size() ? ",\n" : "\n");
    *sink.out << "]\n";
  } else {
    *sink.out << "sigma,feasible,validated,speedup_vs_coo,r_f,metadata_bytes,smem_bytes,"
                 "mean_seconds,preprocess_seconds,note\n"
              << body.str();
  }
  if (!any) throw config_error("no feasible sigma in the sweep");
  return all_ok ? 0 : kExitValidation;
}

const char* status_name(int s) {
  return s == 0 ? "converged" : s == 1 ? "max_iterations" : "breakdown";
}

int cmd_pagerank(mbx_context* ctx, const Args& a) {
  if (a.pos.size() != 1) throw usage_error("pagerank needs exactly one adjacency path");
  const std::string path = a.pos[0];
  const Kernel k = kernel_options(a);
  const std::string backend = a.get("backend", "merbit");
  if (backend != "merbit") throw config_error("unknown kernel id '" + backend + "'");
  const mbx_simt_config c = k.config();
  Loaded L;
  load(ctx, path, k.precision, L);
  Matrix P;
  check(mbx_matrix_build_transition(ctx, L.a.h, &P.h));  // build_transition on the GPU
  Tile t;
  check(mbx_matrix_generate_tile(ctx, P.h, &c, &t.h));
  double xc = 0.0;
  check(mbx_matrix_build_xcache(ctx, P.h, -1, &xc));
  mbx_pagerank_config cfg{a.num("damping", 0.85), a.num("err-tol", 1e-10),
                          a.integer("max-iters", 210), a.integer("reference-iters", 210)};
  std::vector<char> pi(std::max<int64_t>(L.n_rows, 1) * k.vs());
  mbx_pagerank_result r{};
  check(mbx_pagerank(ctx, P.h, t.h, &c, &cfg, nullptr, pi.data(), nullptr, nullptr, &r));
  Sink sink(a.get("out"));
  *sink.out << json_object({{"workload", json_string("pagerank")},
                            {"dataset", json_string(dataset_id(path))},
                            {"backend", json_string("merbit-b200")},
                            {"precision", json_string(k.pname())},
                            {"vertices", std::to_string(L.n_rows)},
                            {"edges", std::to_string(L.nnz)},
                            {"iterations", std::to_string(r.iterations)},
                            {"final_err", json_double(r.final_err)},
                            {"status", json_string(status_name(r.status))},
                            {"preprocess_seconds", json_double(r.preprocess_seconds + xc)},
                            {"iterate_seconds", json_double(r.iterate_seconds)},
                            {"l1_residual", json_double(r.l1_residual)},
                            {"mass", json_double(r.mass)}})
            << '\n';
  return 0;
}

int cmd_bicgstab(mbx_context* ctx, const Args& a) {
  if (a.pos.size() != 1) throw usage_error("bicgstab needs exactly one matrix path");
  const std::string path = a.pos[0];
  const Kernel k = kernel_options(a);
  const mbx_simt_config c = k.config();
  Loaded L;
  load(ctx, path, k.precision, L);
  Tile t;
  check(mbx_matrix_generate_tile(ctx, L.a.h, &c, &t.h));
  const auto b = as_precision(seed_vector(L.n_rows, -1.0, 1.0, k.seed), k.precision);
  mbx_bicgstab_config cfg{a.num("tol", 1e-10), a.integer("max-iters", 20000)};
  std::vector<char> x(std::max<int64_t>(L.n_rows, 1) * k.vs());
  mbx_bicgstab_result r{};
  check(mbx_bicgstab(ctx, L.a.h, t.h, &c, &cfg, b.data(), x.data(), nullptr, &r));
  Fields f = {{"workload", json_string("bicgstab")},
              {"dataset", json_string(dataset_id(path))},
              {"backend", json_string("merbit-b200")},
              {"precision", json_string(k.pname())},
              {"rows", std::to_string(L.n_rows)},
              {"nnz", std::to_string(L.nnz)},
              {"iterations", std::to_string(r.iterations)},
              {"final_residual", json_double(r.final_residual)},
              {"status", json_string(status_name(r.status))},
              {"preprocess_seconds", json_double(r.preprocess_seconds)},
              {"iterate_seconds", json_double(r.iterate_seconds)}};
  if (r.status == 2) f.emplace_back("breakdown", json_string(r.breakdown_reason));
  Sink sink(a.get("out"));
  *sink.out << json_object(f) << '\n';
  return r.status == 2 ? kExitBreakdown : 0;
}

int cmd_convert(mbx_context* ctx, const Args& a) {
  if (a.pos.size() != 1) throw usage_error("convert needs exactly one matrix path");
  if (!a.has("out")) throw usage_error("convert needs --out");
  const Kernel k = kernel_options(a);
  Loaded L;
  load(ctx, a.pos[0], MBX_F64, L);  // normalize_coo: sorted, duplicates summed in fp64
  const HostCsr h = download(L, 8);
  mbx_coo norm{};
  std::vector<int64_t> rows(std::max<int64_t>(L.nnz, 1)), cols(std::max<int64_t>(L.nnz, 1));
  for (int64_t r = 0; r < L.n_rows; ++r)
    for (int64_t q = h.ro[r]; q < h.ro[r + 1]; ++q) {
      rows[q] = r;
      cols[q] = h.cols[q];
    }
  norm.n_rows = L.n_rows;
  norm.n_cols = L.n_cols;
  norm.nnz = L.nnz;
  norm.rows = rows.data();
  norm.cols = cols.data();
  norm.vals = const_cast<double*>(reinterpret_cast<const double*>(h.vals.data()));
  check(mbx_matrix_cache_write(a.get("out").c_str(), &norm));
  std::cout << "wrote matrix cache " << a.get("out") << '\n';
  if (a.has("tile")) {
    Loaded Lp;
    load(ctx, a.pos[0], k.precision, Lp);
    const mbx_simt_config c = k.config();
    Tile t;
    check(mbx_matrix_generate_tile(ctx, Lp.a.h, &c, &t.h));
    check(mbx_tile_cache_write(t.h, a.get("tile").c_str(), k.precision));
    std::cout << "wrote tile cache " << a.get("tile") << '\n';
  }
  return 0;
}

// fixtures.hpp generators (host inputs for the other verbs)
int cmd_gen(const Args& a) {
  if (a.pos.size() != 1) throw usage_error("gen needs exactly one fixture name");
  if (!a.has("out")) throw usage_error("gen needs --out");
  const std::string f = a.pos[0];
  int64_t n_rows = 0, n_cols = 0;
  std::vector<std::tuple<int64_t, int64_t, double>> e;
  if (f == "walkthrough") {  // fixtures.hpp:17-36
    const int64_t ro[] = {0, 5, 5, 10, 13, 20, 26, 32, 34};
    const int64_t cols[] = {0, 2, 3, 5, 7, 1, 2, 4, 6, 7, 0, 3, 6, 0, 1, 2, 4,
                            5, 6, 7, 0, 1, 3, 4, 5, 7, 1, 2, 3, 4, 6, 7, 3, 5};
    n_rows = n_cols = 8;
    for (int64_t r = 0; r < 8; ++r)
      for (int64_t q = ro[r]; q < ro[r + 1]; ++q) e.emplace_back(r, cols[q], double(q + 1));
  } else if (f == "laplacian") {  // fixtures.hpp:40-56
    const int64_t g = a.integer("grid", 8);
    n_rows = n_cols = g * g;
    for (int64_t i = 0; i < g; ++i)
      for (int64_t j = 0; j < g; ++j) {
        const int64_t v = i * g + j;
        std::vector<std::pair<int64_t, double>> row = {{v, 4.0}};
        if (i > 0) row.emplace_back(v - g, -1.0);
        if (i + 1 < g) row.emplace_back(v + g, -1.0);
        if (j > 0) row.emplace_back(v - 1, -1.0);
        if (j + 1 < g) row.emplace_back(v + 1, -1.0);
        std::sort(row.begin(), row.end());
        for (auto& [c, w] : row) e.emplace_back(v, c, w);
      }
  } else if (f == "ring") {  // fixtures.hpp:58-78
    const int64_t n = a.integer("nodes", 100), chords = a.integer("chords", 260);
    n_rows = n_cols = n;
    std::vector<std::pair<int64_t, int64_t>> ed;
    for (int64_t i = 0; i < n; ++i) ed.emplace_back(i, (i + 1) % n);
    std::mt19937_64 rng(uint64_t(a.integer("seed", 42)));
    for (int64_t k = 0; k < chords; ++k) {
      const int64_t from = int64_t(rng() % uint64_t(n)), to = int64_t(rng() % uint64_t(n));
      if (from != to) ed.emplace_back(from, to);
    }
    // coo_to_csr: row-major order, duplicate chords merged by summing values
    std::stable_sort(ed.begin(), ed.end());
    for (size_t k = 0; k < ed.size(); ++k) {
      if (k > 0 && ed[k] == ed[k - 1])
        std::get<2>(e.back()) += 1.0;
      else
        e.emplace_back(ed[k].first, ed[k].second, 1.0);
    }
  } else if (f == "dense-row") {  // fixtures.hpp:93-110
    const int64_t w = a.integer("width", 64);
    n_rows = 1;
    n_cols = w;
    const auto v = seed_vector(w, 0.5, 1.5, uint64_t(a.integer("seed", 1)));
    for (int64_t c = 0; c < w; ++c) e.emplace_back(0, c, v[c]);
  } else if (f == "singular") {  // fixtures.hpp:83-91
    n_rows = n_cols = 2;
    e.emplace_back(0, 0, 1.0);
  } else {
    throw config_error("unknown fixture '" + f + "'");
  }
  std::vector<int64_t> rows, cols;
  std::vector<double> vals;
  for (auto& [r, c, v] : e) {
    rows.push_back(r);
    cols.push_back(c);
    vals.push_back(v);
  }
  mbx_coo coo{n_rows, n_cols, int64_t(e.size()), rows.data(), cols.data(), vals.data()};
  check(mbx_mm_write(a.get("out").c_str(), &coo));
  std::cout << "wrote " << n_rows << "x" << n_cols << " matrix (" << e.size()
            << " nonzeros) to " << a.get("out") << '\n';
  return 0;
}

void usage() {
  std::cerr << "usage: merbit_b200 <validate|bench|sigma-sweep|pagerank|bicgstab|convert|gen> "
               "[args] [--options]\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    usage();
    return argc < 2 ? kExitUsage : 0;
  }
  const std::string verb = argv[1];
  try {
    const Args a = parse_args(argc, argv, 2);
    for (const char* k : {"iters", "warmup", "damping", "err-tol", "max-iters", "reference-iters",
                          "tol", "grid", "nodes", "chords", "width", "seed", "omega", "sigma",
                          "block-size", "device"})
      a.num(k, 0.0);  // malformed numbers are usage errors, before any device work
    if (verb == "gen") return cmd_gen(a);
    static const char* kVerbs[] = {"validate", "bench", "sigma-sweep", "pagerank", "bicgstab",
                                   "convert"};
    if (std::find_if(std::begin(kVerbs), std::end(kVerbs),
                     [&](const char* v) { return verb == v; }) == std::end(kVerbs)) {
      usage();
      return kExitUsage;
    }
    if (a.pos.size() != 1) throw usage_error(verb + " needs exactly one matrix path");
    kernel_options(a);  // option errors before any device work
    const int device = int(a.integer("device", 0));
    Context ctx(device);
    if (verb == "validate") return cmd_validate(ctx.get(), a);
    if (verb == "bench") return cmd_bench(ctx.get(), a);
    if (verb == "sigma-sweep") return cmd_sigma_sweep(ctx.get(), a);
    if (verb == "pagerank") return cmd_pagerank(ctx.get(), a);
    if (verb == "bicgstab") return cmd_bicgstab(ctx.get(), a);
    if (verb == "convert") return cmd_convert(ctx.get(), a);
    usage();
    return kExitUsage;
  } catch (const usage_error& e) {
    std::cerr << "usage error: " << e.what() << '\n';
    return kExitUsage;
  } catch (const io_error& e) {
    std::cerr << "input error: " << e.what() << '\n';
    return kExitInput;
  } catch (const parse_error& e) {
    std::cerr << "input error: " << e.what() << '\n';
    return kExitInput;
  } catch (const corruption_error& e) {
    std::cerr << "input error: " << e.what() << '\n';
    return kExitInput;
  } catch (const dimension_error& e) {
    std::cerr << "input error: " << e.what() << '\n';
    return kExitInput;
  } catch (const capacity_error& e) {
    std::cerr << "configuration error: " << e.what() << '\n';
    return kExitConfig;
  } catch (const config_error& e) {
    std::cerr << "configuration error: " << e.what() << '\n';
    return kExitConfig;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
