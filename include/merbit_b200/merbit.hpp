// merbit_b200/merbit.hpp -- C++ mirror of the reference API for the MERBIT
// hot path, header-only over the C ABI (merbit_b200.h, libmerbit_b200.so).
//
// Names, argument meaning and error behaviour follow
// /root/reference/proj/include/merbit:
//   SimtConfig::make, select_sigma            config.hpp:18-42, src/config.cpp:12-43
//   TileMetadata, generate_tile                tile.hpp:27-58, src/tile.cpp:17-85
//   DualBuffer                                 dual_buffer.hpp:19-42
//   spmv_merbit(.., DualBuffer&, .., trace)    merbit_spmv.hpp:136-352
//   SpmvBackend, MerbitB200Backend, make_backend   backend.hpp:22-34, 112-169
//   PageRankConfig, PageRankResult, pagerank   solvers.hpp:76-218
// and the exception taxonomy of types.hpp:23-65 (status codes are mapped
// back to the same exception classes, so CHECK_THROWS_AS-style tests and the
// CLI's exit-code mapping keep working).
//
// Differences, by design: the matrix lives on the device (DeviceCsr, made
// once from a host CsrMatrix-like triple of vectors); apply() returns a host
// vector that stays valid until the next apply(), exactly the reference's
// lifetime rule (backend.hpp:17-21).  The PageRank power loop runs fused on
// the device; on_iteration, when set, copies each iterate to the host
// (mbx_pagerank_observed).
#pragma once

#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "merbit_b200.h"

namespace merbit_b200 {

using index_t = std::int64_t;  // types.hpp:13

class error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class io_error : public error {
 public:
  using error::error;
};
class parse_error : public error {
 public:
  using error::error;
};
class config_error : public error {
 public:
  using error::error;
};
class dimension_error : public error {
 public:
  using error::error;
};
class capacity_error : public error {
 public:
  using error::error;
};
class corruption_error : public error {
 public:
  using error::error;
};
class device_error : public error {
 public:
  using error::error;
};

inline void check(int rc) {
  if (rc == MBX_OK) return;
  const std::string msg = mbx_last_error();
  switch (rc) {
    case MBX_IO_ERROR: throw io_error(msg);
    case MBX_PARSE_ERROR: throw parse_error(msg);
    case MBX_CONFIG_ERROR: throw config_error(msg);
    case MBX_DIMENSION_ERROR: throw dimension_error(msg);
    case MBX_CAPACITY_ERROR: throw capacity_error(msg);
    case MBX_CORRUPTION_ERROR: throw corruption_error(msg);
    case MBX_CUDA_ERROR:
    case MBX_NCCL_ERROR:
    case MBX_UNSUPPORTED: throw device_error(msg);
    default: throw error(msg);
  }
}

enum class ScalarPrecision { f32, f64 };

template <typename T>
constexpr int precision_of() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "f32 or f64");
  return std::is_same_v<T, float> ? MBX_F32 : MBX_F64;
}

// ---- SimtConfig (config.hpp:18-38) ----------------------------------------
struct SimtConfig {
  int omega = 32;
  int sigma = 14;
  int block_size = 128;
  int offset_bits = 9;

  static SimtConfig make(int omega, int sigma, int block_size) {
    mbx_simt_config c{};
    check(mbx_config_make(omega, sigma, block_size, &c));
    return SimtConfig{c.omega, c.sigma, c.block_size, c.offset_bits};
  }
  int warps_per_block() const { return block_size / omega; }
  index_t steps_per_lane() const { return sigma; }
  index_t steps_per_tile() const { return index_t(omega) * sigma; }
  index_t steps_per_block() const { return index_t(block_size) * sigma; }
  mbx_simt_config c() const { return mbx_simt_config{omega, sigma, block_size, offset_bits}; }
  friend bool operator==(const SimtConfig&, const SimtConfig&) = default;
};

inline int select_sigma(ScalarPrecision p, std::optional<int> override = {}) {
  return mbx_select_sigma(p == ScalarPrecision::f64 ? MBX_F64 : MBX_F32,
                          override.value_or(0));
}

// ---- device context --------------------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) {
    mbx_context* c = nullptr;
    check(mbx_context_create(device, &c));
    h_.reset(c);
  }
  mbx_context* get() const { return h_.get(); }
  void synchronize() const { check(mbx_context_synchronize(h_.get())); }

 private:
  struct Del {
    void operator()(mbx_context* c) const { mbx_context_destroy(c); }
  };
  std::unique_ptr<mbx_context, Del> h_;
};

// ---- device-resident CsrMatrix<T> (csr.hpp:29-38) -----------------------------
template <typename T>
class DeviceCsr {
 public:
  DeviceCsr(Context& ctx, index_t n_rows, index_t n_cols, const std::vector<index_t>& row_offsets,
            const std::vector<index_t>& col_indices, const std::vector<T>& values)
      : ctx_(&ctx), n_rows_(n_rows), n_cols_(n_cols) {
    mbx_matrix* m = nullptr;
    check(mbx_matrix_upload(ctx.get(), precision_of<T>(), n_rows, n_cols, row_offsets.data(),
                            col_indices.data(), values.data(), &m));
    h_.reset(m);
    nnz_ = row_offsets.empty() ? 0 : row_offsets.back();
  }
  // Any type with the reference CsrMatrix<T> fields (n_rows, n_cols,
  // row_offsets, col_indices, values), e.g. merbit::CsrMatrix<T> itself.
  template <typename Csr>
  static DeviceCsr from(Context& ctx, const Csr& a) {
    return DeviceCsr(ctx, a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values);
  }
  mbx_matrix* get() const { return h_.get(); }
  // x hub cache (mbx_matrix_build_xcache); returns its device seconds.
  double build_xcache(int max_hubs = -1) {
    double s = 0.0;
    check(mbx_matrix_build_xcache(ctx_->get(), h_.get(), max_hubs, &s));
    return s;
  }
  index_t n_rows() const { return n_rows_; }
  index_t n_cols() const { return n_cols_; }
  index_t nnz() const { return nnz_; }
  Context& context() const { return *ctx_; }

 private:
  struct Del {
    void operator()(mbx_matrix* m) const { mbx_matrix_destroy(m); }
  };
  Context* ctx_;
  index_t n_rows_, n_cols_, nnz_ = 0;
  std::unique_ptr<mbx_matrix, Del> h_;
};

// ---- DegreeStats (csr.hpp:108-140), reduced on the device --------------------
struct DegreeStats {
  double mean_degree = 0.0;
  bool low_degree = false;
  index_t max_degree = 0;
  index_t empty_rows = 0;
};

template <typename T>
DegreeStats degree_stats(const DeviceCsr<T>& a, int sigma_threshold) {
  mbx_degree_stats d{};
  check(mbx_matrix_degree_stats(a.context().get(), a.get(), sigma_threshold, &d));
  return DegreeStats{d.mean_degree, d.low_degree != 0, d.max_degree, d.empty_rows};
}

// ---- TileMetadata (tile.hpp:27-44) -------------------------------------------
struct TileMetadata {
  int omega = 0;
  int sigma = 0;
  index_t n_rows = 0;
  index_t nnz = 0;
  index_t tile_num = 0;
  index_t lane_num = 0;
  std::vector<std::uint32_t> tile_x;
  std::vector<std::uint32_t> tile_y;
  std::vector<std::uint32_t> lane_desc;

  static constexpr std::uint32_t kLongRowMask = 0x80000000u;
  static std::uint32_t row_of(std::uint32_t v) { return v & ~kLongRowMask; }
  static bool is_marked(std::uint32_t v) { return (v & kLongRowMask) != 0; }
  index_t lane_steps(index_t j) const {
    const index_t total = nnz + n_rows;
    return std::min<index_t>(sigma, total - j * sigma);
  }
};

// Device-resident TILE handle.
class DeviceTile {
 public:
  DeviceTile(mbx_tile* t) : h_(t) { check(mbx_tile_get_info(t, &info_)); }
  mbx_tile* get() const { return h_.get(); }
  const mbx_tile_info& info() const { return info_; }
  double preprocess_seconds() const { return info_.preprocess_seconds; }
  TileMetadata download() const {
    TileMetadata t;
    t.omega = info_.omega;
    t.sigma = info_.sigma;
    t.n_rows = info_.n_rows;
    t.nnz = info_.nnz;
    t.tile_num = info_.tile_num;
    t.lane_num = info_.lane_num;
    t.tile_x.resize(t.tile_num + 1);
    t.tile_y.resize(t.tile_num + 1);
    t.lane_desc.resize(t.lane_num);
    check(mbx_tile_download(h_.get(), t.tile_x.data(), t.tile_y.data(), t.lane_desc.data()));
    return t;
  }

 private:
  struct Del {
    void operator()(mbx_tile* t) const { mbx_tile_destroy(t); }
  };
  std::unique_ptr<mbx_tile, Del> h_;
  mbx_tile_info info_{};
};

// generate_tile(span row_offsets, n_rows, nnz, c) (tile.hpp:51-53), on the GPU;
// arrays byte-identical to the reference.
inline TileMetadata generate_tile(Context& ctx, std::span<const index_t> row_offsets,
                                  index_t n_rows, index_t nnz, const SimtConfig& c) {
  mbx_tile* t = nullptr;
  const mbx_simt_config cc = c.c();
  check(mbx_generate_tile(ctx.get(), row_offsets.empty() ? nullptr : row_offsets.data(), n_rows,
                          nnz, &cc, &t));
  return DeviceTile(t).download();
}

template <typename T>
DeviceTile generate_tile(const DeviceCsr<T>& a, const SimtConfig& c) {
  mbx_tile* t = nullptr;
  const mbx_simt_config cc = c.c();
  check(mbx_matrix_generate_tile(a.context().get(), a.get(), &cc, &t));
  return DeviceTile(t);
}

// ---- DualBuffer (dual_buffer.hpp:19-42) --------------------------------------
template <typename T>
class DualBuffer {
 public:
  explicit DualBuffer(index_t n)
      : bufs_{std::vector<T>(static_cast<std::size_t>(n), T(0)),
              std::vector<T>(static_cast<std::size_t>(n), T(0))} {}
  index_t size() const { return static_cast<index_t>(bufs_[0].size()); }
  int parity() const { return parity_; }
  std::vector<T>& active() { return bufs_[parity_]; }
  std::vector<T>& inactive() { return bufs_[parity_ ^ 1]; }
  const std::vector<T>& last_output() const { return bufs_[parity_ ^ 1]; }
  void flip() { parity_ ^= 1; }

 private:
  std::vector<T> bufs_[2];
  int parity_ = 0;
};

// merbit_spmv.hpp:21-28: routing counters and, with collect_deposits, the
// (row, partial) contributions of the decomposition (mbx_spmv_deposits;
// unordered, rows in the caller's vertex order)
template <typename T = double>
struct SpmvTraceT {
  bool collect_deposits = false;
  std::int64_t fast_tiles = 0, normal_tiles = 0, skipped_tiles = 0;
  std::vector<std::pair<index_t, T>> deposits;
};
using SpmvTrace = SpmvTraceT<double>;

// spmv_merbit (merbit_spmv.hpp:136-352): out.active() = A x on the GPU,
// companion zeroed, parity flipped.
template <typename T, typename TT = double>
void spmv_merbit(const DeviceCsr<T>& a, const DeviceTile& t, const SimtConfig& c,
                 std::span<const T> x, DualBuffer<T>& out, SpmvTraceT<TT>* trace = nullptr) {
  if (static_cast<index_t>(x.size()) != a.n_cols())
    throw dimension_error("spmv: x has " + std::to_string(x.size()) + " entries, matrix has " +
                          std::to_string(a.n_cols()) + " columns");
  if (out.size() != a.n_rows())
    throw dimension_error("spmv: output pair sized " + std::to_string(out.size()) + " for " +
                          std::to_string(a.n_rows()) + " rows");
  const mbx_simt_config cc = c.c();
  mbx_spmv_trace tr{};
  check(mbx_spmv(a.context().get(), a.get(), t.get(), &cc, x.data(), out.active().data(),
                 trace ? &tr : nullptr));
  std::fill(out.inactive().begin(), out.inactive().end(), T(0));
  out.flip();
  if (trace) {
    trace->fast_tiles += tr.fast_tiles;
    trace->normal_tiles += tr.normal_tiles;
    trace->skipped_tiles += tr.skipped_tiles;
    if (trace->collect_deposits) {
      std::int64_t cap = 0, got = 0;
      check(mbx_spmv_deposits(a.context().get(), a.get(), t.get(), &cc, nullptr, nullptr,
                              nullptr, 0, &cap));
      std::vector<std::int64_t> rows(static_cast<std::size_t>(cap > 0 ? cap : 1));
      std::vector<T> amounts(rows.size());
      check(mbx_spmv_deposits(a.context().get(), a.get(), t.get(), &cc, x.data(), rows.data(),
                              amounts.data(), cap, &got));
      for (std::int64_t k = 0; k < got && k < cap; ++k)
        trace->deposits.emplace_back(static_cast<index_t>(rows[static_cast<std::size_t>(k)]),
                                     static_cast<TT>(amounts[static_cast<std::size_t>(k)]));
    }
  }
}

// ---- backends (backend.hpp:22-169) --------------------------------------------
template <typename T>
class SpmvBackend {
 public:
  virtual ~SpmvBackend() = default;
  virtual const std::vector<T>& apply(std::span<const T> x) = 0;
  virtual std::string name() const = 0;
  double preprocess_seconds() const { return preprocess_seconds_; }

 protected:
  double preprocess_seconds_ = 0.0;
};

// MerbitBackend (backend.hpp:112-136) on the GPU: uploads the matrix and
// builds the TILE and the x hub cache once (T_p = their device time).
template <typename T>
class MerbitB200Backend final : public SpmvBackend<T> {
 public:
  template <typename Csr>
  MerbitB200Backend(Context& ctx, const Csr& a, const SimtConfig& c)
      : config_(c), matrix_(DeviceCsr<T>::from(ctx, a)), tile_(generate_tile(matrix_, c)),
        buffer_(a.n_rows) {
    this->preprocess_seconds_ = tile_.preprocess_seconds() + matrix_.build_xcache();
  }
  const std::vector<T>& apply(std::span<const T> x) override {
    spmv_merbit(matrix_, tile_, config_, x, buffer_);
    return buffer_.last_output();
  }
  std::string name() const override { return "merbit-b200"; }
  const DeviceTile& tile() const { return tile_; }
  const DeviceCsr<T>& matrix() const { return matrix_; }
  const SimtConfig& config() const { return config_; }

 private:
  SimtConfig config_;
  DeviceCsr<T> matrix_;
  DeviceTile tile_;
  DualBuffer<T> buffer_;
};

enum class BackendKind { merbit_b200 };

template <typename T, typename Csr>
std::unique_ptr<SpmvBackend<T>> make_backend(BackendKind kind, Context& ctx, const Csr& a,
                                             const SimtConfig& c) {
  switch (kind) {
    case BackendKind::merbit_b200: return std::make_unique<MerbitB200Backend<T>>(ctx, a, c);
  }
  throw config_error("unknown backend kind");
}

// ---- PageRank (solvers.hpp:76-218) --------------------------------------------
enum class SolveStatus { converged, max_iterations, breakdown };

template <typename T>
struct PageRankConfig {
  T damping = T(0.85);
  T err_tol = T(1e-10);
  index_t max_iters = 210;
  index_t reference_iters = 210;
};

template <typename T>
struct PageRankResult {
  std::vector<T> pi;
  std::vector<T> reference_pi;
  index_t iterations = 0;
  double final_err = std::numeric_limits<double>::infinity();
  SolveStatus status = SolveStatus::max_iterations;
  double preprocess_seconds = 0.0;
  double iterate_seconds = 0.0;
  double l1_residual = 0.0;  // ||pi_k - pi_{k-1}||_1, fused on the device
};

// pagerank<T>(p, cfg, backend, on_iteration): yardstick, damping/teleport
// update, dangling redistribution, mass check, ERR and early exit -- all fused
// into the SpMV commit on the device; pi reaches the host once, at the end,
// or after every iteration when on_iteration is set (solvers.hpp:157-158,
// 209: called after the mass check, before the convergence test).
template <typename T>
PageRankResult<T> pagerank(
    MerbitB200Backend<T>& backend, const PageRankConfig<T>& cfg,
    std::vector<double>* residual_history = nullptr,
    const std::function<void(index_t, const std::vector<T>&, double)>& on_iteration = {}) {
  const auto& a = backend.matrix();
  if (a.n_rows() != a.n_cols()) throw dimension_error("pagerank needs a square transition matrix");
  const mbx_simt_config cc = backend.config().c();
  PageRankResult<T> r;
  r.pi.resize(a.n_rows());
  r.reference_pi.resize(a.n_rows());
  mbx_pagerank_result res{};
  const mbx_pagerank_config pc{double(cfg.damping), double(cfg.err_tol), cfg.max_iters,
                               cfg.reference_iters};
  if (residual_history) residual_history->assign(std::max<index_t>(cfg.max_iters, 1), 0.0);
  if (!on_iteration) {
    check(mbx_pagerank(a.context().get(), a.get(), backend.tile().get(), &cc, &pc, nullptr,
                       r.pi.data(), r.reference_pi.data(),
                       residual_history ? residual_history->data() : nullptr, &res));
  } else {
    struct Obs {
      const std::function<void(index_t, const std::vector<T>&, double)>* fn;
      std::vector<T> it;
      std::exception_ptr failure;
    } obs{&on_iteration, std::vector<T>(a.n_rows()), nullptr};
    auto tramp = [](int64_t iter, const void* pi, double err, void* user) -> int {
      auto* o = static_cast<Obs*>(user);
      try {
        std::memcpy(o->it.data(), pi, o->it.size() * sizeof(T));
        (*o->fn)(index_t(iter), o->it, err);
        return 0;
      } catch (...) {  // stops the run; rethrown once the C call has returned
        o->failure = std::current_exception();
        return 1;
      }
    };
    const int rc = mbx_pagerank_observed(
        a.context().get(), a.get(), backend.tile().get(), &cc, &pc, nullptr, r.pi.data(),
        r.reference_pi.data(), residual_history ? residual_history->data() : nullptr, tramp, &obs,
        &res);
    if (obs.failure) std::rethrow_exception(obs.failure);
    check(rc);
  }
  if (residual_history) residual_history->resize(res.iterations);
  r.iterations = res.iterations;
  r.final_err = res.final_err;
  r.status = res.status == 0 ? SolveStatus::converged : SolveStatus::max_iterations;
  r.preprocess_seconds = backend.preprocess_seconds();
  r.iterate_seconds = res.iterate_seconds;
  r.l1_residual = res.l1_residual;
  return r;
}

// ---- BiCGSTAB (solvers.hpp:224-373) -------------------------------------------
template <typename T>
struct BicgstabConfig {
  T tol = T(1e-10);  // on ||A*x - b|| / ||b||, recomputed each pass
  index_t max_iters = 20000;
};

template <typename T>
struct BicgstabResult {
  std::vector<T> x;
  std::vector<double> residual_history;  // true relative residual per pass
  index_t iterations = 0;
  double final_residual = std::numeric_limits<double>::infinity();
  SolveStatus status = SolveStatus::max_iterations;
  std::string breakdown_reason;
  double preprocess_seconds = 0.0;
  double iterate_seconds = 0.0;
};

inline const char* solve_status_name(SolveStatus s) {
  switch (s) {
    case SolveStatus::converged: return "converged";
    case SolveStatus::max_iterations: return "max_iterations";
    case SolveStatus::breakdown: return "breakdown";
  }
  return "unknown";
}

// bicgstab<T>(a, b, cfg, backend): every SpMV, inner product and vector
// update runs on the device (mbx_bicgstab); x reaches the host once.
template <typename T>
BicgstabResult<T> bicgstab(MerbitB200Backend<T>& backend, std::span<const T> b,
                           const BicgstabConfig<T>& cfg = {}) {
  const auto& a = backend.matrix();
  if (a.n_rows() != a.n_cols()) throw dimension_error("bicgstab needs a square system");
  if (static_cast<index_t>(b.size()) != a.n_rows())
    throw dimension_error("bicgstab: right-hand side has " + std::to_string(b.size()) +
                          " entries for " + std::to_string(a.n_rows()) + " rows");
  const mbx_simt_config cc = backend.config().c();
  BicgstabResult<T> r;
  r.x.resize(a.n_rows());
  r.residual_history.assign(std::max<index_t>(cfg.max_iters, 1), 0.0);
  const mbx_bicgstab_config bc{double(cfg.tol), cfg.max_iters};
  mbx_bicgstab_result res{};
  check(mbx_bicgstab(a.context().get(), a.get(), backend.tile().get(), &cc, &bc, b.data(),
                     r.x.data(), r.residual_history.data(), &res));
  r.iterations = res.iterations;
  r.final_residual = res.final_residual;
  r.status = res.status == 0   ? SolveStatus::converged
             : res.status == 1 ? SolveStatus::max_iterations
                               : SolveStatus::breakdown;
  r.breakdown_reason = res.breakdown_reason;
  const bool early = r.status == SolveStatus::breakdown && r.breakdown_reason != "diverged";
  r.residual_history.resize(r.iterations - (early ? 1 : 0));
  r.preprocess_seconds = backend.preprocess_seconds();
  r.iterate_seconds = res.iterate_seconds;
  return r;
}

}  // namespace merbit_b200
