// ref_shim.cpp -- a C ABI over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources where they lie (/root/reference/proj/src/*.cpp, headers
// from /root/reference/proj/include and tests/support) into
// oracle/_ref/libmerbit_ref.so.  Nothing here re-implements reference logic:
// every entry point converts plain arrays into the reference's own types and
// calls the reference function named beside it.  Used to pin the C
// restatement (oracle/merbit_oracle.c), to write tests/golden/, and as the
// CPU arm of bench.py (--impl reference and the cpu_baseline field).
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "merbit/backend.hpp"
#include "merbit/config.hpp"
#include "merbit/fixtures.hpp"
#include "merbit/merbit_spmv.hpp"
#include "merbit/matrix_market.hpp"
#include "merbit/merge_path.hpp"
#include "merbit/merge_spmv.hpp"
#include "merbit/random.hpp"
#include "merbit/reference.hpp"
#include "merbit/solvers.hpp"
#include "merbit/tile.hpp"
#include "support/generators.hpp"

using namespace merbit;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const config_error& e) {
    g_err = e.what();
    return 4;
  } catch (const dimension_error& e) {
    g_err = e.what();
    return 5;
  } catch (const capacity_error& e) {
    g_err = e.what();
    return 6;
  } catch (const corruption_error& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename T>
CsrMatrix<T> make_csr(int64_t n_rows, int64_t n_cols, const int64_t* ro,
                      const int32_t* cols, const T* vals) {
  CsrMatrix<T> a;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.row_offsets.assign(ro, ro + n_rows + 1);
  const int64_t nnz = ro[n_rows];
  a.col_indices.resize(static_cast<std::size_t>(nnz));
  for (int64_t k = 0; k < nnz; ++k) a.col_indices[k] = cols[k];
  a.values.assign(vals, vals + nnz);
  return a;
}

void export_csr(const CsrMatrix<double>& a, int64_t* n_rows, int64_t* n_cols,
                int64_t* nnz, int64_t** ro, int32_t** cols, double** vals) {
  *n_rows = a.n_rows;
  *n_cols = a.n_cols;
  *nnz = a.nnz();
  *ro = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (a.n_rows + 1)));
  *cols = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (a.nnz() + 1)));
  *vals = static_cast<double*>(std::malloc(sizeof(double) * (a.nnz() + 1)));
  std::memcpy(*ro, a.row_offsets.data(), sizeof(int64_t) * (a.n_rows + 1));
  for (int64_t k = 0; k < a.nnz(); ++k) {
    (*cols)[k] = static_cast<int32_t>(a.col_indices[k]);
    (*vals)[k] = a.values[k];
  }
}

// Persistent CPU engine for timing: owns the matrix, the pool and a
// MerbitBackend (backend.hpp:112-136), exactly as the reference CLI builds
// them (merbit_cli.cpp:268-286).
template <typename T>
struct RefEngine {
  CsrMatrix<T> a;
  SimtConfig c;
  std::unique_ptr<ThreadPool> pool;
  std::unique_ptr<SpmvBackend<T>> backend;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_config_make(int omega, int sigma, int block, int* offset_bits) {
  return guarded([&] {
    *offset_bits = SimtConfig::make(omega, sigma, block).offset_bits;
  });
}

int ref_select_sigma(int precision, int override_sigma) {
  const ScalarPrecision p = precision == 1 ? ScalarPrecision::f64 : ScalarPrecision::f32;
  return override_sigma > 0 ? select_sigma(p, override_sigma) : select_sigma(p);
}

int ref_merge_search(const int64_t* ro, int64_t n_rows, int64_t nnz,
                     int64_t diag, int64_t* x, int64_t* y, int* probes) {
  return guarded([&] {
    const PathCoord c = merge_search(
        std::span<const index_t>(ro, static_cast<std::size_t>(n_rows + 1)),
        diag, n_rows, nnz, probes);
    *x = c.x;
    *y = c.y;
  });
}

int ref_generate_tile(const int64_t* ro, int64_t n_rows, int64_t nnz,
                      int omega, int sigma, int block, uint32_t* tile_x,
                      uint32_t* tile_y, uint32_t* lane_desc,
                      double* seconds) {
  return guarded([&] {
    const SimtConfig c = SimtConfig::make(omega, sigma, block);
    const auto t0 = std::chrono::steady_clock::now();
    const TileMetadata t = generate_tile(
        std::span<const index_t>(ro, ro ? static_cast<std::size_t>(n_rows + 1) : 0),
        n_rows, nnz, c);
    if (seconds) *seconds = detail::seconds_since(t0);
    std::memcpy(tile_x, t.tile_x.data(), 4 * t.tile_x.size());
    std::memcpy(tile_y, t.tile_y.data(), 4 * t.tile_y.size());
    if (!t.lane_desc.empty())
      std::memcpy(lane_desc, t.lane_desc.data(), 4 * t.lane_desc.size());
  });
}

#define REF_SPMV(T, SUFFIX)                                                   \
  int ref_spmv_merbit_##SUFFIX(int64_t n_rows, int64_t n_cols,                \
                               const int64_t* ro, const int32_t* cols,        \
                               const T* vals, const T* x, int omega,          \
                               int sigma, int block, int nthreads, T* y,      \
                               int64_t* counters) {                           \
    return guarded([&] {                                                      \
      const SimtConfig c = SimtConfig::make(omega, sigma, block);             \
      const CsrMatrix<T> a = make_csr<T>(n_rows, n_cols, ro, cols, vals);     \
      const TileMetadata t = generate_tile(a, c);                             \
      DualBuffer<T> buf(a.n_rows);                                            \
      std::unique_ptr<ThreadPool> pool;                                       \
      if (nthreads > 1) pool = std::make_unique<ThreadPool>(nthreads);        \
      SpmvTrace<T> trace;                                                     \
      spmv_merbit(a, t, c, std::span<const T>(x, n_cols), buf, pool.get(),    \
                  &trace);                                                    \
      std::memcpy(y, buf.last_output().data(), sizeof(T) * n_rows);           \
      if (counters) {                                                         \
        counters[0] = trace.fast_tiles;                                       \
        counters[1] = trace.normal_tiles;                                     \
        counters[2] = trace.skipped_tiles;                                    \
      }                                                                       \
    });                                                                       \
  }                                                                           \
  int ref_spmv_csr_##SUFFIX(int64_t n_rows, int64_t n_cols, const int64_t* ro, \
                            const int32_t* cols, const T* vals, const T* x,   \
                            T* y) {                                           \
    return guarded([&] {                                                      \
      const CsrMatrix<T> a = make_csr<T>(n_rows, n_cols, ro, cols, vals);     \
      spmv_csr_reference(a, std::span<const T>(x, n_cols),                    \
                         std::span<T>(y, n_rows));                            \
    });                                                                       \
  }                                                                           \
  void* ref_engine_create_##SUFFIX(int64_t n_rows, int64_t n_cols,            \
                                   const int64_t* ro, const int32_t* cols,    \
                                   const T* vals, int omega, int sigma,       \
                                   int block, int nthreads) {                 \
    RefEngine<T>* e = nullptr;                                                \
    const int rc = guarded([&] {                                              \
      auto eng = std::make_unique<RefEngine<T>>();                            \
      eng->a = make_csr<T>(n_rows, n_cols, ro, cols, vals);                   \
      eng->c = SimtConfig::make(omega, sigma, block);                         \
      if (nthreads > 1) eng->pool = std::make_unique<ThreadPool>(nthreads);   \
      static CooTriples unused;                                               \
      eng->backend = make_backend<T>(BackendKind::merbit, eng->a, unused,     \
                                     eng->c, eng->pool.get());                \
      e = eng.release();                                                      \
    });                                                                       \
    return rc == 0 ? e : nullptr;                                             \
  }                                                                           \
  int ref_engine_apply_##SUFFIX(void* h, const T* x, T* y) {                  \
    return guarded([&] {                                                      \
      auto* e = static_cast<RefEngine<T>*>(h);                                \
      const std::vector<T>& out =                                             \
          e->backend->apply(std::span<const T>(x, e->a.n_cols));              \
      if (y) std::memcpy(y, out.data(), sizeof(T) * e->a.n_rows);             \
    });                                                                       \
  }                                                                           \
  double ref_engine_preprocess_seconds_##SUFFIX(void* h) {                    \
    return static_cast<RefEngine<T>*>(h)->backend->preprocess_seconds();      \
  }                                                                           \
  int ref_engine_pagerank_##SUFFIX(void* h, double damping, double err_tol,   \
                                   int64_t max_iters, int64_t ref_iters,      \
                                   T* pi, int64_t* iterations,                \
                                   double* final_err, double* seconds) {      \
    return guarded([&] {                                                      \
      auto* e = static_cast<RefEngine<T>*>(h);                                \
      PageRankConfig<T> cfg;                                                  \
      cfg.damping = static_cast<T>(damping);                                  \
      cfg.err_tol = static_cast<T>(err_tol);                                  \
      cfg.max_iters = max_iters;                                              \
      cfg.reference_iters = ref_iters;                                        \
      const PageRankResult<T> r = pagerank<T>(e->a, cfg, *e->backend);       \
      if (pi) std::memcpy(pi, r.pi.data(), sizeof(T) * r.pi.size());          \
      *iterations = r.iterations;                                             \
      *final_err = r.final_err;                                               \
      *seconds = r.iterate_seconds;                                           \
    });                                                                       \
  }                                                                           \
  void ref_engine_destroy_##SUFFIX(void* h) {                                 \
    delete static_cast<RefEngine<T>*>(h);                                     \
  }

REF_SPMV(double, f64)
REF_SPMV(float, f32)

// bicgstab<T> over the csr backend (solvers.hpp:268-373); status 0/1/2 as
// SolveStatus converged / max_iterations / breakdown.
#define REF_BICGSTAB(T, SUFFIX)                                                   \
  int ref_bicgstab_csr_##SUFFIX(int64_t n, const int64_t* ro, const int32_t* cols, \
                                const T* vals, const T* b, double tol,            \
                                int64_t max_iters, T* x, double* hist,            \
                                int64_t* iterations, double* final_residual,      \
                                int* status, char* reason, int reason_len) {      \
    return guarded([&] {                                                          \
      const CsrMatrix<T> a = make_csr<T>(n, n, ro, cols, vals);                   \
      CsrReferenceBackend<T> backend(a);                                          \
      BicgstabConfig<T> cfg;                                                      \
      cfg.tol = static_cast<T>(tol);                                              \
      cfg.max_iters = max_iters;                                                  \
      const auto r = bicgstab<T>(a, std::span<const T>(b, b + n), cfg, backend);  \
      std::memcpy(x, r.x.data(), sizeof(T) * n);                                  \
      for (std::size_t i = 0; i < r.residual_history.size(); ++i)                 \
        hist[i] = r.residual_history[i];                                          \
      *iterations = r.iterations;                                                 \
      *final_residual = r.final_residual;                                         \
      *status = r.status == SolveStatus::converged       ? 0                      \
                : r.status == SolveStatus::max_iterations ? 1                     \
                                                          : 2;                    \
      std::snprintf(reason, reason_len, "%s", r.breakdown_reason.c_str());        \
    });                                                                           \
  }

// spmv_merge_runtime<T> (merge_spmv.hpp:21-82), single-threaded
#define REF_MERGE_RUNTIME(T, SUFFIX)                                              \
  int ref_spmv_merge_runtime_##SUFFIX(int64_t n_rows, int64_t n_cols,             \
                                      const int64_t* ro, const int32_t* cols,     \
                                      const T* vals, const T* x, int sigma, T* y) { \
    return guarded([&] {                                                          \
      const CsrMatrix<T> a = make_csr<T>(n_rows, n_cols, ro, cols, vals);         \
      const SimtConfig c = SimtConfig::make(32, sigma, 32);                       \
      const auto out = spmv_merge_runtime<T>(a, std::span<const T>(x, x + n_cols), c); \
      std::memcpy(y, out.data(), sizeof(T) * out.size());                        \
    });                                                                           \
  }

extern "C" {
REF_MERGE_RUNTIME(double, f64)
REF_MERGE_RUNTIME(float, f32)
REF_BICGSTAB(double, f64)
REF_BICGSTAB(float, f32)

// ---- file formats (tile.cpp:161-234, matrix_market.cpp) -----------------
// generate_tile on the given rows + write_tile_cache
int ref_tile_cache_write(const char* path, int64_t n_rows, int64_t nnz, const int64_t* ro,
                         int omega, int sigma, int f64) {
  return guarded([&] {
    const SimtConfig c = SimtConfig::make(omega, sigma, omega);
    const TileMetadata t = generate_tile(std::span<const index_t>(ro, ro + n_rows + 1), n_rows,
                                         nnz, c);
    write_tile_cache(path, t, f64 ? ScalarPrecision::f64 : ScalarPrecision::f32);
  });
}

// read_tile_cache: counts + arrays (malloc'd, ref_free)
int ref_tile_cache_read(const char* path, int* omega, int* sigma, int64_t* n_rows,
                        int64_t* nnz, int64_t* tile_num, int64_t* lane_num, uint32_t** tx,
                        uint32_t** ty, uint32_t** ld, int* f64) {
  return guarded([&] {
    const TileCacheContents c = read_tile_cache(path);
    const TileMetadata& t = c.tile;
    *omega = t.omega;
    *sigma = t.sigma;
    *n_rows = t.n_rows;
    *nnz = t.nnz;
    *tile_num = t.tile_num;
    *lane_num = t.lane_num;
    *f64 = c.precision == ScalarPrecision::f64 ? 1 : 0;
    auto dup = [](const std::vector<uint32_t>& v) {
      auto* p = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (v.size() + 1)));
      std::memcpy(p, v.data(), sizeof(uint32_t) * v.size());
      return p;
    };
    *tx = dup(t.tile_x);
    *ty = dup(t.tile_y);
    *ld = dup(t.lane_desc);
  });
}

static void export_coo_arrays(const CooTriples& coo, int64_t* n_rows, int64_t* n_cols,
                              int64_t* nnz, int64_t** rows, int64_t** cols, double** vals) {
  const std::size_t n = coo.entries.size();
  *n_rows = coo.n_rows;
  *n_cols = coo.n_cols;
  *nnz = static_cast<int64_t>(n);
  *rows = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (n + 1)));
  *cols = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (n + 1)));
  *vals = static_cast<double*>(std::malloc(sizeof(double) * (n + 1)));
  for (std::size_t k = 0; k < n; ++k) {
    (*rows)[k] = coo.entries[k].row;
    (*cols)[k] = coo.entries[k].col;
    (*vals)[k] = coo.entries[k].value;
  }
}

static CooTriples import_coo(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                             const int64_t* cols, const double* vals) {
  CooTriples coo;
  coo.n_rows = n_rows;
  coo.n_cols = n_cols;
  coo.entries.reserve(static_cast<std::size_t>(nnz));
  for (int64_t k = 0; k < nnz; ++k) coo.entries.push_back({rows[k], cols[k], vals[k]});
  return coo;
}

// 0 = Matrix Market text, 1 = MBMX cache, 2 = load_matrix_any
int ref_matrix_read(const char* path, int which, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                    int64_t** rows, int64_t** cols, double** vals) {
  return guarded([&] {
    const CooTriples coo = which == 0   ? parse_matrix_market_file(path)
                           : which == 1 ? read_matrix_cache(path)
                                        : load_matrix_any(path);
    export_coo_arrays(coo, n_rows, n_cols, nnz, rows, cols, vals);
  });
}

// 0 = Matrix Market text, 1 = MBMX cache
int ref_matrix_write(const char* path, int which, int64_t n_rows, int64_t n_cols, int64_t nnz,
                     const int64_t* rows, const int64_t* cols, const double* vals) {
  return guarded([&] {
    const CooTriples coo = import_coo(n_rows, n_cols, nnz, rows, cols, vals);
    if (which == 0)
      write_matrix_market_file(path, coo);
    else
      write_matrix_cache(path, coo);
  });
}

// coo_to_csr<T> (csr.hpp:70-88): CSR arrays (malloc'd)
int ref_coo_to_csr_f64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                       const int64_t* cols, const double* vals, int64_t* out_nnz, int64_t** ro,
                       int32_t** ocols, double** ovals) {
  return guarded([&] {
    const CsrMatrix<double> a = coo_to_csr<double>(import_coo(n_rows, n_cols, nnz, rows, cols,
                                                              vals));
    int64_t nr, nc, m;
    export_csr(a, &nr, &nc, &m, ro, ocols, ovals);
    *out_nnz = m;
  });
}
}

// pagerank<T> over the csr backend (solvers.hpp:154-218); status 0/1 as
// SolveStatus converged / max_iterations.
int ref_pagerank_csr_f64(int64_t n, const int64_t* ro, const int32_t* cols,
                         const double* vals, double damping, double err_tol,
                         int64_t max_iters, int64_t ref_iters, double* pi,
                         double* ref_pi, int64_t* iterations,
                         double* final_err, int* status) {
  return guarded([&] {
    const CsrMatrix<double> p = make_csr<double>(n, n, ro, cols, vals);
    CsrReferenceBackend<double> backend(p);
    PageRankConfig<double> cfg;
    cfg.damping = damping;
    cfg.err_tol = err_tol;
    cfg.max_iters = max_iters;
    cfg.reference_iters = ref_iters;
    const auto r = pagerank<double>(p, cfg, backend);
    std::memcpy(pi, r.pi.data(), sizeof(double) * n);
    std::memcpy(ref_pi, r.reference_pi.data(), sizeof(double) * n);
    *iterations = r.iterations;
    *final_err = r.final_err;
    *status = r.status == SolveStatus::converged ? 0 : 1;
  });
}

int ref_pagerank_csr_f32(int64_t n, const int64_t* ro, const int32_t* cols,
                         const float* vals, double damping, double err_tol,
                         int64_t max_iters, int64_t ref_iters, float* pi,
                         int64_t* iterations, double* final_err,
                         int* status) {
  return guarded([&] {
    const CsrMatrix<float> p = make_csr<float>(n, n, ro, cols, vals);
    CsrReferenceBackend<float> backend(p);
    PageRankConfig<float> cfg;
    cfg.damping = static_cast<float>(damping);
    cfg.err_tol = static_cast<float>(err_tol);
    cfg.max_iters = max_iters;
    cfg.reference_iters = ref_iters;
    const auto r = pagerank<float>(p, cfg, backend);
    std::memcpy(pi, r.pi.data(), sizeof(float) * n);
    *iterations = r.iterations;
    *final_err = r.final_err;
    *status = r.status == SolveStatus::converged ? 0 : 1;
  });
}

int ref_build_transition_f64(int64_t n, const int64_t* ro,
                             const int32_t* cols, int64_t* p_ro,
                             int32_t* p_cols, double* p_vals) {
  return guarded([&] {
    std::vector<double> ones(static_cast<std::size_t>(ro[n]), 1.0);
    const CsrMatrix<double> adj = make_csr<double>(n, n, ro, cols, ones.data());
    const CsrMatrix<double> p = build_transition(adj);
    std::memcpy(p_ro, p.row_offsets.data(), sizeof(int64_t) * (n + 1));
    for (int64_t k = 0; k < p.nnz(); ++k) {
      p_cols[k] = static_cast<int32_t>(p.col_indices[k]);
      p_vals[k] = p.values[k];
    }
  });
}

int ref_random_matrix_csr(int shape, uint64_t seed, int64_t* n_rows,
                          int64_t* n_cols, int64_t* nnz, int64_t** ro,
                          int32_t** cols, double** vals) {
  return guarded([&] {
    const CsrMatrix<double> a = coo_to_csr<double>(testing::random_matrix(
        testing::kAllShapes[shape], seed));
    export_csr(a, n_rows, n_cols, nnz, ro, cols, vals);
  });
}

int ref_ring_with_chords_csr(int64_t n, int64_t extra, uint64_t seed,
                             int64_t* nnz, int64_t** ro, int32_t** cols,
                             double** vals) {
  return guarded([&] {
    const CsrMatrix<double> a = ring_with_chords<double>(n, extra, seed);
    int64_t nr, nc;
    export_csr(a, &nr, &nc, nnz, ro, cols, vals);
  });
}

void ref_seed_test_vector(int64_t n, double lo, double hi, uint64_t seed,
                          double* out) {
  const auto v = seed_test_vector<double>(n, lo, hi, seed);
  std::memcpy(out, v.data(), sizeof(double) * n);
}

}  // extern "C"
