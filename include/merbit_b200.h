/*
 * merbit_b200.h -- C ABI of the B200-native MERBIT library (libmerbit_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/merbit): one-time TILE preprocessing
 * (generate_tile), repeated descriptor-driven SpMV (spmv_merbit) and the
 * PageRank driver (pagerank), all executed on an sm_100a GPU.  Plain pointers
 * and sizes only; no C++ or torch types cross it.  The C++ mirror of the
 * reference API (SimtConfig, TileMetadata, DualBuffer, SpmvBackend,
 * make_backend, pagerank) is include/merbit_b200/merbit.hpp, header-only over
 * these entry points; INTEGRATION.md shows the reference-side binding.
 *
 * Conventions
 *  - Every function returns an mbx_status; on failure mbx_last_error() holds
 *    a thread-local message.  Status codes mirror the reference's exception
 *    taxonomy (include/merbit/types.hpp:23-65) so the C++ wrapper can rethrow
 *    the same types, plus CUDA/NCCL/unsupported codes.
 *  - "_host" pointers are host memory; "_dev" pointers are device memory of
 *    the context's device.  Host-buffer calls synchronize the context stream
 *    before returning; device-buffer calls are stream-ordered and
 *    asynchronous.
 *  - A context is one device + one stream; it is not thread-safe (the
 *    reference's backends are single-caller too, backend.hpp:17-21).
 *  - There is no CPU fallback: with no usable sm_100 device every compute
 *    entry point fails with MBX_CUDA_ERROR.
 */
#ifndef MERBIT_B200_H
#define MERBIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MBX_API __attribute__((visibility("default")))

typedef enum {
  MBX_OK = 0,
  MBX_ERROR = 1,            /* merbit::error               */
  MBX_IO_ERROR = 2,         /* merbit::io_error            */
  MBX_PARSE_ERROR = 3,      /* merbit::parse_error         */
  MBX_CONFIG_ERROR = 4,     /* merbit::config_error        */
  MBX_DIMENSION_ERROR = 5,  /* merbit::dimension_error     */
  MBX_CAPACITY_ERROR = 6,   /* merbit::capacity_error      */
  MBX_CORRUPTION_ERROR = 7, /* merbit::corruption_error    */
  MBX_CUDA_ERROR = 8,
  MBX_NCCL_ERROR = 9,
  MBX_UNSUPPORTED = 10
} mbx_status;

typedef enum { MBX_F32 = 0, MBX_F64 = 1 } mbx_precision;

/* SimtConfig (include/merbit/config.hpp:18-38). */
typedef struct {
  int32_t omega;
  int32_t sigma;
  int32_t block_size;
  int32_t offset_bits;
} mbx_simt_config;

/* TileMetadata header (include/merbit/tile.hpp:27-44). */
typedef struct {
  int32_t omega;
  int32_t sigma;
  int64_t n_rows;
  int64_t nnz;
  int64_t tile_num;
  int64_t lane_num;
  double preprocess_seconds; /* device time of the K1 kernels (T_p) */
} mbx_tile_info;

/* SpmvTrace routing counters (include/merbit/merbit_spmv.hpp:21-28). */
typedef struct {
  int64_t fast_tiles;
  int64_t normal_tiles;
  int64_t skipped_tiles;
} mbx_spmv_trace;

/* PageRankConfig (include/merbit/solvers.hpp:76-82). */
typedef struct {
  double damping;          /* 0.85 */
  double err_tol;          /* 1e-10 */
  int64_t max_iters;       /* 210 */
  int64_t reference_iters; /* 210; the yardstick power run (178-191) */
} mbx_pagerank_config;

/* PageRankResult (solvers.hpp:84-93) plus the device-side reductions. */
typedef struct {
  int64_t iterations;
  double final_err;          /* ERR vs the yardstick, inf-norm relative */
  int32_t status;            /* 0 converged, 1 max_iterations */
  double preprocess_seconds; /* T_p of the TILE used */
  double iterate_seconds;    /* T_r: device time of the power loop */
  double l1_residual;        /* ||pi_k - pi_{k-1}||_1 of the last iteration */
  double mass;               /* ||pi_k||_1 */
  double dangling_mass;      /* sum of pi_k over dangling vertices */
} mbx_pagerank_result;

/* BicgstabConfig (solvers.hpp:224-228). */
typedef struct {
  double tol;        /* 1e-10 (converted to T like BicgstabConfig<T>) */
  int64_t max_iters; /* 20000 */
} mbx_bicgstab_config;

/* BicgstabResult (solvers.hpp:230-240); x and the residual history are
 * returned through the caller's buffers. */
typedef struct {
  int64_t iterations;
  double final_residual;     /* ||A x - b|| / ||b|| of the last pass */
  int32_t status;            /* 0 converged, 1 max_iterations, 2 breakdown */
  char breakdown_reason[32]; /* "rho", "rhat_dot_v", "t_dot_t", "omega", "diverged" */
  double preprocess_seconds; /* T_p of the TILE used */
  double iterate_seconds;    /* device time of the iteration loop */
} mbx_bicgstab_result;

/* CooTriples (include/merbit/csr.hpp:22-26) as three host arrays in entry
 * order; arrays returned by the library are freed with mbx_coo_free. */
typedef struct {
  int64_t n_rows;
  int64_t n_cols;
  int64_t nnz;
  int64_t* rows;
  int64_t* cols;
  double* vals;
} mbx_coo;

typedef struct mbx_context_s mbx_context;
typedef struct mbx_matrix_s mbx_matrix;
typedef struct mbx_tile_s mbx_tile;
typedef struct mbx_pagerank_plan_s mbx_pagerank_plan;

/* ---- errors / build info ------------------------------------------------ */
MBX_API const char* mbx_last_error(void);
MBX_API const char* mbx_build_info(void);

/* ---- configuration (host-only; no device needed) ------------------------ */
/* SimtConfig::make (src/config.cpp:12-38): validates 2*ceil_log2(w*s)+s<=32
 * and block_size % omega == 0; derives offset_bits. */
MBX_API int mbx_config_make(int omega, int sigma, int block_size,
                            mbx_simt_config* out);
/* select_sigma (src/config.cpp:40-43): 14 for f32, 7 for f64; override>0
 * wins.  Returns sigma (never fails). */
MBX_API int mbx_select_sigma(int precision, int override_sigma);
/* TILE counts (src/tile.cpp:33-35). */
MBX_API int mbx_tile_counts(int64_t nnz, int64_t n_rows,
                            const mbx_simt_config* c, int64_t* tile_num,
                            int64_t* lane_num);
/* metadata_footprint (src/tile.cpp:146-154). */
MBX_API double mbx_metadata_footprint(int64_t nnz, int64_t n_rows,
                                      const mbx_simt_config* c, double r_f);
/* merge_search (src/merge_path.cpp:8-36) on host arrays. */
MBX_API int mbx_merge_search(const int64_t* row_offsets_host, int64_t n_rows,
                             int64_t nnz, int64_t diag, int64_t* x,
                             int64_t* y);
/* Multi-GPU row partition: cut the merge path at diagonals
 * floor(g*(m+n)/parts) with merge_search and snap each cut to its row start.
 * row_bounds_host has parts+1 entries, [0] = 0, [parts] = n_rows. */
MBX_API int mbx_plan_row_shards(const int64_t* row_offsets_host,
                                int64_t n_rows, int64_t nnz, int parts,
                                int64_t* row_bounds_host);
/* Cost-weighted row partition: cut where ro[r] + row_weight * r crosses
 * g/parts of nnz + row_weight * n_rows (row_weight = cost of one row's
 * commit in nonzeros; 1.0 is the merge-path cut above).  The PageRank commit
 * measured ~3.4 nonzeros per row on B200. */
MBX_API int mbx_plan_row_shards_weighted(const int64_t* row_offsets_host,
                                         int64_t n_rows, int64_t nnz, int parts,
                                         double row_weight,
                                         int64_t* row_bounds_host);

/* ---- context -------------------------------------------------------------- */
MBX_API int mbx_device_count(int* count);
MBX_API int mbx_context_create(int device, mbx_context** out);
MBX_API int mbx_context_destroy(mbx_context* ctx);
/* Adopt a caller stream (cudaStream_t as void*); NULL restores the
 * context's own stream. */
MBX_API int mbx_context_set_stream(mbx_context* ctx, void* stream);
MBX_API void* mbx_context_stream(mbx_context* ctx);
MBX_API int mbx_context_synchronize(mbx_context* ctx);
/* Kernel launch shape of K2 (omega == 32): warps per CTA, resident CTAs per
 * SM (persistent grid), hub-cache cap (-1 auto, 0 off).  Both shape
 * arguments 0 (the default): automatic -- 32 warps x 1 CTA, except 16 x 2
 * for a small matrix without a hub table. */
MBX_API int mbx_context_set_tuning(mbx_context* ctx, int warps_per_cta,
                                   int ctas_per_sm, int max_hubs);
/* Shared-memory budget per SM for K2 (bytes; the rest is L1) and how K2
 * stages the next tile: 0 nothing, 1 L2 prefetch of its streams, 2 TMA bulk
 * copy of its column slots + descriptors into shared memory (slot layout),
 * -1 auto (2 for fp64, 0 for fp32).  smem_per_sm -1: 160 KB for fp32, 128 KB
 * for fp64.  Defaults -1 / -1. */
MBX_API int mbx_context_set_tuning_ex(mbx_context* ctx, int smem_per_sm,
                                      int prefetch);
/* K2 data layout: 1 (default) = lane-major slot copy of the matrix, built
 * once per TILE next to it (omega 32 with the default sigma: 14 for f32, 7
 * for f64); 0 = CSR order staged through shared memory (any omega/sigma). */
MBX_API int mbx_context_set_layout(mbx_context* ctx, int layout);
/* Number of merbit kernels this context launched so far. */
MBX_API int64_t mbx_context_launch_count(const mbx_context* ctx);

/* ---- matrices (device-resident CSR: T values, int32 columns, u32 rows) --- */
/* Copies a host CsrMatrix<T> (include/merbit/csr.hpp:29-38) to the device
 * once: int64 col_indices narrow to int32 (n_cols < 2^31), row_offsets to
 * u32 (nnz < 2^32, the TILE capacity rule of tile.cpp:23-26). */
MBX_API int mbx_matrix_upload(mbx_context* ctx, int precision, int64_t n_rows,
                              int64_t n_cols, const int64_t* row_offsets_host,
                              const int64_t* col_indices_host,
                              const void* values_host, mbx_matrix** out);
/* Same, with int32 column indices on the host. */
MBX_API int mbx_matrix_upload_i32(mbx_context* ctx, int precision,
                                  int64_t n_rows, int64_t n_cols,
                                  const int64_t* row_offsets_host,
                                  const int32_t* col_indices_host,
                                  const void* values_host, mbx_matrix** out);
/* Synthetic R-MAT input generated on the device (counter-based; identical to
 * oracle/mo_rmat_csr).  kind 0: adjacency A (rows = source) with values
 * lo + (hi-lo)*U(value_seed, k); kind 1: PageRank transition P = A^T D^-1
 * (rows = destination, values 1/outdeg, solvers.hpp:36-74). */
MBX_API int mbx_matrix_generate_rmat(mbx_context* ctx, int precision,
                                     int scale, int edge_factor,
                                     uint64_t seed, int kind,
                                     uint64_t value_seed, double lo,
                                     double hi, mbx_matrix** out);
/* BASELINE config C5: 27-point stencil on a grid_dim^3 grid (diagonal 26,
 * neighbours -1; the 3-D five_point_laplacian, fixtures.hpp:40-56). */
MBX_API int mbx_matrix_generate_stencil27(mbx_context* ctx, int precision,
                                          int64_t grid_dim, mbx_matrix** out);
/* BASELINE config C3: 2^log2_rows rows, power-law row lengths
 * max(1, 2^20 / (rank+1)^0.8) by a seeded rank permutation, exactly
 * n - floor(0.9 n) empty rows, strictly increasing columns spread over
 * [0, n), values in [-1, 1). */
MBX_API int mbx_matrix_generate_powerlaw(mbx_context* ctx, int precision,
                                         int log2_rows, uint64_t seed,
                                         mbx_matrix** out);
MBX_API int mbx_matrix_info(const mbx_matrix* m, int* precision,
                            int64_t* n_rows, int64_t* n_cols, int64_t* nnz);
/* Any output pointer may be NULL.  row_offsets as int64. */
MBX_API int mbx_matrix_download(const mbx_matrix* m,
                                int64_t* row_offsets_host,
                                int32_t* col_indices_host, void* values_host);
/* Device pointers of the matrix arrays (for fused/device-side callers). */
MBX_API int mbx_matrix_device_ptrs(const mbx_matrix* m, const void** values,
                                   const int32_t** col_indices,
                                   const uint32_t** row_offsets);
MBX_API int mbx_matrix_destroy(mbx_matrix* m);
/* x hub cache (no reference counterpart; an sm_100a-specific preprocessing
 * step next to generate_tile): ranks columns by reference count and stages
 * the most referenced x entries in shared memory during SpMV.  Results are
 * bitwise identical with and without it.  max_hubs < 0: automatic -- no
 * table for a matrix with fewer than 4096 nonzeros per resident K2 warp
 * (there the SpMV is latency-bound and a table does not pay), else as many
 * hubs as the shared-memory budget of the context tuning allows; > 0: at
 * most that many, whatever the size; 0: remove the cache. */
/* Slot copy currently cached on the matrix: slots (0 if none) and the
 * seconds its one-time build took (part of preprocessing). */
MBX_API int mbx_matrix_slot_info(const mbx_matrix* m, int64_t* slots, double* seconds);
MBX_API int mbx_matrix_build_xcache(mbx_context* ctx, mbx_matrix* m,
                                    int max_hubs, double* seconds);
MBX_API int mbx_matrix_xcache_info(const mbx_matrix* m, int* hubs,
                                   double* coverage);
/* Gather locality measured by the last mbx_matrix_build_xcache sample: the
 * mean number of distinct 32-byte sectors of x that 32 consecutive nonzeros
 * touch (-1 when the build did not sample: automatic mode on a small matrix,
 * or never built).  Below 16 the fp32 K2 prefetches each next tile into L2. */
MBX_API int mbx_matrix_gather_profile(const mbx_matrix* m, double* sectors_per_32);
/* The hub columns (xcache_info's count of them) into host_out, in slot
 * order: ascending column ids. */
MBX_API int mbx_matrix_hub_columns(const mbx_matrix* m, int32_t* host_out);
/* Compact form: once the K2 slot copy for TILE t exists (an SpMV or a
 * PageRank plan with t built it), free the CSR values and columns -- the slot
 * copy holds every (value, column) -- keeping a private copy of t's arrays.
 * Any later call that reads the CSR (download, relabel, row slices, the
 * yardstick, comparators, another TILE's slot copy, plan creation) rebuilds
 * it from the slot copy first.  Resident bytes drop from CSR + slots to
 * about the slot copy alone. */
MBX_API int mbx_matrix_compact(mbx_matrix* m, const mbx_tile* t);
/* Device bytes the matrix holds now: CSR arrays, row offsets, slot copy, hub
 * cache, vertex map, comparator state, a compact form's TILE copy. */
MBX_API int mbx_matrix_resident_bytes(const mbx_matrix* m, int64_t* bytes);
/* Frees the matrix's derived device copies -- the K2 slot copy, the x hub
 * cache and the COO comparator's row array -- keeping only the CSR.  Plans
 * over the matrix rebuild what they need before their next run. */
MBX_API int mbx_matrix_release_caches(mbx_matrix* m);
/* Device pointers of the hub-encoded column array and the hub column list
 * (NULL when no cache is built). */
MBX_API int mbx_matrix_xcache_ptrs(const mbx_matrix* m,
                                   const int32_t** cols_hub,
                                   const int32_t** hub_cols);

/* ---- TILE preprocessing (K1) --------------------------------------------- */
/* generate_tile(span row_offsets, n_rows, nnz, c) (src/tile.cpp:17-85) on
 * the GPU; the arrays are byte-identical to the reference's. */
MBX_API int mbx_generate_tile(mbx_context* ctx,
                              const int64_t* row_offsets_host, int64_t n_rows,
                              int64_t nnz, const mbx_simt_config* c,
                              mbx_tile** out);
/* generate_tile(const CsrMatrix&, c) (tile.hpp:54-58) from the resident
 * matrix. */
MBX_API int mbx_matrix_generate_tile(mbx_context* ctx, const mbx_matrix* m,
                                     const mbx_simt_config* c,
                                     mbx_tile** out);
MBX_API int mbx_tile_get_info(const mbx_tile* t, mbx_tile_info* info);
MBX_API int mbx_tile_download(const mbx_tile* t, uint32_t* tile_x_host,
                              uint32_t* tile_y_host,
                              uint32_t* lane_desc_host);
/* Adopt host TILE arrays (e.g. an MBTL cache, tile.cpp:161-234). */
MBX_API int mbx_tile_upload(mbx_context* ctx, const mbx_tile_info* info,
                            const uint32_t* tile_x_host,
                            const uint32_t* tile_y_host,
                            const uint32_t* lane_desc_host, mbx_tile** out);
MBX_API int mbx_tile_destroy(mbx_tile* t);

/* ---- SpMV (K2 + K3) ------------------------------------------------------- */
/* spmv_merbit (include/merbit/merbit_spmv.hpp:136-352): y = A x.  Every row
 * of y is assigned (no zero-on-entry requirement).  Errors as the reference:
 * config_error on omega/sigma or shape mismatch with the TILE (140-151),
 * dimension_error is the caller's (sizes are implied by the matrix).
 * trace may be NULL. */
MBX_API int mbx_spmv(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                     const mbx_simt_config* c, const void* x_host,
                     void* y_host, mbx_spmv_trace* trace);
MBX_API int mbx_spmv_device(mbx_context* ctx, const mbx_matrix* m,
                            const mbx_tile* t, const mbx_simt_config* c,
                            const void* x_dev, void* y_dev);
/* Routing counters only (device classification of every tile with the
 * kernel's own predicate). */
MBX_API int mbx_spmv_trace_counts(mbx_context* ctx, const mbx_tile* t,
                                  mbx_spmv_trace* trace);
/* SpmvTrace::deposits (merbit_spmv.hpp:21-28, 339-349): the (row, partial
 * sum) contributions the MERBIT decomposition forms for y = A x -- per lane,
 * one at each Down step and one for the row it leaves open; per lane of a
 * long-row tile, its lane-strided subtotal.  Per-row totals reproduce y up to
 * regrouping (the conservation property tests/test_kernel.cpp:136-158
 * checks).  rows_host / amounts_host NULL: *count = the capacity that always
 * suffices.  Otherwise at most `capacity` pairs are written (unordered) and
 * *count is the total; rows in the caller's vertex order (the terminal row
 * n_rows may appear, as in the reference). */
MBX_API int mbx_spmv_deposits(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                              const mbx_simt_config* c, const void* x_host,
                              int64_t* rows_host, void* amounts_host, int64_t capacity,
                              int64_t* count);
/* Plain row-parallel CSR SpMV on the device (the yardstick kernel of
 * pagerank, solvers.hpp:178-191, and a non-MERBIT comparator). */
MBX_API int mbx_spmv_csr_device(mbx_context* ctx, const mbx_matrix* m,
                                const void* x_dev, void* y_dev);

/* The paper's baselines on the same device: kind 0
 * csr_vector (warp per row), 1 coo_atomic (CooReferenceBackend, backend.hpp:
 * 67-84), 2 merge_runtime (spmv_merge_runtime, merge_spmv.hpp:21-82, with
 * this sigma), 3 merge_cub (cub::DeviceSpmv::CsrMV, library), 4..7 cuSPARSE
 * cusparseSpMV COO ALG1, COO ALG2, CSR ALG1, CSR ALG2 (the paper's baseline,
 * PAPER.md:32; libcusparse resolved with dlopen, MBX_UNSUPPORTED when absent;
 * 32-bit indices: nnz < 2^31). */
MBX_API int mbx_spmv_baseline_device(mbx_context* ctx, const mbx_matrix* m, int kind,
                                     int sigma, const void* x_dev, void* y_dev);

/* Mean device time of one multiply (CUDA events; x uploaded once, warm-up
 * untimed): kind -1 = MERBIT (K2+K3 with t), 0..7 = the comparators above. */
MBX_API int mbx_bench_spmv(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                           const mbx_simt_config* c, int kind, int iters, int warmup,
                           const void* x_host, double* mean_seconds);

/* ---- PageRank (K2/K3 in fused mode) --------------------------------------- */
/* One-shot pagerank<T>(p, cfg, backend) (solvers.hpp:154-218): yardstick,
 * power loop with the damping/teleport update, dangling redistribution, L1
 * residual, mass check and ERR fused into the SpMV commit; early exit when
 * ERR < err_tol.  pi0_host may be NULL (uniform 1/n, as the reference).
 * reference_pi_host / residual_history_host (max_iters doubles) may be NULL.
 * The context keeps the call's plan (2 pi buffers, scalars, the captured
 * power-loop graph) for the next call with the same matrix, TILE and configs;
 * it is dropped when the matrix or TILE is destroyed, the tuning changes, or
 * by mbx_context_release_cache. */
MBX_API int mbx_pagerank(mbx_context* ctx, const mbx_matrix* p,
                         const mbx_tile* t, const mbx_simt_config* c,
                         const mbx_pagerank_config* cfg, const void* pi0_host,
                         void* pi_host, void* reference_pi_host,
                         double* residual_history_host,
                         mbx_pagerank_result* result);
/* pagerank with the reference's on_iteration hook (solvers.hpp:157-158, 209):
 * iteration by iteration (no graph), each iterate copied to the host in the
 * original vertex order and handed to observer(r, pi, ERR, user) after the
 * mass check and before the convergence test -- a test / monitoring path.
 * Results as mbx_pagerank (bitwise: the same kernels run). */
typedef int (*mbx_pagerank_observer)(int64_t iteration, const void* pi_host, double err,
                                     void* user);  /* nonzero: abort the run (MBX_ERROR) */
MBX_API int mbx_pagerank_observed(mbx_context* ctx, const mbx_matrix* p,
                                  const mbx_tile* t, const mbx_simt_config* c,
                                  const mbx_pagerank_config* cfg, const void* pi0_host,
                                  void* pi_host, void* reference_pi_host,
                                  double* residual_history_host,
                                  mbx_pagerank_observer observer, void* user,
                                  mbx_pagerank_result* result);
/* Free the plan mbx_pagerank keeps between calls (no-op when none). */
MBX_API int mbx_context_release_cache(mbx_context* ctx);
/* Reusable plan: device buffers, dangling mask and the CUDA graph of the
 * power loop are built once. */
MBX_API int mbx_pagerank_plan_create(mbx_context* ctx, const mbx_matrix* p,
                                     const mbx_tile* t,
                                     const mbx_simt_config* c,
                                     const mbx_pagerank_config* cfg,
                                     mbx_pagerank_plan** out);
/* Runs the yardstick (if reference_iters > 0) and the power loop.  pi0_dev
 * may be NULL (uniform).  The final iterate is left on the device
 * (mbx_pagerank_plan_pi). Asynchronous; call mbx_pagerank_plan_result after
 * a stream sync. */
MBX_API int mbx_pagerank_plan_run(mbx_pagerank_plan* plan,
                                  const void* pi0_dev);
MBX_API int mbx_pagerank_plan_result(mbx_pagerank_plan* plan,
                                     mbx_pagerank_result* result,
                                     double* residual_history_host);
MBX_API const void* mbx_pagerank_plan_pi(const mbx_pagerank_plan* plan);
MBX_API const void* mbx_pagerank_plan_reference_pi(
    const mbx_pagerank_plan* plan);
MBX_API int mbx_pagerank_plan_destroy(mbx_pagerank_plan* plan);

/* ---- BiCGSTAB (K2/K3 SpMVs + device dot/axpy kernels) ------------------- */
/* bicgstab<T>(a, b, cfg, backend) (solvers.hpp:268-373): unpreconditioned
 * BiCGSTAB, three SpMVs per pass (the third for the true-residual stopping
 * test), breakdown reported with the reference's reason string.  Inner
 * products accumulate in fp64 (rounded to T once); vector updates round in T
 * exactly as written.  dimension_error on a non-square system, config_error
 * on a TILE that does not belong to the matrix.  residual_history_host
 * (max_iters doubles) may be NULL. */
MBX_API int mbx_bicgstab(mbx_context* ctx, const mbx_matrix* a, const mbx_tile* t,
                         const mbx_simt_config* c, const mbx_bicgstab_config* cfg,
                         const void* b_host, void* x_host,
                         double* residual_history_host, mbx_bicgstab_result* result);

/* ---- file formats (host) ------------------------------- */
/* MBTL TILE cache, byte-identical to write_tile_cache / read_tile_cache
 * (src/tile.cpp:161-234).  precision: MBX_F32 / MBX_F64 (header byte). */
MBX_API int mbx_tile_cache_write_host(const char* path, const mbx_tile_info* info,
                                      const uint32_t* tile_x, const uint32_t* tile_y,
                                      const uint32_t* lane_desc, int precision);
/* Arrays are allocated by the library (free with mbx_free); counts follow
 * from the header (tile.cpp:214-218).  io_error / parse_error /
 * corruption_error as the reference. */
MBX_API int mbx_tile_cache_read_host(const char* path, mbx_tile_info* info,
                                     uint32_t** tile_x, uint32_t** tile_y,
                                     uint32_t** lane_desc, int* precision);
/* Device TILE <-> MBTL file. */
MBX_API int mbx_tile_cache_write(const mbx_tile* t, const char* path, int precision);
MBX_API int mbx_tile_cache_load(mbx_context* ctx, const char* path, mbx_tile** out,
                                int* precision);
/* Matrix Market coordinate text (parse_matrix_market, matrix_market.cpp:
 * 47-133): real / integer / pattern, general / symmetric; parse_error
 * "origin:line: what" on malformed input. */
MBX_API int mbx_mm_read(const char* path, mbx_coo* out);
MBX_API int mbx_mm_parse(const char* text, int64_t len, const char* origin, mbx_coo* out);
/* "coordinate real general", 1-based, shortest round-trip values
 * (write_matrix_market, matrix_market.cpp:156-168). */
MBX_API int mbx_mm_write(const char* path, const mbx_coo* coo);
/* MBMX binary matrix cache (write/read_matrix_cache, matrix_market.cpp:
 * 178-225) and the magic-sniffing loader (load_matrix_any, 227-238). */
MBX_API int mbx_matrix_cache_write(const char* path, const mbx_coo* coo);
MBX_API int mbx_matrix_cache_read(const char* path, mbx_coo* out);
MBX_API int mbx_matrix_load_any(const char* path, mbx_coo* out);
MBX_API void mbx_coo_free(mbx_coo* coo);
MBX_API void mbx_free(void* p);
/* coo_to_csr<T> (csr.hpp:43-88) on the device: bounds check
 * (dimension_error), stable row-major sort, duplicates summed in fp64 in
 * entry order, one rounding to T -- the result is a resident matrix. */
MBX_API int mbx_matrix_from_coo(mbx_context* ctx, int precision, const mbx_coo* coo,
                                mbx_matrix** out);
/* build_transition (solvers.hpp:36-74) on the device: P[i][j] = T(1)/T(outdeg j)
 * for every adjacency entry j -> i, rows in ascending source order, dangling
 * columns empty; dimension_error on a non-square adjacency. */
MBX_API int mbx_matrix_build_transition(mbx_context* ctx, const mbx_matrix* adjacency,
                                        mbx_matrix** out);
/* Locality preprocessing (no reference counterpart): the symmetric relabel
 * P' = Q P Q^T with vertex v -> rank of its column count (descending, ties by
 * id), rows sorted, columns ascending -- hot columns of x become contiguous
 * (R-MAT s27 PageRank: 1.9x).  PageRank on P' gives pi'[rank[v]] = pi[v] up
 * to summation order.  The new matrix keeps the vertex map: the host-facing
 * mbx_spmv (x, y) and mbx_pagerank (pi0, pi, yardstick) stay in the ORIGINAL
 * vertex order; device-pointer entry points (mbx_spmv_device, plans, shard
 * groups) work in the new order.
 * rank_host (n int32) may be NULL. */
/* DegreeStats (include/merbit/csr.hpp:108-140): mean degree nnz/n_rows,
 * low_degree = mean <= sigma_threshold (callers pass select_sigma), the
 * longest row and the number of empty rows -- one reduction over the
 * resident row offsets.  dimension_error for a matrix with no rows. */
typedef struct {
  double mean_degree;
  int32_t low_degree;
  int32_t pad_;
  int64_t max_degree;
  int64_t empty_rows;
} mbx_degree_stats;
MBX_API int mbx_matrix_degree_stats(mbx_context* ctx, const mbx_matrix* m,
                                    int sigma_threshold, mbx_degree_stats* out);
MBX_API int mbx_matrix_relabel_by_degree(mbx_context* ctx, const mbx_matrix* m,
                                         mbx_matrix** out, int32_t* rank_host);

/* ---- multi-GPU row-sharded PageRank (one process per GPU) ---------------- */
/* GPU g owns rows [row_bounds[g], row_bounds[g+1]) of P (mbx_plan_row_shards)
 * with its own TILE; pi travels between iterations through one in-place
 * ncclAllGather per iteration over NVLink, the rank's reduction scalars
 * riding in the tail of its chunk.  Replaces the reference's single-process
 * pagerank loop (solvers.hpp:154-218) for the sharded case, yardstick
 * included: reference_iters > 0 runs the CSR power iterations (178-191)
 * through the same exchange and ERR is taken against each rank's rows of
 * pi*. */
typedef struct mbx_shard_group_s mbx_shard_group;
/* ncclGetUniqueId (128 bytes), to be broadcast by the caller's bootstrap. */
MBX_API int mbx_nccl_unique_id(void* id128);
/* Rows [r0, r1) of a resident matrix as a new matrix (columns unchanged). */
MBX_API int mbx_matrix_row_slice(mbx_context* ctx, const mbx_matrix* m,
                                 int64_t r0, int64_t r1, mbx_matrix** out);
/* nlocal shards (ranks rank0 .. rank0+nlocal-1) of a world-rank group.
 * nccl_id NULL: every shard is local (nlocal == world), all on this context's
 * device sharing one buffer -- no exchange is needed (single-GPU check of the
 * sharded path).  Otherwise nlocal == 1 and NCCL connects the world. */
MBX_API int mbx_shard_group_create(mbx_context* ctx, int64_t n_global,
                                   int world, const int64_t* row_bounds_host,
                                   int rank0, int nlocal,
                                   mbx_matrix* const* local_matrices,
                                   mbx_tile* const* local_tiles,
                                   const mbx_simt_config* c,
                                   const mbx_pagerank_config* cfg,
                                   const void* nccl_id,
                                   mbx_shard_group** out);
/* Fused compute + exchange (no collective library on the iteration path):
 * the PageRank commit of K2/K3 stores every non-dangling pi_new -- and K3
 * the rank's scalar tail -- straight into every peer's exchange buffer
 * (CUDA IPC mappings, NVLink/NVSwitch P2P stores), so the transfer overlaps
 * the SpMV tile by tile; one device barrier per iteration (system-scope
 * release/acquire epochs in peer memory, bounded: a missing peer fails the
 * run instead of hanging) replaces the all-gather.  Setup is two-phase
 * through the caller's bootstrap (MPI, torch.distributed, ...):
 *   create_peer -> export (MBX_SHARD_BLOB_BYTES) -> all-gather the world's
 *   blobs in rank order -> connect.
 * One shard per group (this rank's rows), world <= 8, the yardstick
 * (reference_iters > 0) included.  Ranks may share a device (the 2- and
 * 3-process tests) or a process (peers of the same pid use raw pointers).
 * run / result / gather_pi / download_local / destroy as above; destroy is
 * collective (a final barrier). */
#define MBX_SHARD_BLOB_BYTES 512
MBX_API int mbx_shard_group_create_peer(mbx_context* ctx, int64_t n_global,
                                        int world, const int64_t* row_bounds_host,
                                        int rank, mbx_matrix* local_matrix,
                                        mbx_tile* local_tile,
                                        const mbx_simt_config* c,
                                        const mbx_pagerank_config* cfg,
                                        mbx_shard_group** out);
MBX_API int mbx_shard_group_export(mbx_shard_group* group, void* blob);
MBX_API int mbx_shard_group_connect(mbx_shard_group* group, const void* blobs);
/* Peer groups: enqueue the final barrier without waiting (destroy does it
 * and then waits); lets one thread retire several ranks' groups. */
MBX_API int mbx_shard_group_quiesce(mbx_shard_group* group);
/* pi0_dev: optional start vector (n_global entries on this device; each
 * shard reads its own rows); NULL = uniform 1/n like the reference. */
MBX_API int mbx_shard_group_run(mbx_shard_group* group, const void* pi0_dev);
MBX_API int mbx_shard_group_result(mbx_shard_group* group,
                                   mbx_pagerank_result* result,
                                   double* residual_history_host);
/* The full pi (n_global entries) -- every rank holds all of it. */
MBX_API int mbx_shard_group_gather_pi(mbx_shard_group* group, void* pi_host);
/* Only this process's rows (its shards in rank order). */
MBX_API int mbx_shard_group_download_local(mbx_shard_group* group,
                                           void* pi_local_host);
MBX_API int mbx_shard_group_destroy(mbx_shard_group* group);

#ifdef __cplusplus
}
#endif
#endif /* MERBIT_B200_H */
