/*
 * merbit_oracle.h -- CPU restatement of the MERBIT reference path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2605_07391_b200/,
 * include/) may include, link or call this.  It is used by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline leg.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj) and is pinned against the compiled reference
 * (oracle/_ref, built by oracle/Makefile) and the committed golden vectors in
 * tests/golden/ (see tests/test_oracle.py).
 *
 * Status codes follow the product's C-ABI (include/merbit_b200.h):
 *   0 ok, 1 generic, 4 config, 5 dimension, 6 capacity, 7 corruption.
 */
#ifndef MERBIT_ORACLE_H
#define MERBIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MO_OK = 0, MO_ERR = 1, MO_ERR_CONFIG = 4, MO_ERR_DIMENSION = 5,
       MO_ERR_CAPACITY = 6, MO_ERR_CORRUPTION = 7 };

/* ---- config (src/config.cpp:5-43) ---------------------------------------- */
int mo_ceil_log2(int64_t x);
int mo_config_make(int omega, int sigma, int block_size, int* offset_bits);

/* ---- merge path (src/merge_path.cpp:8-59) -------------------------------- */
int mo_merge_search(const int64_t* row_offsets, int64_t n_rows, int64_t nnz,
                    int64_t diag, int64_t* x, int64_t* y, int* probes);
/* steps[k] = 0 Right, 1 Down; length nnz + n_rows */
void mo_sequential_path(const int64_t* row_offsets, int64_t n_rows,
                        int64_t nnz, uint8_t* steps);

/* ---- TILE (src/tile.cpp:17-133, descriptor.hpp:31-52) -------------------- */
void mo_tile_counts(int64_t nnz, int64_t n_rows, int omega, int sigma,
                    int64_t* tile_num, int64_t* lane_num);
int mo_generate_tile(const int64_t* row_offsets, int64_t n_rows, int64_t nnz,
                     int omega, int sigma, int offset_bits, uint32_t* tile_x,
                     uint32_t* tile_y, uint32_t* lane_desc);
int mo_reconstruct_path(const uint32_t* tile_x, const uint32_t* tile_y,
                        const uint32_t* lane_desc, int64_t n_rows, int64_t nnz,
                        int omega, int sigma, int offset_bits, uint8_t* steps);

/* ---- SpMV oracles (include/merbit/reference.hpp:15-67) -------------------
 * csr_f64 / csr_f32: fixed left-to-right row sums in the value precision
 *   (spmv_csr_reference<double/float>).
 * csr_f32_acc64: the fp32 gate oracle -- same fp32 inputs, fp64 accumulation;
 *   absrow[r] = sum |a_rk| |x_k| (the row-sum magnitude of the tolerance).
 * Rows are independent, so nthreads only splits the row loop. */
void mo_spmv_csr_f64(int64_t n_rows, const int64_t* ro, const int32_t* cols,
                     const double* vals, const double* x, double* y,
                     double* absrow, int nthreads);
void mo_spmv_csr_f32(int64_t n_rows, const int64_t* ro, const int32_t* cols,
                     const float* vals, const float* x, float* y);
void mo_spmv_csr_f32_acc64(int64_t n_rows, const int64_t* ro,
                           const int32_t* cols, const float* vals,
                           const float* x, double* y, double* absrow,
                           int nthreads);

/* ---- MERBIT SpMV restatement (include/merbit/merbit_spmv.hpp:136-352) ----
 * y is assigned (all rows written); counters = {fast, normal, skipped}. */
int mo_spmv_merbit_f64(int64_t n_rows, int64_t nnz, const int32_t* cols,
                       const double* vals, const double* x,
                       const uint32_t* tile_x, const uint32_t* tile_y,
                       const uint32_t* lane_desc, int omega, int sigma,
                       int offset_bits, int block_size, double* y,
                       int64_t* counters);
int mo_spmv_merbit_f32(int64_t n_rows, int64_t nnz, const int32_t* cols,
                       const float* vals, const float* x,
                       const uint32_t* tile_x, const uint32_t* tile_y,
                       const uint32_t* lane_desc, int omega, int sigma,
                       int offset_bits, int block_size, float* y,
                       int64_t* counters);

/* ---- PageRank (include/merbit/solvers.hpp:36-218) ------------------------
 * build_transition: P = A^T D^-1 from an adjacency pattern.  Outputs are
 * caller-allocated (n+1, nnz, nnz). */
void mo_build_transition_f64(int64_t n, const int64_t* adj_ro,
                             const int32_t* adj_cols, int64_t* p_ro,
                             int32_t* p_cols, double* p_vals);
void mo_build_transition_f32(int64_t n, const int64_t* adj_ro,
                             const int32_t* adj_cols, int64_t* p_ro,
                             int32_t* p_cols, float* p_vals);
/* pagerank over the CSR backend.  status: 0 converged, 1 max_iterations.
 * Returns MO_ERR on a zero-norm iterate, MO_ERR_CONFIG on bad config. */
int mo_pagerank_f64(int64_t n, const int64_t* ro, const int32_t* cols,
                    const double* vals, double damping, double err_tol,
                    int64_t max_iters, int64_t reference_iters, double* pi,
                    double* reference_pi, int64_t* iterations,
                    double* final_err, int* status, int nthreads);
int mo_pagerank_f32(int64_t n, const int64_t* ro, const int32_t* cols,
                    const float* vals, float damping, float err_tol,
                    int64_t max_iters, int64_t reference_iters, float* pi,
                    float* reference_pi, int64_t* iterations,
                    double* final_err, int* status);

/* ---- fixtures (include/merbit/fixtures.hpp, random.hpp,
 *      tests/support/generators.hpp) ---------------------------------------
 * Allocating constructors: *ro (n_rows+1), *cols (nnz), *vals (nnz, double
 * -- cast to T by the caller exactly like coo_to_csr<T>).  Free with
 * mo_free. */
void mo_free(void* p);
int mo_random_matrix_csr(int shape, uint64_t seed, int64_t* n_rows,
                         int64_t* n_cols, int64_t* nnz, int64_t** ro,
                         int32_t** cols, double** vals);
int mo_ring_with_chords_csr(int64_t n, int64_t extra_edges, uint64_t seed,
                            int64_t* nnz, int64_t** ro, int32_t** cols,
                            double** vals);
int mo_single_dense_row_csr(int64_t width, uint64_t seed, int64_t** ro,
                            int32_t** cols, double** vals);
void mo_seed_test_vector(int64_t n, double lo, double hi, uint64_t seed,
                         double* out);

/* ---- counter-based synthetic inputs (shared bit-for-bit with the GPU
 *      generator in paper_2605_07391_b200/csrc/generators.cu) -------------
 * R-MAT (a,b,c,d) = (.57,.19,.19,.05), edge_factor * 2^scale raw edges,
 * duplicates merged, self loops kept, natural vertex order.
 * transposed = 0: rows = source (adjacency A);  1: rows = destination
 * (the pattern of the PageRank transition P = A^T D^-1). */
int mo_rmat_csr(int scale, int edge_factor, uint64_t seed, int transposed,
                int nthreads, int64_t* nnz, int64_t** ro, int32_t** cols);
/* values[k] = lo + (hi-lo) * U(seed, k), U = top 53 bits of a splitmix hash */
void mo_hash_uniform(uint64_t seed, int64_t count, double lo, double hi,
                     double* out);
void mo_hash_uniform_f32(uint64_t seed, int64_t count, double lo, double hi,
                         float* out);
/* P values for a transposed pattern: vals[k] = T(1)/T(outdeg(cols[k])) */
void mo_transition_values_f32(int64_t n, int64_t nnz, const int32_t* cols,
                              float* vals);
void mo_transition_values_f64(int64_t n, int64_t nnz, const int32_t* cols,
                              double* vals);

/* bicgstab over the csr backend (solvers.hpp:268-373).  status 0 converged,
 * 1 max_iterations, 2 breakdown; reason 0 none, 1 rho, 2 rhat_dot_v,
 * 3 t_dot_t, 4 omega, 5 diverged.  hist (max_iters doubles) may be NULL. */
int mo_bicgstab_f64(int64_t n, const int64_t* ro, const int32_t* cols,
                    const double* vals, const double* b, double tol,
                    int64_t max_iters, double* x, double* hist,
                    int64_t* iterations, double* final_residual, int* status,
                    int* reason);
int mo_bicgstab_f32(int64_t n, const int64_t* ro, const int32_t* cols,
                    const float* vals, const float* b, float tol,
                    int64_t max_iters, float* x, double* hist,
                    int64_t* iterations, double* final_residual, int* status,
                    int* reason);

#ifdef __cplusplus
}
#endif
#endif
