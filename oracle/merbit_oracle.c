/*
 * merbit_oracle.c -- CPU restatement of the MERBIT reference path.
 *
 * TEST INFRASTRUCTURE ONLY (see merbit_oracle.h).  Each function cites the
 * reference function it restates (paths under /root/reference/proj).  The
 * restatement is pinned against the compiled reference (oracle/_ref) by
 * tests/test_oracle.py and against tests/golden/.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no fast-math: the fp
 * restatements must round exactly like the reference's plain C++).
 */
#define _GNU_SOURCE
#include "merbit_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define MIN(a, b) ((a) < (b) ? (a) : (b))
#define MAX(a, b) ((a) > (b) ? (a) : (b))

void mo_free(void* p) { free(p); }

/* ========================================================================
 * config -- src/config.cpp:5-38
 * ======================================================================== */
int mo_ceil_log2(int64_t x) {
  int k = 0;
  if (x < 1) return -1;
  while (((int64_t)1 << k) < x) ++k;
  return k;
}

int mo_config_make(int omega, int sigma, int block_size, int* offset_bits) {
  if (omega < 1 || sigma < 1) return MO_ERR_CONFIG;
  if (block_size < omega || block_size % omega != 0) return MO_ERR_CONFIG;
  int ob = mo_ceil_log2((int64_t)omega * sigma);
  if (2 * ob + sigma > 32) return MO_ERR_CONFIG;
  if (offset_bits) *offset_bits = ob;
  return MO_OK;
}

/* ========================================================================
 * merge path -- src/merge_path.cpp:8-59
 * ======================================================================== */
int mo_merge_search(const int64_t* ro, int64_t n_rows, int64_t nnz,
                    int64_t diag, int64_t* x, int64_t* y, int* probes) {
  if (diag < 0 || diag > nnz + n_rows) return MO_ERR_DIMENSION;
  int64_t lo = MAX(diag - nnz, 0);
  int64_t hi = MIN(diag, n_rows);
  int p = 0;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    ++p;
    /* row `mid` is finished before this diagonal (merge_path.cpp:28) */
    if (ro[mid + 1] <= diag - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (probes) *probes = p;
  *x = diag - lo;
  *y = MIN(lo, n_rows);
  return MO_OK;
}

void mo_sequential_path(const int64_t* ro, int64_t n_rows, int64_t nnz,
                        uint8_t* steps) {
  int64_t x = 0, y = 0, k = 0;
  while (x < nnz || y < n_rows) {
    if (y < n_rows && x < ro[y + 1]) {
      steps[k++] = 0;
      ++x;
    } else {
      steps[k++] = 1;
      ++y;
    }
  }
}

/* ========================================================================
 * TILE -- src/tile.cpp:17-133, include/merbit/descriptor.hpp:31-52
 * ======================================================================== */
void mo_tile_counts(int64_t nnz, int64_t n_rows, int omega, int sigma,
                    int64_t* tile_num, int64_t* lane_num) {
  const int64_t total = nnz + n_rows;
  const int64_t span = (int64_t)omega * sigma;
  *lane_num = total == 0 ? 0 : (total + sigma - 1) / sigma;
  *tile_num = total == 0 ? 0 : (total + span - 1) / span;
}

int mo_generate_tile(const int64_t* ro, int64_t n_rows, int64_t nnz,
                     int omega, int sigma, int ob, uint32_t* tile_x,
                     uint32_t* tile_y, uint32_t* lane_desc) {
  if (n_rows >= ((int64_t)1 << 31)) return MO_ERR_CAPACITY; /* tile.cpp:19 */
  if (nnz > (int64_t)0xFFFFFFFF) return MO_ERR_CAPACITY;    /* tile.cpp:23 */
  const int64_t total = nnz + n_rows;
  int64_t tiles, lanes;
  mo_tile_counts(nnz, n_rows, omega, sigma, &tiles, &lanes);
  const uint32_t field = 1u << ob;
  for (int64_t i = 0; i < tiles; ++i) {
    int64_t tsx = 0, tsy = 0;
    int any_down = 0;
    for (int lid = 0; lid < omega; ++lid) {
      const int64_t j = i * omega + lid;
      if (j >= lanes) break; /* only existing lanes vote (tile.cpp:46) */
      const int64_t diag = j * sigma;
      int64_t x, y;
      mo_merge_search(ro, n_rows, nnz, diag, &x, &y, NULL);
      if (lid == 0) {
        tsx = x;
        tsy = y;
      }
      const uint32_t xo = (uint32_t)(x - tsx), yo = (uint32_t)(y - tsy);
      if (xo >= field || yo >= field) return MO_ERR_CAPACITY;
      const int64_t steps = MIN((int64_t)sigma, total - diag);
      uint32_t flags = 0;
      for (int64_t k = 0; k < steps; ++k) {
        if (y < n_rows && x < ro[y + 1]) {
          ++x;
        } else {
          flags |= 1u << k;
          ++y;
          any_down = 1;
        }
      }
      lane_desc[j] = (flags << (2 * ob)) | (yo << ob) | xo;
    }
    tile_x[i] = (uint32_t)tsx;
    tile_y[i] = (uint32_t)tsy | (any_down ? 0u : 0x80000000u);
  }
  tile_x[tiles] = (uint32_t)nnz; /* terminal entry, never marked (80-83) */
  tile_y[tiles] = (uint32_t)n_rows;
  return MO_OK;
}

int mo_reconstruct_path(const uint32_t* tile_x, const uint32_t* tile_y,
                        const uint32_t* lane_desc, int64_t n_rows, int64_t nnz,
                        int omega, int sigma, int ob, uint8_t* steps_out) {
  int64_t tiles, lanes;
  mo_tile_counts(nnz, n_rows, omega, sigma, &tiles, &lanes);
  const int64_t total = nnz + n_rows;
  const uint32_t mask = (1u << ob) - 1u;
  int64_t x = 0, y = 0, k_out = 0;
  for (int64_t j = 0; j < lanes; ++j) {
    const int64_t t = j / omega;
    const uint32_t d = lane_desc[j];
    const int64_t lx = (int64_t)tile_x[t] + (d & mask);
    const int64_t ly = (int64_t)(tile_y[t] & 0x7FFFFFFFu) + ((d >> ob) & mask);
    if (lx != x || ly != y) return MO_ERR_CORRUPTION;
    const uint32_t flags = d >> (2 * ob);
    const int64_t steps = MIN((int64_t)sigma, total - j * sigma);
    for (int64_t k = 0; k < steps; ++k) {
      if ((flags >> k) & 1u) {
        if (steps_out) steps_out[k_out] = 1;
        ++y;
      } else {
        if (steps_out) steps_out[k_out] = 0;
        ++x;
      }
      ++k_out;
    }
  }
  if (x != nnz || y != n_rows) return MO_ERR_CORRUPTION;
  return MO_OK;
}

/* ========================================================================
 * CSR oracles -- include/merbit/reference.hpp:15-46
 * ======================================================================== */
typedef struct {
  int64_t r0, r1;
  const int64_t* ro;
  const int32_t* cols;
  const void* vals;
  const void* x;
  void* y;
  double* absrow;
  int kind; /* 0: f64, 1: f32 in / f64 accumulate */
} csr_job;

static void* csr_worker(void* arg) {
  csr_job* jb = (csr_job*)arg;
  for (int64_t r = jb->r0; r < jb->r1; ++r) {
    double s = 0.0, a = 0.0;
    if (jb->kind == 0) {
      const double* v = (const double*)jb->vals;
      const double* x = (const double*)jb->x;
      for (int64_t k = jb->ro[r]; k < jb->ro[r + 1]; ++k) {
        const double p = v[k] * x[jb->cols[k]];
        s += p;
        a += fabs(p);
      }
    } else {
      const float* v = (const float*)jb->vals;
      const float* x = (const float*)jb->x;
      for (int64_t k = jb->ro[r]; k < jb->ro[r + 1]; ++k) {
        const double p = (double)v[k] * (double)x[jb->cols[k]];
        s += p;
        a += fabs(p);
      }
    }
    ((double*)jb->y)[r] = s;
    if (jb->absrow) jb->absrow[r] = a;
  }
  return NULL;
}

static void csr_parallel(int64_t n_rows, const int64_t* ro, const int32_t* cols,
                         const void* vals, const void* x, double* y,
                         double* absrow, int kind, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  csr_job jobs[256];
  /* split by nonzeros so hub rows do not serialise one worker */
  const int64_t nnz = ro[n_rows];
  int64_t r = 0;
  for (int t = 0; t < nthreads; ++t) {
    const int64_t target = nnz / nthreads * (t + 1);
    int64_t r1 = r;
    if (t == nthreads - 1) {
      r1 = n_rows;
    } else {
      while (r1 < n_rows && ro[r1] < target) ++r1;
    }
    jobs[t] = (csr_job){r, r1, ro, cols, vals, x, y, absrow, kind};
    r = r1;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, csr_worker, &jobs[t]);
  csr_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

void mo_spmv_csr_f64(int64_t n_rows, const int64_t* ro, const int32_t* cols,
                     const double* vals, const double* x, double* y,
                     double* absrow, int nthreads) {
  csr_parallel(n_rows, ro, cols, vals, x, y, absrow, 0, nthreads);
}

void mo_spmv_csr_f32_acc64(int64_t n_rows, const int64_t* ro,
                           const int32_t* cols, const float* vals,
                           const float* x, double* y, double* absrow,
                           int nthreads) {
  csr_parallel(n_rows, ro, cols, vals, x, y, absrow, 1, nthreads);
}

void mo_spmv_csr_f32(int64_t n_rows, const int64_t* ro, const int32_t* cols,
                     const float* vals, const float* x, float* y) {
  for (int64_t r = 0; r < n_rows; ++r) {
    float s = 0.0f;
    for (int64_t k = ro[r]; k < ro[r + 1]; ++k) s += vals[k] * x[cols[k]];
    y[r] = s;
  }
}

/* ========================================================================
 * MERBIT SpMV restatement -- include/merbit/merbit_spmv.hpp:58-352
 * (fast_tile_reduce 58-77, warp_segmented_sum 85-117, block loop 182-324,
 *  ordered carry fold 330-337).  Generated for double and float.
 * ======================================================================== */
static int64_t bit_ceil64(int64_t v) {
  int64_t w = 1;
  while (w < v) w <<= 1;
  return w;
}

#define DEFINE_MERBIT(T, NAME)                                                 \
  int NAME(int64_t n_rows, int64_t nnz, const int32_t* cols, const T* vals,    \
           const T* x, const uint32_t* tile_x, const uint32_t* tile_y,         \
           const uint32_t* lane_desc, int omega, int sigma, int ob,            \
           int block_size, T* y, int64_t* counters) {                          \
    int64_t tiles, lanes;                                                      \
    mo_tile_counts(nnz, n_rows, omega, sigma, &tiles, &lanes);                 \
    const int64_t total = nnz + n_rows;                                        \
    const int wpb = block_size / omega;                                        \
    if (wpb < 1) return MO_ERR_CONFIG;                                         \
    const int64_t blocks = (tiles + wpb - 1) / wpb;                            \
    const uint32_t mask = (1u << ob) - 1u;                                     \
    const int64_t width = bit_ceil64(omega);                                   \
    T* scratch = (T*)malloc(sizeof(T) * ((size_t)(block_size + 1) * sigma + 1)); \
    T* sub = (T*)malloc(sizeof(T) * width);                                    \
    T* lane_sum = (T*)malloc(sizeof(T) * omega);                               \
    T* run_sum = (T*)malloc(sizeof(T) * omega);                                \
    T* tmp_sum = (T*)malloc(sizeof(T) * omega);                                \
    int64_t* lane_row = (int64_t*)malloc(sizeof(int64_t) * omega);             \
    uint8_t* lane_flag = (uint8_t*)malloc(omega);                              \
    uint8_t* run_flag = (uint8_t*)malloc(omega);                               \
    uint8_t* tmp_flag = (uint8_t*)malloc(omega);                               \
    int* ccount = (int*)calloc((size_t)MAX(blocks, 1), sizeof(int));          \
    int64_t* crow = (int64_t*)calloc((size_t)MAX(blocks, 1) * 2, sizeof(int64_t)); \
    T* csum = (T*)calloc((size_t)MAX(blocks, 1) * 2, sizeof(T));               \
    int64_t fast = 0, normal = 0, skipped = 0;                                 \
    for (int64_t r = 0; r < n_rows; ++r) y[r] = (T)0;                          \
    for (int64_t b = 0; b < blocks; ++b) {                                     \
      const int64_t bs = b * wpb, be = MIN(bs + wpb, tiles);                   \
      const int64_t x_bs = tile_x[bs];                                         \
      const int64_t y_bs = tile_y[bs] & 0x7FFFFFFFu;                           \
      const int64_t y_be = tile_y[be] & 0x7FFFFFFFu;                           \
      const int64_t m_b = (int64_t)tile_x[be] - x_bs;                          \
      const int64_t y_se = y_be - y_bs;                                        \
      T* products = scratch;                                                   \
      T* partials = scratch + m_b;                                             \
      for (int64_t r = 0; r <= y_se; ++r) partials[r] = (T)0;                  \
      for (int64_t i = bs; i < be; ++i) {                                      \
        const int64_t x_ws = tile_x[i], x_se = (int64_t)tile_x[i + 1] - x_ws;  \
        if (x_se == 0) { ++skipped; continue; }                                \
        const uint32_t ty = tile_y[i];                                         \
        const int64_t y_bw = (int64_t)(ty & 0x7FFFFFFFu) - y_bs;               \
        const int64_t x_bw = x_ws - x_bs;                                      \
        if (ty & 0x80000000u) {                                                \
          for (int64_t s = 0; s < width; ++s) sub[s] = (T)0;                   \
          for (int lid = 0; lid < omega; ++lid) {                              \
            T acc = (T)0;                                                      \
            for (int64_t k = lid; k < x_se; k += omega)                        \
              acc += vals[x_ws + k] * x[cols[x_ws + k]];                       \
            sub[lid] = acc;                                                    \
          }                                                                    \
          for (int64_t st = width / 2; st >= 1; st /= 2)                       \
            for (int64_t k = 0; k < st; ++k) sub[k] += sub[k + st];            \
          partials[y_bw] += sub[0];                                            \
          ++fast;                                                              \
          continue;                                                            \
        }                                                                      \
        ++normal;                                                              \
        for (int64_t k = 0; k < x_se; ++k)                                     \
          products[x_bw + k] = vals[x_ws + k] * x[cols[x_ws + k]];             \
        for (int lid = 0; lid < omega; ++lid) {                                \
          const int64_t j = i * omega + lid;                                   \
          if (j >= lanes) {                                                    \
            lane_sum[lid] = (T)0; lane_row[lid] = 0; lane_flag[lid] = 1;       \
            continue;                                                          \
          }                                                                    \
          const uint32_t d = lane_desc[j];                                     \
          const uint32_t flags = d >> (2 * ob);                                \
          const int64_t steps = MIN((int64_t)sigma, total - j * sigma);        \
          int64_t xo = d & mask, yo = (d >> ob) & mask;                        \
          T sum = (T)0;                                                        \
          int first = 1, flag = lid == 0;                                      \
          for (int64_t k = 0; k < steps; ++k) {                                \
            if ((flags >> k) & 1u) {                                           \
              if (first) { partials[y_bw + yo] += sum; first = 0; }            \
              else partials[y_bw + yo] = sum;                                  \
              sum = (T)0; ++yo; flag = 1;                                      \
            } else {                                                           \
              sum += products[x_bw + xo]; ++xo;                                \
            }                                                                  \
          }                                                                    \
          lane_sum[lid] = sum; lane_row[lid] = yo; lane_flag[lid] = (uint8_t)flag; \
        }                                                                      \
        for (int l = 0; l < omega; ++l) {                                      \
          run_sum[l] = lane_sum[l]; run_flag[l] = lane_flag[l];                \
        }                                                                      \
        for (int off = 1; off < omega; off <<= 1) {                            \
          int all = 1;                                                         \
          for (int l = 0; l < omega; ++l) if (!run_flag[l]) { all = 0; break; } \
          if (all) break;                                                      \
          for (int l = 0; l < omega; ++l) {                                    \
            const int src = l >= off ? l - off : l;                            \
            tmp_sum[l] = run_sum[src]; tmp_flag[l] = run_flag[src];            \
          }                                                                    \
          for (int l = 0; l < omega; ++l)                                      \
            if (l >= off && !run_flag[l]) {                                    \
              run_sum[l] += tmp_sum[l]; run_flag[l] = tmp_flag[l];             \
            }                                                                  \
        }                                                                      \
        for (int l = 0; l < omega; ++l) {                                      \
          if (!lane_flag[l]) continue;                                         \
          const int src = l == 0 ? omega - 1 : l - 1;                          \
          partials[y_bw + lane_row[src]] += run_sum[src];                      \
        }                                                                      \
      }                                                                        \
      if (y_se == 0) {                                                         \
        ccount[b] = 1; crow[2 * b] = y_bs; csum[2 * b] = partials[0];          \
      } else {                                                                 \
        ccount[b] = 2; crow[2 * b] = y_bs; csum[2 * b] = partials[0];          \
        for (int64_t r = 1; r < y_se; ++r) y[y_bs + r] = partials[r];          \
        crow[2 * b + 1] = y_be; csum[2 * b + 1] = partials[y_se];              \
      }                                                                        \
    }                                                                          \
    for (int64_t b = 0; b < blocks; ++b)                                       \
      for (int e = 0; e < ccount[b]; ++e)                                      \
        if (crow[2 * b + e] < n_rows) y[crow[2 * b + e]] += csum[2 * b + e];   \
    if (counters) { counters[0] = fast; counters[1] = normal; counters[2] = skipped; } \
    free(scratch); free(sub); free(lane_sum); free(run_sum); free(tmp_sum);    \
    free(lane_row); free(lane_flag); free(run_flag); free(tmp_flag);           \
    free(ccount); free(crow); free(csum);                                      \
    return MO_OK;                                                              \
  }

DEFINE_MERBIT(double, mo_spmv_merbit_f64)
DEFINE_MERBIT(float, mo_spmv_merbit_f32)

/* ========================================================================
 * PageRank -- include/merbit/solvers.hpp:36-218
 * ======================================================================== */
#define DEFINE_TRANSITION(T, NAME)                                             \
  void NAME(int64_t n, const int64_t* adj_ro, const int32_t* adj_cols,         \
            int64_t* p_ro, int32_t* p_cols, T* p_vals) {                       \
    const int64_t nnz = adj_ro[n];                                             \
    for (int64_t i = 0; i <= n; ++i) p_ro[i] = 0;                              \
    for (int64_t k = 0; k < nnz; ++k) ++p_ro[adj_cols[k] + 1];                 \
    for (int64_t i = 0; i < n; ++i) p_ro[i + 1] += p_ro[i];                    \
    int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)MAX(n, 1));   \
    for (int64_t i = 0; i < n; ++i) cursor[i] = p_ro[i];                       \
    for (int64_t j = 0; j < n; ++j) {                                          \
      const int64_t b = adj_ro[j], e = adj_ro[j + 1];                          \
      const T w = e > b ? (T)1 / (T)(e - b) : (T)0;                            \
      for (int64_t k = b; k < e; ++k) {                                        \
        const int64_t s = cursor[adj_cols[k]]++;                               \
        p_cols[s] = (int32_t)j;                                                \
        p_vals[s] = w;                                                         \
      }                                                                        \
    }                                                                          \
    free(cursor);                                                              \
  }

DEFINE_TRANSITION(double, mo_build_transition_f64)
DEFINE_TRANSITION(float, mo_build_transition_f32)

static uint8_t* dangling_flags(int64_t n, const int64_t* ro, const int32_t* cols) {
  uint8_t* seen = (uint8_t*)calloc((size_t)MAX(n, 1), 1);
  for (int64_t k = 0; k < ro[n]; ++k) seen[cols[k]] = 1;
  return seen; /* seen[j] == 0 <=> column j dangling (solvers.hpp:133-145) */
}

static double rank_error_f64(int64_t n, const double* pi, const double* star) {
  double err = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double s = star[i], d = pi[i] - s;
    if (s == 0.0) {
      if (d != 0.0) return INFINITY;
      continue;
    }
    err = MAX(err, fabs(d / s));
  }
  return err;
}

int mo_pagerank_f64(int64_t n, const int64_t* ro, const int32_t* cols,
                    const double* vals, double damping, double err_tol,
                    int64_t max_iters, int64_t reference_iters, double* pi_out,
                    double* ref_out, int64_t* iterations, double* final_err,
                    int* status, int nthreads) {
  if (n < 1) return MO_ERR_DIMENSION;
  if (!(damping >= 0.0 && damping <= 1.0)) return MO_ERR_CONFIG;
  if (!(err_tol > 0.0)) return MO_ERR_CONFIG;
  uint8_t* seen = dangling_flags(n, ro, cols);
  double* pi = (double*)malloc(sizeof(double) * n);
  double* w = (double*)malloc(sizeof(double) * n);
  double* star = ref_out;
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t i = 0; i < n; ++i) pi[i] = 1.0 / (double)n;
    const int64_t iters = pass == 0 ? reference_iters : max_iters;
    if (pass == 1) {
      *iterations = 0;
      *final_err = INFINITY;
      *status = 1;
    }
    for (int64_t r = 1; r <= iters; ++r) {
      mo_spmv_csr_f64(n, ro, cols, vals, pi, w, NULL, nthreads);
      double dm = 0.0; /* sequential dangling sum (solvers.hpp:104-107) */
      for (int64_t j = 0; j < n; ++j)
        if (!seen[j]) dm += pi[j];
      const double base = (damping * dm + (1.0 - damping)) / (double)n;
      for (int64_t i = 0; i < n; ++i) pi[i] = damping * w[i] + base;
      if (pass == 0) continue;
      double mass = 0.0;
      for (int64_t i = 0; i < n; ++i) mass += fabs(pi[i]);
      if (mass == 0.0) {
        free(seen); free(pi); free(w);
        return MO_ERR;
      }
      *iterations = r;
      *final_err = rank_error_f64(n, pi, star);
      if (*final_err < err_tol) {
        *status = 0;
        break;
      }
    }
    if (pass == 0) memcpy(star, pi, sizeof(double) * n);
  }
  memcpy(pi_out, pi, sizeof(double) * n);
  free(seen); free(pi); free(w);
  return MO_OK;
}

int mo_pagerank_f32(int64_t n, const int64_t* ro, const int32_t* cols,
                    const float* vals, float damping, float err_tol,
                    int64_t max_iters, int64_t reference_iters, float* pi_out,
                    float* ref_out, int64_t* iterations, double* final_err,
                    int* status) {
  if (n < 1) return MO_ERR_DIMENSION;
  if (!(damping >= 0.0f && damping <= 1.0f)) return MO_ERR_CONFIG;
  if (!(err_tol > 0.0f)) return MO_ERR_CONFIG;
  uint8_t* seen = dangling_flags(n, ro, cols);
  float* pi = (float*)malloc(sizeof(float) * n);
  float* w = (float*)malloc(sizeof(float) * n);
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t i = 0; i < n; ++i) pi[i] = 1.0f / (float)n;
    const int64_t iters = pass == 0 ? reference_iters : max_iters;
    if (pass == 1) {
      *iterations = 0;
      *final_err = INFINITY;
      *status = 1;
    }
    for (int64_t r = 1; r <= iters; ++r) {
      mo_spmv_csr_f32(n, ro, cols, vals, pi, w);
      float dm = 0.0f;
      for (int64_t j = 0; j < n; ++j)
        if (!seen[j]) dm += pi[j];
      const float base = (damping * dm + (1.0f - damping)) / (float)n;
      for (int64_t i = 0; i < n; ++i) pi[i] = damping * w[i] + base;
      if (pass == 0) continue;
      float mass = 0.0f;
      for (int64_t i = 0; i < n; ++i) mass += fabsf(pi[i]);
      if (mass == 0.0f) {
        free(seen); free(pi); free(w);
        return MO_ERR;
      }
      *iterations = r;
      double err = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        const double s = ref_out[i], d = (double)pi[i] - s;
        if (s == 0.0) {
          if (d != 0.0) { err = INFINITY; break; }
          continue;
        }
        err = MAX(err, fabs(d / s));
      }
      *final_err = err;
      if (err < (double)err_tol) {
        *status = 0;
        break;
      }
    }
    if (pass == 0) memcpy(ref_out, pi, sizeof(float) * n);
  }
  memcpy(pi_out, pi, sizeof(float) * n);
  free(seen); free(pi); free(w);
  return MO_OK;
}

/* ========================================================================
 * fixtures -- mt19937_64 (std), random.hpp:14-31, fixtures.hpp:60-111,
 * tests/support/generators.hpp:49-130, csr.hpp:43-89
 * ======================================================================== */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) |
                         (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

static double mt_unit(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
static double mt_uniform_in(mt64* g, double lo, double hi) {
  return lo + (hi - lo) * mt_unit(g);
}

void mo_seed_test_vector(int64_t n, double lo, double hi, uint64_t seed,
                         double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = mt_uniform_in(&g, lo, hi);
}

typedef struct {
  int64_t row, col, ord;
  double value;
} coo_e;

typedef struct {
  int64_t n_rows, n_cols, size, cap;
  coo_e* e;
} coo_t;

static void coo_push(coo_t* c, int64_t r, int64_t col, double v) {
  if (c->size == c->cap) {
    c->cap = c->cap ? c->cap * 2 : 1024;
    c->e = (coo_e*)realloc(c->e, sizeof(coo_e) * (size_t)c->cap);
  }
  c->e[c->size] = (coo_e){r, col, c->size, v};
  c->size++;
}

static int coo_cmp(const void* a, const void* b) {
  const coo_e* x = (const coo_e*)a;
  const coo_e* y = (const coo_e*)b;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return x->ord < y->ord ? -1 : (x->ord > y->ord);
}

/* normalize_coo + coo_to_csr: stable row-major sort, duplicates summed in
 * insertion order in double (csr.hpp:43-89). */
static int coo_to_csr(coo_t* c, int64_t* nnz, int64_t** ro, int32_t** cols,
                      double** vals) {
  qsort(c->e, (size_t)c->size, sizeof(coo_e), coo_cmp);
  int64_t m = 0;
  for (int64_t k = 0; k < c->size; ++k) {
    if (m > 0 && c->e[m - 1].row == c->e[k].row && c->e[m - 1].col == c->e[k].col)
      c->e[m - 1].value += c->e[k].value;
    else
      c->e[m++] = c->e[k];
  }
  *nnz = m;
  *ro = (int64_t*)calloc((size_t)c->n_rows + 1, sizeof(int64_t));
  *cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)MAX(m, 1));
  *vals = (double*)malloc(sizeof(double) * (size_t)MAX(m, 1));
  for (int64_t k = 0; k < m; ++k) {
    ++(*ro)[c->e[k].row + 1];
    (*cols)[k] = (int32_t)c->e[k].col;
    (*vals)[k] = c->e[k].value;
  }
  for (int64_t r = 0; r < c->n_rows; ++r) (*ro)[r + 1] += (*ro)[r];
  free(c->e);
  c->e = NULL;
  return MO_OK;
}

int mo_random_matrix_csr(int shape, uint64_t seed, int64_t* n_rows,
                         int64_t* n_cols, int64_t* nnz, int64_t** ro,
                         int32_t** cols, double** vals) {
  mt64 g;
  mt64_seed(&g, seed);
#define PICK(bound) ((int64_t)(mt64_next(&g) % (uint64_t)(bound)))
  coo_t c = {0, 0, 0, 0, NULL};
  c.n_rows = 1 + PICK(512);
  c.n_cols = 1 + PICK(512);
  int64_t target = PICK(MIN((int64_t)20000, c.n_rows * c.n_cols));
  switch (shape) {
    case 0: /* uniform */
      for (int64_t k = 0; k < target; ++k) {
        const int64_t r = PICK(c.n_rows);
        const int64_t cc = PICK(c.n_cols);
        coo_push(&c, r, cc, mt_uniform_in(&g, -1.0, 1.0));
      }
      break;
    case 1: { /* power_law_rows */
      double wsum = 0.0;
      for (int64_t r = 0; r < c.n_rows; ++r) wsum += 1.0 / (double)(r + 1);
      for (int64_t r = 0; r < c.n_rows && target > 0; ++r) {
        const double share = (1.0 / (double)(r + 1)) / wsum;
        int64_t len = (int64_t)llround(share * (double)target);
        len = MIN(len, c.n_cols);
        for (int64_t k = 0; k < len; ++k) {
          const int64_t cc = PICK(c.n_cols);
          coo_push(&c, r, cc, mt_uniform_in(&g, -1.0, 1.0));
        }
      }
      break;
    }
    case 2: { /* banded */
      const int64_t hb = 1 + PICK(8);
      for (int64_t r = 0; r < c.n_rows; ++r) {
        const int64_t center =
            c.n_cols <= 1 ? 0 : (r * (c.n_cols - 1)) / MAX(c.n_rows - 1, (int64_t)1);
        for (int64_t d = -hb; d <= hb; ++d) {
          const int64_t cc = center + d;
          if (cc >= 0 && cc < c.n_cols) coo_push(&c, r, cc, mt_uniform_in(&g, -1.0, 1.0));
        }
      }
      break;
    }
    case 3: { /* single_dense_row */
      const int64_t hub = PICK(c.n_rows);
      target = MIN((int64_t)20000, c.n_cols * 4);
      for (int64_t k = 0; k < target; ++k) {
        const int64_t cc = PICK(c.n_cols);
        coo_push(&c, hub, cc, mt_uniform_in(&g, -1.0, 1.0));
      }
      for (int64_t k = 0; k < MIN(c.n_rows, (int64_t)32); ++k) {
        const int64_t r = PICK(c.n_rows);
        const int64_t cc = PICK(c.n_cols);
        coo_push(&c, r, cc, mt_uniform_in(&g, -1.0, 1.0));
      }
      break;
    }
    case 4: /* all_empty */
      break;
    case 5: { /* mostly_empty_rows */
      const int64_t live = MAX((int64_t)1, c.n_rows / 10);
      for (int64_t k = 0; k < target; ++k) {
        const int64_t r = (PICK(live) * MAX(c.n_rows / live, (int64_t)1)) % c.n_rows;
        const int64_t cc = PICK(c.n_cols);
        coo_push(&c, r, cc, mt_uniform_in(&g, -1.0, 1.0));
      }
      break;
    }
    default:
      return MO_ERR_CONFIG;
  }
#undef PICK
  *n_rows = c.n_rows;
  *n_cols = c.n_cols;
  return coo_to_csr(&c, nnz, ro, cols, vals);
}

int mo_ring_with_chords_csr(int64_t n, int64_t extra, uint64_t seed,
                            int64_t* nnz, int64_t** ro, int32_t** cols,
                            double** vals) {
  coo_t c = {n, n, 0, 0, NULL};
  for (int64_t i = 0; i < n; ++i) coo_push(&c, i, (i + 1) % n, 1.0);
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t e = 0; e < extra; ++e) {
    const int64_t from = (int64_t)(mt64_next(&g) % (uint64_t)n);
    const int64_t to = (int64_t)(mt64_next(&g) % (uint64_t)n);
    if (from == to) continue;
    coo_push(&c, from, to, 1.0);
  }
  return coo_to_csr(&c, nnz, ro, cols, vals);
}

int mo_single_dense_row_csr(int64_t width, uint64_t seed, int64_t** ro,
                            int32_t** cols, double** vals) {
  *ro = (int64_t*)malloc(sizeof(int64_t) * 2);
  (*ro)[0] = 0;
  (*ro)[1] = width;
  *cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)MAX(width, 1));
  *vals = (double*)malloc(sizeof(double) * (size_t)MAX(width, 1));
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t k = 0; k < width; ++k) {
    (*cols)[k] = (int32_t)k;
    (*vals)[k] = mt_uniform_in(&g, 0.5, 1.5);
  }
  return MO_OK;
}

/* ========================================================================
 * counter-based synthetic inputs (bit-identical to csrc/generators.cu)
 * ======================================================================== */
static inline uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* thresholds floor(p * 2^53) for cumulative (a, a+b, a+b+c) */
#define RMAT_T1 5134103575202365ULL
#define RMAT_T2 6845471433603153ULL
#define RMAT_T3 8556839292003942ULL

static inline uint64_t rmat_key(uint64_t seedmix, int scale, uint64_t e,
                                int transposed) {
  uint64_t src = 0, dst = 0;
  for (int l = 0; l < scale; ++l) {
    const uint64_t u = smix(seedmix ^ ((e << 6) | (uint64_t)l)) >> 11;
    const uint64_t bit = 1ULL << (scale - 1 - l);
    if (u < RMAT_T1) {
    } else if (u < RMAT_T2) {
      dst |= bit;
    } else if (u < RMAT_T3) {
      src |= bit;
    } else {
      src |= bit;
      dst |= bit;
    }
  }
  return transposed ? (dst << scale) | src : (src << scale) | dst;
}

typedef struct {
  uint64_t* keys;
  uint64_t e0, e1, seedmix;
  int scale, transposed;
} key_job;

static void* key_worker(void* arg) {
  key_job* j = (key_job*)arg;
  for (uint64_t e = j->e0; e < j->e1; ++e)
    j->keys[e] = rmat_key(j->seedmix, j->scale, e, j->transposed);
  return NULL;
}

static void radix_sort_u64(uint64_t* a, uint64_t* tmp, uint64_t n, int bits) {
  const int D = 11;
  uint64_t* src = a;
  uint64_t* dst = tmp;
  int passes = 0;
  for (int shift = 0; shift < bits; shift += D) {
    static uint64_t cnt[1 << 11];
    memset(cnt, 0, sizeof(cnt));
    for (uint64_t i = 0; i < n; ++i) ++cnt[(src[i] >> shift) & ((1u << D) - 1)];
    uint64_t s = 0;
    for (int b = 0; b < (1 << D); ++b) {
      const uint64_t c = cnt[b];
      cnt[b] = s;
      s += c;
    }
    for (uint64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & ((1u << D) - 1)]++] = src[i];
    uint64_t* t = src;
    src = dst;
    dst = t;
    ++passes;
  }
  if (passes & 1) memcpy(a, src, sizeof(uint64_t) * n);
}

int mo_rmat_csr(int scale, int edge_factor, uint64_t seed, int transposed,
                int nthreads, int64_t* nnz, int64_t** ro, int32_t** cols) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return MO_ERR_CONFIG;
  const uint64_t n = 1ULL << scale;
  const uint64_t m_raw = (uint64_t)edge_factor << scale;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * m_raw);
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * m_raw);
  if (!keys || !tmp) {
    free(keys);
    free(tmp);
    return MO_ERR;
  }
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  key_job jobs[256];
  const uint64_t seedmix = smix(seed);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (key_job){keys, m_raw * t / nthreads, m_raw * (t + 1) / nthreads,
                        seedmix, scale, transposed};
    if (t) pthread_create(&th[t], NULL, key_worker, &jobs[t]);
  }
  key_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  radix_sort_u64(keys, tmp, m_raw, 2 * scale);
  free(tmp);
  uint64_t m = 0;
  for (uint64_t i = 0; i < m_raw; ++i)
    if (m == 0 || keys[m - 1] != keys[i]) keys[m++] = keys[i];
  *nnz = (int64_t)m;
  *ro = (int64_t*)calloc(n + 1, sizeof(int64_t));
  *cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)MAX(m, 1));
  const uint64_t cmask = (1ULL << scale) - 1;
  for (uint64_t k = 0; k < m; ++k) {
    ++(*ro)[(keys[k] >> scale) + 1];
    (*cols)[k] = (int32_t)(keys[k] & cmask);
  }
  for (uint64_t r = 0; r < n; ++r) (*ro)[r + 1] += (*ro)[r];
  free(keys);
  return MO_OK;
}

void mo_hash_uniform(uint64_t seed, int64_t count, double lo, double hi,
                     double* out) {
  const uint64_t sm = smix(seed);
  for (int64_t k = 0; k < count; ++k)
    out[k] = lo + (hi - lo) * ((double)(smix(sm ^ (uint64_t)k) >> 11) * 0x1.0p-53);
}

void mo_hash_uniform_f32(uint64_t seed, int64_t count, double lo, double hi,
                         float* out) {
  const uint64_t sm = smix(seed);
  for (int64_t k = 0; k < count; ++k)
    out[k] = (float)(lo + (hi - lo) *
                              ((double)(smix(sm ^ (uint64_t)k) >> 11) * 0x1.0p-53));
}

#define DEFINE_TVALS(T, NAME)                                                  \
  void NAME(int64_t n, int64_t nnz, const int32_t* cols, T* vals) {            \
    int64_t* deg = (int64_t*)calloc((size_t)MAX(n, 1), sizeof(int64_t));       \
    for (int64_t k = 0; k < nnz; ++k) ++deg[cols[k]];                          \
    for (int64_t k = 0; k < nnz; ++k) vals[k] = (T)1 / (T)deg[cols[k]];        \
    free(deg);                                                                 \
  }

DEFINE_TVALS(float, mo_transition_values_f32)
DEFINE_TVALS(double, mo_transition_values_f64)

/* ========================================================================
 * bicgstab over the csr backend -- include/merbit/solvers.hpp:268-373
 * (dot: sequential sum in T, 243-248; norm2: fp64, 250-255).  status: 0
 * converged, 1 max_iterations, 2 breakdown; reason 1 rho, 2 rhat_dot_v,
 * 3 t_dot_t, 4 omega, 5 diverged.
 * ======================================================================== */
#define MO_BICGSTAB(T, SUFFIX, SPMV)                                              \
  static T mo_dot_##SUFFIX(int64_t n, const T* a, const T* b) {                  \
    T s = (T)0;                                                                   \
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];                             \
    return s;                                                                     \
  }                                                                               \
  int mo_bicgstab_##SUFFIX(int64_t n, const int64_t* ro, const int32_t* cols,    \
                           const T* vals, const T* b, T tol, int64_t max_iters,   \
                           T* x, double* hist, int64_t* iterations,               \
                           double* final_residual, int* status, int* reason) {    \
    double bb = 0.0;                                                              \
    for (int64_t i = 0; i < n; ++i) bb += (double)b[i] * (double)b[i];            \
    const double b_norm = sqrt(bb);                                               \
    for (int64_t i = 0; i < n; ++i) x[i] = (T)0;                                  \
    *iterations = 0;                                                              \
    *final_residual = INFINITY;                                                   \
    *status = 1;                                                                  \
    *reason = 0;                                                                  \
    if (b_norm == 0.0) {                                                          \
      *status = 0;                                                                \
      *final_residual = 0.0;                                                      \
      return MO_OK;                                                               \
    }                                                                             \
    T* r = (T*)malloc(sizeof(T) * (n + 1));                                       \
    T* rh = (T*)malloc(sizeof(T) * (n + 1));                                      \
    T* p = (T*)calloc(n + 1, sizeof(T));                                          \
    T* v = (T*)calloc(n + 1, sizeof(T));                                          \
    T* s = (T*)calloc(n + 1, sizeof(T));                                          \
    T* t = (T*)calloc(n + 1, sizeof(T));                                          \
    T* ax = (T*)calloc(n + 1, sizeof(T));                                         \
    memcpy(r, b, sizeof(T) * n);                                                  \
    memcpy(rh, b, sizeof(T) * n);                                                 \
    T rho = (T)1, alpha = (T)1, omega = (T)1;                                     \
    for (int64_t iter = 1; iter <= max_iters; ++iter) {                           \
      const T rho_new = mo_dot_##SUFFIX(n, rh, r);                                \
      if (rho_new == (T)0 || !isfinite((double)rho_new)) {                        \
        *status = 2; *reason = 1; *iterations = iter; break;                      \
      }                                                                           \
      if (iter == 1) {                                                            \
        memcpy(p, r, sizeof(T) * n);                                              \
      } else {                                                                    \
        const T beta = (rho_new / rho) * (alpha / omega);                         \
        for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]); \
      }                                                                           \
      SPMV(n, ro, cols, vals, p, v);                                              \
      const T rhat_v = mo_dot_##SUFFIX(n, rh, v);                                 \
      if (rhat_v == (T)0 || !isfinite((double)rhat_v)) {                          \
        *status = 2; *reason = 2; *iterations = iter; break;                      \
      }                                                                           \
      alpha = rho_new / rhat_v;                                                   \
      for (int64_t i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];                 \
      SPMV(n, ro, cols, vals, s, t);                                              \
      const T t_t = mo_dot_##SUFFIX(n, t, t);                                     \
      if (t_t == (T)0 || !isfinite((double)t_t)) {                                \
        *status = 2; *reason = 3; *iterations = iter; break;                      \
      }                                                                           \
      omega = mo_dot_##SUFFIX(n, t, s) / t_t;                                     \
      if (omega == (T)0 || !isfinite((double)omega)) {                            \
        *status = 2; *reason = 4; *iterations = iter; break;                      \
      }                                                                           \
      for (int64_t i = 0; i < n; ++i) {                                           \
        x[i] += alpha * p[i] + omega * s[i];                                      \
        r[i] = s[i] - omega * t[i];                                               \
      }                                                                           \
      rho = rho_new;                                                              \
      SPMV(n, ro, cols, vals, x, ax);                                             \
      double rr = 0.0;                                                            \
      for (int64_t i = 0; i < n; ++i) {                                           \
        const double d = (double)ax[i] - (double)b[i];                            \
        rr += d * d;                                                              \
      }                                                                           \
      const double resid = sqrt(rr) / b_norm;                                     \
      if (hist) hist[iter - 1] = resid;                                           \
      *iterations = iter;                                                         \
      *final_residual = resid;                                                    \
      if (!isfinite(resid)) { *status = 2; *reason = 5; break; }                  \
      if (resid < (double)tol) { *status = 0; break; }                            \
    }                                                                             \
    free(r); free(rh); free(p); free(v); free(s); free(t); free(ax);              \
    return MO_OK;                                                                 \
  }

static void mo_spmv_ref_f64(int64_t n, const int64_t* ro, const int32_t* cols,
                            const double* vals, const double* x, double* y) {
  mo_spmv_csr_f64(n, ro, cols, vals, x, y, NULL, 1);
}
static void mo_spmv_ref_f32(int64_t n, const int64_t* ro, const int32_t* cols,
                            const float* vals, const float* x, float* y) {
  mo_spmv_csr_f32(n, ro, cols, vals, x, y);
}
MO_BICGSTAB(double, f64, mo_spmv_ref_f64)
MO_BICGSTAB(float, f32, mo_spmv_ref_f32)
