// comparators.cu -- the paper's baselines on the same device (SURVEY 8f,
// row f2), so MERBIT's speedups are measured against GPU competitors and not
// only against the reference CPU path:
//
//   kind 0  csr_vector     warp per row, fp64 accumulation (csr_kernel in
//                          kernels.cu; the pagerank yardstick engine)
//   kind 1  coo_atomic     CooReferenceBackend (backend.hpp:67-84) on the GPU:
//                          thread per nonzero, warp-segmented pre-reduction of
//                          equal rows, one atomicAdd per row segment (the
//                          paper's "speedup vs COO" denominator)
//   kind 2  merge_runtime  MergeRuntimeBackend (merge_spmv.hpp:21-82): every
//                          lane binary-searches its own diagonal at multiply
//                          time, walks sigma steps against row_offsets, stores
//                          the rows it closes, and leaves a carry; carries are
//                          folded in ascending lane order (long runs by a warp)
//   kind 3  merge_cub      cub::DeviceSpmv::CsrMV (Merrill & Garland
//                          merge-path SpMV), library code, int32 offsets
//
// No preprocessing is cached by kinds 0, 2, 3; kind 1 expands the row
// indices once per matrix (the COO row array).
#define CUB_IGNORE_DEPRECATED_API 1
#include <cub/cub.cuh>

#include <string>

#include "mbx_internal.h"

namespace mbx {
namespace {

constexpr unsigned kFull = 0xffffffffu;

template <typename T>
__device__ __forceinline__ T mul_round(T a, T b);
template <>
__device__ __forceinline__ float mul_round<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_round<double>(double a, double b) {
  return __dmul_rn(a, b);
}

__global__ void expand_rows_kernel(const uint32_t* __restrict__ ro, int64_t n_rows,
                                   int32_t* __restrict__ rows) {
  // one warp per row: rows[k] = r for k in [ro[r], ro[r+1])
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lid = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w; r < n_rows; r += nw)
    for (uint32_t k = ro[r] + lid; k < ro[r + 1]; k += 32) rows[k] = int32_t(r);
}

template <typename T>
__global__ void __launch_bounds__(256)
    coo_atomic_kernel(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                      const T* __restrict__ vals, const T* __restrict__ x, T* __restrict__ y,
                      int64_t nnz) {
  const int lid = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nnz; base += stride) {
    const int64_t k = base + threadIdx.x;
    const bool ok = k < nnz;
    const int32_t r = ok ? rows[k] : -1;
    T p = ok ? mul_round(vals[k], __ldg(x + cols[k])) : T(0);
    // inclusive segmented scan over lanes of equal row (rows are sorted)
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const T u = __shfl_up_sync(kFull, p, off);
      const int32_t ru = __shfl_up_sync(kFull, r, off);
      if (lid >= off && ru == r) p += u;
    }
    const int32_t rn = __shfl_down_sync(kFull, r, 1);
    if (ok && (lid == 31 || rn != r)) atomicAdd(y + r, p);  // last lane of the segment
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
    merge_runtime_kernel(const uint32_t* __restrict__ ro, const int32_t* __restrict__ cols,
                         const T* __restrict__ vals, const T* __restrict__ x, T* __restrict__ y,
                         int64_t n, int64_t m, int sigma, int64_t lanes,
                         int64_t* __restrict__ carry_row, T* __restrict__ carry_val) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= lanes) return;
  const int64_t total = n + m;
  const int64_t diag = j * sigma;
  const int64_t steps = diag + sigma < total ? sigma : total - diag;
  // merge_search (merge_path.cpp:8-36), predicate of line 28
  int64_t lo = diag - m > 0 ? diag - m : 0, hi = diag < n ? diag : n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (int64_t(ro[mid + 1]) <= diag - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  int64_t px = diag - lo, py = lo < n ? lo : n;
  int64_t end = py < n ? int64_t(ro[py + 1]) : 0;
  T sum = T(0);
  for (int64_t k = 0; k < steps; ++k) {
    if (py < n && px < end) {
      sum += mul_round(vals[px], __ldg(x + cols[px]));
      ++px;
    } else {
      y[py] = sum;  // closes row py (a partial if the row began in an earlier lane)
      sum = T(0);
      ++py;
      end = py < n ? int64_t(ro[py + 1]) : 0;
    }
  }
  carry_row[j] = py;
  carry_val[j] = sum;
}

// y[row] += carries in ascending lane order (merge_spmv.hpp:74-79); a run of
// equal rows is folded by its first lane, runs longer than 32 lanes by the
// whole warp (lane-strided + butterfly)
template <typename T>
__global__ void __launch_bounds__(256)
    merge_fold_kernel(const int64_t* __restrict__ crow, const T* __restrict__ cval, int64_t lanes,
                      int64_t n, T* __restrict__ y) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lid = threadIdx.x & 31;
  int64_t r = -1;
  bool start = false, lng = false;
  T sum = T(0);
  if (e < lanes) {
    r = crow[e];
    start = r < n && (e == 0 || crow[e - 1] != r);
    if (start) {
      // y[r] += c_j one carry at a time, in lane order (the reference's fold)
      sum = y[r];
      int64_t k = e;
      const int64_t lim = e + 32 < lanes ? e + 32 : lanes;
      for (; k < lim && crow[k] == r; ++k) sum += cval[k];
      lng = k == lim && k < lanes && crow[k] == r;
    }
  }
  unsigned long_lanes = __ballot_sync(kFull, lng);
  while (long_lanes) {
    const int src = __ffs(long_lanes) - 1;
    long_lanes &= long_lanes - 1;
    const int64_t e0 = __shfl_sync(kFull, e, src);
    const int64_t rr = __shfl_sync(kFull, r, src);
    T part = T(0);
    for (int64_t w = e0;; w += 32) {
      const int64_t k = w + lid;
      const bool in = k < lanes && crow[k] == rr;
      if (in) part += cval[k];
      if (__ballot_sync(kFull, in) != kFull) break;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
    part = __shfl_sync(kFull, part, 0);
    if (lid == src) sum = y[rr] + part;
  }
  if (start) y[r] = sum;
}

template <typename T>
void launch_baseline_t(mbx_context* ctx, const mbx_matrix* m, int kind, int sigma, const T* x,
                       T* y) {
  cudaStream_t s = ctx->stream;
  const int64_t n = m->n_rows, nnz = m->nnz;
  const T* vals = static_cast<const T*>(m->vals);
  if (kind == 1) {
    if (!m->coo_rows) {
      MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->coo_rows), nnz * 4 + 256, s));
      if (n > 0) {
        expand_rows_kernel<<<unsigned(ctx->sm_count) * 16, 256, 0, s>>>(m->ro, n, m->coo_rows);
        ++ctx->launches;
      }
    }
    MBX_CUDA(cudaMemsetAsync(y, 0, n * sizeof(T), s));
    if (nnz > 0) {
      const int64_t blocks = std::min<int64_t>((nnz + 255) / 256, int64_t(ctx->sm_count) * 32);
      coo_atomic_kernel<T><<<unsigned(blocks), 256, 0, s>>>(m->coo_rows, m->cols, vals, x, y, nnz);
      ++ctx->launches;
    }
  } else if (kind == 2) {
    const int64_t total = n + nnz;
    if (total == 0) return;
    const int64_t lanes = (total + sigma - 1) / sigma;
    const size_t need = size_t(lanes) * (8 + sizeof(T)) + 512;
    char* ws = static_cast<char*>(scratch(ctx, need));
    int64_t* crow = reinterpret_cast<int64_t*>(ws);
    T* cval = reinterpret_cast<T*>(ws + ((size_t(lanes) * 8 + 255) / 256) * 256);
    const unsigned blocks = unsigned((lanes + 255) / 256);
    merge_runtime_kernel<T><<<blocks, 256, 0, s>>>(m->ro, m->cols, vals, x, y, n, nnz, sigma,
                                                   lanes, crow, cval);
    merge_fold_kernel<T><<<blocks, 256, 0, s>>>(crow, cval, lanes, n, y);
    ctx->launches += 2;
  } else if (kind == 3) {
    if (nnz >= (int64_t(1) << 31) || n >= (int64_t(1) << 31))
      fail(MBX_CAPACITY_ERROR, "merge_cub needs int32 row offsets (nnz < 2^31)");
    size_t tb = 0;
    const int* ro = reinterpret_cast<const int*>(m->ro);
    MBX_CUDA(cub::DeviceSpmv::CsrMV(nullptr, tb, vals, ro, m->cols, x, y, int(n),
                                    int(m->n_cols), int(nnz), s));
    void* temp = scratch(ctx, tb + 256);
    MBX_CUDA(cub::DeviceSpmv::CsrMV(temp, tb, vals, ro, m->cols, x, y, int(n), int(m->n_cols),
                                    int(nnz), s));
    ++ctx->launches;
  } else {
    fail(MBX_CONFIG_ERROR, "unknown baseline kind " + std::to_string(kind));
  }
  MBX_CUDA(cudaGetLastError());
}

template <typename F>
int cguard(F&& f) {
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
}  // namespace mbx

extern "C" {

MBX_API int mbx_spmv_baseline_device(mbx_context* ctx, const mbx_matrix* m, int kind, int sigma,
                                     const void* x, void* y) {
  return mbx::cguard([&] {
    MBX_CUDA(cudaSetDevice(ctx->device));
    if (kind == 0) {
      const int rc = mbx_spmv_csr_device(ctx, m, x, y);
      if (rc) mbx::fail(rc, mbx_last_error());
      return;
    }
    if (sigma < 1) mbx::fail(MBX_CONFIG_ERROR, "sigma must be >= 1");
    if (m->precision == MBX_F32)
      mbx::launch_baseline_t<float>(ctx, m, kind, sigma, static_cast<const float*>(x),
                                    static_cast<float*>(y));
    else
      mbx::launch_baseline_t<double>(ctx, m, kind, sigma, static_cast<const double*>(x),
                                     static_cast<double*>(y));
  });
}

// Device-resident timing of one multiply kind on this matrix (CUDA events on
// the context stream): kind -1 = MERBIT (K2+K3 with the given TILE), 0..3 the
// comparators above.  x is uploaded once; warm-up launches are untimed.
MBX_API int mbx_bench_spmv(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                           const mbx_simt_config* c, int kind, int iters, int warmup,
                           const void* x_host, double* mean_seconds) {
  return mbx::cguard([&] {
    if (iters < 1) mbx::fail(MBX_CONFIG_ERROR, "--iters must be at least 1");
    MBX_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t vs = mbx::value_size(m->precision);
    void *x = nullptr, *y = nullptr;
    MBX_CUDA(cudaMallocAsync(&x, m->n_cols * vs + 256, s));
    MBX_CUDA(cudaMallocAsync(&y, m->n_rows * vs + 256, s));
    if (m->n_cols) MBX_CUDA(cudaMemcpyAsync(x, x_host, m->n_cols * vs, cudaMemcpyHostToDevice, s));
    auto once = [&] {
      const int rc = kind < 0 ? mbx_spmv_device(ctx, m, t, c, x, y)
                              : mbx_spmv_baseline_device(ctx, m, kind, c->sigma, x, y);
      if (rc) mbx::fail(rc, mbx_last_error());
    };
    cudaEvent_t e0, e1;
    MBX_CUDA(cudaEventCreate(&e0));
    MBX_CUDA(cudaEventCreate(&e1));
    try {
      for (int i = 0; i < warmup; ++i) once();
      MBX_CUDA(cudaEventRecord(e0, s));
      for (int i = 0; i < iters; ++i) once();
      MBX_CUDA(cudaEventRecord(e1, s));
      MBX_CUDA(cudaEventSynchronize(e1));
    } catch (...) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaFreeAsync(x, s);
      cudaFreeAsync(y, s);
      throw;
    }
    float ms = 0.f;
    MBX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *mean_seconds = double(ms) * 1e-3 / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(x, s);
    cudaFreeAsync(y, s);
    MBX_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
