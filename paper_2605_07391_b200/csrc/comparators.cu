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
//   kind 4-7 cuSPARSE      cusparseSpMV: COO ALG1, COO ALG2, CSR ALG1, CSR
//                          ALG2 -- the paper's own baseline (PAPER.md:32,
//                          494-496: speedups are quoted against cuSPARSE COO).
//                          libcusparse is resolved with dlopen at first use so
//                          the library itself links nothing but the runtime;
//                          the descriptors and the work buffer (and the ALG2
//                          preprocessing) are built once per matrix and kind.
//
// No preprocessing is cached by kinds 0, 2, 3; kind 1 expands the row
// indices once per matrix (the COO row array).
#define CUB_IGNORE_DEPRECATED_API 1
#include <cub/cub.cuh>

#include <cusparse.h>
#include <dlfcn.h>

#include <mutex>
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


// ---- cuSPARSE (dlopen) ------------------------------------------------------
struct SparseApi {
  decltype(&cusparseCreate) create = nullptr;
  decltype(&cusparseDestroy) destroy = nullptr;
  decltype(&cusparseSetStream) set_stream = nullptr;
  decltype(&cusparseCreateCoo) create_coo = nullptr;
  decltype(&cusparseCreateCsr) create_csr = nullptr;
  decltype(&cusparseDestroySpMat) destroy_spmat = nullptr;
  decltype(&cusparseCreateDnVec) create_dnvec = nullptr;
  decltype(&cusparseDestroyDnVec) destroy_dnvec = nullptr;
  decltype(&cusparseDnVecSetValues) dnvec_set = nullptr;
  decltype(&cusparseSpMV_bufferSize) buffer_size = nullptr;
  decltype(&cusparseSpMV) spmv = nullptr;
  decltype(&cusparseSpMV_preprocess) preprocess = nullptr;  // optional
  std::string error;
};

const SparseApi& sparse_api() {
  static SparseApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libcusparse.so.12", "/usr/local/cuda/lib64/libcusparse.so.12",
                             "libcusparse.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) {
      api.error = "cuSPARSE comparator: libcusparse.so.12 not found";
      return;
    }
    auto sym = [&](auto& fn, const char* name, bool required = true) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && required && api.error.empty())
        api.error = std::string("cuSPARSE comparator: missing ") + name;
    };
    sym(api.create, "cusparseCreate");
    sym(api.destroy, "cusparseDestroy");
    sym(api.set_stream, "cusparseSetStream");
    sym(api.create_coo, "cusparseCreateCoo");
    sym(api.create_csr, "cusparseCreateCsr");
    sym(api.destroy_spmat, "cusparseDestroySpMat");
    sym(api.create_dnvec, "cusparseCreateDnVec");
    sym(api.destroy_dnvec, "cusparseDestroyDnVec");
    sym(api.dnvec_set, "cusparseDnVecSetValues");
    sym(api.buffer_size, "cusparseSpMV_bufferSize");
    sym(api.spmv, "cusparseSpMV");
    sym(api.preprocess, "cusparseSpMV_preprocess", false);
  });
  if (!api.error.empty()) fail(MBX_UNSUPPORTED, api.error);
  return api;
}

#define MBX_SPARSE(call)                                                              \
  do {                                                                                \
    const cusparseStatus_t st_ = (call);                                              \
    if (st_ != CUSPARSE_STATUS_SUCCESS)                                               \
      fail(MBX_CUDA_ERROR, "cuSPARSE status " + std::to_string(int(st_)) + " in " #call); \
  } while (0)

}  // namespace

struct SparseState {
  cusparseSpMatDescr_t mat = nullptr;
  cusparseDnVecDescr_t vx = nullptr, vy = nullptr;
  void* buffer = nullptr;
};

void free_sparse_state(mbx_context* ctx, const mbx_matrix* m) {
  for (SparseState*& s : m->sparse) {
    if (!s) continue;
    const SparseApi& api = sparse_api();
    if (s->mat) api.destroy_spmat(s->mat);
    if (s->vx) api.destroy_dnvec(s->vx);
    if (s->vy) api.destroy_dnvec(s->vy);
    if (s->buffer) cudaFreeAsync(s->buffer, ctx->stream);
    delete s;
    s = nullptr;
  }
}

void free_sparse_handle(mbx_context* ctx) {
  if (ctx->cusparse) {
    sparse_api().destroy(static_cast<cusparseHandle_t>(ctx->cusparse));
    ctx->cusparse = nullptr;
  }
}

namespace {

// kinds 4..7: cusparseSpMV with COO ALG1 / COO ALG2 / CSR ALG1 / CSR ALG2
void launch_cusparse(mbx_context* ctx, const mbx_matrix* m, int kind, const void* x, void* y) {
  const SparseApi& api = sparse_api();
  if (m->nnz >= (int64_t(1) << 31))
    fail(MBX_CAPACITY_ERROR, "cuSPARSE comparator: 32-bit indices need nnz < 2^31");
  cudaStream_t s = ctx->stream;
  if (m->n_rows == 0) return;
  if (m->nnz == 0) {  // cuSPARSE rejects empty matrices: y = 0
    MBX_CUDA(cudaMemsetAsync(y, 0, m->n_rows * value_size(m->precision), s));
    return;
  }
  if (!ctx->cusparse) {
    cusparseHandle_t h;
    MBX_SPARSE(api.create(&h));
    ctx->cusparse = h;
  }
  cusparseHandle_t h = static_cast<cusparseHandle_t>(ctx->cusparse);
  MBX_SPARSE(api.set_stream(h, s));
  const bool coo = kind == 4 || kind == 5;
  const cusparseSpMVAlg_t alg = kind == 4   ? CUSPARSE_SPMV_COO_ALG1
                                : kind == 5 ? CUSPARSE_SPMV_COO_ALG2
                                : kind == 6 ? CUSPARSE_SPMV_CSR_ALG1
                                            : CUSPARSE_SPMV_CSR_ALG2;
  const cudaDataType dt = m->precision == MBX_F32 ? CUDA_R_32F : CUDA_R_64F;
  const double one64 = 1.0, zero64 = 0.0;
  const float one32 = 1.0f, zero32 = 0.0f;
  const void* alpha = m->precision == MBX_F32 ? static_cast<const void*>(&one32) : &one64;
  const void* beta = m->precision == MBX_F32 ? static_cast<const void*>(&zero32) : &zero64;
  SparseState*& st = m->sparse[kind - 4];
  if (!st) {
    if (coo && !m->coo_rows) {
      MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->coo_rows), m->nnz * 4 + 256, s));
      if (m->n_rows > 0) {
        expand_rows_kernel<<<unsigned(ctx->sm_count) * 16, 256, 0, s>>>(m->ro, m->n_rows,
                                                                        m->coo_rows);
        ++ctx->launches;
      }
    }
    auto ns = std::make_unique<SparseState>();
    if (coo)
      MBX_SPARSE(api.create_coo(&ns->mat, m->n_rows, m->n_cols, m->nnz, m->coo_rows, m->cols,
                                m->vals, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, dt));
    else
      MBX_SPARSE(api.create_csr(&ns->mat, m->n_rows, m->n_cols, m->nnz, m->ro, m->cols, m->vals,
                                CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO,
                                dt));
    MBX_SPARSE(api.create_dnvec(&ns->vx, m->n_cols, const_cast<void*>(x), dt));
    MBX_SPARSE(api.create_dnvec(&ns->vy, m->n_rows, y, dt));
    size_t bytes = 0;
    MBX_SPARSE(api.buffer_size(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, ns->mat, ns->vx, beta,
                               ns->vy, dt, alg, &bytes));
    MBX_CUDA(cudaMallocAsync(&ns->buffer, bytes > 0 ? bytes : 256, s));
    if (api.preprocess)
      MBX_SPARSE(api.preprocess(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, ns->mat, ns->vx, beta,
                                ns->vy, dt, alg, ns->buffer));
    st = ns.release();
  }
  MBX_SPARSE(api.dnvec_set(st->vx, const_cast<void*>(x)));
  MBX_SPARSE(api.dnvec_set(st->vy, y));
  MBX_SPARSE(api.spmv(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, st->mat, st->vx, beta, st->vy,
                      dt, alg, st->buffer));
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
    mbx::DeviceGuard dg(ctx->device);
    mbx::ensure_csr(ctx, m);
    if (kind == 0) {
      const int rc = mbx_spmv_csr_device(ctx, m, x, y);
      if (rc) mbx::fail(rc, mbx_last_error());
      return;
    }
    if (kind >= 4 && kind <= 7) {
      mbx::launch_cusparse(ctx, m, kind, x, y);
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
// the context stream): kind -1 = MERBIT (K2+K3 with the given TILE), 0..7 the
// comparators above.  x is uploaded once; warm-up launches are untimed.
MBX_API int mbx_bench_spmv(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                           const mbx_simt_config* c, int kind, int iters, int warmup,
                           const void* x_host, double* mean_seconds) {
  return mbx::cguard([&] {
    if (iters < 1) mbx::fail(MBX_CONFIG_ERROR, "--iters must be at least 1");
    mbx::DeviceGuard dg(ctx->device);
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
