// cusparse_bench.cu -- the paper's comparator on B200:
// cuSPARSE SpMV (CSR ALG1/ALG2, COO ALG1/ALG2) against MERBIT (K2+K3 through
// the product C ABI) on the same device-resident matrices.  The paper reports
// MERBIT vs cuSPARSE COO speedups on an RTX 4090.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//   scripts/cusparse_bench.cu -o scripts/cusparse_bench -L paper_2605_07391_b200
//   -lmerbit_b200 -lcusparse -Xlinker -rpath,'$ORIGIN/../paper_2605_07391_b200'
#include <cuda_runtime.h>
#include <cusparse.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "merbit_b200.h"

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                    \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)
#define CS(x)                                                                        \
  do {                                                                               \
    cusparseStatus_t st_ = (x);                                                      \
    if (st_ != CUSPARSE_STATUS_SUCCESS) {                                            \
      printf("cuSPARSE %d at %d\n", int(st_), __LINE__);                             \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)
#define MB(x)                                                      \
  do {                                                             \
    if ((x) != 0) {                                                \
      printf("mbx error %s at %d\n", mbx_last_error(), __LINE__); \
      exit(1);                                                     \
    }                                                              \
  } while (0)

__global__ void expand_rows(const uint32_t* ro, int64_t n, int32_t* rows) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x)
    for (uint32_t k = ro[r]; k < ro[r + 1]; ++k) rows[k] = int32_t(r);
}

__global__ void fill_ones(void* x, int64_t n, int f64) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (f64)
      static_cast<double*>(x)[i] = 1.0 + 1e-3 * double(i & 1023);
    else
      static_cast<float*>(x)[i] = 1.0f + 1e-3f * float(i & 1023);
  }
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? atoi(argv[1]) : 24;
  const int f64 = argc > 2 ? atoi(argv[2]) : 0;
  const int kind = argc > 3 ? atoi(argv[3]) : 1;  // 1: PageRank transition, 0: adjacency
  mbx_context* ctx;
  MB(mbx_context_create(0, &ctx));
  cudaStream_t s = static_cast<cudaStream_t>(mbx_context_stream(ctx));
  mbx_matrix* A;
  MB(mbx_matrix_generate_rmat(ctx, f64 ? MBX_F64 : MBX_F32, scale, 16, 1, kind, 2, 0.0, 1.0, &A));
  int64_t n, nnz;
  MB(mbx_matrix_info(A, nullptr, &n, nullptr, &nnz));
  const void* vals;
  const int32_t* cols;
  const uint32_t* ro;
  MB(mbx_matrix_device_ptrs(A, &vals, &cols, &ro));
  const size_t vs = f64 ? 8 : 4;
  void *x, *y;
  int32_t* rows;
  CK(cudaMalloc(&x, n * vs));
  CK(cudaMalloc(&y, n * vs));
  CK(cudaMalloc(&rows, nnz * 4));
  fill_ones<<<1184, 256, 0, s>>>(x, n, f64);
  expand_rows<<<1184, 256, 0, s>>>(ro, n, rows);
  CK(cudaStreamSynchronize(s));
  // MERBIT: TILE + x cache, then K2+K3
  mbx_simt_config c;
  MB(mbx_config_make(32, f64 ? 7 : 14, 128, &c));
  mbx_tile* t;
  MB(mbx_matrix_generate_tile(ctx, A, &c, &t));
  double xs;
  MB(mbx_matrix_build_xcache(ctx, A, -1, &xs));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 20;
  auto timeit = [&](auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) fn();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms * 1e-3 / reps;
  };
  const double bytes = double(nnz) * (vs + 4) + 2.0 * n * vs + 4.0 * (n + 1);
  auto report = [&](const char* name, double sec) {
    printf("{\"scale\": %d, \"dtype\": \"%s\", \"kernel\": \"%s\", \"us\": %.1f, \"gflops\": %.1f, "
           "\"gbs\": %.1f, \"nnz\": %lld}\n",
           scale, f64 ? "f64" : "f32", name, sec * 1e6, 2.0 * nnz / sec / 1e9, bytes / sec / 1e9,
           (long long)nnz);
    fflush(stdout);
  };
  const double t_merbit =
      timeit([&] { MB(mbx_spmv_device(ctx, A, t, &c, x, y)); });
  report("merbit_b200", t_merbit);

  cusparseHandle_t h;
  CS(cusparseCreate(&h));
  CS(cusparseSetStream(h, s));
  const cudaDataType dt = f64 ? CUDA_R_64F : CUDA_R_32F;
  cusparseSpMatDescr_t csr, coo;
  CS(cusparseCreateCsr(&csr, n, n, nnz, const_cast<uint32_t*>(ro), const_cast<int32_t*>(cols),
                       const_cast<void*>(vals), CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                       CUSPARSE_INDEX_BASE_ZERO, dt));
  CS(cusparseCreateCoo(&coo, n, n, nnz, rows, const_cast<int32_t*>(cols), const_cast<void*>(vals),
                       CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, dt));
  cusparseDnVecDescr_t vx, vy;
  CS(cusparseCreateDnVec(&vx, n, x, dt));
  CS(cusparseCreateDnVec(&vy, n, y, dt));
  const double one = 1.0, zero = 0.0;
  const float onef = 1.f, zerof = 0.f;
  const void* alpha = f64 ? static_cast<const void*>(&one) : static_cast<const void*>(&onef);
  const void* beta = f64 ? static_cast<const void*>(&zero) : static_cast<const void*>(&zerof);
  struct Case {
    const char* name;
    cusparseSpMatDescr_t m;
    cusparseSpMVAlg_t alg;
  } cases[] = {{"cusparse_csr_alg1", csr, CUSPARSE_SPMV_CSR_ALG1},
               {"cusparse_csr_alg2", csr, CUSPARSE_SPMV_CSR_ALG2},
               {"cusparse_coo_alg1", coo, CUSPARSE_SPMV_COO_ALG1},
               {"cusparse_coo_alg2", coo, CUSPARSE_SPMV_COO_ALG2}};
  for (const Case& k : cases) {
    size_t ws = 0;
    CS(cusparseSpMV_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, k.m, vx, beta, vy, dt,
                               k.alg, &ws));
    void* buf = nullptr;
    CK(cudaMalloc(&buf, ws + 256));
    const double sec = timeit([&] {
      CS(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, k.m, vx, beta, vy, dt, k.alg,
                      buf));
    });
    report(k.name, sec);
    printf("{\"speedup_merbit_vs_%s\": %.3f}\n", k.name, sec / t_merbit);
    CK(cudaFree(buf));
  }
  return 0;
}
