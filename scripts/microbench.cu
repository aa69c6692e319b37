// microbench.cu -- ceilings for the SpMV access pattern on the real R-MAT
// matrix (generated through the product C ABI): pure streaming of
// values+columns, pure x gathers with several cache policies, and gathers
// through a shared-memory hub table of varying size.  Not part of the
// product; used to decide kernel design (profiles/).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include
//      scripts/microbench.cu -o scripts/microbench -L paper_2605_07391_b200
//      -lmerbit_b200 -Xlinker -rpath,'$ORIGIN/../paper_2605_07391_b200'
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "merbit_b200.h"

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA %s at %d: %s\n", cudaGetErrorString(e), __LINE__, #x);         \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)
#define MB(x)                                                      \
  do {                                                             \
    if ((x) != 0) {                                                \
      printf("mbx error %s at %d\n", mbx_last_error(), __LINE__); \
      exit(1);                                                     \
    }                                                              \
  } while (0)

__device__ float g_sink;

template <int MODE>
__global__ void stream_kernel(const float4* __restrict__ v, const int4* __restrict__ c, int64_t nv,
                              float* out) {
  float acc = 0.f;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 a;
    int4 b;
    if (MODE == 0) {
      a = __ldg(v + i);
      b = __ldg(c + i);
    } else {
      asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(v + i));
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(c + i));
    }
    acc += a.x + a.y + a.z + a.w + float(b.x ^ b.y ^ b.z ^ b.w);
  }
  if (acc == 1234.5f) *out = acc;
}

// MODE 0: __ldg gathers; 1: ld.global.nc.L1::no_allocate; 2: ld.global.cg;
// 3: hub smem table (cols encoded, sign bit) + __ldg
template <int MODE>
__global__ void gather_kernel(const float4* __restrict__ v, const int4* __restrict__ c,
                              const float* __restrict__ x, int64_t nv, const int* hub_cols,
                              int hubs, float* out) {
  extern __shared__ float hub[];
  if (MODE == 3) {
    for (int i = threadIdx.x; i < hubs; i += blockDim.x) hub[i] = __ldg(x + hub_cols[i]);
    __syncthreads();
  }
  float acc = 0.f;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 a;
    int4 b;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(v + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(c + i));
    int cc[4] = {b.x, b.y, b.z, b.w};
    float vv[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float xv;
      if (MODE == 0) {
        xv = __ldg(x + cc[e]);
      } else if (MODE == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(xv) : "l"(x + cc[e]));
      } else if (MODE == 2) {
        asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(xv) : "l"(x + cc[e]));
      } else {
        xv = cc[e] < 0 ? hub[cc[e] & 0x7fffffff] : __ldg(x + cc[e]);
      }
      acc += vv[e] * xv;
    }
  }
  if (acc == 1234.5f) *out = acc;
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? atoi(argv[1]) : 24;
  mbx_context* ctx;
  MB(mbx_context_create(0, &ctx));
  mbx_matrix* P;
  MB(mbx_matrix_generate_rmat(ctx, MBX_F32, scale, 16, 1, 1, 2, 0.0, 1.0, &P));
  int64_t n, nnz;
  MB(mbx_matrix_info(P, nullptr, &n, nullptr, &nnz));
  const void* vals;
  const int32_t* cols;
  const uint32_t* ro;
  MB(mbx_matrix_device_ptrs(P, &vals, &cols, &ro));
  cudaStream_t s = static_cast<cudaStream_t>(mbx_context_stream(ctx));
  float* x;
  float* out;
  CK(cudaMalloc(&x, n * 4));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(x, 0, n * 4));
  const int64_t nv = nnz / 4;
  const double stream_bytes = double(nv) * 32.0;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto timeit = [&](auto launch, const char* name, double bytes) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    printf("{\"kernel\": \"%s\", \"us\": %.1f, \"gbs\": %.1f, \"gather_per_ns\": %.1f}\n", name,
           ms * 1e3, bytes / (ms * 1e-3) / 1e9, double(nv * 4) / (ms * 1e6));
  };
  printf("{\"n\": %lld, \"nnz\": %lld}\n", (long long)n, (long long)nnz);
  for (int tpb : {256, 512, 1024}) {
    for (int bps : {1, 2, 4, 8}) {
      if (tpb * bps > 2048) continue;
      const int grid = sms * bps;
      char name[128];
      snprintf(name, sizeof name, "stream_ldg t%d b%d", tpb, bps);
      timeit([&] { stream_kernel<0><<<grid, tpb, 0, s>>>((const float4*)vals, (const int4*)cols, nv, out); }, name, stream_bytes);
      snprintf(name, sizeof name, "stream_noalloc t%d b%d", tpb, bps);
      timeit([&] { stream_kernel<1><<<grid, tpb, 0, s>>>((const float4*)vals, (const int4*)cols, nv, out); }, name, stream_bytes);
      snprintf(name, sizeof name, "gather_ldg t%d b%d", tpb, bps);
      timeit([&] { gather_kernel<0><<<grid, tpb, 0, s>>>((const float4*)vals, (const int4*)cols, x, nv, nullptr, 0, out); }, name, stream_bytes);
      snprintf(name, sizeof name, "gather_nc_noalloc t%d b%d", tpb, bps);
      timeit([&] { gather_kernel<1><<<grid, tpb, 0, s>>>((const float4*)vals, (const int4*)cols, x, nv, nullptr, 0, out); }, name, stream_bytes);
      snprintf(name, sizeof name, "gather_cg t%d b%d", tpb, bps);
      timeit([&] { gather_kernel<2><<<grid, tpb, 0, s>>>((const float4*)vals, (const int4*)cols, x, nv, nullptr, 0, out); }, name, stream_bytes);
    }
  }
  // hub tables of several sizes
  CK(cudaFuncSetAttribute(gather_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int cap : {1024, 2048, 4096, 8192, 16384, 32768}) {
    MB(mbx_context_set_tuning(ctx, 32, 1, cap));
    double secs;
    MB(mbx_matrix_build_xcache(ctx, P, cap, &secs));
    int hubs;
    double cov;
    MB(mbx_matrix_xcache_info(P, &hubs, &cov));
    const int32_t *ch, *hc;
    MB(mbx_matrix_xcache_ptrs(P, &ch, &hc));
    (void)secs;
    printf("{\"hub_cap\": %d, \"hubs\": %d, \"coverage\": %.3f}\n", cap, hubs, cov);
    if (!ch) continue;
    for (int tpb : {512, 1024}) {
      for (int bps : {1, 2}) {
        if (tpb * bps > 2048) continue;
        const size_t smem = size_t(hubs) * 4;
        if (smem * bps > 220 * 1024) continue;
        char name[128];
        snprintf(name, sizeof name, "gather_hub%d t%d b%d", hubs, tpb, bps);
        timeit([&] { gather_kernel<3><<<sms * bps, tpb, smem, s>>>((const float4*)vals, (const int4*)ch, x, nv, hc, hubs, out); }, name, stream_bytes);
      }
    }
  }
  return 0;
}
