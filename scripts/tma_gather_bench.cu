// tma_gather_bench.cu -- does TMA tile::gather4 beat LSU gathers for the
// SpMV x[col] pattern on B200?  x is viewed as a 2D tensor [n/8][8] fp32
// (one 32-byte sector per row); each thread covers 4 nonzeros and issues one
// gather4 for the 4 sectors holding x[col0..col3], then reads its values from
// shared memory.  Compared against plain __ldg gathers on the same matrix.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//   scripts/tma_gather_bench.cu -o scripts/tma_gather_bench -L paper_2605_07391_b200
//   -lmerbit_b200 -lcuda -Xlinker -rpath,'$ORIGIN/../paper_2605_07391_b200'
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "merbit_b200.h"

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("CUDA %s at %d: %s\n", cudaGetErrorString(e), __LINE__, #x);              \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// STAGES buffers per warp; each stage = 32 threads x 4 sectors x 32 B = 4 KB
template <int STAGES>
__global__ void __launch_bounds__(256) tma_gather_kernel(const __grid_constant__ CUtensorMap tmap,
                                                         const float4* __restrict__ v,
                                                         const int4* __restrict__ c, int64_t nv,
                                                         float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  float* buf = reinterpret_cast<float*>(smem) + size_t(warp) * STAGES * 32 * 32;
  __shared__ __align__(8) uint64_t bar[8][STAGES];
  if (lid == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp][s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  float acc = 0.f;
  const int64_t wstride = int64_t(gridDim.x) * (blockDim.x >> 5) * 32;
  int64_t i0 = (int64_t(blockIdx.x) * (blockDim.x >> 5) + warp) * 32;
  uint32_t phase[STAGES] = {};
  // prologue: issue STAGES batches
  float4 vv[STAGES];
  int4 cc[STAGES];
#pragma unroll
  for (int s = 0; s < STAGES; ++s) {
    const int64_t i = i0 + s * wstride + lid;
    if (i0 + s * wstride < nv) {
      if (lid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[warp][s])),
                     "r"(int((nv - (i0 + s * wstride) < 32 ? nv - (i0 + s * wstride) : 32) * 128)));
      __syncwarp();
      if (i < nv) {
        vv[s] = __ldg(v + i);
        cc[s] = __ldg(c + i);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + (s * 32 + lid) * 32)),
            "l"(&tmap), "r"(0), "r"(cc[s].x >> 3), "r"(cc[s].y >> 3), "r"(cc[s].z >> 3),
            "r"(cc[s].w >> 3), "r"(smem_u32(&bar[warp][s]))
            : "memory");
      }
    }
  }
  for (int64_t base = i0; base < nv; base += STAGES * wstride) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int64_t bs = base + s * wstride;
      if (bs >= nv) break;
      const int64_t i = bs + lid;
      // wait for stage s
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
            : "=r"(done)
            : "r"(smem_u32(&bar[warp][s])), "r"(phase[s]));
      }
      phase[s] ^= 1;
      if (i < nv) {
        const float* sec = buf + (s * 32 + lid) * 32;
        acc += vv[s].x * sec[0 * 8 + (cc[s].x & 7)] + vv[s].y * sec[1 * 8 + (cc[s].y & 7)] +
               vv[s].z * sec[2 * 8 + (cc[s].z & 7)] + vv[s].w * sec[3 * 8 + (cc[s].w & 7)];
      }
      __syncwarp();
      // refill stage s with the batch STAGES ahead
      const int64_t nb = bs + STAGES * wstride;
      if (nb < nv) {
        if (lid == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[warp][s])),
                       "r"(int((nv - nb < 32 ? nv - nb : 32) * 128)));
        __syncwarp();
        const int64_t j = nb + lid;
        if (j < nv) {
          vv[s] = __ldg(v + j);
          cc[s] = __ldg(c + j);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + (s * 32 + lid) * 32)),
              "l"(&tmap), "r"(0), "r"(cc[s].x >> 3), "r"(cc[s].y >> 3), "r"(cc[s].z >> 3),
              "r"(cc[s].w >> 3), "r"(smem_u32(&bar[warp][s]))
              : "memory");
        }
      }
    }
  }
  if (acc == 1234.5f) *out = acc;
}

// Hybrid: warps [0, tma_warps) gather the TMA share [0, split) of the
// vectors with gather4 (2 stages); the other warps gather [split, nv) with
// LSU __ldg.  Both engines run concurrently inside every SM.
__global__ void __launch_bounds__(512) hybrid_kernel(const __grid_constant__ CUtensorMap tmap,
                                                     const float4* __restrict__ v,
                                                     const int4* __restrict__ c,
                                                     const float* __restrict__ x, int64_t nv,
                                                     int64_t split, int tma_warps, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  __shared__ __align__(8) uint64_t bar[16][2];
  float acc = 0.f;
  if (warp < tma_warps) {
    float* buf = reinterpret_cast<float*>(smem) + size_t(warp) * 2 * 32 * 32;
    if (lid == 0)
      for (int s = 0; s < 2; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    const int64_t wstride = int64_t(gridDim.x) * tma_warps * 32;
    const int64_t i0 = (int64_t(blockIdx.x) * tma_warps + warp) * 32;
    uint32_t phase[2] = {0, 0};
    float4 vv[2];
    int4 cc[2];
    auto issue = [&](int s, int64_t b) {
      if (lid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[warp][s])),
                     "r"(int((split - b < 32 ? split - b : 32) * 128)));
      __syncwarp();
      const int64_t j = b + lid;
      if (j < split) {
        vv[s] = __ldg(v + j);
        cc[s] = __ldg(c + j);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + (s * 32 + lid) * 32)),
            "l"(&tmap), "r"(0), "r"(cc[s].x >> 3), "r"(cc[s].y >> 3), "r"(cc[s].z >> 3),
            "r"(cc[s].w >> 3), "r"(smem_u32(&bar[warp][s]))
            : "memory");
      }
    };
    for (int s = 0; s < 2; ++s)
      if (i0 + s * wstride < split) issue(s, i0 + s * wstride);
    for (int64_t base = i0; base < split; base += 2 * wstride) {
      for (int s = 0; s < 2; ++s) {
        const int64_t bs = base + s * wstride;
        if (bs >= split) break;
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
              : "=r"(done)
              : "r"(smem_u32(&bar[warp][s])), "r"(phase[s]));
        phase[s] ^= 1;
        if (bs + lid < split) {
          const float* sec = buf + (s * 32 + lid) * 32;
          acc += vv[s].x * sec[(cc[s].x & 7)] + vv[s].y * sec[8 + (cc[s].y & 7)] +
                 vv[s].z * sec[16 + (cc[s].z & 7)] + vv[s].w * sec[24 + (cc[s].w & 7)];
        }
        __syncwarp();
        if (bs + 2 * wstride < split) issue(s, bs + 2 * wstride);
      }
    }
  } else {
    const int lw = warp - tma_warps, nlw = (blockDim.x >> 5) - tma_warps;
    for (int64_t i = split + (int64_t(blockIdx.x) * nlw + lw) * 32 + lid; i < nv;
         i += int64_t(gridDim.x) * nlw * 32) {
      const float4 a = __ldg(v + i);
      const int4 b = __ldg(c + i);
      acc += a.x * __ldg(x + b.x) + a.y * __ldg(x + b.y) + a.z * __ldg(x + b.z) + a.w * __ldg(x + b.w);
    }
  }
  if (acc == 1234.5f) *out = acc;
}

__global__ void ldg_gather_kernel(const float4* __restrict__ v, const int4* __restrict__ c,
                                  const float* __restrict__ x, int64_t nv, float* out) {
  float acc = 0.f;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float4 a = __ldg(v + i);
    const int4 b = __ldg(c + i);
    acc += a.x * __ldg(x + b.x) + a.y * __ldg(x + b.y) + a.z * __ldg(x + b.z) + a.w * __ldg(x + b.w);
  }
  if (acc == 1234.5f) *out = acc;
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? atoi(argv[1]) : 24;
  mbx_context* ctx;
  if (mbx_context_create(0, &ctx)) return 1;
  mbx_matrix* P;
  if (mbx_matrix_generate_rmat(ctx, MBX_F32, scale, 16, 1, 1, 2, 0.0, 1.0, &P)) return 1;
  int64_t n, nnz;
  mbx_matrix_info(P, nullptr, &n, nullptr, &nnz);
  const void* vals;
  const int32_t* cols;
  const uint32_t* ro;
  mbx_matrix_device_ptrs(P, &vals, &cols, &ro);
  float *x, *out;
  CK(cudaMalloc(&x, n * 4 + 1024));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(x, 0, n * 4));
  const int64_t nv = nnz / 4;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto timeit = [&](auto launch, const char* name) {
    launch();
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < 5; ++i) launch();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 5;
    printf("{\"kernel\": \"%s\", \"us\": %.1f, \"gather_per_ns\": %.1f}\n", name, ms * 1e3,
           double(nv * 4) / (ms * 1e6));
    fflush(stdout);
  };
  timeit([&] { ldg_gather_kernel<<<sms * 8, 256, 0, s>>>((const float4*)vals, (const int4*)cols, x, nv, out); },
         "ldg_gather");
  CUtensorMap tmap;
  cuuint64_t gdim[2] = {8, cuuint64_t((n + 7) / 8)};
  cuuint64_t gstride[1] = {32};
  for (int boxrows : {1, 4}) {
    cuuint32_t box[2] = {8, cuuint32_t(boxrows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, gdim, gstride,
                                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("{\"encode_box_rows\": %d, \"result\": %d}\n", boxrows, int(r));
    if (r != CUDA_SUCCESS) continue;
    for (int tw : {2, 4, 6, 8}) {
      for (double f : {0.2, 0.3, 0.4}) {
        const int64_t split = int64_t(double(nv) * f);
        const size_t smem = size_t(tw) * 2 * 32 * 32 * 4;
        CK(cudaFuncSetAttribute(hybrid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        char name[96];
        snprintf(name, sizeof name, "hybrid tma_warps%d/16 share%.1f b2", tw, f);
        timeit([&] { hybrid_kernel<<<sms * 2, 512, smem, s>>>(tmap, (const float4*)vals, (const int4*)cols, x, nv, split, tw, out); }, name);
      }
    }
    for (int bps : {2, 4, 8}) {
      char name[64];
      snprintf(name, sizeof name, "tma_gather4 box%d stages2 b%d", boxrows, bps);
      const size_t smem2 = 8 * 2 * 32 * 32 * 4;
      CK(cudaFuncSetAttribute(tma_gather_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
      timeit([&] { tma_gather_kernel<2><<<sms * bps, 256, smem2, s>>>(tmap, (const float4*)vals, (const int4*)cols, nv, out); }, name);
      snprintf(name, sizeof name, "tma_gather4 box%d stages4 b%d", boxrows, bps);
      const size_t smem4 = 8 * 4 * 32 * 32 * 4;
      CK(cudaFuncSetAttribute(tma_gather_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4));
      if (smem4 * bps <= 220 * 1024)
        timeit([&] { tma_gather_kernel<4><<<sms * bps, 256, smem4, s>>>(tmap, (const float4*)vals, (const int4*)cols, nv, out); }, name);
    }
    break;
  }
  return 0;
}
