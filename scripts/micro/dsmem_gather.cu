// Microbenchmark: scattered 4-byte gathers from (a) local shared memory,
// (b) distributed shared memory across a thread-block cluster of C CTAs
// (ld.shared::cluster through mapa), (c) an L2-resident global array --
// gathers per SM per cycle, 1 CTA x 1024 threads per SM, 148 CTAs.
// Question: can a cluster-shared x hub table (C x the entries at the same
// shared memory per SM) serve hub gathers as fast as an L2 hit?
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

constexpr int T = 20000;      // table entries per CTA
constexpr int ITERS = 2048;
constexpr int UNROLL = 8;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int C, int MODE>  // MODE 0: LDS local, 1: ld.shared::cluster, 2: global
__global__ void __launch_bounds__(1024, 1) gather_kernel(const float* __restrict__ g, uint32_t gmask,
                                                         float* out, long long* cycles) {
  extern __shared__ float tab[];
  for (int i = threadIdx.x; i < T; i += blockDim.x) tab[i] = float(i + blockIdx.x);
  if constexpr (C > 1) cg::this_cluster().sync(); else __syncthreads();
  const uint32_t base = uint32_t(__cvta_generic_to_shared(tab));
  uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    float v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      s = s * 1664525u + 1013904223u;
      const uint32_t h = s >> 8;
      if constexpr (MODE == 0) {
        v[u] = tab[h % T];
      } else if constexpr (MODE == 1) {
        const uint32_t idx = h % (uint32_t(T) * C);
        const uint32_t rank = idx % C, loc = idx / C;
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base), "r"(rank));
        float x;
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(ra + loc * 4));
        v[u] = x;
      } else {
        v[u] = __ldg(g + (h & gmask));
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += v[u];
  }
  long long t1 = clock64();
  if constexpr (C > 1) cg::this_cluster().sync();
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int C, int MODE>
void run(const char* name, const float* g, uint32_t gmask, float* out, long long* cyc) {
  auto k = gather_kernel<C, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T * 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = T * 4;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, g, gmask, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("%s: launch failed %s\n", name, cudaGetErrorString(e));
      return;
    }
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(148);
  cudaMemcpy(c.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (auto v : c) mx = v > mx ? v : mx;
  const double loads = 148.0 * 1024 * ITERS * UNROLL;
  printf("{\"case\": \"%s\", \"ms\": %.4f, \"gathers_per_s\": %.4g, \"gathers_per_sm_cycle\": %.3f}\n",
         name, ms, loads / (ms * 1e-3), 1024.0 * ITERS * UNROLL / double(mx));
}

int main() {
  const size_t n = size_t(16) << 20;  // 64 MB of floats: L2-resident-ish
  float *g, *out;
  long long* cyc;
  cudaMalloc(&g, n * 4);
  cudaMemset(g, 0, n * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  run<1, 0>("lds_local", g, n - 1, out, cyc);
  run<1, 1>("cluster1_ld_shared_cluster", g, n - 1, out, cyc);
  run<2, 1>("cluster2_dsmem", g, n - 1, out, cyc);
  run<4, 1>("cluster4_dsmem", g, n - 1, out, cyc);
  run<1, 2>("global_64MB", g, n - 1, out, cyc);
  run<1, 2>("global_4MB", g, (1u << 20) - 1, out, cyc);
  return 0;
}
