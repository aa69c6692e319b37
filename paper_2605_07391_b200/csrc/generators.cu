// generators.cu -- device-side synthetic inputs (BASELINE configs C1/C2/C4).
//
// Counter-based R-MAT (Graph500 a,b,c,d = .57,.19,.19,.05), bit-identical to
// oracle/merbit_oracle.c:mo_rmat_csr so the CPU checker sees the same matrix:
// edge e, level l draws u = splitmix64(splitmix64(seed) ^ (e<<6 | l)) >> 11
// and compares it with floor(p * 2^53) thresholds (pure integer math).
// Duplicates are merged (normalize_coo, csr.hpp:43-68), self loops kept,
// natural vertex order.  kind 1 emits the PageRank transition directly:
// rows = destination, columns = source ascending, value T(1)/T(outdeg)
// (build_transition, solvers.hpp:36-74).
#include <cub/cub.cuh>

#include "mbx_internal.h"

namespace mbx {
namespace {

__host__ __device__ __forceinline__ uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

constexpr uint64_t kT1 = 5134103575202365ULL;  // floor(0.57 * 2^53)
constexpr uint64_t kT2 = 6845471433603153ULL;  // floor(0.76 * 2^53)
constexpr uint64_t kT3 = 8556839292003942ULL;  // floor(0.95 * 2^53)

__global__ void rmat_keys_kernel(uint64_t* __restrict__ keys, uint64_t m_raw, uint64_t seedmix,
                                 int scale, int transposed) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m_raw;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t src = 0, dst = 0;
    for (int l = 0; l < scale; ++l) {
      const uint64_t u = smix(seedmix ^ ((e << 6) | uint64_t(l))) >> 11;
      const uint64_t bit = 1ULL << (scale - 1 - l);
      if (u < kT1) {
      } else if (u < kT2) {
        dst |= bit;
      } else if (u < kT3) {
        src |= bit;
      } else {
        src |= bit;
        dst |= bit;
      }
    }
    keys[e] = transposed ? ((dst << scale) | src) : ((src << scale) | dst);
  }
}

__global__ void csr_from_keys_kernel(const uint64_t* __restrict__ keys, const uint64_t* d_m,
                                     int scale, uint64_t n, uint32_t* __restrict__ ro,
                                     int32_t* __restrict__ cols) {
  const uint64_t m = *d_m;
  const uint64_t cmask = (1ULL << scale) - 1;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[k];
    const uint64_t r = key >> scale;
    cols[k] = int32_t(key & cmask);
    const int64_t rp = k > 0 ? int64_t(keys[k - 1] >> scale) : -1;
    for (int64_t rr = rp + 1; rr <= int64_t(r); ++rr) ro[rr] = uint32_t(k);
    if (k == m - 1)
      for (uint64_t rr = r + 1; rr <= n; ++rr) ro[rr] = uint32_t(m);
  }
}

__global__ void zero_rows_if_empty_kernel(const uint64_t* d_m, uint32_t* ro, uint64_t n) {
  if (*d_m != 0) return;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += uint64_t(gridDim.x) * blockDim.x)
    ro[i] = 0;
}

template <typename T>
__global__ void uniform_values_kernel(T* __restrict__ vals, uint64_t m, uint64_t sm, double lo,
                                      double hi) {
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const double u = double(smix(sm ^ k) >> 11) * 0x1.0p-53;
    // lo + (hi - lo) * u without FMA contraction (matches the C oracle)
    vals[k] = T(__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u)));
  }
}

__global__ void outdeg_kernel(const int32_t* __restrict__ cols, uint64_t m, uint32_t* deg) {
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(deg + cols[k], 1u);
}

template <typename T>
__global__ void transition_values_kernel(const int32_t* __restrict__ cols, uint64_t m,
                                         const uint32_t* __restrict__ deg, T* __restrict__ vals) {
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += uint64_t(gridDim.x) * blockDim.x)
    vals[k] = T(1) / T(deg[cols[k]]);
}

unsigned grid(mbx_context* ctx) { return unsigned(ctx->sm_count) * 16; }

// ---- C5: 27-point stencil on a g^3 grid (diagonal 26, neighbours -1), the
// 3-D generalisation of five_point_laplacian (fixtures.hpp:40-56). ----------
__host__ __device__ __forceinline__ uint32_t span3(int64_t i, int64_t g) {
  return 3u - (i == 0) - (i == g - 1);
}

__global__ void stencil_counts_kernel(int64_t g, uint32_t* cnt) {
  const int64_t n = g * g * g;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = r / (g * g), j = (r / g) % g, k = r % g;
    cnt[r] = g == 1 ? 1u : span3(i, g) * span3(j, g) * span3(k, g);
  }
}

template <typename T>
__global__ void stencil_fill_kernel(int64_t g, const uint32_t* __restrict__ ro,
                                    int32_t* __restrict__ cols, T* __restrict__ vals) {
  const int64_t n = g * g * g;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = r / (g * g), j = (r / g) % g, k = r % g;
    uint32_t p = ro[r];
    for (int di = -1; di <= 1; ++di) {
      if (i + di < 0 || i + di >= g) continue;
      for (int dj = -1; dj <= 1; ++dj) {
        if (j + dj < 0 || j + dj >= g) continue;
        for (int dk = -1; dk <= 1; ++dk) {
          if (k + dk < 0 || k + dk >= g) continue;
          const int64_t c = ((i + di) * g + (j + dj)) * g + (k + dk);  // ascending
          cols[p] = int32_t(c);
          vals[p] = c == r ? T(26) : T(-1);
          ++p;
        }
      }
    }
  }
}

// ---- C3: power-law rows, exactly 10 % empty rows (seeded permutation),
// long rows scattered, strictly increasing columns spread over [0, n),
// values in [-1, 1).  Row length by permuted rank q:
//   L(q) = max(1, floor(2^20 / (q+1)^0.8))  for q < n - n/10, else 0. ------
__host__ __device__ __forceinline__ uint64_t perm_bits(uint64_t v, int bits, uint64_t key) {
  // bijection on [0, 2^bits): odd multiply + xor-shift rounds, masked
  const uint64_t mask = (bits >= 64) ? ~0ULL : ((1ULL << bits) - 1);
  for (int round = 0; round < 4; ++round) {
    v = (v * 0x9E3779B97F4A7C15ULL + (key >> (round * 8))) & mask;
    v ^= v >> ((bits + 1) / 2);
    v &= mask;
  }
  return v;
}

__global__ void powerlaw_counts_kernel(int log2n, uint64_t key, uint32_t* cnt) {
  const int64_t n = int64_t(1) << log2n;
  const int64_t live = n - n / 10;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = int64_t(perm_bits(uint64_t(r), log2n, key));
    uint32_t L = 0;
    if (q < live) {
      const double l = floor(1048576.0 / pow(double(q + 1), 0.8));
      L = uint32_t(l < 1.0 ? 1.0 : (l > double(n) ? double(n) : l));
    }
    cnt[r] = L;
  }
}

template <typename T>
__global__ void powerlaw_fill_kernel(int64_t n, const uint32_t* __restrict__ ro, uint64_t sm,
                                     int32_t* __restrict__ cols, T* __restrict__ vals) {
  // one warp per row (rows up to 2^20 long)
  const int lid = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w; r < n; r += nw) {
    const uint32_t b = ro[r], L = ro[r + 1] - b;
    for (uint32_t t = lid; t < L; t += 32) {
      const int64_t lo = int64_t(t) * n / L, hi = int64_t(t + 1) * n / L;  // [lo, hi) nonempty
      const uint64_t h = smix(sm ^ (uint64_t(r) << 21) ^ t);
      cols[b + t] = int32_t(lo + int64_t(h % uint64_t(hi - lo)));
      const double u = double(smix(h) >> 11) * 0x1.0p-53;
      vals[b + t] = T(__dadd_rn(-1.0, __dmul_rn(2.0, u)));
    }
  }
}

__global__ void widen_u32_kernel(const uint32_t* __restrict__ in, int64_t n,
                                 uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

__global__ void narrow_u64_kernel(const uint64_t* __restrict__ in, int64_t n,
                                  uint32_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = uint32_t(in[i]);
}

// row offsets from per-row counts (64-bit inclusive scan), arrays allocated
void csr_from_counts(mbx_context* ctx, int precision, int64_t n, uint32_t* cnt, mbx_matrix* m) {
  cudaStream_t s = ctx->stream;
  MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->ro), (n + 1) * 4 + 64, s));
  // 64-bit scan so an overflow of the 32-bit cursor is detected, not wrapped
  uint64_t* ro64 = nullptr;
  MBX_CUDA(cudaMallocAsync(&ro64, (n + 1) * 8, s));
  MBX_CUDA(cudaMemsetAsync(ro64, 0, 8, s));
  widen_u32_kernel<<<grid(ctx), 256, 0, s>>>(cnt, n, ro64 + 1);
  ++ctx->launches;
  size_t tb = 0;
  MBX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, ro64 + 1, ro64 + 1, n, s));
  void* temp = nullptr;
  MBX_CUDA(cudaMallocAsync(&temp, tb, s));
  MBX_CUDA(cub::DeviceScan::InclusiveSum(temp, tb, ro64 + 1, ro64 + 1, n, s));
  uint64_t nnz = 0;
  MBX_CUDA(cudaMemcpyAsync(&nnz, ro64 + n, 8, cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(temp, s);
  if (nnz > 0xFFFFFFFFULL) {
    cudaFreeAsync(ro64, s);
    fail(MBX_CAPACITY_ERROR, "generated nonzero count exceeds the 32-bit tile cursor");
  }
  narrow_u64_kernel<<<grid(ctx), 256, 0, s>>>(ro64, n + 1, m->ro);
  ++ctx->launches;
  cudaFreeAsync(ro64, s);
  const size_t vs = value_size(precision);
  m->precision = precision;
  m->n_rows = m->n_cols = n;
  m->nnz = int64_t(nnz);
  MBX_CUDA(cudaMallocAsync(&m->vals, nnz * vs + 256, s));
  MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->cols), nnz * 4 + 256, s));
  MBX_CUDA(cudaMemsetAsync(m->vals, 0, nnz * vs + 256, s));
  MBX_CUDA(cudaMemsetAsync(m->cols, 0, nnz * 4 + 256, s));
}

}  // namespace

void generate_rmat(mbx_context* ctx, int precision, int scale, int edge_factor, uint64_t seed,
                   int kind, uint64_t value_seed, double lo, double hi, mbx_matrix* m) {
  cudaStream_t s = ctx->stream;
  const uint64_t n = 1ULL << scale;
  const uint64_t m_raw = uint64_t(edge_factor) << scale;
  uint64_t *keys = nullptr, *sorted = nullptr, *d_m = nullptr;
  MBX_CUDA(cudaMallocAsync(&keys, m_raw * 8, s));
  MBX_CUDA(cudaMallocAsync(&sorted, m_raw * 8, s));
  MBX_CUDA(cudaMallocAsync(&d_m, 64, s));
  rmat_keys_kernel<<<grid(ctx), 256, 0, s>>>(keys, m_raw, smix(seed), scale, kind == 1);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
  size_t tb = 0, tb2 = 0;
  const int64_t items = int64_t(m_raw);
  MBX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, items, 0, 2 * scale, s));
  MBX_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, sorted, keys, d_m, items, s));
  void* temp = nullptr;
  MBX_CUDA(cudaMallocAsync(&temp, std::max(tb, tb2), s));
  MBX_CUDA(cub::DeviceRadixSort::SortKeys(temp, tb, keys, sorted, items, 0, 2 * scale, s));
  MBX_CUDA(cub::DeviceSelect::Unique(temp, tb2, sorted, keys, d_m, items, s));
  MBX_CUDA(cudaFreeAsync(temp, s));
  MBX_CUDA(cudaFreeAsync(sorted, s));
  uint64_t nnz = 0;
  MBX_CUDA(cudaMemcpyAsync(&nnz, d_m, 8, cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaStreamSynchronize(s));
  if (nnz > 0xFFFFFFFFULL) {
    cudaFreeAsync(keys, s);
    cudaFreeAsync(d_m, s);
    fail(MBX_CAPACITY_ERROR, "generated nonzero count exceeds the 32-bit tile cursor");
  }
  const size_t vs = value_size(precision);
  m->precision = precision;
  m->n_rows = m->n_cols = int64_t(n);
  m->nnz = int64_t(nnz);
  MBX_CUDA(cudaMallocAsync(&m->vals, nnz * vs + 256, s));
  MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->cols), nnz * 4 + 256, s));
  MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->ro), (n + 1) * 4 + 64, s));
  MBX_CUDA(cudaMemsetAsync(m->vals, 0, nnz * vs + 256, s));
  MBX_CUDA(cudaMemsetAsync(m->cols, 0, nnz * 4 + 256, s));
  csr_from_keys_kernel<<<grid(ctx), 256, 0, s>>>(keys, d_m, scale, n, m->ro, m->cols);
  zero_rows_if_empty_kernel<<<grid(ctx), 256, 0, s>>>(d_m, m->ro, n);
  ctx->launches += 2;
  MBX_CUDA(cudaGetLastError());
  MBX_CUDA(cudaFreeAsync(keys, s));
  MBX_CUDA(cudaFreeAsync(d_m, s));
  if (kind == 0) {
    const uint64_t sm = smix(value_seed);
    if (precision == MBX_F32)
      uniform_values_kernel<float><<<grid(ctx), 256, 0, s>>>(static_cast<float*>(m->vals), nnz, sm, lo, hi);
    else
      uniform_values_kernel<double><<<grid(ctx), 256, 0, s>>>(static_cast<double*>(m->vals), nnz, sm, lo, hi);
    ++ctx->launches;
  } else {
    uint32_t* deg = nullptr;
    MBX_CUDA(cudaMallocAsync(&deg, n * 4 + 64, s));
    MBX_CUDA(cudaMemsetAsync(deg, 0, n * 4 + 64, s));
    outdeg_kernel<<<grid(ctx), 256, 0, s>>>(m->cols, nnz, deg);
    if (precision == MBX_F32)
      transition_values_kernel<float><<<grid(ctx), 256, 0, s>>>(m->cols, nnz, deg, static_cast<float*>(m->vals));
    else
      transition_values_kernel<double><<<grid(ctx), 256, 0, s>>>(m->cols, nnz, deg, static_cast<double*>(m->vals));
    ctx->launches += 2;
    MBX_CUDA(cudaFreeAsync(deg, s));
  }
  MBX_CUDA(cudaGetLastError());
  MBX_CUDA(cudaStreamSynchronize(s));
}

void generate_stencil27(mbx_context* ctx, int precision, int64_t g, mbx_matrix* m) {
  cudaStream_t s = ctx->stream;
  const int64_t n = g * g * g;
  uint32_t* cnt = nullptr;
  MBX_CUDA(cudaMallocAsync(&cnt, n * 4 + 64, s));
  stencil_counts_kernel<<<grid(ctx), 256, 0, s>>>(g, cnt);
  ++ctx->launches;
  csr_from_counts(ctx, precision, n, cnt, m);
  if (precision == MBX_F32)
    stencil_fill_kernel<float><<<grid(ctx), 256, 0, s>>>(g, m->ro, m->cols,
                                                         static_cast<float*>(m->vals));
  else
    stencil_fill_kernel<double><<<grid(ctx), 256, 0, s>>>(g, m->ro, m->cols,
                                                          static_cast<double*>(m->vals));
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
  cudaFreeAsync(cnt, s);
  MBX_CUDA(cudaStreamSynchronize(s));
}

void generate_powerlaw(mbx_context* ctx, int precision, int log2n, uint64_t seed, mbx_matrix* m) {
  cudaStream_t s = ctx->stream;
  const int64_t n = int64_t(1) << log2n;
  uint32_t* cnt = nullptr;
  MBX_CUDA(cudaMallocAsync(&cnt, n * 4 + 64, s));
  powerlaw_counts_kernel<<<grid(ctx), 256, 0, s>>>(log2n, smix(seed), cnt);
  ++ctx->launches;
  csr_from_counts(ctx, precision, n, cnt, m);
  const uint64_t sm = smix(seed ^ 0x5851F42D4C957F2DULL);
  if (precision == MBX_F32)
    powerlaw_fill_kernel<float><<<grid(ctx), 256, 0, s>>>(n, m->ro, sm, m->cols,
                                                          static_cast<float*>(m->vals));
  else
    powerlaw_fill_kernel<double><<<grid(ctx), 256, 0, s>>>(n, m->ro, sm, m->cols,
                                                           static_cast<double*>(m->vals));
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
  cudaFreeAsync(cnt, s);
  MBX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mbx
