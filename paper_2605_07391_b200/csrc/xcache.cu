// xcache.cu -- x hub cache preprocessing.
//
// Random x[col] gathers cost one L1->L2 request each and are the limiter of
// the SpMV kernel on power-law inputs (ncu: l1tex2xbar request port ~81%,
// hottest L2 slices ~95% while DRAM sits at ~27%).  The most referenced
// columns ("hubs") are therefore staged once per CTA in shared memory by K2.
// This pass ranks columns by reference count (stable: ties keep ascending
// column order), keeps those referenced more often than the number of CTAs
// that will each load them, and writes a second column array where every
// hub reference becomes (INT32_MIN | slot).  The TILE is untouched and the
// SpMV result is bitwise identical with or without the cache (the same
// x value is read, the summation order does not change).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "mbx_internal.h"

namespace mbx {
namespace {

// Column reference counts.  The hottest columns of a power-law graph take
// most of the increments, and one L2 atomic unit serialises them (R-MAT s20:
// 258 us for 16 M nonzeros); the first kPrivCols columns -- where a degree-
// relabelled graph keeps its hubs, and R-MAT its lowest ids -- are counted
// in shared memory per block and flushed once.
constexpr int kPrivCols = 12288;  // 48 KB of shared counters

__global__ void __launch_bounds__(512) count_cols_kernel(const int32_t* __restrict__ cols,
                                                         int64_t nnz, int64_t ncols,
                                                         uint32_t* __restrict__ cnt) {
  __shared__ uint32_t h[kPrivCols];
  const int lim = int(ncols < kPrivCols ? ncols : kPrivCols);
  for (int i = threadIdx.x; i < lim; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t c = cols[k];
    if (c < kPrivCols)
      atomicAdd(&h[c], 1u);
    else
      atomicAdd(cnt + c, 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < lim; i += blockDim.x)
    if (h[i]) atomicAdd(cnt + i, h[i]);
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    v[i] = int32_t(i);
}

__global__ void fill_kernel(int32_t* v, int64_t n, int32_t val) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    v[i] = val;
}

__global__ void slot_map_kernel(const int32_t* __restrict__ hub_cols, int h, int32_t* slot_of) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < h) slot_of[hub_cols[i]] = i;
}

__global__ void encode_kernel(const int32_t* __restrict__ cols, int64_t nnz,
                              const int32_t* __restrict__ slot_of, int32_t* __restrict__ out) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t c = cols[k];
    const int32_t s = slot_of[c];
    out[k] = s >= 0 ? int32_t(0x80000000u | uint32_t(s)) : c;
  }
}

}  // namespace

void launch_count_columns(mbx_context* ctx, const int32_t* cols, int64_t nnz, int64_t ncols,
                          uint32_t* cnt) {
  if (nnz <= 0) return;
  count_cols_kernel<<<unsigned(ctx->sm_count) * 2, 512, 0, ctx->stream>>>(cols, nnz, ncols, cnt);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

void build_xcache(mbx_context* ctx, mbx_matrix* m, int max_hubs) {
  cudaStream_t s = ctx->stream;
  if (m->cols_hub) {
    cudaFreeAsync(m->cols_hub, s);
    m->cols_hub = nullptr;
  }
  if (m->hub_cols) {
    cudaFreeAsync(m->hub_cols, s);
    m->hub_cols = nullptr;
  }
  m->hub_avail = 0;
  m->hub_coverage = 0.0;
  ++m->version;  // invalidates slot copies built over the old encoding
  ++m->gen;      // and the graphs captured over the old buffers
  const Tuning& tu = ctx->tuning;
  int slots = max_hub_slots(ctx, tu.warps_per_cta, tu.ctas_per_sm,
                            m->precision == MBX_F32 ? 14 : 7, m->precision);
  if (max_hubs >= 0) slots = std::min(slots, max_hubs);
  if (slots <= 0 || m->nnz == 0 || m->n_cols == 0) return;
  const int64_t n = m->n_cols;
  const unsigned grid = unsigned(ctx->sm_count) * 8;
  uint32_t *cnt = nullptr, *cnt_sorted = nullptr;
  int32_t *ids = nullptr, *ids_sorted = nullptr;
  MBX_CUDA(cudaMallocAsync(&cnt, n * 4, s));
  MBX_CUDA(cudaMallocAsync(&cnt_sorted, n * 4, s));
  MBX_CUDA(cudaMallocAsync(&ids, n * 4, s));
  MBX_CUDA(cudaMallocAsync(&ids_sorted, n * 4, s));
  MBX_CUDA(cudaMemsetAsync(cnt, 0, n * 4, s));
  count_cols_kernel<<<unsigned(ctx->sm_count) * 2, 512, 0, s>>>(m->cols, m->nnz, n, cnt);
  iota_kernel<<<grid, 256, 0, s>>>(ids, n);
  ctx->launches += 2;
  size_t tb = 0;
  MBX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, cnt, cnt_sorted, ids,
                                                      ids_sorted, n, 0, 32, s));
  void* temp = nullptr;
  MBX_CUDA(cudaMallocAsync(&temp, tb, s));
  MBX_CUDA(cub::DeviceRadixSort::SortPairsDescending(temp, tb, cnt, cnt_sorted, ids, ids_sorted,
                                                      n, 0, 32, s));
  const int cand = int(std::min<int64_t>(slots, n));
  std::vector<uint32_t> hc(cand);
  std::vector<int32_t> hid(cand);
  MBX_CUDA(cudaMemcpyAsync(hc.data(), cnt_sorted, size_t(cand) * 4, cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaMemcpyAsync(hid.data(), ids_sorted, size_t(cand) * 4, cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaStreamSynchronize(s));
  // A hub pays off only if it is referenced several times more often than
  // it costs to load (once per resident CTA per SpMV), and the per-CTA table
  // load (a serial preamble before any tile) must stay a small fraction
  // (<= 2 %) of that CTA's share of the gathers -- small matrices get small
  // tables (R-MAT s20 in natural order: measured 10 % preamble with an
  // uncapped table).  The load is counted in 128-byte lines: hubs that share
  // a line with an earlier hub ride along for free, so the contiguous hub
  // block of a degree-relabelled matrix (its hubs ARE vertices 0..h-1) costs
  // 1/32 of a scattered one and small relabelled graphs get full tables.
  const int64_t ctas = int64_t(ctx->sm_count) * tu.ctas_per_sm;
  const uint32_t min_refs = uint32_t(4 * ctas);
  const uint32_t min_refs_shared = uint32_t(std::max<int64_t>(ctas / 8, 2));
  const int64_t cap_lines = m->nnz / (ctas * 50);
  const int line_shift = m->precision == MBX_F32 ? 5 : 4;  // entries per 128-byte line
  std::vector<uint8_t> line_seen;
  int h = 0;
  int64_t covered = 0, lines = 0;
  while (h < cand) {
    const int64_t line = int64_t(hid[h]) >> line_shift;
    if (line_seen.size() <= size_t(line)) line_seen.resize(size_t(line) + 1, 0);
    const bool fresh = !line_seen[size_t(line)];
    if (hc[h] <= (fresh ? min_refs : min_refs_shared)) break;
    if (fresh && lines + 1 > cap_lines) break;
    if (fresh) {
      line_seen[size_t(line)] = 1;
      ++lines;
    }
    covered += hc[h++];
  }
  if (h > 0) {
    MBX_CUDA(cudaMallocAsync(&m->hub_cols, size_t(h) * 4 + 64, s));
    MBX_CUDA(cudaMemcpyAsync(m->hub_cols, ids_sorted, size_t(h) * 4, cudaMemcpyDeviceToDevice, s));
    int32_t* slot_of = reinterpret_cast<int32_t*>(cnt);  // reuse
    fill_kernel<<<grid, 256, 0, s>>>(slot_of, n, -1);
    slot_map_kernel<<<(h + 255) / 256, 256, 0, s>>>(m->hub_cols, h, slot_of);
    MBX_CUDA(cudaMallocAsync(&m->cols_hub, m->nnz * 4 + 256, s));
    MBX_CUDA(cudaMemsetAsync(m->cols_hub, 0, m->nnz * 4 + 256, s));
    encode_kernel<<<grid, 256, 0, s>>>(m->cols, m->nnz, slot_of, m->cols_hub);
    ctx->launches += 3;
    MBX_CUDA(cudaGetLastError());
    m->hub_avail = h;
    m->hub_coverage = double(covered) / double(m->nnz);
  }
  cudaFreeAsync(temp, s);
  cudaFreeAsync(cnt, s);
  cudaFreeAsync(cnt_sorted, s);
  cudaFreeAsync(ids, s);
  cudaFreeAsync(ids_sorted, s);
  MBX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mbx

