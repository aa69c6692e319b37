// xcache.cu -- x hub cache preprocessing.
//
// Random x[col] gathers cost one L1->L2 request each and are the limiter of
// the SpMV kernel on power-law inputs (ncu: l1tex2xbar request port ~81%,
// hottest L2 slices ~95% while DRAM sits at ~27%).  The most referenced
// columns ("hubs") are therefore staged once per CTA in shared memory by K2.
// This pass ranks columns by their reference count in a sample of the
// nonzeros (stable: ties keep ascending column order) and keeps those
// referenced more often than the number of CTAs that will each load them;
// the slot copy K2 walks then encodes every hub reference as
// (INT32_MIN | slot).  The TILE is untouched and the
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

// word map of the (ascending) hub list: map[w].x = the hubs among columns
// 32w..32w+31 as bits, map[w].y = slot of the first of them
__global__ void hub_word_kernel(const int32_t* __restrict__ hub_cols, int h, uint2* map,
                                uint32_t* bloom) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= h) return;
  const int32_t c = hub_cols[i];
  const int32_t w = c >> 5;
  atomicOr(&map[w].x, 1u << (c & 31));
  if (i == 0 || (hub_cols[i - 1] >> 5) != w) map[w].y = uint32_t(i);
  const uint32_t b = hub_bloom_bit(c);
  atomicOr(bloom + (b >> 5), 1u << (b & 31));
}

__global__ void encode_kernel(const int32_t* __restrict__ cols, int64_t nnz,
                              const uint2* __restrict__ map, int32_t* __restrict__ out) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x)
    out[k] = hub_word_encode(map, cols[k]);
}

}  // namespace

void launch_count_columns(mbx_context* ctx, const int32_t* cols, int64_t nnz, int64_t ncols,
                          uint32_t* cnt) {
  if (nnz <= 0) return;
  count_cols_kernel<<<unsigned(ctx->sm_count) * 2, 512, 0, ctx->stream>>>(cols, nnz, ncols, cnt);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

namespace {

// Column reference counts over a sample of the nonzeros: every S-th run of
// 32 consecutive nonzeros (one warp-coalesced load each), so the selection
// costs at most ~2^22 scattered increments whatever the matrix size.  The
// counts only rank candidate hubs: a hub's value in shared memory is the same
// x entry, so results do not depend on which columns are chosen.
constexpr int64_t kSampleRuns = int64_t(1) << 17;  // 32 nonzeros each (4 M samples)

// Also the gather locality of the sample: how many distinct 32-byte sectors
// of x a run of 32 consecutive nonzeros touches (a stencil ~10, a random
// or power-law matrix ~30), which picks K2's next-tile staging.
// Distinct 32-byte x sectors in runs of 32 consecutive nonzeros (every
// stride-th run) -- the pilot that tells a local matrix (a stencil) from a
// request-bound one before any counting.
__global__ void sector_sample_kernel(const int32_t* __restrict__ cols, int64_t nnz,
                                     int64_t stride_runs, int sector_shift,
                                     unsigned long long* __restrict__ out) {
  const int lid = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t full = nnz / 32;
  unsigned long long sec = 0, nr = 0;
  for (int64_t r = w * stride_runs; r < full; r += nw * stride_runs) {
    const int32_t c = __ldg(cols + r * 32 + lid);
    const unsigned same = __match_any_sync(0xffffffffu, c >> sector_shift);
    sec += __popc(__ballot_sync(0xffffffffu, lid == __ffs(same) - 1));
    ++nr;
  }
  if (lid == 0 && nr) {
    atomicAdd(out, sec);
    atomicAdd(out + 1, nr);
  }
}

// The first kSamplePriv columns are counted in shared memory per block and
// flushed once (only the entries the block touched): R-MAT's hottest column
// ids are the lowest ones -- column 0 alone takes 0.76^scale of the
// references, serialised at one L2 atomic unit -- and a degree-relabelled
// graph keeps all its hubs there.
constexpr int kSamplePriv = 4096;

__global__ void __launch_bounds__(1024) count_sample_kernel(
    const int32_t* __restrict__ cols, int64_t nnz, int64_t stride_runs, int sector_shift,
    uint32_t* __restrict__ cnt, uint32_t* __restrict__ cmax,
    unsigned long long* __restrict__ sectors, unsigned long long* __restrict__ full_runs,
    const unsigned long long* __restrict__ pilot, int local_sectors) {
  // a local matrix (pilot: sectors, runs) gets no table: nothing to count
  if (pilot && pilot[1] && pilot[0] < (unsigned long long)local_sectors * pilot[1]) return;
  __shared__ uint32_t priv[kSamplePriv];
  for (int i = threadIdx.x; i < kSamplePriv; i += blockDim.x) priv[i] = 0;
  __syncthreads();
  const int lid = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t runs = (nnz + 31) / 32;
  uint32_t mx = 0;  // the largest count this thread produced
  unsigned long long sec = 0, nr = 0;
  for (int64_t r = w * stride_runs; r < runs; r += nw * stride_runs) {
    const int64_t k = r * 32 + lid;
    const int32_t c = k < nnz ? __ldg(cols + k) : -1;
    if (c >= kSamplePriv)
      mx = max(mx, atomicAdd(cnt + c, 1u) + 1u);
    else if (c >= 0)
      atomicAdd(priv + c, 1u);
    if (r * 32 + 32 <= nnz) {  // warp-uniform: a full run
      const unsigned same = __match_any_sync(0xffffffffu, c >> sector_shift);
      const unsigned leaders = __ballot_sync(0xffffffffu, lid == __ffs(same) - 1);
      sec += __popc(leaders);
      ++nr;
    }
  }
  __syncthreads();
  // flush: the last block to add to a column sees its full count
  for (int i = threadIdx.x; i < kSamplePriv; i += blockDim.x)
    if (priv[i]) mx = max(mx, atomicAdd(cnt + i, priv[i]) + priv[i]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lid == 0) {
    if (mx) atomicMax(cmax, mx);
    if (nr) {
      atomicAdd(sectors, sec);
      atomicAdd(full_runs, nr);
    }
  }
}

// candidates: columns whose sampled count exceeds `t`
__global__ void flag_above_kernel(const uint32_t* __restrict__ cnt, int64_t n, uint32_t t,
                                  uint8_t* __restrict__ flag) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    flag[i] = cnt[i] > t;
}

__global__ void gather_counts_kernel(const uint32_t* __restrict__ cnt,
                                     const int32_t* __restrict__ ids, int64_t k,
                                     uint32_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = cnt[ids[i]];
}

// Histogram of the sampled counts (bins 1..kHistBins-1, the last one
// holding every count >= kHistBins-1, whose true sum and maximum are kept
// aside): what the selection below needs to pick the hub SET without sorting.
constexpr int kHistBins = 8192;

struct HubPick {
  unsigned long long sectors;    // distinct x sectors over the sampled full runs ...
  unsigned long long full_runs;  // ... and the number of those runs
  unsigned long long covered;  // sampled references of the chosen hubs
  unsigned long long capsum;   // sum of the counts in the last bin
  uint32_t capmax;             // largest count in the last bin (0: empty)
  uint32_t cmax;               // largest sampled count (count_sample_kernel)
  int32_t h;                   // hubs chosen
  uint32_t tau;                // every count > tau is a hub ...
  int32_t need;                // ... and the first `need` columns with count == tau
  int32_t ties;                // columns with count == tau
  int32_t fallback;            // ties inside the last bin: rank by sorting instead
  int32_t pad;
  unsigned long long psectors;  // pilot sample (automatic mode): distinct sectors ...
  unsigned long long pruns;     // ... over this many full runs
};

// Gathers this local (fewer distinct x sectors per run than this) coalesce
// and hit L1: no hub table is built for them (automatic mode), and K2 takes
// the L2 prefetch staging (resolve_prefetch).
constexpr int kLocalSectors = 16;

__global__ void __launch_bounds__(512) count_hist_kernel(const uint32_t* __restrict__ cnt,
                                                         int64_t n, uint32_t* __restrict__ hist,
                                                         HubPick* pick, int64_t S,
                                                         int64_t min_refs) {
  if (int64_t(pick->cmax) * S <= min_refs) return;  // no table (counted by the sample)
  __shared__ uint32_t h[kHistBins];
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  // counts 1..kLow-1 (most sampled columns: every thread of a block would
  // hit the same few bins) are tallied in registers and added once per warp
  constexpr int kLow = 4;
  uint32_t low[kLow] = {};
  auto tally = [&](uint32_t c) {
    if (c < kLow) {
#pragma unroll
      for (int b = 1; b < kLow; ++b) low[b] += c == uint32_t(b) ? 1u : 0u;
      return;
    }
    if (c >= kHistBins - 1) {
      atomicAdd(&pick->capsum, (unsigned long long)c);
      atomicMax(&pick->capmax, c);
    }
    atomicAdd(&h[c < kHistBins - 1 ? c : kHistBins - 1], 1u);
  };
  // 16-byte loads, two per step in flight (cnt is 256-byte aligned)
  const int64_t n4 = n / 4;
  const int64_t tstride = int64_t(gridDim.x) * blockDim.x;
  const uint4* c4 = reinterpret_cast<const uint4*>(cnt);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += 2 * tstride) {
    const uint4 a = __ldcs(c4 + i);
    const uint4 b = i + tstride < n4 ? __ldcs(c4 + i + tstride) : make_uint4(0, 0, 0, 0);
    tally(a.x);
    tally(a.y);
    tally(a.z);
    tally(a.w);
    tally(b.x);
    tally(b.y);
    tally(b.z);
    tally(b.w);
  }
  for (int64_t i = n4 * 4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += tstride)
    tally(cnt[i]);
#pragma unroll
  for (int b = 1; b < kLow; ++b) {
    const uint32_t t = __reduce_add_sync(0xffffffffu, low[b]);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(&h[b], t);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

// One block: the hub set = the hmax columns of largest count above t (ties
// in ascending column order), i.e. exactly what sorting by (count desc,
// column asc) and taking the first min(hmax, #above t) picks.  pick must be
// zeroed before count_hist_kernel.
__global__ void __launch_bounds__(1024) hub_pick_kernel(const uint32_t* __restrict__ hist,
                                                        uint32_t t, int64_t hmax,
                                                        HubPick* pick, int64_t S,
                                                        int64_t min_refs) {
  if (int64_t(pick->cmax) * S <= min_refs) return;
  constexpr int kPer = kHistBins / 1024;
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ uint32_t top, s_tau;
  __shared__ unsigned long long tot;
  __shared__ int s_h;
  const int tid = threadIdx.x;
  const int r = 1023 - tid;  // bins [kPer*r, kPer*r + kPer): thread 0 holds the top
  if (tid == 0) {
    top = 0;
    s_h = 0;
    s_tau = 0;
  }
  __syncthreads();
  unsigned long long own = 0;
  uint32_t hv[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int b = kPer * r + k;
    hv[k] = hist[b];
    if (hv[k]) atomicMax(&top, uint32_t(b));
    if (b > int64_t(t)) own += hv[k];
  }
  unsigned long long above = 0;  // selectable columns in the bins above this thread's
  Scan(ts).ExclusiveSum(own, above);
  if (tid == 1023) tot = above + own;
  __syncthreads();
  if (tid == 0) pick->fallback = t >= uint32_t(kHistBins - 1) ? 1 : 0;
  const unsigned long long want = tot < (unsigned long long)(hmax > 0 ? hmax : 0)
                                      ? tot
                                      : (unsigned long long)(hmax > 0 ? hmax : 0);
  if (want > 0 && above < want && above + own >= want) {
    // this thread's bins hold the crossing
    unsigned long long cum = above;
    for (int k = kPer - 1; k >= 0; --k) {
      const int b = kPer * r + k;
      if (b <= int64_t(t) || hv[k] == 0) continue;
      if (cum + hv[k] >= want) {
        s_tau = uint32_t(b);
        s_h = int(want);
        pick->need = int32_t(want - cum);
        pick->ties = int32_t(hv[k]);
        if (b == kHistBins - 1 && want - cum < hv[k]) pick->fallback = 1;
        break;
      }
      cum += hv[k];
    }
  }
  __syncthreads();
  if (s_h == 0) return;  // block-uniform
  // sampled references the hubs cover: the bins above tau + need * tau
  const uint32_t tau = s_tau;
  unsigned long long cov = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int b = kPer * r + k;
    if (uint32_t(b) > tau)
      cov += b == kHistBins - 1 ? pick->capsum : (unsigned long long)b * hv[k];
  }
  unsigned long long cs = 0;
  Scan(ts).ExclusiveSum(cov, cs);
  if (tid == 1023) {
    pick->covered = cs + cov + (unsigned long long)pick->need * tau;
    pick->h = s_h;
    pick->tau = tau;
  }
}

// The hub set, ascending: every column counted above tau, plus the columns
// counted exactly tau up to the need-th such column in column order.  Three
// passes over chunks of kPickChunk columns, no global sort or select:
// pick_count (per chunk: columns above tau, ties), pick_scan (one block: the
// chunk holding the need-th tie, the exact cut inside it, every chunk's
// output offset), pick_write (per chunk: a block scan places its hubs).
constexpr int kPickChunk = 8192;
constexpr int kPickThreads = 256;
constexpr int kPickPer = kPickChunk / kPickThreads;  // consecutive columns per thread

__global__ void __launch_bounds__(kPickThreads) pick_count_kernel(
    const uint32_t* __restrict__ cnt, int64_t n, uint32_t tau, uint32_t* __restrict__ above,
    uint32_t* __restrict__ ties) {
  using Reduce = cub::BlockReduce<uint32_t, kPickThreads>;
  __shared__ typename Reduce::TempStorage tr;
  const int64_t base = int64_t(blockIdx.x) * kPickChunk;
  uint32_t ka = 0, kt = 0;
  for (int i = threadIdx.x * 4; i < kPickChunk && base + i < n; i += kPickThreads * 4) {
    if (base + i + 4 <= n) {  // 16-byte loads (cnt is 256-byte aligned)
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(cnt + base + i));
      ka += (v.x > tau) + (v.y > tau) + (v.z > tau) + (v.w > tau);
      kt += (v.x == tau) + (v.y == tau) + (v.z == tau) + (v.w == tau);
    } else {
      for (int j = 0; j < 4 && base + i + j < n; ++j) {
        ka += cnt[base + i + j] > tau;
        kt += cnt[base + i + j] == tau;
      }
    }
  }
  const uint32_t ta = Reduce(tr).Sum(ka);
  __syncthreads();
  const uint32_t tt = Reduce(tr).Sum(kt);
  if (threadIdx.x == 0) {
    above[blockIdx.x] = ta;
    ties[blockIdx.x] = tt;
  }
}

__global__ void __launch_bounds__(1024) pick_scan_kernel(
    const uint32_t* __restrict__ cnt, int64_t n, uint32_t tau,
    const uint32_t* __restrict__ above, const uint32_t* __restrict__ ties, int64_t nchunks,
    int64_t need, int64_t* __restrict__ chunk_off, int64_t* __restrict__ cut) {
  using Scan = cub::BlockScan<int64_t, 1024>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int64_t s_chunk, s_before, carry_t, carry_o;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_chunk = -1;
    s_before = 0;
    carry_t = 0;
    carry_o = 0;
  }
  __syncthreads();
  for (int64_t b0 = 0; b0 < nchunks; b0 += 1024) {  // block-uniform trip count
    const int64_t b = b0 + tid;
    const int64_t vt = b < nchunks ? int64_t(ties[b]) : 0;
    int64_t ex = 0;
    Scan(ts).ExclusiveSum(vt, ex);
    const int64_t t0 = carry_t + ex;  // ties in the chunks before b
    if (vt > 0 && t0 < need && t0 + vt >= need) {
      s_chunk = b;
      s_before = t0;
    }
    // ties this chunk admits, then the output offsets
    const int64_t adm = vt == 0 ? 0 : (t0 >= need ? 0 : (t0 + vt <= need ? vt : need - t0));
    const int64_t sel = (b < nchunks ? int64_t(above[b]) : 0) + adm;
    __syncthreads();
    int64_t off = 0;
    Scan(ts).ExclusiveSum(sel, off);
    if (b < nchunks) chunk_off[b] = carry_o + off;
    __syncthreads();
    if (tid == 1023) {
      carry_t += ex + vt;
      carry_o += off + sel;
    }
    __syncthreads();
  }
  if (s_chunk < 0) {  // no tie admitted
    if (tid == 0) *cut = 0;
    return;
  }
  // inside the crossing chunk: 8 consecutive columns per thread
  const int64_t base = s_chunk * kPickChunk + int64_t(tid) * 8;
  int64_t k = 0;
  for (int j = 0; j < 8; ++j) k += (base + j < n && cnt[base + j] == tau) ? 1 : 0;
  int64_t ex = 0;
  Scan(ts).ExclusiveSum(k, ex);
  const int64_t want = need - s_before;  // the want-th tie of the chunk (1-based)
  if (ex < want && ex + k >= want) {
    int64_t seen = ex;
    for (int j = 0; j < 8; ++j)
      if (base + j < n && cnt[base + j] == tau && ++seen == want) {
        *cut = base + j + 1;
        break;
      }
  }
}

__global__ void __launch_bounds__(kPickThreads) pick_write_kernel(
    const uint32_t* __restrict__ cnt, int64_t n, uint32_t tau, const int64_t* __restrict__ cut,
    const int64_t* __restrict__ chunk_off, int32_t* __restrict__ out) {
  using Scan = cub::BlockScan<uint32_t, kPickThreads>;
  __shared__ typename Scan::TempStorage ts;
  const int64_t base = int64_t(blockIdx.x) * kPickChunk + int64_t(threadIdx.x) * kPickPer;
  const int64_t cu = *cut;
  uint32_t c[kPickPer];
#pragma unroll
  for (int j = 0; j < kPickPer; j += 4) {
    if (base + j + 4 <= n) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(cnt + base + j));
      c[j] = v.x;
      c[j + 1] = v.y;
      c[j + 2] = v.z;
      c[j + 3] = v.w;
    } else {
      for (int q = 0; q < 4; ++q) c[j + q] = base + j + q < n ? cnt[base + j + q] : 0u;
    }
  }
  uint32_t mine = 0;
#pragma unroll
  for (int j = 0; j < kPickPer; ++j)
    mine += (c[j] > tau || (c[j] == tau && base + j < cu)) ? 1u : 0u;
  uint32_t ex = 0;
  Scan(ts).ExclusiveSum(mine, ex);
  if (!mine) return;
  int64_t o = chunk_off[blockIdx.x] + ex;
#pragma unroll
  for (int j = 0; j < kPickPer; ++j)
    if (c[j] > tau || (c[j] == tau && base + j < cu)) out[o++] = int32_t(base + j);
}

}  // namespace

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
  m->hub_prefix = 0;
  m->hub_coverage = 0.0;
  m->gather_sectors = -1.0;
  ++m->version;  // invalidates slot copies built over the old encoding
  ++m->gen;      // and the graphs captured over the old buffers
  const Tuning& tu = ctx->tuning;
  int slots = max_hub_slots(ctx, tu.warps_per_cta, tu.ctas_per_sm,
                            m->precision == MBX_F32 ? 14 : 7, m->precision, m->n_cols);
  if (max_hubs >= 0) slots = std::min(slots, max_hubs);
  if (slots <= 0 || m->nnz == 0 || m->n_cols == 0) return;
  // Automatic mode: a table only pays once K2 is bound by its gather
  // requests, not on a latency-bound small matrix (small_matrix_nnz).
  if (max_hubs < 0 && m->nnz < small_matrix_nnz(ctx)) return;
  const int64_t n = m->n_cols;
  const int64_t runs = (m->nnz + 31) / 32;
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
  // sample stride: at most ~kSampleRuns runs, but never so sparse that a
  // column at the hub threshold expects fewer than 16 sampled references
  // (a stencil's 27-reference columns must not pass by sampling luck)
  const int64_t S = std::max<int64_t>(
      1, std::min<int64_t>((runs + kSampleRuns - 1) / kSampleRuns, int64_t(min_refs) / 16));
  uint32_t* cnt = nullptr;
  MBX_CUDA(cudaMallocAsync(&cnt, n * 4 + 64, s));
  MBX_CUDA(cudaMemsetAsync(cnt, 0, n * 4, s));
  uint32_t* hist = nullptr;
  HubPick* dpick = nullptr;
  MBX_CUDA(cudaMallocAsync(&hist, kHistBins * 4 + sizeof(HubPick) + 64, s));
  dpick = reinterpret_cast<HubPick*>(hist + kHistBins);
  MBX_CUDA(cudaMemsetAsync(hist, 0, kHistBins * 4 + sizeof(HubPick), s));
  const int sector_shift = m->precision == MBX_F32 ? 3 : 2;
  const bool pilot = max_hubs < 0;  // automatic mode: local matrices get no table
  if (pilot) {
    constexpr int64_t kPilotRuns = int64_t(1) << 14;
    sector_sample_kernel<<<unsigned(ctx->sm_count) * 2, 256, 0, s>>>(
        m->cols, m->nnz, std::max<int64_t>(1, runs / kPilotRuns), sector_shift, &dpick->psectors);
    ++ctx->launches;
  }
  count_sample_kernel<<<unsigned(ctx->sm_count) * 2, 1024, 0, s>>>(
      m->cols, m->nnz, S, sector_shift, cnt, &dpick->cmax, &dpick->sectors, &dpick->full_runs,
      pilot ? &dpick->psectors : nullptr, kLocalSectors);
  ++ctx->launches;
  // one pass over the counts: their histogram, then the hub set's
  // threshold (hub_pick_kernel) -- one host synchronisation for the lot
  const int64_t cap_lines = m->nnz / (ctas * 50);
  const uint32_t t = uint32_t(min_refs_shared / S);
  const int64_t hmax = std::min<int64_t>(slots, cap_lines << (m->precision == MBX_F32 ? 5 : 4));
  count_hist_kernel<<<unsigned(ctx->sm_count) * 2, 512, 0, s>>>(cnt, n, hist, dpick, S,
                                                                int64_t(min_refs));
  hub_pick_kernel<<<1, 1024, 0, s>>>(hist, t, hmax, dpick, S, int64_t(min_refs));
  ctx->launches += 2;
  MBX_CUDA(cudaGetLastError());
  HubPick pick{};
  MBX_CUDA(cudaMemcpyAsync(&pick, dpick, sizeof(HubPick), cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(hist, s);
  m->gather_sectors = pick.full_runs ? double(pick.sectors) / double(pick.full_runs) : -1.0;
  const uint32_t cmax = pick.cmax;
  size_t tb = 0;
  void* temp = nullptr;
  // (stream-ordered: the selection's kernels, the slot copy and K2 follow
  // on the same stream, so nothing waits for them on the host)
  auto done = [&] { cudaFreeAsync(cnt, s); };
  if (pilot && pick.pruns && pick.psectors < (unsigned long long)kLocalSectors * pick.pruns) {
    // local gathers (the sample and selection kernels returned at once)
    m->gather_sectors = double(pick.psectors) / double(pick.pruns);
    return done();
  }
  // no column can reach even the shared-line threshold (a stencil: at most
  // 27 references per column): no table, nothing more to do
  if (int64_t(cmax) * S <= int64_t(min_refs)) return done();
  m->hub_prefix = 0;
  if (m->vmap) {
    // degree-relabelled: columns are already ranked by count (vertex v has
    // the v-th largest column count), so the candidates are the prefix in
    // order -- no selection, no sort, and the slot copy encodes a hub as
    // c < h without a lookup.  The sampled counts are noisy but the true ones
    // descend: their suffix maximum is the ranking used.
    const int cand = int(std::min<int64_t>(slots, n));
    std::vector<uint32_t> raw(cand), hc(cand);
    MBX_CUDA(cudaMemcpyAsync(raw.data(), cnt, size_t(cand) * 4, cudaMemcpyDeviceToHost, s));
    MBX_CUDA(cudaStreamSynchronize(s));
    if (cand > 0) hc[cand - 1] = raw[cand - 1];
    for (int i = cand - 2; i >= 0; --i) hc[i] = std::max(raw[i], hc[i + 1]);
    const int line_shift = m->precision == MBX_F32 ? 5 : 4;
    int h = 0;
    int64_t covered = 0;
    while (h < cand) {
      const bool fresh = (h & ((1 << line_shift) - 1)) == 0;
      if (int64_t(hc[h]) * S <= int64_t(fresh ? min_refs : min_refs_shared)) break;
      if (fresh && (int64_t(h) >> line_shift) + 1 > cap_lines) break;
      covered += int64_t(raw[h++]) * S;
    }
    if (h > 0) {
      MBX_CUDA(cudaMallocAsync(&m->hub_cols, size_t(h) * 4 + 64, s));
      iota_kernel<<<(h + 255) / 256, 256, 0, s>>>(m->hub_cols, h);
      ++ctx->launches;
      m->hub_avail = h;
      m->hub_prefix = 1;
      m->hub_coverage = std::min(1.0, double(covered) / double(m->nnz));
    }
    return done();
  }
  if (!pick.fallback) {
    // the hub set straight from the threshold: every column counted above
    // tau, plus the first `need` (in column order) counted exactly tau --
    // selected in ascending column order, which is the slot order
    const int h = pick.h;
    if (h > 0) {
      const int64_t nchunks = (n + kPickChunk - 1) / kPickChunk;
      uint32_t* chunk_cnt = nullptr;  // above | ties
      int64_t* chunk_off = nullptr;   // nchunks offsets, then the tie cut
      MBX_CUDA(cudaMallocAsync(&chunk_cnt, size_t(nchunks) * 8 + 64, s));
      MBX_CUDA(cudaMallocAsync(&chunk_off, size_t(nchunks + 1) * 8 + 64, s));
      int64_t* cut = chunk_off + nchunks;
      pick_count_kernel<<<unsigned(nchunks), kPickThreads, 0, s>>>(cnt, n, pick.tau, chunk_cnt,
                                                                   chunk_cnt + nchunks);
      pick_scan_kernel<<<1, 1024, 0, s>>>(cnt, n, pick.tau, chunk_cnt, chunk_cnt + nchunks,
                                          nchunks, int64_t(pick.need), chunk_off, cut);
      MBX_CUDA(cudaMallocAsync(&m->hub_cols, size_t(h) * 4 + 64, s));
      pick_write_kernel<<<unsigned(nchunks), kPickThreads, 0, s>>>(cnt, n, pick.tau, cut,
                                                                   chunk_off, m->hub_cols);
      ctx->launches += 3;
      cudaFreeAsync(chunk_cnt, s);
      cudaFreeAsync(chunk_off, s);
      m->hub_avail = h;
      m->hub_coverage = std::min(1.0, double(pick.covered) * double(S) / double(m->nnz));
    }
    return done();
  }
  // (ties among counts past the histogram's last bin) candidates: every
  // column whose (scaled) sampled count passes the lower threshold, ranked
  // by count descending (stable: ties in column order)
  uint8_t* flag = nullptr;
  int32_t *cid = nullptr, *cid_sorted = nullptr;
  uint32_t *ccnt = nullptr, *ccnt_sorted = nullptr;
  int64_t* dk = nullptr;
  MBX_CUDA(cudaMallocAsync(&flag, n + 64, s));
  MBX_CUDA(cudaMallocAsync(&dk, 64, s));
  const unsigned grid = unsigned(ctx->sm_count) * 8;
  flag_above_kernel<<<grid, 256, 0, s>>>(cnt, n, t, flag);
  ++ctx->launches;
  MBX_CUDA(cudaMallocAsync(&cid, n * 4 + 64, s));
  cub::CountingInputIterator<int32_t> it(0);
  tb = 0;
  MBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flag, cid, dk, n, s));
  MBX_CUDA(cudaMallocAsync(&temp, tb + 64, s));
  MBX_CUDA(cub::DeviceSelect::Flagged(temp, tb, it, flag, cid, dk, n, s));
  int64_t K = 0;
  MBX_CUDA(cudaMemcpyAsync(&K, dk, 8, cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(temp, s);
  cudaFreeAsync(flag, s);
  cudaFreeAsync(dk, s);
  if (K == 0) {
    cudaFreeAsync(cid, s);
    return done();
  }
  MBX_CUDA(cudaMallocAsync(&ccnt, K * 4 + 64, s));
  MBX_CUDA(cudaMallocAsync(&ccnt_sorted, K * 4 + 64, s));
  MBX_CUDA(cudaMallocAsync(&cid_sorted, K * 4 + 64, s));
  gather_counts_kernel<<<grid, 256, 0, s>>>(cnt, cid, K, ccnt);
  ++ctx->launches;
  tb = 0;
  MBX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, ccnt, ccnt_sorted, cid,
                                                      cid_sorted, int(K), 0, 32, s));
  MBX_CUDA(cudaMallocAsync(&temp, tb + 64, s));
  MBX_CUDA(cub::DeviceRadixSort::SortPairsDescending(temp, tb, ccnt, ccnt_sorted, cid,
                                                      cid_sorted, int(K), 0, 32, s));
  const int cand = int(std::min<int64_t>(slots, K));
  std::vector<uint32_t> hc(cand);
  std::vector<int32_t> hid(cand);
  MBX_CUDA(cudaMemcpyAsync(hc.data(), ccnt_sorted, size_t(cand) * 4, cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaMemcpyAsync(hid.data(), cid_sorted, size_t(cand) * 4, cudaMemcpyDeviceToHost, s));
  MBX_CUDA(cudaStreamSynchronize(s));
  // Each multiply gathers the hub values into a contiguous block once
  // (hub_gather_kernel) and every CTA copies that block with coalesced
  // loads: a hub costs ~1/32 of a request per CTA, so the table fills up to
  // the shared-memory budget with every column referenced more than
  // min_refs_shared times, under the same 2 %-of-a-CTA's-gathers line cap
  // as a relabelled prefix.
  const int line_shift = m->precision == MBX_F32 ? 5 : 4;  // entries per 128-byte line
  int h = 0;
  int64_t covered = 0;
  while (h < cand) {
    if (int64_t(hc[h]) * S <= int64_t(min_refs_shared)) break;
    if ((h & ((1 << line_shift) - 1)) == 0 && (int64_t(h) >> line_shift) + 1 > cap_lines) break;
    covered += int64_t(hc[h++]) * S;
  }
  if (h > 0) {
    // slots in ascending column order: a column's slot is then its rank
    // among the hub columns, which hub_word_map encodes in n/32 words
    MBX_CUDA(cudaMallocAsync(&m->hub_cols, size_t(h) * 4 + 64, s));
    size_t tk = 0;
    MBX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tk, cid_sorted, m->hub_cols, h, 0, 32, s));
    void* tsort = nullptr;
    MBX_CUDA(cudaMallocAsync(&tsort, tk + 64, s));
    MBX_CUDA(cub::DeviceRadixSort::SortKeys(tsort, tk, cid_sorted, m->hub_cols, h, 0, 32, s));
    cudaFreeAsync(tsort, s);
    m->hub_avail = h;
    // estimated from the sample when S > 1
    m->hub_coverage = std::min(1.0, double(covered) / double(m->nnz));
  }
  cudaFreeAsync(temp, s);
  cudaFreeAsync(ccnt, s);
  cudaFreeAsync(ccnt_sorted, s);
  cudaFreeAsync(cid, s);
  cudaFreeAsync(cid_sorted, s);
  done();
}

// The hub lookup of the encoders (caller frees): n_cols/32 + 1 words, 8 bytes
// each (4 MB at R-MAT scale 24), so the per-nonzero test hits L2 instead of
// an n_cols-entry slot table.
uint2* hub_word_map(mbx_context* ctx, const mbx_matrix* m) {
  cudaStream_t s = ctx->stream;
  uint2* map = nullptr;
  const size_t words = hub_map_words(m->n_cols);
  const size_t bytes = words * 8 + size_t(kHubBloomWords) * 4;
  MBX_CUDA(cudaMallocAsync(&map, bytes + 64, s));
  MBX_CUDA(cudaMemsetAsync(map, 0, bytes, s));
  hub_word_kernel<<<(m->hub_avail + 255) / 256, 256, 0, s>>>(
      m->hub_cols, m->hub_avail, map, reinterpret_cast<uint32_t*>(map + words));
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
  return map;
}

// The hub-encoded column array of the staged (layout 0) and generic K2
// paths: every reference to a hub becomes (INT32_MIN | slot).  The default
// slot-layout K2 encodes its slot copy directly and never needs it.
void ensure_cols_hub(mbx_context* ctx, const mbx_matrix* m_) {
  mbx_matrix* m = const_cast<mbx_matrix*>(m_);
  if (m->cols_hub || m->hub_avail <= 0) return;
  cudaStream_t s = ctx->stream;
  uint2* map = hub_word_map(ctx, m);
  MBX_CUDA(cudaMallocAsync(&m->cols_hub, m->nnz * 4 + 256, s));
  MBX_CUDA(cudaMemsetAsync(m->cols_hub, 0, m->nnz * 4 + 256, s));
  encode_kernel<<<unsigned(ctx->sm_count) * 8, 256, 0, s>>>(m->cols, m->nnz, map, m->cols_hub);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
  cudaFreeAsync(map, s);
}

}  // namespace mbx

