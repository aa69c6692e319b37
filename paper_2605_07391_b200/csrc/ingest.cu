// ingest.cu -- device side of the file formats:
//
//  * mbx_matrix_from_coo: coo_to_csr<T> (include/merbit/csr.hpp:43-88) on the
//    GPU for Matrix Market / MBMX inputs of any size.  normalize_coo's
//    contract is kept exactly: bounds check (dimension_error), stable
//    row-major order, duplicates summed in fp64 in their stable order (one
//    sequential run per key), one rounding to T at the end.  Stable LSD
//    radix sort of (row * n_cols + col) gives the same permutation as
//    std::stable_sort on (row, col).
//  * mbx_tile_cache_write / mbx_tile_cache_load: MBTL files straight from /
//    into a device TILE (layout in io.cpp).
#include <cub/cub.cuh>

#include <type_traits>

#include <memory>
#include <string>
#include <vector>

#include "mbx_internal.h"

namespace mbx {

void write_tile_cache_host(const std::string& path, const mbx_tile_info& info,
                           const uint32_t* tx, const uint32_t* ty, const uint32_t* ld,
                           int precision);
void read_tile_cache_host(const std::string& path, mbx_tile_info* info, uint32_t** tx,
                          uint32_t** ty, uint32_t** ld, int* precision);

namespace {

__global__ void coo_keys_kernel(const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                                int64_t n, int64_t n_rows, int64_t n_cols,
                                unsigned long long* __restrict__ keys, int64_t* __restrict__ idx,
                                int* bad) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = r[k], col = c[k];
    if (row < 0 || row >= n_rows || col < 0 || col >= n_cols) atomicExch(bad, 1);
    keys[k] = (unsigned long long)(row) * (unsigned long long)(n_cols) +
              (unsigned long long)(col);
    idx[k] = k;
  }
}

__global__ void run_heads_kernel(const unsigned long long* __restrict__ keys, int64_t n,
                                 int64_t* __restrict__ head) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x)
    head[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

// one thread per run head: the run's values summed left to right in fp64
// (normalize_coo: merged.back().value += e.value), then rounded to T once
template <typename T>
__global__ void merge_runs_kernel(const unsigned long long* __restrict__ keys,
                                  const int64_t* __restrict__ idx, const double* __restrict__ v,
                                  const int64_t* __restrict__ head,
                                  const int64_t* __restrict__ pos,
                                  int64_t n, int64_t n_cols, int64_t* __restrict__ out_row,
                                  int32_t* __restrict__ out_col, T* __restrict__ out_val) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x) {
    if (!head[k]) continue;
    const unsigned long long key = keys[k];
    double s = v[idx[k]];
    for (int64_t j = k + 1; j < n && keys[j] == key; ++j) s += v[idx[j]];
    const int64_t p = pos[k];
    out_row[p] = int64_t(key / (unsigned long long)n_cols);
    out_col[p] = int32_t(key % (unsigned long long)n_cols);
    out_val[p] = static_cast<T>(s);
  }
}

// row_offsets[r] = first merged entry with row >= r (rows are sorted)
__global__ void row_offsets_kernel(const int64_t* __restrict__ rows, int64_t m, int64_t n_rows,
                                   uint32_t* __restrict__ ro) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rows[mid] < r)
        lo = mid + 1;
      else
        hi = mid;
    }
    ro[r] = uint32_t(lo);
  }
}

// build_transition (solvers.hpp:36-74): every adjacency entry j -> i becomes
// the key (i * n + j) of P with the weight T(1) / T(outdeg(j)) computed in T
template <typename T>
__global__ void transition_keys_kernel(const uint32_t* __restrict__ ro,
                                       const int32_t* __restrict__ cols, int64_t n,
                                       unsigned long long* __restrict__ keys,
                                       T* __restrict__ w) {
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lid = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = wid; j < n; j += nw) {
    const uint32_t b = ro[j], e = ro[j + 1];
    const T weight = e > b ? T(1) / static_cast<T>(e - b) : T(0);
    for (uint32_t k = b + lid; k < e; k += 32) {
      keys[k] = (unsigned long long)(cols[k]) * (unsigned long long)(n) + (unsigned long long)(j);
      w[k] = weight;
    }
  }
}

__global__ void split_keys_kernel(const unsigned long long* __restrict__ keys, int64_t m,
                                  int64_t n, int64_t* __restrict__ rows,
                                  int32_t* __restrict__ cols) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += int64_t(gridDim.x) * blockDim.x) {
    rows[k] = int64_t(keys[k] / (unsigned long long)n);
    cols[k] = int32_t(keys[k] % (unsigned long long)n);
  }
}

// ---- degree_stats (csr.hpp:119-140): longest row and empty rows
__global__ void degree_stats_kernel(const uint32_t* __restrict__ ro, int64_t n,
                                    unsigned long long* out /* [0] max, [1] empty */) {
  unsigned long long mx = 0, empty = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long d = ro[r + 1] - ro[r];
    mx = d > mx ? d : mx;
    empty += d == 0;
  }
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = m2 > mx ? m2 : mx;
    empty += __shfl_xor_sync(0xffffffffu, empty, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, mx);
    if (empty) atomicAdd(out + 1, empty);
  }
}

// ---- degree relabelling (a locality preprocessing for graphs whose x
// does not fit L2): vertex v gets the rank of its column count, descending
// (ties: ascending id), applied to rows and columns alike
__global__ void count_columns_kernel(const int32_t* __restrict__ cols, int64_t nnz,
                                     uint32_t* __restrict__ cnt) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + cols[k], 1u);
}

__global__ void iota32_kernel(int32_t* v, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    v[i] = int32_t(i);
}

__global__ void invert_order_kernel(const int32_t* __restrict__ order, int64_t n,
                                    int32_t* __restrict__ rank) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    rank[order[i]] = int32_t(i);
}

// vertex v -> inner[v] -> outer[inner[v]]
__global__ void compose_map_kernel(const int32_t* __restrict__ inner,
                                   const int32_t* __restrict__ outer, int64_t n,
                                   int32_t* __restrict__ out) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += int64_t(gridDim.x) * blockDim.x)
    out[v] = outer[inner[v]];
}

__global__ void relabel_keys_kernel(const uint32_t* __restrict__ ro,
                                    const int32_t* __restrict__ cols, int64_t n,
                                    const int32_t* __restrict__ rank,
                                    unsigned long long* __restrict__ keys) {
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lid = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = wid; r < n; r += nw) {
    const unsigned long long rr = (unsigned long long)rank[r] * (unsigned long long)n;
    for (uint32_t k = ro[r] + lid; k < ro[r + 1]; k += 32)
      keys[k] = rr + (unsigned long long)rank[cols[k]];
  }
}

// new row lengths: row rank[r] of P' is row r of P
__global__ void relabel_lengths_kernel(const uint32_t* __restrict__ ro, int64_t n,
                                       const int32_t* __restrict__ rank,
                                       uint32_t* __restrict__ len) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x)
    len[rank[r]] = ro[r + 1] - ro[r];
}

// row r of P goes to row rank[r] of P' with its columns renamed (unsorted;
// a segmented sort orders them).  Each thread takes kScatterRun consecutive
// nonzeros and finds its first row once (binary search), so a hub row of
// 10^5..10^6 entries is spread over the whole grid instead of one warp.
constexpr int kScatterRun = 16;
template <typename T>
__global__ void relabel_scatter_kernel(const uint32_t* __restrict__ ro,
                                       const int32_t* __restrict__ cols,
                                       const T* __restrict__ vals, int64_t n, int64_t m,
                                       const int32_t* __restrict__ rank,
                                       const uint32_t* __restrict__ ro2,
                                       int32_t* __restrict__ cols2, T* __restrict__ vals2) {
  const int64_t chunks = (m + kScatterRun - 1) / kScatterRun;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < chunks;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k0 = t * kScatterRun;
    const int64_t k1 = k0 + kScatterRun < m ? k0 + kScatterRun : m;
    // last row r with ro[r] <= k0
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (int64_t(ro[mid]) <= k0) lo = mid; else hi = mid - 1;
    }
    int64_t r = lo;
    int64_t end = ro[r + 1];
    int64_t d = int64_t(ro2[rank[r]]) - int64_t(ro[r]);
    for (int64_t k = k0; k < k1; ++k) {
      while (k >= end) {  // next non-empty row
        ++r;
        end = ro[r + 1];
        d = int64_t(ro2[rank[r]]) - int64_t(ro[r]);
      }
      cols2[k + d] = rank[cols[k]];
      vals2[k + d] = vals[k];
    }
  }
}

// rows of at least `long_row` entries: (begin, length) pairs, appended
__global__ void long_rows_kernel(const uint32_t* __restrict__ ro, int64_t n, int64_t long_row,
                                 long long* __restrict__ out, unsigned int* count, unsigned cap) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t len = int64_t(ro[r + 1]) - ro[r];
    if (len >= long_row) {
      const unsigned i = atomicAdd(count, 1u);
      if (i < cap) {
        out[2 * i] = ro[r];
        out[2 * i + 1] = len;
      }
    }
  }
}

// Mid-length rows (R-MAT's degree clusters put ~70 % of the nonzeros in
// rows of 256..4096 entries) would each take CUB's one-CTA multi-pass
// large-segment path; they are sorted in shared memory instead: one CTA per
// row, a bitonic network over the row padded to a power of two.
constexpr int64_t kMidLo = 128, kMidHi = 8192;  // measured best split at s24 (38.7 ms)

__global__ void mid_rows_kernel(const uint32_t* __restrict__ ro, int64_t n, int64_t lo,
                                int64_t hi, long long* __restrict__ out,
                                unsigned int* count) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t len = int64_t(ro[r + 1]) - ro[r];
    if (len > lo && len <= hi) {
      const unsigned i = atomicAdd(count, 1u);
      out[2 * i] = ro[r];
      out[2 * i + 1] = len;
    }
  }
}

template <typename T>
__global__ void bitonic_rows_kernel(const int32_t* __restrict__ kin, const T* __restrict__ vin,
                                    int32_t* __restrict__ kout, T* __restrict__ vout,
                                    const long long* __restrict__ segs) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int64_t b = segs[2 * blockIdx.x];
  const int len = int(segs[2 * blockIdx.x + 1]);
  int pw = 1;
  while (pw < len) pw <<= 1;
  T* sv = reinterpret_cast<T*>(sm);
  int32_t* sk = reinterpret_cast<int32_t*>(sv + pw);
  for (int i = threadIdx.x; i < pw; i += blockDim.x) {
    sk[i] = i < len ? kin[b + i] : INT32_MAX;
    if (i < len) sv[i] = vin[b + i];
  }
  __syncthreads();
  for (int k = 2; k <= pw; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < pw; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const int32_t a = sk[i], c = sk[ixj];
          if ((a > c) == up) {
            sk[i] = c;
            sk[ixj] = a;
            const T t = sv[i];
            sv[i] = sv[ixj];
            sv[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    kout[b + i] = sk[i];
    vout[b + i] = sv[i];
  }
}

// begin / end offsets of a row batch relative to its first row; rows of at
// least `long_row` entries get an empty segment (sorted separately)
__global__ void rebase_offsets_kernel(const uint32_t* __restrict__ ro, int64_t r0, int64_t rows,
                                      int64_t long_row, int64_t mid_lo, int64_t mid_hi,
                                      int32_t* __restrict__ beg, int32_t* __restrict__ end) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = int64_t(ro[r0 + i]) - ro[r0], e = int64_t(ro[r0 + i + 1]) - ro[r0];
    const int64_t len = e - b;
    beg[i] = int32_t(b);
    end[i] = int32_t(len >= long_row || (len > mid_lo && len <= mid_hi) ? b : e);
  }
}

template <typename F>
int iguard(F&& f) {
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

unsigned grid_of(int64_t n, const mbx_context* ctx) {
  const int64_t b = (n + 255) / 256;
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(b, int64_t(ctx->sm_count) * 16)));
}

}  // namespace
}  // namespace mbx

extern "C" {

MBX_API int mbx_matrix_from_coo(mbx_context* ctx, int precision, const mbx_coo* coo,
                                mbx_matrix** out) {
  return mbx::iguard([&] {
    using mbx::fail;
    if (precision != MBX_F32 && precision != MBX_F64)
      fail(MBX_CONFIG_ERROR, "precision must be MBX_F32 or MBX_F64");
    if (coo->n_rows < 0 || coo->n_cols < 0 || coo->nnz < 0)
      fail(MBX_DIMENSION_ERROR, "negative COO dimensions");
    if (coo->n_cols >= (int64_t(1) << 31))
      fail(MBX_CAPACITY_ERROR, "n_cols must be < 2^31 (int32 device column indices)");
    if (coo->nnz > 0 && (!coo->rows || !coo->cols || !coo->vals))
      fail(MBX_DIMENSION_ERROR, "null COO arrays");
    mbx::DeviceGuard dg(ctx->device);  // the caller's device is restored
    cudaStream_t s = ctx->stream;
    const int64_t n = coo->nnz, nr = coo->n_rows, nc = coo->n_cols;
    auto dm = [&](size_t b) {
      void* p = nullptr;
      MBX_CUDA(cudaMallocAsync(&p, std::max<size_t>(b, 256), s));
      return p;
    };
    std::vector<void*> tmp;
    auto tm = [&](size_t b) {
      void* p = dm(b);
      tmp.push_back(p);
      return p;
    };
    auto release = [&] {
      for (void* p : tmp) cudaFreeAsync(p, s);
      tmp.clear();
    };
    auto m = std::make_unique<mbx_matrix>();
    m->ctx = ctx;
    m->precision = precision;
    m->n_rows = nr;
    m->n_cols = nc;
    const size_t vs = mbx::value_size(precision);
    try {
      int64_t merged = 0;
      int64_t* mrow = nullptr;
      if (n > 0) {
        auto* rows = static_cast<int64_t*>(tm(n * 8));
        auto* cols = static_cast<int64_t*>(tm(n * 8));
        auto* vals = static_cast<double*>(tm(n * 8));
        MBX_CUDA(cudaMemcpyAsync(rows, coo->rows, n * 8, cudaMemcpyHostToDevice, s));
        MBX_CUDA(cudaMemcpyAsync(cols, coo->cols, n * 8, cudaMemcpyHostToDevice, s));
        MBX_CUDA(cudaMemcpyAsync(vals, coo->vals, n * 8, cudaMemcpyHostToDevice, s));
        auto* keys = static_cast<unsigned long long*>(tm(n * 8));
        auto* keys2 = static_cast<unsigned long long*>(tm(n * 8));
        auto* idx = static_cast<int64_t*>(tm(n * 8));
        auto* idx2 = static_cast<int64_t*>(tm(n * 8));
        int* bad = static_cast<int*>(tm(64));
        MBX_CUDA(cudaMemsetAsync(bad, 0, 4, s));
        mbx::coo_keys_kernel<<<mbx::grid_of(n, ctx), 256, 0, s>>>(rows, cols, n, nr, nc, keys,
                                                                   idx, bad);
        ++ctx->launches;
        int hbad = 0;
        MBX_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaStreamSynchronize(s));
        if (hbad) {
          // normalize_coo reports the first offending entry (csr.hpp:44-51)
          for (int64_t k = 0; k < n; ++k)
            if (coo->rows[k] < 0 || coo->rows[k] >= nr || coo->cols[k] < 0 || coo->cols[k] >= nc)
              fail(MBX_DIMENSION_ERROR, "coo entry (" + std::to_string(coo->rows[k]) + ", " +
                                            std::to_string(coo->cols[k]) + ") outside " +
                                            std::to_string(nr) + "x" + std::to_string(nc));
        }
        const unsigned long long span =
            (unsigned long long)std::max<int64_t>(nr, 1) * (unsigned long long)std::max<int64_t>(nc, 1);
        int bits = 1;
        while (bits < 64 && (1ull << bits) < span) ++bits;
        size_t tb = 0;
        MBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, idx, idx2, n, 0, bits, s));
        void* temp = tm(tb);
        MBX_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys2, idx, idx2, n, 0, bits, s));
        auto* head = static_cast<int64_t*>(tm(n * 8 + 8));
        auto* pos = static_cast<int64_t*>(tm(n * 8 + 8));
        mbx::run_heads_kernel<<<mbx::grid_of(n, ctx), 256, 0, s>>>(keys2, n, head);
        size_t sb = 0;
        MBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, head, pos, n, s));
        void* st = tm(sb);
        MBX_CUDA(cub::DeviceScan::ExclusiveSum(st, sb, head, pos, n, s));
        int64_t last[2];
        MBX_CUDA(cudaMemcpyAsync(&last[0], pos + n - 1, 8, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaMemcpyAsync(&last[1], head + n - 1, 8, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaStreamSynchronize(s));
        merged = last[0] + last[1];
        if (merged > int64_t(0xFFFFFFFF))
          fail(MBX_CAPACITY_ERROR, "nonzero count " + std::to_string(merged) +
                                       " exceeds the 32-bit tile cursor");
        m->nnz = merged;
        m->vals = dm(merged * vs + 256);
        m->cols = static_cast<int32_t*>(dm(merged * 4 + 256));
        MBX_CUDA(cudaMemsetAsync(m->vals, 0, merged * vs + 256, s));
        MBX_CUDA(cudaMemsetAsync(m->cols, 0, merged * 4 + 256, s));
        mrow = static_cast<int64_t*>(tm(merged * 8));
        if (precision == MBX_F32)
          mbx::merge_runs_kernel<float><<<mbx::grid_of(n, ctx), 256, 0, s>>>(
              keys2, idx2, vals, head, pos, n, nc, mrow, m->cols, static_cast<float*>(m->vals));
        else
          mbx::merge_runs_kernel<double><<<mbx::grid_of(n, ctx), 256, 0, s>>>(
              keys2, idx2, vals, head, pos, n, nc, mrow, m->cols, static_cast<double*>(m->vals));
        ctx->launches += 2;
      } else {
        m->vals = dm(256);
        m->cols = static_cast<int32_t*>(dm(256));
        MBX_CUDA(cudaMemsetAsync(m->vals, 0, 256, s));
        MBX_CUDA(cudaMemsetAsync(m->cols, 0, 256, s));
        mrow = static_cast<int64_t*>(tm(8));
      }
      m->ro = static_cast<uint32_t*>(dm((nr + 1) * 4 + 64));
      mbx::row_offsets_kernel<<<mbx::grid_of(nr + 1, ctx), 256, 0, s>>>(mrow, merged, nr, m->ro);
      ++ctx->launches;
      MBX_CUDA(cudaGetLastError());
      MBX_CUDA(cudaStreamSynchronize(s));
      release();
    } catch (...) {
      release();
      cudaStreamSynchronize(s);
      for (void* p : {m->vals, static_cast<void*>(m->cols), static_cast<void*>(m->ro)})
        if (p) cudaFree(p);
      throw;
    }
    *out = m.release();
  });
}

MBX_API int mbx_matrix_build_transition(mbx_context* ctx, const mbx_matrix* a,
                                        mbx_matrix** out) {
  return mbx::iguard([&] {
    mbx::DeviceGuard dg0(ctx->device);
    mbx::ensure_csr(ctx, a);
    using mbx::fail;
    if (a->n_rows != a->n_cols)
      fail(MBX_DIMENSION_ERROR, "transition matrix needs a square adjacency (" +
                                    std::to_string(a->n_rows) + "x" + std::to_string(a->n_cols) +
                                    ")");
    cudaStream_t s = ctx->stream;
    const int64_t n = a->n_rows, m = a->nnz;
    const size_t vs = mbx::value_size(a->precision);
    auto dm = [&](size_t b) {
      void* p = nullptr;
      MBX_CUDA(cudaMallocAsync(&p, std::max<size_t>(b, 256), s));
      return p;
    };
    auto p = std::make_unique<mbx_matrix>();
    p->ctx = ctx;
    p->precision = a->precision;
    p->n_rows = p->n_cols = n;
    p->nnz = m;
    p->vals = dm(m * vs + 256);
    p->cols = static_cast<int32_t*>(dm(m * 4 + 256));
    p->ro = static_cast<uint32_t*>(dm((n + 1) * 4 + 64));
    MBX_CUDA(cudaMemsetAsync(p->vals, 0, m * vs + 256, s));
    MBX_CUDA(cudaMemsetAsync(p->cols, 0, m * 4 + 256, s));
    auto* keys = static_cast<unsigned long long*>(dm(m * 8 + 8));
    auto* keys2 = static_cast<unsigned long long*>(dm(m * 8 + 8));
    void* w = dm(m * vs + 8);
    auto* rows = static_cast<int64_t*>(dm(m * 8 + 8));
    const unsigned grid = unsigned(ctx->sm_count) * 16;
    if (m > 0) {
      if (a->precision == MBX_F32)
        mbx::transition_keys_kernel<float><<<grid, 256, 0, s>>>(a->ro, a->cols, n, keys,
                                                               static_cast<float*>(w));
      else
        mbx::transition_keys_kernel<double><<<grid, 256, 0, s>>>(a->ro, a->cols, n, keys,
                                                                static_cast<double*>(w));
      const unsigned long long span = (unsigned long long)n * (unsigned long long)n;
      int bits = 1;
      while (bits < 64 && (1ull << bits) < span) ++bits;
      // stable: equal (i, j) pairs keep their order, rows keep ascending sources
      size_t tb = 0;
      if (a->precision == MBX_F32) {
        MBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, static_cast<float*>(w),
                                                 static_cast<float*>(p->vals), m, 0, bits, s));
        void* tmp = dm(tb);
        MBX_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, static_cast<float*>(w),
                                                 static_cast<float*>(p->vals), m, 0, bits, s));
        cudaFreeAsync(tmp, s);
      } else {
        MBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2,
                                                 static_cast<double*>(w),
                                                 static_cast<double*>(p->vals), m, 0, bits, s));
        void* tmp = dm(tb);
        MBX_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, static_cast<double*>(w),
                                                 static_cast<double*>(p->vals), m, 0, bits, s));
        cudaFreeAsync(tmp, s);
      }
      mbx::split_keys_kernel<<<grid, 256, 0, s>>>(keys2, m, n, rows, p->cols);
      ctx->launches += 3;
    }
    mbx::row_offsets_kernel<<<mbx::grid_of(n + 1, ctx), 256, 0, s>>>(rows, m, n, p->ro);
    ++ctx->launches;
    MBX_CUDA(cudaGetLastError());
    for (void* q : {static_cast<void*>(keys), static_cast<void*>(keys2), w,
                    static_cast<void*>(rows)})
      cudaFreeAsync(q, s);
    MBX_CUDA(cudaStreamSynchronize(s));
    *out = p.release();
  });
}

MBX_API int mbx_matrix_degree_stats(mbx_context* ctx, const mbx_matrix* m, int sigma_threshold,
                                    mbx_degree_stats* out) {
  return mbx::iguard([&] {
    mbx::DeviceGuard dg0(ctx->device);
    mbx::ensure_csr(ctx, m);
    if (m->n_rows <= 0) mbx::fail(MBX_DIMENSION_ERROR, "degree stats of a matrix with no rows");
    cudaStream_t s = ctx->stream;
    unsigned long long* d = nullptr;
    MBX_CUDA(cudaMallocAsync(&d, 16, s));
    MBX_CUDA(cudaMemsetAsync(d, 0, 16, s));
    mbx::degree_stats_kernel<<<mbx::grid_of(m->n_rows, ctx), 256, 0, s>>>(m->ro, m->n_rows, d);
    ++ctx->launches;
    MBX_CUDA(cudaGetLastError());
    unsigned long long h[2];
    MBX_CUDA(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(d, s);
    MBX_CUDA(cudaStreamSynchronize(s));
    out->mean_degree = double(m->nnz) / double(m->n_rows);
    out->low_degree = out->mean_degree <= sigma_threshold ? 1 : 0;
    out->pad_ = 0;
    out->max_degree = int64_t(h[0]);
    out->empty_rows = int64_t(h[1]);
  });
}

MBX_API int mbx_matrix_relabel_by_degree(mbx_context* ctx, const mbx_matrix* a,
                                         mbx_matrix** out, int32_t* rank_host) {
  return mbx::iguard([&] {
    mbx::DeviceGuard dg0(ctx->device);
    mbx::ensure_csr(ctx, a);
    using mbx::fail;
    if (a->n_rows != a->n_cols) fail(MBX_DIMENSION_ERROR, "relabelling needs a square matrix");
    cudaStream_t s = ctx->stream;
    const int64_t n = a->n_rows, m = a->nnz;
    const size_t vs = mbx::value_size(a->precision);
    // scratch is released on every exit; the new matrix's buffers too unless
    // the call succeeds (a CUDA error part-way must not leak pool memory)
    struct Scratch {
      cudaStream_t s;
      std::vector<void*> tmp, kept;
      bool done = false;
      ~Scratch() {
        for (void* q : tmp) cudaFreeAsync(q, s);
        if (!done)
          for (void* q : kept) cudaFreeAsync(q, s);
      }
    } scratch{s, {}, {}};
    std::vector<void*>& tmp = scratch.tmp;
    auto dm = [&](size_t b, bool keep = false) {
      void* p = nullptr;
      MBX_CUDA(cudaMallocAsync(&p, std::max<size_t>(b, 256), s));
      (keep ? scratch.kept : tmp).push_back(p);
      return p;
    };
    const unsigned grid = unsigned(ctx->sm_count) * 16;
    auto* cnt = static_cast<uint32_t*>(dm(n * 4 + 64));
    auto* cnt2 = static_cast<uint32_t*>(dm(n * 4 + 64));
    auto* ids = static_cast<int32_t*>(dm(n * 4 + 64));
    auto* order = static_cast<int32_t*>(dm(n * 4 + 64));
    auto* rank = static_cast<int32_t*>(dm(n * 4 + 64));
    MBX_CUDA(cudaMemsetAsync(cnt, 0, n * 4 + 64, s));
    mbx::launch_count_columns(ctx, a->cols, m, n, cnt);
    mbx::iota32_kernel<<<grid, 256, 0, s>>>(ids, n);
    size_t tb = 0;
    MBX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, cnt, cnt2, ids, order, n, 0,
                                                        32, s));
    void* t1 = dm(tb);
    MBX_CUDA(cub::DeviceRadixSort::SortPairsDescending(t1, tb, cnt, cnt2, ids, order, n, 0, 32,
                                                        s));
    mbx::invert_order_kernel<<<grid, 256, 0, s>>>(order, n, rank);
    auto p = std::make_unique<mbx_matrix>();
    p->ctx = ctx;
    p->precision = a->precision;
    p->n_rows = p->n_cols = n;
    p->nnz = m;
    p->vals = dm(m * vs + 256, true);
    p->cols = static_cast<int32_t*>(dm(m * 4 + 256, true));
    p->ro = static_cast<uint32_t*>(dm((n + 1) * 4 + 64, true));
    MBX_CUDA(cudaMemsetAsync(p->vals, 0, m * vs + 256, s));
    MBX_CUDA(cudaMemsetAsync(p->cols, 0, m * 4 + 256, s));
    // P' = Q P Q^T without a global key sort: the new row offsets come from
    // the permuted row lengths, every row is copied to its new place with
    // renamed columns, and one segmented sort per row batch restores
    // ascending columns (8 bytes of scratch per nonzero at fp32 instead of
    // the ~30 of a 64-bit (row, column) key sort -- the first call in a
    // process pays for every byte the memory pool grows by)
    {
      auto* len = static_cast<uint32_t*>(dm((n + 1) * 4 + 64));
      MBX_CUDA(cudaMemsetAsync(len, 0, (n + 1) * 4 + 64, s));
      mbx::relabel_lengths_kernel<<<grid, 256, 0, s>>>(a->ro, n, rank, len);
      size_t tbs = 0;
      MBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tbs, len, p->ro, n + 1, s));
      void* ts = dm(tbs);
      MBX_CUDA(cub::DeviceScan::ExclusiveSum(ts, tbs, len, p->ro, n + 1, s));
      ctx->launches += 2;
    }
    if (m) {
      auto* cols_b = static_cast<int32_t*>(dm(m * 4 + 256));
      void* vals_b = dm(m * vs + 256);
      // unsorted rows into the B buffers, sorted by the segmented sort into p
      if (a->precision == MBX_F32)
        mbx::relabel_scatter_kernel<float><<<grid, 256, 0, s>>>(
            a->ro, a->cols, static_cast<const float*>(a->vals), n, m, rank, p->ro, cols_b,
            static_cast<float*>(vals_b));
      else
        mbx::relabel_scatter_kernel<double><<<grid, 256, 0, s>>>(
            a->ro, a->cols, static_cast<const double*>(a->vals), n, m, rank, p->ro, cols_b,
            static_cast<double*>(vals_b));
      ++ctx->launches;
      // row batches of < 2^30 nonzeros (CUB's item counts are int); one
      // batch needs no host copy of the offsets, only the long-row list
      constexpr int64_t kBatch = int64_t(1) << 30;
      // rows this long would be sorted by one CTA each (CUB's large-segment
      // path): they get a device-wide radix sort of their own instead
      constexpr int64_t kLongRow = 65536;
      const bool single = m < kBatch;
      std::vector<uint32_t> ro_h;
      std::vector<long long> longs;  // (begin, length) pairs
      if (!single) {
        ro_h.resize(n + 1);
        MBX_CUDA(cudaMemcpyAsync(ro_h.data(), p->ro, (n + 1) * 4, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaStreamSynchronize(s));
        for (int64_t r = 0; r < n; ++r)
          if (int64_t(ro_h[r + 1]) - ro_h[r] >= kLongRow) {
            longs.push_back(ro_h[r]);
            longs.push_back(int64_t(ro_h[r + 1]) - ro_h[r]);
          }
      } else {
        const unsigned cap = unsigned(m / kLongRow + 1);  // at most m / kLongRow such rows
        auto* lbuf = static_cast<long long*>(dm(size_t(cap) * 16 + 64));
        auto* lcnt = static_cast<unsigned int*>(dm(64));
        MBX_CUDA(cudaMemsetAsync(lcnt, 0, 4, s));
        mbx::long_rows_kernel<<<grid, 256, 0, s>>>(p->ro, n, kLongRow, lbuf, lcnt, cap);
        ++ctx->launches;
        unsigned nl = 0;
        MBX_CUDA(cudaMemcpyAsync(&nl, lcnt, 4, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaStreamSynchronize(s));
        longs.resize(size_t(nl) * 2);
        if (nl)
          MBX_CUDA(cudaMemcpyAsync(longs.data(), lbuf, size_t(nl) * 16, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaStreamSynchronize(s));
      }
      // mid-length rows: (begin, length) lists for the shared-memory sort,
      // rows of <= 1024 entries first (the small class)
      // a mid row has > kMidLo entries, so there are at most m / kMidLo
      long long* mids = static_cast<long long*>(dm(size_t(m / mbx::kMidLo + 1) * 16 + 64));
      int64_t nmid = 0, nmid_small = 0;
      {
        auto* mcnt = static_cast<unsigned int*>(dm(64));
        MBX_CUDA(cudaMemsetAsync(mcnt, 0, 8, s));
        mbx::mid_rows_kernel<<<grid, 256, 0, s>>>(p->ro, n, mbx::kMidLo, 1024, mids, mcnt);
        unsigned c1 = 0;
        MBX_CUDA(cudaMemcpyAsync(&c1, mcnt, 4, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaStreamSynchronize(s));
        mbx::mid_rows_kernel<<<grid, 256, 0, s>>>(p->ro, n, 1024, mbx::kMidHi, mids + 2 * c1,
                                                  mcnt + 1);
        unsigned c2 = 0;
        MBX_CUDA(cudaMemcpyAsync(&c2, mcnt + 1, 4, cudaMemcpyDeviceToHost, s));
        MBX_CUDA(cudaStreamSynchronize(s));
        ctx->launches += 2;
        nmid_small = c1;
        nmid = int64_t(c1) + c2;
      }
      auto* offs = static_cast<int32_t*>(dm((n + 1) * 4 + 64));
      auto* offe = static_cast<int32_t*>(dm((n + 1) * 4 + 64));
      void* tsort = nullptr;
      size_t tsort_bytes = 0;
      for (int64_t r0 = 0; r0 < n;) {
        int64_t r1 = n;
        if (!single) {  // furthest r1 with ro[r1] - ro[r0] < kBatch (a longer row stands alone)
          int64_t lo = r0 + 1, hi = n;
          while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (int64_t(ro_h[mid]) - int64_t(ro_h[r0]) < kBatch) lo = mid; else hi = mid - 1;
          }
          r1 = lo;
        }
        const int64_t rows = r1 - r0;
        const int64_t base = single ? 0 : int64_t(ro_h[r0]);
        const int64_t items = single ? m : int64_t(ro_h[r1]) - base;
        if (items > 0) {
          mbx::rebase_offsets_kernel<<<mbx::grid_of(rows + 1, ctx), 256, 0, s>>>(
              p->ro, r0, rows, kLongRow, mbx::kMidLo, mbx::kMidHi, offs, offe);
          ++ctx->launches;
          // ping-pong between the B buffers and p (no internal copies in
          // the temp storage); a batch that ends in B is copied over
          auto sort = [&](auto* vb, auto* vp) {
            using V = std::remove_pointer_t<decltype(vb)>;
            cub::DoubleBuffer<int32_t> kd(cols_b + base, p->cols + base);
            cub::DoubleBuffer<V> vd(vb + base, vp + base);
            size_t need = 0;
            MBX_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, need, kd, vd, int(items),
                                                         int(rows), offs, offe, s));
            if (need > tsort_bytes) {
              if (tsort) cudaFreeAsync(tsort, s);
              MBX_CUDA(cudaMallocAsync(&tsort, need, s));
              tsort_bytes = need;
            }
            MBX_CUDA(cub::DeviceSegmentedSort::SortPairs(tsort, need, kd, vd, int(items),
                                                         int(rows), offs, offe, s));
            if (kd.Current() != p->cols + base)
              MBX_CUDA(cudaMemcpyAsync(p->cols + base, kd.Current(), items * 4,
                                       cudaMemcpyDeviceToDevice, s));
            if (vd.Current() != vp + base)
              MBX_CUDA(cudaMemcpyAsync(vp + base, vd.Current(), items * sizeof(V),
                                       cudaMemcpyDeviceToDevice, s));
            // the long rows of this batch: their unsorted copy is still in B
            int bits = 1;
            while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
            for (size_t i = 0; i < longs.size(); i += 2) {
              const int64_t b = longs[i], len = longs[i + 1];
              if (b < base || b >= base + items) continue;
              size_t need2 = 0;
              MBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need2, cols_b + b, p->cols + b,
                                                       vb + b, vp + b, int(len), 0, bits, s));
              if (need2 > tsort_bytes) {
                if (tsort) cudaFreeAsync(tsort, s);
                MBX_CUDA(cudaMallocAsync(&tsort, need2, s));
                tsort_bytes = need2;
              }
              MBX_CUDA(cub::DeviceRadixSort::SortPairs(tsort, need2, cols_b + b, p->cols + b,
                                                       vb + b, vp + b, int(len), 0, bits, s));
              ++ctx->launches;
            }
          };
          if (a->precision == MBX_F32)
            sort(static_cast<float*>(vals_b), static_cast<float*>(p->vals));
          else
            sort(static_cast<double*>(vals_b), static_cast<double*>(p->vals));
          ++ctx->launches;
        }
        r0 = r1;
      }
      // the mid-length rows, in shared memory, once every batch's copy-back
      // is done (their unsorted copy is still in the B buffers); two size
      // classes so short rows do not reserve a long row's tile
      auto mid_sort = [&](auto* vb, auto* vp) {
        using V = std::remove_pointer_t<decltype(vb)>;
        const size_t es = sizeof(V) + 4;
        MBX_CUDA(cudaFuncSetAttribute(mbx::bitonic_rows_kernel<V>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(mbx::kMidHi) * es)));
        if (nmid_small)
          mbx::bitonic_rows_kernel<V><<<unsigned(nmid_small), 256, 1024 * es, s>>>(
              cols_b, vb, p->cols, vp, mids);
        if (nmid > nmid_small)
          mbx::bitonic_rows_kernel<V><<<unsigned(nmid - nmid_small), 1024,
                                        size_t(mbx::kMidHi) * es, s>>>(
              cols_b, vb, p->cols, vp, mids + 2 * nmid_small);
        ctx->launches += 2;
        MBX_CUDA(cudaGetLastError());
      };
      if (nmid) {
        if (a->precision == MBX_F32)
          mid_sort(static_cast<float*>(vals_b), static_cast<float*>(p->vals));
        else
          mid_sort(static_cast<double*>(vals_b), static_cast<double*>(p->vals));
      }
      if (tsort) cudaFreeAsync(tsort, s);
    }
    ctx->launches += 3;
    MBX_CUDA(cudaGetLastError());
    if (rank_host && n)
      MBX_CUDA(cudaMemcpyAsync(rank_host, rank, n * 4, cudaMemcpyDeviceToHost, s));
    // the new matrix keeps the vertex map (composed with the input's own)
    p->vmap = static_cast<int32_t*>(dm(n * 4 + 64, true));
    if (a->vmap) {
      mbx::compose_map_kernel<<<grid, 256, 0, s>>>(a->vmap, rank, n, p->vmap);
      ++ctx->launches;
    } else if (n) {
      MBX_CUDA(cudaMemcpyAsync(p->vmap, rank, n * 4, cudaMemcpyDeviceToDevice, s));
    }
    MBX_CUDA(cudaStreamSynchronize(s));
    scratch.done = true;
    *out = p.release();
  });
}

MBX_API int mbx_tile_cache_write(const mbx_tile* t, const char* path, int precision) {
  return mbx::iguard([&] {
    std::vector<uint32_t> tx(t->info.tile_num + 1), ty(t->info.tile_num + 1),
        ld(std::max<int64_t>(t->info.lane_num, 1));
    const int rc = mbx_tile_download(t, tx.data(), ty.data(), ld.data());
    if (rc) mbx::fail(rc, mbx_last_error());
    mbx::write_tile_cache_host(path, t->info, tx.data(), ty.data(), ld.data(), precision);
  });
}

MBX_API int mbx_tile_cache_load(mbx_context* ctx, const char* path, mbx_tile** out,
                                int* precision) {
  return mbx::iguard([&] {
    mbx_tile_info info{};
    uint32_t *tx = nullptr, *ty = nullptr, *ld = nullptr;
    mbx::read_tile_cache_host(path, &info, &tx, &ty, &ld, precision);
    const int rc = mbx_tile_upload(ctx, &info, tx, ty, ld, out);
    std::free(tx);
    std::free(ty);
    std::free(ld);
    if (rc) mbx::fail(rc, mbx_last_error());
  });
}

}  // extern "C"
