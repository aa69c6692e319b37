// kernels.cu -- the sm_100a kernels of the MERBIT hot path.
//
//  K1 gen_tile_kernel      generate_tile (src/tile.cpp:17-85; paper Alg. 2)
//  K2 spmv_slot_kernel     spmv_merbit tile loop (merbit_spmv.hpp:182-324;
//                          paper Alg. 3-5) over the lane-major slot copy
//                          (default: omega 32, default sigma)
//     spmv_w32_kernel      the same over CSR order staged through shared
//                          memory (any sigma at omega 32; layout 0)
//     spmv_generic_kernel  any omega (the reference's small test configs)
//                          -- all three fuse the PageRank update
//                          (solvers.hpp:99-115) into the commit in PR mode
//  K3 fixup_kernel         ordered boundary-carry fold (merbit_spmv.hpp:
//                          328-337) + PageRank scalar finalisation
//  csr_kernel              spmv_csr_reference (reference.hpp:15-46): the
//                          pagerank yardstick (solvers.hpp:178-191)
//
// Design: SpMV is gather-bound integer/fp work, so no tensor
// cores.  Values/columns stream once with non-allocating loads tagged L2
// evict-first; x is gathered through the read-only path and kept
// L2-resident, its most referenced entries staged in shared memory (the hub
// table); every row of y is ASSIGNED exactly once (interior rows by the warp
// that closes them, boundary rows by K3), so no zero-fill, no atomics, and
// bitwise run-to-run determinism.
#include <atomic>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "mbx_internal.h"


namespace mbx {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;  // K2 CTA: 8 warps

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 16-byte streaming loads (values / columns are touched exactly once).
__device__ __forceinline__ void ld_stream16(const float* p, float (&v)[4], uint64_t pol) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_stream16(const double* p, double (&v)[2], uint64_t pol) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v[0]), "=d"(v[1])
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_cols(const int32_t* p, int (&c)[4], uint64_t pol) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3])
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_cols(const int32_t* p, int (&c)[2], uint64_t pol) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
               : "=r"(c[0]), "=r"(c[1])
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(pol));
  return v;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// Opt a kernel in to the device's full dynamic shared memory once per
// (kernel, device).  `done` is the calling launcher's own bitmask of devices
// (one per kernel instantiation -- kernels of one signature share a pointer
// TYPE, so the memo cannot live in a template over that type), updated
// atomically: cudaFuncSetAttribute is idempotent, so two threads racing on
// the same device both set it and both see the bit.
template <typename K>
void allow_max_smem(K kern, int device, std::atomic<uint64_t>& done) {
  const uint64_t bit = device < 64 ? (uint64_t(1) << device) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return;
  int optin = 0;
  MBX_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  MBX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// Programmatic dependent launch (PDL): K2 and K3 are launched so that the
// next one is scheduled while the previous one drains (its launch latency and
// CTA rasterisation overlap the tail); each waits for its predecessor's
// completion and memory before reading anything it produced, and lets its
// own dependent launch right away (whose CTAs then wait the same way).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// cudaLaunchKernelEx with the PDL attribute (MBX_PDL=0 disables it)
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MBX_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
// (used for the plain SpMV: inside the PageRank graphs, whose kernel
// boundaries are already cheap, it measured 1 % slower)
template <typename... KArgs, typename... Args>
void launch_pdl(bool on, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = on && pdl_enabled() ? 1 : 0;
  MBX_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

template <typename T>
struct VecOf {
  static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// x hub table preamble: hub[i] = x[hub_cols[i]], eight independent gathers
// in flight per thread (a one-at-a-time loop costs ~hubs/blockDim serial L2
// round trips before the CTA's first tile).
template <typename T>
__device__ __forceinline__ void stage_hubs(T* hub, const T* __restrict__ x,
                                           const int32_t* __restrict__ hub_cols, int hc,
                                           const T* __restrict__ hub_x) {
  if (hub_x) {
    // the hub values are contiguous (a degree-relabelled x, whose hubs are
    // its first entries, or the per-multiply hub gather): 16-byte copies,
    // 1/32 of the requests of a scattered table
    constexpr int V = 16 / int(sizeof(T));
    const int nv = hc / V;
    for (int i = threadIdx.x; i < nv; i += blockDim.x)
      reinterpret_cast<float4*>(hub)[i] = __ldg(reinterpret_cast<const float4*>(hub_x) + i);
    for (int i = nv * V + threadIdx.x; i < hc; i += blockDim.x) hub[i] = __ldg(hub_x + i);
    __syncthreads();
    return;
  }
  constexpr int U = 8;
  for (int i0 = threadIdx.x; i0 < hc; i0 += blockDim.x * U) {
    int idx[U];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      idx[u] = i < hc ? __ldg(hub_cols + i) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = idx[u] >= 0 ? __ldg(x + idx[u]) : T(0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < hc) hub[i] = v[u];
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Product staging: values[p] * x[col[p]] for p in [x0, x1).  ACCUM: return
// this lane's running sum (fast path, merbit_spmv.hpp:58-77); else store
// products to buf[p - x0] (merbit_spmv.hpp:244-249).  Lanes own aligned
// 16-byte vectors, so the element->lane map is a pure function of x0.
// ---------------------------------------------------------------------------
template <typename T, bool ACCUM, int MAXV, bool HUB>
__device__ __forceinline__ T stage_products(const T* __restrict__ vals,
                                            const int32_t* __restrict__ cols,
                                            const T* __restrict__ x, const T* hub,
                                            int64_t x0, int64_t x1, T* buf, int lid,
                                            uint64_t pol) {
  constexpr int N = VecOf<T>::N;
  const int64_t a0 = x0 & ~int64_t(N - 1);
  const int nvec = static_cast<int>((x1 - a0 + N - 1) / N);
  // Three explicit phases so each tile pays one DRAM latency (all column and
  // value vectors in flight together) and one L2 latency (all gathers in
  // flight together) instead of one of each per 16-byte vector.
  int col[MAXV][N];
  T val[MAXV][N];
#pragma unroll
  for (int it = 0; it < MAXV; ++it) {
    const int v = lid + 32 * it;
    if (v < nvec) {
      ld_cols(cols + a0 + int64_t(v) * N, col[it], pol);
    } else {
#pragma unroll
      for (int e = 0; e < N; ++e) col[it][e] = 0;
    }
  }
  // element (it, e) sits at tile-relative position k = lead + (lid+32it)*N + e;
  // it is live iff 0 <= k < cnt -- one unsigned compare
  const int lead = static_cast<int>(a0 - x0);  // in (-N, 0]
  const unsigned cnt = static_cast<unsigned>(x1 - x0);
  T xv[MAXV][N];
#pragma unroll
  for (int it = 0; it < MAXV; ++it) {
#pragma unroll
    for (int e = 0; e < N; ++e) {
      const unsigned k = static_cast<unsigned>(lead + (lid + 32 * it) * N + e);
      // hub columns (sign bit set) are served from shared memory; the rest
      // are gathered through the read-only path
      if (k >= cnt)
        xv[it][e] = T(0);
      else if (HUB && col[it][e] < 0)
        xv[it][e] = hub[col[it][e] & 0x7FFFFFFF];
      else
        xv[it][e] = __ldg(x + col[it][e]);
    }
  }
  // values last: their DRAM latency overlaps the gathers' L2 latency, and
  // the column registers are already free (64-register budget at 1024 thr)
#pragma unroll
  for (int it = 0; it < MAXV; ++it) {
    const int v = lid + 32 * it;
    if (v < nvec) {
      ld_stream16(vals + a0 + int64_t(v) * N, val[it], pol);
    } else {
#pragma unroll
      for (int e = 0; e < N; ++e) val[it][e] = T(0);
    }
  }
  T acc = T(0);
#pragma unroll
  for (int it = 0; it < MAXV; ++it) {
#pragma unroll
    for (int e = 0; e < N; ++e) {
      const unsigned k = static_cast<unsigned>(lead + (lid + 32 * it) * N + e);
      if (k < cnt) {
        const T p = val[it][e] * xv[it][e];
        if (ACCUM)
          acc += p;
        else
          buf[k] = p;
      }
    }
  }
  return acc;
}

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }

// ---------------------------------------------------------------------------
// PageRank commit of one finished row w = (P pi_old)[row]:
//   pi_new = damping * w + base  (rank_update, solvers.hpp:99-115)
// plus the fused reductions (fp64): L1 residual, dangling mass of pi_new
// (feeds the next iteration's base), mass (zero-norm check, 201-206) and
// ERR vs the yardstick (rank_error, 118-131).
// ---------------------------------------------------------------------------
struct PrAcc {
  double resid = 0.0, dang = 0.0, mass = 0.0, err = 0.0;
};

// po = pi_old[row], dang = row is a dangling vertex (both may be preloaded).
// With a constant yardstick s (reference_iters == 0) the accumulator holds
// max|pi - s| and the division happens once in pr_block_finish: division by
// a positive constant is monotone, so max(fl(|d|/s)) == fl(max|d| / s) and
// ERR stays bitwise equal to rank_error's formula.
// c * w + base with the product rounded first, as rank_update computes it
// (solvers.hpp:110-112; no contraction into an FMA)
template <typename T>
__device__ __forceinline__ T pr_value(const PrArgs& pr, T base, T w) {
  return mul_rn(static_cast<T>(pr.damping), w) + base;
}

// pi_new[row] = pn, plus (row shards) the exchange copy of a non-dangling
// vertex in this rank's buffer and, fused exchange, in every peer's
template <typename T>
__device__ __forceinline__ void pr_store(const PrArgs& pr, int64_t row, T pn,
                                         T* __restrict__ out) {
  out[row] = pn;
  if (pr.xout) {
    const int32_t q = pr.xmap[row];
    if (q >= 0) {
      static_cast<T*>(pr.xout)[q] = pn;
      for (int k = 0; k < pr.npeer; ++k) static_cast<T*>(pr.xpeer[k])[q] = pn;  // NVLink
    }
  }
}

// One committed row's share of the fused reductions.  |pn - po| is formed
// in T (the reference's own precision for pi) and accumulated in fp64.
template <typename T>
__device__ __forceinline__ void pr_accum(const PrArgs& pr, int64_t row, T pn, T po, bool dang,
                                         PrAcc& a) {
  a.resid += static_cast<double>(fabs(pn - po));
  if (dang) a.dang += static_cast<double>(pn);
  a.mass += fabs(static_cast<double>(pn));
  if (pr.yardstick) {
    const double s = static_cast<double>(reinterpret_cast<const T*>(pr.yardstick)[row]);
    const double d = static_cast<double>(pn) - s;
    if (s == 0.0) {
      if (d != 0.0) a.err = INFINITY;
    } else {
      a.err = fmax(a.err, fabs(d / s));
    }
  } else {
    a.err = fmax(a.err, fabs(static_cast<double>(pn) - pr.yard_const));
  }
}

template <typename T>
__device__ __forceinline__ void pr_commit_v(const PrArgs& pr, T base, int64_t row, T w, T po,
                                            bool dang, T* __restrict__ out, PrAcc& a) {
  const T pn = pr_value(pr, base, w);
  pr_store(pr, row, pn, out);
  pr_accum(pr, row, pn, po, dang, a);
}

__device__ __forceinline__ bool pr_dang(const PrArgs& pr, int64_t row) {
  return pr.dang_from >= 0 ? row >= pr.dang_from
                           : ((__ldg(pr.dangling + (row >> 5)) >> (row & 31)) & 1u) != 0u;
}

template <typename T>
__device__ __forceinline__ void pr_commit(const PrArgs& pr, T base, int64_t row,
                                          T w, T* __restrict__ out, PrAcc& a) {
  pr_commit_v<T>(pr, base, row, w, reinterpret_cast<const T*>(pr.pi_old)[row], pr_dang(pr, row),
                 out, a);
}

// K2, PageRank: the range's head and tail rows go through the carry table;
// K3 commits them and its row reduction must skip them
__device__ __forceinline__ void mark_carry_rows(const PrArgs& pr, uint32_t head_row,
                                                uint32_t tail_row, int64_t n_rows) {
  if (int64_t(head_row) < n_rows) atomicOr(pr.carry_mask + (head_row >> 5), 1u << (head_row & 31));
  if (int64_t(tail_row) < n_rows) atomicOr(pr.carry_mask + (tail_row >> 5), 1u << (tail_row & 31));
}

// iteration bookkeeping of host-unrolled launches (prev/next/iter baked in)
// and of the device-driven loop (derived from *iter_dev)
__device__ __forceinline__ bool pr_skip(const PrArgs& pr) {
  return *pr.stop || (pr.iter_dev && *pr.iter_dev >= pr.max_iters);
}
__device__ __forceinline__ const PrScalars* pr_prev(const PrArgs& pr) {
  return pr.iter_dev ? pr.scal_base + *pr.iter_dev : pr.prev;
}
__device__ __forceinline__ PrScalars* pr_next(const PrArgs& pr) {
  // a baked `next` wins (row shards: the parity's chunk tail)
  return pr.next ? pr.next : pr.scal_base + *pr.iter_dev + 1;
}
__device__ __forceinline__ int pr_iter(const PrArgs& pr) {
  return pr.iter_dev ? int(*pr.iter_dev + 1) : pr.iter;
}

template <typename T>
__device__ __forceinline__ T pr_base(const PrArgs& pr) {
  // base = (damping * dangling_mass + 1 - damping) / n, in fp64 then T
  return static_cast<T>((pr.damping * pr_prev(pr)->dangling + (1.0 - pr.damping)) * pr.inv_n);
}

// Deterministic block reduction of PrAcc (fixed butterfly + fixed warp order)
// followed by the last-block finalisation into *out.
__device__ void pr_block_finish(PrAcc a, const PrArgs& pr, double* block_part,
                                unsigned int* counter, PrScalars* out, bool check_stop,
                                bool advance = false) {
  __shared__ double sm[4][32];
  __shared__ bool is_last;
  // fused exchange: this thread's NVLink stores are performed system-wide
  // before the grid completes (the peer barrier that follows publishes them)
  if (pr.npeer) __threadfence_system();
  a.resid = warp_sum(a.resid);
  a.dang = warp_sum(a.dang);
  a.mass = warp_sum(a.mass);
  a.err = warp_max(a.err);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (l == 0) {
    sm[0][w] = a.resid;
    sm[1][w] = a.dang;
    sm[2][w] = a.mass;
    sm[3][w] = a.err;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0, d = 0, m = 0, e = 0;
    for (int i = 0; i < nw; ++i) {
      r += sm[0][i];
      d += sm[1][i];
      m += sm[2][i];
      e = fmax(e, sm[3][i]);
    }
    double* bp = block_part + 4 * blockIdx.x;
    bp[0] = r;
    bp[1] = d;
    bp[2] = m;
    bp[3] = e;
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    is_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  PrAcc t;
  // L2-coherent (.cg) 16-byte loads of the other blocks' partials, unrolled so
  // the round trips overlap (a volatile loop pays one L2 latency per load)
  const unsigned nb = gridDim.x;
#pragma unroll 4
  for (unsigned int b = threadIdx.x; b < nb; b += blockDim.x) {
    const double2 a01 = __ldcg(reinterpret_cast<const double2*>(block_part + 4 * b));
    const double2 a23 = __ldcg(reinterpret_cast<const double2*>(block_part + 4 * b + 2));
    t.resid += a01.x;
    t.dang += a01.y;
    t.mass += a23.x;
    t.err = fmax(t.err, a23.y);
  }
  t.resid = warp_sum(t.resid);
  t.dang = warp_sum(t.dang);
  t.mass = warp_sum(t.mass);
  t.err = warp_max(t.err);
  __syncthreads();
  if (l == 0) {
    sm[0][w] = t.resid;
    sm[1][w] = t.dang;
    sm[2][w] = t.mass;
    sm[3][w] = t.err;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0, d = 0, m = 0, e = 0;
    for (int i = 0; i < nw; ++i) {
      r += sm[0][i];
      d += sm[1][i];
      m += sm[2][i];
      e = fmax(e, sm[3][i]);
    }
    if (!pr.yardstick) {  // constant yardstick: e = max|pi - s| so far
      const double s = pr.yard_const;
      e = s == 0.0 ? (e != 0.0 ? INFINITY : 0.0) : e / s;
    }
    out->resid = r;
    out->dangling = d;
    out->mass = m;
    out->err = e;
    for (int k = 0; k < pr.npeer; ++k) {  // the tail travels with the chunk
      PrScalars* o = reinterpret_cast<PrScalars*>(
          static_cast<char*>(pr.xpeer[k]) +
          (reinterpret_cast<char*>(out) - static_cast<char*>(pr.xout)));
      o->resid = r;
      o->dangling = d;
      o->mass = m;
      o->err = e;
    }
    if (pr.npeer) __threadfence_system();
    if (check_stop && pr.stop) {
      if (m == 0.0) {
        *pr.stop = 2;  // zero-norm iterate (solvers.hpp:202-205)
        *pr.stop_iter = pr_iter(pr);
      } else if (e < pr.err_tol) {
        *pr.stop = 1;  // converged (solvers.hpp:210-213)
        *pr.stop_iter = pr_iter(pr);
      }
    }
    *counter = 0;  // ready for the next launch
    // device-driven loop: this iteration is complete (every block of this
    // grid has read the old count; the next K2 is stream-ordered after us)
    if (advance && pr.iter_dev) *pr.iter_dev += 1;
  }
}

// ---------------------------------------------------------------------------
// K2, omega == 32: one warp walks `chunks_per_range` consecutive tiles.
// ---------------------------------------------------------------------------
template <typename T>
struct SpmvParams {
  const T* vals;
  const int32_t* cols;
  const T* x;
  T* y;
  const uint32_t* tile_x;
  const uint32_t* tile_y;
  const uint32_t* lane_desc;
  const int32_t* hub_cols;
  const T* hub_x;  // contiguous hub values (nullptr: gather x[hub_cols])
  uint32_t* carry_row;
  T* carry_val;
  Geometry g;
  PrArgs pr;
};

// Per-lane MERBIT walk of the lane's sigma steps (paper Alg. 4,
// merbit_spmv.hpp:251-297) + warp segmented sum (Alg. 5, 85-117), with the
// carry of the previous tile entering at lane 0.  Rows closed inside the
// chunk land in buf[cnt + row - y0]; returns the new carry (open row y1).
template <typename T, int SIGMA>
__device__ __forceinline__ T lane_walk_and_scan(T* buf, int cnt, int sigma, uint32_t d,
                                                int steps, int ob, int lid, T carry,
                                                int xo, int r0) {
  const uint32_t flags = d >> (2 * ob);
  int r = r0;
  T sum = T(0), head = T(0);
  bool had_down = false;
  const int S = SIGMA > 0 ? SIGMA : sigma;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    if (k < steps) {
      if ((flags >> k) & 1u) {
        if (!had_down) {
          head = sum;  // first closure: the row may extend into earlier lanes
          had_down = true;
        } else {
          buf[cnt + r] = sum;  // row opened and closed inside this lane
        }
        sum = T(0);
        ++r;
      } else {
        sum += buf[xo++];
      }
    }
  }
  T tail = sum;
  if (lid == 0) {
    if (had_down)
      head += carry;
    else
      tail += carry;
  }
  // inclusive segmented scan of the trailing sums (flag = lane closed a row)
  T S_ = tail;
  bool F = had_down;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T su = __shfl_up_sync(kFull, S_, off);
    const bool fu = __shfl_up_sync(kFull, F, off);
    if (lid >= off && !F) {
      S_ += su;
      F = fu;
    }
  }
  const T prevS = __shfl_up_sync(kFull, S_, 1);
  if (had_down) buf[cnt + r0] = head + (lid > 0 ? prevS : T(0));
  return __shfl_sync(kFull, S_, 31);
}

// One warp range: `chunks_per_range` consecutive tiles (chunk == tile here).
template <typename T, int SIGMA, bool PR, bool HUB, bool PF>
__device__ __forceinline__ void w32_range(const SpmvParams<T>& p, const T* hub, T* buf,
                                          int64_t range, int lid, uint64_t pol, T base) {
  const Geometry& g = p.g;
  const int sigma = SIGMA > 0 ? SIGMA : g.sigma;
  const int64_t c0 = range * g.chunks_per_range;
  const int nc = static_cast<int>(imin64(c0 + g.chunks_per_range, g.num_chunks) - c0);
  const int64_t total = g.nnz + g.n_rows;
  const int ob = g.ob;
  const uint32_t omask = (1u << ob) - 1u;
  constexpr int MAXV = SIGMA > 0 ? (32 * SIGMA + 2 * VecOf<T>::N + 31) / (32 * VecOf<T>::N) + 1 : 8;

  // tile cursors of this range, one coalesced load
  uint32_t mtx = 0, mty = 0;
  if (lid <= nc) {
    mtx = ld_stream_u32(p.tile_x + c0 + lid, pol);
    mty = ld_stream_u32(p.tile_y + c0 + lid, pol);
  }
  const uint32_t head_row = __shfl_sync(kFull, mty, 0) & ~kLongRowMask;
  const uint32_t tail_row = __shfl_sync(kFull, mty, nc) & ~kLongRowMask;
  T carry = T(0), head_val = T(0);
  bool head_open = true;

  for (int ci = 0; ci < nc; ++ci) {
    const int64_t c = c0 + ci;
    const uint32_t x0 = __shfl_sync(kFull, mtx, ci);
    const uint32_t x1 = __shfl_sync(kFull, mtx, ci + 1);
    const uint32_t ty0 = __shfl_sync(kFull, mty, ci);
    const uint32_t y0 = ty0 & ~kLongRowMask;
    const uint32_t y1 = __shfl_sync(kFull, mty, ci + 1) & ~kLongRowMask;
    const int cnt = static_cast<int>(x1 - x0);
    const int nrows = static_cast<int>(y1 - y0);
    if (PF && ci + 1 < nc) {
      // warm L2 with the next tile's value/column/descriptor lines so its
      // loads do not pay DRAM latency on the critical path
      const uint32_t px1 = __shfl_sync(kFull, mtx, ci + 2);
      const uintptr_t vb = reinterpret_cast<uintptr_t>(p.vals + x1) & ~uintptr_t(127);
      const uintptr_t ve = reinterpret_cast<uintptr_t>(p.vals + px1);
      const uintptr_t cb = reinterpret_cast<uintptr_t>(p.cols + x1) & ~uintptr_t(127);
      const uintptr_t ce = reinterpret_cast<uintptr_t>(p.cols + px1);
      const int nvl = static_cast<int>((ve - vb + 127) >> 7);
      const int ncl = static_cast<int>((ce - cb + 127) >> 7);
      for (int l = lid; l <= nvl + ncl; l += 32) {
        const uintptr_t a = l < nvl ? vb + (uintptr_t(l) << 7)
                            : l < nvl + ncl ? cb + (uintptr_t(l - nvl) << 7)
                                            : reinterpret_cast<uintptr_t>(p.lane_desc + (c + 1) * 32);
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a));
      }
    }
    if (ty0 & kLongRowMask) {
      // long-row tile: every step Right, one row (merbit_spmv.hpp:230-237)
      T s = stage_products<T, true, MAXV, HUB>(p.vals, p.cols, p.x, hub, x0, x1, buf, lid, pol);
      carry += warp_sum(s);
      continue;
    }
    if (cnt == 0) {
      // no nonzero: every step closes a row (merbit_spmv.hpp:217-224); the
      // first closes the carried row, the rest are empty rows.
      for (int k = lid; k < nrows; k += 32) buf[k] = k == 0 ? carry : T(0);
      carry = T(0);
    } else {
      // descriptor first: its load overlaps the staging loads/gathers
      const int64_t j = c * 32 + lid;
      const bool valid = j < g.lane_num;
      const uint32_t d = valid ? ld_stream_u32(p.lane_desc + j, pol) : 0u;
      const int steps = valid ? static_cast<int>(imin64(sigma, total - j * sigma)) : 0;
      stage_products<T, false, MAXV, HUB>(p.vals, p.cols, p.x, hub, x0, x1, buf, lid, pol);
      __syncwarp();
      carry = lane_walk_and_scan<T, SIGMA>(buf, cnt, sigma, d, steps, ob, lid, carry,
                                           static_cast<int>(d & omask),
                                           static_cast<int>((d >> ob) & omask));
    }
    __syncwarp();
    // coalesced commit of the rows closed in this tile (Alg. 6 load_mem)
    for (int k = lid; k < nrows; k += 32) {
      const T w = buf[cnt + k];
      if (k == 0 && head_open) {
        head_val = w;  // range head row: may continue from the previous range
        continue;
      }
      const int64_t row = int64_t(y0) + k;
      if (PR)
        pr_store<T>(p.pr, row, pr_value(p.pr, base, w), p.y);
      else
        p.y[row] = w;
    }
    if (nrows > 0) head_open = false;
    __syncwarp();
  }
  if (lid == 0) {
    p.carry_row[2 * range] = head_row;
    p.carry_val[2 * range] = head_open ? T(0) : head_val;
    p.carry_row[2 * range + 1] = tail_row;
    p.carry_val[2 * range + 1] = carry;
    if (PR) mark_carry_rows(p.pr, head_row, tail_row, g.n_rows);
  }
}

// K2, omega == 32: persistent CTAs; the x hub table is staged once per CTA,
// then each warp strides over ranges (all ranges carry equal merge-path work).
template <typename T, int SIGMA, bool PR, bool HUB, bool PF>
__global__ void __launch_bounds__(1024) spmv_w32_kernel(SpmvParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geometry& g = p.g;
  const int sigma = SIGMA > 0 ? SIGMA : g.sigma;
  if (PR && pr_skip(p.pr)) return;
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  T* hub = reinterpret_cast<T*>(smem_raw);
  const int hub_pad = HUB ? ((g.hub_count + 3) & ~3) : 0;
  T* buf = hub + hub_pad + size_t(warp) * (32 * sigma + 1);
  if (HUB) stage_hubs<T>(hub, p.x, p.hub_cols, g.hub_count, p.hub_x);
  const uint64_t pol = evict_first_policy();
  T base = T(0);
  if (PR) base = pr_base<T>(p.pr);
  const int64_t wstride = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t range = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp; range < g.num_ranges;
       range += wstride)
    w32_range<T, SIGMA, PR, HUB, PF>(p, hub, buf, range, lid, pol, base);
  if (PR && p.pr.npeer) __threadfence_system();  // NVLink stores performed (fused exchange)
}

// ---------------------------------------------------------------------------
// K2, any omega: lanes locate themselves through their own tile entry
// (lane start = tile start + descriptor offsets).  No fast/skip routing;
// used for the reference's small test configurations (omega = 4, ...).
// ---------------------------------------------------------------------------
template <typename T, bool PR>
__global__ void __launch_bounds__(kThreads) spmv_generic_kernel(SpmvParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geometry& g = p.g;
  const int sigma = g.sigma;
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int64_t range = int64_t(blockIdx.x) * g.warps_per_cta + warp;
  if (range >= g.num_ranges) return;
  if (PR && pr_skip(p.pr)) return;
  T* buf = reinterpret_cast<T*>(smem_raw) + size_t(warp) * (32 * sigma + 1);
  const uint64_t pol = evict_first_policy();
  const int64_t c0 = range * g.chunks_per_range;
  const int nc = static_cast<int>(imin64(c0 + g.chunks_per_range, g.num_chunks) - c0);
  const int64_t total = g.nnz + g.n_rows;
  const int ob = g.ob;
  const uint32_t omask = (1u << ob) - 1u;

  T carry = T(0), head_val = T(0);
  bool head_open = true;
  T base = T(0);
  if (PR) base = pr_base<T>(p.pr);
  uint32_t head_row = 0, y1 = 0;

  for (int ci = 0; ci < nc; ++ci) {
    const int64_t j = (c0 + ci) * 32 + lid;
    const bool valid = j < g.lane_num;
    int64_t lx = g.nnz, ly = g.n_rows;
    uint32_t d = 0;
    int steps = 0;
    if (valid) {
      const int64_t tile = j / g.omega;
      d = p.lane_desc[j];
      lx = int64_t(p.tile_x[tile]) + (d & omask);
      ly = int64_t(p.tile_y[tile] & ~kLongRowMask) + ((d >> ob) & omask);
      steps = static_cast<int>(imin64(sigma, total - j * sigma));
    }
    const uint32_t flags = d >> (2 * ob);
    const int live = steps >= 32 ? -1 : int((1u << steps) - 1u);
    const int downs = __popc(flags & uint32_t(live));
    const int rights = steps - downs;
    const int64_t x0 = __shfl_sync(kFull, lx, 0);
    const int64_t yy0 = __shfl_sync(kFull, ly, 0);
    const int64_t x1 = __shfl_sync(kFull, lx + rights, 31);
    const int64_t yy1 = __shfl_sync(kFull, ly + downs, 31);
    if (ci == 0) head_row = static_cast<uint32_t>(yy0);
    y1 = static_cast<uint32_t>(yy1);
    const int cnt = static_cast<int>(x1 - x0);
    const int nrows = static_cast<int>(yy1 - yy0);
    stage_products<T, false, 12, false>(p.vals, p.cols, p.x, nullptr, x0, x1, buf, lid, pol);
    __syncwarp();
    carry = lane_walk_and_scan<T, 0>(buf, cnt, sigma, d, steps, ob, lid, carry,
                                      static_cast<int>(lx - x0), static_cast<int>(ly - yy0));
    __syncwarp();
    for (int k = lid; k < nrows; k += 32) {
      const T w = buf[cnt + k];
      if (k == 0 && head_open) {
        head_val = w;
        continue;
      }
      const int64_t row = yy0 + k;
      if (PR)
        pr_store<T>(p.pr, row, pr_value(p.pr, base, w), p.y);
      else
        p.y[row] = w;
    }
    if (nrows > 0) head_open = false;
    __syncwarp();
  }
  if (lid == 0) {
    p.carry_row[2 * range] = head_row;
    p.carry_val[2 * range] = head_open ? T(0) : head_val;
    p.carry_row[2 * range + 1] = y1;
    p.carry_val[2 * range + 1] = carry;
    if (PR) mark_carry_rows(p.pr, head_row, y1, g.n_rows);
  }
  if (PR && p.pr.npeer) __threadfence_system();  // NVLink stores performed (fused exchange)
}

// ---------------------------------------------------------------------------
// K2 over the lane-major slot layout (omega == 32, default sigma).
//
// The slot copy (built once per TILE by build_slots_kernel) stores, for
// chunk c, the element lane l consumes at step i at
//   c*32*SIGMA + (i/G)*32*G + l*G + i%G      (G = 8/sizeof(T) elements)
// -- zero for Down steps; for marked tiles lane l step i holds element
// 32*i + l, i.e. exactly the lane-strided order of fast_tile_reduce
// (merbit_spmv.hpp:58-77).  Each lane therefore receives its own sigma
// operands with coalesced 8-byte loads and walks them in registers: no
// product staging, no shared-memory transposition (the L1 data pipe was
// the co-limiter with the gather request port, profiles/).
// ---------------------------------------------------------------------------
template <typename T, int SIGMA>
__device__ __forceinline__ void load_slot_vals(const T* base, int lid, T (&v)[SIGMA],
                                               uint64_t pol);
template <>
__device__ __forceinline__ void load_slot_vals<float, 14>(const float* base, int lid,
                                                          float (&v)[14], uint64_t pol) {
#pragma unroll
  for (int g = 0; g < 7; ++g)
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
        : "=f"(v[2 * g]), "=f"(v[2 * g + 1])
        : "l"(base + g * 64 + 2 * lid), "l"(pol));
}
template <>
__device__ __forceinline__ void load_slot_vals<double, 7>(const double* base, int lid,
                                                          double (&v)[7], uint64_t pol) {
#pragma unroll
  for (int i = 0; i < 7; ++i)
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
        : "=d"(v[i])
        : "l"(base + i * 32 + lid), "l"(pol));
}
template <int SIGMA, int G>
__device__ __forceinline__ void load_slot_cols(const int32_t* base, int lid, int (&c)[SIGMA],
                                               uint64_t pol) {
  if constexpr (G == 2) {
#pragma unroll
    for (int g = 0; g < SIGMA / 2; ++g)
      asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
          : "=r"(c[2 * g]), "=r"(c[2 * g + 1])
          : "l"(base + g * 64 + 2 * lid), "l"(pol));
  } else {
#pragma unroll
    for (int i = 0; i < SIGMA; ++i)
      asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
          : "=r"(c[i])
          : "l"(base + i * 32 + lid), "l"(pol));
  }
}

template <typename T>
struct SlotParams {
  const T* svals;
  const int32_t* scols;
  const T* x;
  T* y;
  const uint32_t* tile_x;
  const uint32_t* tile_y;
  const uint32_t* lane_desc;
  const int32_t* hub_cols;
  const T* hub_x;  // contiguous hub values (nullptr: gather x[hub_cols])
  uint32_t* carry_row;
  T* carry_val;
  Geometry g;
  PrArgs pr;
};

// gather x for the steps in `mask` (bit i: slot i is a live element)
#ifndef MBX_GATHER
#define MBX_GATHER 0
#endif
#ifndef MBX_GATHER_NOHUB
#define MBX_GATHER_NOHUB 1
#endif
template <typename T, int SIGMA, bool HUB>
__device__ __forceinline__ void gather_slots(const T* __restrict__ x, const T* hub,
                                             const int (&col)[SIGMA], uint32_t mask,
                                             T (&xv)[SIGMA]) {
#pragma unroll
  for (int i = 0; i < SIGMA; ++i) {
    const int c = col[i];
    if (!HUB && MBX_GATHER_NOHUB) {
      // no hub table (small, stencil-like or uniform matrices): every slot
      // gathers, branch-free -- a dead slot holds column 0 (an L1 hit) and
      // its product is masked by the walk
      xv[i] = __ldg(x + c);
    } else if (MBX_GATHER == 1) {
      // every slot, no branches: a dead slot (column 0) reads x[0] (an L1
      // hit) and its product is masked by the walk; a hub reference is a
      // generic load from shared memory
      const T* p = (HUB && c < 0) ? hub + (c & 0x7FFFFFFF) : x + c;
      xv[i] = *p;
    } else if (MBX_GATHER == 2) {
      xv[i] = (HUB && c < 0) ? hub[c & 0x7FFFFFFF] : __ldg(x + c);
    } else {
      xv[i] = T(0);
      if ((mask >> i) & 1u) {
        if (HUB && c < 0)
          xv[i] = hub[c & 0x7FFFFFFF];
        else
          xv[i] = __ldg(x + c);
      }
    }
  }
}

// Inclusive segmented scan of the lanes' trailing sums (Alg. 5,
// merbit_spmv.hpp:85-117) with the previous tile's carry entering at lane 0;
// returns the new carry (lane 31's run) and sets `headv` (the value of the
// lane's first closed row, valid iff had_down).
template <typename T>
__device__ __forceinline__ T seg_scan(T sum, T head, bool had_down, int lid, T carry, T& headv) {
  T tail = sum;
  if (lid == 0) {
    if (had_down)
      head += carry;
    else
      tail += carry;
  }
  T S_ = tail;
  bool F = had_down;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T su = __shfl_up_sync(kFull, S_, off);
    const bool fu = __shfl_up_sync(kFull, F, off);
    if (lid >= off && !F) {
      S_ += su;
      F = fu;
    }
  }
  const T prevS = __shfl_up_sync(kFull, S_, 1);
  headv = head + (lid > 0 ? prevS : T(0));
  return __shfl_sync(kFull, S_, 31);
}


// ---- TMA bulk staging of the next tile's column slots + descriptors ----
// (mode 2 of the slot kernel): one lane per warp arms the warp's mbarrier
// with the byte count and issues two cp.async.bulk copies global -> shared;
// the lanes wait on the barrier's phase, read their operands with LDS, and
// the buffer is re-armed for the following tile.  The column stream then
// pays its DRAM latency behind the previous tile's gathers and commit.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t phase) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(m)), "r"(phase)
        : "memory");
  } while (!done);
}
// lane 0 only: stage chunk c's column slots (TS int32) and its 32
// descriptors into the warp's buffers (the generic-proxy reads of the
// previous contents are ordered before the async-proxy writes)
__device__ __forceinline__ void stage_chunk(uint64_t* m, int32_t* colbuf, uint32_t* descbuf,
                                            const int32_t* scols, const uint32_t* lane_desc,
                                            int64_t c, int ts, uint64_t pol) {
  const uint32_t cbytes = uint32_t(ts) * 4u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)),
               "r"(cbytes + 128u)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(colbuf)),
      "l"(scols + c * ts), "r"(cbytes), "r"(smem_u32(m)), "l"(pol)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], 128, [%2], %3;" ::"r"(smem_u32(descbuf)),
      "l"(lane_desc + c * 32), "r"(smem_u32(m)), "l"(pol)
      : "memory");
}
template <int SIGMA, int G>
__device__ __forceinline__ void lds_slot_cols(const int32_t* colbuf, int lid, int (&c)[SIGMA]) {
  if constexpr (G == 2) {
#pragma unroll
    for (int g = 0; g < SIGMA / 2; ++g) {
      const int2 v = *reinterpret_cast<const int2*>(colbuf + g * 64 + 2 * lid);
      c[2 * g] = v.x;
      c[2 * g + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < SIGMA; ++i) c[i] = colbuf[i * 32 + lid];
  }
}

// per-warp staging area of mode 2 (after the row buffers and accumulators)
template <int SIGMA>
struct StageBytes {
  static constexpr size_t value = size_t(32 * SIGMA) * 4 + 128 + 16;
};

#ifndef MBX_META_PF
#define MBX_META_PF 1
#endif
// a range's tile entries (lane i <= nc holds entry c0 + i), loaded one range
// ahead so the walk of a range starts without a memory round trip
__device__ __forceinline__ void load_range_meta(const uint32_t* tile_x, const uint32_t* tile_y,
                                                const Geometry& g, int64_t range, int lid,
                                                uint64_t pol, uint32_t& mtx, uint32_t& mty) {
  mtx = mty = 0;
  if (range < 0) return;
  const int64_t c0 = range * g.chunks_per_range;
  const int nc = static_cast<int>(imin64(c0 + g.chunks_per_range, g.num_chunks) - c0);
  if (lid <= nc) {
    mtx = ld_stream_u32(tile_x + c0 + lid, pol);
    mty = ld_stream_u32(tile_y + c0 + lid, pol);
  }
}

template <typename T, int SIGMA, bool PR, bool HUB, int MODE>
__device__ __forceinline__ void slot_range(const SlotParams<T>& p, const T* hub, T* rowbuf,
                                           int64_t range, int lid, uint64_t pol, T base,
                                           unsigned char* stg, uint32_t& phase,
                                           int64_t next_range, uint32_t& pmx, uint32_t& pmy) {
  constexpr bool PF = MODE == 1;
  constexpr bool TMA = MODE == 2;
  int32_t* colbuf = reinterpret_cast<int32_t*>(stg);
  uint32_t* descbuf = reinterpret_cast<uint32_t*>(stg + size_t(32 * SIGMA) * 4);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stg + size_t(32 * SIGMA) * 4 + 128);
  constexpr int G = 8 / int(sizeof(T));
  constexpr int TS = 32 * SIGMA;
  const Geometry& g = p.g;
  const int64_t c0 = range * g.chunks_per_range;
  const int nc = static_cast<int>(imin64(c0 + g.chunks_per_range, g.num_chunks) - c0);
  const int64_t total = g.nnz + g.n_rows;
  const int ob = g.ob;
  const uint32_t omask = (1u << ob) - 1u;

  uint32_t mtx = 0, mty = 0;
  if (MBX_META_PF) {
    mtx = pmx;
    mty = pmy;
    load_range_meta(p.tile_x, p.tile_y, g, next_range, lid, pol, pmx, pmy);
  } else if (lid <= nc) {
    mtx = ld_stream_u32(p.tile_x + c0 + lid, pol);
    mty = ld_stream_u32(p.tile_y + c0 + lid, pol);
  }
  const uint32_t head_row = __shfl_sync(kFull, mty, 0) & ~kLongRowMask;
  const uint32_t tail_row = __shfl_sync(kFull, mty, nc) & ~kLongRowMask;
  T carry = T(0), head_val = T(0);
  bool head_open = true;

  for (int ci = 0; ci < nc; ++ci) {
    const int64_t c = c0 + ci;
    const uint32_t x0 = __shfl_sync(kFull, mtx, ci);
    const uint32_t x1 = __shfl_sync(kFull, mtx, ci + 1);
    const uint32_t ty0 = __shfl_sync(kFull, mty, ci);
    const uint32_t y0 = ty0 & ~kLongRowMask;
    const uint32_t y1 = __shfl_sync(kFull, mty, ci + 1) & ~kLongRowMask;
    const int cnt = static_cast<int>(x1 - x0);
    const int nrows = static_cast<int>(y1 - y0);
    const T* vb = p.svals + c * TS;
    const int32_t* cb = p.scols + c * TS;
    if (TMA) {
      mbar_wait(mbar, phase);  // chunk c's columns + descriptors have landed
      phase ^= 1u;
    }
    // the next chunk this warp walks: c + 1, or the first of its next range
    const int64_t cnext = ci + 1 < nc ? c + 1
                          : next_range >= 0 ? next_range * g.chunks_per_range : int64_t(-1);
    // TMA: every lane has its operands in registers -> re-arm the buffer
    auto restage = [&]() {
      if (TMA) {
        __syncwarp();
        if (lid == 0 && cnext >= 0)
          stage_chunk(mbar, colbuf, descbuf, p.scols, p.lane_desc, cnext, TS, pol);
      }
    };
    auto get_cols = [&](int (&col)[SIGMA]) {
      if (TMA)
        lds_slot_cols<SIGMA, G>(colbuf, lid, col);
      else
        load_slot_cols<SIGMA, G>(cb, lid, col, pol);
    };
    if (PF && lid == 0 && cnext >= 0) {
      // one bulk L2 prefetch per stream for the next tile this warp walks
      // (the next one of this range, or the first of its next range, with
      // that range's tile entries and descriptors): its slots then arrive at
      // L2 latency instead of DRAM latency
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.scols + cnext * TS),
                   "r"(unsigned(TS * 4)));
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.svals + cnext * TS),
                   "r"(unsigned(TS * sizeof(T))));
      if (ci + 1 == nc) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.lane_desc + cnext * 32));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.tile_x + cnext));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.tile_y + cnext));
      }
    }
    if (ty0 & kLongRowMask) {
      // marked tile: one row; lane-strided subtotals + halving tree
      // (fast_tile_reduce, merbit_spmv.hpp:58-77) -- the butterfly's lane 0
      // adds exactly the halving tree's operand pairs
      int col[SIGMA];
      get_cols(col);
      restage();
      uint32_t live = 0;
#pragma unroll
      for (int i = 0; i < SIGMA; ++i) live |= (32 * i + lid < cnt ? 1u : 0u) << i;
      T xv[SIGMA], v[SIGMA];
      gather_slots<T, SIGMA, HUB>(p.x, hub, col, live, xv);
      load_slot_vals<T, SIGMA>(vb, lid, v, pol);
      T s = T(0);
#pragma unroll
      for (int i = 0; i < SIGMA; ++i)
        if ((live >> i) & 1u) s += mul_rn(v[i], xv[i]);
      s = __shfl_sync(kFull, warp_sum(s), 0);
      carry += s;
      continue;
    }
    if (cnt == 0) {
      // no nonzero: the first closure ends the carried row, the rest are
      // empty rows (merbit_spmv.hpp:217-224)
      restage();
      if (PR) {
        if (nrows > 0) {
          if (head_open) head_val = carry;
          const T pb = pr_value(p.pr, base, T(0));  // an empty row: c * 0 + base
          for (int kk = lid; kk < nrows; kk += 32) {
            if (kk == 0 && head_open) continue;
            pr_store<T>(p.pr, int64_t(y0) + kk, kk == 0 ? pr_value(p.pr, base, carry) : pb, p.y);
          }
          head_open = false;
        }
        carry = T(0);
        continue;
      }
      for (int k = lid; k < nrows; k += 32) {
        const T w = k == 0 ? carry : T(0);
        if (k == 0 && head_open) {
          head_val = w;
          continue;
        }
        p.y[int64_t(y0) + k] = w;
      }
      carry = T(0);
      if (nrows > 0) head_open = false;
      continue;
    }
    const int64_t j = c * 32 + lid;
    const bool valid = j < g.lane_num;
    const uint32_t d = !valid ? 0u : TMA ? descbuf[lid] : ld_stream_u32(p.lane_desc + j, pol);
    const int steps = valid ? static_cast<int>(imin64(SIGMA, total - j * SIGMA)) : 0;
    const uint32_t live = steps >= 32 ? kFull : ((1u << steps) - 1u);
    const uint32_t dmask = (d >> (2 * ob)) & live;
    const uint32_t rmask = ~(d >> (2 * ob)) & live;
    const int r0 = static_cast<int>((d >> ob) & omask);
    const bool direct = nrows > kSlotRowBuf;  // warp-uniform
    int col[SIGMA];
    get_cols(col);
    restage();
    T xv[SIGMA], v[SIGMA];
    gather_slots<T, SIGMA, HUB>(p.x, hub, col, rmask, xv);
    load_slot_vals<T, SIGMA>(vb, lid, v, pol);
    // per-lane walk (Alg. 4, merbit_spmv.hpp:251-297) in registers, as
    // predicated selects (no divergent branches per step): a Down step
    // closes a row -- the lane's first closure is its head, later ones are
    // rows opened and closed inside the lane -- and a Right step adds its
    // product; rows beyond the commit buffer go straight to y (PageRank:
    // already rank-updated)
    T sum = T(0), head = T(0);
    bool had_down = false;
    auto walk = [&](T* sink, bool upd) {
      int r = r0;
#pragma unroll
      for (int i = 0; i < SIGMA; ++i) {
        const bool dn = (dmask >> i) & 1u;
        const bool rt = (rmask >> i) & 1u;
        const T prod = mul_rn(v[i], xv[i]);
        if (dn && had_down) sink[r] = upd ? pr_value(p.pr, base, sum) : sum;
        head = (dn && !had_down) ? sum : head;
        had_down = had_down || dn;
        sum = dn ? T(0) : (rt ? sum + prod : sum);
        r += dn ? 1 : 0;
      }
    };
    if (!direct)
      walk(rowbuf, false);
    else
      walk(p.y + y0, PR);
    T headv;
    carry = seg_scan<T>(sum, head, had_down, lid, carry, headv);
    if (!direct) {
      if (had_down) rowbuf[r0] = headv;
      __syncwarp();
      // coalesced commit of the tile's rows (Alg. 6 load_mem)
      for (int k = lid; k < nrows; k += 32) {
        const T w = rowbuf[k];
        if (k == 0 && head_open) {
          head_val = w;
          continue;
        }
        const int64_t row = int64_t(y0) + k;
        if (PR)
          pr_store<T>(p.pr, row, pr_value(p.pr, base, w), p.y);
        else
          p.y[row] = w;
      }
      __syncwarp();
    } else {
      // more rows than the row buffer: the sums went straight to y
      const bool opens = had_down && r0 == 0;  // this lane closes the tile's row 0
      const unsigned who = __ballot_sync(kFull, opens);
      const T hv = __shfl_sync(kFull, headv, who ? __ffs(who) - 1 : 0);
      if (had_down && !(opens && head_open))
        p.y[int64_t(y0) + r0] = PR ? pr_value(p.pr, base, headv) : headv;
      if (PR && p.pr.xout) {
        // row shards: the exchange copies of the tile's rows, coalesced
        __syncwarp();
        for (int k = lid; k < nrows; k += 32)
          if (!(k == 0 && head_open)) pr_store<T>(p.pr, int64_t(y0) + k, p.y[int64_t(y0) + k], p.y);
      }
      if (head_open && who) head_val = hv;
    }
    if (nrows > 0) head_open = false;
  }
  if (lid == 0) {
    p.carry_row[2 * range] = head_row;
    p.carry_val[2 * range] = head_open ? T(0) : head_val;
    p.carry_row[2 * range + 1] = tail_row;
    p.carry_val[2 * range + 1] = carry;
    if (PR) mark_carry_rows(p.pr, head_row, tail_row, g.n_rows);
  }
}

template <typename T, int SIGMA, bool PR, bool HUB, int MODE>
__global__ void __launch_bounds__(1024) spmv_slot_kernel(SlotParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geometry& g = p.g;
  pdl_wait();     // the previous kernel's x / scalars are complete
  pdl_trigger();  // K3 may be scheduled (its CTAs wait for this grid)
  if (PR && pr_skip(p.pr)) return;
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  T* hub = reinterpret_cast<T*>(smem_raw);
  const int hub_pad = HUB ? ((g.hub_count + 3) & ~3) : 0;
  // per warp: the row buffer (kSlotRowBuf T); mode 2: then the staging areas
  constexpr size_t kWarpBytes = kSlotRowBuf * sizeof(T);
  unsigned char* wbase = reinterpret_cast<unsigned char*>(hub + hub_pad);
  T* rowbuf = reinterpret_cast<T*>(wbase + size_t(warp) * kWarpBytes);
  if (HUB) stage_hubs<T>(hub, p.x, p.hub_cols, g.hub_count, p.hub_x);
  const uint64_t pol = evict_first_policy();
  T base = T(0);
  if (PR) base = pr_base<T>(p.pr);
  const int64_t wstride = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t first = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  // mode 2: the warp's staging area (columns, descriptors, mbarrier)
  unsigned char* stg = wbase + size_t(blockDim.x >> 5) * kWarpBytes +
                       size_t(warp) * StageBytes<SIGMA>::value;
  uint32_t phase = 0;
  if (MODE == 2 && lid == 0) {
    uint64_t* mbar = reinterpret_cast<uint64_t*>(stg + size_t(32 * SIGMA) * 4 + 128);
    mbar_init(mbar);
    if (first < g.num_ranges)
      stage_chunk(mbar, reinterpret_cast<int32_t*>(stg),
                  reinterpret_cast<uint32_t*>(stg + size_t(32 * SIGMA) * 4), p.scols, p.lane_desc,
                  first * g.chunks_per_range, 32 * SIGMA, pol);
  }
  uint32_t pmx = 0, pmy = 0;
  if (MBX_META_PF)
    load_range_meta(p.tile_x, p.tile_y, g, first < g.num_ranges ? first : -1, lid, pol, pmx, pmy);
  for (int64_t range = first; range < g.num_ranges; range += wstride)
    slot_range<T, SIGMA, PR, HUB, MODE>(p, hub, rowbuf, range, lid, pol, base, stg, phase,
                                        range + wstride < g.num_ranges ? range + wstride : -1,
                                        pmx, pmy);
  if (PR && p.pr.npeer) __threadfence_system();  // NVLink stores performed (fused exchange)
}

// hub encoding of a column: prefix > 0 -- the hubs are columns 0..prefix-1
// (degree-relabelled), slot c; else the hub word map (nullptr: no hubs)
__device__ __forceinline__ int32_t hub_encode(const uint2* __restrict__ map, int prefix,
                                              int32_t c, const uint32_t* bloom = nullptr) {
  if (prefix > 0) return c < prefix ? int32_t(0x80000000u | uint32_t(c)) : c;
  if (!map) return c;
  if (bloom) {  // shared-memory Bloom filter: most non-hubs never touch the map
    const uint32_t b = hub_bloom_bit(c);
    if (!((bloom[b >> 5] >> (b & 31)) & 1u)) return c;
  }
  return hub_word_encode(map, c);
}

// slot copy CTAs resident per SM: 4 caps the fp32 kernel at 64 registers
// (no spills) -- 32 warps instead of 24 keep more of the copy in flight
// (s24 natural 1.41 -> 1.16 ms, relabelled 0.84 -> 0.77 ms, C5 5.9 -> 5.2 ms)
#ifndef MBX_SLOT_MINB
#define MBX_SLOT_MINB 4
#endif
// One warp per chunk: the chunk's CSR run (at most 32*SIGMA nonzeros) is
// read coalesced into shared memory and hub-encoded there, then every lane
// picks its SIGMA slots out of it (a long-row chunk element-interleaved, a
// normal one along its lane descriptor) and the warp writes them with 8-byte
// stores, 256 contiguous bytes per instruction.
template <typename T, int SIGMA>
__global__ void __launch_bounds__(256, MBX_SLOT_MINB) build_slots_kernel(
    const T* __restrict__ vals, const int32_t* __restrict__ cols, const uint2* __restrict__ map,
    int prefix, const uint32_t* __restrict__ tile_x, const uint32_t* __restrict__ tile_y,
    const uint32_t* __restrict__ lane_desc, int64_t lane_num, int64_t num_chunks, int64_t total,
    int ob, T* __restrict__ svals, int32_t* __restrict__ scols,
    const uint32_t* __restrict__ gbloom) {
  constexpr int G = 8 / int(sizeof(T));
  constexpr int E = 32 * SIGMA;
  static_assert(SIGMA % G == 0, "slot groups");
  __shared__ T sv[8][E];
  __shared__ int32_t sc[8][E];
  extern __shared__ uint32_t sbloom[];  // natural-order hubs: the Bloom filter
  const uint32_t* bl = nullptr;
  if (gbloom) {
    for (int i = threadIdx.x; i < kHubBloomWords; i += blockDim.x) sbloom[i] = gbloom[i];
    __syncthreads();
    bl = sbloom;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t omask = (1u << ob) - 1u;
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t c = int64_t(blockIdx.x) * (blockDim.x >> 5) + w; c < num_chunks; c += nw) {
    const int64_t x0 = tile_x[c];
    const int n = int(imin64(int64_t(tile_x[c + 1]) - x0, E));
    {  // every load of the run in flight at once
      T lv[SIGMA];
      int32_t lc[SIGMA];
#pragma unroll
      for (int i = 0; i < SIGMA; ++i) {
        const int k = i * 32 + l;
        lv[i] = k < n ? __ldcs(vals + x0 + k) : T(0);
        lc[i] = k < n ? __ldcs(cols + x0 + k) : 0;
      }
#pragma unroll
      for (int i = 0; i < SIGMA; ++i) {
        const int k = i * 32 + l;
        if (k < n) {
          sv[w][k] = lv[i];
          sc[w][k] = hub_encode(map, prefix, lc[i], bl);
        }
      }
    }
    __syncwarp();
    T v[SIGMA];
    int32_t q[SIGMA];
    if (tile_y[c] & kLongRowMask) {
#pragma unroll
      for (int i = 0; i < SIGMA; ++i) {
        const int k = i * 32 + l;
        v[i] = k < n ? sv[w][k] : T(0);
        q[i] = k < n ? sc[w][k] : 0;
      }
    } else {
      const int64_t j = c * 32 + l;
      uint32_t d = 0;
      int steps = 0;
      if (j < lane_num) {
        d = lane_desc[j];
        steps = static_cast<int>(imin64(SIGMA, total - j * SIGMA));
      }
      int k = int(d & omask);
      const uint32_t fl = d >> (2 * ob);
#pragma unroll
      for (int i = 0; i < SIGMA; ++i) {
        v[i] = T(0);
        q[i] = 0;
        if (i < steps && !((fl >> i) & 1u)) {
          if (k < n) {
            v[i] = sv[w][k];
            q[i] = sc[w][k];
          } else {  // not reached for a well-formed TILE; stay exact anyway
            v[i] = vals[x0 + k];
            q[i] = hub_encode(map, prefix, cols[x0 + k]);
          }
          ++k;
        }
      }
    }
    __syncwarp();
    const int64_t sb = c * E + int64_t(l) * G;
    if constexpr (G == 2) {
#pragma unroll
      for (int g = 0; g < SIGMA / 2; ++g) {
        *reinterpret_cast<float2*>(svals + sb + g * 64) = make_float2(v[2 * g], v[2 * g + 1]);
        *reinterpret_cast<int2*>(scols + sb + g * 64) = make_int2(q[2 * g], q[2 * g + 1]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < SIGMA; ++i) {
        svals[sb + i * 32] = v[i];
        scols[sb + i * 32] = q[i];
      }
    }
  }
}

// Inverse of build_slots_kernel: the CSR values / columns back from the
// slot copy (hub references decoded through hub_cols).  A compacted matrix
// (mbx_matrix_compact) keeps only the slot copy and rebuilds its CSR with
// this on first use.
template <typename T>
__global__ void unslot_kernel(const T* __restrict__ svals, const int32_t* __restrict__ scols,
                              const int32_t* __restrict__ hub_cols,
                              const uint32_t* __restrict__ tile_x,
                              const uint32_t* __restrict__ tile_y,
                              const uint32_t* __restrict__ lane_desc, int64_t lane_num,
                              int64_t num_chunks, int64_t total, int sigma, int ob,
                              T* __restrict__ vals, int32_t* __restrict__ cols) {
  constexpr int G = 8 / int(sizeof(T));
  const uint32_t omask = (1u << ob) - 1u;
  auto decode = [&](int32_t c) { return c < 0 ? __ldg(hub_cols + (c & 0x7FFFFFFF)) : c; };
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < num_chunks * 32;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = j >> 5;
    const int l = static_cast<int>(j & 31);
    const int64_t x0 = tile_x[c], x1 = tile_x[c + 1];
    const int64_t sb = c * 32 * sigma + int64_t(l) * G;
    if (tile_y[c] & kLongRowMask) {
      for (int i = 0; i < sigma; ++i) {
        const int64_t e = x0 + int64_t(i) * 32 + l;
        const int64_t pos = sb + int64_t(i / G) * 32 * G + (i % G);
        if (e < x1) {
          vals[e] = svals[pos];
          cols[e] = decode(scols[pos]);
        }
      }
    } else {
      uint32_t d = 0;
      int steps = 0;
      if (j < lane_num) {
        d = lane_desc[j];
        steps = static_cast<int>(imin64(sigma, total - j * sigma));
      }
      int64_t x = x0 + (d & omask);
      const uint32_t fl = d >> (2 * ob);
      for (int i = 0; i < steps; ++i) {
        if (!((fl >> i) & 1u)) {
          const int64_t pos = sb + int64_t(i / G) * 32 * G + (i % G);
          vals[x] = svals[pos];
          cols[x] = decode(scols[pos]);
          ++x;
        }
      }
    }
  }
}

template <typename T, int SIGMA, bool PR, bool HUB>
void launch_slot(mbx_context* ctx, const SlotParams<T>& p, size_t smem) {
  auto kern = p.g.prefetch == 2   ? spmv_slot_kernel<T, SIGMA, PR, HUB, 2>
              : p.g.prefetch == 1 ? spmv_slot_kernel<T, SIGMA, PR, HUB, 1>
                                  : spmv_slot_kernel<T, SIGMA, PR, HUB, 0>;
  static std::atomic<uint64_t> done[3];  // per (T, SIGMA, PR, HUB), staging mode
  allow_max_smem(kern, ctx->device, done[p.g.prefetch == 2 ? 2 : p.g.prefetch ? 1 : 0]);
  const int64_t need = (p.g.num_ranges + p.g.warps_per_cta - 1) / p.g.warps_per_cta;
  const unsigned grid = static_cast<unsigned>(imin64(p.g.grid, need));
  launch_pdl(!PR, kern, grid, unsigned(p.g.warps_per_cta * 32), smem, ctx->stream, p);
}

// ---------------------------------------------------------------------------
// K3: boundary rows.  Carries are ordered by range, rows nondecreasing; each
// run of equal rows is summed left to right (ascending block order, exactly
// the reference's fold order) and ASSIGNED; the terminal row n is dropped.
// ---------------------------------------------------------------------------
constexpr int kFixupRun = 32;  // carries one thread folds before the warp takes over
// PageRank K3: a persistent grid of blocks of 256 (measured: 3 per SM beats
// 4 and 6, whose lower register budgets cost more than the extra warps gain)
constexpr int kK3BlocksPerSM = 3;

// One carry entry e (the thread's): the first entry of each run of equal
// rows folds the run left to right (merbit_spmv.hpp:330-337) -- runs longer
// than kFixupRun (rows spanning many ranges) are folded by the whole warp in
// a fixed lane-strided order + butterfly.  Called by all 32 lanes.
template <typename T, bool PR>
__device__ __forceinline__ void fold_carry(const uint32_t* __restrict__ crow,
                                           const T* __restrict__ cval, int64_t ne, int64_t e,
                                           int64_t n_rows, T* __restrict__ y, const PrArgs& pr,
                                           T base, PrAcc& acc) {
  const int lid = threadIdx.x & 31;
  uint32_t r = 0;
  bool start = false, lng = false;
  T sum = T(0);
  if (e < ne) {
    r = crow[e];
    start = e == 0 || crow[e - 1] != r;
    if (start) {
      int64_t k = e;
      const int64_t lim = imin64(ne, e + kFixupRun);
      for (; k < lim && crow[k] == r; ++k) sum += cval[k];
      lng = k == lim && k < ne && crow[k] == r;
    }
  }
  unsigned long_lanes = __ballot_sync(kFull, lng);
  while (long_lanes) {
    const int src = __ffs(long_lanes) - 1;
    long_lanes &= long_lanes - 1;
    const int64_t e0 = __shfl_sync(kFull, e, src);
    const uint32_t rr = __shfl_sync(kFull, r, src);
    // 128 carries per round trip: four independent loads per lane in
    // flight, folded in a fixed (lane, round) order -> deterministic
    T part = T(0);
    for (int64_t w = e0;; w += 128) {
      uint32_t rk[4];
      T vk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t k = w + 32 * j + lid;
        rk[j] = k < ne ? crow[k] : ~rr;
        vk[j] = k < ne ? cval[k] : T(0);
      }
      bool all_in = true;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool in = rk[j] == rr;
        if (in) part += vk[j];
        all_in = all_in && in;
      }
      if (__ballot_sync(kFull, all_in) != kFull) break;
    }
    part = __shfl_sync(kFull, warp_sum(part), 0);
    if (lid == src) sum = part;
  }
  if (start && int64_t(r) < n_rows) {
    if (PR)
      pr_commit<T>(pr, base, r, sum, y, acc);
    else
      y[r] = sum;
  }
}

// K3.  Plain SpMV: one thread per carry entry.  PageRank: a persistent grid
// (kK3BlocksPerSM per SM) strides over the carry entries, then streams the
// reductions of every other row, then the last block finalises the scalars.
template <typename T, bool PR>
__global__ void __launch_bounds__(256, PR ? kK3BlocksPerSM : 1)
    fixup_kernel(const uint32_t* __restrict__ crow, const T* __restrict__ cval,
                 int64_t num_ranges, int64_t n_rows, T* __restrict__ y, PrArgs pr) {
  pdl_wait();     // K2's carries, rows and marks are complete
  pdl_trigger();
  if (PR && pr_skip(pr)) return;
  const int64_t ne = 2 * num_ranges;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  PrAcc acc;
  T base = T(0);
  if (PR) base = pr_base<T>(pr);
  if (!PR) {
    fold_carry<T, PR>(crow, cval, ne, tid, n_rows, y, pr, base, acc);
    return;
  }
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  // warp-uniform trip count (the fold uses warp collectives)
  for (int64_t e0 = tid - (threadIdx.x & 31); e0 < ne; e0 += nt)
    fold_carry<T, PR>(crow, cval, ne, e0 + (threadIdx.x & 31), n_rows, y, pr, base, acc);
  if (PR) {
    // the reductions over every row K2 committed (all but the carry rows,
    // whose share the fold above took): pi_new (just written, L2-resident)
    // and pi_old streamed once -- K2 itself only stores pi_new.
    // each thread takes 16 (fp32) / 8 (fp64) consecutive rows per step: four
    // 16-byte loads of pi_new, four of pi_old, one carry-mask word
    constexpr int kV = 16 / int(sizeof(T));  // rows per 16-byte vector
    constexpr int kR = 4 * kV;               // rows per thread and step
    using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    const T* pold = reinterpret_cast<const T*>(pr.pi_old);
    const int64_t full = n_rows / kR;  // whole groups; the tail row by row
    for (int64_t gi = tid; gi < full; gi += nt) {
      const int64_t r0 = gi * kR;
      V a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = *reinterpret_cast<const V*>(y + r0 + u * kV);
        b[u] = __ldg(reinterpret_cast<const V*>(pold + r0 + u * kV));
      }
      const uint32_t mw = __ldg(pr.carry_mask + (r0 >> 5)) >> (r0 & 31);
      constexpr uint32_t gmask = kR >= 32 ? ~0u : ((1u << kR) - 1u);
      const bool dall = pr.dang_from >= 0 && r0 >= pr.dang_from;
      const bool dnone = pr.dang_from >= 0 && r0 + kR <= pr.dang_from;
      if (!pr.yardstick && (dall || dnone)) {
        // the common group: all or none dangling, constant yardstick --
        // partial sums in T over the group's rows that are not carry rows
        // (the fold took those), one fp64 add each; ERR from the group's
        // extremes (|pi - s| peaks at one of them, and rounding is
        // monotone: the same value as the per-row maximum)
        const uint32_t live = ~mw & gmask;
        T rs = T(0), ms = T(0), ds = T(0), hi = -INFINITY, lo = INFINITY;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const T* pa = reinterpret_cast<const T*>(&a[u]);
          const T* pb = reinterpret_cast<const T*>(&b[u]);
#pragma unroll
          for (int v = 0; v < kV; ++v) {
            const bool in = (live >> (u * kV + v)) & 1u;
            rs += in ? fabs(pa[v] - pb[v]) : T(0);
            ms += in ? fabs(pa[v]) : T(0);
            ds += in ? pa[v] : T(0);
            hi = in ? fmax(hi, pa[v]) : hi;
            lo = in ? fmin(lo, pa[v]) : lo;
          }
        }
        acc.resid += static_cast<double>(rs);
        acc.mass += static_cast<double>(ms);
        if (dall) acc.dang += static_cast<double>(ds);
        if (live)
          acc.err = fmax(acc.err, fmax(fabs(static_cast<double>(hi) - pr.yard_const),
                                       fabs(static_cast<double>(lo) - pr.yard_const)));
        continue;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const T* pa = reinterpret_cast<const T*>(&a[u]);
        const T* pb = reinterpret_cast<const T*>(&b[u]);
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          const int q = u * kV + v;
          const int64_t row = r0 + q;
          if (!((mw >> q) & 1u)) pr_accum<T>(pr, row, pa[v], pb[v], pr_dang(pr, row), acc);
        }
      }
    }
    for (int64_t row = full * kR + tid; row < n_rows; row += nt)
      if (!((__ldg(pr.carry_mask + (row >> 5)) >> (row & 31)) & 1u))
        pr_accum<T>(pr, row, y[row], __ldg(pold + row), pr_dang(pr, row), acc);
    pr_block_finish(acc, pr, pr.block_part, pr.done_counter, pr_next(pr), pr.check_stop != 0,
                    pr.check_stop != 0);  // row shards: the combine kernel advances
  }
}

// ---------------------------------------------------------------------------
// K1: generate_tile.  One thread per lane: merge_search on its diagonal
// (merge_path.cpp:8-36), the sigma-step walk (tile.cpp:59-69), the packed
// descriptor (descriptor.hpp:31-43); the tile's lane group votes the
// long-row mark (tile.cpp:75-77).  Arrays are byte-identical to the
// reference.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void d_merge_search(const uint32_t* __restrict__ ro, int64_t n,
                                               int64_t m, int64_t diag, int64_t& x,
                                               int64_t& y) {
  int64_t lo = diag - m > 0 ? diag - m : 0;
  int64_t hi = diag < n ? diag : n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (int64_t(__ldg(ro + mid + 1)) <= diag - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  x = diag - lo;
  y = lo < n ? lo : n;
}

__global__ void gen_tile_kernel(const uint32_t* __restrict__ ro, int64_t n, int64_t m,
                                int omega, int sigma, int ob, int64_t lane_num,
                                uint32_t* __restrict__ tile_x, uint32_t* __restrict__ tile_y,
                                uint32_t* __restrict__ lane_desc, int small_omega) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lid = threadIdx.x & 31;
  const bool valid = j < lane_num;
  const int64_t total = m + n;
  int64_t x = 0, y = 0;
  const int64_t diag = j * sigma;
  int64_t tsx, tsy;
  int leader = 0;
  if (valid) d_merge_search(ro, n, m, diag, x, y);
  if (small_omega) {
    leader = lid & ~(omega - 1);
    tsx = __shfl_sync(kFull, x, leader);
    tsy = __shfl_sync(kFull, y, leader);
  } else {
    tsx = tsy = 0;
    if (valid) d_merge_search(ro, n, m, (j / omega) * int64_t(omega) * sigma, tsx, tsy);
  }
  uint32_t flags = 0;
  if (valid) {
    const int64_t steps = imin64(sigma, total - diag);
    int64_t cx = x, cy = y;
    int64_t end = cy < n ? int64_t(__ldg(ro + cy + 1)) : 0;
    for (int64_t k = 0; k < steps; ++k) {
      if (cy < n && cx < end) {
        ++cx;
      } else {
        flags |= 1u << k;
        ++cy;
        end = cy < n ? int64_t(__ldg(ro + cy + 1)) : 0;
      }
    }
    lane_desc[j] = (flags << (2 * ob)) | (uint32_t(y - tsy) << ob) | uint32_t(x - tsx);
  }
  if (small_omega) {
    const unsigned ballot = __ballot_sync(kFull, valid && flags != 0u);
    const unsigned gmask = omega >= 32 ? kFull : ((1u << omega) - 1u);
    const bool any_down = ((ballot >> leader) & gmask) != 0u;
    if (valid && lid == leader) {
      tile_x[j / omega] = uint32_t(tsx);
      tile_y[j / omega] = uint32_t(tsy) | (any_down ? 0u : kLongRowMask);
    }
  }
}

// K1 for omega dividing 32 (the default 32): one CTA per kK1Lanes lanes, no
// per-lane search.  The merge path moves down exactly at diagonal
// e_r = ro[r+1] + r (the step after row r's last nonzero), so a lane's step
// flags are the row ends that fall in its sigma diagonals, and its start
// row is the CTA's start row plus the row ends before it.  The CTA's start
// rows come from one global merge-path search per CTA boundary
// (gen_tile_bounds_kernel, all in parallel); the CTA then reads its rows'
// offsets once, coalesced, scatters each row end into its lane's flag word
// (shared-memory atomicOr), and a block scan of the flag popcounts gives
// every lane's (x, y).  The per-lane binary search of gen_tile_kernel cost
// ~log2(n) dependent loads per lane.  Output byte-identical.
#ifndef MBX_K1_THREADS
#define MBX_K1_THREADS 128
#endif
#ifndef MBX_K1_PER
#define MBX_K1_PER 4
#endif
constexpr int kK1Threads = MBX_K1_THREADS;
constexpr int kK1Per = MBX_K1_PER;             // lanes per thread (a multiple of 4)
// (CTA shape measured, scripts/prof/k1_ab.sh: 128 x 4 lanes 1-2 % ahead of 256 x 4,
// 512 x 4 +6 %, 128 x 8 +13-30 %)
constexpr int kK1Lanes = kK1Threads * kK1Per;  // lanes per CTA

__global__ void gen_tile_bounds_kernel(const uint32_t* __restrict__ ro, int64_t n, int64_t m,
                                       int sigma, int64_t blocks, int64_t* __restrict__ bnd) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b > blocks) return;
  int64_t x, y;
  d_merge_search(ro, n, m, imin64(b * kK1Lanes * sigma, m + n), x, y);
  bnd[b] = y;
}

__global__ void __launch_bounds__(kK1Threads) gen_tile_scan_kernel(
    const uint32_t* __restrict__ ro, int64_t n, int64_t m, int omega, int sigma, int ob,
    int64_t lane_num, const int64_t* __restrict__ bnd, uint32_t* __restrict__ tile_x,
    uint32_t* __restrict__ tile_y, uint32_t* __restrict__ lane_desc) {
  __shared__ __align__(16) uint32_t fl[kK1Lanes];
  __shared__ __align__(16) int pre[kK1Lanes + 4];  // row ends before each lane (CTA-relative)
  __shared__ int wsum[kK1Threads / 32];
  const int tid = threadIdx.x, lid = tid & 31, wid = tid >> 5;
  const int64_t j0 = int64_t(blockIdx.x) * kK1Lanes;
  const int64_t d0 = j0 * sigma;
  const int64_t total = m + n;
  const int64_t span = imin64(int64_t(kK1Lanes) * sigma, total - d0);  // this CTA's diagonals
  const int64_t y0 = bnd[blockIdx.x];
  const int64_t r1 = imin64(bnd[blockIdx.x + 1], n - 1);  // last row that can end inside
#pragma unroll
  for (int v = 0; v < kK1Per / 4; ++v)
    reinterpret_cast<uint4*>(fl)[tid * (kK1Per / 4) + v] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const float inv_sigma = 1.0f / float(sigma);
#pragma unroll 8
  for (int64_t r = y0 + tid; r <= r1; r += kK1Threads) {
    const int64_t p = int64_t(__ldg(ro + r + 1)) + r - d0;  // e_r - d0 >= 0
    if (p < span) {
      const int q = int(p);  // < kK1Lanes * sigma <= 2^16: q / sigma from the
      int l = __float2int_rz(float(q) * inv_sigma);  // float reciprocal, corrected
      l += (l + 1) * sigma <= q ? 1 : 0;
      l -= l * sigma > q ? 1 : 0;
      atomicOr(&fl[l], 1u << (q - l * sigma));
    }
  }
  __syncthreads();
  uint32_t f[kK1Per];
  int cl[kK1Per];
  int c = 0;
#pragma unroll
  for (int v = 0; v < kK1Per / 4; ++v) {
    const uint4 f4 = reinterpret_cast<const uint4*>(fl)[tid * (kK1Per / 4) + v];
    f[4 * v] = f4.x;
    f[4 * v + 1] = f4.y;
    f[4 * v + 2] = f4.z;
    f[4 * v + 3] = f4.w;
  }
#pragma unroll
  for (int k = 0; k < kK1Per; ++k) {
    cl[k] = __popc(f[k]);
    c += cl[k];
  }
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(kFull, inc, o);
    if (lid >= o) inc += v;
  }
  if (lid == 31) wsum[wid] = inc;
  __syncthreads();
  int base = inc - c;
  for (int w = 0; w < wid; ++w) base += wsum[w];
  // this thread's lanes' prefixes stay in registers; the block sees them
  // through 16-byte stores (conflict-free, unlike kK1Per-strided words)
  int pv[kK1Per];
#pragma unroll
  for (int k = 0; k < kK1Per; ++k) {
    pv[k] = base;
    base += cl[k];
  }
#pragma unroll
  for (int v = 0; v < kK1Per / 4; ++v)
    reinterpret_cast<int4*>(pre)[tid * (kK1Per / 4) + v] =
        make_int4(pv[4 * v], pv[4 * v + 1], pv[4 * v + 2], pv[4 * v + 3]);
  if (tid == kK1Threads - 1) pre[kK1Lanes] = base;
  __syncthreads();
  uint32_t d[kK1Per];
#pragma unroll
  for (int k = 0; k < kK1Per; ++k) {
    const int l = kK1Per * tid + k;
    const int ld = l & ~(omega - 1);  // the tile's first lane
    const int pl = pv[k], pld = pre[ld];
    // offsets from the tile's start point, in 32 bits: rows and nonzeros
    // consumed by the lanes before this one in its tile
    const int dy = pl - pld;
    const int dx = (l - ld) * sigma - dy;
    d[k] = (f[k] << (2 * ob)) | (uint32_t(dy) << ob) | uint32_t(dx);
    const int64_t j = j0 + l;
    if (l == ld && j < lane_num) {
      const int64_t tsy = y0 + pld;
      const int64_t tsx = j * sigma - tsy;
      const bool any_down = pre[imin64(ld + omega, kK1Lanes)] > pld;
      tile_x[j / omega] = uint32_t(tsx);
      tile_y[j / omega] = uint32_t(tsy) | (any_down ? 0u : kLongRowMask);
    }
  }
  const int64_t j = j0 + kK1Per * tid;
  if (j + kK1Per - 1 < lane_num) {
#pragma unroll
    for (int v = 0; v < kK1Per / 4; ++v)
      reinterpret_cast<uint4*>(lane_desc + j)[v] =
          make_uint4(d[4 * v], d[4 * v + 1], d[4 * v + 2], d[4 * v + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < kK1Per; ++k)
      if (j + k < lane_num) lane_desc[j + k] = d[k];
  }
}

// omega not dividing 32: tile entries from the tile's first lane and an OR
// over the tile's descriptor flags.
__global__ void gen_tile_entries_kernel(const uint32_t* __restrict__ ro, int64_t n, int64_t m,
                                        int omega, int sigma, int ob, int64_t lane_num,
                                        int64_t tile_num, uint32_t* __restrict__ tile_x,
                                        uint32_t* __restrict__ tile_y,
                                        const uint32_t* __restrict__ lane_desc) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= tile_num) return;
  int64_t x, y;
  d_merge_search(ro, n, m, t * int64_t(omega) * sigma, x, y);
  bool any_down = false;
  for (int64_t j = t * omega; j < imin64((t + 1) * omega, lane_num); ++j)
    any_down |= (lane_desc[j] >> (2 * ob)) != 0u;
  tile_x[t] = uint32_t(x);
  tile_y[t] = uint32_t(y) | (any_down ? 0u : kLongRowMask);
}

__global__ void tile_terminal_kernel(uint32_t* tile_x, uint32_t* tile_y, int64_t tile_num,
                                     int64_t m, int64_t n) {
  tile_x[tile_num] = uint32_t(m);
  tile_y[tile_num] = uint32_t(n);  // never marked (tile.cpp:80-83)
}

// Routing counters with the kernel's predicate (merbit_spmv.hpp:217-237).
__global__ void trace_kernel(const uint32_t* __restrict__ tile_x,
                             const uint32_t* __restrict__ tile_y, int64_t tile_num,
                             unsigned long long* counters) {
  __shared__ unsigned long long s[3];
  if (threadIdx.x < 3) s[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < tile_num) {
    const uint32_t xs = tile_x[i + 1] - tile_x[i];
    const int k = xs == 0 ? 2 : ((tile_y[i] & kLongRowMask) ? 0 : 1);
    atomicAdd(&s[k], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < 3 && s[threadIdx.x]) atomicAdd(&counters[threadIdx.x], s[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// Plain CSR (warp per row, fp64 accumulation): the pagerank yardstick and a
// non-MERBIT comparator.
// ---------------------------------------------------------------------------
template <typename T, bool PR>
__global__ void __launch_bounds__(256) csr_kernel(const uint32_t* __restrict__ ro,
                                                  const int32_t* __restrict__ cols,
                                                  const T* __restrict__ vals,
                                                  const T* __restrict__ x, T* __restrict__ y,
                                                  int64_t n_rows, PrArgs pr) {
  const int lid = threadIdx.x & 31;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  PrAcc acc;
  T base = T(0);
  if (PR) base = pr_base<T>(pr);
  for (int64_t r = wid; r < n_rows; r += nwarps) {
    double s = 0.0;
    for (uint32_t k = ro[r] + lid; k < ro[r + 1]; k += 32)
      s += double(vals[k]) * double(__ldg(x + cols[k]));
    s = warp_sum(s);
    if (lid == 0) {
      if (PR)
        pr_commit<T>(pr, base, r, T(s), y, acc);
      else
        y[r] = T(s);
    }
  }
  if (PR) pr_block_finish(acc, pr, pr.block_part, pr.done_counter, pr.next, false);
}

template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

// The PageRank yardstick (solvers.hpp:178-191): the reference runs it over
// its CSR backend, whose spmv_csr_reference sums each row left to right in T
// (reference.hpp:28-37).  One thread per row reproduces that order and
// rounding exactly (products rounded, then added; no FMA contraction), so
// pi* -- and with it ERR and the stop iteration -- equal the reference's.
template <typename T>
__global__ void __launch_bounds__(256) csr_rowserial_pr_kernel(
    const uint32_t* __restrict__ ro, const int32_t* __restrict__ cols,
    const T* __restrict__ vals, const T* __restrict__ x, T* __restrict__ y, int64_t n_rows,
    PrArgs pr) {
  PrAcc acc;
  const T base = pr_base<T>(pr);
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    T s = T(0);
    const uint32_t k1 = __ldg(ro + r + 1);
    uint32_t k = __ldg(ro + r);
    for (; k + 4 <= k1; k += 4) {  // loads run ahead of the dependent adds
      T p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) p[u] = mul_rn(__ldg(vals + k + u), __ldg(x + __ldg(cols + k + u)));
#pragma unroll
      for (int u = 0; u < 4; ++u) s = add_rn(s, p[u]);
    }
    for (; k < k1; ++k) s = add_rn(s, mul_rn(__ldg(vals + k), __ldg(x + __ldg(cols + k))));
    pr_commit<T>(pr, base, r, s, y, acc);
  }
  pr_block_finish(acc, pr, pr.block_part, pr.done_counter, pr.next, false);
}

// SpmvTrace deposit log (merbit_spmv.hpp:21-28, 339-349): every partial row
// sum the MERBIT decomposition forms, one thread per lane -- a normal lane
// deposits at each Down step the partial of the row it closes and, after its
// last step, the partial of the row it leaves open (the segmented sum and the
// carries only regroup these); a lane of a marked (long-row) tile deposits
// its lane-strided subtotal (fast_tile_reduce).  Every staged product lands
// in exactly one deposit, so per-row totals reproduce y up to regrouping.
template <typename T>
__global__ void deposit_kernel(const T* __restrict__ vals, const int32_t* __restrict__ cols,
                               const T* __restrict__ x, const uint32_t* __restrict__ tile_x,
                               const uint32_t* __restrict__ tile_y,
                               const uint32_t* __restrict__ lane_desc, int64_t lane_num,
                               int64_t total, int omega, int sigma, int ob,
                               unsigned long long* counter, int64_t capacity,
                               int64_t* __restrict__ rows, T* __restrict__ amounts) {
  const uint32_t omask = (1u << ob) - 1u;
  auto deposit = [&](int64_t row, T v) {
    const unsigned long long k = atomicAdd(counter, 1ull);
    if (int64_t(k) < capacity) {
      rows[k] = row;
      amounts[k] = v;
    }
  };
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < lane_num;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t tile = j / omega;
    const int l = int(j % omega);
    const uint32_t ty = tile_y[tile];
    const int64_t x0 = tile_x[tile], y0 = ty & ~kLongRowMask;
    if (ty & kLongRowMask) {
      const int64_t x1 = tile_x[tile + 1];
      if (x0 + l >= x1) continue;
      T s = T(0);
      for (int64_t e = x0 + l; e < x1; e += omega) s = add_rn(s, mul_rn(vals[e], x[cols[e]]));
      deposit(y0, s);
      continue;
    }
    const uint32_t d = lane_desc[j];
    const int steps = int(imin64(sigma, total - j * sigma));
    int64_t xx = x0 + (d & omask), yy = y0 + ((d >> ob) & omask);
    const uint32_t fl = d >> (2 * ob);
    T sum = T(0);
    for (int k = 0; k < steps; ++k) {
      if ((fl >> k) & 1u) {
        deposit(yy, sum);
        sum = T(0);
        ++yy;
      } else {
        sum = add_rn(sum, mul_rn(vals[xx], x[cols[xx]]));
        ++xx;
      }
    }
    if (steps > 0) deposit(yy, sum);
  }
}

}  // namespace

void launch_deposits(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t, const void* x,
                     unsigned long long* counter, int64_t capacity, int64_t* rows,
                     void* amounts) {
  ensure_csr(ctx, m);
  const int64_t lanes = t->info.lane_num;
  if (lanes == 0) return;
  const unsigned grid = unsigned(imin64((lanes + 255) / 256, int64_t(ctx->sm_count) * 16));
  const int64_t total = m->nnz + m->n_rows;
  if (m->precision == MBX_F32)
    deposit_kernel<float><<<grid, 256, 0, ctx->stream>>>(
        static_cast<const float*>(m->vals), m->cols, static_cast<const float*>(x), t->tile_x,
        t->tile_y, t->lane_desc, lanes, total, t->info.omega, t->info.sigma, t->offset_bits,
        counter, capacity, rows, static_cast<float*>(amounts));
  else
    deposit_kernel<double><<<grid, 256, 0, ctx->stream>>>(
        static_cast<const double*>(m->vals), m->cols, static_cast<const double*>(x), t->tile_x,
        t->tile_y, t->lane_desc, lanes, total, t->info.omega, t->info.sigma, t->offset_bits,
        counter, capacity, rows, static_cast<double*>(amounts));
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

namespace {

// pi_0 (copy or uniform) and its dangling mass.
template <typename T>
__global__ void pr_init_kernel(const T* __restrict__ pi0, T* __restrict__ pi, int64_t n,
                               PrArgs pr) {
  PrAcc acc;
  const T u = T(1) / static_cast<T>(n);  // T(1)/static_cast<T>(n) (solvers.hpp:193)
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T v = pi0 ? pi0[i] : u;
    pi[i] = v;
    if ((pr.dangling[i >> 5] >> (i & 31)) & 1u) acc.dang += double(v);
    acc.mass += fabs(double(v));
  }
  pr_block_finish(acc, pr, pr.block_part, pr.done_counter, pr.next, false);
}

__global__ void seen_columns_kernel(const int32_t* __restrict__ cols, int64_t nnz,
                                    uint32_t* seen) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = uint32_t(cols[k]);
    const uint32_t bit = 1u << (c & 31);
    if (!(__ldg(seen + (c >> 5)) & bit)) atomicOr(seen + (c >> 5), bit);
  }
}

__global__ void invert_mask_kernel(uint32_t* mask, int64_t n) {
  const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t words = (n + 31) / 32;
  if (w >= words) return;
  uint32_t v = ~mask[w];
  const int64_t lim = n - w * 32;
  if (lim < 32) v &= (1u << lim) - 1u;
  mask[w] = v;
}

__global__ void narrow_cols_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                                   int64_t n, int64_t limit, int* bad) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = src[i];
    if (v < 0 || v >= limit) *bad = 1;
    dst[i] = int32_t(v);
  }
}

__global__ void narrow_rows_kernel(const int64_t* __restrict__ src, uint32_t* __restrict__ dst,
                                   int64_t n, int* bad) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = src[i];
    if (v < 0 || v > int64_t(0xFFFFFFFF) || (i > 0 && src[i - 1] > v)) *bad = 1;
    dst[i] = uint32_t(v);
  }
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148LL * 64) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<unsigned>(b);
}

template <typename T, int SIGMA, bool PR, bool HUB>
void launch_w32(mbx_context* ctx, const SpmvParams<T>& p, size_t smem) {
  auto kern = p.g.prefetch == 1 ? spmv_w32_kernel<T, SIGMA, PR, HUB, true>
                                : spmv_w32_kernel<T, SIGMA, PR, HUB, false>;
  static std::atomic<uint64_t> done[2];  // per (T, SIGMA, PR, HUB), prefetch variant
  allow_max_smem(kern, ctx->device, done[p.g.prefetch == 1 ? 1 : 0]);
  const int64_t need = (p.g.num_ranges + p.g.warps_per_cta - 1) / p.g.warps_per_cta;
  const unsigned grid = static_cast<unsigned>(imin64(p.g.grid, need));
  kern<<<grid, p.g.warps_per_cta * 32, smem, ctx->stream>>>(p);
}

// The hub values of this multiply, contiguous: hub_x[i] = x[hub_cols[i]]
// (once per multiply; every CTA then stages them with coalesced copies)
template <typename T>
__global__ void hub_gather_kernel(const T* __restrict__ x, const int32_t* __restrict__ hub_cols,
                                  int hc, T* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < hc; i += gridDim.x * blockDim.x)
    out[i] = __ldg(x + __ldg(hub_cols + i));
}

template <typename T, bool PR>
void launch_spmv_t(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                   const Geometry& g, const void* x, void* y, void* ws, const PrArgs* pr) {
  if (g.num_ranges == 0) return;
  SpmvParams<T> p;
  p.vals = static_cast<const T*>(m->vals);
  p.cols = g.hub_count > 0 ? m->cols_hub : m->cols;
  p.hub_cols = m->hub_cols;
  p.x = static_cast<const T*>(x);
  p.y = static_cast<T*>(y);
  p.tile_x = t->tile_x;
  p.tile_y = t->tile_y;
  p.lane_desc = t->lane_desc;
  p.g = g;
  const int64_t ne = 2 * g.num_ranges;
  p.carry_row = static_cast<uint32_t*>(ws);
  const size_t row_bytes = ((ne * 4 + 255) / 256) * 256;
  p.carry_val = reinterpret_cast<T*>(static_cast<char*>(ws) + row_bytes);
  if (pr) p.pr = *pr;
  p.hub_x = nullptr;
  if (g.hub_count > 0) {
    if (m->hub_prefix) {
      p.hub_x = p.x;  // the hubs are x's first entries
    } else {
      T* hx = reinterpret_cast<T*>(static_cast<char*>(ws) + row_bytes +
                                   ((ne * sizeof(T) + 255) / 256) * 256);
      hub_gather_kernel<T><<<unsigned((g.hub_count + 255) / 256), 256, 0, ctx->stream>>>(
          p.x, m->hub_cols, g.hub_count, hx);
      ++ctx->launches;
      p.hub_x = hx;
    }
  }
  if (g.slots) {
    SlotParams<T> q;
    q.svals = static_cast<const T*>(m->slots.vals);
    q.scols = m->slots.cols;
    q.x = p.x;
    q.y = p.y;
    q.tile_x = p.tile_x;
    q.tile_y = p.tile_y;
    q.lane_desc = p.lane_desc;
    q.hub_cols = p.hub_cols;
    q.hub_x = p.hub_x;
    q.carry_row = p.carry_row;
    q.carry_val = p.carry_val;
    q.g = g;
    q.pr = p.pr;
    constexpr int kDefSigma = sizeof(T) == 4 ? 14 : 7;
    const size_t smem = spmv_smem_bytes(g, m->precision);
    if (g.hub_count > 0)
      launch_slot<T, kDefSigma, PR, true>(ctx, q, smem);
    else
      launch_slot<T, kDefSigma, PR, false>(ctx, q, smem);
  } else if (g.omega == 32) {
    const size_t smem = spmv_smem_bytes(g, m->precision);
    constexpr int kDefSigma = sizeof(T) == 4 ? 14 : 7;
    if (g.hub_count > 0) {
      if (g.sigma == kDefSigma)
        launch_w32<T, kDefSigma, PR, true>(ctx, p, smem);
      else
        launch_w32<T, 0, PR, true>(ctx, p, smem);
    } else {
      if (g.sigma == kDefSigma)
        launch_w32<T, kDefSigma, PR, false>(ctx, p, smem);
      else
        launch_w32<T, 0, PR, false>(ctx, p, smem);
    }
  } else {
    p.g.warps_per_cta = kThreads / 32;
    const size_t smem = size_t(p.g.warps_per_cta) * (32 * g.sigma + 1) * sizeof(T);
    const unsigned grid =
        static_cast<unsigned>((g.num_ranges + p.g.warps_per_cta - 1) / p.g.warps_per_cta);
    spmv_generic_kernel<T, PR><<<grid, kThreads, smem, ctx->stream>>>(p);
  }
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
  const unsigned fgrid = static_cast<unsigned>(fixup_blocks(g, PR));
  launch_pdl(!PR, fixup_kernel<T, PR>, fgrid, 256u, 0, ctx->stream, p.carry_row,
             static_cast<const T*>(p.carry_val), g.num_ranges, g.n_rows, p.y, p.pr);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

}  // namespace

// K2's next-tile staging when the tuning leaves it to the library.  Matrices
// whose gathers are local (few distinct x sectors per 32 nonzeros: a
// stencil) stream at HBM speed, and the L2 prefetch of the next tile keeps
// the stream fed (C5 fp32 2.50 -> 2.35 ms, fp64 4.23 -> 4.16 ms against
// modes 0 / 2); on gather-bound matrices its extra requests cost (R-MAT s24
// fp32 +10 %, C3 fp64 +7 %), and there fp64 takes the TMA staging (mode 2:
// s24 fp64 SpMV -9 %) and fp32 none.
int resolve_prefetch(int tuning, int precision, double gather_sectors) {
  if (tuning >= 0) return tuning;
  if (gather_sectors > 0.0 && gather_sectors < 16.0) return 1;
  return precision == MBX_F64 ? 2 : 0;
}

size_t stage_bytes(int sigma) { return size_t(32 * sigma) * 4 + 128 + 16; }

size_t spmv_smem_bytes(const Geometry& g, int precision) {
  const size_t vs = value_size(precision);
  const size_t hub = g.hub_count > 0 ? size_t((g.hub_count + 3) & ~3) : 0;
  if (g.slots)  // hub | per warp: row buffer | (mode 2) per warp: staged column
                // slots + descriptors + mbarrier
    return hub * vs + size_t(g.warps_per_cta) * (kSlotRowBuf * vs +
                                                 (g.prefetch == 2 ? stage_bytes(g.sigma) : 0));
  return (hub + size_t(g.warps_per_cta) * (32 * g.sigma + 1)) * vs;
}

int default_sigma(int precision) { return precision == MBX_F32 ? 14 : 7; }

// Shared memory K2 takes per SM by default: what it does not take stays L1
// (256 KB unified per SM).  Measured on degree-relabelled R-MAT PageRank
// fp32 (scripts/prof/pr_iter.py, SMEM=): up to x = 128 MB (s25) the hubs
// win -- 160 KB: s24 790 vs 830 us at 128 KB, s25 1693 vs 1745 us; at
// 256 MB (s26) 128 KB and 96 KB tie (3.82 ms, 160 KB 4.02 ms); at 512 MB
// (s27) 96 KB is best (9.05 vs 9.21 ms at 128 KB, 10.0 ms at 160 KB).
int default_smem_budget(int precision, int64_t n_cols) {
  const int64_t xbytes = n_cols * int64_t(value_size(precision));
  if (xbytes > (int64_t(384) << 20)) return 96 * 1024;
  if (xbytes > (int64_t(192) << 20)) return 128 * 1024;
  return precision == MBX_F32 ? 160 * 1024 : 128 * 1024;
}

int max_hub_slots(const mbx_context* ctx, int warps_per_cta, int ctas_per_sm, int sigma,
                  int precision, int64_t n_cols) {
  int per_sm = 0, optin = 0;
  MBX_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                  ctx->device));
  MBX_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int64_t reserve = 1024;  // per-CTA system reservation
  const int budget = ctx->tuning.smem_per_sm > 0 ? ctx->tuning.smem_per_sm
                                                  : default_smem_budget(precision, n_cols);
  if (budget < per_sm) per_sm = budget;
  int64_t per_cta = per_sm / ctas_per_sm - reserve;
  if (per_cta > optin) per_cta = optin;
  const int64_t vs = int64_t(value_size(precision));
  const bool slot_layout = ctx->tuning.layout == 1 && sigma == default_sigma(precision);
  const int64_t bufs =
      slot_layout ? int64_t(warps_per_cta) *
                        (kSlotRowBuf * vs +
                         (resolve_prefetch(ctx->tuning.prefetch, precision) == 2
                              ? int64_t(stage_bytes(sigma))
                              : 0))
                  : int64_t(warps_per_cta) * (32 * sigma + 1) * vs;
  const int64_t slots = (per_cta - bufs) / vs - 4;
  return slots > 0 ? int(slots & ~int64_t(3)) : 0;
}


int64_t fixup_blocks(const Geometry& g, bool pagerank) {
  // plain SpMV: one thread per carry entry; PageRank: one resident wave
  const int64_t carry = (2 * g.num_ranges + 255) / 256;
  const int64_t b = pagerank ? int64_t(g.sms) * kK3BlocksPerSM : carry;
  return b > 0 ? b : 1;
}

// Condition of the device-driven PageRank loop: replay the body while
// iterations remain and no stop was decided.
__global__ void pr_loop_cond_kernel(cudaGraphConditionalHandle h, const int64_t* iter_dev,
                                    int64_t max_iters, const int* stop) {
  cudaGraphSetConditional(h, (*iter_dev < max_iters && !*stop) ? 1u : 0u);
}

void launch_pr_loop_cond(mbx_context* ctx, cudaGraphConditionalHandle h, const int64_t* iter_dev,
                         int64_t max_iters, const int* stop) {
  pr_loop_cond_kernel<<<1, 1, 0, ctx->stream>>>(h, iter_dev, max_iters, stop);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

size_t spmv_workspace_bytes(const Geometry& g, int precision, bool pagerank) {
  // carry rows | carry values | the multiply's contiguous hub values
  const int64_t ne = 2 * g.num_ranges;
  const size_t vs = value_size(precision);
  size_t b = ((ne * 4 + 255) / 256) * 256 + ((ne * vs + 255) / 256) * 256;
  b += ((size_t(g.hub_count) * vs + 255) / 256) * 256;
  (void)pagerank;
  return b + 256;
}

void free_slots(mbx_context* ctx, const mbx_matrix* m) {
  if (m->slots.vals || m->slots.cols) ++m->gen;
  if (m->slots.vals) cudaFreeAsync(m->slots.vals, ctx->stream);
  if (m->slots.cols) cudaFreeAsync(m->slots.cols, ctx->stream);
  m->slots = mbx_matrix::SlotCache{};
}

bool ensure_slots(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t, const Geometry& g) {
  if (ctx->tuning.layout != 1 || g.omega != 32 || g.sigma != default_sigma(m->precision) ||
      g.num_chunks == 0)
    return false;
  const int hub = g.hub_count > 0 ? 1 : 0;
  mbx_matrix::SlotCache& sc = m->slots;
  if (sc.vals && sc.tile_serial == t->serial && sc.version == m->version && sc.hub == hub)
    return true;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  MBX_CUDA(cudaStreamIsCapturing(ctx->stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) return false;  // never build inside a capture
  ensure_csr(ctx, m);  // a compacted matrix rebuilds its CSR from the old slots first
  free_slots(ctx, m);
  const int64_t count = g.num_chunks * 32 * g.sigma;
  const size_t vs = value_size(m->precision);
  cudaEvent_t e0, e1;
  MBX_CUDA(cudaEventCreate(&e0));
  MBX_CUDA(cudaEventCreate(&e1));
  MBX_CUDA(cudaMallocAsync(&sc.vals, count * vs + 256, ctx->stream));
  MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc.cols), count * 4 + 256, ctx->stream));
  MBX_CUDA(cudaEventRecord(e0, ctx->stream));  // build time, not the allocation
  // the hub encoding is applied while the slots are written (no encoded
  // copy of the CSR columns is kept)
  const int prefix = hub && m->hub_prefix ? m->hub_avail : 0;
  uint2* map = hub && !prefix ? hub_word_map(ctx, m) : nullptr;
  const unsigned grid = grid_for((g.num_chunks + 7) / 8, 1, int64_t(ctx->sm_count) * 8);
  const int64_t total = g.nnz + g.n_rows;
  const uint32_t* bloom =
      map ? reinterpret_cast<const uint32_t*>(map + hub_map_words(m->n_cols)) : nullptr;
  const size_t dyn = map ? size_t(kHubBloomWords) * 4 : 0;
  if (m->precision == MBX_F32)
    build_slots_kernel<float, 14><<<grid, 256, dyn, ctx->stream>>>(
        static_cast<const float*>(m->vals), m->cols, map, prefix, t->tile_x, t->tile_y,
        t->lane_desc, g.lane_num, g.num_chunks, total, g.ob, static_cast<float*>(sc.vals), sc.cols,
        bloom);
  else
    build_slots_kernel<double, 7><<<grid, 256, dyn, ctx->stream>>>(
        static_cast<const double*>(m->vals), m->cols, map, prefix, t->tile_x, t->tile_y,
        t->lane_desc, g.lane_num, g.num_chunks, total, g.ob, static_cast<double*>(sc.vals), sc.cols,
        bloom);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
  MBX_CUDA(cudaEventRecord(e1, ctx->stream));
  if (map) cudaFreeAsync(map, ctx->stream);
  MBX_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  MBX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  sc.tile_serial = t->serial;
  sc.version = m->version;
  sc.hub = hub;
  sc.count = count;
  sc.seconds = ms * 1e-3;
  return true;
}

void compact_matrix(mbx_context* ctx, mbx_matrix* m, const mbx_tile* t) {
  mbx_matrix::SlotCache& sc = m->slots;
  if (!sc.vals || sc.tile_serial != t->serial)
    fail(MBX_CONFIG_ERROR, "compact: the matrix holds no slot copy for this TILE (run an SpMV "
                           "or create a PageRank plan with it first)");
  if (!m->vals) return;  // already compact
  cudaStream_t s = ctx->stream;
  // a private copy of the TILE the slot copy follows (the caller may destroy
  // its TILE handle); then the CSR values and columns go
  const int64_t tn = t->info.tile_num, ln = t->info.lane_num;
  auto* tc = new mbx_matrix::CompactTile;
  tc->info = t->info;
  tc->ob = t->offset_bits;
  MBX_CUDA(cudaMallocAsync(&tc->tile_x, (tn + 1) * 4 + 256, s));
  MBX_CUDA(cudaMallocAsync(&tc->tile_y, (tn + 1) * 4 + 256, s));
  MBX_CUDA(cudaMallocAsync(&tc->lane_desc, ln * 4 + 256, s));
  MBX_CUDA(cudaMemcpyAsync(tc->tile_x, t->tile_x, (tn + 1) * 4, cudaMemcpyDeviceToDevice, s));
  MBX_CUDA(cudaMemcpyAsync(tc->tile_y, t->tile_y, (tn + 1) * 4, cudaMemcpyDeviceToDevice, s));
  MBX_CUDA(cudaMemcpyAsync(tc->lane_desc, t->lane_desc, ln * 4, cudaMemcpyDeviceToDevice, s));
  if (m->cols_hub) {  // derived from the CSR columns: rebuilt on demand
    cudaFreeAsync(m->cols_hub, s);
    m->cols_hub = nullptr;
  }
  cudaFreeAsync(m->vals, s);
  cudaFreeAsync(m->cols, s);
  m->vals = nullptr;
  m->cols = nullptr;
  m->compact = tc;
  ++m->gen;  // graphs captured over a non-slot path would read the freed CSR
  MBX_CUDA(cudaStreamSynchronize(s));
}

void ensure_csr(mbx_context* ctx, const mbx_matrix* m_) {
  mbx_matrix* m = const_cast<mbx_matrix*>(m_);
  if (m->vals || !m->compact) return;
  mbx_matrix::CompactTile* tc = m->compact;
  cudaStream_t s = ctx->stream;
  const size_t vs = value_size(m->precision);
  void* vals = nullptr;
  int32_t* cols = nullptr;
  MBX_CUDA(cudaMallocAsync(&vals, m->nnz * vs + 256, s));
  MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cols), m->nnz * 4 + 256, s));
  const int64_t chunks = (tc->info.lane_num + 31) / 32;
  const int64_t total = m->nnz + m->n_rows;
  const unsigned grid = grid_for(chunks * 32, 256, int64_t(ctx->sm_count) * 16);
  if (chunks > 0) {
    if (m->precision == MBX_F32)
      unslot_kernel<float><<<grid, 256, 0, s>>>(
          static_cast<const float*>(m->slots.vals), m->slots.cols, m->hub_cols, tc->tile_x,
          tc->tile_y, tc->lane_desc, tc->info.lane_num, chunks, total, tc->info.sigma, tc->ob,
          static_cast<float*>(vals), cols);
    else
      unslot_kernel<double><<<grid, 256, 0, s>>>(
          static_cast<const double*>(m->slots.vals), m->slots.cols, m->hub_cols, tc->tile_x,
          tc->tile_y, tc->lane_desc, tc->info.lane_num, chunks, total, tc->info.sigma, tc->ob,
          static_cast<double*>(vals), cols);
    ++ctx->launches;
    MBX_CUDA(cudaGetLastError());
  }
  m->vals = vals;
  m->cols = cols;
  free_compact_tile(ctx, m);
  MBX_CUDA(cudaStreamSynchronize(s));
}

void free_compact_tile(mbx_context* ctx, const mbx_matrix* m_) {
  mbx_matrix* m = const_cast<mbx_matrix*>(m_);
  if (!m->compact) return;
  cudaFreeAsync(m->compact->tile_x, ctx->stream);
  cudaFreeAsync(m->compact->tile_y, ctx->stream);
  cudaFreeAsync(m->compact->lane_desc, ctx->stream);
  delete m->compact;
  m->compact = nullptr;
}

void launch_spmv(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t, const Geometry& g,
                 const void* x, void* y, void* ws, const PrArgs* pr) {
  if (m->precision == MBX_F32) {
    if (pr)
      launch_spmv_t<float, true>(ctx, m, t, g, x, y, ws, pr);
    else
      launch_spmv_t<float, false>(ctx, m, t, g, x, y, ws, nullptr);
  } else {
    if (pr)
      launch_spmv_t<double, true>(ctx, m, t, g, x, y, ws, pr);
    else
      launch_spmv_t<double, false>(ctx, m, t, g, x, y, ws, nullptr);
  }
}

void launch_generate_tile(mbx_context* ctx, const uint32_t* ro, int64_t n_rows, int64_t nnz,
                          const mbx_simt_config& c, mbx_tile* t) {
  const int64_t lanes = t->info.lane_num, tiles = t->info.tile_num;
  const bool small = c.omega <= 32 && (32 % c.omega) == 0;
  if (lanes > 0) {
    const int64_t blocks = (lanes + 255) / 256;
    if (small) {
      const int64_t cblocks = (lanes + kK1Lanes - 1) / kK1Lanes;
      int64_t* bnd = nullptr;
      MBX_CUDA(cudaMallocAsync(&bnd, size_t(cblocks + 1) * 8 + 64, ctx->stream));
      gen_tile_bounds_kernel<<<static_cast<unsigned>((cblocks + 256) / 256), 256, 0,
                               ctx->stream>>>(ro, n_rows, nnz, c.sigma, cblocks, bnd);
      gen_tile_scan_kernel<<<static_cast<unsigned>(cblocks), kK1Threads, 0, ctx->stream>>>(
          ro, n_rows, nnz, c.omega, c.sigma, c.offset_bits, lanes, bnd, t->tile_x, t->tile_y,
          t->lane_desc);
      ++ctx->launches;
      cudaFreeAsync(bnd, ctx->stream);
    } else
      gen_tile_kernel<<<static_cast<unsigned>(blocks), 256, 0, ctx->stream>>>(
          ro, n_rows, nnz, c.omega, c.sigma, c.offset_bits, lanes, t->tile_x, t->tile_y,
          t->lane_desc, small ? 1 : 0);
    ++ctx->launches;
    MBX_CUDA(cudaGetLastError());
    if (!small) {
      gen_tile_entries_kernel<<<static_cast<unsigned>((tiles + 255) / 256), 256, 0,
                                ctx->stream>>>(ro, n_rows, nnz, c.omega, c.sigma,
                                               c.offset_bits, lanes, tiles, t->tile_x,
                                               t->tile_y, t->lane_desc);
      ++ctx->launches;
      MBX_CUDA(cudaGetLastError());
    }
  }
  tile_terminal_kernel<<<1, 1, 0, ctx->stream>>>(t->tile_x, t->tile_y, tiles, nnz, n_rows);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

void launch_trace_counts(mbx_context* ctx, const mbx_tile* t, unsigned long long* counters) {
  const int64_t tiles = t->info.tile_num;
  if (tiles == 0) return;
  trace_kernel<<<static_cast<unsigned>((tiles + 255) / 256), 256, 0, ctx->stream>>>(
      t->tile_x, t->tile_y, tiles, counters);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

int csr_pr_blocks(mbx_context* ctx, const mbx_matrix* m) {
  return static_cast<int>(grid_for(m->n_rows * 32, 256, int64_t(ctx->sm_count) * 8));
}

void launch_csr(mbx_context* ctx, const mbx_matrix* m, const void* x, void* y,
                const PrArgs* pr, double* cta_part, unsigned int* counter) {
  if (m->n_rows == 0) return;
  ensure_csr(ctx, m);
  const unsigned grid = static_cast<unsigned>(csr_pr_blocks(ctx, m));
  PrArgs a;
  if (pr) {
    a = *pr;
    a.block_part = cta_part;
    a.done_counter = counter;
  }
  if (pr) {  // the yardstick: row-serial sums in T, the reference's order
    if (m->precision == MBX_F32)
      csr_rowserial_pr_kernel<float><<<grid, 256, 0, ctx->stream>>>(
          m->ro, m->cols, static_cast<const float*>(m->vals), static_cast<const float*>(x),
          static_cast<float*>(y), m->n_rows, a);
    else
      csr_rowserial_pr_kernel<double><<<grid, 256, 0, ctx->stream>>>(
          m->ro, m->cols, static_cast<const double*>(m->vals), static_cast<const double*>(x),
          static_cast<double*>(y), m->n_rows, a);
  } else if (m->precision == MBX_F32) {
    if (pr)
      csr_kernel<float, true><<<grid, 256, 0, ctx->stream>>>(
          m->ro, m->cols, static_cast<const float*>(m->vals), static_cast<const float*>(x),
          static_cast<float*>(y), m->n_rows, a);
    else
      csr_kernel<float, false><<<grid, 256, 0, ctx->stream>>>(
          m->ro, m->cols, static_cast<const float*>(m->vals), static_cast<const float*>(x),
          static_cast<float*>(y), m->n_rows, a);
  } else {
    if (pr)
      csr_kernel<double, true><<<grid, 256, 0, ctx->stream>>>(
          m->ro, m->cols, static_cast<const double*>(m->vals), static_cast<const double*>(x),
          static_cast<double*>(y), m->n_rows, a);
    else
      csr_kernel<double, false><<<grid, 256, 0, ctx->stream>>>(
          m->ro, m->cols, static_cast<const double*>(m->vals), static_cast<const double*>(x),
          static_cast<double*>(y), m->n_rows, a);
  }
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

int64_t dangling_suffix_start(mbx_context* ctx, const uint32_t* mask_dev, int64_t n) {
  const int64_t words = (n + 31) / 32;
  if (n <= 0) return 0;
  std::vector<uint32_t> m(words);
  MBX_CUDA(cudaMemcpyAsync(m.data(), mask_dev, words * 4, cudaMemcpyDeviceToHost, ctx->stream));
  MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t f = n;  // walk down from the top while rows are dangling
  while (f > 0 && ((m[(f - 1) >> 5] >> ((f - 1) & 31)) & 1u)) --f;
  for (int64_t w = 0; w < (f >> 5); ++w)  // nothing dangling below f
    if (m[w]) return -1;
  for (int64_t r = f & ~int64_t(31); r < f; ++r)
    if ((m[r >> 5] >> (r & 31)) & 1u) return -1;
  return f;
}

// Loads the PageRank start / yardstick kernels of `precision` now.  With
// CUDA's lazy module loading the FIRST launch of a kernel loads its module,
// which waits for the kernels already running in the context; a caller that
// has a spinning peer barrier in flight (several ranks of a fused shard
// group in one process) would block there until the barrier gives up.
void preload_pr_kernels(int precision) {
  cudaFuncAttributes a;
  if (precision == MBX_F32) {
    MBX_CUDA(cudaFuncGetAttributes(&a, pr_init_kernel<float>));
    MBX_CUDA(cudaFuncGetAttributes(&a, csr_rowserial_pr_kernel<float>));
  } else {
    MBX_CUDA(cudaFuncGetAttributes(&a, pr_init_kernel<double>));
    MBX_CUDA(cudaFuncGetAttributes(&a, csr_rowserial_pr_kernel<double>));
  }
}

void launch_pr_init(mbx_context* ctx, int precision, int64_t n, const void* pi0, void* pi,
                    const uint32_t* dangling, PrScalars* out, double* block_part,
                    unsigned int* counter) {
  PrArgs a;
  a.dangling = dangling;
  a.next = out;
  a.block_part = block_part;
  a.done_counter = counter;
  const unsigned grid = grid_for(n, 256, int64_t(ctx->sm_count) * 4);
  if (precision == MBX_F32)
    pr_init_kernel<float><<<grid, 256, 0, ctx->stream>>>(static_cast<const float*>(pi0),
                                                         static_cast<float*>(pi), n, a);
  else
    pr_init_kernel<double><<<grid, 256, 0, ctx->stream>>>(static_cast<const double*>(pi0),
                                                          static_cast<double*>(pi), n, a);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

void launch_dangling_mask(mbx_context* ctx, const mbx_matrix* m_, uint32_t* mask) {
  mbx_matrix* m = const_cast<mbx_matrix*>(m_);
  const int64_t words = (m->n_cols + 31) / 32;
  const size_t bytes = size_t(words > 0 ? words : 1) * 4;
  // the empty columns depend on the pattern alone: computed once per matrix
  // (a compacted matrix then needs no CSR for later PageRank plans)
  if (m->dmask) {
    MBX_CUDA(cudaMemcpyAsync(mask, m->dmask, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  ensure_csr(ctx, m);
  MBX_CUDA(cudaMemsetAsync(mask, 0, bytes, ctx->stream));
  if (m->nnz > 0) {
    seen_columns_kernel<<<grid_for(m->nnz, 256), 256, 0, ctx->stream>>>(m->cols, m->nnz, mask);
    ++ctx->launches;
  }
  if (words > 0) {
    invert_mask_kernel<<<static_cast<unsigned>((words + 255) / 256), 256, 0, ctx->stream>>>(
        mask, m->n_cols);
    ++ctx->launches;
  }
  MBX_CUDA(cudaGetLastError());
  MBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->dmask), bytes + 64, ctx->stream));
  MBX_CUDA(cudaMemcpyAsync(m->dmask, mask, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
}

template <typename T>
__global__ void vertex_map_kernel(int64_t n, const int32_t* __restrict__ map,
                                  const T* __restrict__ src, T* __restrict__ dst, bool to_new) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += int64_t(gridDim.x) * blockDim.x) {
    if (to_new)
      dst[map[v]] = src[v];
    else
      dst[v] = src[map[v]];
  }
}

void launch_vertex_map(mbx_context* ctx, int precision, int64_t n, const int32_t* map,
                       const void* src, void* dst, bool to_new) {
  if (n == 0) return;
  const unsigned grid = grid_for(n, 256, int64_t(ctx->sm_count) * 8);
  if (precision == MBX_F32)
    vertex_map_kernel<float><<<grid, 256, 0, ctx->stream>>>(
        n, map, static_cast<const float*>(src), static_cast<float*>(dst), to_new);
  else
    vertex_map_kernel<double><<<grid, 256, 0, ctx->stream>>>(
        n, map, static_cast<const double*>(src), static_cast<double*>(dst), to_new);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

void launch_narrow_cols(mbx_context* ctx, const int64_t* src, int32_t* dst, int64_t n,
                        int64_t limit, int* bad) {
  if (n == 0) return;
  narrow_cols_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, dst, n, limit, bad);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

void launch_narrow_rows(mbx_context* ctx, const int64_t* src, uint32_t* dst, int64_t n,
                        int* bad) {
  if (n == 0) return;
  narrow_rows_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, dst, n, bad);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

}  // namespace mbx
