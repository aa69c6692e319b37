// solvers.cu -- unpreconditioned BiCGSTAB on the device:
// bicgstab<T> of include/merbit/solvers.hpp:224-373 with its three SpMVs per
// iteration running through K2/K3 (the same TILE and slot copy as PageRank)
// and every dot / axpy as a device kernel.
//
// The recurrence is the reference's, step for step (numbers refer to the
// comments at solvers.hpp:303-356): scalars are T values (rho, alpha, omega,
// beta) computed in T from T operands; inner products accumulate in fp64
// with a fixed reduction tree (deterministic) and are rounded to T once;
// vector updates round every product/sum in T exactly as written (no FMA
// contraction).  The stopping test is the reference's true residual
// ||A x - b|| / ||b|| (a third SpMV per pass), accumulated in fp64.
// Breakdown (zero or non-finite denominator) stops the device loop with the
// reference's reason string.  Host code only enqueues: the scalars, the
// stop flag and the residual history live on the device; the host reads
// one pinned flag per pass with one pass of look-ahead.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include "mbx_internal.h"

namespace mbx {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;

enum : int {
  kReasonNone = 0,
  kReasonRho = 1,
  kReasonRhatV = 2,
  kReasonTT = 3,
  kReasonOmega = 4,
  kReasonDiverged = 5,
};

const char* reason_name(int r) {
  switch (r) {
    case kReasonRho: return "rho";
    case kReasonRhatV: return "rhat_dot_v";
    case kReasonTT: return "t_dot_t";
    case kReasonOmega: return "omega";
    case kReasonDiverged: return "diverged";
    default: return "";
  }
}

// Device-resident recurrence state.  T-valued scalars are stored as the
// double holding the exact T value.
struct BiState {
  double rho, alpha, omega, beta, rho_new;
  double b_norm, resid;
  int64_t iterations;
  int status;  // -1 running, 0 converged, 2 breakdown (max_iterations: host)
  int reason;
  int stop;
  int pad;
};

enum Mode : int { kRho, kAlpha, kOmega, kResid, kBnorm };

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ bool finite_t(T v) {
  return isfinite(static_cast<double>(v));
}

template <typename T>
__device__ void breakdown(BiState* s, int reason, int iter) {
  s->status = 2;
  s->reason = reason;
  s->iterations = iter;
  s->stop = 1;
}

// One or two fp64 inner products over n, a fixed grid-stride assignment,
// warp butterflies, a fixed warp order per block and a fixed block order in
// the last block -- then the scalar step of the recurrence that consumes them.
template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads)
    bi_reduce_kernel(const T* __restrict__ a, const T* __restrict__ b, int64_t n, BiState* st,
                     double* hist, double* part, unsigned int* counter, double tol, int iter) {
  if (MODE != kBnorm && st->stop) return;
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double av = static_cast<double>(a[i]);
    if (MODE == kRho || MODE == kAlpha) {
      s0 += av * static_cast<double>(b[i]);
    } else if (MODE == kOmega) {
      s0 += av * av;
      s1 += av * static_cast<double>(b[i]);
    } else if (MODE == kResid) {
      const double d = av - static_cast<double>(b[i]);
      s0 += d * d;
    } else {
      s0 += av * av;
    }
  }
  __shared__ double sm[2][32];
  __shared__ bool is_last;
  s0 = warp_sum_d(s0);
  s1 = warp_sum_d(s1);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) {
    sm[0][w] = s0;
    sm[1][w] = s1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int i = 0; i < nw; ++i) {
      t0 += sm[0][i];
      t1 += sm[1][i];
    }
    part[2 * blockIdx.x] = t0;
    part[2 * blockIdx.x + 1] = t1;
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // the last block folds the block partials: fixed thread->block map, warp
  // butterflies, warps in order (deterministic); L2-coherent loads in flight
  // together instead of one serial round trip per block
  double q0 = 0.0, q1 = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(part) + i);
    q0 += v.x;
    q1 += v.y;
  }
  q0 = warp_sum_d(q0);
  q1 = warp_sum_d(q1);
  __syncthreads();
  if (l == 0) {
    sm[0][w] = q0;
    sm[1][w] = q1;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double d0 = 0.0, d1 = 0.0;
  for (int i = 0; i < nw; ++i) {
    d0 += sm[0][i];
    d1 += sm[1][i];
  }
  *counter = 0;
  if (MODE == kBnorm) {
    st->b_norm = sqrt(d0);
  } else if (MODE == kRho) {
    // (1) rho_k = <r_hat, r_{k-1}>; (2) beta = (rho_k / rho_{k-1}) * (alpha / omega)
    const T rn = static_cast<T>(d0);
    if (rn == T(0) || !finite_t(rn)) {
      breakdown<T>(st, kReasonRho, iter);
      return;
    }
    st->rho_new = static_cast<double>(rn);
    if (iter > 1) {
      const T q1 = rn / static_cast<T>(st->rho);
      const T q2 = static_cast<T>(st->alpha) / static_cast<T>(st->omega);
      st->beta = static_cast<double>(T(q1 * q2));
    }
  } else if (MODE == kAlpha) {
    // (5) alpha = rho_k / <r_hat, v>
    const T rv = static_cast<T>(d0);
    if (rv == T(0) || !finite_t(rv)) {
      breakdown<T>(st, kReasonRhatV, iter);
      return;
    }
    st->alpha = static_cast<double>(T(static_cast<T>(st->rho_new) / rv));
  } else if (MODE == kOmega) {
    // (8) omega = <t, s> / <t, t>
    const T tt = static_cast<T>(d0);
    if (tt == T(0) || !finite_t(tt)) {
      breakdown<T>(st, kReasonTT, iter);
      return;
    }
    const T om = static_cast<T>(d1) / tt;
    if (om == T(0) || !finite_t(om)) {
      breakdown<T>(st, kReasonOmega, iter);
      return;
    }
    st->omega = static_cast<double>(om);
  } else {
    // stopping test on the true residual ||A x - b|| / ||b|| (solvers.hpp:357-370)
    const double res = sqrt(d0) / st->b_norm;
    hist[iter - 1] = res;
    st->iterations = iter;
    st->resid = res;
    st->rho = st->rho_new;
    if (!isfinite(res)) {
      breakdown<T>(st, kReasonDiverged, iter);
    } else if (res < tol) {
      st->status = 0;
      st->stop = 1;
    }
  }
}

template <typename T>
__device__ __forceinline__ T mul(T a, T b);
template <>
__device__ __forceinline__ float mul<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add(T a, T b);
template <>
__device__ __forceinline__ float add<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add<double>(double a, double b) { return __dadd_rn(a, b); }

// (3) p = r + beta * (p - omega * v)   (p = r on the first pass)
template <typename T>
__global__ void __launch_bounds__(kThreads)
    bi_p_kernel(const T* __restrict__ r, T* __restrict__ p, const T* __restrict__ v, int64_t n,
                const BiState* st, int iter) {
  if (st->stop) return;
  const T beta = static_cast<T>(st->beta), omega = static_cast<T>(st->omega);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = iter == 1 ? r[i] : add(r[i], mul(beta, add(p[i], -mul(omega, v[i]))));
}

// (6) s = r - alpha * v
template <typename T>
__global__ void __launch_bounds__(kThreads)
    bi_s_kernel(const T* __restrict__ r, const T* __restrict__ v, T* __restrict__ s, int64_t n,
                const BiState* st) {
  if (st->stop) return;
  const T alpha = static_cast<T>(st->alpha);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    s[i] = add(r[i], -mul(alpha, v[i]));
}

// (9) x += alpha * p + omega * s;  (10) r = s - omega * t
template <typename T>
__global__ void __launch_bounds__(kThreads)
    bi_xr_kernel(T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                 const T* __restrict__ s, const T* __restrict__ t, int64_t n, const BiState* st) {
  if (st->stop) return;
  const T alpha = static_cast<T>(st->alpha), omega = static_cast<T>(st->omega);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    x[i] = add(x[i], add(mul(alpha, p[i]), mul(omega, s[i])));
    r[i] = add(s[i], -mul(omega, t[i]));
  }
}

template <typename T>
__global__ void bi_init_kernel(const T* __restrict__ b, T* r, T* rh, T* p, T* v, T* s, T* t, T* x,
                               int64_t n, BiState* st) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    r[i] = b[i];
    rh[i] = b[i];
    p[i] = v[i] = s[i] = t[i] = x[i] = T(0);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rho = st->alpha = st->omega = 1.0;
    st->beta = st->rho_new = 0.0;
    st->b_norm = 0.0;
    st->resid = INFINITY;
    st->iterations = 0;
    st->status = -1;
    st->reason = kReasonNone;
    st->stop = 0;
  }
}

struct Buffers {
  void* vec[9] = {};  // r, r_hat, p, v, s, t, x, ax, b
  BiState* st = nullptr;
  double* hist = nullptr;
  double* part = nullptr;
  unsigned int* counter = nullptr;
  void* ws = nullptr;
};

template <typename T>
void run_bicgstab(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t, const Geometry& g,
                  const mbx_bicgstab_config& cfg, const Buffers& B, int* host_flags,
                  cudaEvent_t* ev, int64_t* passes_launched) {
  cudaStream_t s = ctx->stream;
  const int64_t n = m->n_rows;
  T* r = static_cast<T*>(B.vec[0]);
  T* rh = static_cast<T*>(B.vec[1]);
  T* p = static_cast<T*>(B.vec[2]);
  T* v = static_cast<T*>(B.vec[3]);
  T* sv = static_cast<T*>(B.vec[4]);
  T* tv = static_cast<T*>(B.vec[5]);
  T* x = static_cast<T*>(B.vec[6]);
  T* ax = static_cast<T*>(B.vec[7]);
  const T* b = static_cast<const T*>(B.vec[8]);
  const unsigned grid = static_cast<unsigned>(
      std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, ctx->sm_count * 4)));
  // the reference compares resid < double(cfg.tol) with tol of type T
  const double tol = static_cast<double>(static_cast<T>(cfg.tol));
  int64_t launched = 0;
  for (int64_t iter = 1; iter <= cfg.max_iters; ++iter) {
    const int it = static_cast<int>(iter);
    bi_reduce_kernel<T, kRho><<<grid, kThreads, 0, s>>>(rh, r, n, B.st, B.hist, B.part,
                                                        B.counter, tol, it);
    bi_p_kernel<T><<<grid, kThreads, 0, s>>>(r, p, v, n, B.st, it);
    launch_spmv(ctx, m, t, g, p, v, B.ws, nullptr);  // (4) v = A p
    bi_reduce_kernel<T, kAlpha><<<grid, kThreads, 0, s>>>(rh, v, n, B.st, B.hist, B.part,
                                                          B.counter, tol, it);
    bi_s_kernel<T><<<grid, kThreads, 0, s>>>(r, v, sv, n, B.st);
    launch_spmv(ctx, m, t, g, sv, tv, B.ws, nullptr);  // (7) t = A s
    bi_reduce_kernel<T, kOmega><<<grid, kThreads, 0, s>>>(tv, sv, n, B.st, B.hist, B.part,
                                                          B.counter, tol, it);
    bi_xr_kernel<T><<<grid, kThreads, 0, s>>>(x, r, p, sv, tv, n, B.st);
    launch_spmv(ctx, m, t, g, x, ax, B.ws, nullptr);  // A x for the stopping test
    bi_reduce_kernel<T, kResid><<<grid, kThreads, 0, s>>>(ax, b, n, B.st, B.hist, B.part,
                                                          B.counter, tol, it);
    ctx->launches += 7;
    MBX_CUDA(cudaGetLastError());
    ++launched;
    // stop flag of this pass to pinned memory; decide on the previous pass's
    // flag so the device always has the next pass queued
    const int slot = int(iter & 1);
    MBX_CUDA(cudaMemcpyAsync(host_flags + slot, &B.st->stop, sizeof(int), cudaMemcpyDeviceToHost,
                             s));
    MBX_CUDA(cudaEventRecord(ev[slot], s));
    if (iter >= 2) {
      MBX_CUDA(cudaEventSynchronize(ev[slot ^ 1]));
      if (host_flags[slot ^ 1]) break;
    }
  }
  *passes_launched = launched;
}

}  // namespace
}  // namespace mbx

namespace {

template <typename F>
int bguard(F&& f) {
  try {
    f();
    return MBX_OK;
  } catch (const mbx::Error& e) {
    mbx::set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    mbx::set_last_error(e.what());
    return MBX_ERROR;
  }
}

}  // namespace

extern "C" {

MBX_API int mbx_bicgstab(mbx_context* ctx, const mbx_matrix* a, const mbx_tile* t,
                         const mbx_simt_config* c, const mbx_bicgstab_config* cfg,
                         const void* b_host, void* x_host, double* residual_history_host,
                         mbx_bicgstab_result* result) {
  return bguard([&] {
    using mbx::fail;
    if (a->n_rows != a->n_cols) fail(MBX_DIMENSION_ERROR, "bicgstab needs a square system");
    mbx::validate_config(c);
    mbx::validate_tile(a, t, c);
    if (cfg->max_iters < 0) fail(MBX_CONFIG_ERROR, "bicgstab: max_iters must be >= 0");
    mbx::DeviceGuard dg(ctx->device);  // the caller's current device is restored
    cudaStream_t s = ctx->stream;
    const int64_t n = a->n_rows;
    const size_t vs = mbx::value_size(a->precision);
    mbx_bicgstab_result res{};
    res.preprocess_seconds = t->info.preprocess_seconds;
    res.final_residual = INFINITY;
    res.status = 1;  // max_iterations unless the device says otherwise
    const mbx::Geometry g = mbx::make_geometry(ctx, a, t, c->block_size);
    mbx::Buffers B;
    auto alloc = [&](size_t bytes) {
      void* p = nullptr;
      MBX_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 256), s));
      return p;
    };
    for (void*& v : B.vec) v = alloc(n * vs + 256);
    B.st = static_cast<mbx::BiState*>(alloc(sizeof(mbx::BiState)));
    B.hist = static_cast<double*>(alloc(std::max<int64_t>(cfg->max_iters, 1) * sizeof(double)));
    B.part = static_cast<double*>(alloc(2 * sizeof(double) * (ctx->sm_count * 4 + 1)));
    B.counter = static_cast<unsigned int*>(alloc(64));
    B.ws = alloc(mbx::spmv_workspace_bytes(g, a->precision, false));
    MBX_CUDA(cudaMemsetAsync(B.counter, 0, 64, s));
    if (n) MBX_CUDA(cudaMemcpyAsync(B.vec[8], b_host, n * vs, cudaMemcpyHostToDevice, s));
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->sm_count * 4)));
    int* flags = nullptr;
    MBX_CUDA(cudaMallocHost(&flags, 4 * sizeof(int)));
    cudaEvent_t ev[2], e0, e1;
    for (auto* e : {&ev[0], &ev[1], &e0, &e1}) MBX_CUDA(cudaEventCreate(e));
    auto cleanup = [&] {
      cudaStreamSynchronize(s);
      for (void* v : B.vec) cudaFreeAsync(v, s);
      for (void* v : {static_cast<void*>(B.st), static_cast<void*>(B.hist),
                      static_cast<void*>(B.part), static_cast<void*>(B.counter), B.ws})
        cudaFreeAsync(v, s);
      cudaStreamSynchronize(s);
      cudaFreeHost(flags);
      for (auto e : {ev[0], ev[1], e0, e1}) cudaEventDestroy(e);
    };
    try {
      double b_norm = 0.0;
      if (a->precision == MBX_F32) {
        using T = float;
        T* v[9];
        for (int i = 0; i < 9; ++i) v[i] = static_cast<T*>(B.vec[i]);
        mbx::bi_init_kernel<T><<<grid, 256, 0, s>>>(v[8], v[0], v[1], v[2], v[3], v[4], v[5],
                                                    v[6], n, B.st);
        mbx::bi_reduce_kernel<T, mbx::kBnorm><<<grid, 256, 0, s>>>(v[8], v[8], n, B.st, B.hist,
                                                                   B.part, B.counter, 0.0, 0);
      } else {
        using T = double;
        T* v[9];
        for (int i = 0; i < 9; ++i) v[i] = static_cast<T*>(B.vec[i]);
        mbx::bi_init_kernel<T><<<grid, 256, 0, s>>>(v[8], v[0], v[1], v[2], v[3], v[4], v[5],
                                                    v[6], n, B.st);
        mbx::bi_reduce_kernel<T, mbx::kBnorm><<<grid, 256, 0, s>>>(v[8], v[8], n, B.st, B.hist,
                                                                   B.part, B.counter, 0.0, 0);
      }
      ctx->launches += 2;
      MBX_CUDA(cudaGetLastError());
      MBX_CUDA(cudaMemcpyAsync(&b_norm, &B.st->b_norm, sizeof(double), cudaMemcpyDeviceToHost, s));
      MBX_CUDA(cudaStreamSynchronize(s));
      if (b_norm == 0.0) {  // solvers.hpp:279-283
        res.status = 0;
        res.final_residual = 0.0;
        res.iterations = 0;
      } else {
        int64_t launched = 0;
        MBX_CUDA(cudaEventRecord(e0, s));
        if (a->precision == MBX_F32)
          mbx::run_bicgstab<float>(ctx, a, t, g, *cfg, B, flags, ev, &launched);
        else
          mbx::run_bicgstab<double>(ctx, a, t, g, *cfg, B, flags, ev, &launched);
        MBX_CUDA(cudaEventRecord(e1, s));
        MBX_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        MBX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        res.iterate_seconds = ms * 1e-3;
        mbx::BiState st;
        MBX_CUDA(cudaMemcpy(&st, B.st, sizeof(st), cudaMemcpyDeviceToHost));
        res.iterations = st.iterations;
        res.final_residual = st.iterations > 0 ? st.resid : INFINITY;
        res.status = st.status >= 0 ? st.status : 1;
        std::strncpy(res.breakdown_reason, mbx::reason_name(st.reason),
                     sizeof(res.breakdown_reason) - 1);
        // one history entry per completed pass (a breakdown before the
        // stopping test leaves its pass out, as residual_history.push_back)
        const int64_t hl = st.iterations - (st.status == 2 && st.reason != mbx::kReasonDiverged);
        if (residual_history_host && hl > 0)
          MBX_CUDA(cudaMemcpy(residual_history_host, B.hist, hl * sizeof(double),
                              cudaMemcpyDeviceToHost));
      }
      if (n) MBX_CUDA(cudaMemcpy(x_host, B.vec[6], n * vs, cudaMemcpyDeviceToHost));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    *result = res;
  });
}

}  // extern "C"
