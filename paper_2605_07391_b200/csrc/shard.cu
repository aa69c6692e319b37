// shard.cu -- row-sharded multi-GPU PageRank (BASELINE config C4).
//
// One process per GPU.  GPU g owns the merge-path-balanced row block
// [b_g, b_{g+1}) of P (mbx_plan_row_shards: diagonal cuts snapped to row
// starts) with its own TILE.  Only NON-DANGLING vertices are ever gathered
// (a dangling vertex is an empty column of P), so the exchange carries only
// them: column indices are remapped once into the compacted layout
//   pos(v) = owner(v) * chunk + #{non-dangling u in [b_owner, v)},
// each rank keeps its full rows of pi locally (residual, dangling mass,
// final answer) and its commit also writes the non-dangling entries into its
// exchange chunk, and one in-place ncclAllGather of equal-size chunks per
// iteration delivers every gathered entry to every GPU (R-MAT s24: 44 % of
// the vertices, 2.3x fewer bytes over NVLink than the full vector).  The tail of each chunk carries that rank's
// fp64 reduction scalars (dangling mass, L1 residual, mass, ERR), so the
// same collective doubles as the all-reduce; a one-warp combine kernel folds
// the G tails in rank order (deterministic, identical on every rank) and
// decides convergence.  Iteration = K2 + K3 (PR mode, local rows) ->
// ncclAllGather -> combine, captured once as a CUDA graph.
//
// Fused mode (mbx_shard_group_create_peer / export / connect): no all-gather.
// The commit itself stores each non-dangling pi_new (and K3 the scalar tail)
// into every peer's exchange buffer through CUDA IPC mappings -- P2P stores
// over NVLink spread across the whole SpMV -- and peer_barrier_kernel
// (system-scope release/acquire epochs, bounded wait) ends the iteration.
//
// Virtual mode (nccl_id == NULL, nlocal == world): all shards live in one
// process on one device and write into one shared buffer, so no exchange is
// needed -- the sharded kernels, remap and combine are verified on a single
// GPU (tests/test_gpu_shards.py).
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "mbx_internal.h"

namespace mbx {
namespace {

// NCCL is resolved at first use, not linked: a process that already loaded
// an NCCL (e.g. PyTorch's) keeps using that one -- two libnccl.so.2 of
// different versions in one process break each other's symbol resolution.
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
  static Nccl api{};
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.GetErrorString =
        reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather ||
        !api.AllReduce || !api.GetErrorString) {
      err = "libnccl.so.2 lacks a required symbol";
      api.GetUniqueId = nullptr;
    }
  });
  if (!api.GetUniqueId) fail(MBX_NCCL_ERROR, err);
  return api;
}

#define MBX_NCCL(call)                                                                \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess)                                                            \
      ::mbx::fail(MBX_NCCL_ERROR, std::string("NCCL error ") +                        \
                                      ::mbx::nccl().GetErrorString(r_) + " in " #call); \
  } while (0)

// gpre[v] = number of non-dangling vertices in [0, v) (exclusive scan of seen)
__device__ __forceinline__ int64_t compact_pos(int64_t v, const int64_t* bounds, int world,
                                               int64_t chunk_elems, const int64_t* gpre) {
  int g = 0;
  while (g + 1 < world && bounds[g + 1] <= v) ++g;
  return int64_t(g) * chunk_elems + (gpre[v] - gpre[bounds[g]]);
}

__global__ void remap_cols_kernel(const int32_t* __restrict__ in, int64_t nnz,
                                  const int64_t* __restrict__ bounds, int world,
                                  int64_t chunk_elems, const int64_t* __restrict__ gpre,
                                  int32_t* __restrict__ out) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x)
    out[k] = int32_t(compact_pos(in[k], bounds, world, chunk_elems, gpre));
}

// exchange slot of every local row (-1: dangling, never gathered)
__global__ void xmap_kernel(const uint8_t* __restrict__ seen, int64_t r0, int64_t rows,
                            const int64_t* __restrict__ bounds, int world, int64_t chunk_elems,
                            const int64_t* __restrict__ gpre, int32_t* __restrict__ xmap) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += int64_t(gridDim.x) * blockDim.x)
    xmap[i] = seen[r0 + i] ? int32_t(compact_pos(r0 + i, bounds, world, chunk_elems, gpre)) : -1;
}

__global__ void seen_to_count_kernel(const uint8_t* __restrict__ seen, int64_t n,
                                     int64_t* __restrict__ cnt) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    cnt[i] = seen[i] ? 1 : 0;
}

// exchange copy of a start vector: x[xmap[i]] = pi[i]
template <typename T>
__global__ void scatter_exchange_kernel(const T* __restrict__ pi, int64_t rows,
                                        const int32_t* __restrict__ xmap, T* __restrict__ x) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += int64_t(gridDim.x) * blockDim.x)
    if (xmap[i] >= 0) x[xmap[i]] = pi[i];
}

__global__ void seen_flags_kernel(const int32_t* __restrict__ cols, int64_t nnz, uint8_t* seen) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x)
    seen[cols[k]] = 1;
}

__global__ void local_dangling_kernel(const uint8_t* __restrict__ seen, int64_t r0, int64_t rows,
                                      uint32_t* __restrict__ bits) {
  const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= (rows + 31) / 32) return;
  uint32_t v = 0;
  for (int b = 0; b < 32; ++b) {
    const int64_t i = w * 32 + b;
    if (i < rows && !seen[r0 + i]) v |= 1u << b;
  }
  bits[w] = v;
}

// pi_0 = 1/n on the shard's rows; the rank's dangling count goes to the
// tail as an exact integer, so its mass (count * 1/n in fp64) is exact and
// independent of the reduction order.
template <typename T>
__global__ void shard_init_kernel(T* __restrict__ pi, int64_t rows, T val,
                                  const uint32_t* __restrict__ dangling,
                                  unsigned long long* count, const int32_t* __restrict__ xmap,
                                  T* __restrict__ x) {
  unsigned long long c = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += int64_t(gridDim.x) * blockDim.x) {
    pi[i] = val;
    if (xmap[i] >= 0) x[xmap[i]] = val;
    if ((i & 31) == 0) c += __popc(dangling[i >> 5] & (rows - i >= 32 ? 0xFFFFFFFFu
                                                                       : (1u << (rows - i)) - 1u));
  }
  for (int o = 16; o >= 1; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void shard_init_tail_kernel(const unsigned long long* count, int64_t rows, double val,
                                       PrScalars* tail) {
  tail->dangling = double(*count) * val;
  tail->mass = double(rows) * val;
  tail->resid = 0.0;
  tail->err = 0.0;
}

// Fold the world tails in rank order into the global scalars of iteration
// `iter` and decide convergence (solvers.hpp:201-213).
// iter_dev (device-driven loop): the iteration is *iter_dev + 1, `out` is
// the scalar array's base, and the kernel advances the counter.
__device__ void combine_body(const unsigned char* __restrict__ pi_base, int64_t chunk_bytes,
                             int64_t tail_off, int world, PrScalars* out, int* stop,
                             int* stop_iter, int iter, double err_tol, int64_t* iter_dev,
                             int64_t max_iters) {
  if (stop && *stop) return;
  if (iter_dev) {
    if (*iter_dev >= max_iters) return;
    iter = int(*iter_dev + 1);
    out += iter;
  }
  double d = 0.0, r = 0.0, m = 0.0, e = 0.0;
  for (int g = 0; g < world; ++g) {
    const PrScalars* t =
        reinterpret_cast<const PrScalars*>(pi_base + int64_t(g) * chunk_bytes + tail_off);
    d += t->dangling;
    r += t->resid;
    m += t->mass;
    e = fmax(e, t->err);
  }
  out->dangling = d;
  out->resid = r;
  out->mass = m;
  out->err = e;
  if (iter > 0 && stop) {
    if (m == 0.0) {
      *stop = 2;
      *stop_iter = iter;
    } else if (e < err_tol) {
      *stop = 1;
      *stop_iter = iter;
    }
  }
  if (iter_dev) *iter_dev += 1;
}

__global__ void combine_kernel(const unsigned char* __restrict__ pi_base, int64_t chunk_bytes,
                               int64_t tail_off, int world, PrScalars* out, int* stop,
                               int* stop_iter, int iter, double err_tol, int64_t* iter_dev,
                               int64_t max_iters) {
  if (threadIdx.x == 0)
    combine_body(pi_base, chunk_bytes, tail_off, world, out, stop, stop_iter, iter, err_tol,
                 iter_dev, max_iters);
}


__global__ void shard_loop_cond_kernel(cudaGraphConditionalHandle h, const int64_t* iter_dev,
                                       int64_t max_iters, const int* stop) {
  cudaGraphSetConditional(h, (*iter_dev < max_iters && !*stop) ? 1u : 0u);
}

__global__ void slice_rows_kernel(const uint32_t* __restrict__ ro, int64_t r0, int64_t rows,
                                  uint32_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= rows;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = ro[r0 + i] - ro[r0];
}

// ---- fused exchange (peer shard groups) ------------------------------------
struct PeerFlags {
  uint64_t* f[8];  // every rank's epoch array (own included), mapped
  int world = 1;
  int rank = 0;
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Device barrier across the group: publish this rank's epoch in every
// rank's flag array (release, system scope: the NVLink stores of the
// preceding K2/K3 are ordered before it), then wait until every rank has
// published it here (acquire).  Skipped once the run has stopped -- every
// rank reaches the same stop decision at the same iteration.  Bounded: a
// peer that never arrives sets *err instead of hanging the GPU.
// iter_dev (device-driven loop): the slot is slot + iteration, and nothing
// happens past max_iters (every rank skips the same barriers).
__device__ void peer_barrier_body(const PeerFlags& pf, const uint64_t* __restrict__ base, int slot,
                                  const int* stop, int* err, const int64_t* iter_dev,
                                  int64_t max_iters) {
  if (stop && *stop) return;
  if (iter_dev && *iter_dev >= max_iters) return;
  const uint64_t epoch = *base + uint64_t(slot) + (iter_dev ? uint64_t(*iter_dev + 1) : 0ull);
  __threadfence_system();
  for (int k = 0; k < pf.world; ++k)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pf.f[k] + pf.rank), "l"(epoch)
                 : "memory");
  const uint64_t t0 = globaltimer_ns();
  for (int k = 0; k < pf.world; ++k) {
    while (true) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(pf.f[pf.rank] + k)
                   : "memory");
      if (v >= epoch) break;
      if (globaltimer_ns() - t0 > 30ull * 1000000000ull) {
        atomicExch(err, 1);
        return;
      }
      __nanosleep(128);
    }
  }
}

__global__ void peer_barrier_kernel(PeerFlags pf, const uint64_t* __restrict__ base, int slot,
                                    const int* stop, int* err, const int64_t* iter_dev,
                                    int64_t max_iters) {
  if (threadIdx.x == 0) peer_barrier_body(pf, base, slot, stop, err, iter_dev, max_iters);
}

// fused groups: the barrier and the fold of the tails in one launch
__global__ void barrier_combine_kernel(PeerFlags pf, const uint64_t* __restrict__ base, int slot,
                                       const int* bstop, int* err, const int64_t* biter,
                                       const unsigned char* __restrict__ pi_base,
                                       int64_t chunk_bytes, int64_t tail_off, int world,
                                       PrScalars* out, int* stop, int* stop_iter, int iter,
                                       double err_tol, int64_t* iter_dev, int64_t max_iters) {
  if (threadIdx.x != 0) return;
  peer_barrier_body(pf, base, slot, bstop, err, biter, max_iters);
  combine_body(pi_base, chunk_bytes, tail_off, world, out, stop, stop_iter, iter, err_tol,
               iter_dev, max_iters);
}

__global__ void bump_epoch_kernel(uint64_t* base, uint64_t step) { *base += step; }

// global column flags = OR over the ranks' own flags (read over NVLink)
struct SeenPtrs {
  const uint8_t* p[8];
};
__global__ void seen_or_kernel(SeenPtrs sp, int world, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint8_t v = 0;
    for (int k = 0; k < world; ++k) v |= sp.p[k][i];
    out[i] = v;
  }
}

struct Shard {
  int g = 0;
  int li = 0;  // local index (slot in the group's local-row buffers)
  int32_t* xmap = nullptr;  // local row -> exchange slot, -1 for dangling
  int64_t r0 = 0, r1 = 0;
  mbx_matrix view{};  // the local matrix with remapped columns (non-owning)
  const mbx_tile* tile = nullptr;
  Geometry geo;
  int32_t* cols_remap = nullptr;
  uint32_t* dangling = nullptr;
  int64_t dang_from = -1;  // local dangling rows = [dang_from, rows) when a suffix
  uint32_t* carry_mask = nullptr;  // K2 -> K3: the range boundary rows
  double* block_part = nullptr;
  unsigned int* counter = nullptr;
  void* carry_ws = nullptr;
};

}  // namespace
}  // namespace mbx

struct mbx_shard_group_s {
  mbx_context* ctx = nullptr;
  int precision = MBX_F32;
  size_t vs = 4;
  int world = 1, rank0 = 0, nlocal = 1;
  int64_t n = 0;
  std::vector<int64_t> bounds;
  int64_t chunk_bytes = 0, chunk_elems = 0, tail_off = 0;
  void* pi[2] = {nullptr, nullptr};   // exchange buffers: world compacted chunks (+ tails)
  void* loc[2] = {nullptr, nullptr};  // full local rows of pi, one chunk per local shard
  int64_t lchunk_bytes = 0;
  std::vector<mbx::Shard> shards;
  mbx::PrScalars* gscal = nullptr;
  int* flags = nullptr;
  ncclComm_t comm = nullptr;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_launches = 0;
  mbx_simt_config c{};
  mbx_pagerank_config cfg{};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool ran = false;
  // ---- fused exchange (mbx_shard_group_create_peer / _connect) ----
  bool peer = false, connected = false, quiesced = false;
  mbx_matrix* pmat = nullptr;  // the rank's shard, kept for connect
  mbx_tile* ptile = nullptr;
  uint8_t* seen = nullptr;     // this rank's column flags (shared with the peers)
  uint64_t* pflags = nullptr;  // epochs published by the world (shared)
  uint64_t* run_base = nullptr;
  int* perr = nullptr;
  void* xpeer[2][8] = {};      // every rank's exchange buffer (own = pi[i])
  void* lpeer[2][8] = {};      // every rank's local rows (own = loc[i])
  uint8_t* speer[8] = {};
  mbx::PeerFlags pf{};
  std::vector<void*> opened;   // IPC mappings to close
  int64_t epoch_step = 0;
  // yardstick run (reference_iters > 0, solvers.hpp:178-191): CSR power
  // iterations through the same exchange; this rank's rows of pi* stay here
  void* yloc[2] = {nullptr, nullptr};
  mbx::PrScalars* yscal = nullptr;
  // peer barrier slots of one run: 0 entry, 1 + r yardstick iteration r,
  // main_base + r power iteration r, main_base + max_iters + 1 final
  int64_t main_base = 2;
  int64_t* iter_dev = nullptr;  // device-driven loop (virtual and fused groups)
};

namespace {

template <typename F>
int sguard(F&& f) {
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

void* dm(mbx_context* ctx, size_t b) {
  void* p = nullptr;
  MBX_CUDA(cudaMallocAsync(&p, std::max<size_t>(b, 256), ctx->stream));
  return p;
}

// IPC-shareable allocation (cudaIpcGetMemHandle needs a cudaMalloc base)
void* dm_shared(size_t b) {
  void* p = nullptr;
  MBX_CUDA(cudaMalloc(&p, std::max<size_t>(b, 256)));
  MBX_CUDA(cudaMemset(p, 0, std::max<size_t>(b, 256)));
  return p;
}

// barrier slots of one run: 0 = entry, 1 + r = after iteration r (r >= 0)
void peer_barrier(mbx_shard_group* G, int64_t slot, bool skippable,
                  const int64_t* iter_dev = nullptr) {
  mbx_context* ctx = G->ctx;
  mbx::peer_barrier_kernel<<<1, 32, 0, ctx->stream>>>(G->pf, G->run_base, int(slot),
                                                      skippable ? G->flags : nullptr, G->perr,
                                                      iter_dev, G->cfg.max_iters);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

// main = false: a yardstick iteration (own scalars, never stops).
// dev_loop: a power iteration of the device-driven loop (iteration number
// read from G->iter_dev by the barrier and the combine, which advances it).
void exchange_and_combine(mbx_shard_group* G, int slot, int iter, bool main = true,
                          bool dev_loop = false) {
  mbx_context* ctx = G->ctx;
  unsigned char* base = static_cast<unsigned char*>(G->pi[slot]);
  mbx::PrScalars* out = dev_loop ? G->gscal : (main ? G->gscal : G->yscal) + iter;
  int* stop = main ? G->flags : nullptr;
  int64_t* idev = dev_loop ? G->iter_dev : nullptr;
  if (G->peer) {
    // the chunk already went out with the commit: wait for every rank's,
    // then fold the tails -- one launch
    int64_t bslot;
    bool skippable;
    if (dev_loop) {
      bslot = G->main_base;
      skippable = true;
    } else if (main) {
      bslot = G->main_base + iter;
      skippable = iter > 0;
    } else {
      bslot = 1 + iter;
      skippable = false;
    }
    mbx::barrier_combine_kernel<<<1, 32, 0, ctx->stream>>>(
        G->pf, G->run_base, int(bslot), skippable ? G->flags : nullptr, G->perr,
        dev_loop ? G->iter_dev : nullptr, base, G->chunk_bytes, G->tail_off, G->world, out, stop,
        G->flags + 1, iter, G->cfg.err_tol, idev, G->cfg.max_iters);
    ++ctx->launches;
    MBX_CUDA(cudaGetLastError());
    return;
  }
  if (G->comm) {
    // in-place all-gather: each rank's chunk (pi rows + scalar tail)
    MBX_NCCL(mbx::nccl().AllGather(base + int64_t(G->rank0) * G->chunk_bytes, base, G->chunk_bytes,
                           ncclUint8, G->comm, ctx->stream));
  }
  mbx::combine_kernel<<<1, 32, 0, ctx->stream>>>(base, G->chunk_bytes, G->tail_off, G->world, out,
                                                 stop, G->flags + 1, iter, G->cfg.err_tol, idev,
                                                 G->cfg.max_iters);
  ++ctx->launches;
  MBX_CUDA(cudaGetLastError());
}

void launch_iteration(mbx_shard_group* G, int64_t r, bool dev_loop = false) {
  mbx_context* ctx = G->ctx;
  const int src = int((r - 1) & 1), dst = int(r & 1);
  for (mbx::Shard& s : G->shards) {
    mbx::PrArgs a;
    unsigned char* pold = static_cast<unsigned char*>(G->loc[src]) + int64_t(s.li) * G->lchunk_bytes;
    unsigned char* pnew = static_cast<unsigned char*>(G->loc[dst]) + int64_t(s.li) * G->lchunk_bytes;
    unsigned char* xnew = static_cast<unsigned char*>(G->pi[dst]) + int64_t(s.g) * G->chunk_bytes;
    a.pi_old = pold;
    a.dangling = s.dangling;
    a.dang_from = s.dang_from;
    a.yardstick = G->cfg.reference_iters > 0
                      ? static_cast<unsigned char*>(G->yloc[G->cfg.reference_iters & 1]) +
                            int64_t(s.li) * G->lchunk_bytes
                      : nullptr;
    a.yard_const = G->precision == MBX_F32 ? double(1.0f / float(G->n)) : 1.0 / double(G->n);
    a.damping = G->cfg.damping;
    a.inv_n = 1.0 / double(G->n);
    a.prev = G->gscal + (r - 1);
    a.next = reinterpret_cast<mbx::PrScalars*>(xnew + G->tail_off);
    a.xout = G->pi[dst];
    a.xmap = s.xmap;
    if (G->peer)
      for (int k = 0; k < G->world; ++k)
        if (k != G->rank0) a.xpeer[a.npeer++] = G->xpeer[dst][k];
    a.carry_mask = s.carry_mask;
    a.block_part = s.block_part;
    a.done_counter = s.counter;
    a.stop = G->flags;
    a.stop_iter = G->flags + 1;
    a.iter = int(r);
    a.err_tol = G->cfg.err_tol;
    a.check_stop = 0;
    if (dev_loop) {  // prev from the device counter, next stays the parity's tail
      a.iter_dev = G->iter_dev;
      a.scal_base = G->gscal;
      a.max_iters = G->cfg.max_iters;
      a.prev = nullptr;
    }
    mbx::launch_spmv(ctx, &s.view, s.tile, s.geo, G->pi[src], pnew, s.carry_ws, &a);
  }
  exchange_and_combine(G, dst, int(r), true, dev_loop);
}

// One yardstick iteration: the plain CSR kernel (spmv_csr_reference, as the
// single-GPU yardstick) on every local shard, its commit doing the rank
// update into the local rows of pi* and the exchange copy, then the exchange.
void launch_yard_iteration(mbx_shard_group* G, int64_t r) {
  mbx_context* ctx = G->ctx;
  const int src = int((r - 1) & 1), dst = int(r & 1);
  for (mbx::Shard& s : G->shards) {
    mbx::PrArgs a;
    unsigned char* yold = static_cast<unsigned char*>(G->yloc[src]) + int64_t(s.li) * G->lchunk_bytes;
    unsigned char* ynew = static_cast<unsigned char*>(G->yloc[dst]) + int64_t(s.li) * G->lchunk_bytes;
    unsigned char* xnew = static_cast<unsigned char*>(G->pi[dst]) + int64_t(s.g) * G->chunk_bytes;
    a.pi_old = yold;
    a.dangling = s.dangling;
    a.dang_from = s.dang_from;
    a.yard_const = 1.0;
    a.damping = G->cfg.damping;
    a.inv_n = 1.0 / double(G->n);
    a.prev = G->yscal + (r - 1);
    a.next = reinterpret_cast<mbx::PrScalars*>(xnew + G->tail_off);
    a.xout = G->pi[dst];
    a.xmap = s.xmap;
    if (G->peer)
      for (int k = 0; k < G->world; ++k)
        if (k != G->rank0) a.xpeer[a.npeer++] = G->xpeer[dst][k];
    a.stop = G->flags;
    a.stop_iter = G->flags + 1;
    a.iter = int(r);
    a.check_stop = 0;
    mbx::launch_csr(ctx, &s.view, G->pi[src], ynew, &a, s.block_part, s.counter);
  }
  exchange_and_combine(G, dst, int(r), false);
}

// validation + the fields and buffers every mode shares
void group_init(mbx_shard_group* G, mbx_context* ctx, int64_t n_global, int world,
                const int64_t* bounds, int rank0, int nlocal, mbx_matrix* const* mats,
                const mbx_simt_config* c, const mbx_pagerank_config* cfg, bool peer) {
  G->ctx = ctx;
  G->peer = peer;
  if (world < 1 || nlocal < 1 || rank0 < 0 || rank0 + nlocal > world)
    mbx::fail(MBX_CONFIG_ERROR, "shard group: bad world/rank/nlocal");
  if (!(cfg->damping >= 0.0 && cfg->damping <= 1.0))
    mbx::fail(MBX_CONFIG_ERROR, "damping must lie in [0, 1]");
  if (!(cfg->err_tol > 0.0)) mbx::fail(MBX_CONFIG_ERROR, "err_tol must be positive");
  if (cfg->max_iters < 0) mbx::fail(MBX_CONFIG_ERROR, "iteration counts must be >= 0");
  if (bounds[0] != 0 || bounds[world] != n_global)
    mbx::fail(MBX_DIMENSION_ERROR, "row bounds must cover [0, n)");
  for (int g = 0; g < world; ++g)
    if (bounds[g + 1] < bounds[g]) mbx::fail(MBX_DIMENSION_ERROR, "row bounds must not decrease");
  G->ctx = ctx;
  G->precision = mats[0]->precision;
  G->vs = mbx::value_size(G->precision);
  G->world = world;
  G->rank0 = rank0;
  G->nlocal = nlocal;
  G->n = n_global;
  G->peer = peer;
  G->bounds.assign(bounds, bounds + world + 1);
  G->c = *c;
  G->cfg = *cfg;
  if (G->precision == MBX_F32) {
    G->cfg.damping = double(float(cfg->damping));
    G->cfg.err_tol = double(float(cfg->err_tol));
  }
  int64_t rows_max = 0;
  for (int g = 0; g < world; ++g) rows_max = std::max(rows_max, bounds[g + 1] - bounds[g]);
  G->lchunk_bytes = ((rows_max * int64_t(G->vs) + 255) / 256) * 256 + 256;
  cudaStream_t st = ctx->stream;
  for (int i = 0; i < 2; ++i) {
    if (peer) {
      G->loc[i] = dm_shared(G->lchunk_bytes * nlocal);
    } else {
      G->loc[i] = dm(ctx, G->lchunk_bytes * nlocal);
      MBX_CUDA(cudaMemsetAsync(G->loc[i], 0, G->lchunk_bytes * nlocal, st));
    }
  }
  if (cfg->reference_iters > 0) {
    for (int i = 0; i < 2; ++i) {
      G->yloc[i] = dm(ctx, G->lchunk_bytes * nlocal);
      MBX_CUDA(cudaMemsetAsync(G->yloc[i], 0, G->lchunk_bytes * nlocal, st));
    }
    G->yscal = static_cast<mbx::PrScalars*>(
        dm(ctx, (cfg->reference_iters + 1) * sizeof(mbx::PrScalars)));
  }
  G->main_base = cfg->reference_iters > 0 ? cfg->reference_iters + 3 : 2;
  G->gscal = static_cast<mbx::PrScalars*>(dm(ctx, (cfg->max_iters + 1) * sizeof(mbx::PrScalars)));
  MBX_CUDA(cudaMemsetAsync(G->gscal, 0, (cfg->max_iters + 1) * sizeof(mbx::PrScalars), st));
  G->flags = static_cast<int*>(dm(ctx, 64));
  MBX_CUDA(cudaMemsetAsync(G->flags, 0, 64, st));
}

// column flags of this process's shards (dangling = no rank sets the flag)
void local_seen(mbx_shard_group* G, mbx_matrix* const* mats, uint8_t* seen) {
  mbx_context* ctx = G->ctx;
  for (int i = 0; i < G->nlocal; ++i)
    if (mats[i]->nnz)
      mbx::seen_flags_kernel<<<unsigned(ctx->sm_count) * 8, 256, 0, ctx->stream>>>(
          mats[i]->cols, mats[i]->nnz, seen);
  ctx->launches += G->nlocal;
  MBX_CUDA(cudaGetLastError());
}

// compacted exchange layout from the GLOBAL column flags, then every local
// shard's remapped view, TILE geometry and PageRank workspaces.  chunk_fixed
// > 0 (peer mode): the chunk stride was fixed before the flags were known.
void group_layout(mbx_shard_group* G, mbx_matrix* const* mats, mbx_tile* const* tiles,
                  const uint8_t* seen, int64_t chunk_fixed) {
  mbx_context* ctx = G->ctx;
  cudaStream_t st = ctx->stream;
  const int world = G->world;
  const int64_t n_global = G->n;
  const mbx_simt_config* c = &G->c;
  int64_t* dbounds = static_cast<int64_t*>(dm(ctx, (world + 1) * 8));
  MBX_CUDA(cudaMemcpyAsync(dbounds, G->bounds.data(), (world + 1) * 8, cudaMemcpyHostToDevice, st));
  // gpre = exclusive scan of the global flags
  int64_t* gpre = static_cast<int64_t*>(dm(ctx, (n_global + 1) * 8));
  {
    int64_t* cnt = static_cast<int64_t*>(dm(ctx, (n_global + 1) * 8));
    MBX_CUDA(cudaMemsetAsync(cnt, 0, (n_global + 1) * 8, st));
    mbx::seen_to_count_kernel<<<unsigned(ctx->sm_count) * 8, 256, 0, st>>>(seen, n_global, cnt);
    size_t tb = 0;
    MBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, gpre, n_global + 1, st));
    void* tmp = dm(ctx, tb);
    MBX_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, gpre, n_global + 1, st));
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(cnt, st);
    ctx->launches += 2;
  }
  if (chunk_fixed > 0) {
    G->chunk_bytes = chunk_fixed;
    G->tail_off = chunk_fixed - 256;
  } else {
    // chunk = the largest per-rank non-dangling count (+ the scalar tail)
    std::vector<int64_t> gb(world + 1);
    for (int g = 0; g <= world; ++g)
      MBX_CUDA(cudaMemcpyAsync(&gb[g], gpre + G->bounds[g], 8, cudaMemcpyDeviceToHost, st));
    MBX_CUDA(cudaStreamSynchronize(st));
    int64_t nd_max = 0;
    for (int g = 0; g < world; ++g) nd_max = std::max(nd_max, gb[g + 1] - gb[g]);
    G->tail_off = ((nd_max * int64_t(G->vs) + 255) / 256) * 256;
    G->chunk_bytes = G->tail_off + 256;
  }
  G->chunk_elems = G->chunk_bytes / int64_t(G->vs);
  if (G->chunk_elems * world >= (int64_t(1) << 31))
    mbx::fail(MBX_CAPACITY_ERROR, "exchange layout exceeds int32 column indices");
  if (!G->peer) {
    for (int i = 0; i < 2; ++i) {
      G->pi[i] = dm(ctx, G->chunk_bytes * world);
      MBX_CUDA(cudaMemsetAsync(G->pi[i], 0, G->chunk_bytes * world, st));
    }
  }
  for (int i = 0; i < G->nlocal; ++i) {
    mbx_matrix* m = mats[i];
    const int g = G->rank0 + i;
    if (m->n_rows != G->bounds[g + 1] - G->bounds[g] || m->n_cols != n_global)
      mbx::fail(MBX_DIMENSION_ERROR, "shard matrix shape does not match its row bounds");
    if (tiles[i]->info.n_rows != m->n_rows || tiles[i]->info.nnz != m->nnz ||
        tiles[i]->info.omega != c->omega || tiles[i]->info.sigma != c->sigma)
      mbx::fail(MBX_CONFIG_ERROR, "shard TILE does not match its matrix / config");
    mbx::Shard s;
    s.g = g;
    s.li = i;
    s.r0 = G->bounds[g];
    s.r1 = G->bounds[g + 1];
    s.tile = tiles[i];
    s.cols_remap = static_cast<int32_t*>(dm(ctx, m->nnz * 4 + 256));
    MBX_CUDA(cudaMemsetAsync(s.cols_remap, 0, m->nnz * 4 + 256, st));
    if (m->nnz)
      mbx::remap_cols_kernel<<<unsigned(ctx->sm_count) * 8, 256, 0, st>>>(
          m->cols, m->nnz, dbounds, world, G->chunk_elems, gpre, s.cols_remap);
    s.view = *m;
    s.view.slots = mbx_matrix::SlotCache{};  // the view builds its own
    s.view.coo_rows = nullptr;
    s.view.vmap = nullptr;
    s.view.cols = s.cols_remap;
    s.view.cols_hub = nullptr;
    s.view.hub_cols = nullptr;
    s.view.hub_avail = 0;
    s.view.n_cols = G->chunk_elems * world;
    // x hub cache over the remapped columns (owned by the group)
    mbx::build_xcache(ctx, &s.view, ctx->tuning.max_hubs);
    const int64_t rows = s.r1 - s.r0;
    s.xmap = static_cast<int32_t*>(dm(ctx, rows * 4 + 64));
    if (rows)
      mbx::xmap_kernel<<<unsigned(ctx->sm_count) * 4, 256, 0, st>>>(
          seen, s.r0, rows, dbounds, world, G->chunk_elems, gpre, s.xmap);
    s.dangling = static_cast<uint32_t*>(dm(ctx, ((rows + 31) / 32) * 4 + 64));
    mbx::local_dangling_kernel<<<unsigned((rows + 31) / 32 / 256 + 1), 256, 0, st>>>(
        seen, s.r0, rows, s.dangling);
    s.dang_from = mbx::dangling_suffix_start(ctx, s.dangling, rows);
    s.geo = mbx::make_geometry(ctx, &s.view, s.tile, c->block_size);
    s.carry_mask = static_cast<uint32_t*>(dm(ctx, ((rows + 31) / 32) * 4 + 64));
    MBX_CUDA(cudaMemsetAsync(s.carry_mask, 0, ((rows + 31) / 32) * 4 + 64, st));
    // K3 blocks, or the pr_init grid (sm_count * 4) when a start vector is given
    const int64_t nblk = std::max<int64_t>({mbx::fixup_blocks(s.geo, true) + 1, mbx::fixup_blocks(s.geo, false) + 1, ctx->sm_count * 4 + 1,
                                            int64_t(mbx::csr_pr_blocks(ctx, &s.view))});
    s.block_part = static_cast<double*>(dm(ctx, nblk * 4 * sizeof(double)));
    s.counter = static_cast<unsigned int*>(dm(ctx, 64));
    MBX_CUDA(cudaMemsetAsync(s.counter, 0, 64, st));
    s.carry_ws = dm(ctx, mbx::spmv_workspace_bytes(s.geo, G->precision, true));
    ctx->launches += 2;
    G->shards.push_back(s);
  }
  MBX_CUDA(cudaGetLastError());
  MBX_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(dbounds, st);
  cudaFreeAsync(gpre, st);
  MBX_CUDA(cudaStreamSynchronize(st));
}

// The power loop as one CUDA graph.  Virtual and fused groups: a
// device-driven WHILE node (body = an odd and an even iteration + the
// condition; the combine advances the iteration counter), so an early stop
// launches nothing more and any max_iters fits.  NCCL groups: the unrolled
// fixed-count loop (the collective is not placed inside a conditional body).
void group_capture(mbx_shard_group* G) {
  mbx_context* ctx = G->ctx;
  cudaStream_t st = ctx->stream;
  MBX_CUDA(cudaEventCreate(&G->e0));
  MBX_CUDA(cudaEventCreate(&G->e1));
  const mbx::GraphMode gmode = mbx::graph_mode();
  if (gmode == mbx::GraphMode::eager) return;
  if (!G->comm && G->cfg.max_iters > 0 && gmode == mbx::GraphMode::device_loop) {
    G->iter_dev = static_cast<int64_t*>(dm(ctx, 64));
    MBX_CUDA(cudaMemsetAsync(G->iter_dev, 0, 64, st));
    MBX_CUDA(cudaStreamSynchronize(st));
    cudaGraph_t graph;
    MBX_CUDA(cudaGraphCreate(&graph, 0));
    try {
      cudaGraphConditionalHandle h;
      MBX_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      MBX_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      const int64_t before = ctx->launches;
      MBX_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal));
      try {
        launch_iteration(G, 1, true);
        launch_iteration(G, 2, true);
        mbx::shard_loop_cond_kernel<<<1, 1, 0, st>>>(h, G->iter_dev, G->cfg.max_iters, G->flags);
        ++ctx->launches;
        MBX_CUDA(cudaGetLastError());
      } catch (...) {
        cudaGraph_t dummy;
        cudaStreamEndCapture(st, &dummy);
        throw;
      }
      MBX_CUDA(cudaStreamEndCapture(st, &body));
      const int64_t per_body = ctx->launches - before;
      ctx->launches = before;
      MBX_CUDA(cudaGraphInstantiate(&G->graph, graph, 0));
      G->graph_launches = per_body * ((G->cfg.max_iters + 1) / 2);
    } catch (...) {
      cudaGraphDestroy(graph);
      throw;
    }
    cudaGraphDestroy(graph);
  } else if (G->cfg.max_iters > 0 && G->cfg.max_iters <= 4096) {
    MBX_CUDA(cudaStreamSynchronize(st));
    const int64_t before = ctx->launches;
    cudaGraph_t graph;
    MBX_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      for (int64_t r = 1; r <= G->cfg.max_iters; ++r) launch_iteration(G, r);
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      throw;
    }
    MBX_CUDA(cudaStreamEndCapture(st, &graph));
    MBX_CUDA(cudaGraphInstantiate(&G->graph, graph, 0));
    cudaGraphDestroy(graph);
    G->graph_launches = ctx->launches - before;
    ctx->launches = before;
  }
}

// Blob one rank publishes for the others (mbx_shard_group_export)
constexpr uint32_t kBlobMagic = 0x4d425850u;  // "MBXP"
struct PeerBlob {
  uint32_t magic;
  int32_t rank, world, pid, device;
  int32_t pad;
  uint64_t ptr[6];  // pi0, pi1, loc0, loc1, seen, pflags (same-process peers)
  cudaIpcMemHandle_t h[6];
};
static_assert(sizeof(PeerBlob) <= MBX_SHARD_BLOB_BYTES, "blob size");

void group_free(mbx_shard_group* G) {
  if (!G->ctx) return;  // failed before any allocation
  cudaStream_t st = G->ctx->stream;
  if (G->graph) cudaGraphExecDestroy(G->graph);
  for (mbx::Shard& s : G->shards) {
    mbx::free_slots(G->ctx, &s.view);
    for (void* p : {static_cast<void*>(s.cols_remap), static_cast<void*>(s.dangling),
                    static_cast<void*>(s.xmap),
                    static_cast<void*>(s.view.cols_hub), static_cast<void*>(s.view.hub_cols),
                    static_cast<void*>(s.carry_mask), static_cast<void*>(s.block_part),
                    static_cast<void*>(s.counter), s.carry_ws})
      if (p) cudaFreeAsync(p, st);
  }
  for (void* p : {G->yloc[0], G->yloc[1], static_cast<void*>(G->yscal),
                  static_cast<void*>(G->iter_dev)})
    if (p) cudaFreeAsync(p, st);
  for (void* p : {static_cast<void*>(G->gscal), static_cast<void*>(G->flags),
                  static_cast<void*>(G->run_base), static_cast<void*>(G->perr)})
    if (p) cudaFreeAsync(p, st);
  if (G->e0) cudaEventDestroy(G->e0);
  if (G->e1) cudaEventDestroy(G->e1);
  cudaStreamSynchronize(st);
  if (G->peer) {
    for (void* p : G->opened) cudaIpcCloseMemHandle(p);
    for (void* p : {G->pi[0], G->pi[1], G->loc[0], G->loc[1], static_cast<void*>(G->seen),
                    static_cast<void*>(G->pflags)})
      if (p) cudaFree(p);
  } else {
    for (void* p : {G->pi[0], G->pi[1], G->loc[0], G->loc[1]})
      if (p) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
  if (G->comm) mbx::nccl().CommDestroy(G->comm);
}

// owns a group under construction: a failed create releases what it got
struct GroupDeleter {
  void operator()(mbx_shard_group* G) const {
    group_free(G);
    delete G;
  }
};
using GroupPtr = std::unique_ptr<mbx_shard_group, GroupDeleter>;

// pi_0 = 1/n on the shard's rows (into `rows_buf`), its non-dangling entries
// into its chunk of exchange buffer 0 and its scalars into the chunk tail
void init_shard_uniform(mbx_shard_group* G, const mbx::Shard& s, unsigned char* rows_buf) {
  mbx_context* ctx = G->ctx;
  cudaStream_t st = ctx->stream;
  unsigned char* x0 = static_cast<unsigned char*>(G->pi[0]) + int64_t(s.g) * G->chunk_bytes;
  auto* tail = reinterpret_cast<mbx::PrScalars*>(x0 + G->tail_off);
  const int64_t rows = s.r1 - s.r0;
  auto* cnt = reinterpret_cast<unsigned long long*>(s.counter + 8);
  MBX_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
  const unsigned grid = unsigned(ctx->sm_count) * 4;
  double val;
  if (G->precision == MBX_F32) {
    const float v = 1.0f / float(G->n);  // T(1)/static_cast<T>(n) (solvers.hpp:193)
    val = double(v);
    mbx::shard_init_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<float*>(rows_buf), rows,
                                                        v, s.dangling, cnt, s.xmap,
                                                        static_cast<float*>(G->pi[0]));
  } else {
    val = 1.0 / double(G->n);
    mbx::shard_init_kernel<double><<<grid, 256, 0, st>>>(reinterpret_cast<double*>(rows_buf),
                                                         rows, val, s.dangling, cnt, s.xmap,
                                                         static_cast<double*>(G->pi[0]));
  }
  mbx::shard_init_tail_kernel<<<1, 1, 0, st>>>(cnt, rows, val, tail);
  ctx->launches += 2;
}

// Load every kernel a run launches outside the captured graph before the
// first run: under lazy module loading a first launch waits for the running
// kernels of the context, and with several ranks of a fused group in one
// process that includes a peer barrier spinning until the next rank's run is
// issued -- from this very thread.
void preload_run_kernels(mbx_shard_group* G) {
  cudaFuncAttributes a;
  MBX_CUDA(cudaFuncGetAttributes(&a, mbx::peer_barrier_kernel));
  MBX_CUDA(cudaFuncGetAttributes(&a, mbx::barrier_combine_kernel));
  MBX_CUDA(cudaFuncGetAttributes(&a, mbx::combine_kernel));
  MBX_CUDA(cudaFuncGetAttributes(&a, mbx::bump_epoch_kernel));
  MBX_CUDA(cudaFuncGetAttributes(&a, mbx::shard_init_tail_kernel));
  if (G->precision == MBX_F32) {
    MBX_CUDA(cudaFuncGetAttributes(&a, mbx::shard_init_kernel<float>));
    MBX_CUDA(cudaFuncGetAttributes(&a, mbx::scatter_exchange_kernel<float>));
  } else {
    MBX_CUDA(cudaFuncGetAttributes(&a, mbx::shard_init_kernel<double>));
    MBX_CUDA(cudaFuncGetAttributes(&a, mbx::scatter_exchange_kernel<double>));
  }
  mbx::preload_pr_kernels(G->precision);
}

// peer groups: this shard's start chunk (values + tail) out to every peer
void push_start_chunk(mbx_shard_group* G, const mbx::Shard& s) {
  if (!G->peer) return;
  const unsigned char* x0 = static_cast<unsigned char*>(G->pi[0]) + int64_t(s.g) * G->chunk_bytes;
  for (int k = 0; k < G->world; ++k)
    if (k != G->rank0)
      MBX_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(G->xpeer[0][k]) +
                                   int64_t(s.g) * G->chunk_bytes,
                               x0, G->chunk_bytes, cudaMemcpyDeviceToDevice, G->ctx->stream));
}

}  // namespace

extern "C" {

MBX_API int mbx_nccl_unique_id(void* id128) {
  return sguard([&] {
    ncclUniqueId id;
    MBX_NCCL(mbx::nccl().GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id128, &id, sizeof(id));
  });
}

MBX_API int mbx_matrix_row_slice(mbx_context* ctx, const mbx_matrix* m, int64_t r0, int64_t r1,
                                 mbx_matrix** out) {
  return sguard([&] {
    mbx::DeviceGuard dg(ctx->device);
    mbx::ensure_csr(ctx, m);
    if (r0 < 0 || r1 < r0 || r1 > m->n_rows) mbx::fail(MBX_DIMENSION_ERROR, "row slice out of range");
    uint32_t b[2];
    MBX_CUDA(cudaMemcpyAsync(&b[0], m->ro + r0, 4, cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaMemcpyAsync(&b[1], m->ro + r1, 4, cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    auto s = std::make_unique<mbx_matrix>();
    s->ctx = ctx;
    s->precision = m->precision;
    s->n_rows = r1 - r0;
    s->n_cols = m->n_cols;
    s->nnz = int64_t(b[1]) - int64_t(b[0]);
    const size_t vs = mbx::value_size(m->precision);
    s->vals = dm(ctx, s->nnz * vs + 256);
    s->cols = static_cast<int32_t*>(dm(ctx, s->nnz * 4 + 256));
    s->ro = static_cast<uint32_t*>(dm(ctx, (s->n_rows + 1) * 4 + 64));
    MBX_CUDA(cudaMemsetAsync(s->vals, 0, s->nnz * vs + 256, ctx->stream));
    MBX_CUDA(cudaMemsetAsync(s->cols, 0, s->nnz * 4 + 256, ctx->stream));
    if (s->nnz) {
      MBX_CUDA(cudaMemcpyAsync(s->vals, static_cast<char*>(m->vals) + int64_t(b[0]) * vs,
                               s->nnz * vs, cudaMemcpyDeviceToDevice, ctx->stream));
      MBX_CUDA(cudaMemcpyAsync(s->cols, m->cols + b[0], s->nnz * 4, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    }
    mbx::slice_rows_kernel<<<unsigned(ctx->sm_count) * 4, 256, 0, ctx->stream>>>(m->ro, r0, s->n_rows,
                                                                                 s->ro);
    ++ctx->launches;
    MBX_CUDA(cudaGetLastError());
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = s.release();
  });
}


MBX_API int mbx_shard_group_create(mbx_context* ctx, int64_t n_global, int world,
                                   const int64_t* bounds, int rank0, int nlocal,
                                   mbx_matrix* const* mats, mbx_tile* const* tiles,
                                   const mbx_simt_config* c, const mbx_pagerank_config* cfg,
                                   const void* nccl_id, mbx_shard_group** out) {
  return sguard([&] {
    mbx::DeviceGuard dg(ctx->device);
    for (int i = 0; i < nlocal; ++i) mbx::ensure_csr(ctx, mats[i]);
    if (!nccl_id && nlocal != world)
      mbx::fail(MBX_CONFIG_ERROR, "shard group: without NCCL every shard must be local");
    if (nccl_id && nlocal != 1)
      mbx::fail(MBX_CONFIG_ERROR, "shard group: with NCCL each process holds exactly one shard");
    GroupPtr G(new mbx_shard_group_s);
    group_init(G.get(), ctx, n_global, world, bounds, rank0, nlocal, mats, c, cfg, false);
    cudaStream_t st = ctx->stream;
    // dangling vertices = empty columns of the GLOBAL P
    uint8_t* seen = static_cast<uint8_t*>(dm(ctx, n_global + 64));
    MBX_CUDA(cudaMemsetAsync(seen, 0, n_global + 64, st));
    local_seen(G.get(), mats, seen);
    if (nccl_id) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      MBX_CUDA(cudaStreamSynchronize(st));
      MBX_NCCL(mbx::nccl().CommInitRank(&G->comm, world, id, rank0));
      MBX_NCCL(mbx::nccl().AllReduce(seen, seen, n_global, ncclUint8, ncclMax, G->comm, st));
    }
    group_layout(G.get(), mats, tiles, seen, 0);
    cudaFreeAsync(seen, st);
    group_capture(G.get());
    *out = G.release();
  });
}

MBX_API int mbx_shard_group_create_peer(mbx_context* ctx, int64_t n_global, int world,
                                        const int64_t* bounds, int rank, mbx_matrix* local,
                                        mbx_tile* tile, const mbx_simt_config* c,
                                        const mbx_pagerank_config* cfg, mbx_shard_group** out) {
  return sguard([&] {
    mbx::DeviceGuard dg(ctx->device);
    mbx::ensure_csr(ctx, local);
    if (world < 1 || world > 8)
      mbx::fail(MBX_CONFIG_ERROR, "peer shard group: world must be in [1, 8]");
    GroupPtr G(new mbx_shard_group_s);
    mbx_matrix* const mats[1] = {local};
    group_init(G.get(), ctx, n_global, world, bounds, rank, 1, mats, c, cfg, true);
    G->pmat = local;
    G->ptile = tile;
    // the exchange stride is fixed before the global flags are known: every
    // row of the largest shard could be non-dangling (+ the scalar tail)
    int64_t rows_max = 0;
    for (int g = 0; g < world; ++g) rows_max = std::max(rows_max, bounds[g + 1] - bounds[g]);
    G->chunk_bytes = ((rows_max * int64_t(G->vs) + 255) / 256) * 256 + 256;
    if (G->chunk_bytes / int64_t(G->vs) * world >= (int64_t(1) << 31))
      mbx::fail(MBX_CAPACITY_ERROR, "exchange layout exceeds int32 column indices");
    for (int i = 0; i < 2; ++i) G->pi[i] = dm_shared(G->chunk_bytes * world);
    G->seen = static_cast<uint8_t*>(dm_shared(n_global + 64));
    G->pflags = static_cast<uint64_t*>(dm_shared(8 * 8));
    G->run_base = static_cast<uint64_t*>(dm(ctx, 64));
    G->perr = static_cast<int*>(dm(ctx, 64));
    MBX_CUDA(cudaMemsetAsync(G->run_base, 0, 64, ctx->stream));
    MBX_CUDA(cudaMemsetAsync(G->perr, 0, 64, ctx->stream));
    // entry, yardstick 0..R, power iterations 0..max, the final barrier
    G->epoch_step = G->main_base + G->cfg.max_iters + 2;
    local_seen(G.get(), mats, G->seen);
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = G.release();
  });
}

MBX_API int mbx_shard_group_export(mbx_shard_group* G, void* blob) {
  return sguard([&] {
    mbx::DeviceGuard dg(G->ctx->device);
    if (!G->peer) mbx::fail(MBX_CONFIG_ERROR, "export: not a peer shard group");
    PeerBlob b;
    std::memset(&b, 0, sizeof(b));
    b.magic = kBlobMagic;
    b.rank = G->rank0;
    b.world = G->world;
    b.pid = int32_t(getpid());
    b.device = G->ctx->device;
    void* bufs[6] = {G->pi[0], G->pi[1], G->loc[0], G->loc[1], G->seen, G->pflags};
    for (int i = 0; i < 6; ++i) {
      b.ptr[i] = reinterpret_cast<uint64_t>(bufs[i]);
      MBX_CUDA(cudaIpcGetMemHandle(&b.h[i], bufs[i]));
    }
    std::memset(blob, 0, MBX_SHARD_BLOB_BYTES);
    std::memcpy(blob, &b, sizeof(b));
  });
}

MBX_API int mbx_shard_group_connect(mbx_shard_group* G, const void* blobs) {
  return sguard([&] {
    mbx::DeviceGuard dg(G->ctx->device);
    if (!G->peer) mbx::fail(MBX_CONFIG_ERROR, "connect: not a peer shard group");
    if (G->connected) mbx::fail(MBX_CONFIG_ERROR, "connect: already connected");
    mbx_context* ctx = G->ctx;
    const int world = G->world;
    const int mypid = int(getpid());
    for (int k = 0; k < world; ++k) {
      PeerBlob b;
      std::memcpy(&b, static_cast<const char*>(blobs) + int64_t(k) * MBX_SHARD_BLOB_BYTES,
                  sizeof(b));
      if (b.magic != kBlobMagic || b.rank != k || b.world != world)
        mbx::fail(MBX_CONFIG_ERROR, "connect: blob " + std::to_string(k) +
                                        " is not rank " + std::to_string(k) + " of this group");
      void* p[6];
      if (k == G->rank0) {
        void* own[6] = {G->pi[0], G->pi[1], G->loc[0], G->loc[1], G->seen, G->pflags};
        std::copy(own, own + 6, p);
      } else if (b.pid == mypid) {
        // a peer group of this process: its device pointers are valid here
        if (b.device != ctx->device) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            mbx::fail(MBX_CUDA_ERROR, std::string("peer access: ") + cudaGetErrorString(e));
          cudaGetLastError();
        }
        for (int i = 0; i < 6; ++i) p[i] = reinterpret_cast<void*>(b.ptr[i]);
      } else {
        for (int i = 0; i < 6; ++i) {
          MBX_CUDA(cudaIpcOpenMemHandle(&p[i], b.h[i], cudaIpcMemLazyEnablePeerAccess));
          G->opened.push_back(p[i]);
        }
      }
      G->xpeer[0][k] = p[0];
      G->xpeer[1][k] = p[1];
      G->lpeer[0][k] = p[2];
      G->lpeer[1][k] = p[3];
      G->speer[k] = static_cast<uint8_t*>(p[4]);
      G->pf.f[k] = static_cast<uint64_t*>(p[5]);
    }
    G->pf.world = world;
    G->pf.rank = G->rank0;
    // global column flags: OR of every rank's own (all computed before the
    // caller's all-gather of the blobs)
    cudaStream_t st = ctx->stream;
    uint8_t* gseen = static_cast<uint8_t*>(dm(ctx, G->n + 64));
    mbx::SeenPtrs sp{};
    for (int k = 0; k < world; ++k) sp.p[k] = G->speer[k];
    mbx::seen_or_kernel<<<unsigned(ctx->sm_count) * 8, 256, 0, st>>>(sp, world, G->n, gseen);
    ++ctx->launches;
    MBX_CUDA(cudaGetLastError());
    mbx_matrix* const mats[1] = {G->pmat};
    mbx_tile* const tiles[1] = {G->ptile};
    group_layout(G, mats, tiles, gseen, G->chunk_bytes);
    cudaFreeAsync(gseen, st);
    group_capture(G);
    preload_run_kernels(G);
    G->connected = true;
  });
}

MBX_API int mbx_shard_group_run(mbx_shard_group* G, const void* pi0_dev) {
  return sguard([&] {
    mbx::DeviceGuard dg(G->ctx->device);
    if (G->peer && !G->connected) mbx::fail(MBX_CONFIG_ERROR, "peer shard group not connected");
    if (G->quiesced) mbx::fail(MBX_CONFIG_ERROR, "peer shard group already quiesced");
    mbx_context* ctx = G->ctx;
    cudaStream_t st = ctx->stream;
    MBX_CUDA(cudaMemsetAsync(G->flags, 0, 8, st));
    if (G->peer) {
      // a new epoch range; every rank's previous run (its combines, the
      // caller's reads of its rows) is over once all have entered this one
      mbx::bump_epoch_kernel<<<1, 1, 0, st>>>(G->run_base, uint64_t(G->epoch_step));
      ++ctx->launches;
      peer_barrier(G, 0, false);
    }
    // yardstick (reference_iters > 0, solvers.hpp:178-191): CSR power run
    // from the uniform vector through the same exchange
    const int64_t R = G->cfg.reference_iters;
    if (R > 0) {
      for (mbx::Shard& s : G->shards) {
        init_shard_uniform(G, s, static_cast<unsigned char*>(G->yloc[0]) +
                                     int64_t(s.li) * G->lchunk_bytes);
        push_start_chunk(G, s);
      }
      exchange_and_combine(G, 0, 0, false);
      for (int64_t r = 1; r <= R; ++r) launch_yard_iteration(G, r);
      // nobody overwrites exchange buffer 0 before every rank's last
      // yardstick combine has read it
      if (G->peer) peer_barrier(G, R + 2, false);
    }
    for (mbx::Shard& s : G->shards) {
      unsigned char* x0 = static_cast<unsigned char*>(G->pi[0]) + int64_t(s.g) * G->chunk_bytes;
      unsigned char* p0 = static_cast<unsigned char*>(G->loc[0]) + int64_t(s.li) * G->lchunk_bytes;
      const int64_t rows = s.r1 - s.r0;
      auto* tail = reinterpret_cast<mbx::PrScalars*>(x0 + G->tail_off);
      if (pi0_dev) {
        // caller's start vector: copy this shard's rows, reduce its dangling
        // mass and mass deterministically into the chunk tail, then its
        // non-dangling entries into the exchange chunk
        mbx::launch_pr_init(ctx, G->precision, rows,
                            static_cast<const char*>(pi0_dev) + s.r0 * int64_t(G->vs), p0,
                            s.dangling, tail, s.block_part, s.counter);
        if (rows) {
          if (G->precision == MBX_F32)
            mbx::scatter_exchange_kernel<float><<<unsigned(ctx->sm_count) * 4, 256, 0, st>>>(
                reinterpret_cast<const float*>(p0), rows, s.xmap, static_cast<float*>(G->pi[0]));
          else
            mbx::scatter_exchange_kernel<double><<<unsigned(ctx->sm_count) * 4, 256, 0, st>>>(
                reinterpret_cast<const double*>(p0), rows, s.xmap, static_cast<double*>(G->pi[0]));
          ++ctx->launches;
        }
      } else {
        init_shard_uniform(G, s, p0);
      }
      push_start_chunk(G, s);
    }
    MBX_CUDA(cudaGetLastError());
    exchange_and_combine(G, 0, 0);
    if (G->iter_dev) MBX_CUDA(cudaMemsetAsync(G->iter_dev, 0, 8, st));
    MBX_CUDA(cudaEventRecord(G->e0, st));
    if (G->graph) {
      MBX_CUDA(cudaGraphLaunch(G->graph, st));
      ctx->launches += G->graph_launches;
    } else {
      for (int64_t r = 1; r <= G->cfg.max_iters; ++r) launch_iteration(G, r);
    }
    MBX_CUDA(cudaEventRecord(G->e1, st));
    G->ran = true;
  });
}

MBX_API int mbx_shard_group_result(mbx_shard_group* G, mbx_pagerank_result* res,
                                   double* history) {
  return sguard([&] {
    mbx::DeviceGuard dg(G->ctx->device);
    if (!G->ran) mbx::fail(MBX_ERROR, "shard group has not run");
    cudaStream_t st = G->ctx->stream;
    int flags[2];
    int perr = 0;
    MBX_CUDA(cudaMemcpyAsync(flags, G->flags, 8, cudaMemcpyDeviceToHost, st));
    if (G->perr) MBX_CUDA(cudaMemcpyAsync(&perr, G->perr, 4, cudaMemcpyDeviceToHost, st));
    std::vector<mbx::PrScalars> sc(G->cfg.max_iters + 1);
    MBX_CUDA(cudaMemcpyAsync(sc.data(), G->gscal, sc.size() * sizeof(mbx::PrScalars),
                             cudaMemcpyDeviceToHost, st));
    MBX_CUDA(cudaStreamSynchronize(st));
    if (perr)
      mbx::fail(MBX_NCCL_ERROR, "peer shard group: a rank did not reach the barrier in 30 s");
    const int64_t iters = flags[0] ? flags[1] : G->cfg.max_iters;
    if (flags[0] == 2)
      mbx::fail(MBX_ERROR, "pagerank: zero-norm iterate at iteration " + std::to_string(iters));
    float ms = 0.f;
    MBX_CUDA(cudaEventElapsedTime(&ms, G->e0, G->e1));
    res->iterations = iters;
    res->status = flags[0] == 1 ? 0 : 1;
    res->final_err = iters > 0 ? sc[iters].err : 0.0;
    res->preprocess_seconds = 0.0;
    for (auto& s : G->shards) res->preprocess_seconds += s.tile->info.preprocess_seconds;
    res->iterate_seconds = ms * 1e-3;
    res->l1_residual = iters > 0 ? sc[iters].resid : 0.0;
    res->mass = sc[iters].mass;
    res->dangling_mass = sc[iters].dangling;
    if (history)
      for (int64_t r = 1; r <= G->cfg.max_iters; ++r) history[r - 1] = r <= iters ? sc[r].resid : 0.0;
  });
}

// The full pi (every rank holds all chunks after the final exchange).
MBX_API int mbx_shard_group_gather_pi(mbx_shard_group* G, void* pi_host) {
  return sguard([&] {
    mbx::DeviceGuard dg(G->ctx->device);
    cudaStream_t st = G->ctx->stream;
    int flags[2];
    MBX_CUDA(cudaMemcpyAsync(flags, G->flags, 8, cudaMemcpyDeviceToHost, st));
    MBX_CUDA(cudaStreamSynchronize(st));
    const int64_t iters = flags[0] ? flags[1] : G->cfg.max_iters;
    const int slot = int(iters & 1);
    const unsigned char* base = static_cast<const unsigned char*>(G->loc[slot]);
    // the full rows live with their owners: one all-gather of the local
    // chunks (the exchange buffers hold only the non-dangling entries), or
    // direct reads of the peers' rows (peer groups; every rank finished the
    // last iteration before this rank's final barrier)
    unsigned char* all = nullptr;
    if (G->comm) {
      all = static_cast<unsigned char*>(dm(G->ctx, G->lchunk_bytes * G->world));
      MBX_NCCL(mbx::nccl().AllGather(base, all, G->lchunk_bytes, ncclUint8, G->comm, st));
    }
    for (int g = 0; g < G->world; ++g) {
      const int64_t rows = G->bounds[g + 1] - G->bounds[g];
      const unsigned char* src =
          G->peer ? static_cast<const unsigned char*>(G->lpeer[slot][g])
                  : all ? all + int64_t(g) * G->lchunk_bytes
                        : base + int64_t(g - G->rank0) * G->lchunk_bytes;
      if (rows)
        MBX_CUDA(cudaMemcpyAsync(static_cast<char*>(pi_host) + G->bounds[g] * int64_t(G->vs), src,
                                 rows * G->vs, cudaMemcpyDefault, st));
    }
    MBX_CUDA(cudaStreamSynchronize(st));
    if (all) cudaFreeAsync(all, st);
  });
}

// This process's rows of the final pi (its shards in rank order) to host.
MBX_API int mbx_shard_group_download_local(mbx_shard_group* G, void* pi_local_host) {
  return sguard([&] {
    mbx::DeviceGuard dg(G->ctx->device);
    cudaStream_t st = G->ctx->stream;
    int flags[2];
    MBX_CUDA(cudaMemcpyAsync(flags, G->flags, 8, cudaMemcpyDeviceToHost, st));
    MBX_CUDA(cudaStreamSynchronize(st));
    const int64_t iters = flags[0] ? flags[1] : G->cfg.max_iters;
    const unsigned char* base = static_cast<const unsigned char*>(G->loc[iters & 1]);
    int64_t off = 0;
    for (const mbx::Shard& s : G->shards) {
      const int64_t rows = s.r1 - s.r0;
      if (rows)
        MBX_CUDA(cudaMemcpyAsync(static_cast<char*>(pi_local_host) + off * int64_t(G->vs),
                                 base + int64_t(s.li) * G->lchunk_bytes, rows * G->vs,
                                 cudaMemcpyDeviceToHost, st));
      off += rows;
    }
    MBX_CUDA(cudaStreamSynchronize(st));
  });
}

// Peer groups: enqueue the final barrier (asynchronous).  Its completion
// means no peer can still read or write this rank's buffers.
MBX_API int mbx_shard_group_quiesce(mbx_shard_group* G) {
  return sguard([&] {
    mbx::DeviceGuard dg(G->ctx->device);
    if (!G->peer || !G->connected || G->quiesced) return;
    MBX_CUDA(cudaMemsetAsync(G->flags, 0, 8, G->ctx->stream));  // stop must not skip it
    peer_barrier(G, G->epoch_step - 1, false);
    G->quiesced = true;
  });
}

// Collective for peer groups (quiesce, then wait for the final barrier).
MBX_API int mbx_shard_group_destroy(mbx_shard_group* G) {
  return sguard([&] {
    if (!G) return;
    mbx::DeviceGuard dg(G->ctx->device);
    if (G->peer && G->connected) {
      const int rc = mbx_shard_group_quiesce(G);
      if (rc) mbx::fail(rc, "quiesce failed");
      MBX_CUDA(cudaStreamSynchronize(G->ctx->stream));
    }
    group_free(G);
    delete G;
  });
}

}  // extern "C"
