// mbx_internal.h -- shared internals of libmerbit_b200.so (not installed).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "merbit_b200.h"

namespace mbx {

// Status carrier used inside the library; the C ABI converts it to an int
// plus the thread-local message (capi.cu).
struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void set_last_error(const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);

#define MBX_CUDA(call) ::mbx::cuda_check((call), #call, __FILE__, __LINE__)

constexpr uint32_t kLongRowMask = 0x80000000u;  // tile.hpp:38

// Kernel-side geometry of one SpMV launch.  A "chunk" is 32 consecutive
// lanes (one warp's worth, = one tile when omega == 32); a "range" is
// `chunks_per_range` consecutive chunks walked by one warp with its running
// row partial kept in registers.  Ranges are the unit whose boundary rows go
// through the carry table (the reference's per-block carries,
// merbit_spmv.hpp:119-127).
struct Geometry {
  int64_t n_rows = 0, nnz = 0, lane_num = 0, tile_num = 0;
  int64_t num_chunks = 0, num_ranges = 0;
  int omega = 32, sigma = 14, ob = 9, chunks_per_range = 4;
  int warps_per_cta = 8;
  // persistent launch: grid = sm_count * ctas_per_sm, warps stride over ranges
  int grid = 0;
  int sms = 148;  // multiprocessors of the device
  // x hub cache: the hub_count (0 or hub_avail) hub values are staged in
  // shared memory; encoded columns (sign bit) address them.
  int hub_count = 0;
  int prefetch = 0;
  // 1: K2 walks the lane-major slot copy of the matrix (slots.cu) instead of
  // staging products through shared memory
  int slots = 0;
};

// Launch tuning knobs (context-wide; see mbx_context_set_tuning).
struct Tuning {
  int warps_per_cta = 32;
  int ctas_per_sm = 1;
  // launch shape left to the library (no mbx_context_set_tuning call): small
  // matrices without a hub table take 16 warps x 2 CTAs per SM
  bool shape_auto = true;
  int max_hubs = -1;  // -1: fill the shared-memory budget; 0: disable
  // Shared memory K2 may take per SM.  The rest stays L1, which also stages
  // every in-flight miss: a hub table that squeezes L1 below ~80 KB starves
  // memory-level parallelism (measured, profiles/).
  // -1 (default): 160 KB for fp32, 128 KB for fp64 (measured at R-MAT s24:
  // fp32 PageRank 830 -> 790 us / iteration with 38.6 K instead of 30.5 K hubs;
  // fp64 slower above 128 KB, its TMA staging areas already take 33 KB)
  int smem_per_sm = -1;
  // K2 staging of the next tile: 0 none, 1 L2 prefetch of its value/column
  // lines (measured: costs request-port slots), 2 TMA bulk copy of its column
  // slots + descriptors into shared memory (slot layout; measured: fp64 -9 %,
  // fp32 +8 % at R-MAT s24), -1 auto = 2 for fp64, 0 for fp32
  int prefetch = -1;
  // K2 data layout: 1 = lane-major slots (default, omega 32 with the
  // default sigma), 0 = CSR order staged through shared memory
  int layout = 1;
};

// Rows a slot-layout warp can commit through its shared-memory row buffer;
// tiles closing more rows commit lane by lane.
constexpr int kSlotRowBuf = 64;

// Device-side reduction slots of one fused PageRank iteration.
struct PrScalars {
  double dangling;  // sum of pi over dangling vertices
  double resid;     // sum |pi_new - pi_old|
  double mass;      // sum |pi_new|
  double err;       // max |pi_new - pi*| / pi*  (inf rules of rank_error)
};

struct PrArgs {
  const void* pi_old = nullptr;        // x of this iteration
  const uint32_t* dangling = nullptr;  // bit r set <=> vertex r dangling
  // >= 0: the dangling vertices are exactly the rows >= dang_from (a degree
  // relabelled matrix puts its empty columns last), so the commit compares
  // instead of fetching bitmask words
  int64_t dang_from = -1;
  // bit r set <=> row r is a range boundary row whose final value K3's carry
  // fold writes; K2 sets the bits (every iteration, same rows), K3's
  // streaming reduction skips them (the fold accounts for them)
  uint32_t* carry_mask = nullptr;
  const void* yardstick = nullptr;     // pi*; NULL => constant yard_const
  double yard_const = 0.0;
  double damping = 0.85;
  double inv_n = 0.0;
  const PrScalars* prev = nullptr;  // scalars of pi_old (dangling mass)
  PrScalars* next = nullptr;        // scalars of pi_new (written by K3)
  double* block_part = nullptr;     // 4 doubles per K3 block
  unsigned int* done_counter = nullptr;
  int* stop = nullptr;         // set once converged / failed
  int* stop_iter = nullptr;    // iteration that set stop
  int iter = 0;                // 1-based
  double err_tol = 0.0;
  // 1: K3's last block decides convergence.  0 (row shards): the scalars are
  // partial; the combine kernel after the exchange decides.
  int check_stop = 1;
  // Row shards: pi_new of a non-dangling row is also written to its slot
  // xmap[row] (>= 0) of the compacted exchange buffer xout.
  void* xout = nullptr;
  const int32_t* xmap = nullptr;
  // Fused exchange (peer shard groups): the same store goes to the npeer
  // peers' exchange buffers (same layout as xout, mapped over NVLink with
  // CUDA IPC), and K3's scalar tail follows at the same offset.
  static constexpr int kMaxPeers = 7;
  int npeer = 0;
  void* xpeer[kMaxPeers] = {};
  // Device-driven loop (a CUDA-graph WHILE node replays one body for every
  // iteration): the iteration number is *iter_dev + 1 (iterations completed
  // so far, advanced by K3's last block), prev / next are scal_base[r-1] /
  // scal_base[r], and kernels past max_iters return at once.
  int64_t* iter_dev = nullptr;
  PrScalars* scal_base = nullptr;
  int64_t max_iters = 0;
};

}  // namespace mbx

struct mbx_context_s {
  int device = 0;
  int sm_count = 148;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  // growable scratch (carry table etc.), stream-ordered reuse
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* host_scratch = nullptr;  // pinned staging
  size_t host_scratch_bytes = 0;
  mbx::Tuning tuning;
  uint64_t tuning_epoch = 0;  // bumped by every tuning / layout change
  // mbx_pagerank keeps its last plan (pi buffers, scalars, the captured
  // power-loop graph) for the next call on the same matrix, TILE and
  // configs; dropped when either is destroyed or by mbx_context_release_cache
  struct mbx_pagerank_plan_s* pr_cache = nullptr;
  void* cusparse = nullptr;  // cusparseHandle_t of the cuSPARSE comparators (lazy)
};

namespace mbx {
struct SparseState;  // comparators.cu
}  // namespace mbx

struct mbx_matrix_s {
  mbx_context* ctx = nullptr;
  int precision = MBX_F32;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  void* vals = nullptr;        // T[nnz] (+ pad)
  int32_t* cols = nullptr;     // int32[nnz] (+ pad)
  uint32_t* ro = nullptr;      // u32[n_rows+1]
  // x hub cache (mbx_matrix_build_xcache): hub_cols lists the most
  // referenced columns in ascending column order (slot = rank); cols_hub (built only when a
  // staged / generic K2 needs it) is cols with every reference to hub slot
  // s < hub_avail rewritten as (INT32_MIN | s).
  int32_t* cols_hub = nullptr;
  int32_t* hub_cols = nullptr;
  int hub_avail = 0;
  int hub_prefix = 0;         // 1: hub_cols is 0..hub_avail-1 (degree-relabelled)
  double hub_coverage = 0.0;  // fraction of nonzeros that reference a hub
  // distinct 32-byte x sectors per 32 consecutive nonzeros, from the hub
  // selection's sample (-1: not measured); picks K2's next-tile staging
  double gather_sectors = -1.0;
  uint64_t version = 0;       // bumped whenever cols_hub is rebuilt
  // bumped whenever a device buffer a captured PageRank plan may reference
  // (slot copy, cols_hub, hub_cols) is freed or rebuilt: plans compare it
  // before every replay and re-capture on a change
  mutable uint64_t gen = 0;
  // Lane-major slot copy of (values, [hub-encoded] columns) for one TILE:
  // slot (chunk c, step i, lane l) holds the element lane l consumes at step
  // i (zero for Down steps); built once per (TILE, column encoding) and
  // reused by every SpMV / PageRank iteration (slots.cu).
  struct SlotCache {
    void* vals = nullptr;
    int32_t* cols = nullptr;
    uint64_t tile_serial = 0;
    uint64_t version = 0;
    int hub = 0;
    int64_t count = 0;
    double seconds = 0.0;  // build time (preprocessing)
  };
  mutable SlotCache slots;
  mutable int32_t* coo_rows = nullptr;  // COO row array of the coo_atomic comparator
  // cuSPARSE comparator state (comparators.cu): descriptors + work buffer
  // per algorithm, built on first use
  mutable mbx::SparseState* sparse[4] = {nullptr, nullptr, nullptr, nullptr};
  // mbx_matrix_compact: the CSR values / columns were freed; the slot copy
  // and this private copy of its TILE rebuild them on first use (ensure_csr)
  struct CompactTile {
    mbx_tile_info info{};
    int ob = 0;
    uint32_t* tile_x = nullptr;
    uint32_t* tile_y = nullptr;
    uint32_t* lane_desc = nullptr;
  };
  CompactTile* compact = nullptr;
  // dangling-column bitmask (empty columns), cached by the first PageRank plan
  mutable uint32_t* dmask = nullptr;
  // Set on a matrix made by mbx_matrix_relabel_by_degree: vertex v of the
  // original graph is vertex vmap[v] here.  Host-facing PageRank I/O
  // (pi0 in, pi / yardstick out) stays in the ORIGINAL vertex order.
  int32_t* vmap = nullptr;
};

struct mbx_tile_s {
  mbx_context* ctx = nullptr;
  mbx_tile_info info{};
  int offset_bits = 0;
  uint32_t* tile_x = nullptr;
  uint32_t* tile_y = nullptr;
  uint32_t* lane_desc = nullptr;
  uint64_t serial = 0;  // unique per TILE (slot-cache key)
};

namespace mbx {

size_t value_size(int precision);
void* scratch(mbx_context* ctx, size_t bytes);
void* host_scratch(mbx_context* ctx, size_t bytes);
Geometry make_geometry(const mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                       int block_size);
size_t spmv_smem_bytes(const Geometry& g, int precision);
// hub slots the K2 shared-memory budget leaves for a matrix with n_cols
// columns (the budget shrinks as x outgrows L2: the L1 it leaves matters more)
int max_hub_slots(const mbx_context* ctx, int warps_per_cta, int ctas_per_sm, int sigma,
                  int precision, int64_t n_cols);
// Below this many nonzeros (4096 per resident K2 warp of the tuned launch
// shape) K2 is latency-bound -- a warp walks a handful of tiles: the
// automatic x hub table is skipped (it changes nothing there, R-MAT fp32 SpMV
// with / without, scripts/prof/small_hub_probe.py: s19 34.8 / 31.6 us, s20
// 59.9 / 60.0 us, s21 103 / 114 us, s22 193 / 230 us) and K2 takes the
// small-matrix launch shape (make_geometry).
inline int64_t small_matrix_nnz(const mbx_context* ctx) {
  return int64_t(4096) * ctx->sm_count * ctx->tuning.ctas_per_sm * ctx->tuning.warps_per_cta;
}
// K2's default shared memory per SM (Tuning::smem_per_sm = -1)
int default_smem_budget(int precision, int64_t n_cols);
void build_xcache(mbx_context* ctx, mbx_matrix* m, int max_hubs);
// hub lookup words (hub_cols ascending): .x = hub bits of columns 32w..32w+31,
// .y = slot of the first of them
// The map is followed by a 2^17-bit Bloom filter of the hub columns
// (kHubBloomWords u32, hub_bloom_bit): most non-hub columns are rejected from
// shared memory without touching the map.
uint2* hub_word_map(mbx_context* ctx, const mbx_matrix* m);
constexpr int kHubBloomWords = 4096;
inline size_t hub_map_words(int64_t n_cols) { return size_t(n_cols / 32 + 1); }
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t hub_bloom_bit(int32_t c) {
  return (uint32_t(c) * 0x9E3779B1u) >> 15;  // 17 bits
}
// column c -> (INT32_MIN | slot) for a hub, c otherwise
__device__ __forceinline__ int32_t hub_word_encode(const uint2* __restrict__ map, int32_t c) {
  const uint2 e = __ldg(map + (c >> 5));
  const uint32_t b = 1u << (c & 31);
  return (e.x & b) ? int32_t(0x80000000u | (e.y + uint32_t(__popc(e.x & (b - 1u))))) : c;
}
#endif
// build m->cols_hub (hub-encoded CSR columns) if missing: staged / generic K2
void ensure_cols_hub(mbx_context* ctx, const mbx_matrix* m);
// slots.cu: make m->slots match (t, hub encoding of g); false if the slot
// layout does not apply (then K2 uses the staged CSR order)
bool ensure_slots(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t, const Geometry& g);
void free_slots(mbx_context* ctx, const mbx_matrix* m);
// compacted matrices (mbx_matrix_compact): drop the CSR values / columns,
// rebuild them from the slot copy on first use
void compact_matrix(mbx_context* ctx, mbx_matrix* m, const mbx_tile* t);
void ensure_csr(mbx_context* ctx, const mbx_matrix* m);
void free_compact_tile(mbx_context* ctx, const mbx_matrix* m);
int default_sigma(int precision);
// Tuning::prefetch with -1 (auto) resolved for a precision
int resolve_prefetch(int tuning, int precision, double gather_sectors = -1.0);

// ---- kernels (kernels.cu) ----
void launch_generate_tile(mbx_context* ctx, const uint32_t* ro, int64_t n_rows,
                          int64_t nnz, const mbx_simt_config& c, mbx_tile* t);
void launch_spmv(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                 const Geometry& g, const void* x, void* y, void* carry_ws,
                 const PrArgs* pr);
size_t spmv_workspace_bytes(const Geometry& g, int precision, bool pagerank);
// PageRank partial sums K2 hands to K3: one per warp of the persistent
// omega-32 kernels, one per range otherwise.
// K3 blocks of one SpMV / PageRank iteration (block_part slots it needs).
// K3 grid (plain SpMV / PageRank); PageRank buffers size by the larger
int64_t fixup_blocks(const Geometry& g, bool pagerank);
void launch_trace_counts(mbx_context* ctx, const mbx_tile* t,
                         unsigned long long* counters_dev);
void launch_csr(mbx_context* ctx, const mbx_matrix* m, const void* x, void* y,
                const PrArgs* pr, double* cta_part, unsigned int* counter);
int csr_pr_blocks(mbx_context* ctx, const mbx_matrix* m);
void preload_pr_kernels(int precision);
// SpmvTrace deposits of y = A x (x on the device): (row, partial) pairs via
// an atomic counter; at most `capacity` are written, *counter counts all
void launch_deposits(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t, const void* x,
                     unsigned long long* counter, int64_t capacity, int64_t* rows,
                     void* amounts);
// First row of the dangling set when it is a suffix [f, n) of the rows
// (f = n when empty), else -1: one host pass over the bitmask (preprocessing).
int64_t dangling_suffix_start(mbx_context* ctx, const uint32_t* mask_dev, int64_t n);
// comparators.cu: release the cuSPARSE state of a matrix / a context
void free_sparse_state(mbx_context* ctx, const mbx_matrix* m);
void free_sparse_handle(mbx_context* ctx);
// capi.cu's validation of a SimtConfig and of a TILE against (matrix, config)
void validate_config(const mbx_simt_config* c);
void validate_tile(const mbx_matrix* m, const mbx_tile* t, const mbx_simt_config* c);
// Makes ctx->device current for the scope of a C-ABI call (the caller's
// thread may have another device current) and restores the previous one.
struct DeviceGuard {
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = dev;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
  int prev = 0;
};

// How iterative loops are replayed: one graph with a device-driven WHILE node
// (default), the fixed-count loop captured unrolled, or host launches
// (MBX_GRAPH_MODE = while | unrolled | eager; profilers do not descend into
// conditional graph nodes).
enum class GraphMode { device_loop, unrolled, eager };
inline GraphMode graph_mode() {
  const char* e = std::getenv("MBX_GRAPH_MODE");
  if (e && std::string(e) == "unrolled") return GraphMode::unrolled;
  if (e && std::string(e) == "eager") return GraphMode::eager;
  return GraphMode::device_loop;
}
// cnt[c] += #{k : cols[k] == c} (cnt zeroed by the caller); hot low columns
// are counted in shared memory first
void launch_count_columns(mbx_context* ctx, const int32_t* cols, int64_t nnz, int64_t ncols,
                          uint32_t* cnt);
// the WHILE node's condition kernel of the device-driven PageRank loop
void launch_pr_loop_cond(mbx_context* ctx, cudaGraphConditionalHandle h, const int64_t* iter_dev,
                         int64_t max_iters, const int* stop);
void launch_pr_init(mbx_context* ctx, int precision, int64_t n,
                    const void* pi0, void* pi, const uint32_t* dangling,
                    PrScalars* out, double* block_part, unsigned int* counter);
void launch_dangling_mask(mbx_context* ctx, const mbx_matrix* m,
                          uint32_t* mask_words);
// dst[map[v]] = src[v] (to_new) or dst[v] = src[map[v]] (back), T = precision
void launch_vertex_map(mbx_context* ctx, int precision, int64_t n, const int32_t* map,
                       const void* src, void* dst, bool to_new);
void launch_narrow_cols(mbx_context* ctx, const int64_t* src, int32_t* dst,
                        int64_t n, int64_t limit, int* bad_flag);
void launch_narrow_rows(mbx_context* ctx, const int64_t* src, uint32_t* dst,
                        int64_t n, int* bad_flag);

// ---- generators (generators.cu) ----
void generate_rmat(mbx_context* ctx, int precision, int scale,
                   int edge_factor, uint64_t seed, int kind,
                   uint64_t value_seed, double lo, double hi, mbx_matrix* m);
void generate_stencil27(mbx_context* ctx, int precision, int64_t g, mbx_matrix* m);
void generate_powerlaw(mbx_context* ctx, int precision, int log2n, uint64_t seed,
                       mbx_matrix* m);

}  // namespace mbx
