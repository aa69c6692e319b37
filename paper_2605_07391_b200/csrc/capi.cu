// capi.cu -- the extern "C" boundary (include/merbit_b200.h): handles,
// device memory, host<->device staging, error translation, the PageRank
// plan with its CUDA graph.  No CPU compute path exists: every SpMV /
// TILE / PageRank result comes from the kernels in kernels.cu.
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "mbx_internal.h"

namespace {
thread_local std::string g_last_error;
}

namespace mbx {

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void set_last_error(const std::string& msg) { g_last_error = msg; }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e),
                  cudaGetErrorString(e), file, line, what);
    throw Error{MBX_CUDA_ERROR, buf};
  }
}

size_t value_size(int precision) { return precision == MBX_F64 ? 8 : 4; }

void* scratch(mbx_context* ctx, size_t bytes) {
  if (bytes > ctx->scratch_bytes) {
    if (ctx->scratch) MBX_CUDA(cudaFreeAsync(ctx->scratch, ctx->stream));
    const size_t b = std::max<size_t>(bytes, 1 << 20);
    MBX_CUDA(cudaMallocAsync(&ctx->scratch, b, ctx->stream));
    ctx->scratch_bytes = b;
  }
  return ctx->scratch;
}

Geometry make_geometry(const mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                       int block_size) {
  Geometry g;
  g.n_rows = t->info.n_rows;
  g.nnz = t->info.nnz;
  g.lane_num = t->info.lane_num;
  g.tile_num = t->info.tile_num;
  g.omega = t->info.omega;
  g.sigma = t->info.sigma;
  g.ob = t->offset_bits;
  g.num_chunks = (g.lane_num + 31) / 32;
  g.warps_per_cta = ctx->tuning.warps_per_cta;
  g.grid = ctx->sm_count * ctx->tuning.ctas_per_sm;
  g.sms = ctx->sm_count;
  const bool small = ctx->tuning.shape_auto && !(m->hub_cols && m->hub_avail > 0) &&
                     m->nnz < small_matrix_nnz(ctx);
  if (small) {
    // a small matrix without a hub table is latency-bound (a warp walks ~8
    // tiles): two CTAs of 16 warps per SM retire their tails independently
    // (scripts/prof/c1_shape.py, R-MAT s20 fp32: 58.4 -> 56.9 us)
    g.warps_per_cta = 16;
    g.grid = ctx->sm_count * 2;
  }
  // b/32 tiles per warp range (the reference's block of b/omega tiles), but
  // at least ~8 ranges per resident warp so small matrices do not leave the
  // persistent grid with a long tail
  const int64_t warps = int64_t(g.grid) * g.warps_per_cta;
  const int64_t fit = std::max<int64_t>(1, g.num_chunks / (8 * warps));
  g.chunks_per_range = int(std::max<int64_t>(1, std::min<int64_t>({31, block_size / 32, fit})));
  g.num_ranges = (g.num_chunks + g.chunks_per_range - 1) / g.chunks_per_range;
  g.prefetch = resolve_prefetch(ctx->tuning.prefetch, m->precision, m->gather_sectors);
  // ... and without the fp64 TMA staging, whose round trip per tile only
  // pays on a request-bound matrix (R-MAT s20 fp64: 74.7 us with it, 72.4 us
  // at 16 x 2 without)
  if (small && ctx->tuning.prefetch < 0 && g.prefetch == 2) g.prefetch = 0;
  g.hub_count = 0;
  if (m->hub_cols && m->hub_avail > 0 && g.omega == 32 && ctx->tuning.max_hubs != 0 &&
      (ctx->tuning.max_hubs < 0 || ctx->tuning.max_hubs >= m->hub_avail)) {
    const int slots = max_hub_slots(ctx, g.warps_per_cta, ctx->tuning.ctas_per_sm, g.sigma,
                                    m->precision, m->n_cols);
    if (slots >= m->hub_avail) g.hub_count = m->hub_avail;
  }
  // lane-major slot copy for this TILE (built once, outside any capture)
  g.slots = ensure_slots(const_cast<mbx_context*>(ctx), m, t, g) ? 1 : 0;

  if (!g.slots && g.hub_count > 0) {
    // the staged kernel needs more shared memory per warp than the slot one
    const bool slot_budget = ctx->tuning.layout == 1 && g.sigma == default_sigma(m->precision);
    if (slot_budget) g.hub_count = 0;
  }
  if (!g.slots) ensure_csr(const_cast<mbx_context*>(ctx), m);  // staged / generic K2 read CSR
  if (!g.slots && g.hub_count > 0) ensure_cols_hub(const_cast<mbx_context*>(ctx), m);
  return g;
}

}  // namespace mbx

using mbx::fail;

namespace {
void drop_pr_cache(mbx_context* ctx);
bool pr_cache_refs(const mbx_context* ctx, const void* obj);
}  // namespace

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return MBX_OK;
  } catch (const mbx::Error& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return MBX_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MBX_ERROR;
  }
}

void require(bool ok, int code, const std::string& msg) {
  if (!ok) fail(code, msg);
}

void check_precision(int p) {
  require(p == MBX_F32 || p == MBX_F64, MBX_CONFIG_ERROR, "precision must be MBX_F32 or MBX_F64");
}

struct Device {
  explicit Device(int dev) {
    MBX_CUDA(cudaGetDevice(&prev));
    if (prev != dev) MBX_CUDA(cudaSetDevice(dev));
  }
  ~Device() {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  int prev = 0;
};

void* dmalloc(mbx_context* ctx, size_t bytes) {
  void* p = nullptr;
  MBX_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 256), ctx->stream));
  return p;
}
void dfree(mbx_context* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

int config_offset_bits(int omega, int sigma, int block) {
  if (omega < 1) fail(MBX_CONFIG_ERROR, "omega must be >= 1");
  if (sigma < 1) fail(MBX_CONFIG_ERROR, "sigma must be >= 1");
  if (block < omega)
    fail(MBX_CONFIG_ERROR, "block_size " + std::to_string(block) + " smaller than omega " +
                               std::to_string(omega));
  if (block % omega != 0)
    fail(MBX_CONFIG_ERROR, "block_size " + std::to_string(block) + " not a multiple of omega " +
                               std::to_string(omega));
  int ob = 0;
  while ((int64_t(1) << ob) < int64_t(omega) * sigma) ++ob;
  const int bits = 2 * ob + sigma;
  if (bits > 32)
    fail(MBX_CONFIG_ERROR, "infeasible descriptor layout: 2*ceil_log2(omega*sigma) + sigma = 2*" +
                               std::to_string(ob) + " + " + std::to_string(sigma) + " = " +
                               std::to_string(bits) + " exceeds 32");
  return ob;
}

void check_config(const mbx_simt_config* c) {
  require(c != nullptr, MBX_CONFIG_ERROR, "null config");
  const int ob = config_offset_bits(c->omega, c->sigma, c->block_size);
  require(ob == c->offset_bits, MBX_CONFIG_ERROR, "offset_bits inconsistent with omega*sigma");
}

void check_tile_matches(const mbx_matrix* m, const mbx_tile* t, const mbx_simt_config* c) {
  if (t->info.omega != c->omega || t->info.sigma != c->sigma)
    fail(MBX_CONFIG_ERROR, "tile metadata built for omega=" + std::to_string(t->info.omega) +
                               " sigma=" + std::to_string(t->info.sigma) +
                               ", run requested omega=" + std::to_string(c->omega) +
                               " sigma=" + std::to_string(c->sigma));
  if (t->info.n_rows != m->n_rows || t->info.nnz != m->nnz)
    fail(MBX_CONFIG_ERROR, "tile metadata shape (" + std::to_string(t->info.n_rows) + " rows, " +
                               std::to_string(t->info.nnz) +
                               " nnz) does not match the matrix");
}

void tile_counts(int64_t nnz, int64_t n, int omega, int sigma, int64_t* tn, int64_t* ln) {
  const int64_t total = nnz + n;
  const int64_t span = int64_t(omega) * sigma;
  *ln = total == 0 ? 0 : (total + sigma - 1) / sigma;
  *tn = total == 0 ? 0 : (total + span - 1) / span;
}

mbx_tile* new_tile(mbx_context* ctx, const mbx_simt_config& c, int64_t n_rows, int64_t nnz) {
  static std::atomic<uint64_t> next_serial{1};
  auto t = std::make_unique<mbx_tile>();
  t->ctx = ctx;
  t->serial = next_serial++;
  t->info.omega = c.omega;
  t->info.sigma = c.sigma;
  t->info.n_rows = n_rows;
  t->info.nnz = nnz;
  tile_counts(nnz, n_rows, c.omega, c.sigma, &t->info.tile_num, &t->info.lane_num);
  t->offset_bits = c.offset_bits;
  t->tile_x = static_cast<uint32_t*>(dmalloc(ctx, (t->info.tile_num + 1) * 4 + 64));
  t->tile_y = static_cast<uint32_t*>(dmalloc(ctx, (t->info.tile_num + 1) * 4 + 64));
  t->lane_desc = static_cast<uint32_t*>(dmalloc(ctx, t->info.lane_num * 4 + 256));
  return t.release();
}

void tile_capacity(int64_t n_rows, int64_t nnz) {
  if (n_rows >= (int64_t(1) << 31))
    fail(MBX_CAPACITY_ERROR, "row count " + std::to_string(n_rows) +
                                 " collides with the long-row mark bit (limit 2^31)");
  if (nnz > int64_t(0xFFFFFFFF))
    fail(MBX_CAPACITY_ERROR,
         "nonzero count " + std::to_string(nnz) + " exceeds the 32-bit tile cursor");
}

void generate_tile_timed(mbx_context* ctx, const uint32_t* ro_dev, int64_t n_rows, int64_t nnz,
                         const mbx_simt_config& c, mbx_tile* t) {
  cudaEvent_t e0, e1;
  MBX_CUDA(cudaEventCreate(&e0));
  MBX_CUDA(cudaEventCreate(&e1));
  MBX_CUDA(cudaEventRecord(e0, ctx->stream));
  mbx::launch_generate_tile(ctx, ro_dev, n_rows, nnz, c, t);
  MBX_CUDA(cudaEventRecord(e1, ctx->stream));
  MBX_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  MBX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  t->info.preprocess_seconds = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

// ---- matrix upload ---------------------------------------------------------
mbx_matrix* upload_common(mbx_context* ctx, int precision, int64_t n_rows, int64_t n_cols,
                          const int64_t* ro, const void* cols, bool cols64,
                          const void* vals) {
  check_precision(precision);
  require(n_rows >= 0 && n_cols >= 0, MBX_DIMENSION_ERROR, "negative matrix dimensions");
  require(n_cols < (int64_t(1) << 31), MBX_CAPACITY_ERROR,
          "n_cols must be < 2^31 (int32 device column indices)");
  require(ro != nullptr, MBX_DIMENSION_ERROR, "null row_offsets");
  const int64_t nnz = ro[n_rows];
  require(ro[0] == 0 && nnz >= 0, MBX_DIMENSION_ERROR, "row_offsets must start at 0");
  require(nnz <= int64_t(0xFFFFFFFF), MBX_CAPACITY_ERROR,
          "nonzero count " + std::to_string(nnz) + " exceeds the 32-bit tile cursor");
  require(nnz == 0 || (cols && vals), MBX_DIMENSION_ERROR, "null column or value array");
  Device dg(ctx->device);
  auto m = std::make_unique<mbx_matrix>();
  m->ctx = ctx;
  m->precision = precision;
  m->n_rows = n_rows;
  m->n_cols = n_cols;
  m->nnz = nnz;
  const size_t vs = mbx::value_size(precision);
  m->vals = dmalloc(ctx, nnz * vs + 256);
  m->cols = static_cast<int32_t*>(dmalloc(ctx, nnz * 4 + 256));
  m->ro = static_cast<uint32_t*>(dmalloc(ctx, (n_rows + 1) * 4 + 64));
  MBX_CUDA(cudaMemsetAsync(m->vals, 0, nnz * vs + 256, ctx->stream));
  MBX_CUDA(cudaMemsetAsync(m->cols, 0, nnz * 4 + 256, ctx->stream));
  if (nnz) MBX_CUDA(cudaMemcpyAsync(m->vals, vals, nnz * vs, cudaMemcpyHostToDevice, ctx->stream));
  int* bad = static_cast<int*>(dmalloc(ctx, 64));
  MBX_CUDA(cudaMemsetAsync(bad, 0, 8, ctx->stream));
  {
    int64_t* tmp = static_cast<int64_t*>(dmalloc(ctx, (n_rows + 1) * 8));
    MBX_CUDA(cudaMemcpyAsync(tmp, ro, (n_rows + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
    mbx::launch_narrow_rows(ctx, tmp, m->ro, n_rows + 1, bad);
    dfree(ctx, tmp);
  }
  if (nnz) {
    if (cols64) {
      int64_t* tmp = static_cast<int64_t*>(dmalloc(ctx, nnz * 8));
      MBX_CUDA(cudaMemcpyAsync(tmp, cols, nnz * 8, cudaMemcpyHostToDevice, ctx->stream));
      mbx::launch_narrow_cols(ctx, tmp, m->cols, nnz, n_cols, bad + 1);
      dfree(ctx, tmp);
    } else {
      MBX_CUDA(cudaMemcpyAsync(m->cols, cols, nnz * 4, cudaMemcpyHostToDevice, ctx->stream));
    }
  }
  int hb[2] = {0, 0};
  MBX_CUDA(cudaMemcpyAsync(hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  dfree(ctx, bad);
  if (hb[0] || hb[1]) {
    mbx_matrix* raw = m.release();
    mbx_matrix_destroy(raw);
    fail(MBX_DIMENSION_ERROR, hb[0] ? "row_offsets not nondecreasing / out of u32 range"
                                    : "column index outside [0, n_cols)");
  }
  return m.release();
}

}  // namespace

namespace mbx {
// the C-ABI's config / TILE validation, shared with solvers.cu
void validate_config(const mbx_simt_config* c) { check_config(c); }
void validate_tile(const mbx_matrix* m, const mbx_tile* t, const mbx_simt_config* c) {
  check_tile_matches(m, t, c);
}
}  // namespace mbx

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

MBX_API const char* mbx_last_error(void) { return g_last_error.c_str(); }

MBX_API const char* mbx_build_info(void) {
  return "libmerbit_b200 (sm_100a; MERBIT TILE preprocessing, descriptor SpMV, fused PageRank)";
}

MBX_API int mbx_config_make(int omega, int sigma, int block_size, mbx_simt_config* out) {
  return guarded([&] {
    const int ob = config_offset_bits(omega, sigma, block_size);
    require(out != nullptr, MBX_ERROR, "null output");
    *out = mbx_simt_config{omega, sigma, block_size, ob};
  });
}

MBX_API int mbx_select_sigma(int precision, int override_sigma) {
  if (override_sigma > 0) return override_sigma;
  return precision == MBX_F64 ? 7 : 14;
}

MBX_API int mbx_tile_counts(int64_t nnz, int64_t n_rows, const mbx_simt_config* c,
                            int64_t* tile_num, int64_t* lane_num) {
  return guarded([&] {
    require(c && c->omega >= 1 && c->sigma >= 1, MBX_CONFIG_ERROR, "bad config");
    tile_counts(nnz, n_rows, c->omega, c->sigma, tile_num, lane_num);
  });
}

MBX_API double mbx_metadata_footprint(int64_t nnz, int64_t n_rows, const mbx_simt_config* c,
                                      double r_f) {
  int64_t tn = 0, ln = 0;
  tile_counts(nnz, n_rows, c->omega, c->sigma, &tn, &ln);
  return 8.0 * double(tn + 1) + 4.0 * double(ln) * (1.0 - r_f);
}

MBX_API int mbx_merge_search(const int64_t* ro, int64_t n_rows, int64_t nnz, int64_t diag,
                             int64_t* x, int64_t* y) {
  return guarded([&] {
    if (diag < 0 || diag > nnz + n_rows)
      fail(MBX_DIMENSION_ERROR, "merge_search: diagonal " + std::to_string(diag) +
                                    " outside [0, " + std::to_string(nnz + n_rows) + "]");
    int64_t lo = std::max<int64_t>(diag - nnz, 0), hi = std::min<int64_t>(diag, n_rows);
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ro[mid + 1] <= diag - mid - 1)
        lo = mid + 1;
      else
        hi = mid;
    }
    *x = diag - lo;
    *y = std::min(lo, n_rows);
  });
}

MBX_API int mbx_plan_row_shards(const int64_t* ro, int64_t n_rows, int64_t nnz, int parts,
                                int64_t* bounds) {
  return guarded([&] {
    require(parts >= 1, MBX_CONFIG_ERROR, "parts must be >= 1");
    bounds[0] = 0;
    for (int g = 1; g < parts; ++g) {
      const int64_t diag = (nnz + n_rows) * g / parts;
      int64_t x = 0, y = 0;
      int rc = mbx_merge_search(ro, n_rows, nnz, diag, &x, &y);
      if (rc) fail(rc, g_last_error);
      // snap to the start of the row the cut falls in: shard g owns rows
      // [y(d_g), y(d_{g+1})); a row is never split across GPUs.
      bounds[g] = std::max(bounds[g - 1], y);
    }
    bounds[parts] = n_rows;
  });
}

MBX_API int mbx_plan_row_shards_weighted(const int64_t* ro, int64_t n_rows, int64_t nnz,
                                         int parts, double row_weight, int64_t* bounds) {
  if (row_weight == 1.0) return mbx_plan_row_shards(ro, n_rows, nnz, parts, bounds);
  return guarded([&] {
    require(parts >= 1, MBX_CONFIG_ERROR, "parts must be >= 1");
    require(row_weight >= 0.0 && row_weight < 1e9, MBX_CONFIG_ERROR,
            "row_weight must be in [0, 1e9)");
    require(n_rows >= 0 && ro[n_rows] == nnz, MBX_DIMENSION_ERROR,
            "row_offsets[n_rows] != nnz");
    const double total = static_cast<double>(nnz) + row_weight * static_cast<double>(n_rows);
    bounds[0] = 0;
    for (int g = 1; g < parts; ++g) {
      const double target = total * g / parts;
      // smallest r with ro[r] + w*r >= target (cost is nondecreasing in r)
      int64_t lo = 0, hi = n_rows;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<double>(ro[mid]) + row_weight * static_cast<double>(mid) < target)
          lo = mid + 1;
        else
          hi = mid;
      }
      bounds[g] = std::max(bounds[g - 1], lo);
    }
    bounds[parts] = n_rows;
  });
}

MBX_API int mbx_device_count(int* count) {
  return guarded([&] {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

MBX_API int mbx_context_create(int device, mbx_context** out) {
  return guarded([&] {
    int n = 0;
    MBX_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, MBX_CUDA_ERROR,
            "no CUDA device " + std::to_string(device) + " (have " + std::to_string(n) + ")");
    cudaDeviceProp prop;
    MBX_CUDA(cudaGetDeviceProperties(&prop, device));
    require(prop.major == 10, MBX_UNSUPPORTED,
            std::string("libmerbit_b200 is built for sm_100a; device is ") + prop.name);
    auto ctx = std::make_unique<mbx_context>();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    Device dg(device);
    // keep freed stream-ordered allocations in the pool: per-call buffers
    // (PageRank plans, staging) must not be re-mapped from the OS each call
    cudaMemPool_t pool;
    MBX_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    MBX_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    MBX_CUDA(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
    ctx->stream = ctx->own;
    *out = ctx.release();
  });
}

MBX_API int mbx_context_destroy(mbx_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    Device dg(ctx->device);
    drop_pr_cache(ctx);
    mbx::free_sparse_handle(ctx);
    if (ctx->scratch) cudaFreeAsync(ctx->scratch, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->host_scratch) cudaFreeHost(ctx->host_scratch);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
  });
}

MBX_API int mbx_context_set_stream(mbx_context* ctx, void* stream) {
  return guarded([&] {
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    if (s != ctx->stream) {
      // order the new stream after everything queued so far
      cudaEvent_t ev;
      MBX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      MBX_CUDA(cudaEventRecord(ev, ctx->stream));
      MBX_CUDA(cudaStreamWaitEvent(s, ev, 0));
      cudaEventDestroy(ev);
      ctx->stream = s;
    }
  });
}

MBX_API void* mbx_context_stream(mbx_context* ctx) { return ctx ? ctx->stream : nullptr; }

MBX_API int mbx_context_synchronize(mbx_context* ctx) {
  return guarded([&] { MBX_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

MBX_API int64_t mbx_context_launch_count(const mbx_context* ctx) {
  return ctx ? ctx->launches : 0;
}

MBX_API int mbx_matrix_upload(mbx_context* ctx, int precision, int64_t n_rows, int64_t n_cols,
                              const int64_t* ro, const int64_t* cols, const void* vals,
                              mbx_matrix** out) {
  return guarded(
      [&] { *out = upload_common(ctx, precision, n_rows, n_cols, ro, cols, true, vals); });
}

MBX_API int mbx_matrix_upload_i32(mbx_context* ctx, int precision, int64_t n_rows,
                                  int64_t n_cols, const int64_t* ro, const int32_t* cols,
                                  const void* vals, mbx_matrix** out) {
  return guarded(
      [&] { *out = upload_common(ctx, precision, n_rows, n_cols, ro, cols, false, vals); });
}

MBX_API int mbx_matrix_generate_rmat(mbx_context* ctx, int precision, int scale,
                                     int edge_factor, uint64_t seed, int kind,
                                     uint64_t value_seed, double lo, double hi,
                                     mbx_matrix** out) {
  return guarded([&] {
    check_precision(precision);
    require(scale >= 1 && scale <= 30 && edge_factor >= 1, MBX_CONFIG_ERROR,
            "rmat: scale in [1,30], edge_factor >= 1");
    require(kind == 0 || kind == 1, MBX_CONFIG_ERROR, "rmat kind must be 0 or 1");
    Device dg(ctx->device);
    auto m = std::make_unique<mbx_matrix>();
    m->ctx = ctx;
    mbx::generate_rmat(ctx, precision, scale, edge_factor, seed, kind, value_seed, lo, hi,
                       m.get());
    *out = m.release();
  });
}

MBX_API int mbx_matrix_generate_stencil27(mbx_context* ctx, int precision, int64_t grid_dim,
                                          mbx_matrix** out) {
  return guarded([&] {
    check_precision(precision);
    require(grid_dim >= 1 && grid_dim * grid_dim * grid_dim < (int64_t(1) << 31),
            MBX_CONFIG_ERROR, "stencil grid_dim^3 must be < 2^31");
    Device dg(ctx->device);
    auto m = std::make_unique<mbx_matrix>();
    m->ctx = ctx;
    mbx::generate_stencil27(ctx, precision, grid_dim, m.get());
    *out = m.release();
  });
}

MBX_API int mbx_matrix_generate_powerlaw(mbx_context* ctx, int precision, int log2_rows,
                                         uint64_t seed, mbx_matrix** out) {
  return guarded([&] {
    check_precision(precision);
    require(log2_rows >= 4 && log2_rows <= 30, MBX_CONFIG_ERROR, "log2_rows in [4, 30]");
    Device dg(ctx->device);
    auto m = std::make_unique<mbx_matrix>();
    m->ctx = ctx;
    mbx::generate_powerlaw(ctx, precision, log2_rows, seed, m.get());
    *out = m.release();
  });
}

MBX_API int mbx_matrix_info(const mbx_matrix* m, int* precision, int64_t* n_rows,
                            int64_t* n_cols, int64_t* nnz) {
  return guarded([&] {
    require(m != nullptr, MBX_ERROR, "null matrix");
    if (precision) *precision = m->precision;
    if (n_rows) *n_rows = m->n_rows;
    if (n_cols) *n_cols = m->n_cols;
    if (nnz) *nnz = m->nnz;
  });
}

MBX_API int mbx_matrix_download(const mbx_matrix* m, int64_t* ro, int32_t* cols, void* vals) {
  return guarded([&] {
    mbx_context* ctx = m->ctx;
    Device dg(ctx->device);
    mbx::ensure_csr(ctx, m);  // a compacted matrix rebuilds its CSR
    if (ro) {
      std::vector<uint32_t> r(m->n_rows + 1);
      MBX_CUDA(cudaMemcpyAsync(r.data(), m->ro, (m->n_rows + 1) * 4, cudaMemcpyDeviceToHost,
                               ctx->stream));
      MBX_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int64_t i = 0; i <= m->n_rows; ++i) ro[i] = r[i];
    }
    if (cols && m->nnz)
      MBX_CUDA(cudaMemcpyAsync(cols, m->cols, m->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (vals && m->nnz)
      MBX_CUDA(cudaMemcpyAsync(vals, m->vals, m->nnz * mbx::value_size(m->precision),
                               cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

MBX_API int mbx_matrix_device_ptrs(const mbx_matrix* m, const void** values,
                                   const int32_t** cols, const uint32_t** ro) {
  return guarded([&] {
    {
      Device dg(m->ctx->device);
      mbx::ensure_csr(m->ctx, m);
    }
    if (values) *values = m->vals;
    if (cols) *cols = m->cols;
    if (ro) *ro = m->ro;
  });
}

MBX_API int mbx_context_set_tuning_ex(mbx_context* ctx, int smem_per_sm, int prefetch) {
  return guarded([&] {
    ctx->tuning.smem_per_sm = smem_per_sm;
    ctx->tuning.prefetch = prefetch;
    ++ctx->tuning_epoch;
    drop_pr_cache(ctx);
  });
}

MBX_API int mbx_context_set_tuning(mbx_context* ctx, int warps_per_cta, int ctas_per_sm,
                                   int max_hubs) {
  return guarded([&] {
    const bool automatic = warps_per_cta == 0 && ctas_per_sm == 0;
    require(automatic || (warps_per_cta >= 1 && warps_per_cta <= 32 && ctas_per_sm >= 1 &&
                          ctas_per_sm <= 32),
            MBX_CONFIG_ERROR, "warps_per_cta in [1,32], ctas_per_sm in [1,32] (or both 0)");
    ctx->tuning.warps_per_cta = automatic ? 32 : warps_per_cta;
    ctx->tuning.ctas_per_sm = automatic ? 1 : ctas_per_sm;
    ctx->tuning.max_hubs = max_hubs;
    ctx->tuning.shape_auto = automatic;
    ++ctx->tuning_epoch;
    drop_pr_cache(ctx);
  });
}

MBX_API int mbx_context_set_layout(mbx_context* ctx, int layout) {
  return guarded([&] {
    require(layout == 0 || layout == 1, MBX_CONFIG_ERROR, "layout must be 0 or 1");
    ctx->tuning.layout = layout;
    ++ctx->tuning_epoch;
    drop_pr_cache(ctx);
  });
}

MBX_API int mbx_matrix_slot_info(const mbx_matrix* m, int64_t* slots, double* seconds) {
  return guarded([&] {
    if (slots) *slots = m->slots.vals ? m->slots.count : 0;
    if (seconds) *seconds = m->slots.vals ? m->slots.seconds : 0.0;
  });
}

MBX_API int mbx_matrix_build_xcache(mbx_context* ctx, mbx_matrix* m, int max_hubs,
                                    double* seconds) {
  return guarded([&] {
    Device dg(ctx->device);
    mbx::ensure_csr(ctx, m);
    cudaEvent_t e0, e1;
    MBX_CUDA(cudaEventCreate(&e0));
    MBX_CUDA(cudaEventCreate(&e1));
    MBX_CUDA(cudaEventRecord(e0, ctx->stream));
    mbx::build_xcache(ctx, m, max_hubs);
    MBX_CUDA(cudaEventRecord(e1, ctx->stream));
    MBX_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    MBX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (seconds) *seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

MBX_API int mbx_matrix_xcache_info(const mbx_matrix* m, int* hubs, double* coverage) {
  return guarded([&] {
    if (hubs) *hubs = m->hub_avail;
    if (coverage) *coverage = m->hub_coverage;
  });
}

MBX_API int mbx_matrix_xcache_ptrs(const mbx_matrix* m, const int32_t** cols_hub,
                                   const int32_t** hub_cols) {
  return guarded([&] {
    if (cols_hub) *cols_hub = m->cols_hub;
    if (hub_cols) *hub_cols = m->hub_cols;
  });
}

MBX_API int mbx_matrix_gather_profile(const mbx_matrix* m, double* sectors_per_32) {
  return guarded([&] {
    if (sectors_per_32) *sectors_per_32 = m->gather_sectors;
  });
}

MBX_API int mbx_matrix_hub_columns(const mbx_matrix* m, int32_t* host_out) {
  return guarded([&] {
    if (m->hub_avail <= 0 || !host_out) return;
    mbx_context* ctx = m->ctx;
    Device dg(ctx->device);
    MBX_CUDA(cudaMemcpyAsync(host_out, m->hub_cols, size_t(m->hub_avail) * 4,
                             cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

MBX_API int mbx_matrix_compact(mbx_matrix* m, const mbx_tile* t) {
  return guarded([&] {
    mbx_context* ctx = m->ctx;
    Device dg(ctx->device);
    if (t->ctx != ctx) fail(MBX_CONFIG_ERROR, "compact: TILE of another context");
    mbx::compact_matrix(ctx, m, t);
  });
}

MBX_API int mbx_matrix_resident_bytes(const mbx_matrix* m, int64_t* bytes) {
  return guarded([&] {
    const int64_t vs = int64_t(mbx::value_size(m->precision));
    int64_t b = (m->n_rows + 1) * 4;
    if (m->vals) b += m->nnz * vs;
    if (m->cols) b += m->nnz * 4;
    if (m->cols_hub) b += m->nnz * 4;
    if (m->hub_cols) b += int64_t(m->hub_avail) * 4;
    if (m->slots.vals) b += m->slots.count * (vs + 4);
    if (m->coo_rows) b += m->nnz * 4;
    if (m->vmap) b += m->n_rows * 4;
    if (m->compact)
      b += (2 * (m->compact->info.tile_num + 1) + m->compact->info.lane_num) * 4;
    if (m->dmask) b += ((m->n_cols + 31) / 32) * 4;
    *bytes = b;
  });
}

MBX_API int mbx_matrix_release_caches(mbx_matrix* m) {
  return guarded([&] {
    mbx_context* ctx = m->ctx;
    Device dg(ctx->device);
    mbx::ensure_csr(ctx, m);  // the slot copy is a compacted matrix's only data
    mbx::free_slots(ctx, m);
    if (m->cols_hub || m->hub_cols) {
      dfree(ctx, m->cols_hub);
      dfree(ctx, m->hub_cols);
      m->cols_hub = m->hub_cols = nullptr;
      m->hub_avail = 0;
      m->hub_coverage = 0.0;
      ++m->version;
      ++m->gen;
    }
    mbx::free_sparse_state(ctx, m);
    dfree(ctx, m->coo_rows);
    m->coo_rows = nullptr;
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

MBX_API int mbx_matrix_destroy(mbx_matrix* m) {
  return guarded([&] {
    if (!m) return;
    mbx_context* ctx = m->ctx;
    Device dg(ctx->device);
    if (pr_cache_refs(ctx, m)) drop_pr_cache(ctx);
    dfree(ctx, m->vals);
    dfree(ctx, m->cols);
    dfree(ctx, m->ro);
    dfree(ctx, m->cols_hub);
    dfree(ctx, m->hub_cols);
    mbx::free_slots(ctx, m);
    mbx::free_compact_tile(ctx, m);
    dfree(ctx, m->dmask);
    mbx::free_sparse_state(ctx, m);
    dfree(ctx, m->coo_rows);
    dfree(ctx, m->vmap);
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    delete m;
  });
}

MBX_API int mbx_generate_tile(mbx_context* ctx, const int64_t* ro, int64_t n_rows, int64_t nnz,
                              const mbx_simt_config* c, mbx_tile** out) {
  return guarded([&] {
    check_config(c);
    tile_capacity(n_rows, nnz);  // before touching the data (test_format.cpp:149-158)
    require(n_rows >= 0 && nnz >= 0, MBX_DIMENSION_ERROR, "negative sizes");
    require(ro != nullptr || n_rows + nnz == 0, MBX_DIMENSION_ERROR, "null row_offsets");
    Device dg(ctx->device);
    uint32_t* ro32 = static_cast<uint32_t*>(dmalloc(ctx, (n_rows + 1) * 4 + 64));
    int* bad = static_cast<int*>(dmalloc(ctx, 64));
    MBX_CUDA(cudaMemsetAsync(bad, 0, 8, ctx->stream));
    if (ro) {
      int64_t* tmp = static_cast<int64_t*>(dmalloc(ctx, (n_rows + 1) * 8));
      MBX_CUDA(cudaMemcpyAsync(tmp, ro, (n_rows + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
      mbx::launch_narrow_rows(ctx, tmp, ro32, n_rows + 1, bad);
      dfree(ctx, tmp);
    } else {
      MBX_CUDA(cudaMemsetAsync(ro32, 0, 4, ctx->stream));
    }
    mbx_tile* t = new_tile(ctx, *c, n_rows, nnz);
    generate_tile_timed(ctx, ro32, n_rows, nnz, *c, t);
    int hb = 0;
    MBX_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    dfree(ctx, ro32);
    dfree(ctx, bad);
    if (hb) {
      mbx_tile_destroy(t);
      fail(MBX_DIMENSION_ERROR, "row_offsets not nondecreasing / out of u32 range");
    }
    *out = t;
  });
}

MBX_API int mbx_matrix_generate_tile(mbx_context* ctx, const mbx_matrix* m,
                                     const mbx_simt_config* c, mbx_tile** out) {
  return guarded([&] {
    check_config(c);
    tile_capacity(m->n_rows, m->nnz);
    Device dg(ctx->device);
    mbx_tile* t = new_tile(ctx, *c, m->n_rows, m->nnz);
    generate_tile_timed(ctx, m->ro, m->n_rows, m->nnz, *c, t);
    *out = t;
  });
}

MBX_API int mbx_tile_get_info(const mbx_tile* t, mbx_tile_info* info) {
  return guarded([&] {
    require(t != nullptr, MBX_ERROR, "null tile");
    *info = t->info;
  });
}

MBX_API int mbx_tile_download(const mbx_tile* t, uint32_t* tx, uint32_t* ty, uint32_t* ld) {
  return guarded([&] {
    mbx_context* ctx = t->ctx;
    Device dg(ctx->device);
    if (tx)
      MBX_CUDA(cudaMemcpyAsync(tx, t->tile_x, (t->info.tile_num + 1) * 4, cudaMemcpyDeviceToHost,
                               ctx->stream));
    if (ty)
      MBX_CUDA(cudaMemcpyAsync(ty, t->tile_y, (t->info.tile_num + 1) * 4, cudaMemcpyDeviceToHost,
                               ctx->stream));
    if (ld && t->info.lane_num)
      MBX_CUDA(cudaMemcpyAsync(ld, t->lane_desc, t->info.lane_num * 4, cudaMemcpyDeviceToHost,
                               ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

MBX_API int mbx_tile_upload(mbx_context* ctx, const mbx_tile_info* info, const uint32_t* tx,
                            const uint32_t* ty, const uint32_t* ld, mbx_tile** out) {
  return guarded([&] {
    mbx_simt_config c;
    int rc = mbx_config_make(info->omega, info->sigma, info->omega, &c);
    if (rc) fail(rc, g_last_error);
    tile_capacity(info->n_rows, info->nnz);
    Device dg(ctx->device);
    mbx_tile* t = new_tile(ctx, c, info->n_rows, info->nnz);
    t->info.preprocess_seconds = info->preprocess_seconds;
    MBX_CUDA(cudaMemcpyAsync(t->tile_x, tx, (t->info.tile_num + 1) * 4, cudaMemcpyHostToDevice,
                             ctx->stream));
    MBX_CUDA(cudaMemcpyAsync(t->tile_y, ty, (t->info.tile_num + 1) * 4, cudaMemcpyHostToDevice,
                             ctx->stream));
    if (t->info.lane_num)
      MBX_CUDA(cudaMemcpyAsync(t->lane_desc, ld, t->info.lane_num * 4, cudaMemcpyHostToDevice,
                               ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = t;
  });
}

MBX_API int mbx_tile_destroy(mbx_tile* t) {
  return guarded([&] {
    if (!t) return;
    mbx_context* ctx = t->ctx;
    Device dg(ctx->device);
    if (pr_cache_refs(ctx, t)) drop_pr_cache(ctx);
    dfree(ctx, t->tile_x);
    dfree(ctx, t->tile_y);
    dfree(ctx, t->lane_desc);
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    delete t;
  });
}

MBX_API int mbx_spmv_device(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                            const mbx_simt_config* c, const void* x, void* y) {
  return guarded([&] {
    check_config(c);
    check_tile_matches(m, t, c);
    Device dg(ctx->device);
    const mbx::Geometry g = mbx::make_geometry(ctx, m, t, c->block_size);
    void* ws = mbx::scratch(ctx, mbx::spmv_workspace_bytes(g, m->precision, false));
    mbx::launch_spmv(ctx, m, t, g, x, y, ws, nullptr);
  });
}

MBX_API int mbx_spmv_trace_counts(mbx_context* ctx, const mbx_tile* t, mbx_spmv_trace* trace) {
  return guarded([&] {
    Device dg(ctx->device);
    unsigned long long* d = static_cast<unsigned long long*>(dmalloc(ctx, 64));
    MBX_CUDA(cudaMemsetAsync(d, 0, 24, ctx->stream));
    mbx::launch_trace_counts(ctx, t, d);
    unsigned long long h[3];
    MBX_CUDA(cudaMemcpyAsync(h, d, 24, cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    dfree(ctx, d);
    trace->fast_tiles = int64_t(h[0]);
    trace->normal_tiles = int64_t(h[1]);
    trace->skipped_tiles = int64_t(h[2]);
  });
}

MBX_API int mbx_spmv(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                     const mbx_simt_config* c, const void* x_host, void* y_host,
                     mbx_spmv_trace* trace) {
  return guarded([&] {
    check_config(c);
    check_tile_matches(m, t, c);
    Device dg(ctx->device);
    const size_t vs = mbx::value_size(m->precision);
    void* x = dmalloc(ctx, m->n_cols * vs + 256);
    void* y = dmalloc(ctx, m->n_rows * vs + 256);
    // a degree-relabelled matrix takes x and gives y in the original order
    void* tmp = m->vmap ? dmalloc(ctx, std::max(m->n_rows, m->n_cols) * vs + 256) : nullptr;
    if (m->n_cols)
      MBX_CUDA(cudaMemcpyAsync(m->vmap ? tmp : x, x_host, m->n_cols * vs, cudaMemcpyHostToDevice,
                               ctx->stream));
    if (m->vmap) mbx::launch_vertex_map(ctx, m->precision, m->n_cols, m->vmap, tmp, x, true);
    const mbx::Geometry g = mbx::make_geometry(ctx, m, t, c->block_size);
    void* ws = mbx::scratch(ctx, mbx::spmv_workspace_bytes(g, m->precision, false));
    mbx::launch_spmv(ctx, m, t, g, x, y, ws, nullptr);
    if (m->vmap) mbx::launch_vertex_map(ctx, m->precision, m->n_rows, m->vmap, y, tmp, false);
    if (m->n_rows)
      MBX_CUDA(cudaMemcpyAsync(y_host, m->vmap ? tmp : y, m->n_rows * vs, cudaMemcpyDeviceToHost,
                               ctx->stream));
    dfree(ctx, x);
    dfree(ctx, y);
    dfree(ctx, tmp);
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    if (trace) {
      int rc = mbx_spmv_trace_counts(ctx, t, trace);
      if (rc) fail(rc, g_last_error);
    }
  });
}

MBX_API int mbx_spmv_deposits(mbx_context* ctx, const mbx_matrix* m, const mbx_tile* t,
                              const mbx_simt_config* c, const void* x_host, int64_t* rows_host,
                              void* amounts_host, int64_t capacity, int64_t* count) {
  return guarded([&] {
    check_config(c);
    check_tile_matches(m, t, c);
    Device dg(ctx->device);
    const size_t vs = mbx::value_size(m->precision);
    const int64_t lanes = t->info.lane_num;
    // a lane deposits at most once per step plus its trailing partial
    const int64_t bound = lanes * (int64_t(t->info.sigma) + 1);
    if (!rows_host || !amounts_host) {  // capacity query
      *count = bound;
      return;
    }
    void* x = dmalloc(ctx, m->n_cols * vs + 256);
    void* tmp = m->vmap ? dmalloc(ctx, m->n_cols * vs + 256) : nullptr;
    if (m->n_cols)
      MBX_CUDA(cudaMemcpyAsync(m->vmap ? tmp : x, x_host, m->n_cols * vs, cudaMemcpyHostToDevice,
                               ctx->stream));
    if (m->vmap) mbx::launch_vertex_map(ctx, m->precision, m->n_cols, m->vmap, tmp, x, true);
    const int64_t cap = std::min(capacity, bound);
    auto* counter = static_cast<unsigned long long*>(dmalloc(ctx, 64));
    int64_t* rows = static_cast<int64_t*>(dmalloc(ctx, cap * 8 + 256));
    void* amounts = dmalloc(ctx, cap * vs + 256);
    MBX_CUDA(cudaMemsetAsync(counter, 0, 8, ctx->stream));
    mbx::launch_deposits(ctx, m, t, x, counter, cap, rows, amounts);
    unsigned long long n = 0;
    MBX_CUDA(cudaMemcpyAsync(&n, counter, 8, cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t got = std::min<int64_t>(int64_t(n), cap);
    if (got) {
      MBX_CUDA(cudaMemcpyAsync(rows_host, rows, got * 8, cudaMemcpyDeviceToHost, ctx->stream));
      MBX_CUDA(cudaMemcpyAsync(amounts_host, amounts, got * vs, cudaMemcpyDeviceToHost,
                               ctx->stream));
    }
    std::vector<int32_t> vmap;
    if (m->vmap && got) {  // rows back to the caller's vertex numbering
      vmap.resize(size_t(m->n_rows));
      MBX_CUDA(cudaMemcpyAsync(vmap.data(), m->vmap, m->n_rows * 4, cudaMemcpyDeviceToHost,
                               ctx->stream));
    }
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!vmap.empty()) {
      std::vector<int64_t> orig(size_t(m->n_rows));
      for (int64_t v = 0; v < m->n_rows; ++v) orig[size_t(vmap[size_t(v)])] = v;
      for (int64_t k = 0; k < got; ++k)
        if (rows_host[k] < m->n_rows) rows_host[k] = orig[size_t(rows_host[k])];
    }
    *count = int64_t(n);
    dfree(ctx, x);
    dfree(ctx, tmp);
    dfree(ctx, counter);
    dfree(ctx, rows);
    dfree(ctx, amounts);
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

MBX_API int mbx_spmv_csr_device(mbx_context* ctx, const mbx_matrix* m, const void* x, void* y) {
  return guarded([&] {
    Device dg(ctx->device);
    mbx::ensure_csr(ctx, m);
    mbx::launch_csr(ctx, m, x, y, nullptr, nullptr, nullptr);
  });
}

}  // extern "C"

// ============================================================================
// PageRank plan
// ============================================================================
struct mbx_pagerank_plan_s {
  mbx_context* ctx = nullptr;
  const mbx_matrix* p = nullptr;
  const mbx_tile* t = nullptr;
  mbx_simt_config c{};
  mbx_pagerank_config cfg{};
  mbx::Geometry g;
  int64_t n = 0;
  size_t vs = 4;
  void* pi[2] = {nullptr, nullptr};
  void* ref[2] = {nullptr, nullptr};
  uint32_t* dangling = nullptr;
  int64_t dang_from = -1;  // dangling rows = [dang_from, n) when a suffix
  mbx::PrScalars* scal = nullptr;      // [max_iters + 1]
  mbx::PrScalars* ref_scal = nullptr;  // [reference_iters + 1]
  uint32_t* carry_mask = nullptr;  // K2 -> K3: the range boundary rows
  double* block_part = nullptr;
  unsigned int* counter = nullptr;
  int* flags = nullptr;  // [0] stop, [1] stop_iter
  void* carry_ws = nullptr;
  size_t carry_ws_bytes = 0;  // its size: a re-made geometry may need more
  int64_t block_part_n = 0;   // block_part slots (4 doubles each)
  cudaGraphExec_t graph = nullptr;
  int64_t graph_launches = 0;
  int64_t* iter_dev = nullptr;  // iterations completed (device-driven loop)
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool ran = false;
  // cache key (mbx_pagerank): what the plan was built from
  uint64_t p_version = 0, t_serial = 0, tuning_epoch = 0;
  uint64_t p_gen = 0;  // the matrix's buffer generation the graph captured
  mbx_pagerank_config cfg_in{};
};

namespace {

// drop the context's cached mbx_pagerank plan (if any)
void drop_pr_cache(mbx_context* ctx) {
  if (ctx->pr_cache) {
    mbx_pagerank_plan* pl = ctx->pr_cache;
    ctx->pr_cache = nullptr;
    mbx_pagerank_plan_destroy(pl);
  }
}

bool pr_cache_refs(const mbx_context* ctx, const void* obj) {
  return ctx->pr_cache && (static_cast<const void*>(ctx->pr_cache->p) == obj ||
                           static_cast<const void*>(ctx->pr_cache->t) == obj);
}

bool same_config(const mbx_simt_config& a, const mbx_simt_config& b) {
  return a.omega == b.omega && a.sigma == b.sigma && a.block_size == b.block_size;
}

bool same_config(const mbx_pagerank_config& a, const mbx_pagerank_config& b) {
  return a.damping == b.damping && a.err_tol == b.err_tol && a.max_iters == b.max_iters &&
         a.reference_iters == b.reference_iters;
}

}  // namespace

namespace {

mbx::PrArgs pr_args(mbx_pagerank_plan* pl, int64_t r, const void* yard) {
  mbx::PrArgs a;
  a.pi_old = pl->pi[(r - 1) & 1];
  a.dangling = pl->dangling;
  a.dang_from = pl->dang_from;
  a.yardstick = yard;
  a.yard_const = pl->p->precision == MBX_F32 ? double(1.0f / float(pl->n)) : 1.0 / double(pl->n);
  a.damping = pl->cfg.damping;
  a.inv_n = 1.0 / double(pl->n);
  a.prev = pl->scal + (r - 1);
  a.next = pl->scal + r;
  a.carry_mask = pl->carry_mask;
  a.block_part = pl->block_part;
  a.done_counter = pl->counter;
  a.stop = pl->flags;
  a.stop_iter = pl->flags + 1;
  a.iter = int(r);
  a.err_tol = pl->cfg.err_tol;
  return a;
}

// One body of the device-driven loop: an odd iteration (pi0 -> pi1), an
// even one (pi1 -> pi0), then the WHILE condition.  Every iteration number,
// scalar slot and the stop / max_iters guards come from the device.
void launch_loop_body(mbx_pagerank_plan* pl, cudaGraphConditionalHandle h) {
  const void* yard = pl->cfg.reference_iters > 0 ? pl->ref[pl->cfg.reference_iters & 1] : nullptr;
  for (int64_t r = 1; r <= 2; ++r) {
    mbx::PrArgs a = pr_args(pl, r, yard);
    a.iter_dev = pl->iter_dev;
    a.scal_base = pl->scal;
    a.max_iters = pl->cfg.max_iters;
    a.prev = nullptr;
    a.next = nullptr;
    a.iter = 0;
    mbx::launch_spmv(pl->ctx, pl->p, pl->t, pl->g, pl->pi[(r - 1) & 1], pl->pi[r & 1],
                     pl->carry_ws, &a);
  }
  mbx::launch_pr_loop_cond(pl->ctx, h, pl->iter_dev, pl->cfg.max_iters, pl->flags);
}

void launch_power_loop(mbx_pagerank_plan* pl) {
  const void* yard = pl->cfg.reference_iters > 0 ? pl->ref[pl->cfg.reference_iters & 1] : nullptr;
  for (int64_t r = 1; r <= pl->cfg.max_iters; ++r) {
    const mbx::PrArgs a = pr_args(pl, r, yard);
    mbx::launch_spmv(pl->ctx, pl->p, pl->t, pl->g, pl->pi[(r - 1) & 1], pl->pi[r & 1],
                     pl->carry_ws, &a);
  }
}

}  // namespace

namespace {

// block_part slots a plan's K3 / yardstick / pi_0 grids need
int64_t plan_block_slots(mbx_context* ctx, const mbx_matrix* p, const mbx::Geometry& g) {
  const int64_t k3_blocks = std::max(mbx::fixup_blocks(g, true), mbx::fixup_blocks(g, false)) + 1;
  return std::max<int64_t>({k3_blocks, int64_t(mbx::csr_pr_blocks(ctx, p)),
                            int64_t(ctx->sm_count) * 4 + 1});
}

// Capture the power loop of `pl` (geometry already made): records the
// matrix's buffer generation the graph was captured against.
void capture_plan(mbx_pagerank_plan* pl) {
  mbx_context* ctx = pl->ctx;
  if (pl->graph) {
    cudaGraphExecDestroy(pl->graph);
    pl->graph = nullptr;
  }
  pl->p_gen = pl->p->gen;
  // The power loop as ONE CUDA graph with a device-driven WHILE node: the
  // body (two iterations + the condition) replays until max_iters or the
  // stop decision -- an early exit launches nothing more, and any max_iters
  // fits one small graph.  MBX_GRAPH_MODE=unrolled captures the fixed-count
  // loop instead (ncu does not profile kernels inside conditional nodes),
  // =eager launches every kernel from the host.
  const mbx::GraphMode gmode = mbx::graph_mode();
  if (pl->cfg.max_iters > 0 && gmode == mbx::GraphMode::unrolled && pl->cfg.max_iters <= 4096) {
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t before = ctx->launches;
    cudaGraph_t graph;
    MBX_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
      launch_power_loop(pl);
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &graph);
      throw;
    }
    MBX_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
    MBX_CUDA(cudaGraphInstantiate(&pl->graph, graph, 0));
    cudaGraphDestroy(graph);
    pl->graph_launches = ctx->launches - before;
    ctx->launches = before;
  } else if (pl->cfg.max_iters > 0 && gmode == mbx::GraphMode::device_loop) {
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
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
      MBX_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal));
      try {
        launch_loop_body(pl, h);
      } catch (...) {
        cudaGraph_t dummy;
        cudaStreamEndCapture(ctx->stream, &dummy);
        throw;
      }
      MBX_CUDA(cudaStreamEndCapture(ctx->stream, &body));
      const int64_t per_body = ctx->launches - before;
      ctx->launches = before;
      MBX_CUDA(cudaGraphInstantiate(&pl->graph, graph, 0));
      // launches of a run to max_iters (an early stop launches fewer)
      pl->graph_launches = per_body * ((pl->cfg.max_iters + 1) / 2);
    } catch (...) {
      cudaGraphDestroy(graph);
      throw;
    }
    cudaGraphDestroy(graph);
  }
}

// The matrix freed or rebuilt a buffer the plan's graph / geometry points at
// (slot copy rebuilt for another TILE or hub setting, x hub cache rebuilt):
// make the geometry again (rebuilding the slot copy for this TILE) and
// re-capture before the next replay.
void refresh_plan(mbx_pagerank_plan* pl) {
  if (pl->p->gen == pl->p_gen) return;
  mbx_context* ctx = pl->ctx;
  MBX_CUDA(cudaStreamSynchronize(ctx->stream));
  pl->g = mbx::make_geometry(ctx, pl->p, pl->t, pl->c.block_size);
  // the new geometry's workspace (e.g. a hub table that did not exist at
  // capture: the gathered hub values live after the carries) must fit
  const size_t ws = mbx::spmv_workspace_bytes(pl->g, pl->p->precision, true);
  if (ws > pl->carry_ws_bytes) {
    dfree(ctx, pl->carry_ws);
    pl->carry_ws = dmalloc(ctx, ws);
    pl->carry_ws_bytes = ws;
  }
  const int64_t nb = plan_block_slots(ctx, pl->p, pl->g);
  if (nb > pl->block_part_n) {
    dfree(ctx, pl->block_part);
    pl->block_part = static_cast<double*>(dmalloc(ctx, nb * 4 * sizeof(double)));
    pl->block_part_n = nb;
  }
  capture_plan(pl);
}

}  // namespace

extern "C" {

MBX_API int mbx_pagerank_plan_create(mbx_context* ctx, const mbx_matrix* p, const mbx_tile* t,
                                     const mbx_simt_config* c, const mbx_pagerank_config* cfg,
                                     mbx_pagerank_plan** out) {
  return guarded([&] {
    if (p->n_rows != p->n_cols) fail(MBX_DIMENSION_ERROR, "pagerank needs a square transition matrix");
    if (p->n_rows < 1) fail(MBX_DIMENSION_ERROR, "pagerank needs at least one vertex");
    if (!(cfg->damping >= 0.0 && cfg->damping <= 1.0)) fail(MBX_CONFIG_ERROR, "damping must lie in [0, 1]");
    if (!(cfg->err_tol > 0.0)) fail(MBX_CONFIG_ERROR, "err_tol must be positive");
    require(cfg->max_iters >= 0 && cfg->reference_iters >= 0, MBX_CONFIG_ERROR,
            "iteration counts must be >= 0");
    check_config(c);
    check_tile_matches(p, t, c);
    Device dg(ctx->device);
    auto pl = std::make_unique<mbx_pagerank_plan>();
    pl->ctx = ctx;
    pl->p = p;
    pl->t = t;
    pl->c = *c;
    pl->cfg = *cfg;
    if (p->precision == MBX_F32) {
      // PageRankConfig<float> stores damping / err_tol as float
      pl->cfg.damping = double(float(cfg->damping));
      pl->cfg.err_tol = double(float(cfg->err_tol));
    }
    pl->g = mbx::make_geometry(ctx, p, t, c->block_size);
    pl->n = p->n_rows;
    pl->vs = mbx::value_size(p->precision);
    for (int i = 0; i < 2; ++i) pl->pi[i] = dmalloc(ctx, pl->n * pl->vs + 256);
    if (cfg->reference_iters > 0)
      for (int i = 0; i < 2; ++i) pl->ref[i] = dmalloc(ctx, pl->n * pl->vs + 256);
    pl->dangling = static_cast<uint32_t*>(dmalloc(ctx, ((pl->n + 31) / 32) * 4 + 64));
    mbx::launch_dangling_mask(ctx, p, pl->dangling);
    pl->dang_from = mbx::dangling_suffix_start(ctx, pl->dangling, pl->n);
    pl->scal = static_cast<mbx::PrScalars*>(dmalloc(ctx, (cfg->max_iters + 1) * sizeof(mbx::PrScalars)));
    pl->ref_scal = static_cast<mbx::PrScalars*>(
        dmalloc(ctx, (cfg->reference_iters + 1) * sizeof(mbx::PrScalars)));
    MBX_CUDA(cudaMemsetAsync(pl->scal, 0, (cfg->max_iters + 1) * sizeof(mbx::PrScalars), ctx->stream));
    const size_t mask_bytes = size_t((pl->n + 31) / 32) * 4 + 64;
    pl->carry_mask = static_cast<uint32_t*>(dmalloc(ctx, mask_bytes));
    MBX_CUDA(cudaMemsetAsync(pl->carry_mask, 0, mask_bytes, ctx->stream));
    const int64_t nb = plan_block_slots(ctx, p, pl->g);
    pl->block_part = static_cast<double*>(dmalloc(ctx, nb * 4 * sizeof(double)));
    pl->block_part_n = nb;
    pl->counter = static_cast<unsigned int*>(dmalloc(ctx, 64));
    pl->flags = static_cast<int*>(dmalloc(ctx, 64));
    MBX_CUDA(cudaMemsetAsync(pl->counter, 0, 64, ctx->stream));
    pl->carry_ws_bytes = mbx::spmv_workspace_bytes(pl->g, p->precision, true);
    pl->carry_ws = dmalloc(ctx, pl->carry_ws_bytes);
    MBX_CUDA(cudaEventCreate(&pl->e0));
    MBX_CUDA(cudaEventCreate(&pl->e1));
    pl->iter_dev = static_cast<int64_t*>(dmalloc(ctx, 64));
    MBX_CUDA(cudaMemsetAsync(pl->iter_dev, 0, 64, ctx->stream));
    capture_plan(pl.get());
    *out = pl.release();
  });
}

namespace {

// yardstick + pi_0 of a run (everything before the power loop)
void plan_prologue(mbx_pagerank_plan* pl, const void* pi0);

}  // namespace

MBX_API int mbx_pagerank_plan_run(mbx_pagerank_plan* pl, const void* pi0) {
  return guarded([&] {
    mbx_context* ctx = pl->ctx;
    Device dg(ctx->device);
    refresh_plan(pl);
    plan_prologue(pl, pi0);
    MBX_CUDA(cudaEventRecord(pl->e0, ctx->stream));
    if (pl->graph) {
      MBX_CUDA(cudaGraphLaunch(pl->graph, ctx->stream));
      ctx->launches += pl->graph_launches;
    } else {
      launch_power_loop(pl);
    }
    MBX_CUDA(cudaEventRecord(pl->e1, ctx->stream));
    pl->ran = true;
  });
}

namespace {

void plan_prologue(mbx_pagerank_plan* pl, const void* pi0) {
  {
    mbx_context* ctx = pl->ctx;
    MBX_CUDA(cudaMemsetAsync(pl->flags, 0, 8, ctx->stream));
    if (pl->iter_dev) MBX_CUDA(cudaMemsetAsync(pl->iter_dev, 0, 8, ctx->stream));
    // Yardstick: fixed-count power run on the plain CSR kernel (178-191).
    if (pl->cfg.reference_iters > 0) {
      mbx::launch_pr_init(ctx, pl->p->precision, pl->n, nullptr, pl->ref[0], pl->dangling,
                          pl->ref_scal, pl->block_part, pl->counter);
      for (int64_t r = 1; r <= pl->cfg.reference_iters; ++r) {
        mbx::PrArgs a;
        a.pi_old = pl->ref[(r - 1) & 1];
        a.dangling = pl->dangling;
        a.dang_from = pl->dang_from;
        a.yard_const = 1.0;
        a.damping = pl->cfg.damping;
        a.inv_n = 1.0 / double(pl->n);
        a.prev = pl->ref_scal + (r - 1);
        a.next = pl->ref_scal + r;
        mbx::launch_csr(ctx, pl->p, pl->ref[(r - 1) & 1], pl->ref[r & 1], &a, pl->block_part,
                        pl->counter);
      }
    }
    mbx::launch_pr_init(ctx, pl->p->precision, pl->n, pi0, pl->pi[0], pl->dangling, pl->scal,
                        pl->block_part, pl->counter);
  }
}

}  // namespace

MBX_API int mbx_pagerank_plan_result(mbx_pagerank_plan* pl, mbx_pagerank_result* res,
                                     double* history) {
  return guarded([&] {
    require(pl->ran, MBX_ERROR, "plan has not run");
    mbx_context* ctx = pl->ctx;
    Device dg(ctx->device);
    int flags[2];
    MBX_CUDA(cudaMemcpyAsync(flags, pl->flags, 8, cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<mbx::PrScalars> sc(pl->cfg.max_iters + 1);
    MBX_CUDA(cudaMemcpyAsync(sc.data(), pl->scal, sc.size() * sizeof(mbx::PrScalars),
                             cudaMemcpyDeviceToHost, ctx->stream));
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t iters = flags[0] ? flags[1] : pl->cfg.max_iters;
    if (flags[0] == 2)
      fail(MBX_ERROR, "pagerank: zero-norm iterate at iteration " + std::to_string(iters));
    float ms = 0.f;
    MBX_CUDA(cudaEventElapsedTime(&ms, pl->e0, pl->e1));
    res->iterations = iters;
    res->status = flags[0] == 1 ? 0 : 1;
    res->final_err = iters > 0 ? sc[iters].err : std::numeric_limits<double>::infinity();
    res->preprocess_seconds = pl->t->info.preprocess_seconds;
    res->iterate_seconds = ms * 1e-3;
    res->l1_residual = iters > 0 ? sc[iters].resid : 0.0;
    res->mass = sc[iters].mass;
    res->dangling_mass = sc[iters].dangling;
    if (history)
      for (int64_t r = 1; r <= pl->cfg.max_iters; ++r)
        history[r - 1] = r <= iters ? sc[r].resid : 0.0;
  });
}

MBX_API const void* mbx_pagerank_plan_pi(const mbx_pagerank_plan* pl) {
  // The final iterate of the last run: pi[iterations & 1].  Synchronous read
  // of the stop flag so early exits resolve to the right buffer.
  if (!pl) return nullptr;
  int flags[2] = {0, 0};
  if (cudaMemcpyAsync(flags, pl->flags, 8, cudaMemcpyDeviceToHost, pl->ctx->stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(pl->ctx->stream) != cudaSuccess)
    return nullptr;
  const int64_t iters = flags[0] ? flags[1] : pl->cfg.max_iters;
  return pl->pi[iters & 1];
}

MBX_API const void* mbx_pagerank_plan_reference_pi(const mbx_pagerank_plan* pl) {
  if (!pl || pl->cfg.reference_iters == 0) return nullptr;
  return pl->ref[pl->cfg.reference_iters & 1];
}

MBX_API int mbx_pagerank_plan_destroy(mbx_pagerank_plan* pl) {
  return guarded([&] {
    if (!pl) return;
    mbx_context* ctx = pl->ctx;
    Device dg(ctx->device);
    if (pl->graph) cudaGraphExecDestroy(pl->graph);
    for (void* b : {pl->pi[0], pl->pi[1], pl->ref[0], pl->ref[1]}) dfree(ctx, b);
    dfree(ctx, pl->dangling);
    dfree(ctx, pl->scal);
    dfree(ctx, pl->ref_scal);
    dfree(ctx, pl->carry_mask);
    dfree(ctx, pl->block_part);
    dfree(ctx, pl->counter);
    dfree(ctx, pl->flags);
    dfree(ctx, pl->carry_ws);
    dfree(ctx, pl->iter_dev);
    if (pl->e0) cudaEventDestroy(pl->e0);
    if (pl->e1) cudaEventDestroy(pl->e1);
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    delete pl;
  });
}

MBX_API int mbx_pagerank(mbx_context* ctx, const mbx_matrix* p, const mbx_tile* t,
                         const mbx_simt_config* c, const mbx_pagerank_config* cfg,
                         const void* pi0_host, void* pi_host, void* ref_host, double* history,
                         mbx_pagerank_result* result) {
  return guarded([&] {
    // reuse the context's plan when nothing it was built from has changed
    mbx_pagerank_plan* pl = ctx->pr_cache;
    if (!(pl && pl->p == p && pl->p_version == p->version && pl->t == t &&
          pl->t_serial == t->serial && pl->tuning_epoch == ctx->tuning_epoch &&
          same_config(pl->c, *c) && same_config(pl->cfg_in, *cfg))) {
      drop_pr_cache(ctx);
      pl = nullptr;
      int rc = mbx_pagerank_plan_create(ctx, p, t, c, cfg, &pl);
      if (rc) fail(rc, g_last_error);
      pl->p_version = p->version;
      pl->t_serial = t->serial;
      pl->tuning_epoch = ctx->tuning_epoch;
      pl->cfg_in = *cfg;
    } else {
      ctx->pr_cache = nullptr;  // owned by this call until it succeeds
    }
    std::unique_ptr<mbx_pagerank_plan, int (*)(mbx_pagerank_plan*)> guard(pl, mbx_pagerank_plan_destroy);
    int rc = 0;
    Device dg(ctx->device);
    // a degree-relabelled matrix keeps its vertex map: pi0 / pi / the
    // yardstick cross the boundary in the ORIGINAL vertex order
    void* pi0 = nullptr;
    void* tmp = p->vmap ? dmalloc(ctx, pl->n * pl->vs + 256) : nullptr;
    if (pi0_host) {
      pi0 = dmalloc(ctx, pl->n * pl->vs);
      MBX_CUDA(cudaMemcpyAsync(p->vmap ? tmp : pi0, pi0_host, pl->n * pl->vs,
                               cudaMemcpyHostToDevice, ctx->stream));
      if (p->vmap) mbx::launch_vertex_map(ctx, p->precision, pl->n, p->vmap, tmp, pi0, true);
    }
    rc = mbx_pagerank_plan_run(pl, pi0);
    if (rc) fail(rc, g_last_error);
    rc = mbx_pagerank_plan_result(pl, result, history);
    if (rc) fail(rc, g_last_error);
    auto download = [&](void* host, const void* dev) {
      const void* src = dev;
      if (p->vmap) {
        mbx::launch_vertex_map(ctx, p->precision, pl->n, p->vmap, dev, tmp, false);
        src = tmp;
      }
      MBX_CUDA(cudaMemcpyAsync(host, src, pl->n * pl->vs, cudaMemcpyDeviceToHost, ctx->stream));
      MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    };
    if (pi_host) download(pi_host, pl->pi[result->iterations & 1]);
    if (ref_host) {
      if (cfg->reference_iters > 0) {
        download(ref_host, pl->ref[cfg->reference_iters & 1]);
      } else {
        // zero-iteration yardstick: the uniform start vector
        if (p->precision == MBX_F32) {
          float* r = static_cast<float*>(ref_host);
          for (int64_t i = 0; i < pl->n; ++i) r[i] = 1.0f / float(pl->n);
        } else {
          double* r = static_cast<double*>(ref_host);
          for (int64_t i = 0; i < pl->n; ++i) r[i] = 1.0 / double(pl->n);
        }
      }
    }
    dfree(ctx, pi0);
    dfree(ctx, tmp);
    MBX_CUDA(cudaStreamSynchronize(ctx->stream));
    // kept for the next call (only for objects of this context: their
    // destroy calls are what invalidate it)
    if (p->ctx == ctx && t->ctx == ctx) ctx->pr_cache = guard.release();
  });
}

MBX_API int mbx_pagerank_observed(mbx_context* ctx, const mbx_matrix* p, const mbx_tile* t,
                                  const mbx_simt_config* c, const mbx_pagerank_config* cfg,
                                  const void* pi0_host, void* pi_host, void* ref_host,
                                  double* history, mbx_pagerank_observer observer, void* user,
                                  mbx_pagerank_result* result) {
  return guarded([&] {
    require(observer != nullptr, MBX_CONFIG_ERROR, "observer must not be NULL");
    mbx_pagerank_plan* pl = nullptr;
    int rc = mbx_pagerank_plan_create(ctx, p, t, c, cfg, &pl);
    if (rc) fail(rc, g_last_error);
    std::unique_ptr<mbx_pagerank_plan, int (*)(mbx_pagerank_plan*)> guard(pl,
                                                                         mbx_pagerank_plan_destroy);
    Device dg(ctx->device);
    cudaStream_t st = ctx->stream;
    void* pi0 = nullptr;
    void* tmp = dmalloc(ctx, pl->n * pl->vs + 256);
    struct Bufs {  // released on every exit, the observer's abort included
      mbx_context* ctx;
      void** a;
      void** b;
      ~Bufs() {
        dfree(ctx, *a);
        dfree(ctx, *b);
        *a = *b = nullptr;
      }
    } bufs{ctx, &pi0, &tmp};
    if (pi0_host) {
      pi0 = dmalloc(ctx, pl->n * pl->vs);
      MBX_CUDA(cudaMemcpyAsync(p->vmap ? tmp : pi0, pi0_host, pl->n * pl->vs,
                               cudaMemcpyHostToDevice, st));
      if (p->vmap) mbx::launch_vertex_map(ctx, p->precision, pl->n, p->vmap, tmp, pi0, true);
    }
    plan_prologue(pl, pi0);
    std::vector<unsigned char> iterate(size_t(pl->n) * pl->vs);
    MBX_CUDA(cudaEventRecord(pl->e0, st));
    const void* yard = pl->cfg.reference_iters > 0 ? pl->ref[pl->cfg.reference_iters & 1]
                                                   : nullptr;
    for (int64_t r = 1; r <= pl->cfg.max_iters; ++r) {
      // one iteration, then the iterate and its scalars reach the host
      // (solvers.hpp:197-213: mass check, ERR, on_iteration, convergence)
      const mbx::PrArgs a = pr_args(pl, r, yard);
      mbx::launch_spmv(ctx, pl->p, pl->t, pl->g, pl->pi[(r - 1) & 1], pl->pi[r & 1],
                       pl->carry_ws, &a);
      const void* src = pl->pi[r & 1];
      if (p->vmap) {
        mbx::launch_vertex_map(ctx, p->precision, pl->n, p->vmap, src, tmp, false);
        src = tmp;
      }
      int flags[2];
      mbx::PrScalars sc;
      MBX_CUDA(cudaMemcpyAsync(iterate.data(), src, iterate.size(), cudaMemcpyDeviceToHost, st));
      MBX_CUDA(cudaMemcpyAsync(flags, pl->flags, 8, cudaMemcpyDeviceToHost, st));
      MBX_CUDA(cudaMemcpyAsync(&sc, pl->scal + r, sizeof(sc), cudaMemcpyDeviceToHost, st));
      MBX_CUDA(cudaStreamSynchronize(st));
      if (flags[0] == 2) break;  // zero-norm iterate: reported by plan_result, no callback
      if (observer(r, iterate.data(), sc.err, user) != 0)
        fail(MBX_ERROR, "pagerank: aborted by the on_iteration observer at iteration " +
                            std::to_string(r));
      if (flags[0] == 1) break;
    }
    MBX_CUDA(cudaEventRecord(pl->e1, st));
    pl->ran = true;
    rc = mbx_pagerank_plan_result(pl, result, history);
    if (rc) fail(rc, g_last_error);
    auto download = [&](void* host, const void* dev) {
      const void* s2 = dev;
      if (p->vmap) {
        mbx::launch_vertex_map(ctx, p->precision, pl->n, p->vmap, dev, tmp, false);
        s2 = tmp;
      }
      MBX_CUDA(cudaMemcpyAsync(host, s2, pl->n * pl->vs, cudaMemcpyDeviceToHost, st));
      MBX_CUDA(cudaStreamSynchronize(st));
    };
    if (pi_host) download(pi_host, pl->pi[result->iterations & 1]);
    if (ref_host) {
      if (cfg->reference_iters > 0) {
        download(ref_host, pl->ref[cfg->reference_iters & 1]);
      } else if (p->precision == MBX_F32) {
        float* r = static_cast<float*>(ref_host);
        for (int64_t i = 0; i < pl->n; ++i) r[i] = 1.0f / float(pl->n);
      } else {
        double* r = static_cast<double*>(ref_host);
        for (int64_t i = 0; i < pl->n; ++i) r[i] = 1.0 / double(pl->n);
      }
    }
    MBX_CUDA(cudaStreamSynchronize(st));
  });
}

MBX_API int mbx_context_release_cache(mbx_context* ctx) {
  return guarded([&] {
    Device dg(ctx->device);
    drop_pr_cache(ctx);
  });
}

}  // extern "C"
