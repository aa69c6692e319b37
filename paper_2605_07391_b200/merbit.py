"""Host-side mirror of the reference API for the MERBIT path, over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/merbit (the C++ mirror for C++ callers is
include/merbit_b200/merbit.hpp).  Every compute call goes through
libmerbit_b200.so on the GPU; nothing here computes on the CPU.

    SimtConfig.make / select_sigma          config.hpp:18-42, src/config.cpp
    generate_tile -> Tile (TileMetadata)    tile.hpp:27-58, src/tile.cpp:17-85
    spmv_merbit(.., DualBuffer, trace)      merbit_spmv.hpp:136-352
    SpmvBackend / MerbitB200Backend         backend.hpp:22-34, 112-136
    make_backend / BackendKind              backend.hpp:138-169
    pagerank -> PageRankResult              solvers.hpp:76-218
    bicgstab -> BicgstabResult              solvers.hpp:224-373
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import time

import numpy as np

from . import _lib
from ._lib import (mbx_bicgstab_config, mbx_bicgstab_result, mbx_pagerank_config,
                   mbx_pagerank_result, mbx_simt_config, mbx_spmv_trace, mbx_tile_info)

F32, F64 = 0, 1


# ---------------------------------------------------------------------------
# error taxonomy (include/merbit/types.hpp:23-65)
# ---------------------------------------------------------------------------
class MerbitError(RuntimeError):
    code = 1


class IoError(MerbitError):
    code = 2


class ParseError(MerbitError):
    code = 3


class ConfigError(MerbitError):
    code = 4


class DimensionError(MerbitError):
    code = 5


class CapacityError(MerbitError):
    code = 6


class CorruptionError(MerbitError):
    code = 7


class CudaError(MerbitError):
    code = 8


class NcclError(MerbitError):
    code = 9


class UnsupportedError(MerbitError):
    code = 10


_ERRORS = {c.code: c for c in (MerbitError, IoError, ParseError, ConfigError, DimensionError,
                                CapacityError, CorruptionError, CudaError, NcclError,
                                UnsupportedError)}


def _check(rc):
    if rc != 0:
        msg = _lib.lib().mbx_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, MerbitError)(msg)


def _precision_of(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return F32
    if dt == np.float64:
        return F64
    raise ConfigError(f"unsupported value dtype {dt}")


def _dtype_of(precision: int):
    return np.float32 if precision == F32 else np.float64


def _ptr(a):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------------------
# SimtConfig (config.hpp:18-42)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SimtConfig:
    omega: int = 32
    sigma: int = 14
    block_size: int = 128
    offset_bits: int = 9

    @staticmethod
    def make(omega: int, sigma: int, block_size: int) -> "SimtConfig":
        c = mbx_simt_config()
        _check(_lib.lib().mbx_config_make(omega, sigma, block_size, C.byref(c)))
        return SimtConfig(c.omega, c.sigma, c.block_size, c.offset_bits)

    def warps_per_block(self) -> int:
        return self.block_size // self.omega

    def steps_per_tile(self) -> int:
        return self.omega * self.sigma

    def steps_per_block(self) -> int:
        return self.block_size * self.sigma

    def _c(self) -> mbx_simt_config:
        return mbx_simt_config(self.omega, self.sigma, self.block_size, self.offset_bits)


def select_sigma(precision: str, override: int | None = None) -> int:
    return _lib.lib().mbx_select_sigma(1 if precision == "f64" else 0, override or 0)


def tile_counts(nnz: int, n_rows: int, c: SimtConfig):
    t, l = C.c_int64(), C.c_int64()
    cc = c._c()
    _check(_lib.lib().mbx_tile_counts(nnz, n_rows, C.byref(cc), C.byref(t), C.byref(l)))
    return t.value, l.value


def metadata_footprint(nnz: int, n_rows: int, c: SimtConfig, r_f: float) -> float:
    cc = c._c()
    return _lib.lib().mbx_metadata_footprint(nnz, n_rows, C.byref(cc), r_f)


def merge_search(row_offsets, n_rows: int, nnz: int, diag: int):
    ro = np.ascontiguousarray(row_offsets, np.int64)
    x, y = C.c_int64(), C.c_int64()
    _check(_lib.lib().mbx_merge_search(_ptr(ro), n_rows, nnz, diag, C.byref(x), C.byref(y)))
    return x.value, y.value


# Cost of one row's PageRank commit in nonzeros: least-squares fit of per-shard
# K2 times at R-MAT s24 over 32 shards (t ~ 3.2 ns/nnz + 10.9 ns/row + 20 us).
PAGERANK_ROW_WEIGHT = 3.4


def pagerank_row_weight(n_vertices: int, value_bytes: int = 4) -> float:
    """Row weight for plan_row_shards.  Once pi no longer sits in L2 (s27:
    512 MB) each gathered nonzero costs more relative to a row's commit; with
    round 2's store-only commit and the K2 shared-memory budget that shrinks
    with x, the measured best cut at s27 is 2.5 (slowest of 8 shards 1.186 ms
    vs 1.245 at 2.0, 1.215 at 3.0, 1.452 at 1.5; profiles/r2_shard_recut.json);
    at s24 (64 MB of pi) 3.4."""
    return PAGERANK_ROW_WEIGHT if n_vertices * value_bytes <= (96 << 20) else 2.5


def plan_row_shards(row_offsets, n_rows: int, nnz: int, parts: int,
                    row_weight: float = 1.0) -> np.ndarray:
    """Row bounds of `parts` shards.  row_weight 1.0 is the merge-path cut
    (mbx_plan_row_shards); other weights cut ro[r] + row_weight * r evenly."""
    ro = np.ascontiguousarray(row_offsets, np.int64)
    out = np.zeros(parts + 1, np.int64)
    _check(_lib.lib().mbx_plan_row_shards_weighted(_ptr(ro), n_rows, nnz, parts,
                                                   float(row_weight), _ptr(out)))
    return out


# ---------------------------------------------------------------------------
# context / matrices
# ---------------------------------------------------------------------------
def device_count() -> int:
    n = C.c_int()
    _check(_lib.lib().mbx_device_count(C.byref(n)))
    return n.value


class Context:
    """One device + one stream (not thread-safe, like the reference backends)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        _check(_lib.lib().mbx_context_create(device, C.byref(h)))
        self.h = h

    def set_stream(self, stream_ptr: int | None):
        _check(_lib.lib().mbx_context_set_stream(self.h, stream_ptr))

    def release_cache(self):
        """Free the plan pagerank() keeps between calls."""
        _check(_lib.lib().mbx_context_release_cache(self.h))

    @property
    def stream(self) -> int:
        return _lib.lib().mbx_context_stream(self.h) or 0

    def synchronize(self):
        _check(_lib.lib().mbx_context_synchronize(self.h))

    def set_tuning(self, warps_per_cta: int = 0, ctas_per_sm: int = 0, max_hubs: int = -1,
                   smem_per_sm: int | None = None, prefetch: int | None = None):
        """K2 launch shape (persistent grid; 0, 0: automatic -- 32 x 1, or 16 x 2
        for a small matrix without a hub table), x hub-cache cap (-1 automatic, 0 off,
        > 0 a cap that also forces a table on small matrices),
        shared-memory budget per SM and the next tile's staging (0 none,
        1 L2 prefetch, 2 TMA bulk copy into shared memory, -1 auto)."""
        _check(_lib.lib().mbx_context_set_tuning(self.h, warps_per_cta, ctas_per_sm, max_hubs))
        if smem_per_sm is not None or prefetch is not None:
            _check(_lib.lib().mbx_context_set_tuning_ex(
                self.h, -1 if smem_per_sm is None else smem_per_sm,
                -1 if prefetch is None else prefetch))

    def set_layout(self, layout: int):
        """K2 data layout: 1 lane-major slots (default), 0 staged CSR order."""
        _check(_lib.lib().mbx_context_set_layout(self.h, layout))

    @property
    def launch_count(self) -> int:
        return _lib.lib().mbx_context_launch_count(self.h)

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().mbx_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


@dataclass
class DegreeStats:
    """DegreeStats (include/merbit/csr.hpp:108-113)."""
    mean_degree: float
    low_degree: bool
    max_degree: int
    empty_rows: int


class DeviceMatrix:
    """A CsrMatrix<T> (csr.hpp:29-38) resident on the device."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle
        p, nr, nc, nnz = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.lib().mbx_matrix_info(self.h, C.byref(p), C.byref(nr), C.byref(nc),
                                          C.byref(nnz)))
        self.precision, self.n_rows, self.n_cols, self.nnz = p.value, nr.value, nc.value, nnz.value

    @property
    def dtype(self):
        return _dtype_of(self.precision)

    @classmethod
    def upload(cls, ctx: Context, n_rows, n_cols, row_offsets, col_indices, values):
        ro = np.ascontiguousarray(row_offsets, np.int64)
        vals = np.ascontiguousarray(values)
        prec = _precision_of(vals.dtype)
        h = C.c_void_p()
        cols = np.asarray(col_indices)
        if cols.dtype == np.int64:
            cols = np.ascontiguousarray(cols)
            _check(_lib.lib().mbx_matrix_upload(ctx.h, prec, n_rows, n_cols, _ptr(ro), _ptr(cols),
                                                _ptr(vals), C.byref(h)))
        else:
            cols = np.ascontiguousarray(cols, np.int32)
            _check(_lib.lib().mbx_matrix_upload_i32(ctx.h, prec, n_rows, n_cols, _ptr(ro),
                                                    _ptr(cols), _ptr(vals), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_csr(cls, ctx: Context, a):
        """`a` has n_rows, n_cols, row_offsets, col_indices, values (e.g. oracle.Csr)."""
        return cls.upload(ctx, a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values)

    @classmethod
    def rmat(cls, ctx: Context, scale: int, edge_factor: int = 16, seed: int = 1,
             transition: bool = False, dtype=np.float32, value_seed: int = 2,
             lo: float = 0.0, hi: float = 1.0):
        h = C.c_void_p()
        _check(_lib.lib().mbx_matrix_generate_rmat(ctx.h, _precision_of(dtype), scale,
                                                   edge_factor, seed, 1 if transition else 0,
                                                   value_seed, lo, hi, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def stencil27(cls, ctx: Context, grid_dim: int, dtype=np.float32):
        """BASELINE C5: 27-point stencil on a grid_dim^3 grid."""
        h = C.c_void_p()
        _check(_lib.lib().mbx_matrix_generate_stencil27(ctx.h, _precision_of(dtype), grid_dim,
                                                        C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def powerlaw(cls, ctx: Context, log2_rows: int, seed: int = 3, dtype=np.float64):
        """BASELINE C3: power-law rows with long rows and exactly 10% empty rows."""
        h = C.c_void_p()
        _check(_lib.lib().mbx_matrix_generate_powerlaw(ctx.h, _precision_of(dtype), log2_rows,
                                                       seed, C.byref(h)))
        return cls(ctx, h)

    def download(self, want_values=True):
        ro = np.zeros(self.n_rows + 1, np.int64)
        cols = np.zeros(max(self.nnz, 1), np.int32)
        vals = np.zeros(max(self.nnz, 1), self.dtype) if want_values else None
        _check(_lib.lib().mbx_matrix_download(self.h, _ptr(ro), _ptr(cols), _ptr(vals)))
        return ro, cols[:self.nnz], (vals[:self.nnz] if want_values else None)

    def row_offsets(self):
        """Only the row offsets (int64[n_rows + 1]) on the host: no column or
        value bytes cross the bus (row-shard planning at scale 27 would
        otherwise copy 8.5 GB of columns per rank)."""
        ro = np.zeros(self.n_rows + 1, np.int64)
        _check(_lib.lib().mbx_matrix_download(self.h, _ptr(ro), None, None))
        return ro

    def compact(self, tile: "Tile"):
        """Free the CSR values / columns once the slot copy for `tile`
        exists; they are rebuilt from it when a later call needs them."""
        _check(_lib.lib().mbx_matrix_compact(self.h, tile.h))

    def resident_bytes(self) -> int:
        b = C.c_int64()
        _check(_lib.lib().mbx_matrix_resident_bytes(self.h, C.byref(b)))
        return b.value

    def release_caches(self):
        """Free the slot copy, x hub cache and COO rows (CSR kept)."""
        _check(_lib.lib().mbx_matrix_release_caches(self.h))

    def build_xcache(self, max_hubs: int = -1) -> float:
        """Rank columns by reference count and stage the hottest x entries in
        shared memory during SpMV (results bitwise unchanged).  max_hubs < 0:
        automatic (no table below 4096 nonzeros per resident K2 warp, where
        it does not pay); > 0: at most that many whatever the size; 0: none.
        Returns seconds."""
        secs = C.c_double()
        _check(_lib.lib().mbx_matrix_build_xcache(self.ctx.h, self.h, max_hubs, C.byref(secs)))
        return secs.value

    def xcache_info(self):
        hubs, cov = C.c_int(), C.c_double()
        _check(_lib.lib().mbx_matrix_xcache_info(self.h, C.byref(hubs), C.byref(cov)))
        return hubs.value, cov.value

    def gather_sectors(self) -> float:
        """Distinct 32-byte x sectors per 32 consecutive nonzeros, from the
        last build_xcache's sample (-1: not sampled)."""
        v = C.c_double()
        _check(_lib.lib().mbx_matrix_gather_profile(self.h, C.byref(v)))
        return v.value

    def hub_columns(self) -> np.ndarray:
        """The x hub cache's columns in slot order (ascending ids)."""
        h = self.xcache_info()[0]
        out = np.zeros(max(h, 1), np.int32)
        _check(_lib.lib().mbx_matrix_hub_columns(self.h, out.ctypes.data))
        return out[:h]

    def build_transition(self) -> "DeviceMatrix":
        """build_transition (solvers.hpp:36-74) on the device: P = A^T D^-1 of
        this adjacency pattern, in this matrix's precision."""
        h = C.c_void_p()
        _check(_lib.lib().mbx_matrix_build_transition(self.ctx.h, self.h, C.byref(h)))
        return DeviceMatrix(self.ctx, h)

    def degree_stats(self, sigma_threshold: int):
        """DegreeStats (csr.hpp:108-140) of the resident matrix."""
        d = _lib.mbx_degree_stats()
        _check(_lib.lib().mbx_matrix_degree_stats(self.ctx.h, self.h, int(sigma_threshold),
                                                  C.byref(d)))
        return DegreeStats(d.mean_degree, bool(d.low_degree), d.max_degree, d.empty_rows)

    def relabel_by_degree(self, want_rank: bool = True):
        """(P', rank): the symmetric degree relabelling P' = Q P Q^T on the
        device (vertex v -> rank[v], by descending column count) -- a locality
        preprocessing for graphs whose x exceeds L2.  rank is None when not
        wanted (the matrix keeps its vertex map either way)."""
        h = C.c_void_p()
        rank = np.zeros(max(self.n_rows, 1), np.int32) if want_rank else None
        _check(_lib.lib().mbx_matrix_relabel_by_degree(
            self.ctx.h, self.h, C.byref(h), None if rank is None else rank.ctypes.data))
        return DeviceMatrix(self.ctx, h), (None if rank is None else rank[:self.n_rows])

    def slot_info(self):
        """(slots, build seconds) of the lane-major slot copy cached on this
        matrix (built by the first SpMV / PageRank plan per TILE)."""
        n, sec = C.c_int64(), C.c_double()
        _check(_lib.lib().mbx_matrix_slot_info(self.h, C.byref(n), C.byref(sec)))
        return n.value, sec.value

    def device_ptrs(self):
        v, c, r = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(_lib.lib().mbx_matrix_device_ptrs(self.h, C.byref(v), C.byref(c), C.byref(r)))
        return v.value, c.value, r.value

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().mbx_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# TILE (tile.hpp:27-58)
# ---------------------------------------------------------------------------
class Tile:
    """Device-resident TileMetadata."""

    kLongRowMask = 0x80000000

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle
        info = mbx_tile_info()
        _check(_lib.lib().mbx_tile_get_info(self.h, C.byref(info)))
        self.omega, self.sigma = info.omega, info.sigma
        self.n_rows, self.nnz = info.n_rows, info.nnz
        self.tile_num, self.lane_num = info.tile_num, info.lane_num
        self.preprocess_seconds = info.preprocess_seconds

    def download(self):
        tx = np.zeros(self.tile_num + 1, np.uint32)
        ty = np.zeros(self.tile_num + 1, np.uint32)
        ld = np.zeros(max(self.lane_num, 1), np.uint32)
        _check(_lib.lib().mbx_tile_download(self.h, _ptr(tx), _ptr(ty), _ptr(ld)))
        return tx, ty, ld[:self.lane_num]

    @classmethod
    def upload(cls, ctx: Context, omega, sigma, n_rows, nnz, tile_x, tile_y, lane_desc):
        info = mbx_tile_info(omega, sigma, n_rows, nnz, 0, 0, 0.0)
        h = C.c_void_p()
        tx = np.ascontiguousarray(tile_x, np.uint32)
        ty = np.ascontiguousarray(tile_y, np.uint32)
        ld = np.ascontiguousarray(lane_desc, np.uint32)
        if ld.size == 0:
            ld = np.zeros(1, np.uint32)
        _check(_lib.lib().mbx_tile_upload(ctx.h, C.byref(info), _ptr(tx), _ptr(ty), _ptr(ld),
                                          C.byref(h)))
        return cls(ctx, h)

    def long_row_fraction(self) -> float:
        """tile.cpp:135-144"""
        if self.tile_num == 0:
            return 0.0
        _, ty, _ = self.download()
        return float(np.count_nonzero(ty[:-1] & self.kLongRowMask)) / self.tile_num

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().mbx_tile_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def generate_tile(row_offsets, n_rows: int, nnz: int, c: SimtConfig,
                  ctx: Context | None = None) -> Tile:
    """generate_tile(span row_offsets, n_rows, nnz, c) on the GPU (tile.cpp:17-85)."""
    ctx = ctx or default_context()
    cc = c._c()
    h = C.c_void_p()
    ro = None if row_offsets is None else np.ascontiguousarray(row_offsets, np.int64)
    _check(_lib.lib().mbx_generate_tile(ctx.h, _ptr(ro), n_rows, nnz, C.byref(cc), C.byref(h)))
    return Tile(ctx, h)


def generate_tile_for(m: DeviceMatrix, c: SimtConfig) -> Tile:
    """generate_tile(const CsrMatrix&, c) from the resident matrix (tile.hpp:54-58)."""
    cc = c._c()
    h = C.c_void_p()
    _check(_lib.lib().mbx_matrix_generate_tile(m.ctx.h, m.h, C.byref(cc), C.byref(h)))
    return Tile(m.ctx, h)


# ---------------------------------------------------------------------------
# SpMV (merbit_spmv.hpp)
# ---------------------------------------------------------------------------
@dataclass
class SpmvTrace:
    """merbit_spmv.hpp:21-28: tile-routing counters and, with
    collect_deposits, every (row, partial sum) contribution of the MERBIT
    decomposition (mbx_spmv_deposits; unordered, rows in the caller's
    vertex order)."""
    collect_deposits: bool = False
    fast_tiles: int = 0
    normal_tiles: int = 0
    skipped_tiles: int = 0
    deposits: list = field(default_factory=list)


class DualBuffer:
    """Host ping-pong output pair with the reference contract (dual_buffer.hpp:9-42):
    after a multiply, last_output() holds the result and active() is all zeros."""

    def __init__(self, n: int, dtype=np.float64):
        self._bufs = [np.zeros(n, dtype), np.zeros(n, dtype)]
        self._parity = 0

    def size(self):
        return self._bufs[0].size

    def parity(self):
        return self._parity

    def active(self):
        return self._bufs[self._parity]

    def inactive(self):
        return self._bufs[self._parity ^ 1]

    def last_output(self):
        return self._bufs[self._parity ^ 1]

    def flip(self):
        self._parity ^= 1


def spmv_merbit(m: DeviceMatrix, t: Tile, c: SimtConfig, x, out: DualBuffer,
                trace: SpmvTrace | None = None):
    """y = A x into out.active(); companion zeroed; parity flipped."""
    xv = np.ascontiguousarray(x, m.dtype)
    if xv.size != m.n_cols:
        raise DimensionError(f"spmv: x has {xv.size} entries, matrix has {m.n_cols} columns")
    if out.size() != m.n_rows:
        raise DimensionError(f"spmv: output pair sized {out.size()} for {m.n_rows} rows")
    y = out.active()
    if y.dtype != m.dtype:
        raise ConfigError("DualBuffer dtype does not match the matrix precision")
    cc = c._c()
    tr = mbx_spmv_trace() if trace is not None else None
    _check(_lib.lib().mbx_spmv(m.ctx.h, m.h, t.h, C.byref(cc), _ptr(xv) if xv.size else None,
                               _ptr(y) if y.size else None,
                               C.byref(tr) if tr is not None else None))
    out.inactive()[:] = 0
    out.flip()
    if trace is not None:
        trace.fast_tiles += tr.fast_tiles
        trace.normal_tiles += tr.normal_tiles
        trace.skipped_tiles += tr.skipped_tiles
        if trace.collect_deposits:
            L = _lib.lib()
            cap = C.c_int64()
            _check(L.mbx_spmv_deposits(m.ctx.h, m.h, t.h, C.byref(cc), None, None, None, 0,
                                       C.byref(cap)))
            rows = np.zeros(max(cap.value, 1), np.int64)
            amounts = np.zeros(max(cap.value, 1), m.dtype)
            got = C.c_int64()
            _check(L.mbx_spmv_deposits(m.ctx.h, m.h, t.h, C.byref(cc),
                                       _ptr(xv) if xv.size else None, _ptr(rows),
                                       _ptr(amounts), cap.value, C.byref(got)))
            k = min(got.value, cap.value)
            trace.deposits.extend(zip(rows[:k].tolist(), amounts[:k].tolist()))
    return out.last_output()


def spmv_device(m: DeviceMatrix, t: Tile, c: SimtConfig, x_ptr: int, y_ptr: int):
    cc = c._c()
    _check(_lib.lib().mbx_spmv_device(m.ctx.h, m.h, t.h, C.byref(cc), x_ptr, y_ptr))


BASELINE_KINDS = {"csr_vector": 0, "coo_atomic": 1, "merge_runtime": 2, "merge_cub": 3,
                  "cusparse_coo_alg1": 4, "cusparse_coo_alg2": 5, "cusparse_csr_alg1": 6,
                  "cusparse_csr_alg2": 7}


def spmv_baseline_device(m: DeviceMatrix, kind: str, x_ptr: int, y_ptr: int, sigma: int = 0):
    """The paper's comparators on the GPU (csr_vector, coo_atomic,
    merge_runtime with `sigma`, merge_cub, cuSPARSE COO/CSR ALG1/ALG2);
    device pointers in and out."""
    if sigma <= 0:
        sigma = 14 if m.dtype == np.float32 else 7
    _check(_lib.lib().mbx_spmv_baseline_device(m.ctx.h, m.h, BASELINE_KINDS[kind], sigma,
                                               x_ptr, y_ptr))


def trace_counts(t: Tile) -> SpmvTrace:
    tr = mbx_spmv_trace()
    _check(_lib.lib().mbx_spmv_trace_counts(t.ctx.h, t.h, C.byref(tr)))
    return SpmvTrace(False, tr.fast_tiles, tr.normal_tiles, tr.skipped_tiles)


# ---------------------------------------------------------------------------
# backends (backend.hpp)
# ---------------------------------------------------------------------------
class BackendKind(enum.Enum):
    merbit_b200 = "merbit-b200"


class SpmvBackend:
    """backend.hpp:22-34"""

    def apply(self, x):
        raise NotImplementedError

    def name(self) -> str:
        raise NotImplementedError

    def preprocess_seconds(self) -> float:
        return self._preprocess_seconds


class MerbitB200Backend(SpmvBackend):
    """MerbitBackend (backend.hpp:112-136) on the GPU: the constructor uploads
    the CSR once and builds the TILE and the x hub cache (T_p = their device
    time); apply() returns an internal buffer valid until the next apply()."""

    def __init__(self, a, c: SimtConfig, ctx: Context | None = None, xcache: bool = True):
        self.ctx = ctx or default_context()
        self.c = c
        self.matrix = DeviceMatrix.from_csr(self.ctx, a)
        self.tile_ = generate_tile_for(self.matrix, c)
        xc = self.matrix.build_xcache() if xcache else 0.0
        self._preprocess_seconds = self.tile_.preprocess_seconds + xc
        self.buffer = DualBuffer(self.matrix.n_rows, self.matrix.dtype)

    def apply(self, x):
        return spmv_merbit(self.matrix, self.tile_, self.c, x, self.buffer)

    def name(self):
        return "merbit-b200"

    def tile(self):
        return self.tile_


def make_backend(kind: BackendKind, a, c: SimtConfig, ctx: Context | None = None):
    """make_backend (backend.hpp:152-169) for the GPU kind."""
    if kind is BackendKind.merbit_b200:
        return MerbitB200Backend(a, c, ctx)
    raise ConfigError("unknown backend kind")


# ---------------------------------------------------------------------------
# PageRank (solvers.hpp:76-218)
# ---------------------------------------------------------------------------
@dataclass
class PageRankConfig:
    damping: float = 0.85
    err_tol: float = 1e-10
    max_iters: int = 210
    reference_iters: int = 210

    def _c(self):
        return mbx_pagerank_config(self.damping, self.err_tol, self.max_iters,
                                   self.reference_iters)


@dataclass
class PageRankResult:
    pi: np.ndarray
    reference_pi: np.ndarray | None
    iterations: int
    final_err: float
    status: str
    preprocess_seconds: float
    iterate_seconds: float
    l1_residual: float = 0.0
    mass: float = 0.0
    dangling_mass: float = 0.0
    residual_history: np.ndarray | None = None


def pagerank(p, cfg: PageRankConfig, backend: MerbitB200Backend | None = None,
             c: SimtConfig | None = None, pi0=None, on_iteration=None) -> PageRankResult:
    """pagerank<T>(p, cfg, backend, on_iteration): the power loop runs fused on
    the device.

    `p` is the transition matrix (host CSR) when `backend` is None; otherwise the
    backend's resident matrix and TILE are used.  on_iteration(r, pi, err), when
    given, observes every iterate (solvers.hpp:157-158, 209) -- the loop then
    runs iteration by iteration with a host copy of each iterate."""
    if backend is None:
        dt = np.asarray(p.values).dtype
        c = c or SimtConfig.make(32, select_sigma("f64" if dt == np.float64 else "f32"), 128)
        backend = MerbitB200Backend(p, c)
    m, t, c = backend.matrix, backend.tile_, backend.c
    pi = np.zeros(m.n_rows, m.dtype)
    ref = np.zeros(m.n_rows, m.dtype)
    hist = np.zeros(max(cfg.max_iters, 1), np.float64)
    res = mbx_pagerank_result()
    cc, pc = c._c(), cfg._c()
    p0 = None if pi0 is None else np.ascontiguousarray(pi0, m.dtype)
    if on_iteration is None:
        _check(_lib.lib().mbx_pagerank(m.ctx.h, m.h, t.h, C.byref(cc), C.byref(pc), _ptr(p0),
                                       _ptr(pi), _ptr(ref), _ptr(hist), C.byref(res)))
    else:
        n, dt = m.n_rows, m.dtype
        failure = []

        def trampoline(r, pi_host, err, _user):
            try:
                it = np.ctypeslib.as_array(C.cast(pi_host, C.POINTER(
                    C.c_float if dt == np.float32 else C.c_double)), shape=(n,))
                on_iteration(int(r), it.copy(), float(err))
                return 0
            except BaseException as e:  # stops the run; re-raised after the C call
                failure.append(e)
                return 1
        cb = _lib.PAGERANK_OBSERVER(trampoline)
        rc = _lib.lib().mbx_pagerank_observed(m.ctx.h, m.h, t.h, C.byref(cc), C.byref(pc),
                                              _ptr(p0), _ptr(pi), _ptr(ref), _ptr(hist), cb,
                                              None, C.byref(res))
        if failure:
            raise failure[0]
        _check(rc)
    return PageRankResult(pi=pi, reference_pi=ref, iterations=res.iterations,
                          final_err=res.final_err,
                          status="converged" if res.status == 0 else "max_iterations",
                          preprocess_seconds=res.preprocess_seconds,
                          iterate_seconds=res.iterate_seconds, l1_residual=res.l1_residual,
                          mass=res.mass, dangling_mass=res.dangling_mass,
                          residual_history=hist[:res.iterations])


# ---------------------------------------------------------------------------
# BiCGSTAB (solvers.hpp:224-373)
# ---------------------------------------------------------------------------
_SOLVE_STATUS = {0: "converged", 1: "max_iterations", 2: "breakdown"}


def solve_status_name(status: str) -> str:
    """solve_status_name (solvers.hpp): the status strings are the names."""
    return status


@dataclass
class BicgstabConfig:
    tol: float = 1e-10
    max_iters: int = 20000

    def _c(self):
        return mbx_bicgstab_config(self.tol, self.max_iters)


@dataclass
class BicgstabResult:
    x: np.ndarray
    residual_history: np.ndarray
    iterations: int
    final_residual: float
    status: str
    breakdown_reason: str
    preprocess_seconds: float
    iterate_seconds: float


def bicgstab(a, b, cfg: BicgstabConfig | None = None,
             backend: MerbitB200Backend | None = None) -> BicgstabResult:
    """bicgstab<T>(a, b, cfg, backend): unpreconditioned BiCGSTAB with every
    SpMV, inner product and vector update on the device (K2/K3 + fused
    dot/axpy kernels).  `a` is the host CSR when `backend` is None."""
    cfg = cfg or BicgstabConfig()
    if backend is None:
        dt = np.asarray(a.values).dtype
        c = SimtConfig.make(32, select_sigma("f64" if dt == np.float64 else "f32"), 128)
        backend = MerbitB200Backend(a, c)
    m, t, c = backend.matrix, backend.tile_, backend.c
    if m.n_rows != m.n_cols:
        raise DimensionError("bicgstab needs a square system")
    b = np.ascontiguousarray(b, m.dtype)
    if b.shape != (m.n_rows,):
        raise DimensionError(f"bicgstab: right-hand side has {b.size} entries for "
                             f"{m.n_rows} rows")
    x = np.zeros(m.n_rows, m.dtype)
    hist = np.zeros(max(cfg.max_iters, 1), np.float64)
    res = mbx_bicgstab_result()
    cc, bc = c._c(), cfg._c()
    _check(_lib.lib().mbx_bicgstab(m.ctx.h, m.h, t.h, C.byref(cc), C.byref(bc), _ptr(b), _ptr(x),
                                   hist.ctypes.data_as(C.POINTER(C.c_double)), C.byref(res)))
    reason = res.breakdown_reason.decode()
    hl = res.iterations - (1 if res.status == 2 and reason != "diverged" else 0)
    return BicgstabResult(x=x, residual_history=hist[:hl].copy(),
                          iterations=res.iterations, final_residual=res.final_residual,
                          status=_SOLVE_STATUS[res.status],
                          breakdown_reason=reason,
                          preprocess_seconds=res.preprocess_seconds,
                          iterate_seconds=res.iterate_seconds)


class PageRankPlan:
    """Device-resident reusable power loop (buffers + CUDA graph built once)."""

    def __init__(self, m: DeviceMatrix, t: Tile, c: SimtConfig, cfg: PageRankConfig):
        self.m, self.t, self.c, self.cfg = m, t, c, cfg
        h = C.c_void_p()
        cc, pc = c._c(), cfg._c()
        _check(_lib.lib().mbx_pagerank_plan_create(m.ctx.h, m.h, t.h, C.byref(cc), C.byref(pc),
                                                   C.byref(h)))
        self.h = h

    def run(self, pi0_ptr: int | None = None):
        _check(_lib.lib().mbx_pagerank_plan_run(self.h, pi0_ptr))

    def result(self, want_history=False):
        res = mbx_pagerank_result()
        hist = np.zeros(max(self.cfg.max_iters, 1), np.float64) if want_history else None
        _check(_lib.lib().mbx_pagerank_plan_result(self.h, C.byref(res), _ptr(hist)))
        return res, hist

    def pi_ptr(self) -> int:
        return _lib.lib().mbx_pagerank_plan_pi(self.h) or 0

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().mbx_pagerank_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# multi-GPU row shards (shard.cu)
# ---------------------------------------------------------------------------
def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.lib().mbx_nccl_unique_id(buf))
    return buf.raw


def row_slice(m: DeviceMatrix, r0: int, r1: int) -> DeviceMatrix:
    h = C.c_void_p()
    _check(_lib.lib().mbx_matrix_row_slice(m.ctx.h, m.h, r0, r1, C.byref(h)))
    return DeviceMatrix(m.ctx, h)


def recut_row_shards(row_offsets, bounds, shard_times, row_weight: float) -> np.ndarray:
    """Re-cut row shards from measured per-shard times: shard i's time is
    spread over its rows in proportion to the cut's cost (nnz + row_weight *
    rows), and the resulting cumulative-time curve is cut into equal parts.
    With the shards' own measured times one round took the slowest of 8 s27
    shards from 1.53 to 1.35 ms (mean 1.34) under a fixed 160 KB hub budget;
    bench.py --recut feeds it shard_cost_probe times instead, which track the
    group's cost less well since the budget depends on x
    (profiles/r2_shard_recut.json)."""
    ro = np.ascontiguousarray(row_offsets, np.int64)
    b = np.ascontiguousarray(bounds, np.int64)
    t = np.asarray(shard_times, np.float64)
    parts, n = len(t), int(b[-1])
    if parts != len(b) - 1 or parts < 2 or np.any(t <= 0):
        return b.copy()
    tcum = np.concatenate([[0.0], np.cumsum(t)])
    out = np.zeros(parts + 1, np.int64)
    out[-1] = n
    for k in range(1, parts):
        target = tcum[-1] * k / parts
        i = min(int(np.searchsorted(tcum, target, side="right")) - 1, parts - 1)
        frac = (target - tcum[i]) / t[i]
        r0, r1 = int(b[i]), int(b[i + 1])
        c0 = float(ro[r0]) + row_weight * r0
        c1 = float(ro[r1]) + row_weight * r1
        goal = c0 + frac * (c1 - c0)
        # first row r in [r0, r1] with ro[r] + w*r >= goal (monotone in r)
        lo, hi = r0, r1
        while lo < hi:
            mid = (lo + hi) // 2
            if float(ro[mid]) + row_weight * mid < goal:
                lo = mid + 1
            else:
                hi = mid
        out[k] = min(max(lo, int(out[k - 1])), n)
    return out


def shard_cost_probe(L: DeviceMatrix, t: "Tile", c: SimtConfig, reps: int = 5) -> float:
    """Seconds per PageRank iteration a row shard costs, measured on its own
    GPU without its peers: one plain SpMV of the shard (K2 + K3 with its hub
    table and slot copy) plus the PageRank loop's per-row work beyond it (the
    pi stores, exchange copies and K3's reductions) as 24 bytes per row at
    copy bandwidth -- fitted on s27 8-shard cuts, where the row-heavy last
    shard ran 0.20 ms above its SpMV and the others 0.07 ms
    (profiles/r2_shard_recut.json).  What recut_row_shards balances in a
    multi-process run, where the loop itself waits on the slowest rank."""
    import torch
    dt = torch.float32 if L.dtype == np.float32 else torch.float64
    x = torch.full((L.n_cols,), 1.0 / max(L.n_cols, 1), dtype=dt, device="cuda")
    y = torch.empty(max(L.n_rows, 1), dtype=dt, device="cuda")
    L.build_xcache()
    torch.cuda.synchronize()
    for _ in range(2):
        spmv_device(L, t, c, x.data_ptr(), y.data_ptr())
    L.ctx.synchronize()
    t0 = time.perf_counter()  # the context's own stream, whichever it is
    for _ in range(reps):
        spmv_device(L, t, c, x.data_ptr(), y.data_ptr())
    L.ctx.synchronize()
    secs = (time.perf_counter() - t0) / reps
    L.release_caches()
    return secs + 24.0 * L.n_rows / 6.5e12


def prepare_rank_shard(P: DeviceMatrix, world: int, rank: int, c: SimtConfig,
                       row_weight: float | None = None):
    """One rank's preprocessing of the row-sharded PageRank (bench.py N > 1,
    the path tests/test_gpu_bench_path.py gates): the cost-weighted cut of P's
    rows (only the row offsets come to the host), this rank's row slice and
    its TILE.  Returns (bounds, local matrix, local TILE, row weight)."""
    n = P.n_rows
    w = pagerank_row_weight(n, np.dtype(P.dtype).itemsize) if row_weight is None else row_weight
    bounds = plan_row_shards(P.row_offsets(), n, P.nnz, world, w)
    L = row_slice(P, int(bounds[rank]), int(bounds[rank + 1]))
    return bounds, L, generate_tile_for(L, c), w


def recut_rank_shard(P: DeviceMatrix, bounds, shard_times, rank: int, c: SimtConfig,
                     row_weight: float):
    """The second half of bench.py's N > 1 preprocessing: every rank probes
    its first-cut shard (shard_cost_probe), the times are all-gathered, and
    each rank re-cuts identically (recut_row_shards) and rebuilds its slice
    and TILE.  Returns (bounds, local matrix, local TILE)."""
    b = recut_row_shards(P.row_offsets(), bounds, shard_times, row_weight)
    L = row_slice(P, int(b[rank]), int(b[rank + 1]))
    return b, L, generate_tile_for(L, c)


class ShardGroup:
    """Row-sharded PageRank: `shards` = [(DeviceMatrix, Tile)] owned by this
    process for ranks rank0 .. rank0+len(shards)-1 of `world`.  nccl_id None:
    all shards local, sharing one buffer (single-GPU check of the sharded
    path); otherwise one shard per process joined over NCCL.  cfg.reference_iters
    > 0 runs the reference's yardstick through the same exchange first."""

    def __init__(self, ctx: Context, n_global: int, world: int, bounds, rank0: int, shards,
                 c: SimtConfig, cfg: PageRankConfig, nccl_id: bytes | None = None):
        self.ctx, self.n, self.world, self.cfg = ctx, n_global, world, cfg
        self.keep = shards
        self.bounds = np.ascontiguousarray(bounds, np.int64)
        mats = (C.c_void_p * len(shards))(*[m.h.value for m, _ in shards])
        tiles = (C.c_void_p * len(shards))(*[t.h.value for _, t in shards])
        self.dtype = shards[0][0].dtype
        cc, pc = c._c(), cfg._c()
        idb = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
        h = C.c_void_p()
        _check(_lib.lib().mbx_shard_group_create(ctx.h, n_global, world, _ptr(self.bounds), rank0,
                                                 len(shards), mats, tiles, C.byref(cc), C.byref(pc),
                                                 idb, C.byref(h)))
        self.h = h

    def run(self, pi0_ptr: int | None = None):
        _check(_lib.lib().mbx_shard_group_run(self.h, pi0_ptr))

    def result(self, want_history=False):
        res = mbx_pagerank_result()
        hist = np.zeros(max(self.cfg.max_iters, 1), np.float64) if want_history else None
        _check(_lib.lib().mbx_shard_group_result(self.h, C.byref(res), _ptr(hist)))
        return res, hist

    def gather_pi(self):
        pi = np.zeros(self.n, self.dtype)
        _check(_lib.lib().mbx_shard_group_gather_pi(self.h, _ptr(pi)))
        return pi

    def download_local(self, host_ptr: int):
        """This process's rows of the final pi into host memory at host_ptr."""
        _check(_lib.lib().mbx_shard_group_download_local(self.h, host_ptr))

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().mbx_shard_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


SHARD_BLOB_BYTES = 512


class PeerShardGroup(ShardGroup):
    """This rank's row shard joined to its peers by the FUSED exchange: the
    PageRank commit stores pi_new straight into every peer's exchange buffer
    (CUDA IPC, NVLink P2P) and a device barrier ends each iteration -- no
    collective library on the iteration path.  Setup through any bootstrap:
        g = PeerShardGroup(...); blobs = all_gather(g.export()); g.connect(blobs)
    close() is collective (final barrier)."""

    def __init__(self, ctx: Context, n_global: int, world: int, bounds, rank: int,
                 matrix: DeviceMatrix, tile: Tile, c: SimtConfig, cfg: PageRankConfig):
        self.ctx, self.n, self.world, self.cfg = ctx, n_global, world, cfg
        self.keep = [(matrix, tile)]
        self.bounds = np.ascontiguousarray(bounds, np.int64)
        self.dtype = matrix.dtype
        cc, pc = c._c(), cfg._c()
        h = C.c_void_p()
        _check(_lib.lib().mbx_shard_group_create_peer(ctx.h, n_global, world, _ptr(self.bounds),
                                                      rank, matrix.h, tile.h, C.byref(cc),
                                                      C.byref(pc), C.byref(h)))
        self.h = h

    def export(self) -> bytes:
        b = C.create_string_buffer(SHARD_BLOB_BYTES)
        _check(_lib.lib().mbx_shard_group_export(self.h, b))
        return b.raw

    def connect(self, blobs):
        """blobs: the world's export() results in rank order."""
        allb = b"".join(blobs)
        if len(allb) != SHARD_BLOB_BYTES * self.world:
            raise ConfigError(f"connect: expected {self.world} blobs of {SHARD_BLOB_BYTES} bytes")
        buf = C.create_string_buffer(allb, len(allb))
        _check(_lib.lib().mbx_shard_group_connect(self.h, buf))

    def quiesce(self):
        """Enqueue the final barrier without waiting (close() waits)."""
        _check(_lib.lib().mbx_shard_group_quiesce(self.h))
