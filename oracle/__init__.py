"""CPU oracle for the MERBIT path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference leg may import this package, and only as the checker or the timed
CPU baseline; the product (``paper_2605_07391_b200``) never does.

Two layers, both plain CPU code:

* ``liboracle.so`` -- ``merbit_oracle.c``, a C restatement of the reference
  functions (each cites its /root/reference/proj file:line).
* ``_ref/libmerbit_ref.so`` -- the unmodified reference library compiled from
  its own sources by ``oracle/Makefile`` plus ``ref_shim.cpp`` (a C ABI over
  it).  Absent when /root/reference was never available; ``ref()`` then
  returns None.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REF_SO = os.path.join(_HERE, "_ref", "libmerbit_ref.so")
_ORACLE_SO = os.path.join(_HERE, "liboracle.so")

SHAPES = ("uniform", "power_law_rows", "banded", "single_dense_row",
          "all_empty", "mostly_empty_rows")

i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def build(with_ref: bool | None = None) -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/src")
    targets = ["liboracle.so"] + (["ref"] if with_ref else [])
    subprocess.run(["make", "-s", "-C", _HERE] + targets, check=True)


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_offsets: np.ndarray  # int64[n_rows+1]
    col_indices: np.ndarray  # int32[nnz]
    values: np.ndarray | None  # float64 or float32[nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1]) if self.n_rows >= 0 else 0

    def astype(self, dtype) -> "Csr":
        return Csr(self.n_rows, self.n_cols, self.row_offsets, self.col_indices,
                   None if self.values is None else self.values.astype(dtype))


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code} {msg}")
        self.code = code


def _check(rc, msg=""):
    if rc != 0:
        raise OracleError(rc, msg)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build(with_ref=False)
        L = C.CDLL(_ORACLE_SO)
        L.mo_config_make.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.mo_merge_search.argtypes = [i64p, C.c_int64, C.c_int64, C.c_int64,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int)]
        L.mo_sequential_path.argtypes = [i64p, C.c_int64, C.c_int64, u8p]
        L.mo_tile_counts.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.mo_generate_tile.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                       C.c_int, C.c_int, u32p, u32p, u32p]
        L.mo_reconstruct_path.argtypes = [u32p, u32p, u32p, C.c_int64, C.c_int64,
                                          C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.mo_spmv_csr_f64.argtypes = [C.c_int64, i64p, i32p, f64p, f64p, f64p,
                                      C.c_void_p, C.c_int]
        L.mo_spmv_csr_f32.argtypes = [C.c_int64, i64p, i32p, f32p, f32p, f32p]
        L.mo_spmv_csr_f32_acc64.argtypes = [C.c_int64, i64p, i32p, f32p, f32p,
                                            f64p, C.c_void_p, C.c_int]
        for name, fp in (("mo_spmv_merbit_f64", f64p), ("mo_spmv_merbit_f32", f32p)):
            getattr(L, name).argtypes = [C.c_int64, C.c_int64, i32p, fp, fp, u32p,
                                         u32p, u32p, C.c_int, C.c_int, C.c_int,
                                         C.c_int, fp, i64p]
        L.mo_build_transition_f64.argtypes = [C.c_int64, i64p, i32p, i64p, i32p, f64p]
        L.mo_build_transition_f32.argtypes = [C.c_int64, i64p, i32p, i64p, i32p, f32p]
        L.mo_pagerank_f64.argtypes = [C.c_int64, i64p, i32p, f64p, C.c_double,
                                      C.c_double, C.c_int64, C.c_int64, f64p, f64p,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int), C.c_int]
        L.mo_pagerank_f32.argtypes = [C.c_int64, i64p, i32p, f32p, C.c_float,
                                      C.c_float, C.c_int64, C.c_int64, f32p, f32p,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int)]
        for name, fp, tt in (("mo_bicgstab_f64", f64p, C.c_double),
                             ("mo_bicgstab_f32", f32p, C.c_float)):
            getattr(L, name).argtypes = [C.c_int64, i64p, i32p, fp, fp, tt, C.c_int64, fp,
                                         f64p, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.mo_free.argtypes = [C.c_void_p]
        alloc_args = [C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int32)),
                      C.POINTER(C.POINTER(C.c_double))]
        L.mo_random_matrix_csr.argtypes = [C.c_int, C.c_uint64, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64)] + alloc_args
        L.mo_ring_with_chords_csr.argtypes = [C.c_int64, C.c_int64, C.c_uint64,
                                              C.POINTER(C.c_int64)] + alloc_args
        L.mo_single_dense_row_csr.argtypes = [C.c_int64, C.c_uint64] + alloc_args
        L.mo_seed_test_vector.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64, f64p]
        L.mo_rmat_csr.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                  C.POINTER(C.c_int64), C.POINTER(C.POINTER(C.c_int64)),
                                  C.POINTER(C.POINTER(C.c_int32))]
        L.mo_hash_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, f64p]
        L.mo_hash_uniform_f32.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, f32p]
        L.mo_transition_values_f32.argtypes = [C.c_int64, C.c_int64, i32p, f32p]
        L.mo_transition_values_f64.argtypes = [C.c_int64, C.c_int64, i32p, f64p]
        _lib = L
    return _lib


def _take(ptr, n, dtype):
    """Copy a malloc'd C array into numpy and free it."""
    if n == 0:
        out = np.zeros(0, dtype)
    else:
        out = np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)
    lib().mo_free(C.cast(ptr, C.c_void_p))
    return out


# --------------------------------------------------------------------------
# restatement API
# --------------------------------------------------------------------------
def config_make(omega, sigma, block_size):
    ob = C.c_int()
    _check(lib().mo_config_make(omega, sigma, block_size, C.byref(ob)), "config")
    return ob.value


def select_sigma(precision: str, override=None):
    """src/config.cpp:40-43"""
    if override is not None:
        return int(override)
    return 14 if precision == "f32" else 7


def merge_search(ro, n_rows, nnz, diag):
    x, y, p = C.c_int64(), C.c_int64(), C.c_int()
    _check(lib().mo_merge_search(np.ascontiguousarray(ro, np.int64), n_rows, nnz,
                                 diag, C.byref(x), C.byref(y), C.byref(p)), "merge_search")
    return x.value, y.value, p.value


def sequential_path(ro, n_rows, nnz):
    out = np.zeros(nnz + n_rows, np.uint8)
    lib().mo_sequential_path(np.ascontiguousarray(ro, np.int64), n_rows, nnz, out)
    return out


def tile_counts(nnz, n_rows, omega, sigma):
    t, l = C.c_int64(), C.c_int64()
    lib().mo_tile_counts(nnz, n_rows, omega, sigma, C.byref(t), C.byref(l))
    return t.value, l.value


def generate_tile(ro, n_rows, nnz, omega, sigma):
    ob = config_make(omega, sigma, omega)
    tiles, lanes = tile_counts(nnz, n_rows, omega, sigma)
    tx = np.zeros(tiles + 1, np.uint32)
    ty = np.zeros(tiles + 1, np.uint32)
    ld = np.zeros(max(lanes, 1), np.uint32)
    ro_arr = None if ro is None else np.ascontiguousarray(ro, np.int64)
    _check(lib().mo_generate_tile(None if ro_arr is None else ro_arr.ctypes.data,
                                  n_rows, nnz, omega, sigma, ob, tx, ty, ld),
           "generate_tile")
    return tx, ty, ld[:lanes]


def reconstruct_path(tx, ty, ld, n_rows, nnz, omega, sigma):
    ob = config_make(omega, sigma, omega)
    steps = np.zeros(nnz + n_rows, np.uint8)
    ld = np.ascontiguousarray(ld, np.uint32)
    if ld.size == 0:
        ld = np.zeros(1, np.uint32)
    _check(lib().mo_reconstruct_path(np.ascontiguousarray(tx, np.uint32),
                                     np.ascontiguousarray(ty, np.uint32), ld,
                                     n_rows, nnz, omega, sigma, ob,
                                     steps.ctypes.data if steps.size else None),
           "reconstruct_path")
    return steps


def _vals_or_dummy(a):
    return a if a.size else np.zeros(1, a.dtype)


def spmv_csr_f64(a: Csr, x, nthreads=1, want_abs=False):
    """spmv_csr_reference<double> (reference.hpp:15-46)."""
    y = np.zeros(max(a.n_rows, 1), np.float64)
    ab = np.zeros(max(a.n_rows, 1), np.float64) if want_abs else None
    lib().mo_spmv_csr_f64(a.n_rows, a.row_offsets, _vals_or_dummy(a.col_indices),
                          _vals_or_dummy(a.values.astype(np.float64)),
                          _vals_or_dummy(np.ascontiguousarray(x, np.float64)), y,
                          None if ab is None else ab.ctypes.data, nthreads)
    return (y[:a.n_rows], ab[:a.n_rows]) if want_abs else y[:a.n_rows]


def spmv_csr_f32(a: Csr, x):
    """spmv_csr_reference<float>: sequential fp32 sums (information only)."""
    y = np.zeros(max(a.n_rows, 1), np.float32)
    lib().mo_spmv_csr_f32(a.n_rows, a.row_offsets, _vals_or_dummy(a.col_indices),
                          _vals_or_dummy(a.values.astype(np.float32)),
                          _vals_or_dummy(np.ascontiguousarray(x, np.float32)), y)
    return y[:a.n_rows]


def spmv_csr_f32_acc64(a: Csr, x, nthreads=1):
    """fp32 inputs, fp64 accumulation: the fp32 y gate.  Returns (y, sum|a||x|)."""
    y = np.zeros(max(a.n_rows, 1), np.float64)
    ab = np.zeros(max(a.n_rows, 1), np.float64)
    lib().mo_spmv_csr_f32_acc64(a.n_rows, a.row_offsets, _vals_or_dummy(a.col_indices),
                                _vals_or_dummy(np.ascontiguousarray(a.values, np.float32)),
                                _vals_or_dummy(np.ascontiguousarray(x, np.float32)), y,
                                ab.ctypes.data, nthreads)
    return y[:a.n_rows], ab[:a.n_rows]


def spmv_merbit(a: Csr, x, tile, omega, sigma, block_size):
    """Restated spmv_merbit<T> (merbit_spmv.hpp:136-352); returns (y, counters)."""
    tx, ty, ld = tile
    dt = a.values.dtype
    ob = config_make(omega, sigma, block_size)
    y = np.zeros(max(a.n_rows, 1), dt)
    cnt = np.zeros(3, np.int64)
    fn = lib().mo_spmv_merbit_f64 if dt == np.float64 else lib().mo_spmv_merbit_f32
    _check(fn(a.n_rows, a.nnz, _vals_or_dummy(a.col_indices), _vals_or_dummy(a.values),
              _vals_or_dummy(np.ascontiguousarray(x, dt)), np.ascontiguousarray(tx, np.uint32),
              np.ascontiguousarray(ty, np.uint32), _vals_or_dummy(np.ascontiguousarray(ld, np.uint32)),
              omega, sigma, ob, block_size, y, cnt), "spmv_merbit")
    return y[:a.n_rows], cnt


def build_transition(adj: Csr, dtype=np.float64) -> Csr:
    n = adj.n_rows
    ro = np.zeros(n + 1, np.int64)
    cols = np.zeros(max(adj.nnz, 1), np.int32)
    vals = np.zeros(max(adj.nnz, 1), dtype)
    fn = lib().mo_build_transition_f64 if dtype == np.float64 else lib().mo_build_transition_f32
    fn(n, adj.row_offsets, _vals_or_dummy(adj.col_indices), ro, cols, vals)
    return Csr(n, n, ro, cols[:adj.nnz], vals[:adj.nnz])


def pagerank(p: Csr, damping=0.85, err_tol=1e-10, max_iters=210, reference_iters=210,
             nthreads=1):
    """pagerank<T> over the csr backend (solvers.hpp:154-218) in p.values' dtype."""
    n = p.n_rows
    it, err, st = C.c_int64(), C.c_double(), C.c_int()
    if p.values.dtype == np.float64:
        pi = np.zeros(n, np.float64)
        star = np.zeros(n, np.float64)
        rc = lib().mo_pagerank_f64(n, p.row_offsets, _vals_or_dummy(p.col_indices),
                                   _vals_or_dummy(p.values), damping, err_tol, max_iters,
                                   reference_iters, pi, star, C.byref(it), C.byref(err),
                                   C.byref(st), nthreads)
    else:
        pi = np.zeros(n, np.float32)
        star = np.zeros(n, np.float32)
        rc = lib().mo_pagerank_f32(n, p.row_offsets, _vals_or_dummy(p.col_indices),
                                   _vals_or_dummy(p.values), damping, err_tol, max_iters,
                                   reference_iters, pi, star, C.byref(it), C.byref(err),
                                   C.byref(st))
    _check(rc, "pagerank")
    return dict(pi=pi, reference_pi=star, iterations=it.value, final_err=err.value,
                status="converged" if st.value == 0 else "max_iterations")


_SOLVE_STATUS = {0: "converged", 1: "max_iterations", 2: "breakdown"}
_BREAKDOWN = {0: "", 1: "rho", 2: "rhat_dot_v", 3: "t_dot_t", 4: "omega", 5: "diverged"}


def bicgstab(a: Csr, b, tol=1e-10, max_iters=20000):
    """bicgstab<T> over the csr backend (solvers.hpp:268-373) in a.values' dtype
    (dot products sequential in T, residual norm in fp64)."""
    n = a.n_rows
    dt = a.values.dtype
    x = np.zeros(n, dt)
    hist = np.zeros(max(max_iters, 1), np.float64)
    it, fr, st, why = C.c_int64(), C.c_double(), C.c_int(), C.c_int()
    fn = lib().mo_bicgstab_f64 if dt == np.float64 else lib().mo_bicgstab_f32
    _check(fn(n, a.row_offsets, _vals_or_dummy(a.col_indices), _vals_or_dummy(a.values),
              np.ascontiguousarray(b, dt), tol, max_iters, x, hist, C.byref(it), C.byref(fr),
              C.byref(st), C.byref(why)), "bicgstab")
    reason = _BREAKDOWN[why.value]
    return dict(x=x, residual_history=hist[:_hist_len(it.value, st.value, reason)],
                iterations=it.value, final_residual=fr.value, status=_SOLVE_STATUS[st.value],
                breakdown_reason=reason)


def _hist_len(iterations, status, reason):
    """residual_history gets one entry per completed pass: a breakdown before
    the stopping test (every reason but "diverged") leaves the pass out."""
    return iterations - 1 if status == 2 and reason != "diverged" else iterations


# --------------------------------------------------------------------------
# fixtures / generators
# --------------------------------------------------------------------------
def five_point_laplacian(grid_dim, dtype=np.float64) -> Csr:
    """five_point_laplacian<T>(grid_dim) (fixtures.hpp:41-56): 4 on the
    diagonal, -1 to the grid neighbours, CSR columns ascending."""
    n = grid_dim * grid_dim
    ro, cols, vals = [0], [], []
    for i in range(grid_dim):
        for j in range(grid_dim):
            v = i * grid_dim + j
            ent = [(v, 4.0)]
            if i > 0:
                ent.append((v - grid_dim, -1.0))
            if i + 1 < grid_dim:
                ent.append((v + grid_dim, -1.0))
            if j > 0:
                ent.append((v - 1, -1.0))
            if j + 1 < grid_dim:
                ent.append((v + 1, -1.0))
            ent.sort()
            cols += [c for c, _ in ent]
            vals += [w for _, w in ent]
            ro.append(len(cols))
    return Csr(n, n, np.array(ro, np.int64), np.array(cols, np.int32), np.array(vals, dtype))


def singular_diagonal(dtype=np.float64) -> Csr:
    """singular_diagonal_fixture<T>() (fixtures.hpp:83-91): diag(1, 0)."""
    return Csr(2, 2, np.array([0, 1, 1], np.int64), np.array([0], np.int32),
               np.array([1.0], dtype))
def _alloc_ptrs():
    return C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)(), C.POINTER(C.c_double)()


def random_matrix(shape, seed) -> Csr:
    """coo_to_csr<double>(testing::random_matrix(shape, seed)) (generators.hpp:49-130)."""
    s = SHAPES.index(shape) if isinstance(shape, str) else int(shape)
    nr, nc, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    ro, cols, vals = _alloc_ptrs()
    _check(lib().mo_random_matrix_csr(s, seed, C.byref(nr), C.byref(nc), C.byref(nnz),
                                      C.byref(ro), C.byref(cols), C.byref(vals)))
    return Csr(nr.value, nc.value, _take(ro, nr.value + 1, np.int64),
               _take(cols, nnz.value, np.int32), _take(vals, nnz.value, np.float64))


def ring_with_chords(n, extra, seed) -> Csr:
    nnz = C.c_int64()
    ro, cols, vals = _alloc_ptrs()
    _check(lib().mo_ring_with_chords_csr(n, extra, seed, C.byref(nnz), C.byref(ro),
                                         C.byref(cols), C.byref(vals)))
    return Csr(n, n, _take(ro, n + 1, np.int64), _take(cols, nnz.value, np.int32),
               _take(vals, nnz.value, np.float64))


def single_dense_row(width, seed) -> Csr:
    ro, cols, vals = _alloc_ptrs()
    _check(lib().mo_single_dense_row_csr(width, seed, C.byref(ro), C.byref(cols),
                                         C.byref(vals)))
    return Csr(1, width, _take(ro, 2, np.int64), _take(cols, width, np.int32),
               _take(vals, width, np.float64))


def walkthrough() -> Csr:
    """fixtures.hpp:17-36"""
    ro = np.array([0, 5, 5, 10, 13, 20, 26, 32, 34], np.int64)
    cols = np.array([0, 2, 3, 5, 7, 1, 2, 4, 6, 7, 0, 3, 6, 0, 1, 2, 4, 5, 6, 7,
                     0, 1, 3, 4, 5, 7, 1, 2, 3, 4, 6, 7, 3, 5], np.int32)
    return Csr(8, 8, ro, cols, np.arange(1, 35, dtype=np.float64))


def seed_test_vector(n, lo, hi, seed):
    out = np.zeros(max(n, 1), np.float64)
    lib().mo_seed_test_vector(n, lo, hi, seed, out)
    return out[:n]


def rmat(scale, edge_factor=16, seed=1, transposed=False, nthreads=None) -> Csr:
    """Counter-based R-MAT pattern (values None)."""
    nthreads = nthreads or os.cpu_count() or 1
    nnz = C.c_int64()
    ro, cols = C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
    _check(lib().mo_rmat_csr(scale, edge_factor, seed, int(transposed), nthreads,
                             C.byref(nnz), C.byref(ro), C.byref(cols)), "rmat")
    n = 1 << scale
    return Csr(n, n, _take(ro, n + 1, np.int64), _take(cols, nnz.value, np.int32), None)


def hash_uniform(seed, count, lo=0.0, hi=1.0, dtype=np.float64):
    out = np.zeros(max(count, 1), dtype)
    if dtype == np.float32:
        lib().mo_hash_uniform_f32(seed, count, lo, hi, out)
    else:
        lib().mo_hash_uniform(seed, count, lo, hi, out)
    return out[:count]


def transition_values(n, cols, dtype=np.float32):
    vals = np.zeros(max(cols.size, 1), dtype)
    fn = lib().mo_transition_values_f32 if dtype == np.float32 else lib().mo_transition_values_f64
    fn(n, cols.size, _vals_or_dummy(np.ascontiguousarray(cols, np.int32)), vals)
    return vals[:cols.size]


# --------------------------------------------------------------------------
# the compiled reference (oracle/_ref)
# --------------------------------------------------------------------------
_ref = None


class _Ref:
    """Thin ctypes view of oracle/_ref/libmerbit_ref.so (the real reference)."""

    def __init__(self, path):
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_config_make.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.ref_merge_search.argtypes = [i64p, C.c_int64, C.c_int64, C.c_int64,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int)]
        L.ref_generate_tile.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                        C.c_int, C.c_int, u32p, u32p, u32p,
                                        C.POINTER(C.c_double)]
        for sfx, fp in (("f64", f64p), ("f32", f32p)):
            getattr(L, f"ref_spmv_merbit_{sfx}").argtypes = [
                C.c_int64, C.c_int64, i64p, i32p, fp, fp, C.c_int, C.c_int, C.c_int,
                C.c_int, fp, i64p]
            getattr(L, f"ref_spmv_csr_{sfx}").argtypes = [C.c_int64, C.c_int64, i64p,
                                                          i32p, fp, fp, fp]
            getattr(L, f"ref_engine_create_{sfx}").argtypes = [
                C.c_int64, C.c_int64, i64p, i32p, fp, C.c_int, C.c_int, C.c_int, C.c_int]
            getattr(L, f"ref_engine_create_{sfx}").restype = C.c_void_p
            getattr(L, f"ref_engine_apply_{sfx}").argtypes = [C.c_void_p, fp, C.c_void_p]
            getattr(L, f"ref_engine_preprocess_seconds_{sfx}").argtypes = [C.c_void_p]
            getattr(L, f"ref_engine_preprocess_seconds_{sfx}").restype = C.c_double
            getattr(L, f"ref_engine_pagerank_{sfx}").argtypes = [
                C.c_void_p, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_void_p,
                C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double)]
            getattr(L, f"ref_engine_destroy_{sfx}").argtypes = [C.c_void_p]
        L.ref_pagerank_csr_f64.argtypes = [C.c_int64, i64p, i32p, f64p, C.c_double,
                                           C.c_double, C.c_int64, C.c_int64, f64p, f64p,
                                           C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                           C.POINTER(C.c_int)]
        L.ref_pagerank_csr_f32.argtypes = [C.c_int64, i64p, i32p, f32p, C.c_double,
                                           C.c_double, C.c_int64, C.c_int64, f32p,
                                           C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                           C.POINTER(C.c_int)]
        for name, fp in (("ref_bicgstab_csr_f64", f64p), ("ref_bicgstab_csr_f32", f32p)):
            getattr(L, name).argtypes = [C.c_int64, i64p, i32p, fp, fp, C.c_double, C.c_int64,
                                         fp, f64p, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_double), C.POINTER(C.c_int),
                                         C.c_char_p, C.c_int]
        for name, fp in (("ref_spmv_merge_runtime_f64", f64p), ("ref_spmv_merge_runtime_f32", f32p)):
            getattr(L, name).argtypes = [C.c_int64, C.c_int64, i64p, i32p, fp, fp, C.c_int, fp]
        u32pp = C.POINTER(C.POINTER(C.c_uint32))
        L.ref_tile_cache_write.argtypes = [C.c_char_p, C.c_int64, C.c_int64, i64p, C.c_int,
                                           C.c_int, C.c_int]
        L.ref_tile_cache_read.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                          u32pp, u32pp, u32pp, C.POINTER(C.c_int)]
        coo_out = [C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                   C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int64)),
                   C.POINTER(C.POINTER(C.c_double))]
        L.ref_matrix_read.argtypes = [C.c_char_p, C.c_int] + coo_out
        L.ref_matrix_write.argtypes = [C.c_char_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                       i64p, i64p, f64p]
        L.ref_coo_to_csr_f64.argtypes = [C.c_int64, C.c_int64, C.c_int64, i64p, i64p, f64p,
                                         C.POINTER(C.c_int64), C.POINTER(C.POINTER(C.c_int64)),
                                         C.POINTER(C.POINTER(C.c_int32)),
                                         C.POINTER(C.POINTER(C.c_double))]
        L.ref_build_transition_f64.argtypes = [C.c_int64, i64p, i32p, i64p, i32p, f64p]
        alloc_args = [C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int32)),
                      C.POINTER(C.POINTER(C.c_double))]
        L.ref_random_matrix_csr.argtypes = [C.c_int, C.c_uint64, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64), C.POINTER(C.c_int64)] + alloc_args
        L.ref_ring_with_chords_csr.argtypes = [C.c_int64, C.c_int64, C.c_uint64,
                                               C.POINTER(C.c_int64)] + alloc_args
        L.ref_seed_test_vector.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64, f64p]
        L.ref_free.argtypes = [C.c_void_p]
        self.L = L

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.ref_last_error().decode())

    def _take(self, ptr, n, dtype):
        out = (np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)
               if n else np.zeros(0, dtype))
        self.L.ref_free(C.cast(ptr, C.c_void_p))
        return out

    def config_make(self, omega, sigma, block):
        ob = C.c_int()
        self._check(self.L.ref_config_make(omega, sigma, block, C.byref(ob)))
        return ob.value

    def merge_search(self, ro, n_rows, nnz, diag):
        x, y, p = C.c_int64(), C.c_int64(), C.c_int()
        self._check(self.L.ref_merge_search(np.ascontiguousarray(ro, np.int64), n_rows,
                                            nnz, diag, C.byref(x), C.byref(y), C.byref(p)))
        return x.value, y.value, p.value

    def generate_tile(self, ro, n_rows, nnz, omega, sigma):
        tiles, lanes = tile_counts(nnz, n_rows, omega, sigma)
        tx = np.zeros(tiles + 1, np.uint32)
        ty = np.zeros(tiles + 1, np.uint32)
        ld = np.zeros(max(lanes, 1), np.uint32)
        secs = C.c_double()
        ro_arr = None if ro is None else np.ascontiguousarray(ro, np.int64)
        self._check(self.L.ref_generate_tile(None if ro_arr is None else ro_arr.ctypes.data,
                                             n_rows, nnz, omega, sigma, omega, tx, ty, ld,
                                             C.byref(secs)))
        return tx, ty, ld[:lanes]

    def spmv_merbit(self, a: Csr, x, omega, sigma, block, nthreads=1):
        dt = a.values.dtype
        sfx = "f64" if dt == np.float64 else "f32"
        y = np.zeros(max(a.n_rows, 1), dt)
        cnt = np.zeros(3, np.int64)
        self._check(getattr(self.L, f"ref_spmv_merbit_{sfx}")(
            a.n_rows, a.n_cols, a.row_offsets, _vals_or_dummy(a.col_indices),
            _vals_or_dummy(a.values), _vals_or_dummy(np.ascontiguousarray(x, dt)),
            omega, sigma, block, nthreads, y, cnt))
        return y[:a.n_rows], cnt

    def spmv_csr(self, a: Csr, x):
        dt = a.values.dtype
        sfx = "f64" if dt == np.float64 else "f32"
        y = np.zeros(max(a.n_rows, 1), dt)
        self._check(getattr(self.L, f"ref_spmv_csr_{sfx}")(
            a.n_rows, a.n_cols, a.row_offsets, _vals_or_dummy(a.col_indices),
            _vals_or_dummy(a.values), _vals_or_dummy(np.ascontiguousarray(x, dt)), y))
        return y[:a.n_rows]

    def spmv_merge_runtime(self, a: Csr, x, sigma):
        """The reference's spmv_merge_runtime<T> (merge_spmv.hpp:21-82)."""
        dt = a.values.dtype
        y = np.zeros(a.n_rows, dt)
        fn = (self.L.ref_spmv_merge_runtime_f64 if dt == np.float64
              else self.L.ref_spmv_merge_runtime_f32)
        self._check(fn(a.n_rows, a.n_cols, a.row_offsets, _vals_or_dummy(a.col_indices),
                       _vals_or_dummy(a.values), np.ascontiguousarray(x, dt), sigma,
                       y if a.n_rows else np.zeros(1, dt)))
        return y

    # ---- file formats --------------------------------------------------
    def tile_cache_write(self, path, ro, n_rows, nnz, omega, sigma, f64=False):
        self._check(self.L.ref_tile_cache_write(os.fsencode(path), n_rows, nnz,
                                                np.ascontiguousarray(ro, np.int64), omega, sigma,
                                                1 if f64 else 0))

    def tile_cache_read(self, path):
        om, sg, f64 = C.c_int(), C.c_int(), C.c_int()
        nr, nz, tn, ln = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        tx, ty, ld = (C.POINTER(C.c_uint32)() for _ in range(3))
        self._check(self.L.ref_tile_cache_read(os.fsencode(path), C.byref(om), C.byref(sg),
                                               C.byref(nr), C.byref(nz), C.byref(tn),
                                               C.byref(ln), C.byref(tx), C.byref(ty),
                                               C.byref(ld), C.byref(f64)))
        take = lambda p, n: self._take(p, n, np.uint32)  # noqa: E731
        return dict(omega=om.value, sigma=sg.value, n_rows=nr.value, nnz=nz.value,
                    tile_x=take(tx, tn.value + 1), tile_y=take(ty, tn.value + 1),
                    lane_desc=take(ld, ln.value), f64=bool(f64.value))

    def matrix_read(self, path, which=0):
        """which: 0 parse_matrix_market_file, 1 read_matrix_cache, 2 load_matrix_any."""
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        r, c = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
        v = C.POINTER(C.c_double)()
        self._check(self.L.ref_matrix_read(os.fsencode(path), which, C.byref(nr), C.byref(nc),
                                           C.byref(nz), C.byref(r), C.byref(c), C.byref(v)))
        n = nz.value
        return dict(n_rows=nr.value, n_cols=nc.value, rows=self._take(r, n, np.int64),
                    cols=self._take(c, n, np.int64), vals=self._take(v, n, np.float64))

    def matrix_write(self, path, coo, which=0):
        """which: 0 write_matrix_market_file, 1 write_matrix_cache."""
        self._check(self.L.ref_matrix_write(os.fsencode(path), which, coo["n_rows"],
                                            coo["n_cols"], len(coo["rows"]),
                                            np.ascontiguousarray(coo["rows"], np.int64),
                                            np.ascontiguousarray(coo["cols"], np.int64),
                                            np.ascontiguousarray(coo["vals"], np.float64)))

    def coo_to_csr(self, coo) -> Csr:
        m = C.c_int64()
        ro, cols = C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
        vals = C.POINTER(C.c_double)()
        self._check(self.L.ref_coo_to_csr_f64(coo["n_rows"], coo["n_cols"], len(coo["rows"]),
                                              np.ascontiguousarray(coo["rows"], np.int64),
                                              np.ascontiguousarray(coo["cols"], np.int64),
                                              np.ascontiguousarray(coo["vals"], np.float64),
                                              C.byref(m), C.byref(ro), C.byref(cols),
                                              C.byref(vals)))
        return Csr(coo["n_rows"], coo["n_cols"], self._take(ro, coo["n_rows"] + 1, np.int64),
                   self._take(cols, m.value, np.int32), self._take(vals, m.value, np.float64))

    def bicgstab_csr(self, a: Csr, b, tol=1e-10, max_iters=20000):
        """The reference's own bicgstab<T> over CsrReferenceBackend."""
        n = a.n_rows
        dt = a.values.dtype
        x = np.zeros(n, dt)
        hist = np.zeros(max(max_iters, 1), np.float64)
        it, fr, st = C.c_int64(), C.c_double(), C.c_int()
        why = C.create_string_buffer(32)
        fn = self.L.ref_bicgstab_csr_f64 if dt == np.float64 else self.L.ref_bicgstab_csr_f32
        self._check(fn(n, a.row_offsets, _vals_or_dummy(a.col_indices), _vals_or_dummy(a.values),
                       np.ascontiguousarray(b, dt), tol, max_iters, x, hist, C.byref(it),
                       C.byref(fr), C.byref(st), why, 32))
        reason = why.value.decode()
        return dict(x=x, residual_history=hist[:_hist_len(it.value, st.value, reason)],
                    iterations=it.value, final_residual=fr.value,
                    status=_SOLVE_STATUS[st.value], breakdown_reason=reason)

    def pagerank_csr(self, p: Csr, damping=0.85, err_tol=1e-10, max_iters=210,
                     reference_iters=210):
        n = p.n_rows
        it, err, st = C.c_int64(), C.c_double(), C.c_int()
        if p.values.dtype == np.float64:
            pi, star = np.zeros(n), np.zeros(n)
            self._check(self.L.ref_pagerank_csr_f64(
                n, p.row_offsets, _vals_or_dummy(p.col_indices), _vals_or_dummy(p.values),
                damping, err_tol, max_iters, reference_iters, pi, star, C.byref(it),
                C.byref(err), C.byref(st)))
        else:
            pi, star = np.zeros(n, np.float32), None
            self._check(self.L.ref_pagerank_csr_f32(
                n, p.row_offsets, _vals_or_dummy(p.col_indices), _vals_or_dummy(p.values),
                damping, err_tol, max_iters, reference_iters, pi, C.byref(it),
                C.byref(err), C.byref(st)))
        return dict(pi=pi, reference_pi=star, iterations=it.value, final_err=err.value,
                    status="converged" if st.value == 0 else "max_iterations")

    def build_transition(self, adj: Csr) -> Csr:
        n = adj.n_rows
        ro = np.zeros(n + 1, np.int64)
        cols = np.zeros(max(adj.nnz, 1), np.int32)
        vals = np.zeros(max(adj.nnz, 1), np.float64)
        self._check(self.L.ref_build_transition_f64(n, adj.row_offsets,
                                                    _vals_or_dummy(adj.col_indices),
                                                    ro, cols, vals))
        return Csr(n, n, ro, cols[:adj.nnz], vals[:adj.nnz])

    def random_matrix(self, shape, seed) -> Csr:
        s = SHAPES.index(shape) if isinstance(shape, str) else int(shape)
        nr, nc, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        ro, cols, vals = _alloc_ptrs()
        self._check(self.L.ref_random_matrix_csr(s, seed, C.byref(nr), C.byref(nc),
                                                 C.byref(nnz), C.byref(ro), C.byref(cols),
                                                 C.byref(vals)))
        return Csr(nr.value, nc.value, self._take(ro, nr.value + 1, np.int64),
                   self._take(cols, nnz.value, np.int32),
                   self._take(vals, nnz.value, np.float64))

    def ring_with_chords(self, n, extra, seed) -> Csr:
        nnz = C.c_int64()
        ro, cols, vals = _alloc_ptrs()
        self._check(self.L.ref_ring_with_chords_csr(n, extra, seed, C.byref(nnz),
                                                    C.byref(ro), C.byref(cols), C.byref(vals)))
        return Csr(n, n, self._take(ro, n + 1, np.int64),
                   self._take(cols, nnz.value, np.int32),
                   self._take(vals, nnz.value, np.float64))

    def seed_test_vector(self, n, lo, hi, seed):
        out = np.zeros(max(n, 1), np.float64)
        self.L.ref_seed_test_vector(n, lo, hi, seed, out)
        return out[:n]


class RefEngine:
    """The reference MerbitBackend<T> on ThreadPool(nthreads) (backend.hpp:112-136),
    persistent across calls so timing excludes setup."""

    def __init__(self, a: Csr, omega, sigma, block, nthreads):
        r = ref()
        if r is None:
            raise RuntimeError("oracle/_ref/libmerbit_ref.so not built")
        self.L = r.L
        self.dt = a.values.dtype
        self.sfx = "f64" if self.dt == np.float64 else "f32"
        self.a = a
        self.h = getattr(self.L, f"ref_engine_create_{self.sfx}")(
            a.n_rows, a.n_cols, a.row_offsets, _vals_or_dummy(a.col_indices),
            _vals_or_dummy(a.values), omega, sigma, block, nthreads)
        if not self.h:
            raise OracleError(1, self.L.ref_last_error().decode())
        self.preprocess_seconds = getattr(self.L, f"ref_engine_preprocess_seconds_{self.sfx}")(self.h)

    def apply(self, x, y=None):
        rc = getattr(self.L, f"ref_engine_apply_{self.sfx}")(
            self.h, np.ascontiguousarray(x, self.dt), None if y is None else y.ctypes.data)
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())
        return y

    def pagerank(self, damping, err_tol, max_iters, reference_iters, want_pi=False):
        pi = np.zeros(self.a.n_rows, self.dt) if want_pi else None
        it, err, secs = C.c_int64(), C.c_double(), C.c_double()
        rc = getattr(self.L, f"ref_engine_pagerank_{self.sfx}")(
            self.h, damping, err_tol, max_iters, reference_iters,
            None if pi is None else pi.ctypes.data, C.byref(it), C.byref(err), C.byref(secs))
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())
        return dict(pi=pi, iterations=it.value, final_err=err.value, seconds=secs.value)

    def close(self):
        if self.h:
            getattr(self.L, f"ref_engine_destroy_{self.sfx}")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref():
    """The compiled reference, or None when oracle/_ref was never built."""
    global _ref
    if _ref is None and os.path.exists(_REF_SO):
        _ref = _Ref(_REF_SO)
    return _ref
