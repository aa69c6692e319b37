"""On-disk formats of the MERBIT path over the C ABI.

    CooTriples                               csr.hpp:22-26
    parse_matrix_market(_file)               matrix_market.hpp:14-15
    write_matrix_market_file                 matrix_market.hpp:18-19
    write_matrix_cache / read_matrix_cache   matrix_market.hpp:22-23 (MBMX)
    load_matrix_any                          matrix_market.hpp:26
    write_tile_cache / read_tile_cache       tile.hpp / tile.cpp:161-234 (MBTL)
    matrix_from_coo                          coo_to_csr<T> (csr.hpp:43-88) on the GPU

Parsing and file I/O are host work inside libmerbit_b200.so (io.cpp); the
COO -> CSR normalisation and the TILE upload run on the device (ingest.cu).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import mbx_coo, mbx_tile_info
from .merbit import (F32, F64, Context, DeviceMatrix, Tile, _check, _precision_of,
                     default_context)


@dataclass
class CooTriples:
    n_rows: int
    n_cols: int
    rows: np.ndarray  # int64, entry order
    cols: np.ndarray  # int64
    vals: np.ndarray  # float64

    @property
    def nnz(self) -> int:
        return int(self.rows.size)

    def _c(self):
        self.rows = np.ascontiguousarray(self.rows, np.int64)
        self.cols = np.ascontiguousarray(self.cols, np.int64)
        self.vals = np.ascontiguousarray(self.vals, np.float64)
        return mbx_coo(self.n_rows, self.n_cols, self.nnz,
                       self.rows.ctypes.data_as(C.POINTER(C.c_int64)),
                       self.cols.ctypes.data_as(C.POINTER(C.c_int64)),
                       self.vals.ctypes.data_as(C.POINTER(C.c_double)))


def _take_coo(c: mbx_coo) -> CooTriples:
    n = c.nnz
    try:
        rows = np.ctypeslib.as_array(c.rows, (max(n, 1),))[:n].copy()
        cols = np.ctypeslib.as_array(c.cols, (max(n, 1),))[:n].copy()
        vals = np.ctypeslib.as_array(c.vals, (max(n, 1),))[:n].copy()
    finally:
        _lib.lib().mbx_coo_free(C.byref(c))
    return CooTriples(c.n_rows, c.n_cols, rows, cols, vals)


def parse_matrix_market_file(path: str) -> CooTriples:
    c = mbx_coo()
    _check(_lib.lib().mbx_mm_read(os.fsencode(path), C.byref(c)))
    return _take_coo(c)


def parse_matrix_market(text: str, origin: str = "<memory>") -> CooTriples:
    b = text.encode()
    c = mbx_coo()
    _check(_lib.lib().mbx_mm_parse(b, len(b), origin.encode(), C.byref(c)))
    return _take_coo(c)


def write_matrix_market_file(path: str, coo: CooTriples) -> None:
    cc = coo._c()
    _check(_lib.lib().mbx_mm_write(os.fsencode(path), C.byref(cc)))


def write_matrix_cache(path: str, coo: CooTriples) -> None:
    cc = coo._c()
    _check(_lib.lib().mbx_matrix_cache_write(os.fsencode(path), C.byref(cc)))


def read_matrix_cache(path: str) -> CooTriples:
    c = mbx_coo()
    _check(_lib.lib().mbx_matrix_cache_read(os.fsencode(path), C.byref(c)))
    return _take_coo(c)


def load_matrix_any(path: str) -> CooTriples:
    c = mbx_coo()
    _check(_lib.lib().mbx_matrix_load_any(os.fsencode(path), C.byref(c)))
    return _take_coo(c)


def matrix_from_coo(coo: CooTriples, dtype=np.float64, ctx: Context | None = None) -> DeviceMatrix:
    """coo_to_csr<T>(coo) on the device -> a resident DeviceMatrix."""
    ctx = ctx or default_context()
    cc = coo._c()
    h = C.c_void_p()
    _check(_lib.lib().mbx_matrix_from_coo(ctx.h, _precision_of(np.dtype(dtype)), C.byref(cc),
                                          C.byref(h)))
    return DeviceMatrix(ctx, h)


@dataclass
class TileCacheContents:
    """TileCacheContents (tile.hpp): host TILE arrays + stored precision."""
    omega: int
    sigma: int
    n_rows: int
    nnz: int
    tile_x: np.ndarray
    tile_y: np.ndarray
    lane_desc: np.ndarray
    precision: str  # "f32" | "f64"

    @property
    def tile_num(self) -> int:
        return int(self.tile_x.size) - 1

    @property
    def lane_num(self) -> int:
        return int(self.lane_desc.size)


def write_tile_cache(path: str, tile, precision: str = "f32") -> None:
    """MBTL file from a device Tile or host arrays (omega, sigma, n_rows, nnz,
    tile_x, tile_y, lane_desc attributes)."""
    p = F64 if precision == "f64" else F32
    if isinstance(tile, Tile):
        _check(_lib.lib().mbx_tile_cache_write(tile.h, os.fsencode(path), p))
        return
    tx = np.ascontiguousarray(tile.tile_x, np.uint32)
    ty = np.ascontiguousarray(tile.tile_y, np.uint32)
    ld = np.ascontiguousarray(tile.lane_desc, np.uint32)
    info = mbx_tile_info(tile.omega, tile.sigma, tile.n_rows, tile.nnz, tx.size - 1, ld.size, 0.0)
    u32p = C.POINTER(C.c_uint32)
    _check(_lib.lib().mbx_tile_cache_write_host(os.fsencode(path), C.byref(info),
                                                tx.ctypes.data_as(u32p), ty.ctypes.data_as(u32p),
                                                ld.ctypes.data_as(u32p), p))


def read_tile_cache(path: str) -> TileCacheContents:
    info = mbx_tile_info()
    u32p = C.POINTER(C.c_uint32)
    tx, ty, ld = u32p(), u32p(), u32p()
    prec = C.c_int()
    _check(_lib.lib().mbx_tile_cache_read_host(os.fsencode(path), C.byref(info), C.byref(tx),
                                               C.byref(ty), C.byref(ld), C.byref(prec)))
    L = _lib.lib()

    def take(ptr, n):
        a = np.ctypeslib.as_array(ptr, (max(n, 1),))[:n].copy()
        L.mbx_free(C.cast(ptr, C.c_void_p))
        return a

    return TileCacheContents(info.omega, info.sigma, info.n_rows, info.nnz,
                             take(tx, info.tile_num + 1), take(ty, info.tile_num + 1),
                             take(ld, info.lane_num), "f64" if prec.value == F64 else "f32")


def load_tile_cache(path: str, ctx: Context | None = None) -> tuple[Tile, str]:
    """MBTL file -> device Tile (the cached preprocessing, tile.cpp:201-234)."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    prec = C.c_int()
    _check(_lib.lib().mbx_tile_cache_load(ctx.h, os.fsencode(path), C.byref(h), C.byref(prec)))
    return Tile(ctx, h), ("f64" if prec.value == F64 else "f32")
