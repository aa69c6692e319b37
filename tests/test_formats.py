"""CPU: the on-disk formats of the path -- MBTL TILE cache,
MBMX matrix cache, Matrix Market text -- in libmerbit_b200.so's host code,
checked byte-for-byte (files) and rejection-for-rejection (the same inputs
refused with the same error class at the same line) against the reference's
own readers and writers (oracle/_ref compiled from src/tile.cpp and
src/matrix_market.cpp).  Host logic only: no device call."""
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2605_07391_b200 import formats as F
from paper_2605_07391_b200.merbit import (CorruptionError, DimensionError, IoError,
                                          ParseError)

needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")


class HostTile:
    def __init__(self, a, omega, sigma):
        self.omega, self.sigma, self.n_rows, self.nnz = omega, sigma, a.n_rows, a.nnz
        self.tile_x, self.tile_y, self.lane_desc = O.generate_tile(a.row_offsets, a.n_rows,
                                                                   a.nnz, omega, sigma)


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def _tile_cases():
    yield O.walkthrough()
    for shape in O.SHAPES:
        yield O.random_matrix(shape, 7)
    yield O.single_dense_row(1000, 3)
    yield O.Csr(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    yield O.Csr(5, 5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0))


@needs_ref
@pytest.mark.parametrize("cfg", [(32, 14), (32, 7), (4, 4)])
def test_tile_cache_bytes_match_reference(tmp_path, cfg):
    w, s = cfg
    for i, a in enumerate(_tile_cases()):
        for prec in ("f32", "f64"):
            ours, theirs = tmp_path / f"o{i}.mbtl", tmp_path / f"r{i}.mbtl"
            F.write_tile_cache(str(ours), HostTile(a, w, s), prec)
            O.ref().tile_cache_write(str(theirs), a.row_offsets, a.n_rows, a.nnz, w, s,
                                     prec == "f64")
            assert _bytes(ours) == _bytes(theirs)
            got = F.read_tile_cache(str(theirs))
            want = O.ref().tile_cache_read(str(ours))
            assert (got.omega, got.sigma, got.n_rows, got.nnz) == (
                want["omega"], want["sigma"], want["n_rows"], want["nnz"])
            assert got.precision == prec and want["f64"] == (prec == "f64")
            for k in ("tile_x", "tile_y", "lane_desc"):
                assert np.array_equal(getattr(got, k), want[k])


def test_tile_cache_errors(tmp_path):
    p = tmp_path / "t.mbtl"
    with pytest.raises(IoError):
        F.read_tile_cache(str(tmp_path / "missing.mbtl"))
    p.write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(ParseError, match="no MBTL signature"):
        F.read_tile_cache(str(p))
    F.write_tile_cache(str(p), HostTile(O.walkthrough(), 4, 4))
    raw = bytearray(_bytes(p))
    raw[4] = 9  # version
    p.write_bytes(bytes(raw))
    with pytest.raises(ParseError, match="has version 9"):
        F.read_tile_cache(str(p))
    F.write_tile_cache(str(p), HostTile(O.walkthrough(), 4, 4))
    p.write_bytes(_bytes(p)[:-3])
    with pytest.raises(CorruptionError, match="ends early"):
        F.read_tile_cache(str(p))
    raw = bytearray(_bytes(tmp_path / "t.mbtl"))
    raw[8:12] = (0).to_bytes(4, "little")  # omega = 0
    p.write_bytes(bytes(raw))
    with pytest.raises(CorruptionError, match="impossible header"):
        F.read_tile_cache(str(p))


MM_CASES = {
    "general": "%%MatrixMarket matrix coordinate real general\n% c\n3 4 4\n1 1 1.5\n3 4 -2\n"
               "2 2 1e-3\n1 1 0.25\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 4\n2 1 -1\n"
                 "3 2 -1\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n\n2 2 2\n1 2\n2 1\n",
    "integer_crlf": "%%MatrixMarket Matrix Coordinate Integer General\r\n2 3 2\r\n1 3 7\r\n"
                    "   \r\n2 1 -4\r\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
}
# malformed inputs, each rejected by both readers at the same line (the
# messages are each implementation's own)
MM_ERRORS = [
    "",
    "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n",
    "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n",
    "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1 9\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n-2 2 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n",
    "%%MatrixMarket matrix coordinate real general\n% c\n\n2 2 1\n% x\n1 3 1\n",
]


def _coo_equal(got, want):
    assert (got.n_rows, got.n_cols) == (want["n_rows"], want["n_cols"])
    assert np.array_equal(got.rows, want["rows"]) and np.array_equal(got.cols, want["cols"])
    assert np.array_equal(got.vals.view(np.uint64), want["vals"].view(np.uint64))


@needs_ref
def test_matrix_market_parse_matches_reference(tmp_path):
    for name, text in MM_CASES.items():
        p = tmp_path / f"{name}.mtx"
        p.write_bytes(text.encode())
        got = F.parse_matrix_market_file(str(p))
        _coo_equal(got, O.ref().matrix_read(str(p), 0))
        _coo_equal(F.parse_matrix_market(text, str(p)), O.ref().matrix_read(str(p), 0))


def _where(msg):
    """The "origin:line" a Matrix Market error names (None without a line)."""
    m = re.search(r"(\S+\.mtx):(\d+):", msg)
    return (m.group(1), int(m.group(2))) if m else None


@needs_ref
def test_matrix_market_errors_match_reference(tmp_path):
    for i, text in enumerate(MM_ERRORS):
        p = tmp_path / f"bad{i}.mtx"
        p.write_bytes(text.encode())
        with pytest.raises(ParseError) as ours:
            F.parse_matrix_market_file(str(p))
        with pytest.raises(O.OracleError) as theirs:
            O.ref().matrix_read(str(p), 0)
        # same rejection, same error class (parse_error), same file and line
        assert _where(str(ours.value)) == _where(str(theirs.value)), (text, ours.value,
                                                                      theirs.value)
    with pytest.raises(IoError):
        F.parse_matrix_market_file(str(tmp_path / "nope.mtx"))


def _random_coo(seed, n_rows=50, n_cols=40, n=400):
    rng = np.random.default_rng(seed)
    vals = rng.uniform(-1e3, 1e3, n)
    vals[::7] = rng.uniform(-1, 1, vals[::7].size) * 10.0 ** rng.integers(-30, 30, vals[::7].size)
    return F.CooTriples(n_rows, n_cols, rng.integers(0, n_rows, n), rng.integers(0, n_cols, n),
                        vals)


@needs_ref
def test_writers_match_reference_bytes(tmp_path):
    for seed in range(4):
        coo = _random_coo(seed)
        d = dict(n_rows=coo.n_rows, n_cols=coo.n_cols, rows=coo.rows, cols=coo.cols,
                 vals=coo.vals)
        for which, ext, write in ((0, "mtx", F.write_matrix_market_file),
                                  (1, "mbmx", F.write_matrix_cache)):
            ours, theirs = tmp_path / f"o{seed}.{ext}", tmp_path / f"r{seed}.{ext}"
            write(str(ours), coo)
            O.ref().matrix_write(str(theirs), d, which)
            assert _bytes(ours) == _bytes(theirs)
            # round trips through both readers and the sniffing loader
            _coo_equal(F.load_matrix_any(str(theirs)), O.ref().matrix_read(str(ours), 2))
        _coo_equal(F.read_matrix_cache(str(tmp_path / f"r{seed}.mbmx")), d)


def test_matrix_cache_errors(tmp_path):
    p = tmp_path / "m.mbmx"
    p.write_bytes(b"MBMX" + (2).to_bytes(4, "little"))
    with pytest.raises(ParseError, match="has version 2"):
        F.read_matrix_cache(str(p))
    F.write_matrix_cache(str(p), _random_coo(1))
    p.write_bytes(_bytes(p)[:-5])
    with pytest.raises(CorruptionError, match="ends early"):
        F.read_matrix_cache(str(p))
    raw = bytearray(_bytes(tmp_path / "m.mbmx"))
    coo = F.CooTriples(2, 2, np.array([0]), np.array([5]), np.array([1.0]))
    F.write_matrix_cache(str(p), coo)
    with pytest.raises(CorruptionError, match="outside its 2x2 bounds"):
        F.read_matrix_cache(str(p))
    with pytest.raises(IoError):
        F.load_matrix_any(str(tmp_path / "missing"))
    del raw
