"""CPU: the C-ABI library loads, exports every symbol include/merbit_b200.h
declares, and its host-only entry points (config, counts, merge_search, shard
planning) behave like the reference (no GPU needed, no compute calls)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from paper_2605_07391_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "merbit_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"MBX_API[^;(]*?\b(mbx_\w+)\s*\(", text, re.S)))


def test_library_exports_every_declared_symbol():
    decl = declared_symbols()
    assert len(decl) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mbx_\w+)", out))
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    assert sorted(_lib.SIGNATURES) == decl  # the Python view binds exactly the header
    L = _lib.lib()
    for s in decl:
        assert getattr(L, s) is not None
    assert b"sm_100a" in L.mbx_build_info()


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_simt_config_matches_reference_rules():
    # test_format.cpp:13-35, acceptance.cpp:483-502
    assert mb.SimtConfig.make(32, 14, 32).offset_bits == 9
    assert mb.SimtConfig.make(32, 7, 32).offset_bits == 8
    assert mb.SimtConfig.make(4, 4, 4).offset_bits == 4
    assert mb.SimtConfig.make(1, 1, 1).offset_bits == 0
    with pytest.raises(mb.ConfigError, match=r"2\*ceil_log2\(omega\*sigma\) \+ sigma"):
        mb.SimtConfig.make(32, 20, 32)
    for bad in [(0, 4, 4), (4, 0, 4), (4, 4, 6), (4, 4, 2)]:
        with pytest.raises(mb.ConfigError):
            mb.SimtConfig.make(*bad)
    for omega in (1, 2, 4, 8, 16, 32):
        for sigma in range(1, 41):
            try:
                want = O.config_make(omega, sigma, 4 * omega)
            except O.OracleError:
                want = None
            try:
                got = mb.SimtConfig.make(omega, sigma, 4 * omega).offset_bits
            except mb.ConfigError:
                got = None
            assert got == want
    assert mb.select_sigma("f32") == 14 and mb.select_sigma("f64") == 7
    assert mb.select_sigma("f64", 12) == 12


def test_counts_and_footprint():
    # test_format.cpp:160-175, 212-223
    c = mb.SimtConfig.make(32, 14, 32)
    assert mb.metadata_footprint(434, 14, c, 0.0) == 144.0
    assert mb.metadata_footprint(434, 14, c, 1.0) == 16.0
    c7 = mb.SimtConfig.make(32, 7, 128)
    for shape in O.SHAPES:
        a = O.random_matrix(shape, 55)
        total = a.nnz + a.n_rows
        assert mb.tile_counts(a.nnz, a.n_rows, c7) == ((total + 223) // 224, (total + 6) // 7)


def test_merge_search_host_entry():
    # test_merge_path.cpp:53-73
    ident = np.array([0, 1, 2, 3, 4])
    assert mb.merge_search(ident, 4, 4, 0) == (0, 0)
    assert mb.merge_search(ident, 4, 4, 4) == (2, 2)
    assert mb.merge_search(ident, 4, 4, 8) == (4, 4)
    wide = np.array([0, 5])
    assert mb.merge_search(wide, 1, 5, 3) == (3, 0)
    assert mb.merge_search(wide, 1, 5, 6) == (5, 1)
    with pytest.raises(mb.DimensionError):
        mb.merge_search(np.array([0, 1]), 1, 1, -1)
    with pytest.raises(mb.DimensionError):
        mb.merge_search(np.array([0, 1]), 1, 1, 3)
    for shape in O.SHAPES:
        a = O.random_matrix(shape, 33)
        for d in range(0, a.nnz + a.n_rows + 1, 7):
            assert mb.merge_search(a.row_offsets, a.n_rows, a.nnz, d) == \
                O.merge_search(a.row_offsets, a.n_rows, a.nnz, d)[:2]


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_row_shards_are_merge_path_balanced(parts):
    p = O.rmat(14, 16, 3, transposed=True)
    b = mb.plan_row_shards(p.row_offsets, p.n_rows, p.nnz, parts)
    assert b[0] == 0 and b[-1] == p.n_rows and np.all(np.diff(b) >= 0)
    work = [(p.row_offsets[b[g + 1]] - p.row_offsets[b[g]]) + (b[g + 1] - b[g])
            for g in range(parts)]
    target = (p.nnz + p.n_rows) / parts
    longest = int(np.diff(p.row_offsets).max()) + 1
    assert max(abs(w - target) for w in work) <= longest  # off by at most one row


@pytest.mark.parametrize("weight", [0.0, 1.0, 3.4, 16.0])
@pytest.mark.parametrize("parts", [1, 2, 5, 8])
def test_weighted_row_shards(parts, weight):
    p = O.rmat(14, 16, 5, transposed=True)
    ro = p.row_offsets
    b = mb.plan_row_shards(ro, p.n_rows, p.nnz, parts, weight)
    assert b[0] == 0 and b[-1] == p.n_rows and np.all(np.diff(b) >= 0)
    if weight == 1.0:  # exactly the merge-path cut
        assert np.array_equal(b, mb.plan_row_shards(ro, p.n_rows, p.nnz, parts))
    cost = [(ro[b[g + 1]] - ro[b[g]]) + weight * (b[g + 1] - b[g]) for g in range(parts)]
    target = (p.nnz + weight * p.n_rows) / parts
    longest = int(np.diff(ro).max()) + weight
    assert max(abs(c - target) for c in cost) <= longest + 1e-9
    with pytest.raises(mb.ConfigError):
        mb.plan_row_shards(ro, p.n_rows, p.nnz, parts, -1.0)


def test_no_gpu_means_loud_failure():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    assert mb.device_count() == 0
    with pytest.raises(mb.MerbitError):
        mb.Context(0)
