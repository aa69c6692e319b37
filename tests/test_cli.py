"""CPU: the merbit_b200 CLI (tools/merbit_b200_cli.cpp) and
its BenchRecord schema -- byte-compatible with the reference's bench_record.hpp
(CSV and JSON), fixtures written by `gen` byte-identical to the reference's
Matrix Market writer on the same fixture, and the exit-code contract of
merbit_cli.cpp:1-6.  No device work: verbs that need a GPU are in
tests/test_gpu_cli.py."""
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "merbit_b200")
REF_INC = "/root/reference/proj/include"
JSON_INC = None
for cand in ("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/"
             "thirdparty/nlohmann",):
    if os.path.exists(os.path.join(cand, "json.hpp")):
        JSON_INC = cand


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    return CLI


def run(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=True)


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and JSON_INC and shutil.which("g++")),
                    reason="needs the reference headers and nlohmann json.hpp")
def test_bench_record_bytes_match_reference(tmp_path):
    exe = tmp_path / "brc"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{REF_INC}", f"-I{JSON_INC}",
                    f"-I{os.path.join(ROOT, 'include')}",
                    os.path.join(ROOT, "tests", "cpp", "bench_record_check.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "0 failure(s)" in out.stdout


def _coo_of(a):
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_offsets)).astype(np.int64)
    return dict(n_rows=a.n_rows, n_cols=a.n_cols, rows=rows,
                cols=a.col_indices.astype(np.int64), vals=np.asarray(a.values, np.float64))


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")
def test_gen_fixtures_match_reference_writer(cli, tmp_path):
    cases = {
        ("walkthrough",): O.walkthrough(),
        ("laplacian", "--grid", "6"): O.five_point_laplacian(6),
        ("ring", "--nodes", "100", "--chords", "260", "--seed", "42"):
            O.ring_with_chords(100, 260, 42),
        ("dense-row", "--width", "40", "--seed", "3"): O.single_dense_row(40, 3),
        ("singular",): O.singular_diagonal(),
    }
    for i, (args, fixture) in enumerate(cases.items()):
        ours, theirs = tmp_path / f"o{i}.mtx", tmp_path / f"r{i}.mtx"
        r = run(cli, "gen", *args, "--out", str(ours))
        assert r.returncode == 0, r.stderr
        O.ref().matrix_write(str(theirs), _coo_of(fixture), 0)
        assert ours.read_bytes() == theirs.read_bytes(), args


def test_exit_codes_without_device(cli, tmp_path):
    assert run(cli).returncode == 64
    assert run(cli, "frobnicate").returncode == 64
    assert run(cli, "bench").returncode == 64  # missing matrix path
    assert run(cli, "gen", "walkthrough").returncode == 64  # missing --out
    assert run(cli, "gen", "bogus", "--out", str(tmp_path / "x")).returncode == 4
    assert run(cli, "bench", "m.mtx", "--precision", "f16").returncode == 4
    assert run(cli, "bench", "m.mtx", "--iters", "x").returncode == 64
    r = run(cli, "gen", "walkthrough", "--out", str(tmp_path / "no" / "dir" / "w.mtx"))
    assert r.returncode == 3  # io_error
