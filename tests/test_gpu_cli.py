"""GPU: the merbit_b200 CLI verbs end to end on fixtures it
generates itself, checked against the oracle (pinned to the reference) and
the reference's own writers: bicgstab / pagerank reports, breakdown exit code,
validate, bench rows (BenchRecord identities), convert caches, sigma-sweep."""
import csv
import io
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "merbit_b200")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    return CLI


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_bicgstab_verb(cli, tmp_path):
    lap = tmp_path / "lap.mtx"
    assert run(cli, "gen", "laplacian", "--grid", 32, "--out", lap).returncode == 0
    r = run(cli, "bicgstab", lap)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["status"] == "converged" and rep["final_residual"] < 1e-10
    a = O.five_point_laplacian(32)
    want = O.bicgstab(a, O.seed_test_vector(a.n_rows, -1, 1, 1))  # the CLI's b (seed 1)
    assert abs(rep["iterations"] - want["iterations"]) <= 2
    assert rep["rows"] == a.n_rows and rep["nnz"] == a.nnz
    sing = tmp_path / "s.mtx"
    run(cli, "gen", "singular", "--out", sing)
    r = run(cli, "bicgstab", sing, "--omega", 4, "--sigma", 4)
    assert r.returncode == 5  # kExitBreakdown
    rep = json.loads(r.stdout)
    assert rep["status"] == "breakdown" and rep["breakdown"] in ("rhat_dot_v", "rho")


def test_pagerank_verb(cli, tmp_path):
    ring = tmp_path / "ring.mtx"
    run(cli, "gen", "ring", "--nodes", 100, "--chords", 260, "--seed", 42, "--out", ring)
    r = run(cli, "pagerank", ring)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    p = O.build_transition(O.ring_with_chords(100, 260, 42))
    want = O.pagerank(p)
    assert rep["status"] == want["status"] == "converged"
    assert abs(rep["iterations"] - want["iterations"]) <= 1
    assert rep["vertices"] == 100 and rep["final_err"] < 1e-10


def test_validate_convert_and_tile_cache(cli, tmp_path):
    w = tmp_path / "walk.mtx"
    run(cli, "gen", "walkthrough", "--out", w)
    r = run(cli, "validate", w)
    assert r.returncode == 0 and "validation passed" in r.stdout, r.stdout
    assert "[FAIL]" not in r.stdout
    cache, tile = tmp_path / "walk.mbmx", tmp_path / "walk.mbtl"
    r = run(cli, "convert", w, "--out", cache, "--tile", tile, "--precision", "f32",
            "--omega", 4, "--sigma", 4)
    assert r.returncode == 0, r.stderr
    a = O.walkthrough()
    if O.ref() is not None:
        theirs = tmp_path / "ref.mbtl"
        O.ref().tile_cache_write(str(theirs), a.row_offsets, 8, 34, 4, 4, False)
        assert tile.read_bytes() == theirs.read_bytes()
    r = run(cli, "validate", cache, "--tile", tile)
    assert r.returncode == 0 and "reproduces the merge path" in r.stdout
    bad = bytearray(tile.read_bytes())
    bad[33 + 4] ^= 0x01  # tile_x[1] (header: magic, version, omega, sigma, nnz, n_rows, prec)
    (tmp_path / "bad.mbtl").write_bytes(bytes(bad))
    r = run(cli, "validate", cache, "--tile", tmp_path / "bad.mbtl")
    assert r.returncode == 2  # kExitValidation


def test_bench_rows(cli, tmp_path):
    lap = tmp_path / "lap.mtx"
    run(cli, "gen", "laplacian", "--grid", 64, "--out", lap)
    r = run(cli, "bench", lap, "--kernels", "coo,csr,merge,merge-cub,merbit", "--iters", 50,
            "--warmup", 5)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert [x["kernel"] for x in rows] == ["coo", "csr", "merge", "merge-cub", "merbit"]
    for x in rows:
        mean, base, nnz = float(x["mean_seconds"]), float(x["baseline_seconds"]), int(x["nnz"])
        assert float(x["ct"]) == 2.0 * nnz / mean  # bitwise after the text round trip
        assert float(x["speedup"]) == base / mean
        assert x["schema"] == "1" and x["precision"] == "f64"
    merbit = rows[-1]
    assert int(merbit["omega"]) == 32 and int(merbit["sigma"]) == 7
    assert float(merbit["preprocess_seconds"]) > 0 and float(merbit["metadata_bytes"]) > 0
    rj = run(cli, "bench", lap, "--kernels", "merbit", "--iters", 10, "--format", "json")
    assert json.loads(rj.stdout)[0]["kernel"] == "merbit"


def test_sigma_sweep(cli, tmp_path):
    w = tmp_path / "walk.mtx"
    run(cli, "gen", "walkthrough", "--out", w)
    r = run(cli, "sigma-sweep", w, "--sigmas", "1-20", "--iters", 5, "--precision", "f32")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    for x in rows:
        s = int(x["sigma"])
        ob = int(np.ceil(np.log2(32 * s)))
        assert x["feasible"] == ("1" if 2 * ob + s <= 32 else "0"), s
        if x["feasible"] == "1":
            assert x["validated"] == "1"
