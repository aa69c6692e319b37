"""Regenerate tests/golden/*.json from the REAL reference (oracle/_ref).

Run in the build container (needs /root/reference for oracle/_ref):
    make -C oracle all && python tests/golden/make_golden.py
The JSON files are committed; tests/test_oracle.py pins the C restatement and
the GPU tests pin the device path against them without /root/reference.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIGS = [(32, 14, 128), (32, 7, 128), (4, 4, 16)]


def h(*arrays):
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:32]


def main():
    R = O.ref()
    assert R is not None, "oracle/_ref not built (make -C oracle ref)"
    # --- walkthrough (fixtures.hpp:17-36; test_format.cpp:59-110) ---
    a = O.walkthrough()
    walk = {"row_offsets": a.row_offsets.tolist(), "col_indices": a.col_indices.tolist(),
            "path": "".join("RD"[s] for s in O.sequential_path(a.row_offsets, 8, 34)),
            "tiles": {}, "y_unit": R.spmv_csr(a, np.ones(8)).tolist()}
    for (w, s) in [(4, 4), (32, 14), (32, 7)]:
        tx, ty, ld = R.generate_tile(a.row_offsets, 8, 34, w, s)
        walk["tiles"][f"{w},{s}"] = {"tile_x": tx.tolist(), "tile_y": ty.tolist(),
                                     "lane_desc": ld.tolist()}
    lanes = []
    for d in range(0, 42, 4):
        x, y, _ = R.merge_search(a.row_offsets, 8, 34, d)
        lanes.append([x, y])
    walk["lane_starts_4_4"] = lanes
    json.dump(walk, open(os.path.join(HERE, "walkthrough.json"), "w"), indent=1)

    # --- fuzz corpus (acceptance.cpp:49-57): CSR, TILE and y hashes ---
    corpus = []
    for seed in range(1, 85):
        for si, shape in enumerate(O.SHAPES):
            m = R.random_matrix(shape, seed)
            x = R.seed_test_vector(m.n_cols, -1.0, 1.0, seed)
            e = {"seed": seed, "shape": shape, "n_rows": m.n_rows, "n_cols": m.n_cols,
                 "nnz": m.nnz, "csr": h(m.row_offsets, m.col_indices, m.values),
                 "x": h(x), "tiles": {}, "y_csr_f64": h(R.spmv_csr(m, x))}
            for (w, s, b) in CONFIGS:
                tx, ty, ld = R.generate_tile(m.row_offsets, m.n_rows, m.nnz, w, s)
                ymb, cnt = R.spmv_merbit(m, x, w, s, b)
                e["tiles"][f"{w},{s}"] = {"tile": h(tx, ty, ld), "y_merbit_f64": h(ymb),
                                         "trace": cnt.tolist()}
            corpus.append(e)
    json.dump(corpus, open(os.path.join(HERE, "fuzz_corpus.json"), "w"))

    # --- PageRank (test_solvers.cpp:61-124, acceptance.cpp:362-397) ---
    ring = R.ring_with_chords(100, 260, 42)
    p = R.build_transition(ring)
    r = R.pagerank_csr(p)
    pr = {"ring_100_260_42": {"pi": r["pi"].tolist(), "iterations": r["iterations"],
                              "final_err": r["final_err"], "status": r["status"],
                              "p_hash": h(p.row_offsets, p.col_indices, p.values)}}
    # fixed-iteration fp32 run (reference_iters=0) of the same graph
    p32 = p.astype(np.float32)
    r32 = R.pagerank_csr(p32, 0.85, 1e-30, 50, 0)
    pr["ring_f32_50it"] = {"pi": r32["pi"].astype(np.float64).tolist(),
                           "iterations": r32["iterations"]}
    json.dump(pr, open(os.path.join(HERE, "pagerank.json"), "w"), indent=1)
    print("golden written:", len(corpus), "fuzz matrices")


if __name__ == "__main__":
    main()
