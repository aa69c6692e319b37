"""Slot-copy check: SpMV with and without the x hub cache (bitwise), and the
slot copy decoded back to CSR (compact round trip), for a few TILE shapes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O  # noqa: E402
import paper_2605_07391_b200 as mb  # noqa: E402

ctx = mb.Context(0)
for scale, relabel, block, dt in [(13, 0, 64, np.float32), (13, 0, 128, np.float32),
                                  (13, 1, 64, np.float32), (13, 0, 64, np.float64),
                                  (16, 0, 128, np.float32)]:
    P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=5, transition=True, dtype=dt)
    if relabel:
        P, _ = P.relabel_by_degree(want_rank=False)
    n = P.n_rows
    c = mb.SimtConfig.make(32, 14 if dt == np.float32 else 7, block)
    t = mb.generate_tile_for(P, c)
    x = O.hash_uniform(3, n, 0.0, 1.0, dt)
    y0 = mb.spmv_merbit(P, t, c, x, mb.DualBuffer(n, dt))
    ro, cols, vals = P.download()
    P.build_xcache(1 << 30)  # forced: small matrices get no table automatically
    y1 = mb.spmv_merbit(P, t, c, x, mb.DualBuffer(n, dt))
    hubs = P.xcache_info()[0]
    P.compact(t)
    ro2, cols2, vals2 = P.download()
    bad = np.nonzero(y0 != y1)[0]
    print(f"s{scale} relabel {relabel} block {block} {dt.__name__} hubs {hubs}: "
          f"y mismatches {bad.size} {bad[:8]} cols equal {np.array_equal(cols, cols2)} "
          f"vals equal {np.array_equal(vals, vals2)}", flush=True)
    if not np.array_equal(cols, cols2):
        d = np.nonzero(cols != cols2)[0]
        print("  first col diffs", d[:8], cols[d[:8]], cols2[d[:8]])
