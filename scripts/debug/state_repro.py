"""Process-state repro: small SpMVs with the given (omega, sigma, block, dtype)
configs on a fresh context, then row 0 of an R-MAT s13 transition SpMV
(block 64) against the fp64 oracle.  argv: configs like 4,4,4,f64 32,7,64,f32."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O  # noqa: E402
import paper_2605_07391_b200 as mb  # noqa: E402

ctx = mb.Context(0)
ctx.set_layout(1)
a = O.walkthrough()
for spec in sys.argv[1:]:
    w, s, b, dt = spec.split(",")
    d = np.float64 if dt == "f64" else np.float32
    m = mb.DeviceMatrix.from_csr(ctx, a.astype(d))
    c = mb.SimtConfig.make(int(w), int(s), int(b))
    t = mb.generate_tile_for(m, c)
    y = mb.spmv_merbit(m, t, c, np.ones(8, d), mb.DualBuffer(8, d))
P = mb.DeviceMatrix.rmat(ctx, 13, 16, seed=5, transition=True, dtype=np.float32)
n = P.n_rows
c2 = mb.SimtConfig.make(32, 14, 64)
t2 = mb.generate_tile_for(P, c2)
x = O.hash_uniform(3, n, 0.0, 1.0, np.float32)
y2 = mb.spmv_merbit(P, t2, c2, x, mb.DualBuffer(n, np.float32))
ro, cols, vals = P.download()
want = O.spmv_csr_f64(O.Csr(n, n, ro, cols, vals.astype(np.float64)), x.astype(np.float64))
bad = np.nonzero(np.abs(y2 - want) > 1e-4 * np.maximum(1, np.abs(want)))[0]
print(" ".join(sys.argv[1:]) or "(none)", "-> bad rows", bad.size, bad[:5], y2[0], want[0], flush=True)
