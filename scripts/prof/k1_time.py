"""K1 (generate_tile) time on the bench matrices: python scripts/prof/k1_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402

ctx = mb.Context(0)
tag = os.environ.get("TAG", "")
for name, make, sig in [("s24", lambda: mb.DeviceMatrix.rmat(ctx, 24, 16, seed=1, transition=True,
                                                            dtype=np.float32), 14),
                        ("s24f64", None, 7),
                        ("c5", lambda: mb.DeviceMatrix.stencil27(ctx, 400, np.float32), 14),
                        ("c5f64", None, 7)]:
    if make is not None:
        A = make()
    c = mb.SimtConfig.make(32, sig, 128)
    ts = []
    for _ in range(6):
        t = mb.generate_tile_for(A, c)
        ts.append(t.preprocess_seconds * 1e3)
        del t
    print(f"{tag} {name}: tile {min(ts[1:]):.3f} ms (median {sorted(ts[1:])[2]:.3f})", flush=True)
