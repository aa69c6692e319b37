"""Where does the one-shot mbx_pagerank call spend its time?  (plan create /
run / result / copies / destroy, wall clock)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True)
c = mb.SimtConfig.make(32, 14, 128)
t = mb.generate_tile_for(P, c)
cfg = mb.PageRankConfig(0.85, 1e-30, 100, 0)
L = _lib.lib()
for rep in range(3):
    t0 = time.perf_counter()
    plan = mb.PageRankPlan(P, t, c, cfg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan.run()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res, _ = plan.result()
    t3 = time.perf_counter()
    plan.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print({"create_ms": (t1 - t0) * 1e3, "run_ms": (t2 - t1) * 1e3, "result_ms": (t3 - t2) * 1e3,
           "destroy_ms": (t4 - t3) * 1e3, "iterate_ms": res.iterate_seconds * 1e3}, flush=True)
pi0 = torch.full((P.n_rows,), 1.0 / P.n_rows).pin_memory()
pi = torch.empty(P.n_rows).pin_memory()
cc, pc = c._c(), cfg._c()
rr = _lib.mbx_pagerank_result()
for rep in range(3):
    t0 = time.perf_counter()
    rc = L.mbx_pagerank(ctx.h, P.h, t.h, C.byref(cc), C.byref(pc), pi0.data_ptr(), pi.data_ptr(),
                        None, None, C.byref(rr))
    assert rc == 0
    print({"oneshot_ms": (time.perf_counter() - t0) * 1e3, "iterate_ms": rr.iterate_seconds * 1e3},
          flush=True)
