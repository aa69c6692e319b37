"""Two PageRank plans over the same s24 matrix (and the context's cached plan
behind mbx_pagerank), timed alternately: does buffer placement matter?
  python scripts/prof/plan_pair.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200 import _lib  # noqa: E402

ctx = mb.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
P = mb.DeviceMatrix.rmat(ctx, 24, 16, seed=1, transition=True, dtype=np.float32)
P, _ = P.relabel_by_degree(want_rank=False)
c = mb.SimtConfig.make(32, 14, 128)
t = mb.generate_tile_for(P, c)
P.build_xcache()
prc = mb.PageRankConfig(0.85, 1e-30, 100, 0)
plans = [mb.PageRankPlan(P, t, c, prc) for _ in range(2)]
n = P.n_rows
pi0 = torch.full((n,), 1.0 / n, dtype=torch.float32).pin_memory()
pio = torch.empty(n, dtype=torch.float32).pin_memory()
pi0d = torch.full((n,), 1.0 / n, dtype=torch.float32, device="cuda")
L = _lib.lib()
cc, pc = c._c(), prc._c()
rr = _lib.mbx_pagerank_result()


def cached():
    assert L.mbx_pagerank(ctx.h, P.h, t.h, C.byref(cc), C.byref(pc), pi0.data_ptr(),
                          pio.data_ptr(), None, None, C.byref(rr)) == 0


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for f in (plans[0].run, plans[1].run, cached):
    f()
res = {"A": [], "B": [], "A_pi0dev": [], "cached_e2e": []}
for _ in range(4):
    res["A"].append(timed(plans[0].run))
    res["B"].append(timed(plans[1].run))
    res["A_pi0dev"].append(timed(lambda: plans[0].run(pi0d.data_ptr())))
    res["cached_e2e"].append(timed(cached))
for k, v in res.items():
    print(f"{k}: median {sorted(v)[len(v) // 2]:.2f} ms  {['%.2f' % x for x in v]}", flush=True)
