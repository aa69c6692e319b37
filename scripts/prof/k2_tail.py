"""K2 warp finish-time spread (build with -DMBX_EXP_TAIL: exp/tail):
  MBX_LIB_PATH=exp/tail/libmerbit_b200.so python scripts/prof/k2_tail.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200 import _lib  # noqa: E402

ctx = mb.Context(0)
scale = int(os.environ.get("SCALE", "24"))
P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
if scale >= 24:
    P, _ = P.relabel_by_degree(want_rank=False)
c = mb.SimtConfig.make(32, 14, 128)
t = mb.generate_tile_for(P, c)
P.build_xcache()
buf = np.zeros(2 * 8192, np.uint64)


def report(tag):
    torch.cuda.synchronize()
    _lib.lib().mbx_exp_warp_times(buf.ctypes.data_as(C.c_void_p))
    st, en = buf[:8192].astype(np.int64), buf[8192:].astype(np.int64)
    k = int(np.count_nonzero(en))
    st, en = st[:k], en[:k]
    t0 = st.min()
    span = (en.max() - t0) / 1e3
    e = np.sort((en - t0) / 1e3)
    print(f"{tag}: warps {k}, span {span:.1f} us, start spread {(st.max() - t0) / 1e3:.1f} us, "
          f"finish p10 {e[k // 10]:.1f} p50 {e[k // 2]:.1f} p90 {e[9 * k // 10]:.1f} "
          f"p99 {e[99 * k // 100]:.1f} max {e[-1]:.1f} us; idle share "
          f"{1 - e.mean() / e[-1]:.3f}", flush=True)


x = torch.rand(P.n_cols, device="cuda")
y = torch.empty(P.n_rows, device="cuda")
for _ in range(3):
    mb.spmv_device(P, t, c, x.data_ptr(), y.data_ptr())
    report(f"spmv s{scale} f32")
plan = mb.PageRankPlan(P, t, c, mb.PageRankConfig(0.85, 1e-30, 10, 0))
for _ in range(3):
    plan.run()
    report("pagerank K2 (last iteration)")
