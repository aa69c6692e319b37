"""Profiling / A-B driver: the bench's fused PageRank iteration on R-MAT
(degree-relabelled, hub table), `iters` iterations per run.

  python scripts/prof/pr_iter.py [scale] [iters] [runs]

Prints us/iteration (CUDA events over `runs` runs after one warm-up).  Under
ncu use MBX_GRAPH_MODE=unrolled (ncu does not descend into conditional graph
nodes) and e.g. -k regex:spmv_slot --launch-skip 2 -c 1."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 5
natural = os.environ.get("ORDER", "degree") == "natural"
ctx = mb.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
if os.environ.get("SMEM") or os.environ.get("MODE"):
    # K2 shared-memory budget per SM and staging mode (0 LDG, 1 L2 prefetch,
    # 2 TMA bulk staging of the next tile's columns + descriptors)
    ctx.set_tuning(32, 1, -1, smem_per_sm=int(os.environ.get("SMEM", -1)),
                   prefetch=int(os.environ.get("MODE", -1)))
P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
if not natural:
    P, _ = P.relabel_by_degree(want_rank=False)
c = mb.SimtConfig.make(32, 14, 128)
t = mb.generate_tile_for(P, c)
P.build_xcache()
plan = mb.PageRankPlan(P, t, c, mb.PageRankConfig(0.85, 1e-30, iters, 0))
pi0 = None
warm = int(os.environ.get("PI0WARM", "0"))
if warm:
    # start from the iterate after `warm` iterations (data-dependence check)
    wp = mb.PageRankPlan(P, t, c, mb.PageRankConfig(0.85, 1e-30, warm, 0))
    wp.run()
    torch.cuda.synchronize()
    pi0_t = torch.empty(P.n_rows, dtype=torch.float32, device="cuda")
    import ctypes
    ctypes.CDLL("libcudart.so.12").cudaMemcpy(ctypes.c_void_p(pi0_t.data_ptr()),
                                              ctypes.c_void_p(wp.pi_ptr()),
                                              ctypes.c_size_t(4 * P.n_rows), 3)
    pi0 = pi0_t.data_ptr()
plan.run(pi0)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(runs):
    plan.run(pi0)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
res, _ = plan.result()
print(f"scale {scale} {'natural' if natural else 'degree'} smem {os.environ.get('SMEM', '-')} "
      f"mode {os.environ.get('MODE', '-')} hubs {P.xcache_info()[0]}: "
      f"{ms * 1e3 / (runs * iters):.1f} us/iteration "
      f"({runs * iters / (ms * 1e-3):.0f} it/s), mass {res.mass:.9f}, resid {res.l1_residual:.3e}",
      flush=True)
