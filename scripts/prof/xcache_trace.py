"""Kernel / runtime-API timeline of one build_xcache (torch.profiler, CUPTI):
python scripts/prof/xcache_trace.py [scale] [relabel 0|1]."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
relabel = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = mb.Context(0)
A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
if relabel:
    A, _ = A.relabel_by_degree(want_rank=False)
for _ in range(2):
    A.build_xcache()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    secs = A.build_xcache()
print(f"build_xcache {secs * 1e3:.3f} ms, hubs {A.xcache_info()[0]}")
evs = sorted(prof.events(), key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start if evs else 0
for e in evs[:int(os.environ.get("HEAD", "100000"))]:
    if e.device_type == torch.autograd.DeviceType.CUDA or e.name.startswith("cuda"):
        print(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  {(e.time_range.end - e.time_range.start):8.1f} us  "
              f"{'GPU' if e.device_type == torch.autograd.DeviceType.CUDA else 'API'}  {e.name[:90]}")
