"""Per-kernel device time of one (warm) degree relabelling at R-MAT s24 from
CUPTI records (torch.profiler), not replayed: where the preprocessing goes."""
import collections
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ctx = mb.Context(0)
P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
Q, _ = P.relabel_by_degree(want_rank=False)
del Q
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    Q, _ = P.relabel_by_degree(want_rank=False)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += e.time_range.elapsed_us()
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"{v[0]:4d} {v[1]/1e3:9.3f} ms {100*v[1]/tot:5.1f}% {k}")
print(f"total {tot/1e3:.3f} ms")
