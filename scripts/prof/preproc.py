"""Preprocessing split (TILE, x hub cache, slot copy) against one SpMV, repeated
so first-use costs (memory pool growth, module loading) show separately:
python scripts/prof/preproc.py [case ...], cases s24, s24r (degree-relabelled),
s24f64, s24rf64, s20, c3 (power-law f64), c5, c5f64.  LAYOUT=0 runs K2 on
the staged CSR order (no slot copy); MODE= sets K2's next-tile staging."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402

cases = sys.argv[1:] or ["s24", "s24r", "s24f64", "s24rf64", "s20", "c5"]
ctx = mb.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
if os.environ.get("LAYOUT"):
    ctx.set_layout(int(os.environ["LAYOUT"]))
if os.environ.get("MODE"):  # K2 next-tile staging: 0 none, 1 L2 prefetch, 2 TMA
    ctx.set_tuning(32, 1, -1, prefetch=int(os.environ["MODE"]))


def make(case):
    dt = np.float64 if "f64" in case else np.float32
    if case.startswith("c3"):
        return mb.DeviceMatrix.powerlaw(ctx, 22, seed=3, dtype=np.float64), np.float64
    if case.startswith("c5"):
        return mb.DeviceMatrix.stencil27(ctx, 400, dt), dt
    scale = int(case[1:3])
    A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=dt)
    if case[3:4] == "r":
        A, _ = A.relabel_by_degree(want_rank=False)
    return A, dt


for case in cases:
    A, dt = make(case)
    c = mb.SimtConfig.make(32, 14 if dt == np.float32 else 7, 128)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    x = torch.rand(A.n_cols, device="cuda", dtype=tdt)
    y = torch.empty(A.n_rows, device="cuda", dtype=tdt)
    torch.cuda.synchronize()
    rows = []
    for rep in range(3):
        t = mb.generate_tile_for(A, c)
        xc = A.build_xcache()
        w0 = time.perf_counter()
        mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())  # builds the slot copy
        ctx.synchronize()
        first = time.perf_counter() - w0
        rows.append((t.preprocess_seconds * 1e3, xc * 1e3, A.slot_info()[1] * 1e3, first * 1e3))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
    e0.record(s)
    for _ in range(20):
        mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
    e1.record(s)
    torch.cuda.synchronize()
    sp = e0.elapsed_time(e1) / 20
    best = [min(r[i] for r in rows) for i in range(4)]
    print(f"{case}: nnz {A.nnz} hubs {A.xcache_info()[0]} sectors/32 {A.gather_sectors():.1f} "
          f"spmv {sp:.3f} ms | "
          + " | ".join(f"rep{i} tile {r[0]:.3f} xc {r[1]:.3f} slots {r[2]:.3f} first {r[3]:.3f}"
                       for i, r in enumerate(rows))
          + f" || best pre {sum(best[:3]):.3f} ms = {sum(best[:3]) / sp:.2f}x spmv; "
          f"first-rep pre {sum(rows[0][:3]):.3f} ms = {sum(rows[0][:3]) / sp:.2f}x; "
          f"ysum {float(y.double().sum()):.9e}", flush=True)
    del A, t, x, y
    torch.cuda.synchronize()
