#!/usr/bin/env python
"""Benchmark of the MERBIT hot path on B200 (contract: see DESIGN.md).

Workload at N=1 (BASELINE.json configs[1]): PageRank, 100 fixed iterations
(reference_iters=0, err_tol=1e-30 so every run does all 100), fp32, on the
transition matrix of a synthetic R-MAT scale-24 graph (edge factor 16,
Graph500 a,b,c,d, duplicates merged, natural vertex order), TILE built once
(preprocessing amortised).  One "step" = one 100-iteration PageRank run.

  value      iterations/s with the matrix resident in HBM (CUDA graph replay)
  e2e        same metric through the one-shot C-ABI call mbx_pagerank with
             pinned HOST buffers (pi0 in, pi out) inside the timed region
  roofline   one fused PageRank iteration (K2 spmv_w32<float,14,PR> + K3
             fixup) against measured HBM copy bandwidth: algorithmic bytes
             8m + 16n + 4 per iteration
  spmv       the plain SpMV (K2+K3) on the same matrix: GFLOP/s = 2m/t and
             GB/s over 8m + 12n + 4
  cpu_baseline  the reference's own MerbitBackend<float> PageRank
             (oracle/_ref, ThreadPool(nproc)) on this box's host cores

--impl reference runs only that CPU reference arm and prints its line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV GFLOP/s & HBM GB/s vs roofline; PageRank iters/sec at 1/2/4/8 B200"


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.samples.append([s.strip() for s in line.split(",")])
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                smax.append(float(s[1]))
                for k, name in enumerate(names):
                    if s[4 + k].lower().startswith("active"):
                        reasons.add(name)
            except (ValueError, IndexError):
                continue
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_pagerank(ro, cols, n, iters_per_step, steps, warmup, nthreads, want_line=False):
    """The reference's pagerank<float> with MerbitBackend on ThreadPool(nthreads)
    (oracle/_ref = the unmodified reference compiled from its sources)."""
    import numpy as np

    import oracle as O
    vals = O.transition_values(n, cols, np.float32)
    a = O.Csr(n, n, ro, cols, vals)
    t0 = time.perf_counter()
    eng = O.RefEngine(a, 32, 14, 128, nthreads)
    setup = time.perf_counter() - t0
    for _ in range(warmup):
        eng.pagerank(0.85, 1e-30, iters_per_step, 0)
    secs = 0.0
    done = 0
    for _ in range(steps):
        r = eng.pagerank(0.85, 1e-30, iters_per_step, 0)
        secs += r["seconds"]
        done += r["iterations"]
    eng.close()
    return {"value": done / secs, "seconds": secs, "iterations": done,
            "preprocess_seconds": eng.preprocess_seconds, "setup_seconds": setup}


def run_reference(args):
    """--impl reference: the reference CPU implementation on this box's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle as O
    if O.ref() is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libmerbit_ref.so not built"}))
        return 0
    nthreads = os.cpu_count() or 1
    t0 = time.perf_counter()
    p = O.rmat(args.scale, 16, 1, transposed=True, nthreads=nthreads)
    gen = time.perf_counter() - t0
    iters = args.ref_iters_per_step
    r = cpu_reference_pagerank(p.row_offsets, p.col_indices, p.n_rows, iters,
                               args.steps, args.warmup, nthreads)
    v = r["value"]
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * r["seconds"] / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"pagerank fp32 R-MAT scale {args.scale} (transition, "
                               f"edge factor 16, natural order); {iters} iterations per step",
                   "scale": args.scale, "nnz": p.nnz, "n": p.n_rows, "omega": 32, "sigma": 14,
                   "block_size": 128, "threads": nthreads},
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": nthreads, "kind": "reference",
                         "sample": f"{args.steps} x {iters} PageRank iterations of the "
                                   f"reference MerbitBackend<float> on ThreadPool({nthreads})"},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_preprocess_seconds": r["preprocess_seconds"],
        "input_generation_seconds": gen,
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--iters", type=int, default=100, help="PageRank iterations per step")
    ap.add_argument("--block-size", type=int, default=128)
    ap.add_argument("--ref-iters-per-step", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--spmv-reps", type=int, default=50)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    import paper_2605_07391_b200 as mb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        raise SystemExit("multi-GPU bench path: see bench_multi (not in this build)")
    torch.cuda.set_device(local)
    # A real (non-NULL) stream shared by torch events and the library: the
    # library never runs on the legacy default stream.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = mb.Context(local)
    ctx.set_stream(stream.cuda_stream)

    scale = args.scale
    t0 = time.perf_counter()
    P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
    gen_s = time.perf_counter() - t0
    n, m = P.n_rows, P.nnz
    cfg = mb.SimtConfig.make(32, 14, args.block_size)
    tile = mb.generate_tile_for(P, cfg)
    prc = mb.PageRankConfig(0.85, 1e-30, args.iters, 0)
    plan = mb.PageRankPlan(P, tile, cfg, prc)

    for _ in range(args.warmup):
        plan.run()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        plan.run()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launch_count - launches0
    clocks = sampler.stop()
    ms_total = ev0.elapsed_time(ev1)
    res, hist = plan.result(want_history=True)
    assert res.iterations == args.iters
    iters_per_s = args.iters * args.steps / (ms_total * 1e-3)
    t_iter = ms_total * 1e-3 / (args.iters * args.steps)
    peak, peak_kind = measured_peak()
    b_iter = 8 * m + 16 * n + 4
    achieved = b_iter / t_iter / 1e9

    # plain SpMV on the same matrix (K2 + K3), device buffers
    x = torch.rand(n, device="cuda", dtype=torch.float32)
    y = torch.empty(n, device="cuda", dtype=torch.float32)
    for _ in range(5):
        mb.spmv_device(P, tile, cfg, x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.spmv_reps):
        mb.spmv_device(P, tile, cfg, x.data_ptr(), y.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    t_spmv = e0.elapsed_time(e1) * 1e-3 / args.spmv_reps
    b_spmv = 8 * m + 12 * n + 4

    # e2e: one-shot C-ABI call with pinned host buffers (pi0 in, pi out)
    pi0 = torch.full((n,), 1.0 / n, dtype=torch.float32).pin_memory()
    pi_out = torch.empty(n, dtype=torch.float32).pin_memory()
    import ctypes as C

    from paper_2605_07391_b200 import _lib
    L = _lib.lib()
    cc, pc = cfg._c(), prc._c()
    rr = _lib.mbx_pagerank_result()

    def e2e_call():
        rc = L.mbx_pagerank(ctx.h, P.h, tile.h, C.byref(cc), C.byref(pc), pi0.data_ptr(),
                            pi_out.data_ptr(), None, None, C.byref(rr))
        if rc:
            raise RuntimeError(L.mbx_last_error().decode())
    e2e_call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_call()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_val = args.iters / e2e_s
    mass = float(pi_out.double().sum())

    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        import oracle as O
        if O.ref() is not None:
            ro, cols, _ = P.download(want_values=False)
            nthreads = os.cpu_count() or 1
            r = cpu_reference_pagerank(ro, cols, n, 2, 3, 1, nthreads)
            cpu = {"value": r["value"], "unit": "iters/s", "cores": nthreads,
                   "kind": "reference",
                   "sample": f"3 x 2 PageRank iterations (after 1 warm-up) of the reference "
                             f"MerbitBackend<float> on ThreadPool({nthreads}), same scale-{scale}"
                             f" transition matrix; reference generate_tile took "
                             f"{r['preprocess_seconds']:.2f} s"}
    line = {
        "metric": METRIC, "value": iters_per_s, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"pagerank {args.iters} iterations fp32, R-MAT scale {scale} "
                               f"transition (edge factor 16, natural vertex order), "
                               f"preprocessing amortised",
                   "scale": scale, "n": n, "nnz": m, "omega": 32, "sigma": 14,
                   "block_size": args.block_size,
                   "l2": "inputs (values+cols ~%.1f GB) larger than L2; no flush" % (8 * m / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                     "kernel": "PageRank iteration: spmv_w32_kernel<float,14,PR> + fixup",
                     "bytes_per_launch": b_iter},
        "spmv": {"ms": t_spmv * 1e3, "gflops": 2 * m / t_spmv / 1e9,
                 "gbs": b_spmv / t_spmv / 1e9, "frac": b_spmv / t_spmv / 1e9 / peak,
                 "bytes": b_spmv},
        "preprocess_ms": tile.preprocess_seconds * 1e3,
        "preprocess_over_spmv": tile.preprocess_seconds / t_spmv,
        "e2e": {"value": e2e_val, "unit": "iters/s", "h2d_bytes_per_step": 4 * n,
                "d2h_bytes_per_step": 4 * n, "mass": mass},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "l1_residual_last": res.l1_residual,
        "input_generation_seconds": gen_s,
    }
    if rank == 0:
        print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
