#!/usr/bin/env python
"""Benchmark of the MERBIT hot path on B200 (contract and derivations: DESIGN.md).

Workload (BASELINE.json configs[1]): PageRank, 100 fixed iterations
(reference_iters=0, err_tol=1e-30, so every run does all 100), fp32, on the
transition matrix of a synthetic R-MAT graph (default scale 24: edge factor
16, Graph500 a,b,c,d, duplicates merged; vertices relabelled by degree on the
device as preprocessing, --vertex-order natural keeps R-MAT's numbering),
TILE built once (preprocessing amortised).  One "step" = one 100-iteration
PageRank run.  At N>1 GPUs (torchrun) the SAME matrix is row-sharded
(cost-weighted cut) and pi is exchanged every iteration, by default with P2P
stores fused into the commit (--exchange nccl: one ncclAllGather; chosen
automatically when the GPUs have no peer access): strong scaling.
--scale 27 gives BASELINE config C4.

  value      iterations/s, matrix resident in HBM (CUDA-graph replay), max
             over ranks of the device time
  e2e        same metric with pinned HOST buffers inside the timed region:
             N=1 the one-shot C-ABI call mbx_pagerank (pi0 in, pi out);
             N>1 each rank's pi0 slice H2D + run + its pi slice D2H
  roofline   the fused PageRank iteration on one GPU (K2 spmv_slot_kernel + K3
             fixup) vs measured HBM copy bandwidth; algorithmic bytes per
             iteration 8m + 16n + 4 (fp32)
  spmv       plain SpMV (K2+K3) on the same matrix (fp32) and on an fp64
             R-MAT of the same scale: GFLOP/s = 2m/t, GB/s over 8m+12n+4 /
             12m+20n+4
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
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_per_launch():
    """DRAM bytes (read + write) of one fused PageRank iteration (K2 + K3) at
    scale 24, from the committed `ncu --set full` capture summarised in
    profiles/ncu_traffic.json (null when absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d["pagerank_iteration_s24_f32"]["dram_bytes"]
    except Exception:
        return None


def gather_ceiling():
    """Measured ceiling of scattered 4-byte gathers from an L2-resident array
    (scripts/micro/dsmem_gather.cu, case global_64MB, all 148 SMs) -- the
    bound of an SpMV whose x is gathered at random (null when absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1s2_dsmem_gather.jsonl")) as f:
            for line in f:
                d = json.loads(line)
                if d.get("case") == "global_64MB":
                    return float(d["gathers_per_s"])
    except Exception:
        pass
    return None


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_reference_pagerank(ro, cols, n, iters_per_step, steps, warmup, nthreads):
    """The reference's pagerank<float> with MerbitBackend on ThreadPool(nthreads)
    (oracle/_ref = the unmodified reference compiled from its sources)."""
    import numpy as np

    import oracle as O
    vals = O.transition_values(n, cols, np.float32)
    a = O.Csr(n, n, ro, cols, vals)
    eng = O.RefEngine(a, 32, 14, 128, nthreads)
    for _ in range(warmup):
        eng.pagerank(0.85, 1e-30, iters_per_step, 0)
    secs, done = 0.0, 0
    for _ in range(steps):
        r = eng.pagerank(0.85, 1e-30, iters_per_step, 0)
        secs += r["seconds"]
        done += r["iterations"]
    pre = eng.preprocess_seconds
    eng.close()
    return {"value": done / secs, "seconds": secs, "iterations": done, "preprocess_seconds": pre}


def c1_numbers(mb, ctx, stream, peak, with_ref):
    """BASELINE config 1: R-MAT scale 20 fp32 (values U[0,1)), MERBIT
    preprocessing (TILE + hub table + slot copy, wall clock incl. syncs) and
    one SpMV on the device, beside the reference's generate_tile and one
    spmv_merbit on ThreadPool(nproc) (oracle/_ref) for the same matrix."""
    import numpy as np
    import torch
    A = mb.DeviceMatrix.rmat(ctx, 20, 16, seed=1, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    x = torch.rand(A.n_cols, device="cuda", dtype=torch.float32)
    y = torch.empty(A.n_rows, device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = mb.generate_tile_for(A, c)
    A.build_xcache()
    mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())  # builds the slot copy
    torch.cuda.synchronize()
    first_s = time.perf_counter() - t0
    # steady-state preprocessing split (device-timed TILE and slot copy, the
    # hub table's wall clock incl. its one host sync)
    t = mb.generate_tile_for(A, c)
    xc_s = A.build_xcache()
    mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
    ctx.synchronize()
    split = (t.preprocess_seconds, xc_s, A.slot_info()[1])
    ts = time_device(stream, lambda: mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr()), 50)
    m, n = A.nnz, A.n_rows
    b = 8 * m + 12 * n + 4
    out = {"matrix": "R-MAT scale 20 fp32, values U[0,1)", "nnz": m, "n": n,
           "tile_ms": t.preprocess_seconds * 1e3,
           "preprocess_plus_first_spmv_ms": first_s * 1e3, "spmv_ms": ts * 1e3,
           "preprocess_ms": sum(split) * 1e3, "preprocess_tile_ms": split[0] * 1e3,
           "preprocess_xcache_ms": split[1] * 1e3, "preprocess_slots_ms": split[2] * 1e3,
           "preprocess_over_spmv": sum(split) / ts,
           "gflops": 2 * m / ts / 1e9, "frac": b / ts / 1e9 / peak}
    out.update(comparator_numbers(A, c, x, y, stream, ts, 50))
    if with_ref:
        import oracle as O
        if O.ref() is not None:
            ro, cols, vals = A.download()
            nthreads = os.cpu_count() or 1
            eng = O.RefEngine(O.Csr(n, A.n_cols, ro, cols, vals), 32, 14, 128, nthreads)
            xh = x.cpu().numpy()
            eng.apply(xh)
            reps = 5
            t1 = time.perf_counter()
            for _ in range(reps):
                eng.apply(xh)
            ref_spmv = (time.perf_counter() - t1) / reps
            out.update({"reference_generate_tile_ms": eng.preprocess_seconds * 1e3,
                        "reference_spmv_ms": ref_spmv * 1e3, "reference_threads": nthreads,
                        "speedup_spmv": ref_spmv / ts,
                        "speedup_preprocess": eng.preprocess_seconds / t.preprocess_seconds})
            eng.close()
    return out


def run_reference(args):
    """--impl reference: the reference CPU implementation on this box's cores."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    import oracle as O
    if O.ref() is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libmerbit_ref.so not built"}))
        return 0
    nthreads = os.cpu_count() or 1
    # the same matrix as our arm: scale 24 (C2) at N = 1, 27 (C4) at N > 1
    world = int(os.environ.get("WORLD_SIZE", "1"))
    args.scale = args.scale if args.scale is not None else (24 if world == 1 else 27)
    t0 = time.perf_counter()
    p = O.rmat(args.scale, 16, 1, transposed=True, nthreads=nthreads)
    gen = time.perf_counter() - t0
    # a bounded sample per step: 2 iterations at scale 24, 1 at 27 (~2 s)
    iters = args.ref_iters_per_step if args.ref_iters_per_step else (2 if args.scale <= 25 else 1)
    r = cpu_reference_pagerank(p.row_offsets, p.col_indices, p.n_rows, iters, args.steps,
                               args.warmup, nthreads)
    v = r["value"]
    print(json.dumps({
        "metric": METRIC, "impl": "reference", "value": v, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * r["seconds"] / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"pagerank fp32, R-MAT scale {args.scale} transition (edge factor "
                               f"16, natural vertex order); {iters} iterations per step",
                   "scale": args.scale, "nnz": p.nnz, "n": p.n_rows, "omega": 32, "sigma": 14,
                   "block_size": 128, "threads": nthreads},
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": nthreads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.steps} x {iters} PageRank iterations of the reference "
                                   f"MerbitBackend<float> on ThreadPool({nthreads})"},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_preprocess_seconds": r["preprocess_seconds"],
        "input_generation_seconds": gen}))
    return 0


def single_gpu_rate(mb, stream, P, cfg, steps, iters=100):
    """PageRank iterations/s of P on this one GPU (TILE + hub table + slot
    copy, then `steps` timed runs of `iters` iterations after one warm-up);
    the derived copies are released afterwards so P can be sharded next."""
    t = mb.generate_tile_for(P, cfg)
    xc_s = P.build_xcache()
    plan = mb.PageRankPlan(P, t, cfg, mb.PageRankConfig(0.85, 1e-30, iters, 0))
    pre_ms = (t.preprocess_seconds + xc_s + P.slot_info()[1]) * 1e3
    plan.run()
    ts = time_device(stream, plan.run, steps)
    res, _ = plan.result()
    plan.close()
    del t
    P.release_caches()
    return {"n_gpus": 1, "iters_per_s": iters / ts, "us_per_iteration": ts * 1e6 / iters,
            "steps": steps, "iterations_per_step": iters, "preprocess_ms": pre_ms,
            "mass": res.mass}


def time_device(stream, fn, reps):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


def reference_spmv(mb, A, sigma, sample):
    """The reference's generate_tile + spmv_merbit<T> (MerbitBackend on
    ThreadPool(nproc), oracle/_ref) on the host copy of A: one warm-up and
    three timed applies.  None when oracle/_ref is absent."""
    import numpy as np

    import oracle as O
    if O.ref() is None:
        return None
    ro, cols, vals = A.download()
    nthreads = os.cpu_count() or 1
    eng = O.RefEngine(O.Csr(A.n_rows, A.n_cols, ro, cols, vals), 32, sigma, 128, nthreads)
    x = O.hash_uniform(7, A.n_cols, -1.0, 1.0, vals.dtype)
    eng.apply(x)
    reps = 3
    t1 = time.perf_counter()
    for _ in range(reps):
        eng.apply(x)
    ts = (time.perf_counter() - t1) / reps
    out = {"sample": sample, "nnz": A.nnz, "n": A.n_rows, "threads": nthreads,
           "cpu_model": cpu_model(), "kind": "reference",
           "generate_tile_ms": eng.preprocess_seconds * 1e3, "spmv_ms": ts * 1e3,
           "gflops": 2 * A.nnz / ts / 1e9}
    eng.close()
    del ro, cols, vals
    return out


COMPARATORS = ("coo_atomic", "csr_vector", "merge_runtime", "merge_cub", "cusparse_coo_alg1",
               "cusparse_coo_alg2", "cusparse_csr_alg1", "cusparse_csr_alg2")


def comparator_numbers(A, c, x, y, stream, ts, reps):
    """The paper's comparators on the same device and inputs:
    each one's time and MERBIT's speedup over it; speedup_vs_cusparse_coo is
    the paper's headline ratio (cuSPARSE COO) against
    cuSPARSE's faster COO algorithm, speedup_vs_coo the reference's
    CooReferenceBackend on the GPU (BenchRecord.speedup)."""
    from paper_2605_07391_b200.merbit import spmv_baseline_device
    base = {}
    for kind in COMPARATORS:
        try:
            fn = (lambda k=kind: spmv_baseline_device(A, k, x.data_ptr(), y.data_ptr(), c.sigma))
            fn()
            tb = time_device(stream, fn, reps)
            base[kind] = {"ms": tb * 1e3, "gflops": 2 * A.nnz / tb / 1e9,
                          "merbit_speedup": tb / ts}
        except Exception as e:  # e.g. 32-bit offsets at > 2^31 nonzeros
            base[kind] = {"unavailable": str(e)[:120]}
    out = {"comparators": base}
    if "ms" in base.get("coo_atomic", {}):
        out["speedup_vs_coo"] = base["coo_atomic"]["ms"] * 1e-3 / ts  # BenchRecord.speedup
    coo = [base[k]["ms"] for k in ("cusparse_coo_alg1", "cusparse_coo_alg2") if "ms" in base[k]]
    if coo:
        out["speedup_vs_cusparse_coo"] = min(coo) * 1e-3 / ts
    csr = [base[k]["ms"] for k in ("cusparse_csr_alg1", "cusparse_csr_alg2") if "ms" in base[k]]
    if csr:
        out["speedup_vs_cusparse_csr"] = min(csr) * 1e-3 / ts
    return out


def spmv_numbers(mb, ctx, stream, scale, dtype, reps, peak, make=None, label=None,
                 reference=None):
    """Plain SpMV (K2+K3) on an R-MAT matrix (or make(ctx, dtype)) of the
    given precision."""
    import numpy as np
    import torch
    t_dt = torch.float32 if dtype == np.float32 else torch.float64
    vs = 4 if dtype == np.float32 else 8
    A = (make(ctx, dtype) if make else
         mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=dtype))
    c = mb.SimtConfig.make(32, 14 if vs == 4 else 7, 128)
    x = torch.rand(A.n_cols, device="cuda", dtype=t_dt)
    y = torch.empty(A.n_rows, device="cuda", dtype=t_dt)
    torch.cuda.synchronize()
    pre = []
    for _ in range(2):
        # preprocessing twice: the first pass also pays one-time costs (memory
        # pool growth for the slot copy, lazy kernel loading); the second is
        # the steady-state cost of the algorithm
        t = mb.generate_tile_for(A, c)
        xc_s = A.build_xcache()
        mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        ctx.synchronize()
        pre.append((t.preprocess_seconds, xc_s, A.slot_info()[1]))  # slot copy: first SpMV
    tile_s, xc_s, slot_s = pre[1]
    for _ in range(2):
        mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
    ts = time_device(stream, lambda: mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr()), reps)
    m, n = A.nnz, A.n_rows
    b = m * (vs + 4) + 2 * n * vs + 4 * (n + 1)
    out = {"dtype": "f32" if vs == 4 else "f64", "ms": ts * 1e3, "gflops": 2 * m / ts / 1e9,
           "gbs": b / ts / 1e9, "frac": b / ts / 1e9 / peak, "bytes": b, "nnz": m,
           "preprocess_ms": (tile_s + xc_s + slot_s) * 1e3,
           "preprocess_tile_ms": tile_s * 1e3, "preprocess_xcache_ms": xc_s * 1e3,
           "preprocess_slots_ms": slot_s * 1e3,
           "preprocess_over_spmv": (tile_s + xc_s + slot_s) / ts,
           "preprocess_first_ms": sum(pre[0]) * 1e3,
           "preprocess_first_over_spmv": sum(pre[0]) / ts,
           "xcache_hubs": A.xcache_info()[0], "xcache_coverage": A.xcache_info()[1]}
    # the same K2/K3 over the staged CSR order (layout 0: no slot copy): the
    # preprocessing / steady-state trade the slot copy makes, and after how
    # many SpMVs the copy has paid for itself
    try:
        ctx.set_layout(0)
        mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        ts0 = time_device(stream, lambda: mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr()),
                          max(3, reps // 2))
        out["staged_layout"] = {
            "ms": ts0 * 1e3, "frac": b / ts0 / 1e9 / peak,
            "preprocess_ms": (tile_s + xc_s) * 1e3,
            "preprocess_over_spmv": (tile_s + xc_s) / ts0,
            "slot_copy_pays_after_spmvs": (slot_s / (ts0 - ts)) if ts0 > ts else None}
    finally:
        ctx.set_layout(1)
    out.update(comparator_numbers(A, c, x, y, stream, ts, max(3, reps // 3)))
    if reference is not None:
        # the reference's CPU path on this box (a bounded sample when the full
        # matrix would not fit the host / time budget): reported, not a target
        try:
            if reference == "same":
                ref = reference_spmv(mb, A, c.sigma, "the same matrix")
            else:
                S = reference[0](ctx, dtype)
                ref = reference_spmv(mb, S, c.sigma, reference[1])
                del S
            if ref is not None:
                ref["gpu_speedup_gflops"] = (2 * m / ts / 1e9) / ref["gflops"]
            out["reference_cpu"] = ref
        except Exception as e:
            out["reference_cpu"] = {"unavailable": str(e)[:160]}
    if label:
        tr = mb.trace_counts(t)
        out.update({"matrix": label, "n": n, "fast_tiles": tr.fast_tiles,
                    "normal_tiles": tr.normal_tiles, "skipped_tiles": tr.skipped_tiles})
    del A, t, x, y
    torch.cuda.synchronize()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=None,
                    help="R-MAT scale (default: 24 = C2 at N = 1, 27 = C4 at N > 1)")
    ap.add_argument("--iters", type=int, default=100, help="PageRank iterations per step")
    ap.add_argument("--block-size", type=int, default=128)
    ap.add_argument("--ref-iters-per-step", type=int, default=0,
                    help="reference arm: PageRank iterations per step (0: 2 below scale 26, "
                         "else 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extras (N = 1: SpMV f32/f64, C1, C3, C5, C4 on one GPU; "
                         "N > 1: the one-GPU anchor, the NCCL exchange, C2 sharded)")
    ap.add_argument("--spmv-reps", type=int, default=30)
    ap.add_argument("--recut", action="store_true",
                    help="N > 1: re-cut the row shards from a per-rank cost probe "
                         "(off by default: the weighted cut measured better at s27)")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N > 1: fused = the commit stores into the peers' buffers (P2P, "
                         "one device barrier per iteration); nccl = one ncclAllGather")
    ap.add_argument("--vertex-order", default="degree", choices=["degree", "natural"],
                    help="degree: relabel vertices by column count on the device "
                         "(preprocessing); natural: R-MAT's own numbering")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_07391_b200 as mb
    from paper_2605_07391_b200 import _lib
    from paper_2605_07391_b200.merbit import (PeerShardGroup, ShardGroup, nccl_unique_id,
                                              prepare_rank_shard, recut_rank_shard,
                                              shard_cost_probe)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("MBX_BENCH_ONE_DEVICE") == "1":
        local = 0  # plumbing check of N > 1 on a one-GPU box (fused exchange only)
    if world > 1:
        # gloo only bootstraps (IPC blobs, NCCL id broadcast, barriers,
        # max-over-ranks); the pi exchange is the library's fused P2P stores
        # or its own NCCL all-gather.  NCCL's init log stays on so the
        # communicator's rank count is visible in the run's output.
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = mb.Context(local)
    ctx.set_stream(stream.cuda_stream)
    peak, peak_kind = measured_peak()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    extras = {}

    def peer_ok():
        """The fused exchange stores into the peers' memory: every rank must
        reach every other rank's device over P2P (NVLink), and CUDA IPC
        handles only open on one node (every rank local)."""
        ndev = torch.cuda.device_count()
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        ok = local_world == world and all(torch.cuda.can_device_access_peer(local, j)
                                          for j in range(min(world, ndev)) if j != local)
        t_ok = torch.tensor([1 if ok else 0], dtype=torch.int64)
        dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
        return int(t_ok[0]) == 1

    def make_shard_runner(exchange, n_global, bounds, Lm, tile, prc):
        if exchange == "fused":
            # the commit stores pi_new into every peer's buffer over NVLink
            # (CUDA IPC); gloo only carries the setup blobs
            g = PeerShardGroup(ctx, n_global, world, bounds, rank, Lm, tile, cfg, prc)
            blobs = [None] * world
            dist.all_gather_object(blobs, g.export())
            g.connect(blobs)
            return g
        ids = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        return ShardGroup(ctx, n_global, world, bounds, rank, [(Lm, tile)], cfg, prc, ids[0])

    def cut_rank_shard(M):
        """bench's row cut of M for this rank: the weighted cut, then (with
        --recut) the measured re-cut -- every rank probes its first-cut shard
        on its own GPU (one plain SpMV + the loop's per-row work), the times
        are shared, and every rank re-cuts the same way."""
        b, L, t, w = prepare_rank_shard(M, world, rank, cfg)
        if not args.recut:
            return b, L, t, None
        probe = shard_cost_probe(L, t, cfg)
        times = [None] * world
        dist.all_gather_object(times, probe)
        del L, t
        b2, L, t = recut_rank_shard(M, b, times, rank, cfg, w)
        return b2, L, t, {"probe_ms": [round(v * 1e3, 4) for v in times],
                          "bounds_first": [int(v) for v in b], "bounds": [int(v) for v in b2]}

    def time_shard_runner(g, warmup, steps, iters):
        """iterations/s of a shard group: device time, max over ranks."""
        for _ in range(warmup):
            g.run()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            g.run()
        e1.record(stream)
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1))
        res, _ = g.result()
        assert res.iterations == iters, res.iterations
        return {"iters_per_s": iters * steps / (ms * 1e-3), "ms_per_step": ms / steps,
                "us_per_iteration": ms * 1e3 / (iters * steps), "steps": steps,
                "mass": res.mass}

    scale = args.scale if args.scale is not None else (24 if world == 1 else 27)
    t0 = time.perf_counter()
    P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
    gen_s = time.perf_counter() - t0
    n, m = P.n_rows, P.nnz
    cfg = mb.SimtConfig.make(32, 14, args.block_size)
    prc = mb.PageRankConfig(0.85, 1e-30, args.iters, 0)
    ro_host = None
    relabel_s = relabel_warm_s = 0.0
    P_natural = P
    if args.vertex_order == "degree":
        # locality preprocessing on the device: vertices ranked by descending
        # column count (P' = Q P Q^T); pi crosses the host boundary in the
        # original vertex order (the matrix keeps its vertex map)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        P, _ = P.relabel_by_degree(want_rank=False)
        torch.cuda.synchronize()
        relabel_s = time.perf_counter() - t1
        # the first call also grows the device memory pool (first touch:
        # page-mapping GBs on a fresh box costs 0.05-0.8 s, box to box); so
        # does a second call while the first's output is alive.  The third
        # call reuses the second's freed memory: the relabelling's own cost.
        for _ in range(2):
            t1 = time.perf_counter()
            del_me, _ = P_natural.relabel_by_degree(want_rank=False)
            torch.cuda.synchronize()
            relabel_warm_s = time.perf_counter() - t1
            del del_me
    if world == 1:
        tile = mb.generate_tile_for(P, cfg)
        xc_s = P.build_xcache()  # x hub cache: preprocessing, next to the TILE
        hub_cov = P.xcache_info()[1]
        runner = mb.PageRankPlan(P, tile, cfg, prc)  # builds the K2 slot copy once
        local_rows, local_nnz = n, m
        run = runner.run
        pre_ms = (relabel_s + tile.preprocess_seconds + xc_s + P.slot_info()[1]) * 1e3
        # the CSR values / columns are not read by the loop: keep only the
        # slot copy (rebuilt into CSR on demand)
        resident_full = P.resident_bytes()
        P.compact(tile)
        footprint = {"csr_bytes": m * 8 + 4 * (n + 1),
                     "resident_bytes_before_compact": resident_full,
                     "resident_bytes": P.resident_bytes(),
                     "tile_bytes": 4 * (2 * (tile.tile_num + 1) + tile.lane_num)}
        footprint["resident_over_csr"] = footprint["resident_bytes"] / footprint["csr_bytes"]
        footprint["resident_bytes_per_nnz"] = footprint["resident_bytes"] / m
    else:
        footprint = None
        hub_cov = None  # the shard group builds its own hub tables
        if rank == 0 and not args.no_extras:
            # the one-GPU anchor of THIS matrix, timed on rank 0 before the
            # cut (the other ranks wait): the strong-scaling reference
            extras["n1_anchor"] = single_gpu_rate(mb, stream, P, cfg, 3)
        barrier()
        t_cut = time.perf_counter()
        bounds, Lm, tile, recut = cut_rank_shard(P)
        if recut:
            extras["shard_recut"] = recut
        torch.cuda.synchronize()
        cut_s = time.perf_counter() - t_cut
        del P, P_natural
        P_natural = None
        if args.exchange == "fused" and not peer_ok():
            if rank == 0:
                print("bench: no P2P access between the ranks' GPUs; exchange = nccl",
                      file=sys.stderr)
            args.exchange = "nccl"
        runner = make_shard_runner(args.exchange, n, bounds, Lm, tile, prc)
        local_rows, local_nnz = int(bounds[rank + 1] - bounds[rank]), Lm.nnz
        run = runner.run
        pre_ms = (relabel_s + cut_s) * 1e3  # cut(s), slices, TILEs, probe
        barrier()  # every rank's preprocessing is done before the first run

    for _ in range(args.warmup):
        run()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    launches0 = ctx.launch_count
    # one event per step boundary (recording does not synchronise): the
    # total over the K steps is the value, the per-step median goes beside it
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    evs[0].record(stream)
    for k in range(args.steps):
        run()
        evs[k + 1].record(stream)
    barrier()
    clocks = sampler.stop()
    launches = ctx.launch_count - launches0
    ms_local = evs[0].elapsed_time(evs[-1])
    step_ms = sorted(evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps))
    step_ms_median = max_over_ranks(step_ms[len(step_ms) // 2])
    ms_total = max_over_ranks(ms_local)
    res, hist = runner.result(want_history=True)
    assert res.iterations == args.iters, res.iterations
    iters_per_s = args.iters * args.steps / (ms_total * 1e-3)
    t_iter_local = ms_local * 1e-3 / (args.iters * args.steps)
    b_iter = 8 * local_nnz + 16 * local_rows + 4
    achieved = b_iter / t_iter_local / 1e9
    ceil = gather_ceiling()
    gather_bound = None
    if hub_cov is not None and ceil:
        # every nonzero outside the shared-memory hub table is one scattered
        # x gather (one 32-B L1->L2 request); this, not DRAM, bounds K2 on R-MAT
        g_iter = local_nnz * (1.0 - hub_cov)
        gather_bound = {"gathers_per_iteration": g_iter, "hub_coverage": hub_cov,
                        "achieved_per_s": g_iter / t_iter_local, "ceiling_per_s": ceil,
                        "frac": g_iter / t_iter_local / ceil,
                        "ceiling_source": "profiles/r1s2_dsmem_gather.jsonl global_64MB "
                                          "(scattered 4-B gathers, L2-resident, 148 SMs)"}

    # e2e with pinned host buffers inside the timed region
    if world == 1:
        pi0 = torch.full((n,), 1.0 / n, dtype=torch.float32).pin_memory()
        pi_out = torch.empty(n, dtype=torch.float32).pin_memory()
        L = _lib.lib()
        cc, pc = cfg._c(), prc._c()
        rr = _lib.mbx_pagerank_result()

        def e2e_call():
            rc = L.mbx_pagerank(ctx.h, P.h, tile.h, C.byref(cc), C.byref(pc), pi0.data_ptr(),
                                pi_out.data_ptr(), None, None, C.byref(rr))
            if rc:
                raise RuntimeError(L.mbx_last_error().decode())
        h2d = d2h = 4 * n
    else:
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        pi0 = torch.full((r1 - r0,), 1.0 / n, dtype=torch.float32).pin_memory()
        pi_out = torch.empty(r1 - r0, dtype=torch.float32).pin_memory()
        pi0_dev = torch.empty(n, device="cuda", dtype=torch.float32)

        def e2e_call():
            pi0_dev[r0:r1].copy_(pi0, non_blocking=True)  # this rank's rows of pi0
            runner.run(pi0_dev.data_ptr())
            runner.download_local(pi_out.data_ptr())  # this rank's rows of pi
        h2d = d2h = 4 * (r1 - r0)
    e2e_call()
    barrier()
    e2e_steps = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        t1 = time.perf_counter()
        e2e_call()  # synchronous: ends with pi on the host
        e2e_steps.append(time.perf_counter() - t1)
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    e2e_val = args.iters / e2e_s
    e2e_steps.sort()
    e2e_median_s = max_over_ranks(e2e_steps[len(e2e_steps) // 2])
    mass = float(pi_out.double().sum()) if world == 1 else res.mass
    # the device-resident loop once more right after the e2e window: the two
    # windows see the same clocks / power state only if these agree
    recheck = {}
    if args.steps >= 2:
        barrier()
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(2):
            run()
        r1.record(stream)
        barrier()
        rms = max_over_ranks(r0.elapsed_time(r1)) / 2
        recheck = {"iters_per_s": args.iters / (rms * 1e-3), "ms_per_step": rms, "steps": 2}
    # the two paths interleaved step by step (a device-resident step, then an
    # end-to-end one), so both medians come from the same power / clock
    # window: their difference is what the host copies cost
    interleaved = {}
    if args.steps >= 2:
        dev_ms, e2e_ms = [], []
        for _ in range(args.steps):
            barrier()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            run()
            a1.record(stream)
            torch.cuda.synchronize()
            dev_ms.append(max_over_ranks(a0.elapsed_time(a1)))
            barrier()
            t1 = time.perf_counter()
            e2e_call()
            e2e_ms.append(max_over_ranks((time.perf_counter() - t1) * 1e3))
        dev_ms.sort()
        e2e_ms.sort()
        dm, em = dev_ms[len(dev_ms) // 2], e2e_ms[len(e2e_ms) // 2]
        interleaved = {"steps": args.steps, "device_median_ms": dm, "e2e_median_ms": em,
                       "device_iters_per_s": args.iters / (dm * 1e-3),
                       "e2e_iters_per_s": args.iters / (em * 1e-3),
                       "host_copies_ms": em - dm}

    if world > 1 and not args.no_extras:
        if args.exchange == "fused":
            # north_star's exchange, timed beside the fused one on the same
            # shards: one in-place ncclAllGather of the compacted pi per
            # iteration (NVLink / NVSwitch, NVLS when NCCL enables it)
            if os.environ.get("MBX_BENCH_ONE_DEVICE") == "1":
                extras["nccl_allgather_exchange"] = {
                    "unavailable": "the ranks share one device; NCCL needs one GPU per rank"}
            else:
                g2 = make_shard_runner("nccl", n, bounds, Lm, tile, prc)
                extras["nccl_allgather_exchange"] = time_shard_runner(g2, 2, args.steps,
                                                                      args.iters)
                g2.close()
        if scale != 24:
            # BASELINE C2's matrix (scale 24) sharded the same way: the
            # strong-scaling counterpart of the N = 1 line
            Q = mb.DeviceMatrix.rmat(ctx, 24, 16, seed=1, transition=True, dtype=np.float32)
            if args.vertex_order == "degree":
                Q, _ = Q.relabel_by_degree(want_rank=False)
            nq = Q.n_rows
            qb, QL, qt, qrecut = cut_rank_shard(Q)
            del Q
            gq = make_shard_runner(args.exchange, nq, qb, QL, qt, prc)
            d = time_shard_runner(gq, 2, args.steps, args.iters)
            d["exchange"] = args.exchange
            if qrecut:
                d["shard_recut"] = qrecut
            extras["c2_s24_sharded"] = d
            gq.close()
            del QL, qt

    cpu = None
    if rank == 0 and world == 1:
        if args.vertex_order == "degree" and P_natural is not None and not args.no_extras:
            # the same PageRank in R-MAT's natural vertex order, for comparison
            tn = mb.generate_tile_for(P_natural, cfg)
            P_natural.build_xcache()
            pn = mb.PageRankPlan(P_natural, tn, cfg, mb.PageRankConfig(0.85, 1e-30, 20, 0))
            pn.run()
            tnat = time_device(stream, pn.run, 3) / 20
            extras["pagerank_natural_order"] = {"iters_per_s": 1.0 / tnat,
                                                "us_per_iteration": tnat * 1e6}
            pn.close()
            del tn
        if not args.no_extras:
            extras["spmv_f32"] = spmv_numbers(mb, ctx, stream, scale, np.float32, args.spmv_reps,
                                              peak)
            extras["spmv_f64"] = spmv_numbers(mb, ctx, stream, scale, np.float64, args.spmv_reps,
                                              peak)
            # the same SpMVs after the device degree relabelling (preprocessing)
            for dt, key in ((np.float32, "spmv_f32_relabelled"),
                            (np.float64, "spmv_f64_relabelled")):
                extras[key] = spmv_numbers(
                    mb, ctx, stream, scale, dt, args.spmv_reps, peak,
                    make=lambda cx, d: mb.DeviceMatrix.rmat(
                        cx, scale, 16, seed=1, transition=True, dtype=d).relabel_by_degree(False)[0],
                    label=f"R-MAT scale {scale} transition, degree-relabelled")
            extras["c1_rmat_s20_f32"] = c1_numbers(mb, ctx, stream, peak,
                                                   not args.no_cpu_baseline)
            # BASELINE C3: fp64 power-law, long rows + exactly 10 % empty rows
            extras["c3_powerlaw_f64"] = spmv_numbers(
                mb, ctx, stream, 0, np.float64, args.spmv_reps, peak,
                make=lambda cx, dt: mb.DeviceMatrix.powerlaw(cx, 22, seed=3, dtype=dt),
                label="power-law 2^22 rows, 10% empty, rows up to 2^20 nnz",
                reference=None if args.no_cpu_baseline else "same")
            # BASELINE C5: 27-point stencil, 64M rows (uniform sparsity)
            for dt, key in ((np.float32, "c5_stencil_f32"), (np.float64, "c5_stencil_f64")):
                extras[key] = spmv_numbers(
                    mb, ctx, stream, 0, dt, max(5, args.spmv_reps // 3), peak,
                    make=lambda cx, d: mb.DeviceMatrix.stencil27(cx, 400, d),
                    label="27-point stencil 400^3 (64M rows)",
                    reference=None if args.no_cpu_baseline else (
                        lambda cx, d: mb.DeviceMatrix.stencil27(cx, 160, d),
                        "27-point stencil 160^3 (4.1M rows, 109M nonzeros): a bounded sample "
                        "of C5 (the full 1.7 G-nonzero matrix takes ~20 GB of host memory)"))
            # BASELINE C4's matrix (scale 27, 2.1 G nonzeros) on this one GPU:
            # the anchor of the 2/4/8-GPU runs (bench.py --gpus N defaults to it)
            Q = mb.DeviceMatrix.rmat(ctx, 27, 16, seed=1, transition=True, dtype=np.float32)
            if args.vertex_order == "degree":
                Q, _ = Q.relabel_by_degree(want_rank=False)
            d = single_gpu_rate(mb, stream, Q, cfg, 2, args.iters)
            d.update({"scale": 27, "n": Q.n_rows, "nnz": Q.nnz,
                      "frac": (8 * Q.nnz + 16 * Q.n_rows + 4) / (d["us_per_iteration"] * 1e-6)
                      / 1e9 / peak})
            extras["c4_s27_n1"] = d
            del Q
            torch.cuda.synchronize()
        if not args.no_cpu_baseline:
            import oracle as O
            if O.ref() is not None:
                ro, cols, _ = P_natural.download(want_values=False)  # R-MAT's own numbering
                nthreads = os.cpu_count() or 1
                r = cpu_reference_pagerank(ro, cols, n, 2, 5, 1, nthreads)
                cpu = {"value": r["value"], "unit": "iters/s", "cores": nthreads,
                       "kind": "reference", "cpu_model": cpu_model(),
                       "sample": f"5 x 2 = {r['iterations']} PageRank iterations (after one "
                                 f"2-iteration warm-up) of the reference MerbitBackend<float> on "
                                 f"ThreadPool({nthreads}), same scale-{scale} transition matrix "
                                 f"(natural order); its generate_tile took "
                                 f"{r['preprocess_seconds']:.2f} s"}
    line = {
        "metric": METRIC, "value": iters_per_s, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"pagerank {args.iters} iterations fp32, R-MAT scale {scale} "
                               f"transition (edge factor 16; vertex order: "
                               + ("degree-relabelled on the device as preprocessing, pi "
                                  "returned in the original order" if args.vertex_order ==
                                  "degree" else "natural") + "), preprocessing amortised"
                               + (f", {world} row shards (weighted cut, row weight "
                                  f"{mb.merbit.pagerank_row_weight(n)}"
                                  + (", re-cut from measured shard cost" if args.recut else "")
                                  + "), exchange: "
                                  + ("fused P2P stores in the commit" if args.exchange == "fused"
                                     else "ncclAllGather") if world > 1 else ""),
                   "scale": scale, "n": n, "nnz": m, "omega": 32, "sigma": 14,
                   "block_size": args.block_size,
                   "l2": "inputs (values+cols %.1f GB per GPU) larger than L2; no flush"
                         % (8 * local_nnz / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_per_launch() if scale == 24 and world == 1 else None,
                     "peak_kind": peak_kind, "frac_of_nominal_8tbs": achieved / 8000.0,
                     "kernel": "fused PageRank iteration (spmv_slot_kernel<float,14,PR,HUB> + "
                               "fixup_kernel) on rank 0",
                     "bytes_per_launch": b_iter, "us_per_iteration": t_iter_local * 1e6,
                     "gather_bound": gather_bound},
        "e2e": {"value": e2e_val, "unit": "iters/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "mass": mass,
                "median_step_ms": e2e_median_s * 1e3,
                "median_iters_per_s": args.iters / e2e_median_s,
                "interleaved_with_device_steps": interleaved},
        "median_step_ms": step_ms_median,
        "median_iters_per_s": args.iters / (step_ms_median * 1e-3),
        "recheck_after_e2e": recheck,
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "preprocess_ms": pre_ms,
        "hbm_footprint": footprint,
        "relabel_ms": relabel_s * 1e3,
        "relabel_ms_repeat": relabel_warm_s * 1e3,
        "l1_residual_last": res.l1_residual,
        "input_generation_seconds": gen_s,
    }
    line.update(extras)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        runner.close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
