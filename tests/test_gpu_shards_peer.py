"""GPU: the FUSED exchange of the row-sharded PageRank (peer shard groups,
shard.cu): the K2/K3 commit stores pi_new straight into every peer's
exchange buffer and a device barrier (system-scope release/acquire epochs)
ends each iteration -- no collective library on the iteration path.

Only one GPU is available, so the ranks share it:
* in one process, each rank on its own context and stream (peers of the same
  pid use raw device pointers; the ranks' graphs run concurrently);
* in two processes (CUDA IPC handles exchanged over a gloo bootstrap at
  127.0.0.1; the GPU time-slices the two contexts, so every barrier is a
  real cross-process handoff).
Gate: pi bitwise equal to the virtual shard group on the same bounds (same
shards, TILEs and summation order), which is itself gated against the fp64
oracle in test_gpu_shards.py; run to run bitwise; a second run on the same
group (the epoch ranges of consecutive runs) bitwise equal."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
from conftest import gpu_shared_between_processes

import oracle as O
import paper_2605_07391_b200 as mb
from paper_2605_07391_b200.merbit import PeerShardGroup, ShardGroup, row_slice

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def virtual_pi(ctx, scale, parts, iters, weight=1.0):
    P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=5, transition=True, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    ro, _, _ = P.download(want_values=False)
    b = mb.plan_row_shards(ro, P.n_rows, P.nnz, parts, weight)
    shards = [(m, mb.generate_tile_for(m, c)) for m in
              (row_slice(P, int(b[g]), int(b[g + 1])) for g in range(parts))]
    grp = ShardGroup(ctx, P.n_rows, parts, b, 0, shards, c,
                     mb.PageRankConfig(0.85, 1e-30, iters, 0))
    grp.run()
    res, hist = grp.result(want_history=True)
    pi = grp.gather_pi()
    grp.close()
    return pi, res, hist, b


@pytest.mark.parametrize("parts", [2, 3])
def test_peer_groups_in_one_process(parts):
    iters = 12
    base = mb.Context(0)
    want, wres, whist, b = virtual_pi(base, 12, parts, iters)
    c = mb.SimtConfig.make(32, 14, 128)
    cfg = mb.PageRankConfig(0.85, 1e-30, iters, 0)
    ctxs, groups = [], []
    for r in range(parts):
        cx = mb.Context(0)  # own stream per rank: the ranks' graphs overlap
        P = mb.DeviceMatrix.rmat(cx, 12, 16, seed=5, transition=True, dtype=np.float32)
        L = row_slice(P, int(b[r]), int(b[r + 1]))
        t = mb.generate_tile_for(L, c)
        groups.append(PeerShardGroup(cx, P.n_rows, parts, b, r, L, t, c, cfg))
        ctxs.append(cx)
    blobs = [g.export() for g in groups]
    for g in groups:
        g.connect(blobs)
    for rep in range(2):  # two runs: consecutive epoch ranges
        for g in groups:
            g.run()  # asynchronous: every rank's barrier waits for the others
        for g in groups:
            res, hist = g.result(want_history=True)
            assert res.iterations == iters
            assert res.l1_residual == wres.l1_residual and np.array_equal(hist, whist)
            assert abs(res.mass - 1.0) <= 1e-5
        for g in groups:
            pi = g.gather_pi()
            assert np.array_equal(pi.view(np.uint32), want.view(np.uint32)), rep
    for g in groups:
        g.run()
    for g in groups:
        g.quiesce()  # the final barrier, enqueued on every rank first
    for g in groups:
        g.close()


def test_peer_group_rejects_bad_blobs():
    cx = mb.Context(0)
    P = mb.DeviceMatrix.rmat(cx, 10, 16, seed=5, transition=True, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    b = np.array([0, P.n_rows // 2, P.n_rows], np.int64)
    L = row_slice(P, 0, int(b[1]))
    g = PeerShardGroup(cx, P.n_rows, 2, b, 0, L, mb.generate_tile_for(L, c), c,
                       mb.PageRankConfig(0.85, 1e-30, 4, 0))
    with pytest.raises(mb.ConfigError):
        g.run()  # not connected
    blob = g.export()
    with pytest.raises(mb.ConfigError):
        g.connect([blob, blob])  # rank 1's slot holds rank 0's blob
    with pytest.raises(mb.ConfigError):
        g.connect([blob])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.skipif(not gpu_shared_between_processes(),
                    reason="device 0 is in an exclusive compute mode")
def test_peer_groups_across_processes(tmp_path, world):
    """Two / three processes, CUDA IPC mappings, gloo only for the bootstrap."""
    iters = 8
    base = mb.Context(0)
    want, wres, _, b = virtual_pi(base, 11, world, iters)
    np.save(tmp_path / "bounds.npy", b)
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PYTHONPATH=ROOT)
        procs.append(subprocess.Popen(
            [sys.executable, os.path.join(ROOT, "tests", "peer_rank.py"), str(tmp_path),
             str(iters)], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out.decode())
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
    for r in range(world):
        pi = np.load(tmp_path / f"pi{r}.npy")
        assert np.array_equal(pi.view(np.uint32), want.view(np.uint32)), r
        resid = float(np.load(tmp_path / f"resid{r}.npy"))
        assert resid == wres.l1_residual


def test_peer_groups_early_stop_and_start_vector():
    """Convergence decided after the barrier: on a directed ring pi stays
    uniform, so ERR against the uniform yardstick (reference_iters = 0) drops
    below err_tol at iteration 1 and every rank must stop there and skip the
    remaining barriers consistently (the final barrier still meets).  The
    start vector comes from the caller (its chunk pushed to the peers before
    the first barrier)."""
    import torch
    parts, iters, n = 3, 50, 3000
    ring = O.Csr(n, n, np.arange(n + 1, dtype=np.int64),
                 np.array([(i - 1) % n for i in range(n)], np.int32), np.ones(n))
    base = mb.Context(0)
    c = mb.SimtConfig.make(32, 7, 128)
    cfg = mb.PageRankConfig(0.85, 1e-9, iters, 0)
    b = np.array([0, 700, 2100, n], np.int64)
    P = mb.DeviceMatrix.from_csr(base, ring)
    vs = [(m, mb.generate_tile_for(m, c)) for m in
          (row_slice(P, int(b[g]), int(b[g + 1])) for g in range(parts))]
    virt = ShardGroup(base, n, parts, b, 0, vs, c, cfg)
    pi0_dev = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    virt.run(pi0_dev.data_ptr())
    wres, whist = virt.result(want_history=True)
    want = virt.gather_pi()
    assert wres.status == 0 and wres.iterations == 1  # converged at once
    groups = []
    for r in range(parts):
        cx = mb.Context(0)
        Q = mb.DeviceMatrix.from_csr(cx, ring)
        L = row_slice(Q, int(b[r]), int(b[r + 1]))
        groups.append(PeerShardGroup(cx, n, parts, b, r, L, mb.generate_tile_for(L, c), c, cfg))
    blobs = [g.export() for g in groups]
    for g in groups:
        g.connect(blobs)
    for rep in range(2):
        for g in groups:
            g.run(pi0_dev.data_ptr())
        for g in groups:
            res, hist = g.result(want_history=True)
            assert res.status == 0 and res.iterations == 1
            assert res.final_err == wres.final_err and np.array_equal(hist, whist)
            assert np.array_equal(g.gather_pi(), want)
    for g in groups:
        g.quiesce()
    for g in groups:
        g.close()


def test_peer_group_world_one_and_limits():
    """A one-rank peer group (no peers: the barrier meets itself) equals the
    single-GPU loop bitwise; world > 8 is rejected."""
    cx = mb.Context(0)
    P = mb.DeviceMatrix.rmat(cx, 11, 16, seed=8, transition=True, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(P, c)
    cfg = mb.PageRankConfig(0.85, 1e-30, 9, 0)
    b = np.array([0, P.n_rows], np.int64)
    g = PeerShardGroup(cx, P.n_rows, 1, b, 0, P, t, c, cfg)
    g.connect([g.export()])
    g.run()
    res, _ = g.result()
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, t, c
    single = mb.pagerank(None, cfg, backend=be)
    assert res.iterations == 9
    assert np.array_equal(g.gather_pi().view(np.uint32), single.pi.view(np.uint32))
    g.close()
    with pytest.raises(mb.ConfigError):
        PeerShardGroup(cx, P.n_rows, 9, np.linspace(0, P.n_rows, 10).astype(np.int64), 0, P, t,
                       c, cfg)


def test_peer_groups_with_yardstick():
    """The yardstick phase over the fused exchange (its own barrier slots,
    then a transition barrier before the power loop reuses buffer 0): stop
    iteration and pi equal the virtual group's."""
    parts, n_it = 2, 210
    base = mb.Context(0)
    c = mb.SimtConfig.make(32, 7, 128)
    cfg = mb.PageRankConfig(0.85, 1e-6, n_it, 24)
    P = mb.DeviceMatrix.rmat(base, 11, 16, seed=5, transition=True, dtype=np.float64)
    ro, _, _ = P.download(want_values=False)
    b = mb.plan_row_shards(ro, P.n_rows, P.nnz, parts)
    vs = [(m, mb.generate_tile_for(m, c)) for m in
          (row_slice(P, int(b[g]), int(b[g + 1])) for g in range(parts))]
    virt = ShardGroup(base, P.n_rows, parts, b, 0, vs, c, cfg)
    virt.run()
    wres, _ = virt.result()
    want = virt.gather_pi()
    assert wres.status == 0 and wres.iterations < n_it
    groups = []
    for r in range(parts):
        cx = mb.Context(0)
        Q = mb.DeviceMatrix.rmat(cx, 11, 16, seed=5, transition=True, dtype=np.float64)
        L = row_slice(Q, int(b[r]), int(b[r + 1]))
        groups.append(PeerShardGroup(cx, Q.n_rows, parts, b, r, L, mb.generate_tile_for(L, c),
                                     c, cfg))
    blobs = [g.export() for g in groups]
    for g in groups:
        g.connect(blobs)
    for rep in range(2):
        for g in groups:
            g.run()
        for g in groups:
            res, _ = g.result()
            assert res.iterations == wres.iterations and res.final_err == wres.final_err
            assert np.array_equal(g.gather_pi(), want)
    for g in groups:
        g.quiesce()
    for g in groups:
        g.close()
