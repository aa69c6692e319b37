"""CPU, world_size 2 over gloo: the multi-GPU exchange protocol of shard.cu
(merge-path row bounds from the product's mbx_plan_row_shards, compacted
chunks holding only the NON-DANGLING entries of each rank's rows plus an fp64
scalar tail, columns remapped to pos(v) = owner * chunk + #non-dangling before
v in the owner's rows, one all-gather per iteration, rank-order combine, full
rows kept locally) reproduces the single-process PageRank.  The per-shard multiply here is the
CPU oracle (the checker) -- this test covers the host logic and layout; the
device kernels of the same protocol are covered by tests/test_gpu_shards.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle as O
import paper_2605_07391_b200 as mb

SCALE, ITERS, C_ = 10, 30, 0.85


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = O.rmat(SCALE, 16, 11, transposed=True)
    n = p.n_rows
    vals = O.transition_values(n, p.col_indices, np.float64)
    b = mb.plan_row_shards(p.row_offsets, n, p.nnz, world)  # product host logic
    r0, r1 = int(b[rank]), int(b[rank + 1])
    ro = p.row_offsets[r0:r1 + 1] - p.row_offsets[r0]
    cols = p.col_indices[p.row_offsets[r0]:p.row_offsets[r1]]
    v = vals[p.row_offsets[r0]:p.row_offsets[r1]]
    seen = torch.zeros(n, dtype=torch.uint8)
    seen[torch.from_numpy(cols.astype(np.int64))] = 1
    dist.all_reduce(seen, op=dist.ReduceOp.MAX)  # global empty columns = dangling
    nd = seen.numpy().astype(bool)
    gpre = np.concatenate([[0], np.cumsum(nd)])  # non-dangling before v
    nd_max = max(int(gpre[b[g + 1]] - gpre[b[g]]) for g in range(world))
    chunk = nd_max + 4  # non-dangling pi entries, then 4 fp64 scalars
    owner = np.searchsorted(np.asarray(b), np.arange(n), side="right") - 1
    pos = owner * chunk + (gpre[:n] - gpre[np.asarray(b)[owner]])
    assert nd[cols].all()  # only non-dangling columns are ever gathered
    local = O.Csr(r1 - r0, world * chunk, ro, pos[cols].astype(np.int32), v)
    dang = ~nd[r0:r1]
    xmap = np.where(nd[r0:r1], pos[r0:r1] - rank * chunk, -1)

    def pack(pi):
        mine = torch.zeros(chunk, dtype=torch.float64)
        mine[torch.from_numpy(xmap[xmap >= 0])] = torch.from_numpy(pi[xmap >= 0])
        return mine
    buf = torch.zeros(world * chunk, dtype=torch.float64)
    pi_local = np.full(r1 - r0, 1.0 / n)
    mine = pack(pi_local)
    mine[nd_max] = pi_local[dang].sum()
    dist.all_gather_into_tensor(buf, mine)
    for _ in range(ITERS):
        dm = sum(float(buf[g * chunk + nd_max]) for g in range(world))  # rank order
        w = O.spmv_csr_f64(local, buf.numpy())
        new = C_ * w + (C_ * dm + 1 - C_) / n
        mine = pack(new)
        mine[nd_max] = new[dang].sum()
        mine[nd_max + 1] = np.abs(new - pi_local).sum()
        pi_local = new
        dist.all_gather_into_tensor(buf, mine)
    # the full answer: one gather of the local rows (mbx_shard_group_gather_pi)
    rows_max = int(np.diff(np.asarray(b)).max())
    lbuf = torch.zeros(world * rows_max, dtype=torch.float64)
    lmine = torch.zeros(rows_max, dtype=torch.float64)
    lmine[:r1 - r0] = torch.from_numpy(pi_local)
    dist.all_gather_into_tensor(lbuf, lmine)
    full = np.concatenate([lbuf[g * rows_max:g * rows_max + (b[g + 1] - b[g])].numpy()
                           for g in range(world)])
    q.put((rank, full, [int(x) for x in b]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_exchange_protocol(world):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    out.sort(key=lambda t: t[0])
    assert out[0][2] == out[1][2]  # both ranks derived identical bounds
    assert np.array_equal(out[0][1], out[1][1])  # every rank holds the same pi
    p = O.rmat(SCALE, 16, 11, transposed=True)
    p64 = O.Csr(p.n_rows, p.n_cols, p.row_offsets, p.col_indices,
                O.transition_values(p.n_rows, p.col_indices, np.float64))
    want = O.pagerank(p64, C_, 1e-300, ITERS, 0)["pi"]
    assert np.abs(out[0][1] - want).sum() <= 1e-13


def test_recut_row_shards_properties():
    """recut_row_shards (bench.py's measured re-cut): equal times keep the
    cut, a slow shard gives rows away, bounds stay monotone and span all
    rows, and the cut is exactly the even split of the measured-time curve
    when time is proportional to nnz + w*rows."""
    rng = np.random.default_rng(3)
    deg = rng.integers(0, 40, size=5000)
    ro = np.concatenate([[0], np.cumsum(deg)])
    n, m = 5000, int(ro[-1])
    for w in (1.0, 1.5, 3.4):
        b = mb.plan_row_shards(ro, n, m, 4, w)
        assert np.array_equal(mb.recut_row_shards(ro, b, [1.0] * 4, w), b)
        slow = mb.recut_row_shards(ro, b, [2.0, 1.0, 1.0, 1.0], w)
        assert slow[0] == 0 and slow[-1] == n and np.all(np.diff(slow) >= 0)
        assert slow[1] < b[1]  # the slow shard shrinks
        # time = k_i * cost within shard i: the re-cut evens the time curve
        cost = ro + w * np.arange(n + 1)
        k = np.array([1.0, 2.0, 0.5, 1.5])
        t = [k[i] * (cost[b[i + 1]] - cost[b[i]]) for i in range(4)]
        nb = mb.recut_row_shards(ro, b, t, w)
        curve = np.zeros(n + 1)
        for i in range(4):
            seg = slice(b[i], b[i + 1] + 1)
            curve[seg] = sum(t[:i]) + k[i] * (cost[seg] - cost[b[i]])
        parts = [curve[nb[i + 1]] - curve[nb[i]] for i in range(4)]
        step = k.max() * (w + 40)  # one row's cost at most
        assert max(parts) - min(parts) <= 2 * step
    # malformed input leaves the cut alone
    b = mb.plan_row_shards(ro, n, m, 4, 1.0)
    assert np.array_equal(mb.recut_row_shards(ro, b, [1.0, 0.0, 1.0, 1.0], 1.0), b)
    assert np.array_equal(mb.recut_row_shards(ro, b, [1.0] * 3, 1.0), b)
