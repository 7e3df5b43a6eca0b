"""Host logic of the frame-sharded multi-GPU path (paper_2503_11731_b200/dist.py)
on CPU: shard plans, and the gather of per-rank frame blocks to rank 0 over a
world_size-2 (and 3) gloo process group."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2503_11731_b200 import dist as gd  # noqa: E402


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 3), (3, 4), (0, 2)])
def test_shard_range_partitions(n, world):
    seen = []
    for r in range(world):
        lo, hi = gd.shard_range(n, world, r)
        assert 0 <= lo <= hi <= n
        seen += list(range(lo, hi))
    assert seen == list(range(n))            # contiguous, ordered, disjoint, complete
    c = gd.shard_counts(n, world)
    assert max(c) - min(c) <= 1 and sum(c) == n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame(t, shape):
    """Deterministic stand-in for the rendered frames of timestep t."""
    g = torch.Generator().manual_seed(1000 + t)
    return torch.rand(shape, generator=g)


def _worker(rank, world, port, n_t, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        per_t, shape = 3, (2, 5, 4)
        lo, hi = gd.shard_range(n_t, world, rank)
        full = torch.full((n_t, per_t) + shape, -1.0) if rank == 0 else None
        if rank == 0:   # the root renders straight into its slice of the batch
            local = full[lo:hi]
        else:
            local = torch.empty((hi - lo, per_t) + shape)
        for j, t in enumerate(range(lo, hi)):
            local[j] = _frame(t, (per_t,) + shape)
        for r in gd.gather_blocks(local, full, n_t, world, rank):
            r.wait()
        m = gd.max_over_ranks(float(rank) + 0.5, torch.device("cpu"), world)
        if rank == 0:
            want = torch.stack([_frame(t, (per_t,) + shape) for t in range(n_t)])
            q.put(("ok", bool(torch.equal(full, want)), m))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put(("err", repr(e), None))


@pytest.mark.parametrize("world,n_t", [(2, 8), (2, 5), (3, 7)])
def test_gather_blocks_gloo(world, n_t):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n_t, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == "ok", res
    assert res[1], "gathered batch differs from the frames the ranks rendered"
    assert res[2] == world - 0.5                 # max over ranks
    assert all(p.exitcode == 0 for p in ps)


def test_gather_world1_copies():
    local = torch.arange(12.0).view(3, 4)
    full = torch.zeros(3, 4)
    assert gd.gather_blocks(local, full, 3, 1, 0) == []
    assert torch.equal(full, local)


def _round_worker(rank, world, port, n_t, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        shapes = {"cam": (6, 2, 3, 4), "lidar": (1, 4, 2, 5)}
        lo, hi = gd.shard_range(n_t, world, rank)
        full = {k: torch.full((n_t,) + sh, -1.0) for k, sh in shapes.items()} if rank == 0 else None
        local = {k: (full[k][lo:hi] if rank == 0 else torch.empty((hi - lo,) + sh)) for k, sh in shapes.items()}
        reqs = []
        for j in range(gd.n_rounds(n_t, world)):
            if j < hi - lo:   # "render" item j of this rank's block, then post its round
                for k, sh in shapes.items():
                    local[k][j] = _frame(lo + j, sh) + (0.5 if k == "lidar" else 0.0)
            ops = gd.round_ops(local, full, j, n_t, world, rank)
            if ops:
                reqs += dist.batch_isend_irecv(ops)
        for r in reqs:
            r.wait()
        if rank == 0:
            ok = all(torch.equal(full[k][t], _frame(t, sh) + (0.5 if k == "lidar" else 0.0))
                     for k, sh in shapes.items() for t in range(n_t))
            q.put(("ok", ok, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), None))


@pytest.mark.parametrize("world,n_t", [(2, 8), (3, 7), (4, 6)])
def test_overlapped_gather_rounds_gloo(world, n_t):
    """Round-wise gather (post item j as soon as it is rendered) assembles the
    same batch on rank 0, uneven blocks included."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_round_worker, args=(r, world, port, n_t, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == "ok" and res[1], res
    assert all(p.exitcode == 0 for p in ps)


def _bench_worker(rank, world, port, n_t, schedule, q):
    """bench.py's multi-GPU step bookkeeping (dist.ShardedBatch: slabs, the
    per-frame output views, the timestep shard, both gather schedules) with a
    stub renderer in place of the CUDA path: frame f of timestep t is filled
    with a deterministic function of (t, f)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        # a timestep as in the Chunked batch: 6 cameras (8 channels) then 1 LiDAR (4)
        specs = [(0, 8, 3, 5)] * 6 + [(2, 4, 2, 6)]
        sb = gd.ShardedBatch(specs, n_t, world, rank, torch.device("cpu"))
        lo, hi = gd.shard_range(n_t, world, rank)
        assert (sb.lo, sb.hi) == (lo, hi) and len(sb.outs) == 7 * (hi - lo)
        fpt = sb.frames_per_timestep

        def stub(t, f):
            return _frame(1000 * t + f, tuple(specs[f][1:]))
        reqs = []
        for i, out in enumerate(sb.outs):
            t, f = lo + i // fpt, i % fpt
            out.copy_(stub(t, f))                      # "render" local frame i
            if schedule == "rounds" and f == fpt - 1:
                reqs += sb.round(i // fpt)             # post this timestep's round
        if schedule == "rounds":
            for j in sb.rounds_left():
                reqs += sb.round(j)
            for r in reqs:
                r.wait()
        else:
            sb.gather()
        if rank == 0:
            ok = True
            for t in range(n_t):
                cams = [f for f in range(7) if specs[f][0] == 0]
                for c, f in enumerate(cams):
                    ok &= torch.equal(sb.full[0][6 * t + c], stub(t, f))
                ok &= torch.equal(sb.full[2][t], stub(t, 6))
            q.put(("ok", bool(ok), None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), None))


@pytest.mark.parametrize("schedule", ["end", "rounds"])
@pytest.mark.parametrize("world,n_t", [(4, 10), (4, 3)])
def test_bench_step_bookkeeping_world4_gloo(world, n_t, schedule):
    """World size 4: the sharding, slab and gather bookkeeping bench.py's step
    runs (both gather schedules, uneven and short blocks) assembles the whole
    batch on rank 0 in batch order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_bench_worker, args=(r, world, port, n_t, schedule, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = q.get(timeout=180)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == "ok" and res[1], res
    assert all(p.exitcode == 0 for p in ps)


# ---------------------------------------------------------------- pixel-partitioned frame (NEXT-4)
def test_balanced_and_adaptive_bands():
    from paper_2503_11731_b200 import pixdist as pd
    assert pd.balanced_bands(np.ones(16), 4) == [0, 4, 8, 12, 16]
    b = pd.balanced_bands([0, 0, 10, 0, 0, 0, 0, 10], 2)
    assert b[0] == 0 and b[-1] == 8 and 2 < b[1] <= 7
    for nb in (1, 3, 8):   # every band keeps >= 1 row even with all cost in one row
        b = pd.balanced_bands([0] * 10 + [5] + [0] * 5, nb)
        assert len(b) == nb + 1 and all(b[i + 1] > b[i] for i in range(nb)) and b[-1] == 16
    # time-adaptive: band 0 took 3x longer per pair -> its boundary moves up
    pairs = np.ones(20)
    nb = pd.adapt_bands([0, 10, 20], [30.0, 10.0], pairs)
    assert nb[1] < 10
    # equal measured cost -> unchanged
    assert pd.adapt_bands([0, 10, 20], [10.0, 10.0], pairs) == [0, 10, 20]


def _pix_worker(rank, world, port, q):
    """The sparse all-to-all of pixdist.exchange on gloo: each rank routes its
    shard of synthetic tile rects to bands brute force, sends the routed rows
    (global index, a payload value), and must receive exactly the overlap set
    of its band in ascending global order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        from paper_2503_11731_b200 import pixdist as pd
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n, rows = 997, 23
        g = torch.Generator().manual_seed(7)
        y0 = torch.randint(0, rows, (n,), generator=g)
        y1 = torch.clamp(y0 + torch.randint(0, 6, (n,), generator=g), max=rows - 1)
        vis = torch.rand(n, generator=g) < 0.8
        bounds = pd.balanced_bands(np.ones(rows), world)
        lo, hi = gd.shard_range(n, world, rank)
        rows_out, counts = [], []
        for b in range(world):
            sel = [i for i in range(lo, hi) if vis[i] and y1[i] >= bounds[b] and y0[i] < bounds[b + 1]]
            rows_out += [[float(i), float(i) * 0.5] for i in sel]
            counts.append(len(sel))
        payload = torch.tensor(rows_out, dtype=torch.float32).reshape(-1, 2)
        recv, rc = pd.exchange(payload, counts)
        want = [i for i in range(n) if vis[i] and y1[i] >= bounds[rank] and y0[i] < bounds[rank + 1]]
        ok = recv[:, 0].to(torch.int64).tolist() == want and torch.equal(recv[:, 1], recv[:, 0] * 0.5)
        ok = ok and sum(rc) == len(want)
        q.put(("ok", bool(ok), rank))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), rank))


@pytest.mark.parametrize("world", [2, 3])
def test_pixel_partition_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_pix_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    assert all(r[0] == "ok" and r[1] for r in res), res
