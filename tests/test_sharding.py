"""Multi-rank host logic on CPU (gloo, world_size 2): row sharding covers the
batch exactly once and the timing reduction is a max over ranks."""
import os

import pytest
import torch.multiprocessing as mp

from paper_2409_08970_b200.sharding import max_over_ranks, shard_rows


@pytest.mark.parametrize("batch,world", [(65536, 8), (2048, 3), (5, 4), (0, 2), (4096, 1)])
def test_shard_rows_partition(batch, world):
    seen = []
    for r in range(world):
        s, c = shard_rows(batch, r, world)
        seen.extend(range(s, s + c))
    assert seen == list(range(batch))
    counts = [shard_rows(batch, r, world)[1] for r in range(world)]
    assert max(counts) - min(counts) <= 1


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = max_over_ranks(1.5 + rank)
        s, c = shard_rows(1001, rank, world)
        q.put((rank, m, s, c))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert [o[1] for o in out] == [2.5, 2.5]
    assert out[0][2:] == (0, 501) and out[1][2:] == (501, 500)


def _shard_apply_worker(rank, world, port, q):
    """bench.py's multi-GPU data path with the GPU apply mocked by the C
    restatement (a per-row CPU transform): shard -> apply -> gather."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import bench
    from oracle import checkers as O
    from tests.golden_io import load_golden, setup_of

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R = O.Restatement()
        st = setup_of(load_golden("c1"))
        cfg = bench.CONFIGS["C1"]
        batch = 1001
        x = R.fill_signals(bench.mix_seed(bench.SEED, cfg["n"], cfg["cid"]), cfg["dist"], cfg["n"], batch, cfg["r"])
        start, rows = bench.shard_rows(batch, rank, world)
        assert (start, rows) == shard_rows(batch, rank, world)  # bench's copy agrees with the package's
        y = R.forward(st, x[start:start + rows])
        parts = [None] * world
        dist.all_gather_object(parts, (start, y))
        if rank == 0:
            full = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
            q.put(("ok", bool(np.array_equal(full, R.forward(st, x)))))
        dist.barrier()
    except Exception as e:  # pragma: no cover
        q.put(("error", repr(e)))
    finally:
        dist.destroy_process_group()


def test_bench_shard_apply_gather_gloo_world2():
    """Strong scaling as bench.py runs it (contiguous row shards, no data-path
    collective): the gathered shards are bitwise the single-rank result."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_shard_apply_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
    assert res == ("ok", True), res
