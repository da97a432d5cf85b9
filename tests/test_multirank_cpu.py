"""CPU, world_size 2 over gloo: the batched-pairs sharding (configs 3/5b) and the
max-over-ranks timing reduction bench.py uses.  No GPU: the per-pair runner is a stub."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_02153_b200.batch import run_sharded, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_items, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_sharded(n_items, lambda i: {"owner": rank, "value": i * i}, rank, world)
        # bench.py: device-timed region, max over ranks
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            out.put((res, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for world in (1, 2, 4, 8):
        items = sorted(i for r in range(world) for i in shard(64, r, world))
        assert items == list(range(64))
    with pytest.raises(ValueError):
        shard(8, 2, 2)


@pytest.mark.parametrize("n_items", [8, 7])
def test_two_rank_gloo(n_items):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_items, q)) for r in range(2)]
    for p in procs:
        p.start()
    res, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r["item"] for r in res] == list(range(n_items))
    assert all(r["value"] == r["item"] ** 2 and r["owner"] == r["item"] % 2 for r in res)
    assert tmax == 2.0


def test_lanes_order_runner_reuse_and_errors():
    import threading
    import time

    from paper_1604_02153_b200.batch import run_lanes

    built, active, peak = [], [0], [0]
    lock = threading.Lock()

    def make_runner(k):
        built.append(k)

        def run(i):
            with lock:
                active[0] += 1
                peak[0] = max(peak[0], active[0])
            time.sleep(0.01)
            with lock:
                active[0] -= 1
            return {"sq": i * i}
        return run

    items = [3, 1, 4, 15, 9, 2, 6]
    res = run_lanes(items, make_runner, 3)
    assert [r["item"] for r in res] == items and all(r["sq"] == r["item"] ** 2 for r in res)
    assert sorted(built) == [0, 1, 2] and peak[0] > 1  # one runner per lane, lanes overlap
    assert run_lanes([], make_runner, 4) == []

    def failing(k):
        def run(i):
            if i == 5:
                raise RuntimeError("pair 5 failed")
            return {}
        return run
    with pytest.raises(RuntimeError, match="pair 5"):
        run_lanes(list(range(10)), failing, 2)
    with pytest.raises(ValueError):
        run_lanes([1], failing, 0)


def _lanes_worker(rank, world, port, n_items, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_sharded(n_items, None, rank, world, make_runner=lambda k: (lambda i: {"owner": rank}), lanes=3)
        if rank == 0:
            out.put(res)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_with_lanes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lanes_worker, args=(r, 2, port, 11, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r["item"] for r in res] == list(range(11))
    assert all(r["owner"] == r["item"] % 2 and 0 <= r["lane"] < 3 for r in res)
