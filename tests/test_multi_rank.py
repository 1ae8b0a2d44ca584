"""Multi-rank host logic on CPU (gloo, world_size 2): the shard split, the
max-over-ranks timing reduction and the gather of per-instance scalars that
bench.py / multi-GPU runs use (no GPU needed; the solve itself is per rank)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_07772_b200.shard import gather_scalars, max_over_ranks, shard_range, weak_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 1024, 131072):
        for world in (1, 2, 3, 8):
            rs = [shard_range(r, world, total) for r in range(world)]
            flat = [d for r in rs for d in r]
            assert flat == list(range(total))
            assert max(len(r) for r in rs) - min(len(r) for r in rs) <= 1


def test_weak_range_disjoint():
    rs = [set(weak_range(r, 1024)) for r in range(8)]
    assert sum(len(r) for r in rs) == len(set().union(*rs)) == 8 * 1024


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = max_over_ranks(1.0 + rank)
        draws = shard_range(rank, world, 5)
        outs = {"ee": torch.tensor([10.0 * d for d in draws]),
                "status": torch.tensor([d % 3 for d in draws], dtype=torch.int8),
                "p": torch.zeros(len(draws), 2)}  # dense outputs stay on their rank
        g = gather_scalars(outs)
        q.put((rank, t, None if g is None else {k: v.tolist() for k, v in g.items()}))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, t0, g0), (r1, t1, g1) = res
    assert t0 == t1 == 2.0
    assert g1 is None
    assert g0["ee"] == [0.0, 10.0, 20.0, 30.0, 40.0]
    assert g0["status"] == [0.0, 1.0, 2.0, 0.0, 1.0]
    assert "p" not in g0
