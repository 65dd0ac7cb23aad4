"""Multi-rank plumbing on CPU (gloo, world_size 2): contiguous position
sharding and the gather-to-root of per-rank outputs used by the multi-GPU
bench path (the GPU path runs the same code on NCCL)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_12787_b200.shard import ChunkedGather, chunk_spans, gather_to_root, max_over_ranks, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 1024, 1025, 65536):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert sum(c for _, c in spans) == total
            at = 0
            for s, c in spans:
                assert s == at
                at += c
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = shard_range(total, world, rank)
    # stand-in for this rank's rendered outputs: rows tagged with their global index
    local = torch.arange(start, start + count, dtype=torch.float32)[:, None].repeat(1, 6)
    full = gather_to_root(local, total, world, rank)
    slowest = max_over_ranks(10.0 + rank)
    if rank == 0:
        q.put((full.numpy().tolist(), slowest))
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [10, 11])
def test_gather_to_root_gloo_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, slowest = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [row[0] for row in full] == list(range(total))
    assert all(len(set(row)) == 1 for row in full)
    assert slowest == 11.0


def _chunked_worker(rank, world, port, total, chunk, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = shard_range(total, world, rank)
    buf = torch.full((total if rank == 0 else count, 5), -1.0)
    g = ChunkedGather(total, world, rank, chunk, buf)
    view = g.local_view()
    spans = chunk_spans(count, chunk)
    for k in range(g.n_chunks()):
        if k < len(spans):  # "render" chunk k of this rank's shard into its view
            c0, n = spans[k]
            view[c0:c0 + n] = torch.arange(start + c0, start + c0 + n, dtype=torch.float32)[:, None]
        g.post(k)
    g.wait()
    if rank == 0:
        q.put(buf.numpy().tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total,chunk", [(2, 10, 3), (2, 11, 4), (3, 17, 5), (2, 7, 256)])
def test_chunked_gather_gloo(world, total, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunked_worker, args=(r, world, port, total, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [row[0] for row in full] == list(range(total))
    assert all(len(set(row)) == 1 for row in full)
