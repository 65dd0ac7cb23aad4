"""Multi-GPU render inside the library (csrc/group.cpp): positions
split contiguously over the members, scene + weights replicated, one gather of
the outputs to the root. On the one-GPU test box a group of two contexts on the
same device exercises the sharding and the chunked gather (peer-copy transport:
NCCL cannot put two ranks on one device); a one-member group and a one-rank
communicator run the NCCL code path. Across processes, two ranks that each render
their shard through libswr and gather over gloo reproduce a local render bit for
bit (the bench.py --verify flow as a test)."""
import os
import socket

import numpy as np
import pytest

from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
from paper_2506_12787_b200.shard import shard_range

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene():
    sc = make_scene(3000, seed=21)
    sc.rssi_cal = (12.5, -61.0)
    return sc


def _ck(sc, chunk=None):
    ck = swr.Checkpoint.from_scene(sc, device=0)
    if chunk:
        ck.set_option("chunk", chunk)
    return ck


@pytest.mark.parametrize("B", [1, 300, 301])
def test_group_host_render_equals_single(scene, B):
    pos = random_positions(B, seed=B)
    want = swr.render(_ck(scene), pos, rssi=True)
    g = swr.Group([_ck(scene, 64), _ck(scene, 50)])
    got = g.render(pos, rssi=True)
    for k in want:
        assert np.array_equal(want[k], got[k]), k


@pytest.mark.parametrize("members", [1, 2, 3])
def test_group_device_render_gathers_to_root(scene, members):
    import torch
    B = 301
    pos = random_positions(B, seed=7)
    want = swr.render(_ck(scene), pos, rssi=True)
    g = swr.Group([_ck(scene, 40 + 16 * i) for i in range(members)])
    d_pos = torch.from_numpy(pos).cuda()
    H, W = scene.H, scene.W
    d_spec = torch.full((B, H, W, 2), float("nan"), device="cuda")
    d_pooled = torch.zeros(B, dtype=torch.float64, device="cuda")
    d_rssi = torch.zeros(B, dtype=torch.float64, device="cuda")
    d_rc = torch.zeros((B, 2), dtype=torch.int32, device="cuda")
    d_ang = torch.zeros((B, 2), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    flags = swr.OUT_SPECTRA | swr.OUT_POOLED | swr.OUT_RSSI | swr.OUT_AOA
    g.render_device(d_pos.data_ptr(), B, flags, d_spec.data_ptr(), d_pooled.data_ptr(), d_rssi.data_ptr(),
                    d_rc.data_ptr(), d_ang.data_ptr(), st.cuda_stream)
    st.synchronize()
    assert np.array_equal(d_spec.cpu().numpy(), want["spectra"])
    assert np.array_equal(d_pooled.cpu().numpy(), want["pooled"])
    assert np.array_equal(d_rssi.cpu().numpy(), want["rssi"])
    assert np.array_equal(d_rc.cpu().numpy(), want["aoa_rc"])
    assert np.array_equal(d_ang.cpu().numpy(), want["aoa_ang"])


def test_comm_one_rank_render_gather(scene):
    """The cross-process NCCL gather with one rank (ncclCommInitRank over a fresh
    unique id): rank 0 renders in place, spectra and pooled equal swr.render."""
    import torch
    B = 130
    pos = random_positions(B, seed=9)
    ck = _ck(scene, 48)
    want = swr.render(_ck(scene), pos)
    comm = swr.Comm(ck, swr.nccl_unique_id(), 1, 0)
    d_pos = torch.from_numpy(pos).cuda()
    d_spec = torch.zeros((B, scene.H, scene.W, 2), device="cuda")
    d_pooled = torch.zeros(B, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    comm.render_gather(d_pos.data_ptr(), [B], swr.OUT_SPECTRA | swr.OUT_POOLED, d_spec.data_ptr(),
                       d_pooled.data_ptr(), st.cuda_stream)
    st.synchronize()
    assert np.array_equal(d_spec.cpu().numpy(), want["spectra"])
    assert np.array_equal(d_pooled.cpu().numpy(), want["pooled"])
    comm.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_worker(rank, world, port, B, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_12787_b200.shard import gather_to_root
    sc = make_scene(3000, seed=21)
    ck = swr.Checkpoint.from_scene(sc, device=0)   # every rank: its own context (one GPU on the test box)
    pos = random_positions(B, seed=11)
    s0, n = shard_range(B, world, rank)
    out = swr.render(ck, pos[s0:s0 + n])
    spec = gather_to_root(torch.from_numpy(out["spectra"]), B, world, rank)
    pooled = gather_to_root(torch.from_numpy(out["pooled"]), B, world, rank)
    if rank == 0:
        local = swr.render(ck, pos)
        q.put((bool(np.array_equal(spec.numpy(), local["spectra"])),
               bool(np.array_equal(pooled.numpy(), local["pooled"]))))
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [200, 201])
def test_two_ranks_render_and_gather_over_gloo(B):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok == (True, True)
