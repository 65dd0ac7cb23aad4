"""Multi-GPU plumbing: shard TX positions across ranks, gather outputs to root.

SURVEY.md section 8(e): positions are independent units, so a batch of B
positions is split contiguously across P ranks (one process per GPU), the
scene and MLP weights are replicated on every GPU, and the only collective is
the final gather of the rendered outputs to rank 0 (NCCL over NVLink on the
GPUs; the same code runs on gloo for the CPU tests). Nothing here computes a
spectrum: rendering is libswr.so's job on each rank's own device.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, start + count) share of `total` units for `rank`;
    the first total % world ranks take one extra unit."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def gather_to_root(local: torch.Tensor, total: int, world: int, rank: int, root: int = 0):
    """Gather the ranks' contiguous shards (dim 0) into one tensor on `root`.
    Shards may differ by one row (shard_range); they are padded to a common
    length for the collective and trimmed afterwards. Returns the full tensor
    on root and None elsewhere."""
    if world == 1:
        return local
    per = -(-total // world)
    start, count = shard_range(total, world, rank)
    if local.shape[0] != count:
        raise ValueError("local shard has the wrong length")
    pad = local
    if count < per:
        pad = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[:count] = local
    dev = pad.device
    if pad.is_cuda and dist.get_backend() == "gloo":  # gloo moves host memory only (plumbing tests)
        pad = pad.cpu()
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == root else None
    dist.gather(pad, gather_list=bufs, dst=root)
    if rank == root:
        bufs = [b.to(dev) for b in bufs]
    if rank != root:
        return None
    parts = []
    for r in range(world):
        _, c = shard_range(total, world, r)
        parts.append(bufs[r][:c])
    return torch.cat(parts, dim=0)


def chunk_spans(count: int, chunk: int) -> list[tuple[int, int]]:
    """[(first, n)] chunks of a rank's `count` units, `chunk` at a time."""
    return [(c0, min(chunk, count - c0)) for c0 in range(0, count, chunk)]


class ChunkedGather:
    """Overlapped gather to root ("on a comm stream in
    chunks overlapped with rendering"). Each rank renders its contiguous shard
    chunk by chunk; after chunk k is enqueued, `post(k)` sends it to root with a
    non-blocking point-to-point send (root posts the matching receives straight
    into its full output buffer, so nothing is padded or concatenated). With
    NCCL the transfers run on NCCL's own stream, ordered after the chunk's render
    and concurrent with the next chunk's. `wait()` completes every transfer.

    `out` is the root's [total, ...] buffer (the root renders its own shard
    directly into its slice of it); `local` is a non-root rank's [count, ...]
    buffer."""

    def __init__(self, total: int, world: int, rank: int, chunk: int, buf: torch.Tensor, root: int = 0):
        self.total, self.world, self.rank, self.root, self.chunk = total, world, rank, root, chunk
        self.buf = buf
        self.spans = [shard_range(total, world, r) for r in range(world)]
        self.reqs = []
        # gloo cannot move device memory: stage through host copies (plumbing tests only)
        self.stage = buf.is_cuda and dist.is_initialized() and dist.get_backend() == "gloo"
        self.landing = []

    def local_view(self) -> torch.Tensor:
        """Where this rank writes its shard: its slice of `out` on root, `local` elsewhere."""
        if self.rank == self.root:
            s, c = self.spans[self.rank]
            return self.buf[s:s + c]
        return self.buf

    def n_chunks(self) -> int:
        return max(len(chunk_spans(c, self.chunk)) for _, c in self.spans)

    def post(self, k: int) -> None:
        if self.world == 1:
            return
        if self.rank == self.root:
            for r, (s, c) in enumerate(self.spans):
                if r == self.root:
                    continue
                sp = chunk_spans(c, self.chunk)
                if k < len(sp):
                    c0, n = sp[k]
                    dst = self.buf[s + c0:s + c0 + n]
                    if self.stage:
                        tmp = torch.empty(dst.shape, dtype=dst.dtype)
                        self.landing.append((dst, tmp))
                        dst = tmp
                    self.reqs.append(dist.irecv(dst, src=r))
        else:
            sp = chunk_spans(self.spans[self.rank][1], self.chunk)
            if k < len(sp):
                c0, n = sp[k]
                src = self.buf[c0:c0 + n]
                if self.stage:
                    src = src.cpu()  # synchronous copy after the chunk's render
                    self.landing.append((None, src))  # keep alive until wait()
                self.reqs.append(dist.isend(src, dst=self.root))

    def wait(self) -> None:
        for r in self.reqs:
            r.wait()
        self.reqs = []
        for dst, tmp in self.landing:
            if dst is not None:
                dst.copy_(tmp)
        self.landing = []


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
