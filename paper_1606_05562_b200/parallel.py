"""Multi-GPU plumbing for the codec path.

Frames/images are independent (the codec is intra-only), so they are sharded
contiguously across ranks with no data-path collective.  Config 4's single
exchange is the SUM all-reduce of the per-frame SSE vector: every rank writes
its slice of an int64 [n_total] vector (zeros elsewhere) and one all-reduce
yields both the per-frame and the global SSE (exact, order independent).
torch.distributed provides the process group (NCCL on GPUs, gloo in the CPU
tests); the per-frame work runs in libdct16a.
"""
from __future__ import annotations

import math


def shard(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced shard [start, stop) of n_items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def reduce_sse(local_sse, offset: int, n_total: int, group=None):
    """Place this rank's per-frame SSE (int64 tensor) at `offset` of a zero
    [n_total] vector and SUM all-reduce it across the group."""
    import torch
    import torch.distributed as dist
    full = torch.zeros(n_total, dtype=torch.int64, device=local_sse.device)
    full[offset:offset + local_sse.numel()] = local_sse
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


class FusedSseAllReduce:
    """The config-4 exchange fused into the codec kernel (dct16a_codec_allreduce):
    one int64 [n_total] SSE vector per rank in torch symmetric memory; every
    rank's kernel adds each local frame's SSE into all ranks' vectors over
    peer-mapped memory (NVLink).  Symmetric-memory barriers order the zeroing
    before, and the reads after, every rank's kernel.  Reuse one instance."""

    def __init__(self, n_total: int, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.n_total = n_total
        self.buf = symm.empty(n_total, dtype=torch.int64, device=device)
        self.handle = symm.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        self.peers = list(self.handle.buffer_ptrs)
        if len(self.peers) > 8:
            raise ValueError("dct16a_codec_allreduce supports up to 8 peers")

    def run(self, frames, quant, frame_offset: int, recon=None, desc=None, stream=None):
        """Codec of this rank's frames; returns the all-reduced per-frame SSE (int64)."""
        from . import _lib
        self.buf.zero_()
        self.handle.barrier()            # every rank's vector is zero before any kernel adds
        if frames is not None and frames.shape[0] > 0:
            _lib.dct16a_codec_allreduce(frames, quant, self.peers, frame_offset, recon, desc, stream)
        self.handle.barrier()            # every rank's kernel has finished adding
        return self.buf


def psnr_from_sse(sse_total: int, n_pixels: int, bit_depth: int) -> float:
    """10·log10(peak²·P/SSE), +inf for SSE = 0 (reading A7)."""
    if sse_total == 0:
        return math.inf
    peak = (1 << bit_depth) - 1
    return 10.0 * math.log10(peak * peak * n_pixels / sse_total)


def codec_sharded(local_frames, offset: int, n_total: int, mode: str = "uniform", r: int = 16,
                  step: int = 16, valid_height: int | None = None, group=None, want_recon: bool = False):
    """Run the fused codec on this rank's frames and all-reduce the SSE.
    Returns (recon or None, per-frame SSE int64 [n_total], global PSNR)."""
    from . import codec
    recon, sse_local, _ = codec(local_frames, mode, r=r, step=step, valid_height=valid_height,
                                want_recon=want_recon)
    full = reduce_sse(sse_local, offset, n_total, group)
    n, h, w = local_frames.shape
    vh = h if valid_height is None else valid_height
    bits = 8 if local_frames.element_size() == 1 else 10
    total = int(full.sum().item())
    return recon, full, psnr_from_sse(total, n_total * vh * w, bits)


def strided_ids(n_items: int, world: int, rank: int) -> list[int]:
    """Items r, r + world, r + 2·world, ... — the ids rank `rank` generates when
    every rank needs the whole batch (weak-scaling bench inputs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_items, world))


def allgather_strided(part, n_items: int, world: int, group=None):
    """Reassemble the full batch from every rank's strided part (part = items
    rank, rank + world, ...; shape (len, ...)) with one all_gather of equal-size
    padded buffers; returns the (n_items, ...) tensor in item order on every rank."""
    import torch
    import torch.distributed as dist
    m = (n_items + world - 1) // world
    buf = torch.zeros((m, *part.shape[1:]), dtype=part.dtype, device=part.device)
    buf[:part.shape[0]] = part
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.empty((n_items, *part.shape[1:]), dtype=part.dtype, device=part.device)
    for r in range(world):
        cnt = len(range(r, n_items, world))
        out[r::world] = parts[r][:cnt]
    return out
