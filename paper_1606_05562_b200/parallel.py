"""Multi-GPU plumbing for the codec path.

Frames/images are independent (the codec is intra-only), so they are sharded
contiguously across ranks with no data-path collective.  Config 4's single
exchange is the SUM all-reduce of the per-frame SSE vector: every rank writes
its slice of an int64 [n_total] vector (zeros elsewhere) and one all-reduce
yields both the per-frame and the global SSE (exact, order independent).
torch.distributed provides the process group (NCCL on GPUs, gloo in the CPU
tests and for several ranks sharing one GPU); every per-frame computation,
the PSNR of each frame and of the whole set included, runs in libdct16a.
"""
from __future__ import annotations


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
    if offset < 0 or offset + local_sse.numel() > n_total:
        raise ValueError(f"frames [{offset}, {offset + local_sse.numel()}) outside [0, {n_total})")
    full = torch.zeros(n_total, dtype=torch.int64, device=local_sse.device)
    full[offset:offset + local_sse.numel()] = local_sse
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


def sse_psnr(full_sse, desc, stream=None):
    """Per-frame PSNR, the exact ΣSSE and the PSNR of the whole set from an
    all-reduced per-frame SSE vector, through the library's finaliser
    (dct16a_sse_psnr, readings A7/A8).  Returns device
    tensors (psnr float64 [n], sse_total int64 [1], psnr_total float64 [1])."""
    import torch
    from . import _lib
    n = full_sse.numel()
    psnr = torch.empty(n, dtype=torch.float64, device=full_sse.device)
    tot = torch.empty(1, dtype=torch.int64, device=full_sse.device)
    ptot = torch.empty(1, dtype=torch.float64, device=full_sse.device)
    _lib.dct16a_sse_psnr(full_sse, n, desc, psnr, tot, ptot, stream)
    return psnr, tot, ptot


class FusedSseAllReduce:
    """The config-4 exchange fused into the codec kernel (dct16a_codec_allreduce,
    SURVEY.md §8(f) f2): one int64 [n_total] SSE vector per rank in torch
    symmetric memory; every rank's kernel adds each local frame's SSE into all
    ranks' vectors — through the NVLS multicast address when the group has one
    (multimem.red: one store reaches every GPU through the NVSwitch), else by
    peer-mapped atomics over NVLink.  Symmetric-memory barriers order the
    zeroing before, and the reads after, every rank's kernel.  Reuse one
    instance; the vector returned by run() is overwritten by the next run()."""

    def __init__(self, n_total: int, device, group=None, use_multicast: bool = True):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.n_total = int(n_total)
        self.buf = symm.empty(self.n_total, dtype=torch.int64, device=device)
        self.handle = symm.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        self.peers = list(self.handle.buffer_ptrs)
        if len(self.peers) > 8:
            raise ValueError("dct16a_codec_allreduce supports up to 8 peers")
        mc = int(getattr(self.handle, "multicast_ptr", 0) or 0) if use_multicast else 0
        # the multicast address maps every rank's copy of the vector: one peer entry
        self.targets = [mc] if mc else self.peers
        self.multicast = bool(mc)

    def run(self, frames, quant, frame_offset: int, recon=None, desc=None, stream=None):
        """Codec of this rank's frames; returns the all-reduced per-frame SSE (int64)."""
        import torch
        from . import _lib
        n = 0 if frames is None else int(frames.shape[0])
        if frame_offset < 0 or frame_offset + n > self.n_total:
            raise ValueError(f"frames [{frame_offset}, {frame_offset + n}) outside the vector [0, {self.n_total})")
        cur = torch.cuda.current_stream(self.buf.device)
        if stream is not None and getattr(stream, "cuda_stream", stream) != cur.cuda_stream:
            raise ValueError("run() must be called on torch's current stream (zeroing and barriers use it)")
        self.buf.zero_()
        self.handle.barrier()            # every rank's vector is zero before any kernel adds
        if n > 0:
            _lib.dct16a_codec_allreduce(frames, quant, self.targets, frame_offset, recon, desc, cur,
                                        multicast=self.multicast)
        self.handle.barrier()            # every rank's kernel has finished adding
        return self.buf


class IpcSseAllReduce:
    """The fused in-kernel SSE all-reduce (dct16a_codec_allreduce, peer atomics)
    over CUDA IPC instead of symmetric memory: every rank cudaMallocs its int64
    [n_total] vector, the IPC handles are exchanged over the process group, and
    each rank maps every other rank's vector — which also works for several
    processes sharing one GPU (symmetric memory refuses that), so the
    multi-peer path runs on this pool's single-GPU boxes.  Barriers of the
    process group (after a device synchronisation) order the zeroing before,
    and the reads after, every rank's kernel."""

    def __init__(self, n_total: int, device, group=None):
        import torch
        import torch.distributed as dist
        from cuda.bindings import runtime as rt
        self.rt, self.dist, self.group = rt, dist, group
        self.n_total = int(n_total)
        self.device = torch.device(device)
        self.nbytes = 8 * self.n_total
        err, ptr = rt.cudaMalloc(max(self.nbytes, 8))
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"cudaMalloc: {err}")
        self.ptr = int(ptr)
        err, h = rt.cudaIpcGetMemHandle(self.ptr)
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"cudaIpcGetMemHandle: {err}")
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, bytes(h.reserved), group=group)
        me = dist.get_rank(group)
        self.opened = []
        self.peers = []
        for r, hb in enumerate(handles):
            if r == me:
                self.peers.append(self.ptr)
                continue
            ph = rt.cudaIpcMemHandle_t()
            ph.reserved = hb
            err, pp = rt.cudaIpcOpenMemHandle(ph, rt.cudaIpcMemLazyEnablePeerAccess)
            if err != rt.cudaError_t.cudaSuccess:
                raise RuntimeError(f"cudaIpcOpenMemHandle (rank {r}): {err}")
            self.opened.append(int(pp))
            self.peers.append(int(pp))
        if len(self.peers) > 8:
            raise ValueError("dct16a_codec_allreduce supports up to 8 peers")

    def run(self, frames, quant, frame_offset: int, recon=None, desc=None, stream=None):
        """Codec of this rank's frames; returns the all-reduced per-frame SSE
        (int64 [n_total], a copy of this rank's vector)."""
        import torch
        from . import _lib
        n = 0 if frames is None else int(frames.shape[0])
        if frame_offset < 0 or frame_offset + n > self.n_total:
            raise ValueError(f"frames [{frame_offset}, {frame_offset + n}) outside the vector [0, {self.n_total})")
        rt = self.rt
        rt.cudaMemset(self.ptr, 0, self.nbytes)
        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)       # every rank's vector is zero before any kernel adds
        if n > 0:
            _lib.dct16a_codec_allreduce(frames, quant, self.peers, frame_offset, recon, desc, stream)
        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)       # every rank's kernel has finished adding
        out = torch.empty(self.n_total, dtype=torch.int64, device=self.device)
        rt.cudaMemcpy(out.data_ptr(), self.ptr, self.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
        return out

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def close(self):
        """Unmap the peers' vectors and free this rank's (every rank must call it,
        after the last run(); also on leaving a `with` block)."""
        for pp in self.opened:
            self.rt.cudaIpcCloseMemHandle(pp)
        self.opened = []
        if self.ptr and self.dist.is_initialized():
            self.dist.barrier(group=self.group)   # no rank still maps this vector
        if self.ptr:
            self.rt.cudaFree(self.ptr)
            self.ptr = 0


def codec_sharded(local_frames, offset: int, n_total: int, mode: str = "uniform", r: int = 16,
                  step: int = 16, valid_height: int | None = None, group=None, want_recon: bool = False):
    """Run the fused codec on this rank's frames and all-reduce the SSE.
    Returns (recon or None, per-frame SSE int64 [n_total], per-frame PSNR
    float64 [n_total], global PSNR float64 [1]) — device tensors."""
    import torch
    from . import _lib, codec
    n, h, w = local_frames.shape
    if n:
        recon, sse_local, _ = codec(local_frames, mode, r=r, step=step, valid_height=valid_height,
                                    want_recon=want_recon)
    else:   # an empty shard still takes part in the collective
        recon, sse_local = None, torch.empty(0, dtype=torch.int64, device=local_frames.device)
    full = reduce_sse(sse_local, offset, n_total, group)
    bits = _lib._pixel_depth(local_frames, None)
    desc = _lib.make_desc(w, h, 1, bits, valid_height=valid_height)   # the geometry of one frame
    psnr, _, ptot = sse_psnr(full, desc)
    return recon, full, psnr, ptot
