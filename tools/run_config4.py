#!/usr/bin/env python
"""Config 4 end to end on 1..8 GPUs (BASELINE.json configs[3]): 3840x2160
10-bit frames sharded frame-wise across ranks, fused forward / uniform
quantisation (Δ = 16) / inverse / SSE on each rank (dct16a_codec), then the
single exchange of the path — the SUM all-reduce of the per-frame uint64 SSE
vector over NCCL (paper_1606_05562_b200.parallel.reduce_sse).

Launch: python -m torch.distributed.run --nnodes=1 --nproc-per-node N
        --master-addr 127.0.0.1 --master-port P tools/run_config4.py [--frames F]
(or plainly with python for one GPU).  With fewer GPUs than ranks (--backend
gloo), ranks share the GPUs round-robin: the multi-rank logic (sharding, the
all-reduce over CUDA tensors, the global PSNR) then runs on one B200.  Rank 0 prints one JSON line: global
PSNR from ΣSSE, the per-frame SSE vector (--dump), codec time as the max over
ranks (CUDA events), all-reduce time, blocks/s over all ranks.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import paper_1606_05562_b200 as pkg
    import synth
    from paper_1606_05562_b200 import parallel

    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=1000)
    ap.add_argument("--height", type=int, default=2160)
    ap.add_argument("--width", type=int, default=3840)
    ap.add_argument("--step", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dump", action="store_true", help="print the per-frame SSE vector")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--ipc", action="store_true",
                    help="fuse the SSE all-reduce into the kernel over CUDA IPC-mapped peer vectors "
                         "(parallel.IpcSseAllReduce; works with several ranks on one GPU) and check it against NCCL/gloo")
    ap.add_argument("--fused", action="store_true",
                    help="fuse the SSE all-reduce into the kernel (dct16a_codec_allreduce over symmetric memory) "
                         "and check it against the NCCL path")
    a = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()     # ranks share GPUs when there are fewer GPUs than ranks
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or a.fused or a.ipc:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        if a.backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)

    f0, f1 = parallel.shard(a.frames, world, rank)
    x = torch.from_numpy(synth.frames_10bit(range(f0, f1), H=a.height, W=a.width, total=1000)).to(dev)
    n = f1 - f0
    q = pkg.make_quant("uniform", step=a.step)
    sse = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    d = pkg.desc_of(x) if n else None
    stream = torch.cuda.current_stream(dev)

    def step():
        if n:
            pkg.dct16a_codec(x, q, sse, None, None, d, stream)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.reps):
        step()
    e1.record(stream)
    e1.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / a.reps], dtype=torch.float64, device=dev)
    parallel.reduce_sse(sse[:n], f0, a.frames)          # warm the collective (NCCL setup)
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    full = parallel.reduce_sse(sse[:n], f0, a.frames)
    r1.record(stream)
    r1.synchronize()
    ar_ms = torch.tensor([r0.elapsed_time(r1)], dtype=torch.float64, device=dev)
    fused = None
    if a.fused:
        try:
            fz = parallel.FusedSseAllReduce(a.frames, dev)
        except Exception as e:   # e.g. symmetric memory with several ranks on one GPU
            fused = {"skipped": f"{type(e).__name__}: {str(e).splitlines()[0][:200] if str(e) else ''}"}
        else:
            got = fz.run(x if n else None, q, f0, None, d, stream)
            torch.cuda.synchronize()
            f_e0, f_e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f_e0.record(stream)
            for _ in range(a.reps):
                got = fz.run(x if n else None, q, f0, None, d, stream)
            f_e1.record(stream)
            f_e1.synchronize()
            fused = {"ms": f_e0.elapsed_time(f_e1) / a.reps, "equal_to_nccl": bool(torch.equal(got, full)),
                     "n_peers": len(fz.targets), "multicast": fz.multicast}
    ipc = None
    if a.ipc:
        with parallel.IpcSseAllReduce(a.frames, dev) as iz:
            got = iz.run(x if n else None, q, f0, None, d, stream)
            got = iz.run(x if n else None, q, f0, None, d, stream)   # twice: zeroing between runs
            n_peers = len(iz.peers)
        ok = torch.tensor([1 if torch.equal(got, full) else 0], dtype=torch.int32)
        if world > 1:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)      # every rank's vector, not only rank 0's
        ipc = {"equal_to_collective": bool(ok.item()), "n_peers": n_peers}
    if world > 1:
        if a.backend == "gloo":
            ms, ar_ms = ms.cpu(), ar_ms.cpu()
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(ar_ms, op=dist.ReduceOp.MAX)
    psnr_frames, sse_tot, psnr_tot = parallel.sse_psnr(full, pkg.make_desc(a.width, a.height, 1, 10))
    torch.cuda.synchronize()
    if rank == 0:
        tot = int(sse_tot.item())
        assert tot == int(full.sum().item())
        P = a.frames * a.height * a.width
        blocks = a.frames * (a.height // 16) * (a.width // 16)
        line = {"config": 4, "n_gpus": world, "frames": a.frames, "step": a.step,
                "codec_ms_max_over_ranks": float(ms.item()), "allreduce_ms": float(ar_ms.item()),
                "blocks_per_s": blocks / (float(ms.item()) / 1e3),
                "global_psnr_db": float(psnr_tot.item()), "sse_total": tot, "backend": a.backend if world > 1 else None,
                "pixels": P}
        if fused is not None:
            line["fused_allreduce"] = fused
        if ipc is not None:
            line["ipc_allreduce"] = ipc
        if a.dump:
            line["sse"] = full.cpu().tolist()
            line["psnr"] = psnr_frames.cpu().tolist()
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
