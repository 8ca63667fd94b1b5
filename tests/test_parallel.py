"""Host logic of the multi-GPU path on CPU: contiguous sharding and the
per-frame SSE all-reduce, with a real 2-process gloo group (127.0.0.1)."""
import math
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1606_05562_b200 import parallel  # noqa: E402


def test_shard_covers_and_balances():
    for n in (0, 1, 7, 600, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [parallel.shard(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard(10, 2, 2)


def test_psnr_from_sse():
    assert parallel.psnr_from_sse(0, 10, 8) == math.inf
    assert abs(parallel.psnr_from_sse(256, 256, 8) - 48.1308) < 1e-4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = parallel.shard(n_total, world, rank)
    # per-frame SSE a rank would get from dct16a_codec: a deterministic function of the frame id
    local = torch.tensor([(f * 7919) % 100003 + 2 ** 40 for f in range(a, b)], dtype=torch.int64)
    full = parallel.reduce_sse(local, a, n_total)
    out[rank] = full.tolist()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_total", [(2, 1000), (2, 7), (3, 10)])
def test_sse_allreduce_gloo(world, n_total):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    want = [(f * 7919) % 100003 + 2 ** 40 for f in range(n_total)]
    for r in range(world):
        assert out[r] == want          # every rank holds every frame's SSE, exactly


def _gather_worker(rank, world, port, n_total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = parallel.strided_ids(n_total, world, rank)
    part = torch.tensor([[i * 10 + j for j in range(3)] for i in ids], dtype=torch.int64).reshape(len(ids), 3)
    full = parallel.allgather_strided(part, n_total, world)
    out[rank] = full.tolist()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_total", [(2, 7), (2, 8), (3, 10)])
def test_allgather_strided_gloo(world, n_total):
    """bench.py's input assembly: each rank generates items rank::world, one
    all_gather rebuilds the batch in item order on every rank."""
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n_total, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    want = [[i * 10 + j for j in range(3)] for i in range(n_total)]
    for r in range(world):
        assert out[r] == want
