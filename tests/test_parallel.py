"""Host logic of the multi-GPU path on CPU: contiguous sharding and the
per-frame SSE all-reduce, with a real 2-process gloo group (127.0.0.1)."""
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


def test_reduce_sse_rejects_out_of_range_shards():
    with pytest.raises(ValueError):
        parallel.reduce_sse(torch.zeros(3, dtype=torch.int64), 8, 10)
    with pytest.raises(ValueError):
        parallel.reduce_sse(torch.zeros(3, dtype=torch.int64), -1, 10)
    assert parallel.reduce_sse(torch.arange(3, dtype=torch.int64), 7, 10).tolist() == [0] * 7 + [0, 1, 2]


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
