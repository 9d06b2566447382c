"""N>1 host logic on CPU with the gloo backend, world size 2: the request sharding used by
bench.py is a disjoint, complete partition and the timed-region reduction is a max over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_19385_b200.dist import reduce_max, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e = shard_range(total, rank, world)
    mine = torch.arange(s, e, dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([e - s]))
    gathered = [torch.zeros(int(n.item()), dtype=torch.int64) for n in sizes]
    if len(set(int(n.item()) for n in sizes)) == 1:
        dist.all_gather(gathered, mine)
    else:
        for r in range(world):
            buf = mine if r == rank else gathered[r]
            dist.broadcast(buf, src=r)
            gathered[r] = buf
    mx = reduce_max(10.0 * (rank + 1))
    if rank == 0:
        q.put((sorted(torch.cat(gathered).tolist()), mx))
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [64, 65])
def test_gloo_world2_sharding_and_max(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ids == list(range(total))  # complete and disjoint
    assert mx == 20.0


def test_shard_range_balanced():
    for total in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
