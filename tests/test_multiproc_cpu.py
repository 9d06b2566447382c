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


def test_launch_plan():
    from paper_2605_19385_b200.dist import launch_plan, spawn_argv
    assert launch_plan(1, {}, 1) == "single"
    assert launch_plan(8, {}, 8) == "spawn"
    assert launch_plan(8, {"WORLD_SIZE": "8"}, 8) == "ranked"
    assert launch_plan(1, {"WORLD_SIZE": "1"}, 1) == "single"
    for gpus, env, vis in ((2, {}, 1), (8, {"WORLD_SIZE": "4"}, 8), (0, {}, 8)):
        with pytest.raises(ValueError):
            launch_plan(gpus, env, vis)
    cmd = spawn_argv("py", "bench.py", ["--gpus", "4"], 4, 29500)
    assert cmd[:3] == ["py", "-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-3:] == ["bench.py", "--gpus", "4"]


def test_bench_refuses_more_gpus_than_visible():
    """`python bench.py --gpus 2` on a box with fewer GPUs must fail loudly, not time one GPU and
    report n_gpus = 1."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    visible = torch.cuda.device_count()
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(visible + 1), "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stdout + r.stderr
    assert f"needs {visible + 1} GPUs" in r.stderr


def _gather_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_19385_b200.dist import gather_floats
    vals = gather_floats(100.0 + rank)
    if rank == 0:
        q.put(vals)
    dist.destroy_process_group()


def test_gloo_world2_per_rank_gather():
    """The bench's per-rank img/s gather (rank order) over gloo, world size 2."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    vals = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert vals == [100.0, 101.0]
