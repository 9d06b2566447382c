"""Request sharding across the GPUs of one box: whole requests are partitioned
across ranks, never split, and there is no collective on the data path.  The only collective is
the max-over-ranks reduction of the timed region (bench).  Mirrors the reference's placement
rule -- a request goes to exactly one executor (proj/src/sim.cpp:238-243, 411) -- at rank
granularity: rank r owns a contiguous, balanced block of the global batch."""
from __future__ import annotations


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[start, end) of the requests rank `rank` decodes out of `total` (balanced, contiguous)."""
    if world <= 0 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def reduce_max(value: float, device=None) -> float:
    """Max over ranks of a scalar (identity when torch.distributed is not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def launch_plan(gpus: int, env: dict, visible_gpus: int) -> str:
    """How `bench.py --gpus N` runs (the driver may launch it under torchrun or bare):
      "single"  N == 1 and no torchrun environment;
      "ranked"  under torchrun with WORLD_SIZE == N (this process is one rank);
      "spawn"   N > 1 without torchrun: re-launch through torch.distributed.run, one rank per GPU.
    Raises ValueError (the bench exits non-zero) when the request cannot be honoured: fewer visible
    GPUs than N, or a torchrun world size that disagrees with --gpus -- a silently smaller run would
    report the wrong n_gpus."""
    if gpus < 1:
        raise ValueError(f"--gpus {gpus}: must be >= 1")
    world = env.get("WORLD_SIZE")
    if world is not None and int(world) != gpus:
        raise ValueError(f"--gpus {gpus} but WORLD_SIZE={world}: launch with --nproc-per-node {gpus}")
    if visible_gpus < gpus:
        raise ValueError(f"--gpus {gpus} needs {gpus} GPUs; {visible_gpus} visible")
    if world is not None and int(world) > 1:
        return "ranked"
    return "spawn" if gpus > 1 else "single"


def spawn_argv(python: str, script: str, argv: list, gpus: int, port: int) -> list:
    """torch.distributed.run command line for N ranks on this node (rendezvous on 127.0.0.1)."""
    return [python, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", script] + list(argv)


def gather_floats(value: float, device=None) -> list:
    """Every rank's scalar, in rank order (the value itself when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(value)]
    if dist.get_backend() == "gloo":
        device = None
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]
