"""Replication sharding over GPUs (one process per GPU, torch.distributed).

Replications are independent units: rank r of W owns the
contiguous ids [1 + r*M/W, (r+1)*M/W] (remainder spread over the first
ranks), runs the whole device pipeline for them with no data-path
collective, and the M x |grid| theta matrix (at most a few hundred KB) is
all-gathered once (NCCL over NVLink on GPUs, gloo on CPU).  Because theta
is a pure function of (seed, generator, replication, N), the gathered
matrix is bit-identical for any world size -- the device analogue of the
reference's worker-count invariance (test_harness.py:127-143).
"""

from __future__ import annotations

import numpy as np


def active(flag: bool | None) -> bool:
    if flag is False:
        return False
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return False
    on = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
    if flag and not on:
        raise RuntimeError("distributed=True but torch.distributed is not initialised")
    return on


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first offset, count) of rank's contiguous share of `total` units."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def bind_device() -> None:
    """Under torchrun, put this rank on GPU LOCAL_RANK (mod the visible GPUs)
    unless the caller already moved it off device 0."""
    import os

    import torch

    if "LOCAL_RANK" not in os.environ or not torch.cuda.is_available():
        return
    n = torch.cuda.device_count()
    want = int(os.environ["LOCAL_RANK"]) % max(1, n)
    if torch.cuda.current_device() == 0 and want != 0:
        torch.cuda.set_device(want)


_ERRORS = {"ArithmeticError": ArithmeticError, "ValueError": ValueError,
           "RuntimeError": RuntimeError}


def _raise_collective(status, group=None) -> None:
    """Re-raise the first failing rank's error on EVERY rank (same type), so
    no rank is left blocked in the data gather (the reference raises
    ArithmeticError cleanly from its one process)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    every = [None] * world
    dist.all_gather_object(every, status, group=group)
    for r, st in enumerate(every):
        if st is None:
            continue
        kind, msg = st
        if kind == "ConfigurationError":
            from .harness import ConfigurationError

            raise ConfigurationError(f"rank {r}: {msg}")
        cls = _ERRORS.get(kind, RuntimeError)
        raise cls(f"rank {r}: {kind}: {msg}" if cls is RuntimeError else f"rank {r}: {msg}")


def gather_rows(local: np.ndarray, total: int, group=None) -> np.ndarray:
    """All-gather row blocks of a [count, k] float64 matrix in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    k = local.shape[1]
    counts = [shard(total, world, r)[1] for r in range(world)]
    width = max(counts)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    buf = torch.zeros((width, k), dtype=torch.float64, device=dev)
    buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(dev)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return np.concatenate([o[:c].cpu().numpy() for o, c in zip(outs, counts)], axis=0)


def estimate_sharded(generator: str, model, seed: int, replications: int, grid,
                     group=None, estimator=None) -> np.ndarray:
    """theta[M, |grid|] with replications sharded over the process group."""
    import torch.distributed as dist

    from .harness import estimate_replications

    est = estimator or estimate_replications
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    first, count = shard(replications, world, rank)
    if estimator is None:
        bind_device()
    local, status = np.zeros((count, len(grid))), None
    if count:
        try:
            local = np.asarray(est(generator, model, seed, 1 + first, count, grid))
        except Exception as e:  # noqa: BLE001 -- re-raised on every rank below
            status = (type(e).__name__, str(e))
    _raise_collective(status, group)
    return gather_rows(local, replications, group)
