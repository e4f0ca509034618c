"""Stream sharding across GPUs.

Video streams are independent (only predict/match/update is sequential, and
only within a stream), so the multi-GPU path is pure data parallelism over
streams: one process per GPU owns a disjoint, contiguous block of global
stream ids and runs them batched in one `Tracker` on its own device.  No
collective touches the data path; the only cross-rank traffic is the final
host gather of the track records (kilobytes per stream) and, for timing,
a barrier and a max-reduction of elapsed times.

The reference has no multi-GPU code (SPEC.md:456 lists multi-GPU dispatch as
a non-goal); this module is north_star's "partitioned across the GPUs of one
box by independent video streams ... only a final host gather of track
results".
"""
from __future__ import annotations

import os

SEED_BASE = 1000  # stream seed = 1000 + global stream id


def stream_seed(global_id: int) -> int:
    """Seed of the synthetic stream with this global id (rank independent)."""
    return SEED_BASE + int(global_id)


def shard(rank: int, world: int, per_rank: int | None = None, total: int | None = None):
    """Global stream ids owned by `rank`.

    per_rank=B (weak scaling): rank r owns [r*B, (r+1)*B).
    total=T (strong scaling, C5's 64 streams split over N GPUs): contiguous
    blocks whose sizes differ by at most one, lower ranks first."""
    if (per_rank is None) == (total is None):
        raise ValueError("give exactly one of per_rank / total")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if per_rank is not None:
        if per_rank < 1:
            raise ValueError("per_rank must be >= 1")
        return list(range(rank * per_rank, (rank + 1) * per_rank))
    if total < world:
        raise ValueError(f"{total} streams cannot be split over {world} GPUs")
    base, extra = divmod(int(total), world)
    lo = rank * base + min(rank, extra)
    return list(range(lo, lo + base + (1 if rank < extra else 0)))


def dist_env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None):
    """Initialise torch.distributed when WORLD_SIZE > 1.  backend=None picks
    NCCL when CUDA is available (and binds LOCAL_RANK's device), gloo
    otherwise; FT_DIST_BACKEND or `backend` force one (tests run several
    ranks on one GPU over gloo)."""
    ws, rank, local = dist_env()
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = backend or os.environ.get("FT_DIST_BACKEND") or (
            "nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        if not dist.is_initialized():
            dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws: int) -> None:
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws: int, v: float) -> float:
    """Max over ranks (device timing is reported as the slowest rank)."""
    if ws == 1:
        return float(v)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_tracks(ws: int, rank: int, ids, records):
    """Final host gather: every rank sends {global stream id: record array}
    for its streams to rank 0, which returns the merged dict ordered by
    stream id (other ranks return None).  `records` is the per-stream list a
    Tracker step returns (TRACK_DTYPE arrays)."""
    local = {int(g): r for g, r in zip(ids, records)}
    if ws == 1:
        return dict(sorted(local.items()))
    import torch.distributed as dist
    out = [None] * ws if rank == 0 else None
    dist.gather_object(local, out, dst=0)
    if rank != 0:
        return None
    merged = {}
    for part in out:
        dup = merged.keys() & part.keys()
        if dup:
            raise RuntimeError(f"streams {sorted(dup)} owned by two ranks")
        merged.update(part)
    return dict(sorted(merged.items()))
