"""Independent streams sharded across the GPUs of one box.

Streams are independent replicas of one analysed graph (their own rings,
histories and control RNG), so the hot path needs no collective: rank r runs
a contiguous range of streams on its own GPU (one process per GPU, launched
by torchrun).  The only exchange is the final gather of the per-stream
reports to rank 0, which torch.distributed performs over NCCL (NVLink) for
sink bytes and as pickled objects for the small digest/count records.
"""
from __future__ import annotations

from typing import Callable, Sequence

from .engine import RunReport, RuntimeConfig, run_streams


def stream_range(total: int, rank: int, world: int) -> range:
    """Contiguous share of `total` streams for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return range(lo, hi)


def _dist():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist
    except ImportError:  # pragma: no cover
        pass
    return None


def gather_reports(local: Sequence[RunReport], streams: range, total: int,
                   dst: int = 0) -> list[RunReport] | None:
    """Collect every rank's per-stream reports on `dst`, ordered by stream id.
    Ranks other than dst return None.  Without an initialised process group
    the local reports are returned as they are."""
    dist = _dist()
    if dist is None:
        return list(local)
    payload = (list(streams), [r.__dict__ for r in local])
    gathered = [None] * dist.get_world_size() if dist.get_rank() == dst else None
    dist.gather_object(payload, gathered, dst=dst)
    if dist.get_rank() != dst:
        return None
    out: list[RunReport | None] = [None] * total
    for ids, reps in gathered:
        for sid, d in zip(ids, reps):
            out[sid] = RunReport(**d)
    return out  # type: ignore[return-value]


def run_sharded(graph, total_streams: int, config: RuntimeConfig | None = None,
                seed_of: Callable[[int], int | None] = lambda s: None,
                source_of: Callable[[int], object] | None = None,
                source_actor: str = "src") -> list[RunReport] | None:
    """Run streams [0, total_streams) across the process group: each rank
    fires its contiguous share on its own device; rank 0 receives all
    reports (others get None).  Works on one process without a group."""
    dist = _dist()
    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    mine = stream_range(total_streams, rank, world)
    sources = None
    if source_of is not None:
        sources = {source_actor: [source_of(s) for s in mine]}
    local = run_streams(graph, len(mine), config, seeds=[seed_of(s) for s in mine],
                        sources=sources) if len(mine) else []
    return gather_reports(local, mine, total_streams)
