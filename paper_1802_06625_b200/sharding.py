"""Independent streams sharded across the GPUs of one box.

Streams are independent replicas of one analysed graph (their own rings,
histories and control RNG), so the hot path needs no collective: rank r runs
a contiguous range of streams on its own GPU (one process per GPU, launched
by torchrun).  The only exchange is the final gather of the per-stream
reports to rank 0: captured sink bytes as uint8 tensors through the process
group's backend (NCCL over NVLink on the GPU box), the small digest/count
records as pickled objects.
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
    the local reports are returned as they are.

    The small records (digests, firing counts, occupancies) travel as pickled
    objects; captured sink bytes travel as one uint8 tensor per rank through
    the group's backend -- `dist.gather` over NCCL (NVLink, from the rank's
    device) on the GPU box, gloo on the CPU -- padded to the largest rank."""
    dist = _dist()
    if dist is None:
        return list(local)
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    meta = []
    blobs = []
    for sid, r in zip(streams, local):
        rec = {k: v for k, v in r.__dict__.items() if k != "sink_data"}
        names = sorted(r.sink_data)
        meta.append((sid, rec, [(n, len(r.sink_data[n])) for n in names]))
        blobs.extend(r.sink_data[n] for n in names)
    blob = b"".join(blobs)
    sizes = [None] * world
    dist.all_gather_object(sizes, len(blob))
    gathered_meta = [None] * world if rank == dst else None
    dist.gather_object(meta, gathered_meta, dst=dst)
    pad = max(1, max(sizes))
    nccl = dist.get_backend() == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    t = torch.zeros(pad, dtype=torch.uint8, device=dev)
    if blob:
        t[:len(blob)] = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev)
    parts = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
    dist.gather(t, parts, dst=dst)
    if rank != dst:
        return None
    out: list[RunReport | None] = [None] * total
    for r_meta, part, n in zip(gathered_meta, parts, sizes):
        data = part[:n].cpu().numpy().tobytes()
        off = 0
        for sid, rec, lens in r_meta:
            sinks = {}
            for name, ln in lens:
                sinks[name] = data[off:off + ln]
                off += ln
            out[sid] = RunReport(**rec, sink_data=sinks)
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
