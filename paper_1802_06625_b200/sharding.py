"""Independent streams sharded across the GPUs of one box.

Streams are independent replicas of one analysed graph (their own rings,
histories and control RNG), so the hot path needs no collective: rank r runs
a contiguous range of streams on its own GPU (one process per GPU, launched
by torchrun).  The only exchange is the final gather of the per-stream
reports to rank 0: captured sink bytes as uint8 tensors through the process
group's backend (NCCL over NVLink on the GPU box), the small digest/count
records as pickled objects.  `gather_sink_rings` moves the sink bytes
straight out of the device rings (a zero-copy torch view of the ring storage,
NCCL gather device to device), so no rank round-trips them through the host.
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


class _DeviceBytes:
    """__cuda_array_interface__ over library-owned device memory, so torch can
    view a ring's storage without a copy (torch.as_tensor)."""

    def __init__(self, ptr: int, shape: tuple[int, ...], strides: tuple[int, ...]):
        self.__cuda_array_interface__ = {"shape": shape, "strides": strides, "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


def ring_view(rt, fid: str, n_iter: int):
    """uint8 torch view [S, n_iter * span] of FIFO `fid`'s ring on the
    runtime's device, valid for a run that started from reset (write counter
    0) and fired n_iter <= slots iterations: chunk n of stream s is iteration
    n (fifos.py:87-98 aligned ring, no wrap)."""
    import torch
    st = rt.storage[fid]
    if n_iter > st.slots:
        raise ValueError(f"{fid}: {n_iter} iterations wrap a ring of {st.slots} chunks")
    cai = _DeviceBytes(st.data, (rt.n_streams, n_iter * st.span), (st.stream_stride, 1))
    return torch.as_tensor(cai, device=torch.device("cuda", int(rt.config.device)))


def gather_sink_rings(rt, sink: str, n_iter: int, dst: int = 0):
    """Gather the last run's sink-channel bytes of every rank to `dst`
    directly from the device rings (NCCL gather over NVLink; gloo falls back
    to host tensors).  Returns the [world * S, n_iter * span] uint8 tensor
    (stream-major, rank-contiguous) on dst, None elsewhere.  Without a process
    group the local view is returned."""
    from .graph import PortRef
    a = rt.graph.actor(sink)
    (p,) = a.input_ports
    fid = rt.graph.fifo_into(PortRef(sink, p.id)).id
    view = ring_view(rt, fid, n_iter)
    dist = _dist()
    if dist is None:
        return view
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    t = view.contiguous() if dist.get_backend() == "nccl" else view.cpu()
    parts = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
    dist.gather(t, parts, dst=dst)
    return torch.cat(parts, 0) if rank == dst else None


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
