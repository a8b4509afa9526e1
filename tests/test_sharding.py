"""Stream sharding and the report gather on a world-size-2 gloo group (CPU)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1802_06625_b200.engine import RunReport
from paper_1802_06625_b200.sharding import gather_reports, stream_range


@pytest.mark.parametrize("total,world", [(64, 1), (64, 2), (64, 8), (7, 3), (2, 4)])
def test_stream_range_partitions(total, world):
    ranges = [stream_range(total, r, world) for r in range(world)]
    flat = [s for r in ranges for s in r]
    assert flat == list(range(total))
    sizes = [len(r) for r in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_stream_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        stream_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = 5
    mine = stream_range(total, rank, world)
    local = [RunReport(sink_digests={"sink": f"d{s}"}, firing_counts={"src": 10 + s},
                       sink_data={"sink": bytes([s]) * 3}) for s in mine]
    out = gather_reports(local, mine, total)
    q.put((rank, None if out is None else [(r.sink_digests["sink"], r.firing_counts["src"],
                                            r.sink_data["sink"]) for r in out]))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_reports_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] is None
    assert res[0] == [(f"d{s}", 10 + s, bytes([s]) * 3) for s in range(5)]


def _sharded_worker(rank, world, port, q):
    import hashlib

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import dpd as od
    from paper_1802_06625_b200 import RuntimeConfig
    from paper_1802_06625_b200.apps import predistortion as pd
    from paper_1802_06625_b200.sharding import run_sharded
    S, blocks, B = 5, 6, 256
    reps = run_sharded(pd.build_description(B, 4), S,
                       RuntimeConfig(source_firings=blocks, capture_sinks=True),
                       seed_of=lambda s: 1000 + s,
                       source_of=lambda s: pd.stream_input(s, blocks, B).tobytes())
    if rank == 0:
        ok = []
        for s in range(S):
            want = od.dpd_stream(pd.stream_input(s, blocks, B),
                                 od.subset_schedule(1000 + s, blocks), 4).tobytes()
            ok.append(reps[s].sink_data["sink"] == want and
                      reps[s].sink_digests["sink"] == hashlib.sha256(want).hexdigest())
        q.put(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_run_sharded_two_ranks_one_gpu():
    """Two ranks (both on cuda:0 here; one per GPU on a multi-GPU box) run a
    contiguous share of 5 streams each and rank 0 gathers every report, sink
    bytes included, bit-exact against the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok == [True] * 5
