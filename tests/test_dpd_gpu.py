"""DPD filter bank on the B200 vs the reference's golden vectors and the
oracle: bit-exact sink bytes, firing counts, Eq. 1 counters, occupancy."""
import hashlib

import numpy as np
import pytest

from oracle import dpd as od
from paper_1802_06625_b200 import RuntimeConfig, run, run_streams
from paper_1802_06625_b200.apps import predistortion as pd

pytestmark = pytest.mark.gpu


def dpd_graph(tmp_path, data: bytes, block=256, branches=4, min_active=2):
    p = tmp_path / "input.bin"
    p.write_bytes(data)
    return pd.build_description(block, branches, str(p), min_active)


@pytest.mark.parametrize("epoch_close", ["1", "0"])
@pytest.mark.parametrize("fuse", [True, False])
@pytest.mark.parametrize("epoch", [4096, 7])
def test_default_app_digest(golden, tmp_path, monkeypatch, fuse, epoch, epoch_close):
    # epoch_close "1": the Eq. 1 recheck and the ring advance in one launch
    # (pb_epoch_close); "0": pb_eq1_check after resolve, pb_rings_advance at the end
    monkeypatch.setenv("PB_EPOCH_CLOSE", epoch_close)
    g = golden["dpd"]["default"]
    desc = dpd_graph(tmp_path, pd.make_input(11, 160))
    rep = run(desc, config=RuntimeConfig(source_firings=160, seed=11, fuse=fuse, epoch=epoch))
    assert rep.sink_digests["sink"] == g["sink_digest"]
    assert rep.firing_counts == g["firing_counts"]
    assert rep.eq1_checks == 8 * 160 and rep.eq1_failures == 0
    for fid, occ in rep.max_occupancy.items():
        assert occ <= rep.beta[fid] and occ <= rep.slots[fid], fid


@pytest.mark.parametrize("fuse", [True, False])
def test_small_run_bytes(golden, tmp_path, fuse):
    arr = golden["dpd_small"]
    desc = dpd_graph(tmp_path, arr["small_input"].tobytes())
    rep = run(desc, config=RuntimeConfig(source_firings=6, seed=11, capture_sinks=True,
                                         fuse=fuse))
    assert rep.sink_data["sink"] == arr["small_sink"].tobytes()
    assert rep.eq1_checks == 48 and rep.eq1_failures == 0   # test_apps.py:152-159


def test_impulse_all_active(golden, tmp_path):
    imp = np.zeros(512, np.float32)
    imp[0] = 1.0
    desc = dpd_graph(tmp_path, imp.tobytes(), min_active=4)
    rep = run(desc, config=RuntimeConfig(source_firings=1, seed=11, capture_sinks=True))
    assert rep.sink_data["sink"] == golden["dpd_small"]["impulse_sink"].tobytes()


@pytest.mark.parametrize("fuse", [True, False])
def test_c2_shape_streams(golden, fuse):
    xs = [pd.stream_input(s, 24, 4096) for s in (0, 1)]
    desc = pd.build_description(4096, 4)
    reps = run_streams(desc, 2, RuntimeConfig(source_firings=24, fuse=fuse),
                       seeds=[1000, 1001], sources={"src": [x.tobytes() for x in xs]})
    for s, rep in enumerate(reps):
        assert rep.sink_digests["sink"] == golden["dpd"][f"c2_stream{s}"]["sink_digest"]
        assert rep.firing_counts == golden["dpd"][f"c2_stream{s}"]["firing_counts"]


@pytest.mark.parametrize("fuse", [True, False])
def test_k10_paper_scale(golden, fuse):
    x = pd.stream_input(7, 16, 512)
    desc = pd.build_description(512, 10)
    (rep,) = run_streams(desc, 1, RuntimeConfig(source_firings=16, capture_sinks=True,
                                                fuse=fuse),
                         seeds=[1007], sources={"src": [x.tobytes()]})
    assert rep.sink_data["sink"] == golden["dpd_small"]["k10_sink"].tobytes()


def test_many_streams_against_oracle():
    S, blocks, B = 6, 40, 1024
    xs = [pd.stream_input(s, blocks, B) for s in range(S)]
    desc = pd.build_description(B, 4)
    reps = run_streams(desc, S, RuntimeConfig(source_firings=blocks, epoch=16),
                       seeds=[1000 + s for s in range(S)],
                       sources={"src": [x.tobytes() for x in xs]})
    for s in range(S):
        sets = od.subset_schedule(1000 + s, blocks)
        want = od.dpd_stream(xs[s], sets, 4).tobytes()
        assert reps[s].sink_digests["sink"] == hashlib.sha256(want).hexdigest()
        assert reps[s].firing_counts == od.firing_counts(sets, 4)


def fir_chain(block):
    re, im = pd.branch_taps(2)
    return {"name": "fir_chain", "actors": [
        {"id": "src", "kind": "static", "behavior": "file_source", "params": {"path": "x"},
         "ports": [{"id": "out", "dir": "out"}]},
        {"id": "f", "kind": "static", "behavior": "fir_branch", "params": {"re": re, "im": im},
         "ports": [{"id": "in", "dir": "in"}, {"id": "out", "dir": "out"}]},
        {"id": "sink", "kind": "static", "behavior": "null_sink",
         "ports": [{"id": "in", "dir": "in"}]}],
        "fifos": [{"id": "a", "src": "src.out", "dst": "f.in", "token_bytes": 8 * block},
                  {"id": "b", "src": "f.out", "dst": "sink.in", "token_bytes": 8 * block}],
        "control": {}}


@pytest.mark.parametrize("block", [16, 256, 1000, 4096, 12288])
def test_fir_kernel_bitexact_static_chain(block):
    blocks = 9
    x = pd.stream_input(3, blocks, block)
    # adversarial values: signed zeros, tiny and large magnitudes
    x[0, 0, :8] = [0.0, -0.0, 1e-30, -1e-30, 3e4, -3e4, 1.0, -1.0]
    (rep,) = run_streams(fir_chain(block), 1, RuntimeConfig(source_firings=blocks, epoch=4,
                                                            capture_sinks=True),
                         sources={"src": [x.tobytes()]})
    cr, ci = od.branch_taps(2)
    hr = hi = np.zeros(9, np.float32)
    want = []
    for n in range(blocks):
        yr, yi, hr, hi = od.fir_block(x[n, 0], x[n, 1], cr, ci, hr, hi)
        want.append(np.stack([yr, yi]))
    assert rep.sink_data["sink"] == np.stack(want).tobytes()


TOLERANCE = 1e-5   # north star: max-abs/relative error <= 1e-5 for DPD


@pytest.mark.parametrize("fuse,B,K", [(True, 4096, 4), (False, 4096, 4), (True, 256, 4),
                                       (True, 1000, 10), (True, 16, 4)])
def test_tolerance_mode_within_1e5(fuse, B, K):
    """RuntimeConfig(exact=False): the fused bank runs PB_FIR_MERGED (one FMA
    FIR with the active branches' taps summed, per-branch history as a
    correction), per-actor launches PB_FIR_FMA.  Not bit-exact by design;
    every sample within 1e-5 of the exact reference (relative to
    max(1, |y|)) and control / firing counts still exact."""
    S, blocks = 3, 20
    xs = [pd.stream_input(s, blocks, B) for s in range(S)]
    desc = pd.build_description(B, K)
    reps = run_streams(desc, S,
                       RuntimeConfig(source_firings=blocks, exact=False, fuse=fuse,
                                     capture_sinks=True, epoch=7),
                       seeds=[1000 + s for s in range(S)],
                       sources={"src": [x.tobytes() for x in xs]})
    worst = 0.0
    for s in range(S):
        sets = od.subset_schedule(1000 + s, blocks, length=K)
        want = od.dpd_stream(xs[s], sets, K).astype(np.float64)
        got = np.frombuffer(reps[s].sink_data["sink"], np.float32).reshape(want.shape)
        err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
        worst = max(worst, float(err.max()))
        assert reps[s].firing_counts == od.firing_counts(sets, K)
    assert worst <= TOLERANCE, worst
    assert worst > 0.0   # genuinely the contracted arithmetic
