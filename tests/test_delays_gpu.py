"""Initial delay tokens, the drain phase and delayed cycles on the device,
against the reference engines (tests/golden/delays.json, made by
tests/golden/make_delays.py from interp.interpret and runtime.run):
consumers fire on the delay tokens after the sources stop
(test_interp.py:41-60), delay payloads reach the sinks
(test_runtime.py:57-64), delays on source, middle and sink channels and on
broadcasts, feedback loops through delayed self loops and cycles fed by a
source (epochs capped at the cycle's delay), and a sourceless cycle that
spins until the timeout (test_runtime.py:224-235)."""
import json

import pytest

from conftest import GOLDEN
from paper_1802_06625_b200 import (RuntimeConfig, Timeout, UnsupportedGraph, instantiate, run,
                                   run_streams)
from paper_1802_06625_b200.behaviors import ActorBehavior

pytestmark = pytest.mark.gpu

CASES = json.loads((GOLDEN / "delays.json").read_text())
RUNNABLE = sorted(k for k in CASES if k != "two_cycle")


def description(case, tmp_path):
    """The case's graph; a file source reads the recorded input from tmp_path."""
    desc = json.loads(json.dumps(case["description"]))
    if "input_hex" in case:
        p = tmp_path / "input.bin"
        p.write_bytes(bytes.fromhex(case["input_hex"]))
        for a in desc["actors"]:
            if a.get("behavior") == "file_source":
                a["params"]["path"] = str(p)
    return desc


@pytest.mark.parametrize("epoch", [4096, 1, 3])
@pytest.mark.parametrize("key", RUNNABLE)
def test_delay_graph_matches_reference(key, epoch, tmp_path):
    case = CASES[key]
    want = case["interpret"]
    rep = run(description(case, tmp_path), config=RuntimeConfig(
        source_firings=case["source_firings"], seed=case["seed"], capture_sinks=True,
        epoch=epoch))
    assert rep.firing_counts == want["firing_counts"]
    assert rep.sink_digests == want["sink_digests"]
    for sink, hexdata in want["sink_data_hex"].items():
        assert rep.sink_data[sink].hex() == hexdata, sink
    assert rep.slots == case["run"]["slots"] and rep.beta == case["run"]["beta"]
    for fid, occ in rep.max_occupancy.items():
        assert occ <= rep.beta[fid] and occ <= rep.slots[fid], fid
        assert rep.device_max_occupancy[fid] <= rep.device_slots[fid], fid


@pytest.mark.parametrize("exact", [True, False])
def test_dpd_with_delayed_branch_channel(exact, tmp_path):
    """A delay on a gated branch channel of the DPD app keeps that region out
    of the fused bank (its channel is materialised); bit-exact in the exact
    mode, within 1e-5 in the tolerance mode."""
    import numpy as np
    case = CASES["dpd_branch_delay"]
    rep = run(description(case, tmp_path), config=RuntimeConfig(
        source_firings=case["source_firings"], seed=case["seed"], capture_sinks=True,
        exact=exact))
    assert rep.firing_counts == case["interpret"]["firing_counts"]
    want = np.frombuffer(bytes.fromhex(case["interpret"]["sink_data_hex"]["sink"]), np.float32)
    got = np.frombuffer(rep.sink_data["sink"], np.float32)
    if exact:
        assert rep.sink_digests == case["interpret"]["sink_digests"]
    else:
        assert (np.abs(got - want) / np.maximum(1.0, np.abs(want))).max() <= 1e-5


@pytest.mark.parametrize("key", ["chain_all_d", "feedback_d2_payload", "fed_cycle", "bcast_delay",
                                 "gated_e2_d2_payload", "rate_pair_b_d2"])
def test_delay_graph_streams(key):
    case = CASES[key]
    S = 5
    reps = run_streams(case["description"], S, RuntimeConfig(
        source_firings=case["source_firings"], capture_sinks=True),
        seeds=[case["seed"]] * S)
    for r in reps:
        assert r.firing_counts == case["interpret"]["firing_counts"]
        assert r.sink_digests == case["interpret"]["sink_digests"]


class PyPass(ActorBehavior):
    """passthrough / add_mod (behavior.py:158-173) as a host behaviour."""

    def fire(self, ctx):
        off = int(ctx.params.get("offset", 0))
        live = [v for v in ctx.inputs.values() if len(v)]
        for span in ctx.outputs.values():
            for i in range(len(span)):
                span[i] = (sum(v[i] for v in live) + off) & 0xFF


@pytest.mark.parametrize("key,actors", [("chain_all_d", ["s2"]), ("feedback_d1", ["j"]),
                                        ("fed_cycle", ["b"]), ("bcast_delay", ["s2"])])
def test_host_actors_drain_and_cycle(key, actors):
    case = CASES[key]
    rep = run(case["description"], behaviors={a: PyPass() for a in actors},
              config=RuntimeConfig(source_firings=case["source_firings"], seed=case["seed"],
                                   capture_sinks=True))
    assert rep.firing_counts == case["interpret"]["firing_counts"]
    assert rep.sink_digests == case["interpret"]["sink_digests"]


def test_sourceless_cycle_spins_until_timeout():
    case = CASES["two_cycle"]
    rt = instantiate(case["description"], config=RuntimeConfig(timeout_ms=case["timeout_ms"]))
    try:
        with pytest.raises(Timeout) as exc:
            rt.run()
        assert sorted(exc.value.alive) == case["raises"]["alive"]
        beta = rt.analysis.bounds.beta
        for fid, chan in rt.channels.items():
            assert chan.max_occupancy <= min(beta[fid], chan.plan.slots), fid
        assert rt.firings["a"][0] > 1 and rt.firings["a"][0] == rt.firings["b"][0]
    finally:
        rt.close()
    with pytest.raises(UnsupportedGraph, match="timeout_ms"):
        instantiate(case["description"])
