"""Golden runs of graphs with initial delay tokens, from the REFERENCE engines.

Run here (the build container) only -- it imports /root/reference/pkg:

    python tests/golden/make_delays.py

Writes tests/golden/delays.json: for each graph its description, the number
of source firings, and what the reference interpreter (interp.py:89-229) and
the threaded runtime (runtime.py:345-347) report: sink digests and bytes,
firing counts (including the drain phase: consumers fire on delay tokens
after the sources stop, test_interp.py:41-44), slots and beta; for the
sourceless cycle, the exception the threaded runtime raises at its timeout
(test_runtime.py:224-235).

Cases: the delay layouts the reference tests use (static_chain with delays on
the source's, a middle and the sink's channel, payloads; test_interp.py,
test_runtime.py:57-64), broadcasts to a delayed and an undelayed channel, a
feedback loop through a delayed self loop, a two-actor cycle fed by a source,
rate-2 channels with delays, and two_cycle (fixtures.py:363) without a source.
"""
from __future__ import annotations

import copy
import json
import os
import sys
from pathlib import Path

REF = Path(os.environ.get("PRUNE_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import fixtures as fx  # noqa: E402  (reference test fixtures)
from tokenflow.interp import interpret  # noqa: E402
from tokenflow.model import build_graph  # noqa: E402
from tokenflow.runtime import RuntimeConfig, run  # noqa: E402

OUT = Path(__file__).resolve().parent


def port(pid, d, kind="srp", rate=1):
    return {"id": pid, "dir": d, "kind": kind, "rate": rate}


def chain(stages, delays, payloads=None, rate=1, token_bytes=1):
    desc = fx.static_chain(stages, rate=rate, token_bytes=token_bytes, delays=delays)
    for k, hexdata in (payloads or {}).items():
        desc["fifos"][k]["delay_payload_hex"] = hexdata
    return desc


def feedback(delay=1, payload=None):
    """src -> j (add_mod of the input and its own previous output) -> sink,
    the loop closed by a delayed self loop j.loop_out -> j.loop_in."""
    loop = {"id": "f_loop", "src": "j.loop_out", "dst": "j.loop_in", "rate": 1,
            "delay": delay, "token_bytes": 1}
    if payload:
        loop["delay_payload_hex"] = payload
    return {"name": "feedback", "control": {},
            "actors": [
                {"id": "src", "kind": "static", "behavior": "counter_source",
                 "ports": [port("out", "out")], "params": {}},
                {"id": "j", "kind": "static", "behavior": "add_mod", "params": {"offset": 3},
                 "ports": [port("i1", "in"), port("loop_in", "in"), port("out", "out"),
                           port("loop_out", "out")]},
                {"id": "sink", "kind": "static", "behavior": "null_sink",
                 "ports": [port("in", "in")], "params": {}}],
            "fifos": [{"id": "f_in", "src": "src.out", "dst": "j.i1", "rate": 1, "delay": 0,
                       "token_bytes": 1},
                      loop,
                      {"id": "f_out", "src": "j.out", "dst": "sink.in", "rate": 1, "delay": 0,
                       "token_bytes": 1}]}


def fed_cycle(delay=2, rate=2):
    """a and b feeding each other (the back edge holds the delay) plus a
    source into a and a sink off b."""
    return {"name": "fed_cycle", "control": {},
            "actors": [
                {"id": "src", "kind": "static", "behavior": "counter_source",
                 "ports": [port("out", "out", rate=rate)], "params": {}},
                {"id": "a", "kind": "static", "behavior": "add_mod", "params": {"offset": 1},
                 "ports": [port("i1", "in", rate=rate), port("back", "in", rate=rate),
                           port("out", "out", rate=rate)]},
                {"id": "b", "kind": "static", "behavior": "passthrough", "params": {},
                 "ports": [port("in", "in", rate=rate), port("out", "out", rate=rate),
                           port("tap", "out", rate=rate)]},
                {"id": "sink", "kind": "static", "behavior": "null_sink",
                 "ports": [port("in", "in", rate=rate)], "params": {}}],
            "fifos": [{"id": "f_src", "src": "src.out", "dst": "a.i1", "rate": rate, "delay": 0,
                       "token_bytes": 1},
                      {"id": "f_ab", "src": "a.out", "dst": "b.in", "rate": rate, "delay": 0,
                       "token_bytes": 1},
                      {"id": "f_ba", "src": "b.out", "dst": "a.back", "rate": rate,
                       "delay": delay, "token_bytes": 1},
                      {"id": "f_out", "src": "b.tap", "dst": "sink.in", "rate": rate,
                       "delay": 0, "token_bytes": 1}]}


def broadcast_delayed():
    """src broadcasts to s1 (no delay) and s2 (delay 2); both to sinks."""
    return {"name": "bcast_delay", "control": {},
            "actors": [
                {"id": "src", "kind": "static", "behavior": "counter_source",
                 "ports": [port("out", "out")], "params": {}},
                {"id": "s1", "kind": "static", "behavior": "passthrough", "params": {},
                 "ports": [port("in", "in"), port("out", "out")]},
                {"id": "s2", "kind": "static", "behavior": "add_mod", "params": {"offset": 7},
                 "ports": [port("in", "in"), port("out", "out")]},
                {"id": "k1", "kind": "static", "behavior": "null_sink", "params": {},
                 "ports": [port("in", "in")]},
                {"id": "k2", "kind": "static", "behavior": "null_sink", "params": {},
                 "ports": [port("in", "in")]}],
            "fifos": [{"id": "a", "src": "src.out", "dst": "s1.in", "rate": 1, "delay": 0,
                       "token_bytes": 2},
                      {"id": "b", "src": "src.out", "dst": "s2.in", "rate": 1, "delay": 2,
                       "token_bytes": 2, "delay_payload_hex": "aabbccdd"},
                      {"id": "c", "src": "s1.out", "dst": "k1.in", "rate": 1, "delay": 0,
                       "token_bytes": 2},
                      {"id": "d", "src": "s2.out", "dst": "k2.in", "rate": 1, "delay": 1,
                       "token_bytes": 2}]}


def gated(fid: str, delay: int, payload: str | None = None, builder=None):
    """A reference fixture with initial tokens on one channel (gated or not)."""
    desc = (builder or fx.gated_pipeline)()
    for f in desc["fifos"]:
        if f["id"] == fid:
            f["delay"] = delay
            if payload:
                f["delay_payload_hex"] = payload
    return desc


def dpd_branch_delay(path: str):
    """The reference DPD app (B=256, K=4) with one initial token on the
    branch-2 -> combiner channel (a dynamically gated channel)."""
    from tokenflow.apps import predistortion as rpd
    desc = rpd.build_description(path)
    for f in desc["fifos"]:
        if f["id"] == "f_fir2":
            f["delay"] = 1
            # one 256-sample token of ordinary floats (a NaN payload would
            # compare by its NaN bits, which differ between IEEE implementations)
            import numpy as np
            f["delay_payload_hex"] = np.linspace(-0.75, 0.5, 512, dtype=np.float32).tobytes().hex()
    return desc


def cases() -> dict[str, tuple[dict, int]]:
    return {
        "gated_e1_d1": (gated("f_e1", 1), 6),
        "gated_e2_d2_payload": (gated("f_e2", 2, "0a0b"), 9),
        "gated_src_d1": (gated("f_src", 1), 6),
        "gated_out_d1": (gated("f_out", 1), 6),
        "rate_pair_b_d2": (gated("f_b", 2, None, lambda: fx.rate_pair(2)), 5),
        "chain_mid_d1": (chain(2, {1: 1}), 6),              # test_interp.py:41-44
        "chain_mid_d2": (chain(2, {1: 2}), 4),              # test_interp.py:56-60
        "chain3_mid_d2": (chain(3, {1: 2}), 20),            # test_interp.py:140
        "chain_src_payload": (chain(1, {0: 2}, {0: "0102"}), 4),   # test_runtime.py:57-64
        "chain_sink_d1": (chain(2, {2: 1}), 5),
        "chain_all_d": (chain(3, {0: 1, 1: 2, 2: 1, 3: 3}, {3: "0a0b0c"}), 9),
        "chain_rate2_d4": (chain(2, {1: 4}, rate=2, token_bytes=3), 7),
        "feedback_d1": (feedback(1), 8),
        "feedback_d2_payload": (feedback(2, "1122"), 9),
        "fed_cycle": (fed_cycle(2, 2), 6),
        "fed_cycle_d4": (fed_cycle(4, 2), 5),
        "bcast_delay": (broadcast_delayed(), 5),
    }


def main():
    out = {}
    import tempfile
    from tokenflow.apps import predistortion as rpd
    td = tempfile.mkdtemp()
    inp = Path(td) / "dpd.bin"
    inp.write_bytes(rpd.make_input(11, 12))
    all_cases = dict(cases())
    all_cases["dpd_branch_delay"] = (dpd_branch_delay(str(inp)), 12)
    for name, (desc, n) in all_cases.items():
        g = build_graph(copy.deepcopy(desc))
        rec = {"description": desc, "source_firings": n, "seed": 5}
        if name == "dpd_branch_delay":
            rec["input_hex"] = inp.read_bytes().hex()
        ref = interpret(g, source_firings=n, seed=5, capture_sinks=True)
        rec["interpret"] = {"sink_digests": ref.sink_digests,
                            "sink_data_hex": {k: v.hex() for k, v in ref.sink_data.items()},
                            "firing_counts": ref.firing_counts}
        rep = run(build_graph(copy.deepcopy(desc)),
                  config=RuntimeConfig(source_firings=n, seed=5, capture_sinks=True,
                                       timeout_ms=5000))
        assert rep.sink_digests == ref.sink_digests, name
        assert rep.firing_counts == ref.firing_counts, name
        rec["run"] = {"slots": rep.slots, "beta": rep.beta, "max_occupancy": rep.max_occupancy}
        out[name] = rec
    # sourceless cycle: spins until the timeout (test_runtime.py:224-235)
    from tokenflow.runtime import Timeout
    desc = fx.two_cycle(delay=2, rate=2)
    try:
        run(build_graph(copy.deepcopy(desc)), config=RuntimeConfig(timeout_ms=250))
        raised = None
    except Timeout as e:
        raised = {"type": "Timeout", "alive": sorted(e.alive)}
    out["two_cycle"] = {"description": desc, "timeout_ms": 250, "raises": raised}
    (OUT / "delays.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print(f"wrote {len(out)} cases to {OUT / 'delays.json'}")


if __name__ == "__main__":
    main()
