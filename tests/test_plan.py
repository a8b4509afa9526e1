"""Admission (plan.admit) on the reference's graphs: conditions, rejections."""
import json

from conftest import GOLDEN

import pytest

from paper_1802_06625_b200 import InconsistentGraph, UnsupportedGraph, admit, as_graph
from paper_1802_06625_b200.apps import predistortion as pd
from paper_1802_06625_b200.graph import DanglingPort, DuplicateId, RateMismatch


def test_dpd_conditions_and_bounds():
    p = admit(as_graph(pd.build_description()), c_factor=3)
    assert [c.element for c in p.conds] == [1, 2, 3, 4]
    assert {a: c for a, c in p.actor_cond.items() if c >= 0} == {"b1": 0, "b2": 1, "b3": 2,
                                                                 "b4": 3}
    assert p.fifo_cond["f_in3"] == p.fifo_cond["f_fir3"] == 2
    assert p.fifo_cond["f_src"] == p.fifo_cond["f_out"] == -1
    assert len(p.eq1_ports) == 8
    assert all(v == 3 for v in p.admission.beta.values())   # rate + (C-1)*rate


def test_rule2_skewed_control_rejected():
    # test_acceptance.py:195-203: a delay on c_split only
    desc = pd.build_description()
    for f in desc["fifos"]:
        if f["id"] == "c_split":
            f["delay"] = 1
    with pytest.raises(InconsistentGraph, match="rule 2"):
        admit(as_graph(desc))


def test_eq1_mismatch_rejected():
    desc = pd.build_description()
    # feed branch b2 from the d1 dynamic port: b2's consumer side is gated by
    # element 2, its producer side by element 1
    for f in desc["fifos"]:
        if f["id"] == "f_in2":
            f["src"] = "split.d1"
        if f["id"] == "f_in1":
            f["src"] = "split.d2"
    # the reference's rule 1 catches it (rules.py:162-175)
    with pytest.raises(InconsistentGraph, match="rule 1"):
        admit(as_graph(desc))


def test_data_delay_is_unsupported_not_wrong(golden):
    """Delay tokens are admitted on aligned, always-active channels (also
    from host producers); a delay that is not a multiple of the rate, or on a
    dynamically gated channel, raises UnsupportedGraph instead of running
    wrong."""
    desc = golden["fixtures"]["static_chain"]["description"]
    desc = json.loads(json.dumps(desc))
    desc["fifos"][0]["delay"] = 2          # source -> s1: a host producer
    p = admit(as_graph(desc))
    assert p.extra["s1"] == 2 and p.extra["src"] == 0
    desc = json.loads(json.dumps(golden["fixtures"]["rate_pair_atr3"]["description"]))
    for f in desc["fifos"]:
        if f["rate"] == 3 and f["src"] != "src.out" and not f["dst"].startswith("sink"):
            f["delay"] = 2                 # not a multiple of the rate
            break
    else:
        pytest.skip("no rate-3 device channel in the fixture")
    with pytest.raises(UnsupportedGraph, match="delay"):
        admit(as_graph(desc))
    desc = json.loads(json.dumps(golden["fixtures"]["gated_pipeline"]["description"]))
    for f in desc["fifos"]:
        if f["id"] == "f_m1":
            f["delay"] = 1                 # x.d1 -> m1: gated by the control token
    with pytest.raises((UnsupportedGraph, InconsistentGraph)):
        admit(as_graph(desc))


def test_device_delay_admitted(golden):
    desc = golden["motion"]["diamond_delay2"]["description"]
    p = admit(as_graph(desc))
    assert p.admission.beta["fb"] == 2 + 1 + (p.admission.c_factor - 1) * 1
    from paper_1802_06625_b200.apps import motion
    p = admit(as_graph(motion.build_description()))
    assert p.roles["blur"] == p.roles["detect"] == p.roles["clean"] == "device"


def test_delay_drain_phase_and_cycles(golden):
    """Firings after the sources stop (interp.py drain; test_interp.py:41-44)
    per actor, and the epoch cap a delayed cycle imposes."""
    desc = json.loads(json.dumps(golden["fixtures"]["static_chain"]["description"]))
    desc["fifos"][1]["delay"] = 2          # s1 -> s2, both device actors
    p = admit(as_graph(desc))
    assert p.extra == {"src": 0, "s1": 0, "s2": 2, "s3": 2, "sink": 2}
    assert p.epoch_cap is None
    d = json.loads((GOLDEN / "delays.json").read_text())
    for key, case in d.items():
        p = admit(as_graph(case["description"]))
        if key == "two_cycle":
            assert p.extra == {"a": None, "b": None} and p.epoch_cap == 1
            continue
        want = case["interpret"]["firing_counts"]
        n = case["source_firings"]
        always = {a for a, c in p.actor_cond.items() if c < 0}   # gated ones fire by control
        assert {a: n + e for a, e in p.extra.items() if a in always} == \
            {a: v for a, v in want.items() if a in always}, key
    p = admit(as_graph(d["fed_cycle_d4"]["description"]))
    assert p.epoch_cap == 2 and p.loose == {"f_ba"}
    assert p.order.index("a") < p.order.index("b")


def test_zero_delay_cycle_deadlocks():
    desc = {"name": "cyc", "actors": [
        {"id": "a", "kind": "static", "behavior": "passthrough",
         "ports": [{"id": "in", "dir": "in"}, {"id": "out", "dir": "out"}]},
        {"id": "b", "kind": "static", "behavior": "passthrough",
         "ports": [{"id": "in", "dir": "in"}, {"id": "out", "dir": "out"}]}],
        "fifos": [{"id": "ab", "src": "a.out", "dst": "b.in"},
                  {"id": "ba", "src": "b.out", "dst": "a.in"}], "control": {}}
    with pytest.raises(InconsistentGraph, match="Deadlock"):
        admit(as_graph(desc))


@pytest.mark.parametrize("key", ["static_chain", "broadcast_two_sinks", "clean_single_chain",
                                 "clean_two_component", "gated_pipeline", "rate_pair_atr3"])
def test_reference_fixtures_admitted(golden, key):
    admit(as_graph(golden["fixtures"][key]["description"]))


def test_structural_errors_match_reference_classes():
    desc = pd.build_description()
    bad = json.loads(json.dumps(desc))
    bad["actors"].append(bad["actors"][0])
    with pytest.raises(DuplicateId):
        as_graph(bad)
    bad = json.loads(json.dumps(desc))
    bad["fifos"][0]["dst"] = "split.nope"
    with pytest.raises(DanglingPort):
        as_graph(bad)
    bad = json.loads(json.dumps(desc))
    bad["fifos"][0]["rate"] = 2
    with pytest.raises(RateMismatch):
        as_graph(bad)


def test_reference_graph_object_converts(golden):
    import sys
    from pathlib import Path
    ref = Path("/root/repo/oracle/_ref")
    if not (ref / "tokenflow").is_dir():
        pytest.skip("reference not installed in oracle/_ref")
    sys.path.insert(0, str(ref))
    from tokenflow.model import build_graph
    desc = pd.build_description(4096, 10)
    g_ref = build_graph(desc)
    g = as_graph(g_ref)
    assert g.description() == as_graph(desc).description()


def test_mixed_graph_admitted():
    """BASELINE config 5: the DPD region and the adaptive CNN in one graph."""
    from paper_1802_06625_b200.apps import mixed
    p = admit(as_graph(mixed.build_description(256, 4, 2)))
    assert p.roles["dpd_conf"] == p.roles["cnn_conf"] == "config"
    assert {p.roles[a] for a in ("cnn_l1", "cnn_l2", "cnn_l3", "dpd_b1")} == {"device"}
    assert len(p.conds) == 6     # 4 DPD branches + CNN process / bypass


def test_matmul_chain_found_in_bypass_app():
    """plan.find_matmul_chains: the bypass app's l1 -> l2 -> l3 (link channels
    f_l2, f_l3); a second consumer of l2's output ends the chain at l2."""
    from paper_1802_06625_b200.apps import bypass
    from paper_1802_06625_b200.behaviors import resolve
    from paper_1802_06625_b200.plan import find_matmul_chains

    def chains(desc):
        p = admit(as_graph(desc))
        behaviors = {}
        for a in desc["actors"]:
            b = resolve(a["behavior"])
            if a["behavior"] != "file_source":
                b.init(a["id"], a.get("params", {}), None)
            behaviors[a["id"]] = b
        return [(c.actors, sorted(c.internal_fifos)) for c in find_matmul_chains(p, behaviors)]
    desc = bypass.build_description("x.bin")
    assert chains(desc) == [(["l1", "l2", "l3"], ["f_l2", "f_l3"])]
    # a static chain src -> m1 -> m2 -> m3 -> sink; a second consumer of m2's
    # output ends the chain at m2
    from paper_1802_06625_b200.apps.bypass import layer_weights

    def port(pid, d):
        return {"id": pid, "dir": d, "kind": "srp", "rate": 1}
    acts = [{"id": "src", "kind": "static", "behavior": "file_source", "params": {"path": "x"},
             "ports": [port("out", "out")]},
            {"id": "sink", "kind": "static", "behavior": "null_sink", "ports": [port("in", "in")]}]
    acts += [{"id": f"m{k}", "kind": "static", "behavior": "matmul",
              "params": {"w": layer_weights(k)}, "ports": [port("in", "in"), port("out", "out")]}
             for k in (1, 2, 3)]

    def ff(fid, src, dst):
        return {"id": fid, "src": src, "dst": dst, "rate": 1, "delay": 0, "token_bytes": 256}
    fifos = [ff("a", "src.out", "m1.in"), ff("b", "m1.out", "m2.in"), ff("c", "m2.out", "m3.in"),
             ff("d", "m3.out", "sink.in")]
    lin = {"name": "lin", "actors": acts, "fifos": fifos, "control": {}}
    assert chains(lin) == [(["m1", "m2", "m3"], ["b", "c"])]
    tap = {"id": "tap", "kind": "static", "behavior": "null_sink", "ports": [port("in", "in")]}
    lin2 = dict(lin, actors=acts + [tap], fifos=fifos + [ff("t", "m2.out", "tap.in")])
    assert chains(lin2) == [(["m1", "m2"], ["b"])]


def test_motion_region_found():
    """plan.find_motion_regions: the motion app's blur -> detect -> clean with
    f_cur / f_mask internal and f_prev kept; a delay of 2 on f_prev does not
    match."""
    from paper_1802_06625_b200.apps import motion
    from paper_1802_06625_b200.behaviors import resolve
    from paper_1802_06625_b200.plan import find_motion_regions

    def regions(desc):
        p = admit(as_graph(desc))
        behaviors = {}
        for a in desc["actors"]:
            b = resolve(a["behavior"])
            if a["behavior"] != "file_source":
                b.init(a["id"], a.get("params", {}), None)
            behaviors[a["id"]] = b
        return [(m.blur, m.detect, m.clean, m.cur_fifo, m.prev_fifo, m.mask_fifo, m.side)
                for m in find_motion_regions(p, behaviors)]
    desc = motion.build_description()
    assert regions(desc) == [("blur", "detect", "clean", "f_cur", "f_prev", "f_mask", 64)]
    d2 = dict(desc, fifos=[dict(f, delay=2) if f["id"] == "f_prev" else f
                           for f in desc["fifos"]])
    assert regions(d2) == []
    assert regions(motion.build_description(12)) == []    # not a power-of-two side


def test_bypass_region_found():
    """plan.find_bypass_regions: the bypass app's fork -> l1..l3 -> join with
    the f_bypass edge; the chain's output channel f_chain is internal."""
    from paper_1802_06625_b200.apps import bypass
    from paper_1802_06625_b200.behaviors import resolve
    from paper_1802_06625_b200.plan import find_bypass_regions, find_matmul_chains
    desc = bypass.build_description("x.bin")
    p = admit(as_graph(desc))
    behaviors = {}
    for a in desc["actors"]:
        b = resolve(a["behavior"])
        if a["behavior"] != "file_source":
            b.init(a["id"], a.get("params", {}), None)
        behaviors[a["id"]] = b
    regions = find_bypass_regions(p, behaviors, find_matmul_chains(p, behaviors))
    assert [(r.route, r.merge, r.chain.actors, r.chain_out, r.bypass_fifo, r.out_fifo)
            for r in regions] == [("fork", "join", ["l1", "l2", "l3"], "f_chain", "f_bypass",
                                   "f_out")]
