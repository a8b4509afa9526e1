"""Golden admission verdicts from the REFERENCE analysis (tokenflow.analyze).

Run here (the build container) only -- it imports /root/reference/pkg:

    python tests/golden/make_admission.py

Writes tests/golden/admission.json: for every graph of the corpus, its
description and what `tokenflow.analysis.analyze(build_graph(desc), c)`
returns for c in (2, 3, 5): verdict, violations (rule, subjects),
diagnostics (code, subjects), DPGs (q, x, y, members, components) and the
buffer bounds beta; or the exception type when analyze itself raises.  For
consistent graphs with a source it also records the reference RunReport's
slots and beta (runtime.py:268-269, :323) at c_factor 3.

Corpus:
  * every builder of pkg/tests/fixtures.py (and the parameterised variants
    the reference tests use), the inline layouts of test_rules.py and
    test_analysis.py, and the shipped apps;
  * 600 seeded random descriptions: dynamic pairs joined by static
    subchains with random perturbations (extra feeders, shared members,
    mismatched elements, control delays, double-sided actors, cycles,
    orphans), plus fully random wirings.
"""
from __future__ import annotations

import copy
import json
import os
import random
import sys
from pathlib import Path

REF = Path(os.environ.get("PRUNE_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import fixtures as fx  # noqa: E402  (reference test fixtures)
from tokenflow.analysis import analyze  # noqa: E402
from tokenflow.model import GraphError, build_graph  # noqa: E402

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parent.parent))


def port(pid, d, kind="srp", rate=1):
    return {"id": pid, "dir": d, "kind": kind, "rate": rate}


def named_cases() -> dict[str, dict]:
    cases = {}
    for name in ("static_chain", "broadcast_two_sinks", "clean_single_chain",
                 "clean_two_component", "shared_member_violation", "double_sided_violation",
                 "unencapsulated_violation", "encapsulated_pass", "three_component_split",
                 "diamond_component", "mismatched_elements", "unbalanced_control_delay",
                 "orphan_dynamic", "shared_config", "uncontrolled_port", "two_cycle",
                 "rate_pair", "gated_pipeline", "stranded_tokens"):
        cases[name] = getattr(fx, name)()
    cases["two_cycle_delay0"] = fx.two_cycle(delay=0)
    cases["two_cycle_delay1_rate2"] = fx.two_cycle(delay=1, rate=2)
    cases["static_chain_delays"] = fx.static_chain(stages=2, delays={1: 2})
    cases["static_chain_stages2_token_bytes5"] = fx.static_chain(stages=2, token_bytes=5)
    cases["rate_pair_atr3"] = fx.rate_pair(atr=3)
    # test_rules.py:111-129 -- a dynamic subchain member
    desc = fx.clean_single_chain()
    for a in desc["actors"]:
        if a["id"] == "m1":
            a["kind"] = "dynamic"
            a["ports"] = ([fx.port("ctl", "in", "control_in")] + a["ports"]
                          + [fx.port("d9", "out", "drp")])
        if a["id"] == "y":
            a["ports"].insert(-1, fx.port("e2", "in", "drp"))
    desc["fifos"] += [fx.fifo("c_m", "q.c", "m1.ctl"), fx.fifo("f_d9", "m1.d9", "y.e2")]
    desc["control"]["table"] += [{"port": "q.c", "drp": "m1.d9", "element": 1},
                                 {"port": "q.c", "drp": "y.e2", "element": 1}]
    cases["dynamic_subchain_member"] = desc
    # test_rules.py:148-155 -- several violations sorted
    desc = fx.mismatched_elements()
    for f in desc["fifos"]:
        if f["id"] == "c_x":
            f["delay"] = 1
    cases["mismatched_and_unbalanced"] = desc
    # test_analysis.py:136-146 -- a component spanning two control elements
    desc = fx.clean_two_component()
    desc["control"]["table"] = [r if r["drp"] != "y.e2" else dict(r, element=1)
                                for r in desc["control"]["table"]]
    cases["component_two_elements"] = desc
    # test_analysis.py:148-169 -- one port fanning into two components
    actors, fifos, ctl = fx._pair_scaffold(
        [fx.port("d1", "out", "drp")],
        [fx.port("e1", "in", "drp"), fx.port("e2", "in", "drp")],
        [("q.c", "x.d1", 1), ("q.c", "y.e1", 1), ("q.c", "y.e2", 1)], length=1)
    for k in (1, 2):
        actors.append(fx.actor(f"m{k}", "static", [fx.port("in", "in"), fx.port("out", "out")],
                               "passthrough"))
        fifos += [fx.fifo(f"f_m{k}", "x.d1", f"m{k}.in"),
                  fx.fifo(f"f_e{k}", f"m{k}.out", f"y.e{k}")]
    cases["port_fans_two_components"] = {"name": "fan", "actors": actors, "fifos": fifos,
                                         "control": ctl}
    # test_analysis.py:171-189 -- declared length / element bijection
    desc = fx.three_component_split()
    desc["control"]["value_lengths"] = {"q.c": 4}
    for f in desc["fifos"]:
        if f["id"] in ("c_x", "c_y"):
            f["token_bytes"] = 4
    cases["declared_length_mismatch"] = desc
    desc = fx.three_component_split()
    desc["control"]["table"] = [r if r["drp"] not in ("x.d4", "y.e3") else dict(r, element=2)
                                for r in desc["control"]["table"]]
    cases["elements_not_distinct"] = desc
    # the shipped apps
    from tokenflow.apps import bypass, motion, predistortion
    cases["app_predistortion"] = predistortion.build_description("/nonexistent.bin")
    cases["app_bypass"] = bypass.build_description("/nonexistent.bin")
    cases["app_motion"] = motion.build_description("/nonexistent.bin")
    from paper_1802_06625_b200.apps import mixed, vision
    from paper_1802_06625_b200.apps import predistortion as mypd
    cases["app_dpd_k10"] = mypd.build_description(512, 10)
    cases["app_vision"] = vision.build_description(24)
    cases["app_mixed"] = mixed.build_description()
    return cases


# ------------------------------------------------------------ random corpus

class Builder:
    def __init__(self, rng: random.Random):
        self.rng = rng
        self.actors: dict[str, dict] = {}
        self.fifos: list[dict] = []
        self.lengths: dict[str, int] = {}
        self.table: list[dict] = []
        self.nport: dict[str, int] = {}

    def actor(self, aid, kind, behavior=""):
        self.actors[aid] = {"id": aid, "kind": kind, "behavior": behavior, "params": {},
                            "ports": []}
        self.nport[aid] = 0
        return aid

    def new_port(self, aid, d, kind="srp", rate=1):
        self.nport[aid] += 1
        pid = f"{'i' if d == 'in' else 'o'}{self.nport[aid]}"
        if kind == "drp":
            pid = ("e" if d == "in" else "d") + pid[1:]
        self.actors[aid]["ports"].append(port(pid, d, kind, rate))
        return pid

    def edge(self, src, dst, skind="srp", dkind="srp", rate=None, delay=0, reuse=None):
        rate = rate or self.rng.choice((1, 1, 1, 2))
        if reuse is not None:
            sp = reuse
            rate = next(p["rate"] for p in self.actors[src]["ports"] if p["id"] == sp)
        else:
            sp = self.new_port(src, "out", skind, rate)
        dp = self.new_port(dst, "in", dkind, rate)
        self.fifos.append({"id": f"f{len(self.fifos)}", "src": f"{src}.{sp}", "dst": f"{dst}.{dp}",
                           "rate": rate, "delay": delay, "token_bytes": 1})
        return sp, dp

    def control(self, q, dyn, length, delay=0):
        cp = f"c{len(self.lengths)}"
        if cp not in [p["id"] for p in self.actors[q]["ports"]]:
            self.actors[q]["ports"].append(port(cp, "out", "control_out"))
        self.lengths[f"{q}.{cp}"] = length
        for a in dyn:
            self.actors[a]["ports"].insert(0, port("ctl", "in", "control_in"))
            self.fifos.append({"id": f"c_{a}", "src": f"{q}.{cp}", "dst": f"{a}.ctl", "rate": 1,
                               "delay": delay if self.rng.random() < 0.15 else 0,
                               "token_bytes": length})
        return f"{q}.{cp}"

    def desc(self, name):
        return {"name": name, "actors": list(self.actors.values()), "fifos": self.fifos,
                "control": {"value_lengths": self.lengths, "table": self.table}}


def structured(rng: random.Random, idx: int) -> dict:
    b = Builder(rng)
    n_pairs = rng.choice((1, 1, 2))
    for k in range(n_pairs):
        q = b.actor(f"q{k}", "config", "fixed_policy")
        src = b.actor(f"src{k}", "static", "counter_source")
        x = b.actor(f"x{k}", "dynamic", "route")
        y = b.actor(f"y{k}", "dynamic", "merge")
        snk = b.actor(f"sink{k}", "static", "null_sink")
        b.edge(src, x)
        b.edge(y, snk)
        n_dc = rng.randint(1, 3)
        length = n_dc if rng.random() < 0.8 else rng.randint(1, 4)
        ctl = b.control(q, [x, y], length)
        for c in range(n_dc):
            el = c + 1 if rng.random() < 0.85 else rng.randint(1, max(1, length))
            el = min(el, length)
            kind = rng.random()
            if kind < 0.2:       # direct link
                sp, dp = b.edge(x, y, "drp", "drp")
                b.table += [{"port": ctl, "drp": f"{x}.{sp}", "element": el},
                            {"port": ctl, "drp": f"{y}.{dp}",
                             "element": el if rng.random() < 0.9 else rng.randint(1, length)}]
                continue
            chain = [b.actor(f"m{k}_{c}_{j}", "static", "passthrough")
                     for j in range(rng.randint(1, 3))]
            sp, _ = b.edge(x, chain[0], "drp")
            b.table.append({"port": ctl, "drp": f"{x}.{sp}", "element": el})
            for u, v in zip(chain, chain[1:]):
                b.edge(u, v)
            if rng.random() < 0.25 and len(chain) > 1:     # a parallel branch (diamond)
                par = b.actor(f"p{k}_{c}", "static", "passthrough")
                b.edge(chain[0], par)
                b.edge(par, chain[-1])
            _, dp = b.edge(chain[-1], y, "srp", "drp")
            b.table.append({"port": ctl, "drp": f"{y}.{dp}",
                            "element": el if rng.random() < 0.9 else rng.randint(1, length)})
    # perturbations
    statics = [a for a, d in b.actors.items() if d["kind"] == "static" and
               not a.startswith(("src", "sink"))]
    for _ in range(rng.choice((0, 0, 1, 1, 2, 3))):
        r = rng.random()
        if r < 0.2 and statics:              # outside feeder into a subchain member
            f = b.actor(f"feed{len(b.actors)}", "static", "counter_source")
            b.edge(f, rng.choice(statics))
            if rng.random() < 0.5:           # ... that also feeds a dynamic actor's SRP
                ys = [a for a, d in b.actors.items() if d["kind"] == "dynamic"]
                b.edge(f, rng.choice(ys))
        elif r < 0.35 and len(statics) > 1:  # extra edge between statics (maybe a cycle)
            u, v = rng.sample(statics, 2)
            b.edge(u, v, delay=rng.choice((0, 0, 1, 2)))
        elif r < 0.5 and statics:            # subchain member also feeds another pair's y
            ys = [a for a in b.actors if a.startswith("y")]
            yy = rng.choice(ys)
            u = rng.choice(statics)
            ctls = [fi["src"] for fi in b.fifos if fi["dst"] == f"{yy}.ctl"]
            _, dp = b.edge(u, yy, "srp", "drp")
            b.table.append({"port": ctls[0], "drp": f"{yy}.{dp}", "element": 1})
        elif r < 0.6:                        # orphan dynamic actor
            qs = [a for a, d in b.actors.items() if d["kind"] == "config"]
            o = b.actor(f"o{len(b.actors)}", "dynamic", "route")
            s2 = b.actor(f"s{len(b.actors)}", "static", "counter_source")
            k2 = b.actor(f"k{len(b.actors)}", "static", "null_sink")
            b.edge(s2, o)
            sp, _ = b.edge(o, k2, "drp")
            q = rng.choice(qs)
            cp = next(p["id"] for p in b.actors[q]["ports"] if p["kind"] == "control_out")
            b.actors[o]["ports"].insert(0, port("ctl", "in", "control_in"))
            b.fifos.append({"id": f"c_{o}", "src": f"{q}.{cp}", "dst": f"{o}.ctl", "rate": 1,
                            "delay": 0, "token_bytes": b.lengths[f"{q}.{cp}"]})
            b.table.append({"port": f"{q}.{cp}", "drp": f"{o}.{sp}", "element": 1})
        elif r < 0.7:                        # double-sided dynamic actor
            xs = [a for a in b.actors if a.startswith("x")]
            xx = rng.choice(xs)
            ctls = [fi["src"] for fi in b.fifos if fi["dst"] == f"{xx}.ctl"]
            f = b.actor(f"feed{len(b.actors)}", "static", "counter_source")
            _, dp = b.edge(f, xx, "srp", "drp")
            b.table.append({"port": ctls[0], "drp": f"{xx}.{dp}", "element": 1})
        elif r < 0.8 and statics:            # a static actor feeding back into x (cycle)
            xs = [a for a in b.actors if a.startswith("x")]
            b.edge(rng.choice(statics), rng.choice(xs), delay=rng.choice((0, 1)))
        elif r < 0.9 and len([a for a in b.actors if a.startswith("q")]) > 1:
            # one configuration actor drives the other pair too (shared config)
            pass
        elif statics:                        # member fans out to an extra sink
            k2 = b.actor(f"k{len(b.actors)}", "static", "null_sink")
            b.edge(rng.choice(statics), k2)
    if rng.random() < 0.05 and b.table:     # an uncontrolled port
        b.table.pop(rng.randrange(len(b.table)))
    return b.desc(f"structured{idx}")


def wild(rng: random.Random, idx: int) -> dict:
    """Random wirings of static, dynamic and configuration actors."""
    b = Builder(rng)
    n = rng.randint(3, 9)
    ids = [b.actor(f"a{k}", rng.choice(("static", "static", "dynamic"))) for k in range(n)]
    q = b.actor("q", "config", "fixed_policy")
    dyn = [a for a in ids if b.actors[a]["kind"] == "dynamic"]
    for _ in range(rng.randint(n - 1, 2 * n)):
        u, v = rng.sample(ids, 2)
        sk = "drp" if u in dyn and rng.random() < 0.6 else "srp"
        dk = "drp" if v in dyn and rng.random() < 0.6 else "srp"
        b.edge(u, v, sk, dk, delay=rng.choice((0, 0, 0, 1, 2)))
    for a in ids:
        if not b.actors[a]["ports"]:
            b.edge(a, rng.choice([x for x in ids if x != a]))
    length = rng.randint(1, 3)
    if dyn:
        ctl = b.control(q, dyn, length)
        for a in dyn:
            for p in b.actors[a]["ports"]:
                if p["kind"] == "drp":
                    b.table.append({"port": ctl, "drp": f"{a}.{p['id']}",
                                    "element": rng.randint(1, length)})
    else:
        del b.actors[q]
    # dynamic actors need at least one DRP
    for a in dyn:
        if not any(p["kind"] == "drp" for p in b.actors[a]["ports"]):
            return None
    return b.desc(f"wild{idx}")


def record(desc: dict) -> dict | None:
    try:
        g = build_graph(copy.deepcopy(desc))
    except GraphError:
        return None
    out = {"description": desc, "analysis": {}}
    for c in (2, 3, 5):
        try:
            r = analyze(g, c_factor=c)
        except Exception as e:  # noqa: BLE001
            out["analysis"][str(c)] = {"raises": type(e).__name__}
            continue
        out["analysis"][str(c)] = {
            "verdict": r.verdict,
            "violations": [[v.rule, list(v.subjects)] for v in r.violations],
            "diagnostics": [[d.code, list(d.subjects)] for d in r.diagnostics],
            "dpgs": [{"q": d.q, "x": d.x, "y": d.y, "members": list(d.members),
                      "dcs": [[list(dc.members), [str(p) for p in dc.in_drps],
                               [str(p) for p in dc.out_drps], list(dc.elements)]
                              for dc in d.dcs]} for d in r.dpgs],
            "beta": dict(r.bounds.beta) if r.bounds is not None else None,
        }
    return out


def reference_run_fields(desc: dict) -> dict:
    """slots / beta of the reference RunReport (runtime.py:318-323) at
    c_factor 2, 3 and 5 (4 source firings; graphs without a terminating run
    are skipped)."""
    from tokenflow.runtime import RuntimeConfig, run
    out = {}
    for c in (2, 3, 5):
        try:
            rep = run(build_graph(copy.deepcopy(desc)),
                      config=RuntimeConfig(source_firings=4, c_factor=c, seed=3,
                                           timeout_ms=2000))
        except Exception as e:  # noqa: BLE001
            out[str(c)] = {"raises": type(e).__name__}
            continue
        out[str(c)] = {"slots": rep.slots, "beta": rep.beta,
                       "max_occupancy": rep.max_occupancy,
                       "firing_counts": rep.firing_counts, "sink_digests": rep.sink_digests}
    return out


def main():
    corpus = {}
    for name, desc in named_cases().items():
        rec = record(desc)
        assert rec is not None, name
        if rec["analysis"]["3"].get("verdict") == "consistent" and not name.startswith("app_"):
            rec["reference_run"] = reference_run_fields(desc)
        corpus[name] = rec
    rng = random.Random(1802_06625)
    made = 0
    tries = 0
    while made < 600 and tries < 20000:
        tries += 1
        desc = structured(rng, tries) if tries % 3 else wild(rng, tries)
        if desc is None:
            continue
        rec = record(desc)
        if rec is None:
            continue
        corpus[desc["name"]] = rec
        made += 1
    verdicts = {}
    for rec in corpus.values():
        a = rec["analysis"]["3"]
        key = a.get("verdict", "raises " + a.get("raises", ""))
        verdicts[key] = verdicts.get(key, 0) + 1
    (OUT / "admission.json").write_text(json.dumps(corpus, sort_keys=True, separators=(",", ":")))
    print(f"{len(corpus)} graphs ({made} random, {tries} tries): {verdicts}")


if __name__ == "__main__":
    main()
