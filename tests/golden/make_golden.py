"""Generate the golden vectors under tests/golden/ by running the REFERENCE
package itself (tokenflow, imported from /root/reference/pkg/src).

Run here (the build container) only; /root/reference does not exist on the
GPU box, which reads the committed outputs instead:

    python tests/golden/make_golden.py

Outputs (all small):
  dpd.json         sink digests / firing counts / control sets for DPD cases
  dpd_small.npz    full sink streams + per-branch FIR outputs of short runs
  fixtures.json    sink digests + firing counts of the reference's engine
                   conformance fixtures (pkg/tests/fixtures.py)
  bypass.json      bypass app digests; bypass_small.npz sink bytes
  policies.json    control sequences of the four policies for several seeds
  motion.json      motion app (one-frame delay FIFO): sink digests and firing
                   counts; motion_small.npz the sink bytes of a short run;
                   the static chain fixture with a 2-token delay
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("PRUNE_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import fixtures as fx  # noqa: E402  (reference test fixtures)
from tokenflow import behavior as tb  # noqa: E402
from tokenflow.apps import bypass as rbp  # noqa: E402
from tokenflow.apps import motion as rmo  # noqa: E402
from tokenflow.apps import make_app  # noqa: E402
from tokenflow.apps import predistortion as rpd  # noqa: E402
from tokenflow.interp import interpret  # noqa: E402
from tokenflow.model import build_graph  # noqa: E402
from tokenflow.runtime import RuntimeConfig, run  # noqa: E402

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parent.parent))
from paper_1802_06625_b200.apps import predistortion as mypd  # noqa: E402


class Recorder(rpd.FirBranch):
    def init(self, actor_id, params, seed):
        super().init(actor_id, params, seed)
        self.seen = []

    def fire(self, ctx):
        super().fire(ctx)
        self.seen.append((ctx.firing, bytes(next(iter(ctx.outputs.values())))))


def dpd_case(block, branches, blocks, seed, data: bytes, record=False):
    """Reference interpret() of the DPD graph at a non-default shape
    (SURVEY §8 c3b recipe: module globals BLOCK/TOKEN_BYTES/BRANCHES)."""
    saved = (rpd.BLOCK, rpd.TOKEN_BYTES, rpd.BRANCHES)
    rpd.BLOCK, rpd.TOKEN_BYTES, rpd.BRANCHES = block, block * 8, branches
    try:
        with tempfile.TemporaryDirectory() as td:
            p = Path(td) / "input.bin"
            p.write_bytes(data)
            desc = rpd.build_description(str(p))
            g = build_graph(desc)
            recs = {f"b{k}": Recorder() for k in range(1, branches + 1)} if record else None
            rep = interpret(g, behaviors=recs, source_firings=blocks, seed=seed,
                            capture_sinks=True)
            branch_out = None
            if record:
                branch_out = {k: [(f, np.frombuffer(b, np.float32).copy()) for f, b in r.seen]
                              for k, r in recs.items()}
            return rep, branch_out
    finally:
        rpd.BLOCK, rpd.TOKEN_BYTES, rpd.BRANCHES = saved


def main():
    dpd = {}
    arrays = {}
    # C1: the reference default app (B=256, K=4, 160 blocks, seed 11)
    app = make_app("predistortion")
    rep, _ = dpd_case(256, 4, app.iterations, app.seed, app.input_bytes)
    dpd["default"] = {"block": 256, "branches": 4, "blocks": 160, "seed": 11,
                      "input": "make_input(11, 160)",
                      "input_sha256": hashlib.sha256(app.input_bytes).hexdigest(),
                      "sink_digest": rep.sink_digests["sink"],
                      "firing_counts": rep.firing_counts}
    arrays["default_sink_head"] = np.frombuffer(rep.sink_data["sink"][:4 * 2048], np.uint8)
    # short run with per-branch outputs (kernel-level parity)
    small = rpd.make_input(11, 6)
    rep, br = dpd_case(256, 4, 6, 11, small, record=True)
    dpd["small"] = {"block": 256, "branches": 4, "blocks": 6, "seed": 11,
                    "sink_digest": rep.sink_digests["sink"], "firing_counts": rep.firing_counts}
    arrays["small_input"] = np.frombuffer(small, np.uint8)
    arrays["small_sink"] = np.frombuffer(rep.sink_data["sink"], np.uint8)
    for k, seen in br.items():
        arrays[f"small_{k}_firings"] = np.array([f for f, _ in seen], np.int32)
        arrays[f"small_{k}_out"] = np.stack([o for _, o in seen])
    # C2 shape: B=4096, K=4, per-stream numpy input, seed 1000+s
    for s in (0, 1):
        x = mypd.stream_input(s, 24, 4096)
        rep, _ = dpd_case(4096, 4, 24, 1000 + s, x.tobytes())
        dpd[f"c2_stream{s}"] = {"block": 4096, "branches": 4, "blocks": 24, "seed": 1000 + s,
                                "input": f"stream_input({s}, 24, 4096)",
                                "sink_digest": rep.sink_digests["sink"],
                                "firing_counts": rep.firing_counts}
    # paper-scale branch count K=10 (string-sorted combiner order e1,e10,e2..)
    x = mypd.stream_input(7, 16, 512)
    rep, _ = dpd_case(512, 10, 16, 1007, x.tobytes())
    dpd["k10"] = {"block": 512, "branches": 10, "blocks": 16, "seed": 1007,
                  "input": "stream_input(7, 16, 512)", "sink_digest": rep.sink_digests["sink"],
                  "firing_counts": rep.firing_counts}
    arrays["k10_sink"] = np.frombuffer(rep.sink_data["sink"], np.uint8)
    # all-active impulse (test_acceptance.py:251-281)
    imp = np.zeros(512, np.float32)
    imp[0] = 1.0
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "impulse.bin"
        p.write_bytes(imp.tobytes())
        desc = rpd.build_description(str(p))
        for a in desc["actors"]:
            if a["id"] == "conf":
                a["params"]["min_active"] = 4
        rep = interpret(build_graph(desc), source_firings=1, seed=11, capture_sinks=True)
    arrays["impulse_sink"] = np.frombuffer(rep.sink_data["sink"], np.uint8)
    (OUT / "dpd.json").write_text(json.dumps(dpd, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "dpd_small.npz", **arrays)

    # engine conformance fixtures (test_interp.py:86-98)
    fixtures = {}
    cases = [("static_chain", {}), ("broadcast_two_sinks", {}), ("clean_single_chain", {}),
             ("clean_two_component", {}), ("gated_pipeline", {}), ("rate_pair", {"atr": 3}),
             ("static_chain", {"stages": 2, "token_bytes": 5})]
    for name, kw in cases:
        desc = getattr(fx, name)(**kw)
        g = build_graph(desc)
        rep = interpret(g, source_firings=10, seed=6, capture_sinks=True)
        rt = run(g, config=RuntimeConfig(source_firings=10, seed=6))
        assert rt.sink_digests == rep.sink_digests
        key = name + ("" if not kw else "_" + "_".join(f"{k}{v}" for k, v in kw.items()))
        fixtures[key] = {"builder": name, "kwargs": kw, "description": desc,
                         "source_firings": 10, "seed": 6,
                         "sink_digests": rep.sink_digests, "firing_counts": rep.firing_counts,
                         "eq1_checks": rt.eq1_checks,
                         "sink_data_hex": {k: v.hex() for k, v in rep.sink_data.items()}}
    (OUT / "fixtures.json").write_text(json.dumps(fixtures, indent=1, sort_keys=True))

    # bypass app (matmul chain + marker)
    bp = {}
    app = make_app("bypass")
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "input.bin"
        p.write_bytes(app.input_bytes)
        rep = interpret(app.graph(str(p)), source_firings=app.iterations, seed=app.seed,
                        capture_sinks=True)
    bp["default"] = {"mats": 32, "seed": 5, "sink_digest": rep.sink_digests["sink"],
                     "firing_counts": rep.firing_counts,
                     "input_sha256": hashlib.sha256(app.input_bytes).hexdigest()}
    np.savez_compressed(OUT / "bypass_small.npz",
                        input=np.frombuffer(app.input_bytes, np.uint8),
                        sink=np.frombuffer(rep.sink_data["sink"], np.uint8))
    (OUT / "bypass.json").write_text(json.dumps(bp, indent=1, sort_keys=True))

    # policies: control vectors straight from the reference behaviours
    pol = {}
    for name, params in [("subset_policy", {"length": 4, "min_active": 2}),
                         ("subset_policy", {"length": 10, "min_active": 2}),
                         ("subset_policy", {"length": 30, "min_active": 3}),
                         ("seeded_policy", {"length": 3}),
                         ("seeded_policy", {"length": 7}),
                         ("alternate_policy", {"length": 3}),
                         ("fixed_policy", {"length": 3, "element": 2})]:
        for seed in (None, 0, 5, 11, 351504803, 2**31 - 1):
            b = tb.resolve(name)
            b.init("conf", params, seed)
            vecs = []
            for f in range(64):
                span = bytearray(params["length"])
                ctx = tb.FireContext("conf", f, {"ctl": 1}, {}, {"ctl": memoryview(span)},
                                     params, seed)
                b.fire(ctx)
                vecs.append(bytes(span).hex())
            pol[f"{name}|{json.dumps(params, sort_keys=True)}|{seed}"] = vecs
    (OUT / "policies.json").write_text(json.dumps(pol, indent=1, sort_keys=True))

    # motion detection (one-frame delay FIFO, apps/motion.py)
    mo = {}
    arrays = {}
    for frames, seed in ((16, 7), (40, 3)):
        data = rmo.make_input(seed, frames)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "motion.bin")
            Path(path).write_bytes(data)
            g = build_graph(rmo.build_description(path))
            res = interpret(g, source_firings=frames, seed=seed, capture_sinks=True)
        key = f"{frames}|{seed}"
        mo[key] = {"frames": frames, "seed": seed,
                   "sink_digest": res.sink_digests["sink"],
                   "firing_counts": dict(res.firing_counts)}
        if frames == 16:
            arrays["sink_16_7"] = np.frombuffer(res.sink_data["sink"], dtype=np.uint8)
    # a byte diamond with 2 initial delay tokens on one branch: s1 broadcasts
    # to an undelayed and a delayed channel, add_mod sums both
    def port(pid, d):
        return {"id": pid, "dir": d, "kind": "srp", "rate": 1}
    desc = {"name": "diamond", "control": {}, "actors": [
        {"id": "src", "kind": "static", "behavior": "counter_source", "ports": [port("out", "out")]},
        {"id": "s1", "kind": "static", "behavior": "passthrough",
         "ports": [port("in", "in"), port("out", "out")]},
        {"id": "m", "kind": "static", "behavior": "add_mod", "params": {"offset": 3},
         "ports": [port("a", "in"), port("b", "in"), port("out", "out")]},
        {"id": "sink", "kind": "static", "behavior": "null_sink", "ports": [port("in", "in")]}],
        "fifos": [
            {"id": "f0", "src": "src.out", "dst": "s1.in", "rate": 1, "delay": 0, "token_bytes": 4},
            {"id": "fa", "src": "s1.out", "dst": "m.a", "rate": 1, "delay": 0, "token_bytes": 4},
            {"id": "fb", "src": "s1.out", "dst": "m.b", "rate": 1, "delay": 2, "token_bytes": 4,
             "delay_payload_hex": bytes(range(8)).hex()},
            {"id": "fo", "src": "m.out", "dst": "sink.in", "rate": 1, "delay": 0,
             "token_bytes": 4}]}
    g = build_graph(desc)
    res = interpret(g, source_firings=12, seed=5, capture_sinks=True)
    mo["diamond_delay2"] = {"description": desc, "iterations": 12, "seed": 5,
                            "sink_digest": res.sink_digests["sink"],
                            "firing_counts": dict(res.firing_counts),
                            "sink_hex": res.sink_data["sink"].hex()}
    (OUT / "motion.json").write_text(json.dumps(mo, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "motion_small.npz", **arrays)
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
