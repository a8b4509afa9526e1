"""Python behaviour overrides of actors between sources and sinks
(runtime.py:336-341, interp.py:95-99): the recorder pattern of SURVEY 8(c3b)
(a FirBranch subclass that calls super().fire and records the outputs; the
FIR still runs on the device) against the reference's recorded per-branch
outputs, and pure host behaviours (no device kernel) replacing static and
dynamic actors, against the reference interpreter's digests."""
import numpy as np
import pytest

from paper_1802_06625_b200 import RuntimeConfig, run, run_streams
from paper_1802_06625_b200.apps import predistortion as pd
from paper_1802_06625_b200.behaviors import ActorBehavior, FirBranch

pytestmark = pytest.mark.gpu


class Recorder(FirBranch):
    """tests/golden/make_golden.py's Recorder, against this package."""

    def __init__(self):
        self.seen = []

    def fire(self, ctx):
        super().fire(ctx)
        self.seen.append((ctx.firing, bytes(next(iter(ctx.outputs.values())))))


@pytest.mark.parametrize("epoch", [4096, 4])
def test_recorder_sees_reference_branch_outputs(golden, tmp_path, epoch):
    arr = golden["dpd_small"]
    p = tmp_path / "input.bin"
    p.write_bytes(arr["small_input"].tobytes())
    desc = pd.build_description(256, 4, str(p), 2)
    recs = {f"b{k}": Recorder() for k in range(1, 5)}
    rep = run(desc, behaviors=recs, config=RuntimeConfig(source_firings=6, seed=11,
                                                         capture_sinks=True, epoch=epoch))
    assert rep.sink_data["sink"] == arr["small_sink"].tobytes()
    for k, r in recs.items():
        firings = [f for f, _ in r.seen]
        assert firings == arr[f"small_{k}_firings"].tolist(), k
        got = np.stack([np.frombuffer(b, np.float32) for _, b in r.seen])
        assert np.array_equal(got.view(np.uint32), arr[f"small_{k}_out"].view(np.uint32)), k


class Negate(FirBranch):
    """An observing override that rewrites its outputs: the engine copies
    ctx.outputs back, so downstream actors see the negated branch."""

    def fire(self, ctx):
        out = np.frombuffer(ctx.outputs["out"], np.float32)
        out *= -1.0


def test_observer_writes_reach_downstream(tmp_path):
    x = pd.make_input(11, 6)
    p = tmp_path / "input.bin"
    p.write_bytes(x)
    desc = pd.build_description(256, 4, str(p), 4)     # all branches active
    base = run(desc, config=RuntimeConfig(source_firings=6, seed=11, capture_sinks=True))
    neg = run(desc, behaviors={f"b{k}": Negate() for k in range(1, 5)},
              config=RuntimeConfig(source_firings=6, seed=11, capture_sinks=True))
    a = np.frombuffer(base.sink_data["sink"], np.float32)
    b = np.frombuffer(neg.sink_data["sink"], np.float32)
    assert np.array_equal(a, -b)


class PyAddMod(ActorBehavior):
    """behavior.py:168-173 written as a user behaviour (no device kernel)."""

    def fire(self, ctx):
        off = int(ctx.params.get("offset", 0))
        out = ctx.outputs["out"]
        src = ctx.inputs["in"]
        for i in range(len(out)):
            out[i] = (src[i] + off) & 0xFF


class PyRoute(ActorBehavior):
    """behavior.py:176-184 as a user behaviour: copy to active outputs."""

    def __init__(self):
        self.controls = []

    def control(self, actor_id, firing, values):
        self.controls.append((firing, values))

    def fire(self, ctx):
        (data,) = [v for k, v in ctx.inputs.items()]
        for span in ctx.outputs.values():
            if len(span):
                span[:] = data


class PyMerge(ActorBehavior):
    """behavior.py:187-199: the bytewise sum of the live inputs."""

    def fire(self, ctx):
        out = ctx.outputs["out"]
        live = [v for v in ctx.inputs.values() if len(v)]
        for i in range(len(out)):
            out[i] = sum(v[i] for v in live) & 0xFF


@pytest.mark.parametrize("epoch", [4096, 3])
@pytest.mark.parametrize("which", [("m1",), ("m1", "m2"), ("x",), ("y",), ("x", "m2", "y")])
def test_host_actors_in_gated_pipeline(golden, which, epoch):
    case = golden["fixtures"]["gated_pipeline"]
    make = {"m1": PyAddMod, "m2": PyAddMod, "x": PyRoute, "y": PyMerge}
    beh = {aid: make[aid]() for aid in which}
    rep = run(case["description"], behaviors=beh, config=RuntimeConfig(
        source_firings=case["source_firings"], seed=case["seed"], capture_sinks=True,
        epoch=epoch))
    assert rep.sink_digests == case["sink_digests"]
    assert rep.firing_counts == case["firing_counts"]
    assert rep.eq1_checks == case["eq1_checks"]
    if "x" in which:
        # control() once per firing, in order, with the decoded value
        ctl = beh["x"].controls
        assert [f for f, _ in ctl] == list(range(case["firing_counts"]["x"]))
        assert all(len(v) == 2 for _, v in ctl)


def test_host_actor_streams_use_factories(golden):
    case = golden["fixtures"]["static_chain"]
    S = 3
    reps = run_streams(case["description"], S, RuntimeConfig(
        source_firings=case["source_firings"], capture_sinks=True),
        seeds=[case["seed"]] * S, behaviors={"s2": PyAddMod})
    for r in reps:
        assert r.sink_digests == case["sink_digests"]
        assert r.firing_counts == case["firing_counts"]


class Boom(ActorBehavior):
    def fire(self, ctx):
        raise RuntimeError("boom")


def test_host_actor_exception_is_actor_panic(golden):
    from paper_1802_06625_b200 import ActorPanic
    case = golden["fixtures"]["static_chain"]
    with pytest.raises(ActorPanic) as e:
        run(case["description"], behaviors={"s2": Boom()},
            config=RuntimeConfig(source_firings=4))
    assert e.value.actor == "s2"


def test_overrides_keep_fused_regions_apart(golden, tmp_path):
    """A Python override (here observers: device-behaviour subclasses whose fire
    sees the device result) of a member of a fused region -- the bypass app's
    l2, the motion app's clean -- keeps that region's channels materialised
    (per-actor launches) and the reference's outputs unchanged; the observers
    see every firing."""
    from paper_1802_06625_b200.apps import bypass, motion
    from paper_1802_06625_b200.behaviors import MatMul, PlusMedian
    from paper_1802_06625_b200.engine import DeviceRuntime

    class SeenMM(MatMul):
        def __init__(self):
            self.n = 0

        def fire(self, ctx):
            self.n += 1

    class SeenMedian(PlusMedian):
        def __init__(self):
            self.n = 0

        def fire(self, ctx):
            self.n += 1

    arr = golden["bypass_small"]
    p = tmp_path / "input.bin"
    p.write_bytes(arr["input"].tobytes())
    obs = SeenMM()
    desc = bypass.build_description(str(p))
    cfg = RuntimeConfig(source_firings=32, seed=5, capture_sinks=True)
    rep = run(desc, behaviors={"l2": obs}, config=cfg)
    assert rep.sink_data["sink"] == arr["sink"].tobytes()
    assert obs.n == rep.firing_counts["l2"] == golden["bypass"]["default"]["firing_counts"]["l2"]
    rt = DeviceRuntime(desc, behaviors={"l2": SeenMM()}, config=cfg, n_streams=1, seeds=[5])
    assert "bypass_region" not in [item[0] for item in rt.launches]
    rt.close()

    mp = tmp_path / "motion.bin"
    mp.write_bytes(motion.make_input(7, 16))
    mobs = SeenMedian()
    rep = run(motion.build_description(input_path=str(mp)), behaviors={"clean": mobs},
              config=RuntimeConfig(source_firings=16, seed=7, capture_sinks=True, epoch=5))
    assert rep.sink_data["sink"] == golden["motion_small"]["sink_16_7"].tobytes()
    assert mobs.n == 16
