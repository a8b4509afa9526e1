"""The oracle itself, pinned against the reference's golden vectors."""
import hashlib

import numpy as np

from oracle import dpd as od
from paper_1802_06625_b200.apps import predistortion as pd


def sink_bytes(x, sets, K):
    return od.dpd_stream(x, sets, K).tobytes()


def test_subset_schedule_matches_reference_known_answer():
    # pkg/tests/test_behavior.py:343-348
    sets = od.subset_schedule(11, 6)
    assert [sorted(s) for s in sets] == [[1, 2, 3, 4], [1, 2, 3, 4], [3, 4], [1, 2, 3, 4],
                                        [1, 2, 3, 4], [1, 3]]


def test_actor_seed_frozen_values():
    # pkg/tests/test_behavior.py:115-119
    assert od.actor_seed(0, "conf") == 351504808
    assert od.actor_seed(11, "conf") == 351504803
    assert od.actor_seed(0, "q") == 1962978855
    assert od.actor_seed(123, "src") == 1615078646


def test_taps_frozen():
    for k in range(4):
        re, im = od.branch_taps(k)
        pre, pim = pd.branch_taps(k)
        assert [float(v) for v in re] == pre and [float(v) for v in im] == pim


def test_default_app_digest(golden):
    g = golden["dpd"]["default"]
    data = pd.make_input(11, 160)
    assert hashlib.sha256(data).hexdigest() == g["input_sha256"]
    x = np.frombuffer(data, np.float32).reshape(160, 2, 256)
    sets = od.subset_schedule(11, 160)
    assert hashlib.sha256(sink_bytes(x, sets, 4)).hexdigest() == g["sink_digest"]
    assert od.firing_counts(sets, 4) == g["firing_counts"]


def test_small_run_sink_and_branch_outputs(golden):
    arr = golden["dpd_small"]
    x = np.frombuffer(arr["small_input"].tobytes(), np.float32).reshape(6, 2, 256)
    sets = od.subset_schedule(11, 6)
    out, per = od.dpd_stream(x, sets, 4, return_branches=True)
    assert out.tobytes() == arr["small_sink"].tobytes()
    for k in range(1, 5):
        got = np.stack([o.reshape(-1) for _, o in per[k]])
        assert got.tobytes() == arr[f"small_b{k}_out"].tobytes()


def test_c2_shape_streams(golden):
    for s in (0, 1):
        g = golden["dpd"][f"c2_stream{s}"]
        x = pd.stream_input(s, 24, 4096)
        sets = od.subset_schedule(1000 + s, 24)
        assert hashlib.sha256(sink_bytes(x, sets, 4)).hexdigest() == g["sink_digest"]


def test_k10_string_sorted_combiner(golden):
    g = golden["dpd"]["k10"]
    assert od.combiner_order(10) == [1, 10, 2, 3, 4, 5, 6, 7, 8, 9]
    x = pd.stream_input(7, 16, 512)
    sets = od.subset_schedule(1007, 16, length=10)
    assert sink_bytes(x, sets, 10) == golden["dpd_small"]["k10_sink"].tobytes()


def test_impulse_response(golden):
    x = np.zeros((1, 2, 256), np.float32)
    x[0, 0, 0] = 1.0
    out = od.dpd_stream(x, [{1, 2, 3, 4}], 4)
    assert out.tobytes() == golden["dpd_small"]["impulse_sink"].tobytes()


def test_motion_oracle_matches_reference(golden):
    """oracle/motion.py against the reference motion app run through
    tokenflow.interp.interpret (tests/golden/motion.json)."""
    from oracle import motion as om
    from paper_1802_06625_b200.apps import motion as am
    want = golden["motion_small"]["sink_16_7"].tobytes()
    assert om.motion_stream(am.make_input(7, 16), 16) == want
    for key, case in golden["motion"].items():
        if "|" not in key:
            continue
        got = om.motion_stream(am.make_input(case["seed"], case["frames"]), case["frames"])
        assert hashlib.sha256(got).hexdigest() == case["sink_digest"]
