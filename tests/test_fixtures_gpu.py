"""Engine conformance on the reference's fixture graphs (pkg/tests/fixtures.py,
test_interp.py:86-98): sink digests and firing counts equal the reference
interpreter's, recorded in tests/golden/fixtures.json."""
import pytest

from paper_1802_06625_b200 import RuntimeConfig, run

pytestmark = pytest.mark.gpu


def cases(golden):
    return sorted(golden["fixtures"])


@pytest.mark.parametrize("key", ["static_chain", "broadcast_two_sinks", "clean_single_chain",
                                 "clean_two_component", "gated_pipeline", "rate_pair_atr3",
                                 "static_chain_stages2_token_bytes5"])
@pytest.mark.parametrize("epoch", [4096, 3])
def test_fixture_matches_reference(golden, key, epoch):
    case = golden["fixtures"][key]
    rep = run(case["description"], config=RuntimeConfig(
        source_firings=case["source_firings"], seed=case["seed"], capture_sinks=True,
        epoch=epoch))
    assert rep.sink_digests == case["sink_digests"]
    assert rep.firing_counts == case["firing_counts"]
    assert rep.eq1_checks == case["eq1_checks"]
    for sink, hexdata in case["sink_data_hex"].items():
        assert rep.sink_data[sink].hex() == hexdata


def _admission_cases():
    import json

    from conftest import GOLDEN
    corpus = json.loads((GOLDEN / "admission.json").read_text())
    return {k: v for k, v in corpus.items() if "reference_run" in v}


ADMISSION = _admission_cases()


@pytest.mark.parametrize("c_factor", [2, 3, 5])
@pytest.mark.parametrize("key", sorted(ADMISSION))
def test_run_report_fields_match_reference(key, c_factor):
    """RunReport slots / beta at the caller's c_factor equal the reference
    RunReport's (runtime.py:318-323, fifos.py:87-98, analysis.py:398-411);
    firing counts and digests too; max_occupancy stays within beta and slots
    (test_runtime.py:211-219) and the device rings within their capacity."""
    from paper_1802_06625_b200 import UnsupportedGraph
    case = ADMISSION[key]
    want = case["reference_run"][str(c_factor)]
    if "raises" in want:
        pytest.skip(f"reference run raises {want['raises']}")
    try:
        rep = run(case["description"], config=RuntimeConfig(source_firings=4, c_factor=c_factor,
                                                            seed=3, epoch=3))
    except UnsupportedGraph:
        pytest.skip("outside the executor's class")
    assert rep.slots == want["slots"] and rep.beta == want["beta"]
    assert rep.firing_counts == want["firing_counts"]
    assert rep.sink_digests == want["sink_digests"]
    for fid, occ in rep.max_occupancy.items():
        assert occ <= rep.beta[fid] and occ <= rep.slots[fid], fid
        assert rep.device_max_occupancy[fid] <= rep.device_slots[fid], fid
