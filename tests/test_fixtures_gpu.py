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
