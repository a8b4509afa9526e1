"""The DPD path at BASELINE config 2's full size (64 streams x 256 blocks x
4096 samples, 537 MB per run), checked through size-independent properties:
firing counts of every stream exact against the control replay, two streams
against the oracle, determinism (identical digests across runs), and
linearity of the filter bank under a fixed control schedule
(sink(x + y) = sink(x) + sink(y) within fp32 rounding), which covers every
stream and every block without running the CPU oracle on all of them."""
import numpy as np
import pytest

from oracle import dpd as od
from paper_1802_06625_b200 import RuntimeConfig, run_streams
from paper_1802_06625_b200.apps import predistortion as pd

pytestmark = pytest.mark.gpu

S, BLOCKS, B, K = 64, 256, 4096, 4


def _run(xs, exact):
    desc = pd.build_description(B, K)
    return run_streams(desc, S, RuntimeConfig(source_firings=BLOCKS, epoch=BLOCKS, exact=exact,
                                              capture_sinks=True),
                       seeds=[pd.stream_seed(s) for s in range(S)],
                       sources={"src": [x.tobytes() for x in xs]})


@pytest.mark.parametrize("exact", [False, True])
def test_c2_full_size_properties(exact):
    xs = [pd.stream_input(s, BLOCKS, B) for s in range(S)]
    reps = _run(xs, exact)
    for s in range(S):
        sets = od.subset_schedule(pd.stream_seed(s), BLOCKS, length=K)
        assert reps[s].firing_counts == od.firing_counts(sets, K), s
    for s in (0, S - 1):
        sets = od.subset_schedule(pd.stream_seed(s), BLOCKS, length=K)
        want = od.dpd_stream(xs[s], sets, K)
        got = np.frombuffer(reps[s].sink_data["sink"], np.float32).reshape(want.shape)
        if exact:
            assert got.tobytes() == want.tobytes(), s
        else:
            err = np.abs(got.astype(np.float64) - want) / np.maximum(1.0, np.abs(want))
            assert err.max() <= 1e-5, (s, err.max())
    again = _run(xs, exact)
    assert [r.sink_digests for r in again] == [r.sink_digests for r in reps]


def test_c2_full_size_linearity():
    rng = np.random.default_rng(7)
    xs = [pd.stream_input(s, BLOCKS, B) for s in range(S)]
    ys = [rng.uniform(-1, 1, x.shape).astype(np.float32) for x in xs]
    zs = [(x.astype(np.float64) + y).astype(np.float32) for x, y in zip(xs, ys)]
    rx, ry, rz = _run(xs, False), _run(ys, False), _run(zs, False)
    worst = 0.0
    for s in range(S):
        fx = np.frombuffer(rx[s].sink_data["sink"], np.float32).astype(np.float64)
        fy = np.frombuffer(ry[s].sink_data["sink"], np.float32).astype(np.float64)
        fz = np.frombuffer(rz[s].sink_data["sink"], np.float32).astype(np.float64)
        scale = np.maximum(1.0, np.abs(fx) + np.abs(fy))
        worst = max(worst, float((np.abs(fz - (fx + fy)) / scale).max()))
    assert worst <= 1e-5, worst
