"""BASELINE config 5 on one B200: the mixed graph (DPD filter bank + adaptive
CNN, two host configuration actors, dynamic rates) in one batched run,
several streams; each half against its oracle."""
import numpy as np
import pytest

from oracle import cnn as oc
from oracle import dpd as od
from paper_1802_06625_b200 import RuntimeConfig, run_streams
from paper_1802_06625_b200.apps import mixed, vision
from paper_1802_06625_b200.apps import predistortion as pd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("exact,epoch", [(True, 4096), (False, 3)])
def test_mixed_graph(exact, epoch):
    S, N, B, K, R = 3, 6, 1024, 4, 2
    desc = mixed.build_description(B, K, R)
    xs = [pd.stream_input(s, N, B) for s in range(S)]
    fr = [vision.make_frames(10 + s, N * R) for s in range(S)]
    reps = run_streams(desc, S, RuntimeConfig(source_firings=N, capture_sinks=True, exact=exact,
                                              epoch=epoch),
                       seeds=[500 + s for s in range(S)],
                       sources={"dpd_src": [x.tobytes() for x in xs],
                                "cnn_src": [f.tobytes() for f in fr]})
    p = oc.graph_params(vision.build_description(R))
    for s in range(S):
        sets = od.subset_schedule(500 + s, N, length=K, actor="dpd_conf")
        want = od.dpd_stream(xs[s], sets, K)
        got = np.frombuffer(reps[s].sink_data["dpd_sink"], np.float32).reshape(want.shape)
        if exact:
            assert got.tobytes() == want.tobytes()
        else:
            assert (np.abs(got - want) / np.maximum(1.0, np.abs(want))).max() <= 1e-5
        logits = np.frombuffer(reps[s].sink_data["cnn_sink"], np.float32).reshape(N, R, -1)
        for j in range(N):
            if j % 2 == 0:
                w = oc.forward(fr[s][j * R:(j + 1) * R], p)["logits"]
                assert np.abs(logits[j] - w).max() <= 1e-3
            else:
                assert (logits[j] == np.float32(p["marker"])).all()
        fc = reps[s].firing_counts
        assert fc["dpd_combine"] == fc["cnn_join"] == N
        assert fc["cnn_l1"] == N // 2
        assert sum(fc[f"dpd_b{k}"] for k in range(1, K + 1)) == sum(len(x) for x in sets)
