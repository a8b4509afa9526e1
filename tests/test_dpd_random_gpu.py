"""Randomised DPD filter-bank configurations against the oracle: branch
counts 1..32 (the launch limit), odd block lengths, min_active 0..K, several
streams and epoch splits; bit-exact in the exact mode, <= 1e-5 in the
tolerance mode, control and firing counts exact in both."""
import random

import numpy as np
import pytest

from oracle import dpd as od
from paper_1802_06625_b200 import RuntimeConfig, UnsupportedGraph, run_streams
from paper_1802_06625_b200.apps import predistortion as pd

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = random.Random(seed)
    K = rng.choice([1, 2, 3, 5, 8, 13, 32])
    B = rng.choice([16, 24, 136, 512, 1032, 2048, 4104])
    min_active = rng.randint(0, K)
    S = rng.randint(1, 4)
    blocks = rng.randint(3, 14)
    epoch = rng.choice([1, 2, 5, 4096])
    return K, B, min_active, S, blocks, epoch


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("exact", [True, False])
def test_random_bank(seed, exact):
    K, B, min_active, S, blocks, epoch = _case(seed)
    xs = [pd.stream_input(40 + s, blocks, B) for s in range(S)]
    desc = pd.build_description(B, K, min_active=min_active)
    reps = run_streams(desc, S, RuntimeConfig(source_firings=blocks, capture_sinks=True,
                                              exact=exact, epoch=epoch),
                       seeds=[7 * seed + s for s in range(S)],
                       sources={"src": [x.tobytes() for x in xs]})
    for s in range(S):
        sets = od.subset_schedule(7 * seed + s, blocks, length=K, min_active=min_active)
        want = od.dpd_stream(xs[s], sets, K)
        got = np.frombuffer(reps[s].sink_data["sink"], np.float32).reshape(want.shape)
        if exact:
            assert got.tobytes() == want.tobytes(), (K, B, s)
        else:
            err = np.abs(got.astype(np.float64) - want) / np.maximum(1.0, np.abs(want))
            assert err.max() <= 1e-5, (K, B, s, err.max())
        assert reps[s].firing_counts == od.firing_counts(sets, K)


def test_block_shorter_than_the_halo_is_unsupported():
    """B = 8 < the 12-sample window halo of the FIR kernels: refused, not run wrong."""
    desc = pd.build_description(8, 4)
    x = pd.stream_input(0, 3, 8)
    with pytest.raises(UnsupportedGraph):
        run_streams(desc, 1, RuntimeConfig(source_firings=3),
                    sources={"src": [x.tobytes()]})
