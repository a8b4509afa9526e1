"""Vision graph host side: weight preparation for the tcgen05 kernel and the
oracle's own consistency (direct-loop convolution on a small case)."""
import numpy as np

from oracle import cnn as oc
from paper_1802_06625_b200 import admit, as_graph
from paper_1802_06625_b200.apps import vision
from paper_1802_06625_b200.behaviors import resolve
from paper_1802_06625_b200.cnn_weights import (KC, conv_device_layout, core_layout,
                                               layer_params, tf32_split)


def test_tf32_split_is_exact():
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32)
    hi, lo = tf32_split(x)
    assert (hi + lo == x).all()
    assert ((hi.view(np.uint32) & 0x1FFF) == 0).all()


def test_core_layout_matches_kernel_indexing():
    rows = 32
    t = np.arange(rows * KC, dtype=np.float32).reshape(rows, KC)
    flat = core_layout(t)
    for r in range(rows):
        for k in range(KC):
            off = ((r // 8) * (KC // 4) + k // 4) * 32 + (r % 8) * 4 + k % 4
            assert flat[off] == t[r, k]


def test_conv_device_layout_roundtrip():
    w, _ = layer_params({"seed": 1}, 32, 75)
    dev = conv_device_layout(w).reshape(-1, 2, 32 * KC)
    assert dev.shape[0] == 3   # 75 -> 96 padded K
    rec = np.zeros((32, 3 * KC), np.float32)
    for c in range(3):
        for r in range(32):
            for k in range(KC):
                off = ((r // 8) * (KC // 4) + k // 4) * 32 + (r % 8) * 4 + k % 4
                rec[r, c * KC + k] = dev[c, 0, off] + dev[c, 1, off]
    assert (rec[:, :75] == w).all() and (rec[:, 75:] == 0).all()


def test_oracle_conv_against_direct_loops():
    rng = np.random.default_rng(3)
    x = rng.random((1, 8, 10, 3)).astype(np.float32)
    w = rng.standard_normal((32, 75)).astype(np.float32)
    b = rng.standard_normal(32).astype(np.float32)
    pad = 1
    got = oc.conv_relu_pool(x, w, b, pad)
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0))).astype(np.float64)
    Ho, Wo = 8 + 2 * pad - 4, 10 + 2 * pad - 4
    conv = np.zeros((Ho, Wo, 32))
    for oy in range(Ho):
        for ox in range(Wo):
            for co in range(32):
                acc = b[co]
                for ky in range(5):
                    for kx in range(5):
                        for ci in range(3):
                            acc += xp[0, oy + ky, ox + kx, ci] * w[co, (ky * 5 + kx) * 3 + ci]
                conv[oy, ox, co] = max(acc, 0.0)
    want = conv.reshape(Ho // 2, 2, Wo // 2, 2, 32).max(axis=(1, 3))
    assert np.allclose(got[0], want, rtol=1e-12, atol=1e-12)


def test_vision_graph_admitted_and_behaviours_init():
    desc = vision.build_description(24)
    p = admit(as_graph(desc))
    assert {a: c for a, c in p.actor_cond.items() if c >= 0} == {"l1": 0, "l2": 0, "l3": 0}
    for a in desc["actors"]:
        if a["behavior"] == "file_source":
            continue
        b = resolve(a["behavior"])
        b.init(a["id"], a["params"] if "params" in a else {}, None)
    params = oc.graph_params(desc)
    assert params["l3"][0].shape == (100, 18432)
    assert vision.flops_per_frame() == 104 * 104 * 32 * 150 + 48 * 48 * 32 * 1600 + 3686400
