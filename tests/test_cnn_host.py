"""Vision graph host side: weight preparation for the tcgen05 kernel and the
oracle's own consistency (direct-loop convolution on a small case)."""
import numpy as np

from oracle import cnn as oc
from paper_1802_06625_b200 import admit, as_graph
from paper_1802_06625_b200.apps import vision
from paper_1802_06625_b200.behaviors import resolve
from paper_1802_06625_b200.cnn_weights import (bf16_rn, bf16_split, conv_device_layout,
                                               conv_steps, layer_params)


def test_bf16_rn_matches_torch():
    import torch
    x = np.random.default_rng(0).standard_normal(100000).astype(np.float32) * 37.0
    want = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert (bf16_rn(x) == want).all()


def test_bf16_split_accuracy():
    x = np.random.default_rng(1).standard_normal(100000).astype(np.float32)
    hi, lo = bf16_split(x)
    assert ((hi.view(np.uint32) & 0xFFFF) == 0).all() and ((lo.view(np.uint32) & 0xFFFF) == 0).all()
    rel = np.abs((hi.astype(np.float64) + lo) - x) / np.abs(x)
    assert rel.max() <= 2.0 ** -17


def _unpack(dev, steps):
    """Inverse of conv_device_layout: [S][64][16] fp32 from bf16 bits."""
    bits = dev.reshape(steps, 8, 2, 8, 8).transpose(0, 1, 3, 2, 4).reshape(steps, 64, 16)
    return (bits.astype(np.uint32) << 16).view(np.float32)


def test_conv_device_layout_roundtrip():
    for cin, steps in ((3, 5), (32, 50)):
        w, _ = layer_params({"seed": 1}, 32, 25 * cin)
        dev = conv_device_layout(w, cin)
        assert dev.dtype == np.uint16 and dev.size == steps * 64 * 16
        m = _unpack(dev, steps)
        hi, lo = bf16_split(conv_steps(w, cin))
        assert (m[:, :32] == hi).all() and (m[:, 32:] == lo).all()
        rec = conv_steps(w, cin)
        if cin == 3:   # step ky, index kx*3+ci
            assert (rec[:, :, 15] == 0).all()
            assert (rec.transpose(1, 0, 2)[:, :, :15].reshape(32, 75) == w).all()
        else:          # step (ky, kx, kc), channel 16kc+e
            assert (rec.reshape(25, 2, 32, 16).transpose(2, 0, 1, 3).reshape(32, 800) == w).all()


def test_dense_device_layout_roundtrip():
    from paper_1802_06625_b200.cnn_weights import dense_device_layout
    w, _ = layer_params({"seed": 3}, 100, 256)
    dev = dense_device_layout(w)
    S = 256 // 16
    bits = dev.reshape(S, 28, 2, 8, 8).transpose(1, 3, 0, 2, 4).reshape(224, 256)
    m = (bits.astype(np.uint32) << 16).view(np.float32)
    hi, lo = bf16_split(w)
    assert (m[:100] == hi).all() and (m[112:212] == lo).all()
    assert (m[100:112] == 0).all() and (m[212:] == 0).all()


def emulate_conv(x, w, b, pad):
    """The kernel's arithmetic on the CPU: operands split to bf16 hi/lo,
    D = xh*wh + xl*wh + xh*wl (float64 accumulation ~ TMEM fp32), bias,
    ReLU, 2x2 max pool."""
    F, H, W, Cin = x.shape
    xh, xl = bf16_split(x)
    wh, wl = bf16_split(w)
    xp = [np.pad(a.astype(np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0))) for a in (xh, xl)]
    Ho, Wo = H + 2 * pad - 4, W + 2 * pad - 4
    def im2col(a):
        cols = np.empty((F, Ho, Wo, 25 * Cin))
        for ky in range(5):
            for kx in range(5):
                t = ky * 5 + kx
                cols[..., t * Cin:(t + 1) * Cin] = a[:, ky:ky + Ho, kx:kx + Wo, :]
        return cols
    ch, cl = im2col(xp[0]), im2col(xp[1])
    y = ch @ wh.astype(np.float64).T + cl @ wh.astype(np.float64).T + ch @ wl.astype(np.float64).T
    y = np.maximum(y + b, 0.0)
    return y.reshape(F, Ho // 2, 2, Wo // 2, 2, -1).max(axis=(2, 4))


def test_split_bf16_conv_within_tolerance():
    """bf16x3 meets the stated activation tolerance (1e-4 of max(1,|y|)) on
    the vision graph's own layer shapes."""
    p = oc.graph_params(vision.build_description(1))
    x = vision.make_frames(0, 1)
    want1 = oc.conv_relu_pool(x, *p["l1"])
    got1 = emulate_conv(x, *p["l1"])
    assert (np.abs(got1 - want1) / np.maximum(1, np.abs(want1))).max() <= 2e-5
    x2 = want1.astype(np.float32)
    want2 = oc.conv_relu_pool(x2, *p["l2"])
    got2 = emulate_conv(x2, *p["l2"])
    assert (np.abs(got2 - want2) / np.maximum(1, np.abs(want2))).max() <= 2e-5


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


def test_conv_device_layout_i8_roundtrip():
    """The int8-limb B operand: per K-step rows 0-31 [wh | 0], rows 32-63
    [wl | wh] in core-matrix order, then the dequantisation factors; the limbs
    recombine to the quantised weights, which are within wdq / 2 of W."""
    from paper_1802_06625_b200.cnn_weights import (W_LIMIT, conv_device_layout_i8,
                                                   conv_quant_weights)
    w, _ = layer_params({"seed": 2}, 32, 800)
    dev = conv_device_layout_i8(w, 32)
    S = 50
    assert dev.dtype == np.uint8 and dev.size == S * 2048 + 128
    rows = dev[:S * 2048].view(np.int8).reshape(S, 8, 2, 8, 16).transpose(0, 1, 3, 2, 4)
    rows = rows.reshape(S, 64, 32).astype(np.int64)
    wdq = dev[S * 2048:].view(np.float32)
    q, wdq_ref = conv_quant_weights(w)
    assert (wdq == wdq_ref).all() and np.abs(q).max() <= W_LIMIT
    assert (rows[:, :32, 16:] == 0).all() and (rows[:, 32:, 16:] == rows[:, :32, :16]).all()
    rec = 256 * rows[:, :32, :16] + rows[:, 32:, :16]                 # [S][32][16]
    assert (rec == conv_steps(q.astype(np.float32), 32).astype(np.int64)).all()
    assert (np.abs(q * wdq[:, None].astype(np.float64) - w) <= wdq[:, None] * 0.5 + 1e-12).all()


def test_int8_limb_conv_within_tolerance():
    """The int8-limb layer-2 arithmetic (cnn_weights.conv_i8_reference, which
    the GPU tests hold the kernel to) on the vision graph's own shapes: conv
    tokens within 1e-3 of max(1, |y|) of float64, and the logits it leads to
    within the north star's 1e-3, top-1 equal."""
    from paper_1802_06625_b200.cnn_weights import conv_i8_reference
    p = oc.graph_params(vision.build_description(2))
    x = vision.make_frames(3, 2)
    want = oc.forward(x, p)
    l1 = want["l1"].astype(np.float32)
    got2 = conv_i8_reference(l1, *p["l2"])
    assert (np.abs(got2 - want["l2"]) / np.maximum(1, np.abs(want["l2"]))).max() <= 1e-3
    logits = oc.classify(oc.dense(got2.astype(np.float32), *p["l3"]), *p["join"])
    assert np.abs(logits - want["logits"]).max() <= 1e-3
    assert (logits.argmax(-1) == want["logits"].argmax(-1)).all()
