"""ORACLE (test infrastructure only) for the vision graph — PARITY UNPINNED.

The reference package has no DNN (SPEC.md:640, :655 replace it with 8x8
matmuls), so there is no reference output to pin against.  This is the
builder's frozen float64 restatement of the graph defined in
paper_1802_06625_b200/apps/vision.py (shapes from PAPER.md:674-684, :700):
conv5x5 (zero pad) + bias + ReLU + 2x2 max pool, twice; dense; then
ReLU -> hidden (ReLU) -> logits, or marker logits for bypassed firings.
Device parity is a tolerance (north star: <= 1e-3 on logits, top-1
consistent), stated in tests/test_cnn_gpu.py.
"""
from __future__ import annotations

import numpy as np


def conv_relu_pool(x: np.ndarray, w: np.ndarray, b: np.ndarray, pad: int) -> np.ndarray:
    """x [F,H,W,C] -> [F,Ho/2,Wo/2,32]; w [cout][25*cin] in (ky,kx,ci) order."""
    F, H, W, Cin = x.shape
    xp = np.pad(x.astype(np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    Ho, Wo = H + 2 * pad - 4, W + 2 * pad - 4
    cols = np.empty((F, Ho, Wo, 25 * Cin), np.float64)
    for ky in range(5):
        for kx in range(5):
            t = ky * 5 + kx
            cols[..., t * Cin:(t + 1) * Cin] = xp[:, ky:ky + Ho, kx:kx + Wo, :]
    y = cols @ w.astype(np.float64).T + b.astype(np.float64)
    y = np.maximum(y, 0.0)
    y = y.reshape(F, Ho // 2, 2, Wo // 2, 2, -1).max(axis=(2, 4))
    return y


def dense(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    F = x.shape[0]
    return x.reshape(F, -1).astype(np.float64) @ w.astype(np.float64).T + b


def classify(x, w4, b4, w5, b5):
    h = np.maximum(np.maximum(x, 0.0) @ w4.astype(np.float64).T + b4, 0.0)
    return h @ w5.astype(np.float64).T + b5


def forward(frames: np.ndarray, params: dict) -> dict:
    """All intermediate tokens of a processed firing (float64)."""
    l1 = conv_relu_pool(frames, *params["l1"])
    l2 = conv_relu_pool(l1, *params["l2"])
    l3 = dense(l2, *params["l3"])
    logits = classify(l3, *params["join"])
    return {"l1": l1, "l2": l2, "l3": l3, "logits": logits}


def graph_params(desc: dict) -> dict:
    """Weights of every vision actor, from the description's seeds."""
    from paper_1802_06625_b200.cnn_weights import layer_params
    acts = {a["id"]: a for a in desc["actors"]}
    out = {}
    for aid in ("l1", "l2"):
        p = acts[aid]["params"]
        w, b = layer_params(p, 32, 25 * int(p["cin"]))
        out[aid] = (w, b, int(p["pad"]))
    p = acts["l3"]["params"]
    out["l3"] = layer_params(p, int(p["nout"]), int(p["nin"]))
    p = acts["join"]["params"]
    w4, b4 = layer_params({"seed": int(p["seed"])}, int(p["nhid"]), int(p["nin"]))
    w5, b5 = layer_params({"seed": int(p["seed"]) + 100}, int(p["nout"]), int(p["nhid"]))
    out["join"] = (w4, b4, w5, b5)
    out["marker"] = float(np.float32(p["marker"]))
    return out
