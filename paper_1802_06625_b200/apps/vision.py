"""Adaptive CNN vision graph (the paper's "Adaptive Deep Neural Network",
PAPER.md:674-684, Fig. 9; work sizes :700) on the PRUNE graph model.

    src --frames--> select --d1--> l1 (conv5x5 3->32, ReLU, pool2)
                      |                -> l2 (conv5x5 32->32, ReLU, pool2)
                      |                -> l3 (dense 18432->100)
                      |                -> join.e1
                      +--d2 (bypass)--------------------> join.e2
    conf --ctl--> select, join;  join --logits--> sink

Shapes follow the paper: 96x96x3 fp32 frames, zero-padded by 6 so the first
conv gives 104x104 (pooled 52x52x32), the second 48x48 (pooled 24x24x32),
L3 has 18432*100 = 1.84M weights, token rate atr = 24 frames
per firing on every data channel (:680).  `join` is the paper's
"L3Relu-L5" stage: ReLU, a 100->64 hidden layer and 64->4 logits for the
processed path; bypassed frames get constant marker logits (:682).  The
configuration actor stays separate (the paper merges it into Select-Pad,
which the model forbids, model.py:241-242).  Weights are He-normal from
seeds (paper_1802_06625_b200/cnn_weights.py).  Tokens: NHWC fp32.
"""
from __future__ import annotations

from typing import Any

import numpy as np

H = W = 96
CIN = 3
FRAME_BYTES = H * W * CIN * 4
L1_OUT = (52, 52, 32)
L2_OUT = (24, 24, 32)
N_CLASSES = 4


def build_description(frames_per_firing: int = 24, policy: str = "alternate_policy",
                      input_path: str = "frames.bin", marker: float = -1.0) -> dict[str, Any]:
    R = frames_per_firing

    def port(pid, d, kind="srp"):
        return {"id": pid, "dir": d, "kind": kind, "rate": 1 if "control" in kind else R}

    conf_params: dict[str, Any] = {"length": 2}
    if policy == "fixed_policy":
        conf_params["element"] = 1
    l1b = L1_OUT[0] * L1_OUT[1] * L1_OUT[2] * 4
    l2b = L2_OUT[0] * L2_OUT[1] * L2_OUT[2] * 4
    actors = [
        {"id": "src", "kind": "static", "behavior": "file_source", "params": {"path": input_path},
         "ports": [port("out", "out")]},
        {"id": "conf", "kind": "config", "behavior": policy, "params": conf_params,
         "ports": [port("ctl", "out", "control_out")]},
        {"id": "select", "kind": "dynamic", "behavior": "route",
         "ports": [port("in", "in"), port("ctl", "in", "control_in"),
                   port("d1", "out", "drp"), port("d2", "out", "drp")]},
        {"id": "l1", "kind": "static", "behavior": "conv2d_relu_pool",
         "params": {"h": H, "w": W, "cin": CIN, "cout": 32, "pad": 6, "seed": 1},
         "ports": [port("in", "in"), port("out", "out")]},
        {"id": "l2", "kind": "static", "behavior": "conv2d_relu_pool",
         "params": {"h": 52, "w": 52, "cin": 32, "cout": 32, "pad": 0, "seed": 2},
         "ports": [port("in", "in"), port("out", "out")]},
        {"id": "l3", "kind": "static", "behavior": "dense",
         "params": {"nin": 24 * 24 * 32, "nout": 100, "seed": 3},
         "ports": [port("in", "in"), port("out", "out")]},
        {"id": "join", "kind": "dynamic", "behavior": "classify_merge",
         "params": {"nin": 100, "nhid": 64, "nout": N_CLASSES, "seed": 4, "marker": marker,
                    "bypass_port": "e2"},
         "ports": [port("ctl", "in", "control_in"), port("e1", "in", "drp"),
                   port("e2", "in", "drp"), port("out", "out")]},
        {"id": "sink", "kind": "static", "behavior": "null_sink", "ports": [port("in", "in")]},
    ]
    fifos = [
        {"id": "f_src", "src": "src.out", "dst": "select.in", "rate": R, "token_bytes": FRAME_BYTES},
        {"id": "c_select", "src": "conf.ctl", "dst": "select.ctl", "rate": 1, "token_bytes": 2},
        {"id": "c_join", "src": "conf.ctl", "dst": "join.ctl", "rate": 1, "token_bytes": 2},
        {"id": "f_l1", "src": "select.d1", "dst": "l1.in", "rate": R, "token_bytes": FRAME_BYTES},
        {"id": "f_l2", "src": "l1.out", "dst": "l2.in", "rate": R, "token_bytes": l1b},
        {"id": "f_l3", "src": "l2.out", "dst": "l3.in", "rate": R, "token_bytes": l2b},
        {"id": "f_chain", "src": "l3.out", "dst": "join.e1", "rate": R, "token_bytes": 400},
        {"id": "f_bypass", "src": "select.d2", "dst": "join.e2", "rate": R,
         "token_bytes": FRAME_BYTES},
        {"id": "f_out", "src": "join.out", "dst": "sink.in", "rate": R,
         "token_bytes": N_CLASSES * 4},
    ]
    table = [{"port": "conf.ctl", "drp": "select.d1", "element": 1},
             {"port": "conf.ctl", "drp": "join.e1", "element": 1},
             {"port": "conf.ctl", "drp": "select.d2", "element": 2},
             {"port": "conf.ctl", "drp": "join.e2", "element": 2}]
    return {"name": "vision", "actors": actors, "fifos": fifos,
            "control": {"value_lengths": {"conf.ctl": 2}, "table": table}}


def make_frames(seed: int, n_frames: int) -> np.ndarray:
    """Synthetic RGB frames, uniform [0, 1) fp32, NHWC (BASELINE config 3)."""
    return np.random.default_rng(seed).random((n_frames, H, W, CIN), dtype=np.float32)


def flops_per_frame() -> float:
    """Tensor-core work per processed frame (conv MACs x 2)."""
    l1 = 104 * 104 * 32 * 75 * 2
    l2 = 48 * 48 * 32 * 800 * 2
    l3 = 18432 * 100 * 2
    return float(l1 + l2 + l3)
