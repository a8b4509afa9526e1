"""The reference's adaptive-bypass matrix pipeline (apps/bypass.py:69-132):

    src -> fork (route) -> l1 -> l2 -> l3 (8x8 matmul each) -> join (path_merge) -> sink
                        \\-------------- bypass ---------------/

`conf` (alternate_policy, length 2) sends element 1 (the chain) and element 2
(the bypass) on alternate firings; `join` adds MARKER to bypassed matrices.
One token is one 8x8 float32 matrix.  Every actor is a device kernel
(matmul_kernel, path_merge_kernel; route aliases its input span).
"""
from __future__ import annotations

import random
from typing import Any

import numpy as np

N = 8
TOKEN_BYTES = N * N * 4
MARKER = 0.5


def layer_weights(layer: int) -> list[float]:
    """apps/bypass.py:26-32: exact float32 weights."""
    return [float(np.float32(0.1 + 0.05 * layer - 0.01 * i + 0.02 * k))
            for i in range(N) for k in range(N)]


def build_description(input_path: str = "input.bin") -> dict[str, Any]:
    def port(pid, direction, kind="srp"):
        return {"id": pid, "dir": direction, "kind": kind, "rate": 1}

    actors: list[dict[str, Any]] = [
        {"id": "src", "kind": "static", "behavior": "file_source",
         "params": {"path": input_path}, "ports": [port("out", "out")]},
        {"id": "conf", "kind": "config", "behavior": "alternate_policy", "params": {"length": 2},
         "ports": [port("ctl", "out", "control_out")]},
        {"id": "fork", "kind": "dynamic", "behavior": "route",
         "ports": [port("in", "in"), port("ctl", "in", "control_in"), port("d1", "out", "drp"),
                   port("d2", "out", "drp")]},
        {"id": "join", "kind": "dynamic", "behavior": "path_merge",
         "params": {"marker": MARKER, "bypass_port": "e2"},
         "ports": [port("ctl", "in", "control_in"), port("e1", "in", "drp"),
                   port("e2", "in", "drp"), port("out", "out")]},
        {"id": "sink", "kind": "static", "behavior": "null_sink", "ports": [port("in", "in")]},
    ]
    for layer in (1, 2, 3):
        actors.append({"id": f"l{layer}", "kind": "static", "behavior": "matmul",
                       "params": {"w": layer_weights(layer)},
                       "ports": [port("in", "in"), port("out", "out")]})

    def fifo(fid, src, dst, tb=TOKEN_BYTES):
        return {"id": fid, "src": src, "dst": dst, "rate": 1, "delay": 0, "token_bytes": tb}

    fifos = [fifo("f_src", "src.out", "fork.in"), fifo("c_fork", "conf.ctl", "fork.ctl", 2),
             fifo("c_join", "conf.ctl", "join.ctl", 2), fifo("f_l1", "fork.d1", "l1.in"),
             fifo("f_l2", "l1.out", "l2.in"), fifo("f_l3", "l2.out", "l3.in"),
             fifo("f_chain", "l3.out", "join.e1"), fifo("f_bypass", "fork.d2", "join.e2"),
             fifo("f_out", "join.out", "sink.in")]
    table = [{"port": "conf.ctl", "drp": "fork.d1", "element": 1},
             {"port": "conf.ctl", "drp": "join.e1", "element": 1},
             {"port": "conf.ctl", "drp": "fork.d2", "element": 2},
             {"port": "conf.ctl", "drp": "join.e2", "element": 2}]
    return {"name": "bypass", "actors": actors, "fifos": fifos,
            "control": {"value_lengths": {"conf.ctl": 2}, "table": table}}


def make_input(seed: int, mats: int) -> bytes:
    """apps/bypass.py:135-141: CPython-random uniform(-1, 1) matrices as float32."""
    rng = random.Random(seed)
    return b"".join(np.array([rng.uniform(-1.0, 1.0) for _ in range(N * N)],
                             dtype=np.float32).tobytes() for _ in range(mats))
