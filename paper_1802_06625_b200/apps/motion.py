"""Frame-difference motion detection (the reference app apps/motion.py:74-108),
parameterised by frame side.

    src -> blur -> (f_cur, f_prev: one-frame delay) -> detect -> clean -> sink

One token is one side x side 8-bit frame.  f_prev carries one initial delay
token (a zero frame), so the first firing of `detect` compares against
black; on the device that channel is a ring one chunk longer whose producer
writes one chunk ahead of its consumer (engine.py, pb_span_ref.offset).
Actors: gauss_blur, frame_diff_threshold (threshold 16), plus_median -- all
device image kernels (csrc/pb_image.cu), integer and bit-exact.
"""
from __future__ import annotations

import random
from typing import Any

SIDE = 64


def build_description(side: int = SIDE, input_path: str = "input.bin",
                      threshold: int = 16) -> dict[str, Any]:
    fb = side * side

    def srp(pid, direction):
        return {"id": pid, "dir": direction, "kind": "srp", "rate": 1}

    return {
        "name": "motion",
        "actors": [
            {"id": "src", "kind": "static", "behavior": "file_source",
             "params": {"path": input_path}, "ports": [srp("out", "out")]},
            {"id": "blur", "kind": "static", "behavior": "gauss_blur",
             "ports": [srp("in", "in"), srp("out", "out")]},
            {"id": "detect", "kind": "static", "behavior": "frame_diff_threshold",
             "params": {"threshold": threshold},
             "ports": [srp("cur", "in"), srp("prev", "in"), srp("out", "out")]},
            {"id": "clean", "kind": "static", "behavior": "plus_median",
             "ports": [srp("in", "in"), srp("out", "out")]},
            {"id": "sink", "kind": "static", "behavior": "null_sink", "ports": [srp("in", "in")]},
        ],
        "fifos": [
            {"id": "f_src", "src": "src.out", "dst": "blur.in", "rate": 1, "delay": 0,
             "token_bytes": fb},
            {"id": "f_cur", "src": "blur.out", "dst": "detect.cur", "rate": 1, "delay": 0,
             "token_bytes": fb},
            {"id": "f_prev", "src": "blur.out", "dst": "detect.prev", "rate": 1, "delay": 1,
             "token_bytes": fb},
            {"id": "f_mask", "src": "detect.out", "dst": "clean.in", "rate": 1, "delay": 0,
             "token_bytes": fb},
            {"id": "f_out", "src": "clean.out", "dst": "sink.in", "rate": 1, "delay": 0,
             "token_bytes": fb},
        ],
        "control": {},
    }


def make_input(seed: int, frames: int, side: int = SIDE) -> bytes:
    """apps/motion.py:111-112 (uniform random bytes, CPython random)."""
    return random.Random(seed).randbytes(frames * side * side)
