"""ORACLE (test infrastructure only): numpy restatement of the motion app.

  * blur       — GaussBlur.fire apps/motion.py:32-47: int32 rows pass over
                 columns d..d+side-4 with k = (1 4 6 4 1), then columns, >> 8,
                 2-pixel border copied
  * diff       — FrameDiffThreshold.fire :50-58: 255 where |cur-prev| > thr
  * median     — PlusMedian.fire :61-71: middle of the sorted (centre, up,
                 down, left, right), 1-pixel border copied
  * motion_stream — the interpreter's sink stream (pkg/tests/oracles.py:59-67
                 restates the same): per frame, median(diff(blur_k, blur_{k-1}))
                 with blur_{-1} = the zero delay token
Pinned by tests/golden/motion.json (the reference app run through
tokenflow.interp.interpret) in tests/test_oracle.py.
"""
from __future__ import annotations

import numpy as np

KERNEL = (1, 4, 6, 4, 1)


def blur(frame: np.ndarray) -> np.ndarray:
    a = frame.astype(np.int32)
    side = a.shape[0]
    w = side - 4
    rows = np.zeros((side, w), dtype=np.int32)
    for d, k in enumerate(KERNEL):
        rows += k * a[:, d:d + w]
    cols = np.zeros((w, w), dtype=np.int32)
    for d, k in enumerate(KERNEL):
        cols += k * rows[d:d + w, :]
    out = a.copy()
    out[2:side - 2, 2:side - 2] = cols >> 8
    return out.astype(np.uint8)


def diff(cur: np.ndarray, prev: np.ndarray, threshold: int = 16) -> np.ndarray:
    return np.where(np.abs(cur.astype(np.int32) - prev.astype(np.int32)) > threshold,
                    255, 0).astype(np.uint8)


def median(a: np.ndarray) -> np.ndarray:
    c = a[1:-1, 1:-1]
    stack = np.stack([c, a[:-2, 1:-1], a[2:, 1:-1], a[1:-1, :-2], a[1:-1, 2:]])
    out = a.copy()
    out[1:-1, 1:-1] = np.sort(stack, axis=0)[2]
    return out


def motion_stream(data: bytes, frames: int, side: int = 64, threshold: int = 16) -> bytes:
    x = np.frombuffer(data, dtype=np.uint8)[:frames * side * side].reshape(frames, side, side)
    prev = np.zeros((side, side), dtype=np.uint8)
    out = bytearray()
    for k in range(frames):
        cur = blur(x[k])
        out += median(diff(cur, prev, threshold)).tobytes()
        prev = cur
    return bytes(out)
