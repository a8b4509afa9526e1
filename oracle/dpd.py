"""ORACLE (test infrastructure only): numpy restatement of the DPD hot path.

Follows the reference package step by step:
  * subset_schedule  — SubsetPolicy.pick/_PolicyBase (behavior.py:202-218,
    248-256) with CPython `random` seeded by actor_seed (behavior.py:17-21),
    the same replay as pkg/tests/oracles.py:102-110
  * branch_taps      — predistortion.py:29-33
  * fir_block        — FirBranch.fire predistortion.py:51-65 (one numpy binary
    op at a time, float32 throughout, accumulators from +0, ascending taps)
  * branch_sum       — BranchSum.fire predistortion.py:72-83 (sorted port-id
    order, which is string order: e1, e10, e2, ...)
  * dpd_stream       — the sink stream the interpreter (interp.py:89-229)
    produces for the DPD graph: per block, route to the active branches
    (behavior.py:176-184), each branch filters with its own history of the
    input blocks it was routed, then the combiner sums.
"""
from __future__ import annotations

import random
import zlib

import numpy as np

TAPS = 10


def actor_seed(base, actor_id: str):
    if base is None:
        return None
    return (base ^ zlib.crc32(actor_id.encode())) & 0x7FFFFFFF


def subset_schedule(seed, blocks: int, length: int = 4, min_active: int = 2,
                    actor: str = "conf") -> list[set[int]]:
    s = actor_seed(seed, actor)
    rng = random.Random(s if s is not None else 0)
    sets = []
    for _ in range(blocks):
        size = rng.randint(min(min_active, length), length)
        sets.append(set(rng.sample(range(1, length + 1), size)))
    return sets


def control_tokens(active_sets: list[set[int]], length: int) -> np.ndarray:
    out = np.zeros((len(active_sets), length), dtype=np.uint8)
    for n, s in enumerate(active_sets):
        for k in s:
            out[n, k - 1] = 1
    return out


def branch_taps(k: int) -> tuple[np.ndarray, np.ndarray]:
    re = np.array([np.float32(0.05 * (k + 1) / (t + 1)) for t in range(TAPS)], dtype=np.float32)
    im = np.array([np.float32(0.002 * (k + 1) * (t - 4.5)) for t in range(TAPS)],
                  dtype=np.float32)
    return re, im


def fir_block(xr, xi, cr, ci, hr, hi):
    """Returns (yr, yi, new_hr, new_hi); all float32 (predistortion.py:51-65)."""
    B = xr.shape[-1]
    fr = np.concatenate([hr, xr])
    fi = np.concatenate([hi, xi])
    acc_r = np.zeros(B, dtype=np.float32)
    acc_i = np.zeros(B, dtype=np.float32)
    for t in range(TAPS):
        seg_r = fr[TAPS - 1 - t:TAPS - 1 - t + B]
        seg_i = fi[TAPS - 1 - t:TAPS - 1 - t + B]
        acc_r = acc_r + (cr[t] * seg_r - ci[t] * seg_i)
        acc_i = acc_i + (cr[t] * seg_i + ci[t] * seg_r)
    return acc_r, acc_i, fr[B:].copy(), fi[B:].copy()


def combiner_order(branches: int) -> list[int]:
    """Branch indices (1-based) in sorted(port id) order of `combine`."""
    return [int(p[1:]) for p in sorted(f"e{k}" for k in range(1, branches + 1))]


def dpd_stream(x: np.ndarray, active_sets: list[set[int]], branches: int,
               return_branches: bool = False):
    """x: (blocks, 2, B) float32 planar input -> (blocks, 2, B) sink stream."""
    blocks, _, B = x.shape
    taps = [branch_taps(k) for k in range(branches)]
    hist = [(np.zeros(TAPS - 1, np.float32), np.zeros(TAPS - 1, np.float32))
            for _ in range(branches)]
    out = np.zeros((blocks, 2, B), dtype=np.float32)
    per_branch = {k: [] for k in range(1, branches + 1)}
    order = combiner_order(branches)
    for n in range(blocks):
        ys = {}
        for k in range(1, branches + 1):
            if k not in active_sets[n]:
                continue
            cr, ci = taps[k - 1]
            hr, hi = hist[k - 1]
            yr, yi, hr, hi = fir_block(x[n, 0], x[n, 1], cr, ci, hr, hi)
            hist[k - 1] = (hr, hi)
            ys[k] = (yr, yi)
            per_branch[k].append((n, np.stack([yr, yi])))
        acc_r = np.zeros(B, dtype=np.float32)
        acc_i = np.zeros(B, dtype=np.float32)
        for k in order:
            if k in ys:
                acc_r = acc_r + ys[k][0]
                acc_i = acc_i + ys[k][1]
        out[n, 0], out[n, 1] = acc_r, acc_i
    if return_branches:
        return out, per_branch
    return out


def firing_counts(active_sets: list[set[int]], branches: int) -> dict[str, int]:
    n = len(active_sets)
    counts = {"src": n, "conf": n, "split": n, "combine": n, "sink": n}
    for k in range(1, branches + 1):
        counts[f"b{k}"] = sum(1 for s in active_sets if k in s)
    return counts
