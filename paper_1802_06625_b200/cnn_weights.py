"""Deterministic weights of the vision example and their device layout.

The paper's adaptive DNN has no published weights; the
reference package replaces it with 8x8 matmuls.  Weights here
are He-normal from a seed (`he_normal`), so a graph description only carries
seeds and shapes (or explicit `weights`/`bias` lists).

`conv_device_layout` prepares a conv weight matrix W[cout][K] (K = 25*cin in
(ky, kx, ci) order) for the tcgen05 kernel: per 32-wide K chunk, the TF32
"hi" part (low 13 mantissa bits cleared) and the exact remainder "lo", each
as a 32x32 K-major UMMA operand in core-matrix order [row/8][k/4][row%8][k%4]
(csrc/pb_cnn.cu).
"""
from __future__ import annotations

import numpy as np

KC = 32


def he_normal(seed: int, rows: int, fan_in: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((rows, fan_in)) * np.sqrt(2.0 / fan_in)).astype(np.float32)


def small_bias(seed: int, rows: int) -> np.ndarray:
    rng = np.random.default_rng(seed + 7919)
    return (rng.standard_normal(rows) * 0.01).astype(np.float32)


def layer_params(params, rows: int, fan_in: int) -> tuple[np.ndarray, np.ndarray]:
    """Weights W[rows][fan_in] and bias[rows] from explicit lists
    (params["weights"], params["bias"]) or He-normal from params["seed"]."""
    if "weights" in params:
        w = np.asarray(params["weights"], dtype=np.float32).reshape(rows, fan_in)
        b = np.asarray(params.get("bias") or [0.0] * rows, dtype=np.float32)
        return w, b
    seed = int(params["seed"])
    return he_normal(seed, rows, fan_in), small_bias(seed, rows)


def tf32_split(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    bits = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    hi = (bits & np.uint32(0xFFFFE000)).view(np.float32)
    lo = (x.astype(np.float32) - hi).astype(np.float32)
    return hi, lo


def core_layout(tile: np.ndarray) -> np.ndarray:
    """[rows][KC] -> UMMA K-major no-swizzle order [row/8][k/4][row%8][k%4]."""
    rows = tile.shape[0]
    t = tile.reshape(rows // 8, 8, KC // 4, 4)          # [r8][r%8][k4][k%4]
    return np.ascontiguousarray(t.transpose(0, 2, 1, 3)).reshape(-1)


def conv_device_layout(w: np.ndarray) -> np.ndarray:
    """W[cout][K] -> per chunk [hi core][lo core], K zero-padded to 32."""
    cout, K = w.shape
    chunks = (K + KC - 1) // KC
    wp = np.zeros((cout, chunks * KC), np.float32)
    wp[:, :K] = w
    hi, lo = tf32_split(wp)
    out = []
    for c in range(chunks):
        out.append(core_layout(hi[:, c * KC:(c + 1) * KC]))
        out.append(core_layout(lo[:, c * KC:(c + 1) * KC]))
    return np.concatenate(out)
