"""Deterministic weights of the vision example and their device layout.

The paper's adaptive DNN has no published weights; the
reference package replaces it with 8x8 matmuls.  Weights here
are He-normal from a seed (`he_normal`), so a graph description only carries
seeds and shapes (or explicit `weights`/`bias` lists).

`conv_device_layout` prepares a conv weight matrix W[cout][K] (K = 25*cin in
(ky, kx, ci) order) for the tcgen05 kernel: per 16-wide K-step, the bf16
"hi" part and the bf16-rounded remainder "lo" stacked as one 64-row UMMA B
operand in core-matrix order [row/8][k/8][row%8][k%8] (csrc/pb_cnn.cu).
"""
from __future__ import annotations

import numpy as np

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


def bf16_rn(x: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (round-to-nearest-even), returned as fp32 values."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def bf16_split(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """x = hi + lo + O(2^-17 |x|), hi and lo bf16 (the kernel's converter)."""
    x = np.asarray(x, dtype=np.float32)
    hi = bf16_rn(x)
    lo = bf16_rn((x - hi).astype(np.float32))
    return hi, lo


def conv_steps(w: np.ndarray, cin: int) -> np.ndarray:
    """W[32][25*cin] ((ky,kx,ci) order) -> the kernel's K-steps [steps][32][16].
    cin == 3: step ky holds (kx, ci) at index kx*3+ci (15 used, 1 zero);
    cin % 16 == 0: step (ky, kx, kc) holds channels 16kc..16kc+15."""
    cout = w.shape[0]
    wt = np.asarray(w, np.float32).reshape(cout, 5, 5, cin)
    if cin == 3:
        out = np.zeros((5, cout, 16), np.float32)
        out[:, :, :15] = wt.reshape(cout, 5, 15).transpose(1, 0, 2)
        return out
    if cin % 16:
        raise ValueError("conv: Cin must be 3 or a multiple of 16")
    kc = cin // 16
    return np.ascontiguousarray(
        wt.reshape(cout, 25, kc, 16).transpose(1, 2, 0, 3)).reshape(25 * kc, cout, 16)


def conv_device_layout(w: np.ndarray, cin: int) -> np.ndarray:
    """Per K-step a 2 KB UMMA B operand [wh; wl] (64 rows x 16 bf16) in the
    K-major no-swizzle core layout [row/8][kblock][row%8][8] (csrc/pb_cnn.cu).
    Returned as uint16 bf16 bits."""
    steps = conv_steps(w, cin)
    hi, lo = bf16_split(steps)
    both = np.concatenate([hi, lo], axis=1)                   # [S][64][16]
    bits = (both.view(np.uint32) >> 16).astype(np.uint16)
    S = bits.shape[0]
    core = bits.reshape(S, 8, 8, 2, 8).transpose(0, 1, 3, 2, 4)   # [S][r/8][kb][r%8][8]
    return np.ascontiguousarray(core).reshape(-1)


DENSE_N = 112   # padded outputs per precision half (csrc/pb_cnn.cu kDN)


def dense_device_layout(w: np.ndarray) -> np.ndarray:
    """W[nout][nin] -> per 16-wide K-step a UMMA B operand of 224 rows
    [wh (nout, zero-padded to 112); wl (same)] x 16 bf16 in the K-major
    no-swizzle core layout [row/8][kblock][row%8][8]; steps are contiguous, so
    a 64-wide K chunk is one 28 KB block.  Returned as uint16 bf16 bits."""
    nout, nin = w.shape
    if nout > DENSE_N or nin % 64:
        raise ValueError("dense: nout <= 112 and nin a multiple of 64")
    hi, lo = bf16_split(w)
    rows = np.zeros((2 * DENSE_N, nin), np.float32)
    rows[:nout] = hi
    rows[DENSE_N:DENSE_N + nout] = lo
    bits = (rows.view(np.uint32) >> 16).astype(np.uint16)
    S = nin // 16
    core = bits.reshape(2 * DENSE_N // 8, 8, S, 2, 8).transpose(2, 0, 3, 1, 4)
    return np.ascontiguousarray(core).reshape(-1)


# int8-limb layer (csrc/pb_conv_rows.cu, RowCfg<32, true>): quantisation ranges
X_LIMIT = 32639   # |X| of an activation (per frame: X = rint(x * 32639 / max|x|))
W_LIMIT = 32511   # |W| of a weight (per output channel: W = rint(w / wdq))


def limbs(v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Signed 16-bit integers -> (h, l), v = 256 h + l, both in [-128, 127]."""
    v = np.asarray(v, np.int64)
    h = (v + 128) >> 8
    return h, v - 256 * h


def conv_quant_weights(w: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """W[cout][K] -> (integer weights [cout][K] with |W| <= W_LIMIT, the float32
    per-channel dequantisation factors wdq = max|w| / W_LIMIT)."""
    w = np.asarray(w, np.float32)
    wdq = (np.abs(w).max(axis=1) / np.float32(W_LIMIT)).astype(np.float32)
    scale = np.where(wdq > 0, 1.0 / np.maximum(wdq.astype(np.float64), 1e-300), 0.0)
    q = np.rint(w.astype(np.float64) * scale[:, None]).astype(np.int64)
    return np.clip(q, -W_LIMIT, W_LIMIT), wdq


def conv_device_layout_i8(w: np.ndarray, cin: int) -> np.ndarray:
    """The int8-limb layer's weights (cin = 32): per 16-channel K-step (ky, kx,
    half) a 2 KB UMMA B operand of 64 rows x 32 int8 -- rows 0-31 [wh | 0] (the
    "hi" accumulator columns), rows 32-63 [wl | wh] ("mid") -- against the A
    operand [xh | xl], in the K-major no-swizzle core layout
    [row/8][kblock][row%8][16]; then the 32 float32 factors wdq.  As uint8."""
    if cin % 16:
        raise ValueError("conv int8 limbs: Cin must be a multiple of 16")
    q, wdq = conv_quant_weights(w)
    steps = conv_steps(q.astype(np.float32), cin).astype(np.int64)   # [S][32][16] exact
    wh, wl = limbs(steps)
    S, cout = steps.shape[0], steps.shape[1]
    rows = np.zeros((S, 2 * cout, 32), np.int8)
    rows[:, :cout, :16] = wh
    rows[:, cout:, :16] = wl
    rows[:, cout:, 16:] = wh
    core = rows.reshape(S, 2 * cout // 8, 8, 2, 16).transpose(0, 1, 3, 2, 4)
    return np.concatenate([np.ascontiguousarray(core).reshape(-1).view(np.uint8),
                           wdq.view(np.uint8)])


def conv_i8_reference(x: np.ndarray, w: np.ndarray, b: np.ndarray, pad: int) -> np.ndarray:
    """The int8-limb layer's arithmetic on the CPU (float64 where the device
    sums exactly in s32): per frame X = rint(x * q), q = X_LIMIT / max|x| in
    float32 and the product exact (the kernel's FFMA rounding), limbs of X
    and of the quantised weights, hi = sum xh wh, mid = sum (xh wl + xl wh),
    y = (256 hi + mid) * 256 * max|x| / X_LIMIT * wdq, bias, ReLU, 2x2 max."""
    F, H, W, Cin = x.shape
    x = np.asarray(x, np.float32)
    mx = np.abs(x.reshape(F, -1)).max(axis=1).astype(np.float32)
    q = np.where(mx > 0, np.float32(X_LIMIT) / np.maximum(mx, np.float32(1e-30)),
                 np.float32(0)).astype(np.float32)
    # the device rounds the exact product (one FFMA into a 2^23 magic number)
    X = np.rint(x.astype(np.float64) * q.astype(np.float64)[:, None, None, None]).astype(np.int64)
    xh, xl = limbs(X)
    qw, wdq = conv_quant_weights(w)
    wh, wl = limbs(qw)
    Ho, Wo = H + 2 * pad - 4, W + 2 * pad - 4

    def cols(a):
        ap = np.pad(a.astype(np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0)))
        c = np.empty((F, Ho, Wo, 25 * Cin))
        for ky in range(5):
            for kx in range(5):
                t = ky * 5 + kx
                c[..., t * Cin:(t + 1) * Cin] = ap[:, ky:ky + Ho, kx:kx + Wo, :]
        return c
    ch, cl = cols(xh), cols(xl)
    hi = ch @ wh.T.astype(np.float64)
    mid = ch @ wl.T.astype(np.float64) + cl @ wh.T.astype(np.float64)
    xdq = (mx.astype(np.float64) * (256.0 / X_LIMIT))[:, None, None, None]
    y = (256.0 * hi + mid) * xdq * wdq.astype(np.float64)
    y = np.maximum(y + b, 0.0)
    return y.reshape(F, Ho // 2, 2, Wo // 2, 2, -1).max(axis=(2, 4))
