"""Round-to-nearest quantization primitives — oracle (TEST INFRASTRUCTURE).

* Activations, per token symmetric INT4 (Stage 2b): "the row scales are
  computed by dividing the maximum absolute value of each token by 7 (largest
  representable number in INT4). We then divide each row to its corresponding scale
  and round the result to its nearest integer."  Clip ratio 0.9.
* Weights, per output channel ("per-column") symmetric RTN with the clip ratio from
  "a linear search over the squared error".
* INT4 nibble packing of the "sub-byte format".

Readings: Z7 round half to even; Z8 codes in [-7, 7]; Z9 scale =
clip * amax / 7, then clamp; Z10 all-zero row -> scale 1, codes 0; scales stored as
fp32 (Z11); Z13 weight clip grid 1.00, 0.99, ..., 0.40 with ties toward the larger
ratio; non-finite rows -> scale NaN, codes 0 (SURVEY §8b "Non-finite input").
"""
from __future__ import annotations

import numpy as np

QMAX_SYM4 = 7  # P:233 "7 (largest representable number in INT4)"


def _rne(v: np.ndarray) -> np.ndarray:
    """Round half to even (Z7): numpy.rint is IEEE round-to-nearest-even."""
    return np.rint(v)


def clip32(clip_ratio: float) -> float:
    """The clip ratio as the C ABI receives it (an fp32), widened to fp64."""
    c = float(np.float32(clip_ratio))
    if not (0.0 < c <= 1.0):
        raise ValueError(f"clip ratio must lie in (0, 1], got {clip_ratio}")
    return c


def quantize_sym_rows(y: np.ndarray, clip_ratio: float = 0.9, qmax: int = QMAX_SYM4):
    """Per-row symmetric RTN (clip P:249).

    For each row y (fp64): a = max_k |y_k| (NaN propagates);
      a == 0            -> scale 1, codes 0                       (Z10)
      a not finite      -> scale NaN, codes 0                     (non-finite reading)
      otherwise         s = fp32(clip * a / qmax);  c = clamp(RNE(y / s), -qmax, qmax).
    Returns (codes int64 [rows, K], scale float32 [rows])."""
    y = np.asarray(y, dtype=np.float64)
    if y.ndim != 2:
        raise ValueError("quantize_sym_rows expects a 2-D [rows, K] array")
    clip = clip32(clip_ratio)
    amax = np.max(np.abs(y), axis=1) if y.shape[1] else np.zeros(y.shape[0])
    codes = np.zeros(y.shape, dtype=np.int64)
    scale = np.ones(y.shape[0], dtype=np.float32)
    for r in range(y.shape[0]):
        a = amax[r]
        if a == 0.0:
            continue
        if not np.isfinite(a):
            scale[r] = np.nan
            continue
        s32 = np.float32(clip * a / qmax)
        scale[r] = s32
        codes[r] = np.clip(_rne(y[r] / np.float64(s32)), -qmax, qmax).astype(np.int64)
    return codes, scale


def quantize_sym_groups(y: np.ndarray, group: int = 128, clip_ratio: float = 0.9, qmax: int = QMAX_SYM4):
    """Group-wise symmetric RTN ("group-wise quantization ... group size
    128"): every run of `group` consecutive elements of a row is quantized by the rule of
    quantize_sym_rows with its own scale.  Returns (codes int64 [rows, K], scale float32
    [rows, K / group])."""
    y = np.asarray(y, dtype=np.float64)
    rows, k = y.shape
    if group <= 0 or k % group:
        raise ValueError(f"group {group} must divide K = {k}")
    codes, scale = quantize_sym_rows(y.reshape(rows * (k // group), group), clip_ratio, qmax)
    return codes.reshape(rows, k), scale.reshape(rows, k // group)


def dequantize_sym_groups(codes: np.ndarray, scale: np.ndarray) -> np.ndarray:
    """x^ = c * s_g for the group g of each element."""
    codes = np.asarray(codes, dtype=np.float64)
    g = codes.shape[1] // scale.shape[1]
    return codes * np.repeat(np.asarray(scale, dtype=np.float64), g, axis=1)


def dequantize_sym_rows(codes: np.ndarray, scale: np.ndarray) -> np.ndarray:
    """x^ = c * s."""
    return np.asarray(codes, dtype=np.float64) * np.asarray(scale, dtype=np.float64)[:, None]


def pack_int4(codes: np.ndarray) -> np.ndarray:
    """Two's-complement nibbles, two per byte, low nibble = even index (D1/D2):
    byte j = (c[2j] & 0xF) | ((c[2j+1] & 0xF) << 4).  Last axis must be even."""
    c = np.asarray(codes, dtype=np.int64)
    if c.shape[-1] % 2:
        raise ValueError("packing needs an even number of codes along the last axis")
    if np.any(c < -8) or np.any(c > 15):
        raise ValueError("code out of 4-bit range")
    lo = c[..., 0::2] & 0xF
    hi = c[..., 1::2] & 0xF
    return (lo | (hi << 4)).astype(np.uint8)


def unpack_int4_signed(packed: np.ndarray) -> np.ndarray:
    """Inverse of pack_int4 for signed codes in [-8, 7]."""
    b = np.asarray(packed, dtype=np.int64)
    lo = b & 0xF
    hi = (b >> 4) & 0xF
    lo = np.where(lo >= 8, lo - 16, lo)
    hi = np.where(hi >= 8, hi - 16, hi)
    out = np.empty(b.shape[:-1] + (b.shape[-1] * 2,), dtype=np.int64)
    out[..., 0::2] = lo
    out[..., 1::2] = hi
    return out


def unpack_int4_unsigned(packed: np.ndarray) -> np.ndarray:
    """Inverse of pack_int4 for unsigned codes in [0, 15] (KV cache, D4)."""
    b = np.asarray(packed, dtype=np.int64)
    out = np.empty(b.shape[:-1] + (b.shape[-1] * 2,), dtype=np.int64)
    out[..., 0::2] = b & 0xF
    out[..., 1::2] = (b >> 4) & 0xF
    return out


CLIP_GRID = tuple((100 - i) / 100.0 for i in range(61))  # 1.00 .. 0.40 (Z13)


def rtn_weight_quantize(w: np.ndarray, qmax: int = QMAX_SYM4):
    """Per-output-channel symmetric RTN with clip line search (Z13).

    w: [N, K] (nn.Linear [out, in] layout; one "column" of the paper's [in, out]
    matrix is one row here).  For each channel n and each clip c in CLIP_GRID
    (descending): s = fp32(c * max|w_n| / qmax), q = clamp(RNE(w_n / s)),
    err = sum (w_n - q s)^2; keep the first (largest c) strict minimum.
    Returns (codes int64 [N, K], scale float32 [N], chosen clip float64 [N])."""
    w = np.asarray(w, dtype=np.float64)
    n_out = w.shape[0]
    codes = np.zeros(w.shape, dtype=np.int64)
    scale = np.ones(n_out, dtype=np.float32)
    chosen = np.ones(n_out)
    amax = np.max(np.abs(w), axis=1)
    for n in range(n_out):
        if amax[n] == 0:
            continue
        best = None
        for c in CLIP_GRID:
            s32 = np.float32(c * amax[n] / qmax)
            q = np.clip(_rne(w[n] / np.float64(s32)), -qmax, qmax)
            err = float(np.sum((w[n] - q * np.float64(s32)) ** 2))
            if best is None or err < best[0]:
                best = (err, c, s32, q)
        _, chosen[n], scale[n], q = best
        codes[n] = q.astype(np.int64)
    return codes, scale, chosen
