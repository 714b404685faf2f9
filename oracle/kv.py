"""Quantized KV cache Init (prefill) — oracle (TEST INFRASTRUCTURE).

* Stage 1d (Eqs. 13-14): online per-head H_{d_h} on post-RoPE Q and K.
* Stage 2c: the cache is quantized to low bit-width.
* Setup: "We quantize the KV caches using asymmetric quantization with a group
  size 128 with a constant clipping ratio of 0.95."
* App. performance: routine "Init" builds the cache from the prefill K, V.

Readings: Z14 range forced to include 0: lo = clip*min(min g, 0),
hi = clip*max(max g, 0), s = (hi - lo)/15, z = clamp(RNE(-lo/s), 0, 15),
c = clamp(RNE(x/s) + z, 0, 15); Z10 hi == lo -> s = 1, z = 0, codes 0; Z15 fp32 scale
+ uint8 zero per (token, head); Z16 V is not rotated online (W_v carries H);
the rotated Q is stored back as fp16 (RNE).
"""
from __future__ import annotations

import numpy as np

from .hadamard import hadamard
from .quant import clip32, pack_int4

QMAX_ASYM4 = 15


def quantize_asym_groups(x: np.ndarray, clip_ratio: float = 0.95, qmax: int = QMAX_ASYM4):
    """Asymmetric RTN per group = last axis (Z14).

    x: [..., G] fp64.  Returns (codes int64 [..., G] in [0, qmax],
    scale float32 [...], zero int64 [...])."""
    x = np.asarray(x, dtype=np.float64)
    clip = clip32(clip_ratio)
    flat = x.reshape(-1, x.shape[-1])
    codes = np.zeros(flat.shape, dtype=np.int64)
    scale = np.ones(flat.shape[0], dtype=np.float32)
    zero = np.zeros(flat.shape[0], dtype=np.int64)
    for r in range(flat.shape[0]):
        g = flat[r]
        lo = clip * min(float(np.min(g)), 0.0)
        hi = clip * max(float(np.max(g)), 0.0)
        if not (np.isfinite(lo) and np.isfinite(hi)):
            scale[r] = np.nan
            continue
        if hi == lo:
            continue
        s32 = np.float32((hi - lo) / qmax)
        s = np.float64(s32)
        z = int(np.clip(np.rint(-lo / s), 0, qmax))
        scale[r] = s32
        zero[r] = z
        codes[r] = np.clip(np.rint(g / s) + z, 0, qmax).astype(np.int64)
    return (codes.reshape(x.shape), scale.reshape(x.shape[:-1]), zero.reshape(x.shape[:-1]))


def dequantize_asym(codes, scale, zero) -> np.ndarray:
    """x^ = (c - z) * s."""
    return (np.asarray(codes, dtype=np.float64) - np.asarray(zero, dtype=np.float64)[..., None]) \
        * np.asarray(scale, dtype=np.float64)[..., None]


def kv_init(k: np.ndarray, v: np.ndarray, q: np.ndarray | None = None,
            rotate_k: bool = True, rotate_v: bool = False, clip_ratio: float = 0.95):
    """KV cache Init for one prefill batch.

    k, v: [T, n_kv, d_h] (fp16 values as fp64); q: optional [T, n_q, d_h].
    Returns dict with packed codes [T, n_kv, d_h/2] (unsigned nibbles, low = even
    index), fp32 scales [T, n_kv], uint8 zeros [T, n_kv] for K and V, and the rotated
    q' = fp16(H^ q) per head (or None)."""
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    d_h = k.shape[-1]
    h = hadamard(d_h)
    kr = k @ h.T if rotate_k else k          # k'_h = H^ k_h  (Eq. 14, column convention)
    vr = v @ h.T if rotate_v else v
    kc, ks, kz = quantize_asym_groups(kr, clip_ratio)
    vc, vs, vz = quantize_asym_groups(vr, clip_ratio)
    out = {
        "k_codes": pack_int4(kc), "k_scale": ks, "k_zero": kz.astype(np.uint8),
        "v_codes": pack_int4(vc), "v_scale": vs, "v_zero": vz.astype(np.uint8),
        "k_rot": kr, "v_rot": vr,
        "q_rot": None,
    }
    if q is not None:
        out["q_rot"] = (np.asarray(q, dtype=np.float64) @ h.T).astype(np.float16)  # Eq. 13
    return out
