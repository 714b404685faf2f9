"""Quantized KV cache Append + Decode — oracle (TEST INFRASTRUCTURE).

The paper's decoding routines: "2) Append: During decoding, this routine is called
first to quantize the current keys and values and append them to the cache.  3) Decode:
Finally, this routine is called during decoding with the current query vector.  The routine
computes the attention output using a quantized implementation of flash attention which can
load the quantized cache and compute the final value vector."  Benchmarked for one new token
per sequence on a cache of 2047 tokens (tab:QAttention_bench).

What is computed (fp64):
* Append: the new token's K, Q get RoPE at their position (reading Z22: rounded to
  fp16), then exactly `kv.kv_init` on that one token (per-head H on K and Q, Eqs. 13-14;
  asymmetric INT4 K/V, Z14) written at cache row `position`.
* Decode: standard softmax attention of the (rotated) query against the DEQUANTIZED cache,
  x^ = (c - z) * s (Z14), rows 0 .. seq_len-1:
      score_j = <q, k^_j> * sm_scale,   p = softmax(score),   o = sum_j p_j v^_j,
  with grouped-query attention: query head h reads KV head h // (n_q / n_kv).
  Since Q and K are rotated by the same orthogonal H^, the scores equal those of the
  unrotated vectors (pin P14); V is not rotated online (Z16), so o is in V's space.
  Output rounded to fp16 (RNE).  Reading Z24: sm_scale = 1/sqrt(head_dim) (the standard
  scaled dot product; the paper does not restate it).
"""
from __future__ import annotations

import numpy as np

from .glue import rope
from .kv import dequantize_asym, kv_init


def kv_append(cache: dict, k_new, v_new, q_new, positions, theta: float = 10000.0, clip_ratio: float = 0.95):
    """Append one token per sequence.  cache: dict of arrays
    k_codes/v_codes int64 [B, S_max, n_kv, d] (unpacked codes), k_scale/v_scale float32
    [B, S_max, n_kv], k_zero/v_zero int64 [B, S_max, n_kv]; modified in place.
    k_new, v_new: [B, n_kv, d] pre-RoPE fp16 values; q_new: [B, n_q, d] pre-RoPE.
    positions: [B] row of the new token in each sequence (= its RoPE position).
    Returns the rotated query fp16(H^ fp16(rope(q))) [B, n_q, d]."""
    positions = np.asarray(positions, dtype=np.int64)
    kr = rope(np.asarray(k_new, np.float64), positions).astype(np.float16)  # Z22
    qr = rope(np.asarray(q_new, np.float64), positions).astype(np.float16)
    out = kv_init(kr, np.asarray(v_new, np.float64), qr, clip_ratio=clip_ratio)
    from .quant import unpack_int4_unsigned
    kc = unpack_int4_unsigned(out["k_codes"])
    vc = unpack_int4_unsigned(out["v_codes"])
    for b, pos in enumerate(positions):
        cache["k_codes"][b, pos] = kc[b]
        cache["v_codes"][b, pos] = vc[b]
        cache["k_scale"][b, pos] = out["k_scale"][b]
        cache["v_scale"][b, pos] = out["v_scale"][b]
        cache["k_zero"][b, pos] = out["k_zero"][b]
        cache["v_zero"][b, pos] = out["v_zero"][b]
    return out["q_rot"]


def attention_reference(q, k, v, seq_lens, sm_scale: float | None = None) -> np.ndarray:
    """Plain softmax attention, fp64: q [B, n_q, d], k, v [B, S, n_kv, d] (already real-valued),
    rows 0 .. seq_lens[b]-1 of sequence b.  Returns fp64 [B, n_q, d]."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    B, n_q, d = q.shape
    n_kv = k.shape[2]
    group = n_q // n_kv
    scale = 1.0 / np.sqrt(d) if sm_scale is None else sm_scale
    out = np.zeros((B, n_q, d))
    for b in range(B):
        L = int(seq_lens[b])
        for h in range(n_q):
            kh = k[b, :L, h // group]          # [L, d]
            s = kh @ q[b, h] * scale            # [L]
            p = np.exp(s - s.max())
            p /= p.sum()
            out[b, h] = p @ v[b, :L, h // group]
    return out


def decode_attention(q_rot, cache: dict, seq_lens, sm_scale: float | None = None) -> np.ndarray:
    """Decode: attention of the rotated query against the dequantized INT4 cache.
    q_rot fp16 [B, n_q, d]; cache as in kv_append (unpacked codes).  Returns fp16 [B, n_q, d]."""
    k_hat = dequantize_asym(cache["k_codes"], cache["k_scale"], cache["k_zero"])
    v_hat = dequantize_asym(cache["v_codes"], cache["v_scale"], cache["v_zero"])
    return attention_reference(q_rot, k_hat, v_hat, seq_lens, sm_scale).astype(np.float16)


def empty_cache(B: int, S_max: int, n_kv: int, d: int) -> dict:
    return {"k_codes": np.zeros((B, S_max, n_kv, d), np.int64), "v_codes": np.zeros((B, S_max, n_kv, d), np.int64),
            "k_scale": np.ones((B, S_max, n_kv), np.float32), "v_scale": np.ones((B, S_max, n_kv), np.float32),
            "k_zero": np.zeros((B, S_max, n_kv), np.int64), "v_zero": np.zeros((B, S_max, n_kv), np.int64)}


def cache_init(k, v, S_max: int, clip_ratio: float = 0.95) -> dict:
    """Prefill a cache (routine Init) from post-RoPE K, V [B, T, n_kv, d]: rows 0..T-1."""
    from .quant import unpack_int4_unsigned
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    B, T, n_kv, d = k.shape
    c = empty_cache(B, S_max, n_kv, d)
    for b in range(B):
        out = kv_init(k[b], v[b], None, clip_ratio=clip_ratio)
        c["k_codes"][b, :T] = unpack_int4_unsigned(out["k_codes"])
        c["v_codes"][b, :T] = unpack_int4_unsigned(out["v_codes"])
        c["k_scale"][b, :T] = out["k_scale"]
        c["v_scale"][b, :T] = out["v_scale"]
        c["k_zero"][b, :T] = out["k_zero"]
        c["v_zero"][b, :T] = out["v_zero"]
    return c
