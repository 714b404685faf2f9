"""Decoder-layer glue around the quantized linears — oracle (TEST
INFRASTRUCTURE).  Standard Llama-2 ops in the QuaRot-modified layer (Fig. ffn_quarot P:131-169,
Fig. attn_quarot), fp64:

* RMSNorm without scale ("we leave the computation of RMSNorm (without scaling) in
  FP32"; Eq. 3 P:123 writes it x <- x/||x||).  Reading Z21: Llama's form x / sqrt(mean(x^2) + eps),
  eps = 1e-5; it differs from x/||x|| by the constant sqrt(d) (exactly, for eps = 0), which the
  per-token quantization scale absorbs.
* RoPE ("Pos", Eqs. 10-12): Llama-2's rotary embedding, pairs (i, i + d/2) ("rotate
  half"), inv_freq_i = theta^(-2i/d), theta = 10000, position = index within the sequence.
* SwiGLU: act = silu(gate) * up (Fig. ffn_orig, sigma = SiLU in Llama).
* residual add.

Precision (Fig. ffn_quarot caption): "The result of the matmul between the INT4 weights
and activations on a TensorCore is INT32, which we immediately cast (and scale) to FP16 which is
the default precision of the model."  Every linear output is therefore an fp16 tensor before
the next op, and the elementwise glue runs as the FP16 model's ops (reading Z23): each op's
result is rounded to fp16, i.e. act = fp16(fp16(silu(g)) * u) and x + fp16(y) -> fp16, with the
arithmetic of each op exact (fp64) before its one rounding.
"""
from __future__ import annotations

import numpy as np

from . import kv as okv
from . import layer as olayer

RMS_EPS = 1e-5
ROPE_THETA = 10000.0


def rmsnorm(x: np.ndarray, eps: float = RMS_EPS) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)


def rope(x: np.ndarray, positions: np.ndarray, theta: float = ROPE_THETA) -> np.ndarray:
    """x: [T, n_heads, d]; positions: [T] integers.  Rotate-half RoPE in fp64."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    half = d // 2
    inv_freq = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / d)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]  # [T, half]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def swiglu(gate: np.ndarray, up: np.ndarray) -> np.ndarray:
    """silu(g) * u in fp64 (the full-precision definition)."""
    g = np.asarray(gate, dtype=np.float64)
    return g / (1.0 + np.exp(-g)) * np.asarray(up, dtype=np.float64)


def silu_fp16(gate16: np.ndarray) -> np.ndarray:
    """The FP16 model's activation op: fp16(silu(g)) of fp16 g (one rounding)."""
    g = np.asarray(gate16, dtype=np.float16).astype(np.float64)
    return (g / (1.0 + np.exp(-g))).astype(np.float16)


def swiglu_fp16(gate16: np.ndarray, up16: np.ndarray) -> np.ndarray:
    """SwiGLU of the FP16 model (Fig. ffn_orig, reading Z23): fp16(fp16(silu(g)) * u), g and u
    the fp16 outputs of the gate / up linears."""
    s = silu_fp16(gate16).astype(np.float64)
    return (s * np.asarray(up16, dtype=np.float16).astype(np.float64)).astype(np.float16)


def add_fp16(a16: np.ndarray, b16: np.ndarray) -> np.ndarray:
    """The FP16 model's residual add: fp16(a + b) of two fp16 tensors (one rounding)."""
    with np.errstate(over="ignore"):  # |a + b| > 65504 rounds to inf, as in the FP16 model
        return (np.asarray(a16, np.float16).astype(np.float64)
                + np.asarray(b16, np.float16).astype(np.float64)).astype(np.float16)


def rmsnorm_quant(x: np.ndarray, clip_ratio: float = 0.9, eps: float = RMS_EPS):
    """RMSNorm (fp64, no fp16 round trip) then per-token INT4 quantization (NONE mode):
    Fig. ffn_quarot's norm -> quantize."""
    return olayer.hadamard_quant(rmsnorm(x, eps), "none", clip_ratio=clip_ratio)


def decoder_layer(x, attn_out, w, positions, shapes: dict, clip=0.9, clip_kv=0.95):
    """One QuaRot decoder layer prefill with the attention core excluded (SURVEY §8 a8 /
    config 5): the out_proj input is the supplied `attn_out` rows.

    x: [T, hidden] fp16 residual stream; attn_out: [T, hidden] fp16; w: dict name -> (codes
    int64 [N, K], scale float32 [N]) for qkv, o, gate_up ([gate | up] rows), down.
    Returns dict with the KV cache, rotated Q (fp16), o (fp16, residual added), act (fp16) and the
    layer output (fp16)."""
    n_h, n_kv, d = shapes["n_heads"], shapes["n_kv"], shapes["head_dim"]
    ffn = shapes["ffn"]
    T = x.shape[0]
    cx, _, sx = rmsnorm_quant(x, clip)
    qkv = olayer.int4_linear(cx, sx, *w["qkv"], exact_f64=True)[1]
    qkv64 = qkv.astype(np.float64)
    nq, nk = n_h * d, n_kv * d
    # RoPE output is stored as fp16 (the model's activation precision, Fig. attn_quarot) before
    # the per-head Hadamard and the cache quantization
    q = rope(qkv64[:, :nq].reshape(T, n_h, d), positions).astype(np.float16).astype(np.float64)
    k = rope(qkv64[:, nq:nq + nk].reshape(T, n_kv, d), positions).astype(np.float16).astype(np.float64)
    v = qkv64[:, nq + nk:].reshape(T, n_kv, d)
    cache = okv.kv_init(k, v, q, clip_ratio=clip_kv)
    co, _, so = olayer.hadamard_quant(attn_out, "across_heads", d, clip)
    o = add_fp16(x, olayer.int4_linear(co, so, *w["o"], exact_f64=True)[1])      # x + fp16 linear output
    cn, _, sn = rmsnorm_quant(o, clip)
    gu = olayer.int4_linear(cn, sn, *w["gate_up"], exact_f64=True)[1]            # fp16 [gate | up]
    act = swiglu_fp16(gu[:, :ffn], gu[:, ffn:])
    cd, _, sd = olayer.hadamard_quant(act, "full", d, clip)
    out = add_fp16(o, olayer.int4_linear(cd, sd, *w["down"], exact_f64=True)[1])
    return {"qkv": qkv, "cache": cache, "o": o, "gate_up": gu, "act": act, "out": out}
