"""The QuaRot 4-bit linear layer and its pieces, composed — oracle (TEST INFRASTRUCTURE).

P:860 (App. "4-bit Linear and Attention Layers"): "For a given input of FP16, the layer
optionally computes the Hadamard operation, then calls the quantization kernel to
quantize and save the input in a sub-byte format. In the next step, the quantized
weights and input are passed to the CUTLASS 4-bit GEMM kernel. Finally, the output is
dequantized and cast back to FP16."

Which linear gets which online transform ("1 1/2 Hadamard transforms per layer",
Fig. ffn_quarot, Fig. attn_quarot):
  NONE         QKV and gate/up inputs (the global Q is fused into the weights)
  FULL         down_proj input: H before quantize, W_down <- H W_down
  ACROSS_HEADS out_proj input: Z <- Z (H_{n_h} (x) I)
"""
from __future__ import annotations

import math

import numpy as np

from . import hadamard as had
from .gemm import dequant_epilogue, int_matmul, int_matmul_exact_f64
from .quant import pack_int4, quantize_sym_rows, rtn_weight_quantize

MODES = ("none", "full", "across_heads")


def online_transform(x: np.ndarray, mode: str, head_dim: int = 128) -> np.ndarray:
    """y for each token row according to the mode (fp64, dense)."""
    x = np.asarray(x, dtype=np.float64)
    if mode == "none":
        return x
    if mode == "full":
        return had.apply_full(x)
    if mode == "across_heads":
        return had.apply_across_heads(x, head_dim)
    raise ValueError(f"unknown mode {mode!r}")


def hadamard_quant(x: np.ndarray, mode: str, head_dim: int = 128, clip_ratio: float = 0.9):
    """Rows a1|a2 + a3 of SURVEY §8(a): online transform then per-token symmetric INT4
    RTN and nibble packing.  Returns (codes int64 [M,K], packed uint8 [M,K/2],
    scale float32 [M])."""
    y = online_transform(x, mode, head_dim)
    codes, scale = quantize_sym_rows(y, clip_ratio)
    return codes, pack_int4(codes), scale


def rotate_weight(w: np.ndarray, mode: str, head_dim: int = 128) -> np.ndarray:
    """Offline pairing of the online transform (Z4): with y = T x online, the weight in
    nn.Linear [N, K] layout becomes W' = W T^T so that W' (T x) = W x.
    FULL: W_down <- H W_down (in the paper's [in, out] orientation)."""
    w = np.asarray(w, dtype=np.float64)
    if mode == "none":
        return w
    # rows of W are vectors in the input space: rotate each like an activation row
    return online_transform(w, mode, head_dim)


def quantize_weight(w: np.ndarray, mode: str, head_dim: int = 128):
    """a0: rotate then per-output-channel RTN with clip search.  Returns
    (codes int64 [N,K], packed uint8 [N,K/2], scale float32 [N])."""
    wr = rotate_weight(w, mode, head_dim)
    codes, scale, _ = rtn_weight_quantize(wr)
    return codes, pack_int4(codes), scale


def int4_linear(cx: np.ndarray, sx: np.ndarray, cw: np.ndarray, sw: np.ndarray,
                exact_f64: bool = False):
    """Rows a4 + a5: acc = cx cw^T exactly, y = fp16(acc s_x s_w).  Returns (acc, y)."""
    acc = int_matmul_exact_f64(cx, cw) if exact_f64 else int_matmul(cx, cw)
    return acc, dequant_epilogue(acc, sx, sw)


def quarot_linear(x: np.ndarray, cw: np.ndarray, sw: np.ndarray, mode: str,
                  head_dim: int = 128, clip_ratio: float = 0.9, exact_f64: bool = False):
    """The whole 4-bit linear of P:860 on fp16 input rows x."""
    cx, _, sx = hadamard_quant(x, mode, head_dim, clip_ratio)
    _, y = int4_linear(cx, sx, cw, sw, exact_f64=exact_f64)
    return y


# ---------------------------------------------------------------------------------------
# Full-precision pieces used only by the computational-invariance pins (Eq. 3)
# ---------------------------------------------------------------------------------------

def rmsnorm_noscale(x: np.ndarray) -> np.ndarray:
    """x_i <- x_i / ||x_i|| per row, the scale-free RMSNorm of Eq. (3)."""
    x = np.asarray(x, dtype=np.float64)
    return x / np.linalg.norm(x, axis=-1, keepdims=True)


def silu(v: np.ndarray) -> np.ndarray:
    return v / (1.0 + np.exp(-v))


def ffn_reference(x, w_gate, w_up, w_down, alpha):
    """Fig. ffn_orig: RMSNorm with alpha, gated FFN.  nn.Linear layouts
    w_gate/w_up [F, D], w_down [D, F].  fp64."""
    h = rmsnorm_noscale(x) * alpha[None, :]
    return (silu(h @ w_gate.T) * (h @ w_up.T)) @ w_down.T


def ffn_quarot_fullprecision(xq, w_gate, w_up, w_down, alpha, q_mat):
    """Fig. ffn_quarot without quantization: input XQ, alpha and Q^T fused into
    W_gate/W_up (Eq. 4), online H before W_down and H fused into W_down
    (P:185), W_down post-multiplied by Q.  Returns the rotated output YQ."""
    wg = (w_gate * alpha[None, :]) @ q_mat          # [F,D]: x Q -> (xQ)(Q^T diag(a) W)
    wu = (w_up * alpha[None, :]) @ q_mat
    wd = q_mat.T @ rotate_weight(w_down, "full")    # rows of W_down rotated by H, then Q
    h = rmsnorm_noscale(xq)
    a = silu(h @ wg.T) * (h @ wu.T)
    a = online_transform(a, "full")
    return a @ wd.T


def token_sample(m_total: int, n: int, shards: int = 1) -> np.ndarray:
    """Deterministic sample of token rows for parity at full size: first, last, shard
    boundaries, and evenly spaced interior rows."""
    idx = {0, m_total - 1}
    for g in range(1, shards):
        b = g * m_total // shards
        idx.update({b - 1, b})
    step = max(1, m_total // max(1, n))
    idx.update(range(step // 2, m_total, step))
    return np.array(sorted(i for i in idx if 0 <= i < m_total)[: max(n, len(idx))], dtype=np.int64)


def scale_norm(mode: str, k: int, head_dim: int = 128) -> float:
    """1/sqrt of the transform size (Z5), exposed for tests."""
    if mode == "none":
        return 1.0
    if mode == "full":
        return 1.0 / math.sqrt(k)
    return 1.0 / math.sqrt(k // head_dim)
