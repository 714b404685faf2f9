"""INT4 x INT4 GEMM and the dequantizing epilogue — oracle (TEST INFRASTRUCTURE).

* P:167 (Fig. ffn_quarot caption): "The result of the matmul between the INT4 weights
  and activations on a TensorCore is INT32, which we immediately cast (and scale) to
  FP16".
* P:233 (Stage 2b): "The dequantization is also done by casting the INT32 output of
  GEMM into FP16, multiply the corresponding scale for the row (from input scales) and
  column (from weight scales)."

Reading Z11/Z12: the scale products are formed in fp64 here and rounded once to fp16
(the literal fp16 cast of |acc| up to 1.4e6 would overflow); the GPU forms them in
fp32.  acc is exact: sum_k c_x[m,k] c_w[n,k] over int64.
"""
from __future__ import annotations

import numpy as np

INT32_MAX = 2**31 - 1


def int_matmul(cx: np.ndarray, cw: np.ndarray) -> np.ndarray:
    """acc[m, n] = sum_k cx[m, k] * cw[n, k], int64, by definition (numpy int64 matmul:
    exact integer arithmetic, no BLAS).  Asserts the result fits int32 (D3)."""
    cx = np.asarray(cx, dtype=np.int64)
    cw = np.asarray(cw, dtype=np.int64)
    if cx.shape[1] != cw.shape[1]:
        raise ValueError("inner dimensions differ")
    acc = cx @ cw.T
    if acc.size and np.max(np.abs(acc)) > INT32_MAX:
        raise OverflowError("accumulator exceeds int32")
    return acc


def int_matmul_exact_f64(cx: np.ndarray, cw: np.ndarray) -> np.ndarray:
    """Same integers via fp64 BLAS.  Exact because every product |c_x c_w| <= 64 and
    every partial sum is below 64 * K <= 2^21 << 2^53 (pin: tests compare with
    int_matmul on sub-blocks).  Used for large sampled blocks where the int64
    loop would take minutes."""
    cx = np.asarray(cx, dtype=np.float64)
    cw = np.asarray(cw, dtype=np.float64)
    if cx.shape[1] != cw.shape[1]:
        raise ValueError("inner dimensions differ")
    if cx.shape[1] > 2**21 // 64:
        raise ValueError("K too large for the exactness bound")
    acc = cx @ cw.T
    out = acc.astype(np.int64)
    if not np.array_equal(out.astype(np.float64), acc):
        raise ArithmeticError("fp64 accumulation not exact")
    return out


def dequant_epilogue(acc: np.ndarray, x_scale: np.ndarray, w_scale: np.ndarray) -> np.ndarray:
    """y[m, n] = fp16_RNE(acc[m, n] * s_x[m] * s_w[n]), product in fp64 (Z12)."""
    y = np.asarray(acc, dtype=np.float64) * np.asarray(x_scale, dtype=np.float64)[:, None] \
        * np.asarray(w_scale, dtype=np.float64)[None, :]
    return y.astype(np.float16)


def group_linear(cx: np.ndarray, sx: np.ndarray, cw: np.ndarray, sw: np.ndarray) -> np.ndarray:
    """Group-wise W4A4 linear: y[m, n] = fp16_RNE( sum_g sx[m, g] sw[n, g]
    sum_{k in g} cx[m, k] cw[n, k] ), the per-group integer dot products exact (int64), the
    scaled sum in fp64.  sx [M, K/G], sw [N, K/G]."""
    cx = np.asarray(cx, dtype=np.int64)
    cw = np.asarray(cw, dtype=np.int64)
    ng = sx.shape[1]
    g = cx.shape[1] // ng
    y = np.zeros((cx.shape[0], cw.shape[0]), dtype=np.float64)
    for j in range(ng):
        acc = int_matmul(cx[:, j * g:(j + 1) * g], cw[:, j * g:(j + 1) * g]).astype(np.float64)
        y += acc * np.asarray(sx[:, j], dtype=np.float64)[:, None] * np.asarray(sw[:, j], dtype=np.float64)[None, :]
    return y.astype(np.float16)
