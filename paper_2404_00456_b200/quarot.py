"""Thin Python binding of libquarot.so (include/quarot.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module only
allocates outputs with ``torch.empty`` (PyTorch is the device-memory / stream plumbing),
passes raw device pointers and the current CUDA stream, and raises on a non-OK status.
There is no fallback: if the shared library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# QUAROT_LIB: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("QUAROT_LIB") or os.path.join(_PKG, "libquarot.so")

NONE, FULL, ACROSS_HEADS = 0, 1, 2
RMSNORM = 0x100  # mode flag: scale-free RMSNorm fused into the NONE quantizer
KPERM = 0x200    # mode flag (FULL, K = 28672): codes in the transform-native K order
MODES = {"none": NONE, "full": FULL, "across_heads": ACROSS_HEADS}
KV_ROTATE_K, KV_ROTATE_V = 1, 2

_c_i64, _c_i32, _c_u32, _c_f32, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_float, ctypes.c_void_p

_SIGS = {
    "quarot_hadamard_quant": [_vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_f32, _vp, _c_i64, _vp, _vp],
    "quarot_int4_linear": [_vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp],
    "quarot_int4_matmul_s32": [_vp, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp],
    "quarot_int4_linear_residual": [_vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp,
                                    _c_i64, _vp],
    "quarot_int4_linear_swiglu": [_vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp],
    "quarot_rope": [_vp, _c_i64, _c_i32, _c_i32, _c_i64, _c_i64, _c_i32, _c_f32, _vp],
    "quarot_swiglu": [_vp, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp],
    "quarot_kv_quant": [_vp, _c_i64, _vp, _c_i64, _c_i64, _c_i32, _c_i32, _vp, _c_i64, _c_i32, _c_u32,
                        _c_f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "quarot_kv_quant_rope": [_vp, _c_i64, _vp, _c_i64, _c_i64, _c_i32, _c_i32, _vp, _c_i64, _c_i32, _c_u32,
                             _c_f32, _c_i64, _c_i32, _c_f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "quarot_kv_append": [_vp, _c_i64, _vp, _c_i64, _c_i64, _c_i32, _c_i32, _vp, _c_i64, _c_i32, _c_u32, _c_f32,
                         _vp, _c_f32, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "quarot_kv_decode": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_i64, _c_f32,
                         _vp, _vp, _c_i64, _vp],
    "quarot_kv_decode_workspace_bytes": [_c_i64, _c_i32, _c_i32, _c_i64],
    "quarot_hadamard_quant_group": [_vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32, _c_f32, _vp, _c_i64, _vp,
                                    _c_i64, _vp],
    "quarot_hadamard_quant_group8": [_vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32, _c_f32, _vp, _c_i64, _vp,
                                     _c_i64, _vp],
    "quarot_int4_linear_group": [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32,
                                 _vp, _c_i64, _vp],
    "quarot_int4_linear_group8": [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32,
                                  _vp, _c_i64, _vp],
    "quarot_hadamard_quant8": [_vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_f32, _vp, _c_i64, _vp, _vp],
    "quarot_int8_linear": [_vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp],
    "quarot_int8_matmul_s32": [_vp, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp],
    "quarot_status_string": [_c_i32],
    "quarot_abi_version": [],
    "quarot_base_hadamard": [_c_i32, _vp],
    "quarot_full_kperm": [_c_i64, _vp],
    "quarot_prepare": [],
    "quarot_last_launch_count": [],
    "quarot_last_cuda_error": [],
    "quarot_debug_gemm_mode": [_c_i32],
    "quarot_debug_gemm_group_m": [_c_i32],
    "quarot_debug_hq_full_variant": [_c_i32],
    "quarot_debug_hq_heads_variant": [_c_i32],
    "quarot_debug_kv_variant": [_c_i32],
}
EXPORTS = tuple(_SIGS)


class QuarotError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: status {status}: {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libquarot.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2404_00456_b200.build`")
        h = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(h, name)
            f.argtypes = args
            f.restype = (ctypes.c_char_p if name in ("quarot_status_string", "quarot_last_cuda_error")
                         else ctypes.c_int64 if name == "quarot_kv_decode_workspace_bytes"
                         else None if name.startswith("quarot_debug_") else ctypes.c_int32)
        _lib = h
    return _lib


def _check(fn: str, status: int):
    if status != 0:
        msg = lib().quarot_status_string(status).decode()
        if status == 6:  # QUAROT_ERR_CUDA
            msg += f" ({lib().quarot_last_cuda_error().decode()})"
        raise QuarotError(fn, status, msg)


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev(t: torch.Tensor, name: str, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() >= 1 and t.stride(-1) != 1:
        raise ValueError(f"{name} must have unit stride in its last dimension")
    return t.data_ptr()


def abi_version() -> int:
    return lib().quarot_abi_version()


def last_launch_count() -> int:
    return lib().quarot_last_launch_count()


def base_hadamard(m: int) -> torch.Tensor:
    """The library's stored H_m (host int8), for cross-checking against the oracle."""
    out = torch.empty(m * m, dtype=torch.int8)
    _check("quarot_base_hadamard", lib().quarot_base_hadamard(m, out.data_ptr()))
    return out.view(m, m)


def hadamard_quant(x: torch.Tensor, mode="none", head_dim: int = 128, clip_ratio: float = 0.9,
                   q: torch.Tensor | None = None, scale: torch.Tensor | None = None, stream=None,
                   rmsnorm: bool = False, kperm: bool = False):
    """quarot_hadamard_quant: fp16 x [M, K] -> (packed uint8 q [M, K/2], fp32 scale [M]).
    rmsnorm=True (NONE only): RMS-normalize each row first (scale-free RMSNorm, fused).
    kperm=True (FULL, K = 28672): codes in the transform-native K order (full_kperm)."""
    mode_i = MODES[mode] if isinstance(mode, str) else int(mode)
    if rmsnorm:
        mode_i |= RMSNORM
    if kperm:
        mode_i |= KPERM
    M, K = x.shape
    if q is None:
        q = torch.empty(M, K // 2, dtype=torch.uint8, device=x.device)
    if scale is None:
        scale = torch.empty(M, dtype=torch.float32, device=x.device)
    st = lib().quarot_hadamard_quant(_dev(x, "x", torch.float16), M, K, x.stride(0), mode_i, head_dim,
                                     clip_ratio, _dev(q, "q", torch.uint8), q.stride(0),
                                     _dev(scale, "scale", torch.float32), _stream(stream))
    _check("quarot_hadamard_quant", st)
    return q, scale


def prepare() -> None:
    """quarot_prepare: one-time setup (constant images, tables, kernel attributes) on the current
    CUDA device, so no later call synchronizes the host (e.g. before CUDA-graph capture)."""
    _check("quarot_prepare", lib().quarot_prepare())


def full_kperm(K: int) -> torch.Tensor:
    """quarot_full_kperm: int64 [K] (host), perm[p] = natural element index at native position p."""
    perm = torch.empty(K, dtype=torch.int64)
    _check("quarot_full_kperm", lib().quarot_full_kperm(K, perm.data_ptr()))
    return perm


def permute_k_packed(w: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
    """Offline: packed INT4 rows [N, K/2] reordered along K by `perm` (W'[n][p] = W[n][perm[p]]),
    the weight layout paired with KPERM activations.  A pure nibble permutation (torch ops)."""
    lo, hi = (w & 0xF), (w >> 4)
    codes = torch.stack([lo, hi], -1).reshape(w.shape[0], -1)
    codes = codes[:, perm.to(w.device)]
    return (codes[:, 0::2] | (codes[:, 1::2] << 4)).contiguous()


def int4_linear(xq: torch.Tensor, x_scale: torch.Tensor, wq: torch.Tensor, w_scale: torch.Tensor,
                y: torch.Tensor | None = None, stream=None, residual: torch.Tensor | None = None) -> torch.Tensor:
    """quarot_int4_linear: y fp16 [M, N] = fp16(acc * s_x * s_w) (+ residual, fused:
    quarot_int4_linear_residual)."""
    M, Kh = xq.shape
    N = wq.shape[0]
    if y is None:
        y = torch.empty(M, N, dtype=torch.float16, device=xq.device)
    if residual is None:
        st = lib().quarot_int4_linear(_dev(xq, "xq", torch.uint8), _dev(x_scale, "x_scale", torch.float32), M,
                                      2 * Kh, xq.stride(0), _dev(wq, "wq", torch.uint8),
                                      _dev(w_scale, "w_scale", torch.float32), N, wq.stride(0),
                                      _dev(y, "y", torch.float16), y.stride(0), _stream(stream))
        _check("quarot_int4_linear", st)
    else:
        st = lib().quarot_int4_linear_residual(
            _dev(xq, "xq", torch.uint8), _dev(x_scale, "x_scale", torch.float32), M, 2 * Kh, xq.stride(0),
            _dev(wq, "wq", torch.uint8), _dev(w_scale, "w_scale", torch.float32), N, wq.stride(0),
            _dev(residual, "residual", torch.float16), residual.stride(0), _dev(y, "y", torch.float16), y.stride(0),
            _stream(stream))
        _check("quarot_int4_linear_residual", st)
    return y


def interleave_gate_up(wq: torch.Tensor, w_scale: torch.Tensor):
    """Offline weight layout for quarot_int4_linear_swiglu: [gate (F rows) ; up (F rows)] ->
    rows interleaved in blocks of 8 ([8 gate | 8 up] per 16).  Pure row permutation."""
    F = wq.shape[0] // 2
    if wq.shape[0] != 2 * F or F % 8:
        raise ValueError("gate/up weight needs 2F rows with F % 8 == 0")
    idx = torch.arange(2 * F, device=wq.device).view(2, F // 8, 8).transpose(0, 1).reshape(-1)
    return wq[idx].contiguous(), w_scale[idx].contiguous()


def int4_linear_swiglu(xq: torch.Tensor, x_scale: torch.Tensor, wq_il: torch.Tensor, w_scale_il: torch.Tensor,
                       act: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """quarot_int4_linear_swiglu: act [M, F] = silu(gate) * up from interleaved gate/up weights."""
    M, Kh = xq.shape
    N2 = wq_il.shape[0]
    if act is None:
        act = torch.empty(M, N2 // 2, dtype=torch.float16, device=xq.device)
    st = lib().quarot_int4_linear_swiglu(_dev(xq, "xq", torch.uint8), _dev(x_scale, "x_scale", torch.float32), M,
                                         2 * Kh, xq.stride(0), _dev(wq_il, "wq", torch.uint8),
                                         _dev(w_scale_il, "w_scale", torch.float32), N2, wq_il.stride(0),
                                         _dev(act, "act", torch.float16), act.stride(0), _stream(stream))
    _check("quarot_int4_linear_swiglu", st)
    return act


def rope(x: torch.Tensor, pos0: int = 0, seq_len: int = 2048, theta: float = 10000.0, stream=None) -> torch.Tensor:
    """quarot_rope, in place on x fp16 [T, n_heads, head_dim] (token stride arbitrary, heads
    contiguous): Llama-2 rotary embedding at positions (pos0 + t) % seq_len."""
    T, n, d = x.shape
    if x.stride(2) != 1 or x.stride(1) != d:
        raise ValueError("x: heads of a token must be contiguous [n, d]")
    _check("quarot_rope", lib().quarot_rope(_dev(x, "x", torch.float16), T, n, d, x.stride(0), pos0, seq_len, theta,
                                            _stream(stream)))
    return x


def swiglu(gate_up: torch.Tensor, act: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """quarot_swiglu: act [M, F] = silu(gate_up[:, :F]) * gate_up[:, F:]."""
    M, F2 = gate_up.shape
    F = F2 // 2
    if act is None:
        act = torch.empty(M, F, dtype=torch.float16, device=gate_up.device)
    _check("quarot_swiglu", lib().quarot_swiglu(_dev(gate_up, "gate_up", torch.float16), M, F, gate_up.stride(0),
                                                _dev(act, "act", torch.float16), act.stride(0), _stream(stream)))
    return act


def int4_matmul_s32(xq: torch.Tensor, wq: torch.Tensor, acc: torch.Tensor | None = None,
                    stream=None) -> torch.Tensor:
    """quarot_int4_matmul_s32: raw int32 accumulators [M, N] (parity only)."""
    M, Kh = xq.shape
    N = wq.shape[0]
    if acc is None:
        acc = torch.empty(M, N, dtype=torch.int32, device=xq.device)
    st = lib().quarot_int4_matmul_s32(_dev(xq, "xq", torch.uint8), M, 2 * Kh, xq.stride(0),
                                      _dev(wq, "wq", torch.uint8), N, wq.stride(0),
                                      _dev(acc, "acc", torch.int32), acc.stride(0), _stream(stream))
    _check("quarot_int4_matmul_s32", st)
    return acc


def kv_quant(k: torch.Tensor, v: torch.Tensor, q: torch.Tensor | None = None, flags: int = KV_ROTATE_K,
             clip_ratio: float = 0.95, out: dict | None = None, stream=None, rope: tuple | None = None) -> dict:
    """quarot_kv_quant (KV-cache Init): k, v fp16 [T, n_kv, d] (heads contiguous per token,
    any token stride — e.g. views into a fused QKV output); q optional fp16 [T, n_q, d]
    rotated in place.  rope = (pos0, seq_len, theta) calls quarot_kv_quant_rope instead: K and Q
    are read pre-RoPE and RoPE is applied in the same pass.  Returns dict of codes / scales /
    zeros for K and V."""
    T, n_kv, d = k.shape
    if v.shape != k.shape:
        raise ValueError("k and v shapes differ")
    for name, t in (("k", k), ("v", v), ("q", q)):
        if t is not None and (t.stride(2) != 1 or t.stride(1) != d):
            raise ValueError(f"{name}: heads of a token must be contiguous [n, d]")
    dev = k.device
    if out is None:
        out = {
            "k_codes": torch.empty(T, n_kv, d // 2, dtype=torch.uint8, device=dev),
            "k_scale": torch.empty(T, n_kv, dtype=torch.float32, device=dev),
            "k_zero": torch.empty(T, n_kv, dtype=torch.uint8, device=dev),
            "v_codes": torch.empty(T, n_kv, d // 2, dtype=torch.uint8, device=dev),
            "v_scale": torch.empty(T, n_kv, dtype=torch.float32, device=dev),
            "v_zero": torch.empty(T, n_kv, dtype=torch.uint8, device=dev),
        }
    n_q = 0 if q is None else q.shape[1]
    head = (_dev(k, "k", torch.float16), k.stride(0), _dev(v, "v", torch.float16), v.stride(0), T, n_kv, d,
            None if q is None else _dev(q, "q", torch.float16), 0 if q is None else q.stride(0), n_q, flags,
            clip_ratio)
    outs = (out["k_codes"].data_ptr(), out["k_scale"].data_ptr(), out["k_zero"].data_ptr(),
            out["v_codes"].data_ptr(), out["v_scale"].data_ptr(), out["v_zero"].data_ptr(), _stream(stream))
    if rope is None:
        _check("quarot_kv_quant", lib().quarot_kv_quant(*head, *outs))
    else:
        pos0, seq_len, theta = rope
        _check("quarot_kv_quant_rope", lib().quarot_kv_quant_rope(*head, int(pos0), int(seq_len), float(theta), *outs))
    return out


def hadamard_quant_group(x: torch.Tensor, group: int = 128, clip_ratio: float = 0.9, q: torch.Tensor | None = None,
                         scale: torch.Tensor | None = None, stream=None, mode="none", head_dim: int = 128):
    """quarot_hadamard_quant_group (§8 f3; mode none / full / across_heads): packed INT4 [M, K/2]
    and fp32 scales [M, K/group]."""
    M, K = x.shape
    q = torch.empty(M, K // 2, dtype=torch.uint8, device=x.device) if q is None else q
    scale = torch.empty(M, max(K // group, 1), dtype=torch.float32, device=x.device) if scale is None else scale
    mode_i = MODES[mode] if isinstance(mode, str) else int(mode)
    st = lib().quarot_hadamard_quant_group(_dev(x, "x", torch.float16), M, K, x.stride(0), mode_i, head_dim, group,
                                           clip_ratio,
                                           _dev(q, "q", torch.uint8), q.stride(0), _dev(scale, "scale", torch.float32),
                                           scale.stride(0), _stream(stream))
    _check("quarot_hadamard_quant_group", st)
    return q, scale


def hadamard_quant_group8(x: torch.Tensor, group: int = 128, clip_ratio: float = 0.9, stream=None, mode="none",
                          head_dim: int = 128):
    """quarot_hadamard_quant_group8 (§8 f3): int8 codes [M, K] (one per byte) and fp32 scales [M, K/group]."""
    M, K = x.shape
    q = torch.empty(M, K, dtype=torch.int8, device=x.device)
    scale = torch.empty(M, max(K // group, 1), dtype=torch.float32, device=x.device)
    mode_i = MODES[mode] if isinstance(mode, str) else int(mode)
    st = lib().quarot_hadamard_quant_group8(_dev(x, "x", torch.float16), M, K, x.stride(0), mode_i, head_dim, group,
                                            clip_ratio,
                                            q.data_ptr(), q.stride(0), _dev(scale, "scale", torch.float32),
                                            scale.stride(0), _stream(stream))
    _check("quarot_hadamard_quant_group8", st)
    return q, scale


def int4_linear_group(xq: torch.Tensor, x_scale: torch.Tensor, wq: torch.Tensor, w_scale_t: torch.Tensor,
                      group: int = 128, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """quarot_int4_linear_group (§8 f3, group 64 / 128 / 256): packed INT4 codes xq [M, K/2], wq [N, K/2];
    x_scale [M, K/group]; w_scale_t [K/group, N]; y fp16 [M, N]."""
    M, K = xq.shape[0], 2 * xq.shape[1]
    N = wq.shape[0]
    y = torch.empty(M, N, dtype=torch.float16, device=xq.device) if y is None else y
    st = lib().quarot_int4_linear_group(_dev(xq, "xq", torch.uint8), _dev(x_scale, "x_scale", torch.float32),
                                        x_scale.stride(0), M, K, xq.stride(0), _dev(wq, "wq", torch.uint8),
                                        _dev(w_scale_t, "w_scale_t", torch.float32), w_scale_t.stride(0), N,
                                        wq.stride(0), group, _dev(y, "y", torch.float16), y.stride(0), _stream(stream))
    _check("quarot_int4_linear_group", st)
    return y


def int4_linear_group8(xq: torch.Tensor, x_scale: torch.Tensor, wq: torch.Tensor, w_scale_t: torch.Tensor,
                       y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """quarot_int4_linear_group8 (§8 f3, group 128): int8-stored codes xq [M, K], wq [N, K];
    x_scale [M, K/128]; w_scale_t [K/128, N]; y fp16 [M, N]."""
    M, K = xq.shape
    N = wq.shape[0]
    y = torch.empty(M, N, dtype=torch.float16, device=xq.device) if y is None else y
    st = lib().quarot_int4_linear_group8(xq.data_ptr(), _dev(x_scale, "x_scale", torch.float32), x_scale.stride(0), M,
                                         K, xq.stride(0), wq.data_ptr(), _dev(w_scale_t, "w_scale_t", torch.float32),
                                         w_scale_t.stride(0), N, wq.stride(0), 128, _dev(y, "y", torch.float16),
                                         y.stride(0), _stream(stream))
    _check("quarot_int4_linear_group8", st)
    return y


def hadamard_quant8(x: torch.Tensor, clip_ratio: float = 0.9, rmsnorm: bool = False, q: torch.Tensor | None = None,
                    scale: torch.Tensor | None = None, stream=None, mode="none", head_dim: int = 128):
    """quarot_hadamard_quant8 (A8W8, §8 f4): int8 codes [M, K] and fp32 scales [M]; mode NONE
    (± RMSNorm), FULL (every K = 2^n m) or ACROSS_HEADS (power-of-two head_dim and heads)."""
    M, K = x.shape
    if x.stride(1) != 1:
        raise ValueError("x rows must be contiguous")
    q = torch.empty(M, K, dtype=torch.int8, device=x.device) if q is None else q
    scale = torch.empty(M, dtype=torch.float32, device=x.device) if scale is None else scale
    mode_i = MODES[mode] if isinstance(mode, str) else int(mode)
    st = lib().quarot_hadamard_quant8(_dev(x, "x", torch.float16), M, K, x.stride(0), mode_i | (RMSNORM if rmsnorm else 0),
                                      head_dim, clip_ratio, q.data_ptr(), q.stride(0), scale.data_ptr(), _stream(stream))
    _check("quarot_hadamard_quant8", st)
    return q, scale


def int8_linear(xq: torch.Tensor, x_scale: torch.Tensor, wq: torch.Tensor, w_scale: torch.Tensor,
                y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """quarot_int8_linear (A8W8, §8 f4): int8 [M, K] x int8 [N, K] -> fp16 [M, N]."""
    M, K = xq.shape
    N = wq.shape[0]
    y = torch.empty(M, N, dtype=torch.float16, device=xq.device) if y is None else y
    st = lib().quarot_int8_linear(_dev(xq, "xq", torch.int8), _dev(x_scale, "x_scale", torch.float32), M, K,
                                  xq.stride(0), _dev(wq, "wq", torch.int8), _dev(w_scale, "w_scale", torch.float32), N,
                                  wq.stride(0), y.data_ptr(), y.stride(0), _stream(stream))
    _check("quarot_int8_linear", st)
    return y


def int8_matmul_s32(xq: torch.Tensor, wq: torch.Tensor, stream=None) -> torch.Tensor:
    M, K = xq.shape
    N = wq.shape[0]
    acc = torch.empty(M, N, dtype=torch.int32, device=xq.device)
    st = lib().quarot_int8_matmul_s32(_dev(xq, "xq", torch.int8), M, K, xq.stride(0), _dev(wq, "wq", torch.int8), N,
                                      wq.stride(0), acc.data_ptr(), acc.stride(0), _stream(stream))
    _check("quarot_int8_matmul_s32", st)
    return acc


def kv_cache_empty(B: int, s_max: int, n_kv: int, head_dim: int = 128, device="cuda") -> dict:
    """Allocate a per-sequence INT4 KV cache (layout of quarot_kv_append / quarot_kv_decode)."""
    return {"k_codes": torch.zeros(B, s_max, n_kv, head_dim // 2, dtype=torch.uint8, device=device),
            "k_scale": torch.ones(B, s_max, n_kv, dtype=torch.float32, device=device),
            "k_zero": torch.zeros(B, s_max, n_kv, dtype=torch.uint8, device=device),
            "v_codes": torch.zeros(B, s_max, n_kv, head_dim // 2, dtype=torch.uint8, device=device),
            "v_scale": torch.ones(B, s_max, n_kv, dtype=torch.float32, device=device),
            "v_zero": torch.zeros(B, s_max, n_kv, dtype=torch.uint8, device=device)}


def kv_append(k: torch.Tensor, v: torch.Tensor, q: torch.Tensor | None, positions: torch.Tensor, cache: dict,
              flags: int = KV_ROTATE_K, clip_ratio: float = 0.95, theta: float = 10000.0, stream=None) -> dict:
    """quarot_kv_append (routine Append): k, v [B, n_kv, d], q [B, n_q, d] pre-RoPE fp16
    (q rotated in place); positions int32 [B] on the device; cache from kv_cache_empty."""
    B, n_kv, d = k.shape
    s_max = cache["k_codes"].shape[1]
    for name, t in (("k", k), ("v", v), ("q", q)):
        if t is not None and (t.stride(2) != 1 or t.stride(1) != d):
            raise ValueError(f"{name}: heads of a token must be contiguous [n, d]")
    if positions.dtype != torch.int32 or positions.device != k.device:
        raise ValueError("positions: int32 on the device")
    st = lib().quarot_kv_append(_dev(k, "k", torch.float16), k.stride(0), _dev(v, "v", torch.float16), v.stride(0),
                                B, n_kv, d, None if q is None else _dev(q, "q", torch.float16),
                                0 if q is None else q.stride(0), 0 if q is None else q.shape[1], flags, clip_ratio,
                                positions.data_ptr(), theta, s_max,
                                *(cache[n].data_ptr() for n in ("k_codes", "k_scale", "k_zero", "v_codes", "v_scale",
                                                               "v_zero")), _stream(stream))
    _check("quarot_kv_append", st)
    return cache


def kv_decode(q: torch.Tensor, cache: dict, seq_lens: torch.Tensor, n_kv: int | None = None,
              sm_scale: float | None = None, out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
    """quarot_kv_decode (routine Decode): q fp16 [B, n_q, d] (rotated), seq_lens int32 [B]
    on the device.  Returns fp16 [B, n_q, d]."""
    B, n_q, d = q.shape
    s_max, n_kv_c = cache["k_codes"].shape[1], cache["k_codes"].shape[2]
    n_kv = n_kv_c if n_kv is None else n_kv
    if not q.is_contiguous():
        raise ValueError("q must be contiguous [B, n_q, d]")
    if seq_lens.dtype != torch.int32 or seq_lens.device != q.device:
        raise ValueError("seq_lens: int32 on the device")
    if out is None:
        out = torch.empty_like(q)
    wsb = lib().quarot_kv_decode_workspace_bytes(B, n_q, d, s_max)
    if workspace is None or workspace.numel() * workspace.element_size() < wsb:
        workspace = torch.empty(max(1, wsb // 4), dtype=torch.float32, device=q.device)
    st = lib().quarot_kv_decode(_dev(q, "q", torch.float16),
                                *(cache[n].data_ptr() for n in ("k_codes", "k_scale", "k_zero", "v_codes", "v_scale",
                                                               "v_zero")),
                                seq_lens.data_ptr(), B, n_q, n_kv, d, s_max,
                                float(d ** -0.5 if sm_scale is None else sm_scale), out.data_ptr(),
                                workspace.data_ptr(), workspace.numel() * workspace.element_size(), _stream(stream))
    _check("quarot_kv_decode", st)
    return out


def quarot_linear(x: torch.Tensor, wq: torch.Tensor, w_scale: torch.Tensor, mode="none", head_dim: int = 128,
                  clip_ratio: float = 0.9, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """The 4-bit linear layer of P:860: optional online Hadamard + quantize, INT4 GEMM,
    dequantize to fp16 — two kernel launches."""
    xq, xs = hadamard_quant(x, mode, head_dim, clip_ratio, stream=stream)
    return int4_linear(xq, xs, wq, w_scale, y=y, stream=stream)
