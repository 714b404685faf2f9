"""Parity comparison helpers (test infrastructure).  Tolerances from BASELINE.json
north_star: int32 accumulators bit-exact; INT4 codes within 1 step on at most 1e-4 of
elements; fp16 outputs within 1e-2 relative Frobenius; scales within 1e-5 relative
(SURVEY §8c O10)."""
from __future__ import annotations

import numpy as np

CODE_FLIP_FRACTION = 1e-4
FROB_REL = 1e-2
SCALE_REL = 1e-5


def unpack_signed(packed: np.ndarray) -> np.ndarray:
    b = np.asarray(packed, dtype=np.int64)
    lo, hi = b & 0xF, (b >> 4) & 0xF
    out = np.empty(b.shape[:-1] + (2 * b.shape[-1],), dtype=np.int64)
    out[..., 0::2] = np.where(lo >= 8, lo - 16, lo)
    out[..., 1::2] = np.where(hi >= 8, hi - 16, hi)
    return out


def unpack_unsigned(packed: np.ndarray) -> np.ndarray:
    b = np.asarray(packed, dtype=np.int64)
    out = np.empty(b.shape[:-1] + (2 * b.shape[-1],), dtype=np.int64)
    out[..., 0::2] = b & 0xF
    out[..., 1::2] = (b >> 4) & 0xF
    return out


def code_stats(gpu_codes: np.ndarray, ref_codes: np.ndarray) -> dict:
    d = np.abs(np.asarray(gpu_codes, np.int64) - np.asarray(ref_codes, np.int64))
    n = d.size
    return {"n": int(n), "flips": int(np.count_nonzero(d)), "max_step": int(d.max()) if n else 0,
            "fraction": float(np.count_nonzero(d)) / max(1, n)}


def assert_codes(gpu_codes, ref_codes, what=""):
    st = code_stats(gpu_codes, ref_codes)
    allowed = max(1, int(CODE_FLIP_FRACTION * st["n"]))
    assert st["max_step"] <= 1, f"{what}: code differs by {st['max_step']} steps ({st})"
    assert st["flips"] <= allowed, f"{what}: {st['flips']} flips > {allowed} allowed ({st})"
    return st


# When an fp16 intermediate the oracle cannot observe (RoPE inside the fused KV pass, Z22) is
# rounded on both sides from different-precision arithmetic, a group's extreme element may land
# on the adjacent fp16 value: its scale then moves by up to one fp16 ulp, relative 2^-10.
FP16_ULP_REL = 2.0 ** -10


def assert_scales(gpu_scale, ref_scale, what="", rel_tol=SCALE_REL):
    g = np.asarray(gpu_scale, np.float64)
    r = np.asarray(ref_scale, np.float64)
    assert np.array_equal(np.isnan(g), np.isnan(r)), f"{what}: NaN pattern differs"
    ok = ~np.isnan(r)
    rel = np.abs(g[ok] - r[ok]) / np.maximum(np.abs(r[ok]), 1e-300)
    assert rel.size == 0 or rel.max() <= rel_tol, f"{what}: scale rel diff {rel.max():.3g}"
    return float(rel.max()) if rel.size else 0.0


def frob_rel(y_gpu, y_ref) -> float:
    g = np.asarray(y_gpu, np.float64)
    r = np.asarray(y_ref, np.float64)
    den = np.linalg.norm(r)
    return float(np.linalg.norm(g - r) / den) if den > 0 else float(np.linalg.norm(g))


def max_fp16_ulp(y_gpu, y_ref) -> int:
    a = np.asarray(y_gpu, np.float16).view(np.int16).astype(np.int64)
    b = np.asarray(y_ref, np.float16).view(np.int16).astype(np.int64)
    # map sign-magnitude to a monotone integer line
    a = np.where(a < 0, -(a & 0x7FFF), a)
    b = np.where(b < 0, -(b & 0x7FFF), b)
    return int(np.max(np.abs(a - b))) if a.size else 0
