"""Pins for oracle/quant.py, oracle/gemm.py and oracle/kv.py (CPU only)."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import gemm, kv, layer, quant
from oracle import hadamard as had

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_sym_worked_examples():
    # P6 (clip P:249)
    for key in ("sym_quant_clip1", "sym_quant_clip09"):
        g = GOLD[key]
        codes, scale = quant.quantize_sym_rows(np.array([g["row"]]), g["clip"])
        assert codes[0].tolist() == g["codes"]
        assert float(scale[0]) == g.get("scale", g.get("scale_fp32"))


def test_sym_zero_and_nonfinite_rows():
    codes, scale = quant.quantize_sym_rows(np.array([[0.0] * 8, [1.0, np.nan] + [0.0] * 6,
                                                    [np.inf] + [1.0] * 7]))
    assert np.all(codes == 0)
    assert scale[0] == 1.0 and np.isnan(scale[1]) and np.isnan(scale[2])


def _brute_code(v, s, qmax=7):
    # argmin_q |v - q s| over integers, ties -> even (Z7), then clamp: brute force
    best = None
    for q in range(-qmax - 50, qmax + 51):
        e = abs(v - q * s)
        if best is None or e < best[0] - 1e-300 or (e == best[0] and q % 2 == 0):
            best = (e, q)
    return int(np.clip(best[1], -qmax, qmax))


def test_sym_brute_force_tiny():
    # P7: every code is the nearest representable level; unclipped error <= s/2
    rng = np.random.default_rng(0)
    for _ in range(40):
        y = rng.standard_normal((1, 9)) * rng.uniform(0.1, 10)
        codes, scale = quant.quantize_sym_rows(y, 0.9)
        s = float(scale[0])
        for v, c in zip(y[0], codes[0]):
            assert c == _brute_code(v, s)
            if abs(v) <= 7 * s:
                assert abs(v - c * s) <= s / 2 + 1e-15


def test_sym_exact_ties_round_half_even():
    # clip 1 -> s = 1 exactly for amax 7; 2.5 -> 2, -0.5 -> 0, 1.5 -> 2 (Z7)
    codes, scale = quant.quantize_sym_rows(np.array([[7.0, 2.5, -0.5, 1.5, -6.5]]), 1.0)
    assert scale[0] == 1.0
    assert codes[0].tolist() == [7, 2, 0, 2, -6]


def test_sym_idempotent():
    rng = np.random.default_rng(2)
    y = rng.standard_normal((5, 64))
    c1, s1 = quant.quantize_sym_rows(y, 1.0)
    c2, s2 = quant.quantize_sym_rows(quant.dequantize_sym_rows(c1, s1), 1.0)
    assert np.array_equal(c1, c2)
    assert np.allclose(s1, s2, rtol=1e-6)


def test_sym_scale_invariance_power_of_two():
    # P15: scaling a row by 2^j leaves codes unchanged and scales the scale exactly
    rng = np.random.default_rng(4)
    y = rng.standard_normal((3, 100))
    c1, s1 = quant.quantize_sym_rows(y)
    for j in (-7, 3, 11):
        c2, s2 = quant.quantize_sym_rows(y * 2.0**j)
        assert np.array_equal(c1, c2)
        assert np.array_equal(s2, (s1 * np.float32(2.0**j)).astype(np.float32))


def test_pack_worked_example_and_roundtrip():
    # P8
    g = GOLD["pack_7_m7"]
    assert quant.pack_int4(np.array(g["codes"])).tolist() == g["bytes"]
    # exhaustive bijection over all 256 bytes (signed nibbles)
    allb = np.arange(256, dtype=np.uint8)[None, :]
    assert np.array_equal(quant.pack_int4(quant.unpack_int4_signed(allb)), allb)
    assert np.array_equal(quant.pack_int4(quant.unpack_int4_unsigned(allb) - 0), allb)
    codes = np.array(list(itertools.product(range(-8, 8), repeat=2))).reshape(1, -1)
    assert np.array_equal(quant.unpack_int4_signed(quant.pack_int4(codes)), codes)


def test_rtn_weight_examples():
    # S:258-262 examples for the clip line search
    w = np.array([[-7.0, -3, 0, 2, 7, 5] * 4]) * 0.25  # exactly representable with s = 0.25
    codes, scale, clip = quant.rtn_weight_quantize(w)
    assert clip[0] == 1.0 and scale[0] == np.float32(0.25)
    assert np.allclose(codes * 0.25, w)
    # one outlier among many ones: clipping the outlier lowers the total error
    # (S:261's [1,1,1,1,100] picks 1.0 on the 0.40..1.00 grid, so a denser column is used)
    w2 = np.array([[1.0] * 100 + [10.0]])
    _, _, clip2 = quant.rtn_weight_quantize(w2)
    assert clip2[0] < 1.0
    _, s0, _ = quant.rtn_weight_quantize(np.zeros((1, 8)))
    assert s0[0] == 1.0


def test_rtn_weight_search_is_argmin():
    # the chosen clip has the minimum squared error on the grid (definition, Z13)
    rng = np.random.default_rng(9)
    w = rng.standard_normal((4, 64))
    codes, scale, clip = quant.rtn_weight_quantize(w)
    for n in range(4):
        amax = np.max(np.abs(w[n]))
        errs = []
        for c in quant.CLIP_GRID:
            s = np.float64(np.float32(c * amax / 7))
            q = np.clip(np.rint(w[n] / s), -7, 7)
            errs.append(np.sum((w[n] - q * s) ** 2))
        assert np.sum((w[n] - codes[n] * np.float64(scale[n])) ** 2) == pytest.approx(min(errs), rel=1e-12)


def test_int_matmul_brute_force():
    # P9: exact integer accumulation vs a plain triple loop
    rng = np.random.default_rng(1)
    a = rng.integers(-7, 8, (8, 8))
    b = rng.integers(-7, 8, (8, 8))
    ref = [[sum(int(a[i, k]) * int(b[j, k]) for k in range(8)) for j in range(8)] for i in range(8)]
    assert gemm.int_matmul(a, b).tolist() == ref


def test_int_matmul_f64_exact_on_block_and_bounds():
    rng = np.random.default_rng(2)
    a = rng.integers(-7, 8, (16, 28672))
    b = rng.integers(-7, 8, (12, 28672))
    assert np.array_equal(gemm.int_matmul_exact_f64(a, b), gemm.int_matmul(a, b))
    # worst case fits int32, and so does the x256 scaled accumulator
    worst = gemm.int_matmul(np.full((1, 28672), 7), np.full((1, 28672), -7))
    assert abs(int(worst[0, 0])) == 49 * 28672 < 2**22
    assert 256 * 49 * 28672 < 2**31


def test_epilogue_closed_form():
    # P10
    g = GOLD["epilogue"]
    y = gemm.dequant_epilogue(np.array([[g["acc"]]]), np.array([g["sx"]], np.float32), np.array([g["sw"]], np.float32))
    assert y.dtype == np.float16 and float(y[0, 0]) == g["y"]


def test_asym_worked_example_and_bounds():
    # P11
    g = GOLD["asym_ramp"]
    codes, scale, zero = kv.quantize_asym_groups(np.array([g["group"]]), g["clip"])
    assert codes[0].tolist() == g["codes"] and int(zero[0]) == g["zero"]
    assert float(scale[0]) == g["scale_fp32"]
    rng = np.random.default_rng(3)
    x = rng.standard_normal((50, 128))
    codes, scale, zero = kv.quantize_asym_groups(x, 0.95)
    deq = kv.dequantize_asym(codes, scale, zero)
    for r in range(50):
        s = float(scale[r])
        lo, hi = 0.95 * min(x[r].min(), 0), 0.95 * max(x[r].max(), 0)
        inside = (x[r] >= lo) & (x[r] <= hi)
        # representable range is [(0 - z) s, (15 - z) s]; error <= s/2 inside it (+ z rounding)
        assert np.all(np.abs(x[r][inside] - deq[r][inside]) <= s + 1e-12)
        assert 0 <= zero[r] <= 15 and codes[r].min() >= 0 and codes[r].max() <= 15


def test_asym_brute_force():
    # codes are the nearest level of the affine grid (c - z) s, clamped to [0, 15]
    rng = np.random.default_rng(8)
    for _ in range(30):
        x = rng.standard_normal((1, 16)) * rng.uniform(0.1, 5)
        codes, scale, zero = kv.quantize_asym_groups(x, 0.95)
        s, z = float(scale[0]), int(zero[0])
        for v, c in zip(x[0], codes[0]):
            best = min(range(0, 16), key=lambda q: (abs(v - (q - z) * s), q % 2))
            if abs(v - (best - z) * s) != abs(v - (c - z) * s):
                raise AssertionError((v, c, best))


def test_asym_degenerate_groups():
    codes, scale, zero = kv.quantize_asym_groups(np.zeros((1, 128)))
    assert scale[0] == 1.0 and zero[0] == 0 and np.all(codes == 0)
    # constant positive group: range [0, 0.95c] includes 0
    codes, scale, zero = kv.quantize_asym_groups(np.full((1, 4), 2.0), 1.0)
    assert np.allclose(kv.dequantize_asym(codes, scale, zero), 2.0)


def test_attention_score_invariance():
    # P14: (Q H^)(K H^)^T = Q K^T per head
    rng = np.random.default_rng(6)
    q = rng.standard_normal((10, 4, 128))
    k = rng.standard_normal((12, 4, 128))
    h = had.hadamard(128)
    for hd in range(4):
        a = (q[:, hd] @ h.T) @ (k[:, hd] @ h.T).T
        assert np.allclose(a, q[:, hd] @ k[:, hd].T, atol=1e-11)


def test_kv_init_shapes_and_rotation():
    rng = np.random.default_rng(7)
    k = rng.standard_normal((3, 2, 128)).astype(np.float16)
    v = rng.standard_normal((3, 2, 128)).astype(np.float16)
    q = rng.standard_normal((3, 4, 128)).astype(np.float16)
    out = kv.kv_init(k, v, q)
    assert out["k_codes"].shape == (3, 2, 64) and out["k_codes"].dtype == np.uint8
    assert out["k_scale"].shape == (3, 2) and out["v_zero"].dtype == np.uint8
    assert np.allclose(out["k_rot"], had.apply_per_head(k.reshape(3, 256).astype(np.float64), 128).reshape(3, 2, 128))
    assert np.array_equal(out["v_rot"], v.astype(np.float64))
    assert out["q_rot"].dtype == np.float16


def test_quarot_linear_close_to_fp():
    # end-to-end sanity of the composed oracle: QuaRot W4A4 on the tiny config stays close
    # to the full-precision product (not a parity bar, a smoke pin of composition)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((16, 256)).astype(np.float16)
    x[:, 3] *= 50
    w = rng.standard_normal((256, 256)) / 16
    cw, _, sw = layer.quantize_weight(w, "full")
    y = layer.quarot_linear(x, cw, sw, "full").astype(np.float64)
    ref = x.astype(np.float64) @ w.T
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 0.25


# ---- 8-bit (A8W8): the same RTN definition with qmax = 127 (P:6, tab:rtn_results)
def test_sym8_brute_force_and_ties():
    rng = np.random.default_rng(5)
    for _ in range(30):
        y = rng.standard_normal((1, 11)) * rng.uniform(0.1, 10)
        codes, scale = quant.quantize_sym_rows(y, 0.9, qmax=127)
        s = float(scale[0])
        assert np.isclose(s, 0.9 * np.max(np.abs(y)) / 127, rtol=1e-6)
        for v, c in zip(y[0], codes[0]):
            assert c == _brute_code(v, s, qmax=127)
    # clip 1, amax 127 -> s = 1: exact ties round half to even, the top clamps at 127
    codes, scale = quant.quantize_sym_rows(np.array([[127.0, 2.5, -0.5, 126.5, -3.5]]), 1.0, qmax=127)
    assert scale[0] == 1.0 and codes[0].tolist() == [127, 2, 0, 126, -4]


def test_int8_matmul_exactness_bound():
    # 127 * 127 * K < 2^31 up to K = 131072 (the A8W8 ABI limit), and the fp64 path stays exact
    assert 127 * 127 * 131072 < 2 ** 31
    rng = np.random.default_rng(6)
    a = rng.integers(-127, 128, (5, 3000))
    b = rng.integers(-127, 128, (4, 3000))
    assert np.array_equal(gemm.int_matmul_exact_f64(a, b), a @ b.T)


# ---------------------------------------------------------------------------- group-wise (§8 f3)

def test_group_equal_to_row_when_group_is_k():
    # a single group per row is exactly the per-token rule (special case)
    rng = np.random.default_rng(5)
    y = rng.standard_normal((6, 256))
    c1, s1 = quant.quantize_sym_groups(y, 256)
    c2, s2 = quant.quantize_sym_rows(y)
    assert np.array_equal(c1, c2) and np.array_equal(s1[:, 0], s2)


def test_group_brute_force_nearest_level_and_bound():
    # P7 per group: every unclipped element's code is the nearest level of its own group's
    # scale (ties to even), |y - c s_g| <= s_g / 2, and no group's scale exceeds the row scale
    rng = np.random.default_rng(6)
    y = rng.standard_normal((4, 64)) * np.repeat(rng.uniform(0.01, 10, (4, 4)), 16, axis=1)
    y[1, 5] = 300.0  # one group with an outlier
    codes, scale = quant.quantize_sym_groups(y, 16)
    _, srow = quant.quantize_sym_rows(y)
    assert np.all(scale <= srow[:, None] * (1 + 1e-7))
    for r in range(4):
        for k in range(64):
            s = float(scale[r, k // 16])
            levels = np.arange(-7, 8)
            d = np.abs(y[r, k] - levels * s)
            best = levels[d == d.min()]
            c = codes[r, k]
            if abs(y[r, k]) <= 7 * s:
                assert c in best and (len(best) == 1 or c % 2 == 0)
                assert abs(y[r, k] - c * s) <= s / 2 * (1 + 1e-12)
            else:
                assert c == np.sign(y[r, k]) * 7


def test_group_zero_and_nonfinite_groups():
    y = np.zeros((1, 32))
    y[0, 20] = np.nan
    codes, scale = quant.quantize_sym_groups(y, 16)
    assert scale[0, 0] == 1.0 and np.isnan(scale[0, 1]) and not codes.any()


def test_group_linear_reduces_and_brute_force():
    from oracle import gemm as G
    rng = np.random.default_rng(7)
    cx = rng.integers(-7, 8, (3, 32))
    cw = rng.integers(-7, 8, (5, 32))
    sx = rng.uniform(0.1, 2, (3, 4)).astype(np.float32)
    sw = rng.uniform(0.1, 2, (5, 4)).astype(np.float32)
    y = G.group_linear(cx, sx, cw, sw)
    ref = np.zeros((3, 5))
    for m in range(3):  # triple loop by definition
        for n in range(5):
            for k in range(32):
                ref[m, n] += float(cx[m, k]) * float(cw[n, k]) * float(sx[m, k // 8]) * float(sw[n, k // 8])
    assert np.array_equal(y, ref.astype(np.float16))
    # equal scales in every group reduce to the per-token / per-channel epilogue
    y2 = G.group_linear(cx, np.repeat(sx[:, :1], 4, 1), cw, np.repeat(sw[:, :1], 4, 1))
    assert np.array_equal(y2, G.dequant_epilogue(G.int_matmul(cx, cw), sx[:, 0], sw[:, 0]))


def test_group_dequantize_matches_codes_times_group_scale():
    # x^ = c * s_g for the element's own group; with one group per row it is the per-row rule
    rng = np.random.default_rng(8)
    y = rng.standard_normal((3, 48))
    c, s = quant.quantize_sym_groups(y, 16)
    d = quant.dequantize_sym_groups(c, s)
    for r in range(3):
        for k in range(48):
            assert d[r, k] == c[r, k] * float(s[r, k // 16])
    c1, s1 = quant.quantize_sym_groups(y, 48)
    assert np.array_equal(quant.dequantize_sym_groups(c1, s1), quant.dequantize_sym_rows(c1, s1[:, 0]))
