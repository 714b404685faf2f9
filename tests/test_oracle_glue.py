"""Pins for oracle/glue.py (decoder-layer glue) — CPU only."""
import numpy as np
import pytest
import scipy.special

from oracle import glue
from oracle import hadamard as had
from oracle import layer as olayer


def test_rmsnorm_forms():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 64)) * 3
    y = glue.rmsnorm(x, eps=0.0)
    # Eq. 3's x/||x|| up to the constant sqrt(d) (Z21), and unit RMS
    assert np.allclose(y, np.sqrt(64) * x / np.linalg.norm(x, axis=1, keepdims=True), atol=1e-13)
    assert np.allclose(np.sqrt(np.mean(y * y, axis=1)), 1.0, atol=1e-13)
    # commutes with orthogonal rotations (Eq. 3), eps included
    q = had.randomized(64, rng.choice([-1.0, 1.0], 64))
    assert np.allclose(glue.rmsnorm(x @ q.T) @ q, glue.rmsnorm(x), atol=1e-12)


def test_rmsnorm_quant_codes_equal_plain_quant():
    # a positive per-row scaling never changes the codes (P15): RMSNorm + quant == quant
    rng = np.random.default_rng(1)
    x = rng.standard_normal((4, 128)) * 5
    c1, _, s1 = glue.rmsnorm_quant(x)
    c2, _, s2 = olayer.hadamard_quant(x, "none")
    assert np.array_equal(c1, c2)
    rms = np.sqrt(np.mean(x * x, axis=1) + glue.RMS_EPS)
    assert np.allclose(s1, s2 / rms, rtol=1e-6)


def test_rope_properties():
    rng = np.random.default_rng(2)
    q = rng.standard_normal((6, 2, 8))
    k = rng.standard_normal((6, 2, 8))
    pos = np.arange(6)
    assert np.allclose(glue.rope(q, np.zeros(6)), q, atol=1e-15)  # position 0: identity
    rq = glue.rope(q, pos)
    # each (i, i + d/2) pair is rotated: norms preserved
    assert np.allclose(rq[..., :4] ** 2 + rq[..., 4:] ** 2, q[..., :4] ** 2 + q[..., 4:] ** 2, atol=1e-13)
    # relative-position property of the scores (Eqs. 10-12)
    s1 = np.einsum("hd,hd->h", glue.rope(q[:1], [5])[0], glue.rope(k[:1], [2])[0])
    s2 = np.einsum("hd,hd->h", glue.rope(q[:1], [105])[0], glue.rope(k[:1], [102])[0])
    assert np.allclose(s1, s2, atol=1e-10)


def test_rope_brute_force_rotation():
    # explicit 2x2 rotation by pos * theta^(-2i/d) on pair (i, i + d/2)
    d, pos = 8, 7
    x = np.arange(1, d + 1, dtype=np.float64)[None, None, :]
    y = glue.rope(x, [pos])[0, 0]
    for i in range(d // 2):
        a = pos * 10000.0 ** (-2 * i / d)
        rot = np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]]) @ np.array([x[0, 0, i], x[0, 0, i + d // 2]])
        assert np.allclose([y[i], y[i + d // 2]], rot, atol=1e-13)


def test_swiglu_closed_form():
    rng = np.random.default_rng(3)
    g, u = rng.standard_normal(100) * 4, rng.standard_normal(100)
    assert np.allclose(glue.swiglu(g, u), g * scipy.special.expit(g) * u, atol=1e-14)
    assert glue.swiglu(np.array([0.0]), np.array([5.0]))[0] == 0.0


def test_decoder_layer_close_to_full_precision():
    # composition pin: the quantized chain stays close to the same chain without quantization
    rng = np.random.default_rng(4)
    T, D, F, nh, nkv, d = 8, 256, 448, 2, 1, 128
    shapes = {"n_heads": nh, "n_kv": nkv, "head_dim": d, "ffn": F}
    x = (rng.standard_normal((T, D)) * 0.5).astype(np.float16)
    z = rng.standard_normal((T, D)).astype(np.float16)
    wf = {"qkv": rng.standard_normal(((nh + 2 * nkv) * d, D)) / 16, "o": rng.standard_normal((D, D)) / 16,
          "gate_up": rng.standard_normal((2 * F, D)) / 16, "down": rng.standard_normal((D, F)) / 21}
    modes = {"qkv": "none", "o": "across_heads", "gate_up": "none", "down": "full"}
    w = {}
    for n in wf:
        c, _, s = olayer.quantize_weight(wf[n], modes[n], d)
        w[n] = (c, s)
    out = glue.decoder_layer(x, z, w, np.arange(T), shapes)
    # full precision reference of the same (rotated) layer
    h = glue.rmsnorm(x.astype(np.float64))
    o = olayer.online_transform(z, "across_heads", d) @ olayer.rotate_weight(wf["o"], "across_heads", d).T + x
    gu = glue.rmsnorm(o) @ wf["gate_up"].T
    act = glue.swiglu(gu[:, :F], gu[:, F:])
    ref = olayer.online_transform(act, "full") @ olayer.rotate_weight(wf["down"], "full").T + o
    rel = np.linalg.norm(out["out"].astype(np.float64) - ref) / np.linalg.norm(ref)
    assert rel < 0.3, rel  # W4A4 RTN noise of three chained random linears
    assert out["cache"]["k_codes"].shape == (T, nkv, d // 2)
    # negative control: a down_proj weight that was NOT rotated breaks the pairing (P16)
    w_bad = dict(w)
    c, _, s = olayer.quantize_weight(wf["down"], "none", d)
    w_bad["down"] = (c, s)
    bad = glue.decoder_layer(x, z, w_bad, np.arange(T), shapes)
    rel_bad = np.linalg.norm(bad["out"].astype(np.float64) - ref) / np.linalg.norm(ref)
    assert rel_bad > 2 * rel, (rel, rel_bad)


def _ulp16(a, b):
    a = np.asarray(a, np.float16).view(np.int16).astype(np.int64)
    b = np.asarray(b, np.float16).view(np.int16).astype(np.int64)
    a = np.where(a < 0, -(a & 0x7FFF), a)
    b = np.where(b < 0, -(b & 0x7FFF), b)
    return np.abs(a - b)


def test_fp16_glue_ops_match_torch_half():
    """Pin of reading Z23 (every linear output is FP16, the model's default precision):
    the oracle's FP16 ops equal PyTorch's own fp16 CPU kernels — F.silu on a half tensor, the
    half product, the half add — an independent implementation of the same FP16 model ops."""
    import torch
    rng = np.random.default_rng(5)
    g = (rng.standard_normal(200000) * 4).astype(np.float16)
    u = (rng.standard_normal(200000) * 2).astype(np.float16)
    g[:6] = [0.0, -0.0, 65504.0, -65504.0, 6e-8, -20.0]
    tg, tu = torch.from_numpy(g), torch.from_numpy(u)
    s_t = torch.nn.functional.silu(tg).numpy()
    s_o = glue.silu_fp16(g)
    d = _ulp16(s_o, s_t)
    # torch evaluates silu in fp32 before its one rounding; fp64 vs fp32 may straddle a rounding
    # boundary only in rare near-tie cases
    assert d.max() <= 1 and np.count_nonzero(d) <= 2e-3 * d.size, (d.max(), np.count_nonzero(d))
    # with the same fp16 silu output, the product and the add are single correctly rounded ops
    a_t = (torch.from_numpy(s_o) * tu).numpy()
    assert np.array_equal(glue.swiglu_fp16(g, u).view(np.int16), a_t.view(np.int16))
    r = (rng.standard_normal(200000) * 3).astype(np.float16)
    assert np.array_equal(glue.add_fp16(r, u).view(np.int16), (torch.from_numpy(r) + tu).numpy().view(np.int16))


def test_fp16_glue_special_cases():
    # silu(0) = 0; large positive g: silu(g) = g exactly in fp16; large negative: -0/0
    assert glue.silu_fp16(np.float16([0.0]))[0] == 0
    assert glue.silu_fp16(np.float16([30.0]))[0] == np.float16(30.0)
    assert glue.silu_fp16(np.float16([-30.0]))[0] == 0
    # up = 1: the SwiGLU is the fp16 SiLU itself; residual add of 0 is the identity
    g = np.float16([0.5, -1.25, 3.0, 7.5])
    assert np.array_equal(glue.swiglu_fp16(g, np.ones(4, np.float16)), glue.silu_fp16(g))
    assert np.array_equal(glue.add_fp16(g, np.zeros(4, np.float16)), g)
    # fp16 overflow of the add saturates to inf like the FP16 model
    assert np.isinf(glue.add_fp16(np.float16([65504.0]), np.float16([65504.0]))[0])


def test_decoder_layer_outputs_are_fp16_model_ops():
    """decoder_layer's intermediates are fp16 and its act is the FP16 model's SwiGLU of the fp16
    gate/up linear output, recomputed here with PyTorch's own half kernels (within 1 ulp)."""
    rng = np.random.default_rng(6)
    T, D, F, nh, nkv, d = 4, 256, 448, 2, 1, 128
    shapes = {"n_heads": nh, "n_kv": nkv, "head_dim": d, "ffn": F}
    x = (rng.standard_normal((T, D)) * 0.5).astype(np.float16)
    z = rng.standard_normal((T, D)).astype(np.float16)
    w = {"qkv": (rng.integers(-7, 8, ((nh + 2 * nkv) * d, D)), np.full((nh + 2 * nkv) * d, 0.02, np.float32)),
         "o": (rng.integers(-7, 8, (D, D)), np.full(D, 0.02, np.float32)),
         "gate_up": (rng.integers(-7, 8, (2 * F, D)), np.full(2 * F, 0.02, np.float32)),
         "down": (rng.integers(-7, 8, (D, F)), np.full(D, 0.02, np.float32))}
    out = glue.decoder_layer(x, z, w, np.arange(T), shapes)
    assert out["o"].dtype == out["act"].dtype == out["out"].dtype == out["gate_up"].dtype == np.float16
    import torch
    gu = torch.from_numpy(out["gate_up"])
    act_t = (torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]).numpy()
    assert _ulp16(out["act"], act_t).max() <= 1
