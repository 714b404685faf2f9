"""Pins of the Append / Decode oracle against facts that do not come from
its own formula: closed-form special cases, the hard-attention limit, rotation invariance
(P:225), the GQA head mapping, exactness on representable caches, and the agreement of
Append with Init (routine consistency)."""
import numpy as np

from oracle import attention as oatt
from oracle import hadamard as ohad
from oracle import kv as okv
from oracle.glue import rope


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def test_single_token_returns_its_value():
    q = _rand((1, 2, 8), 0)
    k = _rand((1, 1, 2, 8), 1)
    v = _rand((1, 1, 2, 8), 2)
    o = oatt.attention_reference(q, k, v, [1])
    assert np.allclose(o[0, 0], v[0, 0, 0]) and np.allclose(o[0, 1], v[0, 0, 1])


def test_zero_query_averages_values():
    k = _rand((2, 9, 1, 16), 3)
    v = _rand((2, 9, 1, 16), 4)
    o = oatt.attention_reference(np.zeros((2, 1, 16)), k, v, [9, 4])
    assert np.allclose(o[0, 0], v[0, :9, 0].mean(0))
    assert np.allclose(o[1, 0], v[1, :4, 0].mean(0))  # rows past seq_len are ignored


def test_hard_attention_limit_picks_the_best_key():
    # scaling the scores up makes softmax an argmax: o -> v of the highest-scoring key
    q = _rand((1, 1, 32), 5)
    k = _rand((1, 40, 1, 32), 6)
    v = _rand((1, 40, 1, 32), 7)
    best = int(np.argmax(k[0, :, 0] @ q[0, 0]))
    o = oatt.attention_reference(q, k, v, [40], sm_scale=1e4)
    assert np.allclose(o[0, 0], v[0, best, 0], atol=1e-9)
    # and the score sign matters: the lowest key under a negative scale
    worst = int(np.argmin(k[0, :, 0] @ q[0, 0]))
    o = oatt.attention_reference(q, k, v, [40], sm_scale=-1e4)
    assert np.allclose(o[0, 0], v[0, worst, 0], atol=1e-9)


def test_rotating_q_and_k_leaves_attention_unchanged():
    # P:225 ("Since both queries and keys are rotated, the final attention scores remain unchanged")
    d = 64
    H = ohad.hadamard(d)
    q = _rand((2, 4, d), 8)
    k = _rand((2, 30, 4, d), 9)
    v = _rand((2, 30, 4, d), 10)
    o1 = oatt.attention_reference(q, k, v, [30, 17])
    o2 = oatt.attention_reference(q @ H.T, k @ H.T, v, [30, 17])
    assert np.allclose(o1, o2, atol=1e-12)


def test_gqa_head_mapping():
    # n_q = 4 query heads over n_kv = 2 KV heads: constant value rows identify the KV head
    q = _rand((1, 4, 8), 11)
    k = _rand((1, 5, 2, 8), 12)
    v = np.zeros((1, 5, 2, 8))
    v[..., 0, :] = 3.0
    v[..., 1, :] = -2.0
    o = oatt.attention_reference(q, k, v, [5])
    assert np.allclose(o[0, :2], 3.0) and np.allclose(o[0, 2:], -2.0)


def test_decode_is_exact_on_representable_caches():
    # codes / zeros / scales chosen directly: the dequantized cache is exactly (c - z) * s,
    # so decode must equal plain attention on those values (before the fp16 output rounding)
    rng = np.random.default_rng(13)
    B, S, n_kv, d = 2, 7, 2, 16
    c = oatt.empty_cache(B, S, n_kv, d)
    for key in ("k", "v"):
        c[f"{key}_codes"][:] = rng.integers(0, 16, (B, S, n_kv, d))
        c[f"{key}_zero"][:] = rng.integers(0, 16, (B, S, n_kv))
        c[f"{key}_scale"][:] = np.float32(0.25) * rng.integers(1, 5, (B, S, n_kv))
    kx = (c["k_codes"] - c["k_zero"][..., None]) * c["k_scale"][..., None].astype(np.float64)
    vx = (c["v_codes"] - c["v_zero"][..., None]) * c["v_scale"][..., None].astype(np.float64)
    q = rng.standard_normal((B, 4, d)).astype(np.float16)
    ref = oatt.attention_reference(q.astype(np.float64), kx, vx, [7, 3]).astype(np.float16)
    assert np.array_equal(oatt.decode_attention(q, c, [7, 3]), ref)


def test_append_at_position_zero_is_init():
    # RoPE at position 0 is the identity (angle 0), so appending into row 0 equals Init
    B, n_kv, n_q, d = 3, 2, 4, 128
    k = _rand((B, n_kv, d), 14).astype(np.float16)
    v = _rand((B, n_kv, d), 15).astype(np.float16)
    qn = _rand((B, n_q, d), 16).astype(np.float16)
    c = oatt.empty_cache(B, 4, n_kv, d)
    q_rot = oatt.kv_append(c, k, v, qn, [0, 0, 0])
    ref = okv.kv_init(k.astype(np.float64), v.astype(np.float64), qn.astype(np.float64))
    from oracle.quant import unpack_int4_unsigned
    assert np.array_equal(c["k_codes"][:, 0], unpack_int4_unsigned(ref["k_codes"]))
    assert np.array_equal(c["v_zero"][:, 0], ref["v_zero"])
    assert np.array_equal(q_rot, ref["q_rot"])


def test_append_then_decode_equals_init_of_the_whole_sequence():
    # Init of T+1 post-RoPE tokens == Init of T tokens + Append of token T (per-token groups)
    B, T, n_kv, n_q, d = 2, 6, 2, 4, 64
    rng = np.random.default_rng(17)
    k_pre = rng.standard_normal((B, T + 1, n_kv, d)).astype(np.float16)
    v = rng.standard_normal((B, T + 1, n_kv, d)).astype(np.float16)
    pos = np.arange(T + 1)
    k_post = np.stack([rope(k_pre[b].astype(np.float64), pos) for b in range(B)]).astype(np.float16)
    full = oatt.cache_init(k_post, v, T + 1)
    part = oatt.cache_init(k_post[:, :T], v[:, :T], T + 1)
    q = rng.standard_normal((B, n_q, d)).astype(np.float16)
    oatt.kv_append(part, k_pre[:, T], v[:, T], q, [T, T])
    for key in full:
        assert np.array_equal(full[key], part[key]), key
