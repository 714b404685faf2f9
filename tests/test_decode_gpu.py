"""GPU parity of the quantized-KV decoding routines: Append and Decode
against oracle/attention.py.  The decode cache is built by the ORACLE (cache_init) and handed
to both sides, so the kernel is judged on the same codes the oracle dequantizes."""
import numpy as np
import pytest
import torch

import synth
from oracle import attention as oatt
from oracle import hadamard as ohad
from oracle.quant import pack_int4, unpack_int4_unsigned
from tests import _parity as P

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def q():
    import paper_2404_00456_b200 as q
    q.lib()
    return q


def _to_gpu_cache(c: dict) -> dict:
    """Oracle cache (unpacked int64 codes) -> device tensors in the library layout."""
    out = {}
    for t in ("k", "v"):
        out[f"{t}_codes"] = torch.as_tensor(pack_int4(c[f"{t}_codes"]).astype(np.uint8), device=DEV)
        out[f"{t}_scale"] = torch.as_tensor(c[f"{t}_scale"].astype(np.float32), device=DEV)
        out[f"{t}_zero"] = torch.as_tensor(c[f"{t}_zero"].astype(np.uint8), device=DEV)
    return out


@pytest.mark.parametrize("B,n_kv,n_q,positions", [(4, 8, 64, [0, 5, 2047, 100]), (3, 32, 32, [7, 0, 1]),
                                                  (2, 2, 4, [3, 3])])
def test_kv_append_parity(q, B, n_kv, n_q, positions):
    d, s_max = 128, 2048
    k, v, qq = synth.kv_inputs(B, n_kv, n_q, d, seed=B + n_kv, device=DEV)
    pos = torch.tensor(positions, dtype=torch.int32, device=DEV)
    cache = q.kv_cache_empty(B, s_max, n_kv, d)
    q_dev = qq.clone()
    q.kv_append(k, v, q_dev, pos, cache)
    torch.cuda.synchronize()
    oc = oatt.empty_cache(B, s_max, n_kv, d)
    q_ref = oatt.kv_append(oc, k.cpu().numpy(), v.cpu().numpy(), qq.cpu().numpy(), positions)
    rows = (np.arange(B), np.asarray(positions))
    for t in ("k", "v"):
        got = unpack_int4_unsigned(cache[f"{t}_codes"].cpu().numpy()[rows])
        P.assert_codes(got, oc[f"{t}_codes"][rows], f"{t} codes")
        P.assert_scales(cache[f"{t}_scale"].cpu().numpy()[rows], oc[f"{t}_scale"][rows], f"{t} scale",
                        rel_tol=P.FP16_ULP_REL if t == "k" else P.SCALE_REL)  # RoPE'd K: Z22 rounding
    assert P.frob_rel(q_dev.cpu().numpy(), q_ref) <= 1e-3
    # every other row of the cache is untouched
    mask = np.ones((B, s_max), bool)
    mask[rows] = False
    assert not cache["k_codes"].cpu().numpy()[mask].any() and not cache["v_zero"].cpu().numpy()[mask].any()


@pytest.mark.parametrize("B,n_kv,n_q,seq_lens,s_max", [(3, 8, 64, [2048, 1, 777], 2048),
                                                       (2, 32, 32, [300, 2048], 2048),
                                                       (4, 4, 16, [1, 2, 255, 257], 512),
                                                       (1, 2, 4, [5000], 5000)])
def test_kv_decode_parity(q, B, n_kv, n_q, seq_lens, s_max):
    d = 128
    rng = np.random.default_rng(B * 7 + n_kv)
    T = max(seq_lens)
    k = rng.standard_normal((B, T, n_kv, d))
    k[..., 3] *= 20.0  # planted key outlier channel
    v = rng.standard_normal((B, T, n_kv, d))
    c = oatt.cache_init(k.astype(np.float16), v.astype(np.float16), s_max)  # K rotated by Init
    H = ohad.hadamard(d)
    q_rot = (rng.standard_normal((B, n_q, d)) @ H.T).astype(np.float16)
    ref = oatt.decode_attention(q_rot, c, seq_lens)
    out = q.kv_decode(torch.as_tensor(q_rot, device=DEV), _to_gpu_cache(c),
                      torch.tensor(seq_lens, dtype=torch.int32, device=DEV))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.isfinite(got).all()
    assert P.frob_rel(got, ref) <= P.FROB_REL
    for b in range(B):  # per sequence too (short and long sequences must both be right)
        assert P.frob_rel(got[b], ref[b]) <= P.FROB_REL, b


def test_kv_decode_single_row_returns_its_value(q):
    # a one-row cache: softmax over one element is 1, so o = v^_0 exactly (up to fp16)
    d, n_kv, n_q = 128, 2, 16
    rng = np.random.default_rng(3)
    c = oatt.cache_init(rng.standard_normal((1, 1, n_kv, d)).astype(np.float16),
                        rng.standard_normal((1, 1, n_kv, d)).astype(np.float16), 256)
    qr = rng.standard_normal((1, n_q, d)).astype(np.float16)
    out = q.kv_decode(torch.as_tensor(qr, device=DEV), _to_gpu_cache(c), torch.ones(1, dtype=torch.int32, device=DEV))
    v_hat = (c["v_codes"][0, 0] - c["v_zero"][0, 0][:, None]) * c["v_scale"][0, 0][:, None].astype(np.float64)
    ref = np.repeat(v_hat, n_q // n_kv, axis=0).astype(np.float16)
    assert P.max_fp16_ulp(out.cpu().numpy()[0], ref) <= 1


def test_decode_errors(q):
    qq = torch.zeros(1, 6, 128, dtype=torch.float16, device=DEV)
    cache = q.kv_cache_empty(1, 16, 2)
    with pytest.raises(q.QuarotError):  # G = 3 unsupported
        q.kv_decode(qq, cache, torch.ones(1, dtype=torch.int32, device=DEV))


def test_kv_decode_one_cta_per_pair_writes_output_directly(q):
    """With >= 2 (sequence, KV head) pairs per SM the grid runs one CTA per pair (nsplit 1): the
    decode kernel writes the fp16 output itself (one launch, no combine pass) — same parity bar."""
    B, n_kv, n_q, s_max, d = 40, 8, 64, 1024, 128
    rng = np.random.default_rng(11)
    seq_lens = [int(v) for v in rng.integers(1, s_max + 1, B)]
    seq_lens[0], seq_lens[1] = 1, s_max
    k = rng.standard_normal((B, s_max, n_kv, d))
    k[..., 5] *= 20.0
    v = rng.standard_normal((B, s_max, n_kv, d))
    c = oatt.cache_init(k.astype(np.float16), v.astype(np.float16), s_max)
    H = ohad.hadamard(d)
    q_rot = (rng.standard_normal((B, n_q, d)) @ H.T).astype(np.float16)
    ref = oatt.decode_attention(q_rot, c, seq_lens)
    out = q.kv_decode(torch.as_tensor(q_rot, device=DEV), _to_gpu_cache(c),
                      torch.tensor(seq_lens, dtype=torch.int32, device=DEV))
    launches = q.last_launch_count()
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    if B * n_kv >= 2 * nsm:
        assert launches == 1
    assert np.isfinite(got).all()
    for b in range(B):
        assert P.frob_rel(got[b], ref[b]) <= P.FROB_REL, b
