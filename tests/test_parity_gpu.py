"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element
on seeded inputs.  Bars (BASELINE.json north_star): int32 accumulators bit-exact; INT4
codes within one step on <= 1e-4 of elements; fp16 outputs within 1e-2 relative Frobenius;
scales within 1e-5 relative."""
import numpy as np
import pytest
import torch

import synth
from oracle import gemm as ogemm
from oracle import kv as okv
from oracle import layer as olayer
from oracle import quant as oquant
from tests import _parity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    from paper_2404_00456_b200 import quarot
    quarot.lib()
    assert torch.cuda.is_available()
    return quarot


DEV = "cuda"


def _adversarial_rows(k: int) -> np.ndarray:
    """Edge rows: zero, exact ties at clip 1 scale, one huge outlier, fp16 extremes,
    subnormals, alternating signs."""
    rows = []
    rows.append(np.zeros(k))
    r = np.zeros(k); r[0] = 7.0; r[1:8] = [0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 3.5]; rows.append(r)
    r = np.random.default_rng(0).standard_normal(k) * 0.01; r[k // 3] = 1000.0; rows.append(r)
    r = np.full(k, 65504.0); r[::2] = -65504.0; rows.append(r)
    r = np.full(k, 6e-8); r[1::3] = -6e-8; rows.append(r)
    r = np.ones(k); r[1::2] = -1; rows.append(r)
    return np.stack(rows).astype(np.float16)


def _hq_compare(q, x16: torch.Tensor, mode: str, head_dim: int = 128, clip=0.9, rows=None):
    xq, xs = q.hadamard_quant(x16, mode, head_dim, clip)
    torch.cuda.synchronize()
    sel = slice(None) if rows is None else torch.as_tensor(rows, device=x16.device)
    xh = x16[sel].float().cpu().numpy().astype(np.float64)
    ref_codes, _, ref_scale = olayer.hadamard_quant(xh, mode, head_dim, clip)
    got_codes = P.unpack_signed(xq[sel].cpu().numpy())
    st = P.assert_codes(got_codes, ref_codes, f"{mode} K={x16.shape[1]}")
    P.assert_scales(xs[sel].cpu().numpy(), ref_scale, f"{mode} K={x16.shape[1]}")
    # no code -8 is ever produced (symmetric range [-7, 7], Z8)
    assert not np.any(got_codes == -8)
    return xq, xs, st


@pytest.mark.parametrize("mode,K,hd", [
    ("none", 256, 128), ("none", 4096, 128), ("none", 8192, 128), ("none", 11008, 128),
    ("full", 256, 128), ("full", 448, 128), ("full", 688, 128), ("full", 4096, 128),
    ("full", 11008, 128), ("full", 28672, 128), ("full", 640, 128), ("full", 5120, 128), ("full", 13824, 128),
    ("across_heads", 512, 128), ("across_heads", 4096, 128), ("across_heads", 8192, 128),
    ("across_heads", 8192, 64),
])
def test_hadamard_quant_parity(q, mode, K, hd):
    M = 37  # ragged
    x = synth.activations(M, K, "outlier", seed=K + len(mode), device=DEV)
    x = torch.cat([x, torch.from_numpy(_adversarial_rows(K)).to(DEV)], 0).contiguous()
    _hq_compare(q, x, mode, hd)


def test_hadamard_quant_nonfinite_rows(q):
    K = 4096
    x = synth.activations(4, K, "normal", seed=1, device=DEV)
    x[1, 5] = float("nan")
    x[2, 7] = float("inf")
    for mode in ("none", "full", "across_heads"):
        xq, xs = q.hadamard_quant(x, mode)
        s = xs.cpu().numpy()
        assert np.isfinite(s[0]) and np.isnan(s[1]) and np.isnan(s[2]) and np.isfinite(s[3])
        codes = P.unpack_signed(xq.cpu().numpy())
        assert np.all(codes[1] == 0) and np.all(codes[2] == 0)


def test_hadamard_quant_strided_and_split_invariance(q):
    # leading dimensions > width, and row splits give bitwise identical results
    K, M = 4096, 64
    big = synth.activations(M, K + 64, "outlier", seed=3, device=DEV)
    x = big[:, :K]
    for mode in ("none", "full", "across_heads"):
        xq, xs = q.hadamard_quant(x, mode)
        xq2, xs2 = q.hadamard_quant(x.contiguous(), mode)
        a1, s1 = q.hadamard_quant(x[:20], mode)
        a2, s2 = q.hadamard_quant(x[20:], mode)
        assert torch.equal(xq, xq2) and torch.equal(xs, xs2)
        assert torch.equal(torch.cat([a1, a2]), xq) and torch.equal(torch.cat([s1, s2]), xs)


@pytest.mark.parametrize("mode,K", [("full", 28672), ("full", 11008), ("full", 13824), ("full", 5120),
                                    ("across_heads", 8192), ("across_heads", 4096)])
def test_hadamard_quant_tcgen05_paths(q, mode, K):
    """The tcgen05 quantizers (FULL 1024x28 / 64x172, ACROSS_HEADS n_h 32/64) on what the small
    parity cases do not reach: several rows per persistent CTA (the TMEM / smem rings wrap),
    a leading dimension > K, row splits, and non-finite rows."""
    M = 3 * 148 + 5
    big = synth.activations(M, K + 64, "swiglu" if mode == "full" else "normal", seed=K, device=DEV)
    big[7, 11] = float("nan")
    big[300, 5] = float("inf")
    x = big[:, :K]
    xq, xs = q.hadamard_quant(x, mode)
    xq2, xs2 = q.hadamard_quant(x.contiguous(), mode)
    bits = lambda t: t.view(torch.int32)  # NaN scales compare bitwise
    assert torch.equal(xq, xq2) and torch.equal(bits(xs), bits(xs2))
    a1, s1 = q.hadamard_quant(x[:151], mode)
    a2, s2 = q.hadamard_quant(x[151:], mode)
    assert torch.equal(torch.cat([a1, a2]), xq) and torch.equal(bits(torch.cat([s1, s2])), bits(xs))
    s = xs.cpu().numpy()
    assert np.isnan(s[7]) and np.isnan(s[300]) and np.isfinite(np.delete(s, [7, 300])).all()
    codes = P.unpack_signed(xq.cpu().numpy())
    assert np.all(codes[7] == 0) and np.all(codes[300] == 0)
    rows = [0, 1, 147, 148, 149, 296, 297, 444, 447, M - 1]  # CTA 0 rows 0..3, tail rows
    _hq_compare(q, x.contiguous(), mode, rows=rows)


def _rand_codes_packed(rows, k, seed):
    return synth.packed_weight_codes(rows, k, seed, device=DEV)


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (1, 256, 256), (300, 776, 512), (129, 264, 4096),
                                   (257, 512, 11008), (64, 256, 28672), (600, 1024, 8192)])
def test_int4_gemm_s32_bit_exact(q, M, N, K):
    xq = _rand_codes_packed(M, K, seed=M)
    wq = _rand_codes_packed(N, K, seed=N + 1)
    acc = q.int4_matmul_s32(xq, wq)
    torch.cuda.synchronize()
    cx = P.unpack_signed(xq.cpu().numpy())
    cw = P.unpack_signed(wq.cpu().numpy())
    ref = ogemm.int_matmul_exact_f64(cx, cw) if K > 4096 else ogemm.int_matmul(cx, cw)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("M,N,K", [(2085, 4120, 4096), (1100, 8200, 2176), (2085, 4120, 28672)])
def test_int4_gemm_multi_tile_full_matrix(q, M, N, K):
    # more 256x256 tiles than CTA pairs (>= 2 tiles per persistent pair), so the staging and
    # operand rings run across tile boundaries; ragged M and N, and a K % 256 == 128 tail.
    # Every element is checked: a ring race corrupts ~1 % of entries by one k-step.
    xq = _rand_codes_packed(M, K, seed=M)
    wq = _rand_codes_packed(N, K, seed=N + 1)
    xs = torch.rand(M, device=DEV) * 0.1 + 0.01
    ws = synth.weight_scales(N, seed=9, device=DEV)
    acc = q.int4_matmul_s32(xq, wq)
    y = q.int4_linear(xq, xs, wq, ws)
    torch.cuda.synchronize()
    ref = ogemm.int_matmul_exact_f64(P.unpack_signed(xq.cpu().numpy()), P.unpack_signed(wq.cpu().numpy()))
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), ref)
    yref = ogemm.dequant_epilogue(ref, xs.cpu().numpy(), ws.cpu().numpy())
    assert P.max_fp16_ulp(y.cpu().numpy(), yref) <= 2


def test_int4_gemm_extreme_codes_bit_exact(q):
    # all +-7: the largest accumulators (|acc| = 49 K); checks the x256 scaling path
    M, N, K = 130, 264, 28672
    xq = torch.full((M, K // 2), 0x77, dtype=torch.uint8, device=DEV)
    wq = torch.full((N, K // 2), 0x99, dtype=torch.uint8, device=DEV)  # -7, -7
    wq[::2] = 0x77
    acc = q.int4_matmul_s32(xq, wq).cpu().numpy()
    assert np.all(acc[:, 0::2] == 49 * K) and np.all(acc[:, 1::2] == -49 * K)


@pytest.mark.parametrize("M,N,K", [(200, 264, 256), (129, 1024, 4096), (300, 512, 28672)])
def test_int4_linear_epilogue(q, M, N, K):
    xq = _rand_codes_packed(M, K, seed=7)
    wq = _rand_codes_packed(N, K, seed=8)
    xs = torch.rand(M, device=DEV) * 0.1 + 0.01
    ws = synth.weight_scales(N, seed=9, device=DEV)
    y = q.int4_linear(xq, xs, wq, ws)
    torch.cuda.synchronize()
    cx = P.unpack_signed(xq.cpu().numpy())
    cw = P.unpack_signed(wq.cpu().numpy())
    acc = ogemm.int_matmul_exact_f64(cx, cw)
    ref = ogemm.dequant_epilogue(acc, xs.cpu().numpy(), ws.cpu().numpy())
    got = y.cpu().numpy()
    assert P.frob_rel(got, ref) <= P.FROB_REL
    assert P.max_fp16_ulp(got, ref) <= 2


def test_tiny_config_end_to_end(q):
    # BASELINE config 0: 16 tokens x 256 -> 256, power-of-two Hadamard, RTN weights
    x = synth.activations(16, 256, "outlier", seed=0, device="cpu", n_outliers=1)
    w = synth.dense_weight(256, 256, seed=1).double().numpy()
    cw, pw, sw = olayer.quantize_weight(w, "full")
    y = q.quarot_linear(x.to(DEV), torch.from_numpy(pw).to(DEV), torch.from_numpy(sw).to(DEV), "full")
    ref = olayer.quarot_linear(x.double().numpy(), cw, sw, "full")
    assert P.frob_rel(y.cpu().numpy(), ref) <= P.FROB_REL
    # and close to the full-precision product (QuaRot W4A4 on a rotated layer)
    fp = x.double().numpy() @ w.T
    assert P.frob_rel(y.cpu().numpy(), fp) < 0.2


@pytest.mark.parametrize("T,n_kv,n_q,hd,flags", [(37, 8, 64, 128, 1), (5, 2, 0, 128, 1), (9, 4, 4, 64, 3),
                                                 (3, 2, 2, 256, 1), (11, 8, 8, 128, 0)])
def test_kv_quant_parity(q, T, n_kv, n_q, hd, flags):
    k, v, qq = synth.kv_inputs(T, n_kv, n_q, hd, seed=T, device=DEV)
    k[0, 0] = 0  # degenerate group
    q_dev = None if qq is None else qq.clone()
    out = q.kv_quant(k, v, q_dev, flags=flags)
    torch.cuda.synchronize()
    ref = okv.kv_init(k.cpu().numpy(), v.cpu().numpy(), None if qq is None else qq.cpu().numpy(),
                      rotate_k=bool(flags & 1), rotate_v=bool(flags & 2))
    for t in ("k", "v"):
        P.assert_codes(P.unpack_unsigned(out[f"{t}_codes"].cpu().numpy()),
                       P.unpack_unsigned(ref[f"{t}_codes"]), f"{t} codes")
        P.assert_codes(out[f"{t}_zero"].cpu().numpy(), ref[f"{t}_zero"], f"{t} zero")
        P.assert_scales(out[f"{t}_scale"].cpu().numpy(), ref[f"{t}_scale"], f"{t} scale")
    assert out["k_scale"][0, 0].item() == 1.0 and out["k_zero"][0, 0].item() == 0
    if qq is not None:
        assert P.max_fp16_ulp(q_dev.cpu().numpy(), ref["q_rot"]) <= 1


def test_deterministic_repeat(q):
    x = synth.activations(512, 28672, "swiglu", seed=5, device=DEV)
    a = q.hadamard_quant(x, "full")
    b = q.hadamard_quant(x, "full")
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    wq = _rand_codes_packed(512, 28672, seed=6)
    ws = synth.weight_scales(512, seed=6, device=DEV)
    y1 = q.int4_linear(a[0], a[1], wq, ws)
    y2 = q.int4_linear(a[0], a[1], wq, ws)
    assert torch.equal(y1, y2)


def test_errors_raise_without_launch(q):
    x = torch.zeros(4, 192, dtype=torch.float16, device=DEV)
    with pytest.raises(q.QuarotError):
        q.hadamard_quant(x, "full")  # 192 = 2^4 * 12 unsupported
    assert q.last_launch_count() == 0


def test_kv_quant_from_fused_qkv_views(q):
    # K, V, Q read straight out of a fused QKV output [T, (n_q + 2 n_kv) d] (strided views)
    T, n_q, n_kv, d = 33, 8, 2, 128
    fused = synth.activations(T, (n_q + 2 * n_kv) * d, "normal", seed=2, device=DEV)
    qv = fused[:, : n_q * d].view(T, n_q, d)
    kv_ = fused[:, n_q * d:(n_q + n_kv) * d].view(T, n_kv, d)
    vv = fused[:, (n_q + n_kv) * d:].view(T, n_kv, d)
    k_ref, v_ref, q_ref = (t.cpu().numpy().copy() for t in (kv_, vv, qv))
    out = q.kv_quant(kv_, vv, qv)
    ref = okv.kv_init(k_ref, v_ref, q_ref)
    P.assert_codes(P.unpack_unsigned(out["k_codes"].cpu().numpy()), P.unpack_unsigned(ref["k_codes"]), "k")
    P.assert_codes(P.unpack_unsigned(out["v_codes"].cpu().numpy()), P.unpack_unsigned(ref["v_codes"]), "v")
    assert P.max_fp16_ulp(qv.cpu().numpy(), ref["q_rot"]) <= 1
    # K and V regions of the fused buffer are untouched
    assert np.array_equal(kv_.cpu().numpy(), k_ref) and np.array_equal(vv.cpu().numpy(), v_ref)


@pytest.mark.parametrize("K,group", [(8192, 128), (4096, 64), (11008, 256), (256, 128)])
def test_hadamard_quant_group_parity(q, K, group):
    """group-wise INT4 quantizer against the oracle (codes within one step on
    <= 1e-4 of elements, scales 1e-5), with the adversarial rows and a non-finite group."""
    if K % group:
        pytest.skip("group must divide K")
    M = 37
    x = synth.activations(M, K, "outlier", seed=K + group, device=DEV)
    x = torch.cat([x, torch.from_numpy(_adversarial_rows(K)).to(DEV)], 0).contiguous()
    x[3, group + 1] = float("nan")
    xq, xs = q.hadamard_quant_group(x, group)
    torch.cuda.synchronize()
    ref_c, ref_s = oquant.quantize_sym_groups(x.float().cpu().numpy().astype(np.float64), group)
    got = P.unpack_signed(xq.cpu().numpy())
    P.assert_codes(got, ref_c, f"group {group} K={K}")
    s = xs.cpu().numpy()
    assert np.isnan(s[3, 1]) and np.all(got[3, group:2 * group] == 0)
    fin = np.isfinite(ref_s)
    assert np.array_equal(fin, np.isfinite(s))
    P.assert_scales(s[fin], ref_s[fin], f"group {group} K={K}")


def _group_case(M, N, K, G, seed):
    rng = np.random.default_rng(seed)
    cx = rng.integers(-7, 8, (M, K)).astype(np.int8)
    cw = rng.integers(-8, 8, (N, K)).astype(np.int8)
    sx = rng.uniform(0.001, 0.02, (M, K // G)).astype(np.float32)
    sw = rng.uniform(0.001, 0.02, (N, K // G)).astype(np.float32)
    return cx, cw, sx, sw


def _assert_group_out(got, ref):
    assert P.frob_rel(got, ref) <= 1e-2
    ulp = np.abs(got.astype(np.float32) - ref.astype(np.float32)) / np.maximum(
        np.abs(np.spacing(ref.astype(np.float16))).astype(np.float32), 1e-30)
    assert np.quantile(ulp, 0.999) <= 2.0 and ulp.max() <= 4.0


@pytest.mark.parametrize("G", [64, 128, 256])
@pytest.mark.parametrize("M,N,K", [(300, 520, 512), (128, 256, 256), (513, 1032, 1024), (64, 256, 4096),
                                   (1100, 776, 2304)])
def test_int4_linear_group_parity(q, M, N, K, G):
    """group-wise W4A4 GEMM on PACKED INT4 codes (G = 64 / 128 / 256, weight codes
    incl. -8) against the oracle's group_linear (fp64) on the same codes and scales: fp16 outputs
    within 1e-2 relative Frobenius, 2 fp16 ulp at the 99.9th percentile (4 max).  Covers ragged M / N,
    several tiles per CTA pair and K / 256 k-blocks of G / 32 MMAs per group."""
    from oracle import gemm as og
    from oracle import quant as oq
    cx, cw, sx, sw = _group_case(M, N, K, G, M + N + K + G)
    xq = torch.from_numpy(oq.pack_int4(cx.astype(np.int64))).to(DEV)
    wq = torch.from_numpy(oq.pack_int4(cw.astype(np.int64))).to(DEV)
    y = q.int4_linear_group(xq, torch.from_numpy(sx).to(DEV), wq, torch.from_numpy(sw.T.copy()).to(DEV), group=G)
    torch.cuda.synchronize()
    _assert_group_out(y.cpu().numpy(), og.group_linear(cx, sx, cw, sw))


def test_int4_linear_group_extreme_codes(q):
    """Largest per-group sums (|acc_g| = 7 * 8 * G at G = 256): the accumulator bias stays exact."""
    from oracle import gemm as og
    from oracle import quant as oq
    M, N, K, G = 256, 256, 1024, 256
    cx = np.full((M, K), 7, np.int8)
    cx[1::2] = -7
    cw = np.full((N, K), -8, np.int8)
    cw[::3] = 7
    sx = np.full((M, K // G), 1.0 / 1024, np.float32)
    sw = np.full((N, K // G), 1.0 / 64, np.float32)
    y = q.int4_linear_group(torch.from_numpy(oq.pack_int4(cx.astype(np.int64))).to(DEV), torch.from_numpy(sx).to(DEV),
                            torch.from_numpy(oq.pack_int4(cw.astype(np.int64))).to(DEV),
                            torch.from_numpy(sw.T.copy()).to(DEV), group=G)
    ref = og.group_linear(cx, sx, cw, sw)
    assert np.array_equal(y.cpu().numpy(), ref.astype(np.float16))


@pytest.mark.parametrize("M,N,K", [(300, 520, 512), (513, 1032, 1024)])
def test_int4_linear_group8_parity(q, M, N, K):
    """quarot_int4_linear_group8: the int8-stored-codes variant (G = 128) on the same oracle."""
    from oracle import gemm as og
    cx, cw, sx, sw = _group_case(M, N, K, 128, M + N + K)
    y = q.int4_linear_group8(torch.from_numpy(cx).to(DEV), torch.from_numpy(sx).to(DEV),
                             torch.from_numpy(cw).to(DEV), torch.from_numpy(sw.T.copy()).to(DEV))
    torch.cuda.synchronize()
    _assert_group_out(y.cpu().numpy(), og.group_linear(cx, sx, cw, sw))


@pytest.mark.parametrize("mode,G", [("none", 128), ("full", 64), ("across_heads", 256)])
def test_group_pipeline_quant_then_linear(q, mode, G):
    """quarot_hadamard_quant_group (packed) -> quarot_int4_linear_group against the oracle pipeline
    (online transform, quantize_sym_groups, group_linear); the int8-stored quantizer agrees."""
    from oracle import gemm as og
    from oracle import layer as olayer
    M, K, N = 200, 4096, 264
    x = synth.activations(M, K, "outlier", seed=11, device=DEV)
    xq4, xs4 = q.hadamard_quant_group(x, G, mode=mode)
    xq8, xs8 = q.hadamard_quant_group8(x, G, mode=mode)
    torch.cuda.synchronize()
    got_c = P.unpack_signed(xq4.cpu().numpy())
    assert np.array_equal(got_c, xq8.cpu().numpy().astype(np.int64))
    assert torch.equal(xs4, xs8)
    rng = np.random.default_rng(12)
    cw = rng.integers(-7, 8, (N, K)).astype(np.int8)
    sw = rng.uniform(0.001, 0.02, (N, K // G)).astype(np.float32)
    from oracle import quant as oq
    wq = torch.from_numpy(oq.pack_int4(cw.astype(np.int64))).to(DEV)
    y = q.int4_linear_group(xq4, xs4, wq, torch.from_numpy(sw.T.copy()).to(DEV), group=G)
    torch.cuda.synchronize()
    rc, rs = oquant.quantize_sym_groups(olayer.online_transform(x.float().cpu().numpy().astype(np.float64), mode), G)
    P.assert_codes(got_c, rc, f"group {G} {mode} codes")
    # on the GPU's own codes and scales the GEMM matches group_linear to fp16 ulps; against the
    # oracle's codes (<= 1e-4 flips) within the 1e-2 end-to-end bar
    _assert_group_out(y.cpu().numpy(), og.group_linear(got_c.astype(np.int8), xs4.cpu().numpy(), cw, sw))
    assert P.frob_rel(y.cpu().numpy(), og.group_linear(rc, rs, cw, sw)) <= 1e-2


@pytest.mark.parametrize("clip", [0.9, 1.0, 0.5])
def test_full28_kperm_vs_oracle_clamp_paths(q, clip):
    """The KPERM FULL K = 1024 x 28 kernel (the chain's down_proj quantizer) against the oracle,
    un-permuted: its clamp-free packing (warps none of whose lanes can reach |v * inv| >= 7.5)
    and its clamping path.  Gaussian-like rows take mostly the clamp-free path, the adversarial
    rows (a spike: every transformed element at amax, so every warp clamps; ties; extremes) the
    clamping one, and clip 0.5 saturates many codes in every row."""
    K = 28672
    x = synth.activations(40, K, "swiglu", seed=11, device=DEV)
    x = torch.cat([x, torch.from_numpy(_adversarial_rows(K)).to(DEV)], 0).contiguous()
    xq, xs = q.hadamard_quant(x, "full", clip_ratio=clip, kperm=True)
    perm = q.full_kperm(K)
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(K)
    nat = q.permute_k_packed(xq, inv)
    ref_codes, _, ref_scale = olayer.hadamard_quant(x.float().cpu().numpy().astype(np.float64), "full", 128, clip)
    got = P.unpack_signed(nat.cpu().numpy())
    P.assert_codes(got, ref_codes, f"full-28 kperm clip={clip}")
    P.assert_scales(xs.cpu().numpy(), ref_scale, f"full-28 kperm clip={clip}")
    assert not np.any(got == -8) and np.abs(got).max() == 7


@pytest.mark.parametrize("n_kv,n_q", [(8, 64), (32, 32)])
def test_kv_tc_value_rows_edge_cases(q, n_kv, n_q):
    """KV Init's V rows (tcgen05 kernel: copied to registers, fp16 min / max) on edge rows —
    zero, constant, +-0 mixes, a NaN, an inf, fp16 extremes, a single spike — against the
    oracle's kv_init and bitwise against the CUDA-core kernel (quarot_debug_kv_variant 1), an
    independent implementation of the same arithmetic."""
    T, d = 64, 128
    k, v, qq = synth.kv_inputs(T, n_kv, n_q, d, seed=21, device=DEV)
    v[0, 0] = 0
    v[1, 0] = 0.75
    v[2, 0, ::2] = 0.0
    v[2, 0, 1::2] = -0.0
    v[3, 0, 5] = float("nan")
    v[4, 0, 7] = float("inf")
    v[5, 0, ::2] = 65504.0
    v[5, 0, 1::2] = -65504.0
    v[6, 0] = 0
    v[6, 0, 17] = -3.0
    outs = []
    for variant in (0, 1):
        q.lib().quarot_debug_kv_variant(variant)
        try:
            qc = qq.clone()
            outs.append(q.kv_quant(k, v, qc))
        finally:
            q.lib().quarot_debug_kv_variant(0)
    torch.cuda.synchronize()
    # V is not rotated: both kernels do exactly the same arithmetic (K goes through H_128 on the
    # tensor core in one and in butterflies in the other, so its fp32 sums may round differently)
    for key in ("v_codes", "v_zero"):
        assert torch.equal(outs[0][key], outs[1][key]), key
    assert torch.equal(outs[0]["v_scale"].view(torch.int32), outs[1]["v_scale"].view(torch.int32))  # NaNs bitwise
    sv = outs[0]["v_scale"].cpu().numpy()
    assert np.isnan(sv[3, 0]) and np.isnan(sv[4, 0]) and sv[0, 0] == 1.0
    vc = P.unpack_unsigned(outs[0]["v_codes"].cpu().numpy())
    assert np.all(vc[3, 0] == 0) and np.all(vc[4, 0] == 0)
    fin = np.ones(T, bool)
    fin[[3, 4]] = False
    ref = okv.kv_init(k.cpu().numpy()[fin], v.cpu().numpy()[fin], None if qq is None else qq.cpu().numpy()[fin])
    P.assert_codes(vc[fin], P.unpack_unsigned(ref["v_codes"]), "v codes")
    P.assert_scales(sv[fin], ref["v_scale"], "v scale")
