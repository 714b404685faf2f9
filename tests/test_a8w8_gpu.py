"""GPU parity of the A8W8 path (QuaRot's 8-bit RTN configuration, P:6,
tab:rtn_results): the int8 per-token quantizer (mode NONE, optional RMSNorm) and the native
kind::i8 GEMM, against the oracle (qmax = 127)."""
import numpy as np
import pytest
import torch

import synth
from oracle import gemm as ogemm
from oracle import glue as oglue
from oracle import quant as oquant
from tests import _parity as P

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def q():
    import paper_2404_00456_b200 as q
    q.lib()
    return q


def _codes8(rows, k, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return torch.randint(-127, 128, (rows, k), generator=g, device=DEV, dtype=torch.int32).to(torch.int8)


@pytest.mark.parametrize("K,rms", [(256, False), (4096, True), (8192, False), (8192, True), (1040, False)])
def test_quant8_parity(q, K, rms):
    x = synth.activations(67, K, "outlier", seed=K, device=DEV) * 0.1
    x[5] = 0
    xq, xs = q.hadamard_quant8(x, rmsnorm=rms)
    xh = x.float().cpu().numpy().astype(np.float64)
    y = oglue.rmsnorm(xh) if rms else xh
    rc, rs = oquant.quantize_sym_rows(y, 0.9, qmax=127)
    P.assert_codes(xq.cpu().numpy().astype(np.int64), rc, "int8 codes")
    P.assert_scales(xs.cpu().numpy(), rs, "int8 scales")


@pytest.mark.parametrize("mode,K", [("full", 28672), ("across_heads", 8192), ("across_heads", 4096)])
def test_quant8_transform_parity(q, mode, K):
    """8-bit FULL / ACROSS_HEADS quantizers (the tcgen05 transforms with qmax = 127) against the
    oracle's dense transform + RTN, including a zero row, a non-finite row and multi-row CTAs."""
    from oracle import layer as olayer
    M = 2 * 148 + 7
    x = synth.activations(M, K, "swiglu" if mode == "full" else "normal", seed=K + 3, device=DEV)
    x[5] = 0
    x[9, 3] = float("inf")
    xq, xs = q.hadamard_quant8(x, mode=mode)
    torch.cuda.synchronize()
    rows = [0, 1, 5, 147, 148, 149, 296, M - 1]
    xh = x[rows].float().cpu().numpy().astype(np.float64)
    rc, rs = oquant.quantize_sym_rows(olayer.online_transform(xh, mode, 128), 0.9, qmax=127)
    P.assert_codes(xq[rows].cpu().numpy().astype(np.int64), rc, f"int8 {mode} codes")
    P.assert_scales(xs[rows].cpu().numpy(), rs, f"int8 {mode} scales")
    s9 = xs[9].item()
    assert s9 != s9 and not xq[9].any()  # non-finite row: scale NaN, codes 0
    assert int(xq.abs().max()) <= 127


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (300, 776, 512), (129, 264, 4096), (600, 1024, 8192),
                                   (2085, 4120, 4096), (1100, 8200, 2176)])
def test_int8_gemm_s32_bit_exact(q, M, N, K):
    # includes > 1 tile per CTA pair (double-buffered accumulators), ragged M / N, K % 256 == 128
    xq, wq = _codes8(M, K, M), _codes8(N, K, N + 1)
    acc = q.int8_matmul_s32(xq, wq)
    torch.cuda.synchronize()
    ref = ogemm.int_matmul_exact_f64(xq.cpu().numpy().astype(np.int64), wq.cpu().numpy().astype(np.int64))
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), ref)


def test_int8_gemm_extreme_codes(q):
    M, N, K = 130, 264, 65536  # |acc| = 127 * 127 * K = 1.06e9 < 2^31
    xq = torch.full((M, K), 127, dtype=torch.int8, device=DEV)
    wq = torch.full((N, K), -127, dtype=torch.int8, device=DEV)
    wq[::2] = 127
    acc = q.int8_matmul_s32(xq, wq).cpu().numpy()
    assert np.all(acc[:, 0::2] == 127 * 127 * K) and np.all(acc[:, 1::2] == -127 * 127 * K)


@pytest.mark.parametrize("M,N,K", [(200, 264, 256), (1100, 8200, 4096)])
def test_int8_linear_epilogue(q, M, N, K):
    xq, wq = _codes8(M, K, 7), _codes8(N, K, 8)
    xs = torch.rand(M, device=DEV) * 1e-3 + 1e-4
    ws = synth.weight_scales(N, seed=9, device=DEV) * 0.01
    y = q.int8_linear(xq, xs, wq, ws)
    torch.cuda.synchronize()
    acc = ogemm.int_matmul_exact_f64(xq.cpu().numpy().astype(np.int64), wq.cpu().numpy().astype(np.int64))
    ref = ogemm.dequant_epilogue(acc, xs.cpu().numpy(), ws.cpu().numpy())
    assert P.max_fp16_ulp(y.cpu().numpy(), ref) <= 2


def test_a8w8_linear_end_to_end(q):
    # RMSNorm + int8 quant -> int8 GEMM with RTN-quantized int8 weights vs the oracle
    M, N, K = 96, 512, 1024
    x = synth.activations(M, K, "normal", seed=3, device=DEV)  # incoherent (rotated-like) activations
    w = synth.dense_weight(N, K, seed=4).double().numpy()
    cw, sw, _ = oquant.rtn_weight_quantize(w, qmax=127)
    xq, xs = q.hadamard_quant8(x, rmsnorm=True)
    y = q.int8_linear(xq, xs, torch.as_tensor(cw.astype(np.int8), device=DEV), torch.as_tensor(sw, device=DEV))
    rc, rs = oquant.quantize_sym_rows(oglue.rmsnorm(x.float().cpu().numpy().astype(np.float64)), 0.9, qmax=127)
    ref = ogemm.dequant_epilogue(ogemm.int_matmul_exact_f64(rc, cw), rs, sw)
    assert P.frob_rel(y.cpu().numpy(), ref) <= P.FROB_REL
    # and 8-bit is close to the full-precision linear on outlier-free (rotated) inputs — the
    # paper's "lossless" 8-bit RTN (P:6)
    fp = oglue.rmsnorm(x.float().cpu().numpy().astype(np.float64)) @ w.T
    assert P.frob_rel(y.cpu().numpy(), fp) <= 2e-2
