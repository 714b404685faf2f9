"""GPU parity of the 8-bit transform quantizers at every width (A8W8 QuaRot, P:6,
tab:rtn_results) and of the group-wise quantizers after the FULL / ACROSS_HEADS transforms
(tab:group_wise_ablation 256G / 128G / 64G), against the oracle's dense
fp64 transform (oracle.layer.online_transform) followed by its RTN (oracle.quant)."""
import numpy as np
import pytest
import torch

import synth
from oracle import layer as olayer
from oracle import quant as oquant
from tests import _parity as P

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def q():
    import paper_2404_00456_b200 as q
    q.lib()
    return q


def _rows(M):
    return sorted({0, 1, 5, 9, 147, 148, 149, 296, M - 1} & set(range(M)))


def _inputs(M, K, kind, seed):
    x = synth.activations(M, K, kind, seed=seed, device=DEV)
    x[5] = 0
    x[9, 3] = float("inf")
    return x


# the tcgen05 kernels (11008 = 64 x 172, 13824 = 128 x 108, 5120 = 256 x 20, 28672 = 1024 x 28) and the
# shared-memory kernel (every other 2^n m, including m = 1)
@pytest.mark.parametrize("K", [11008, 13824, 5120, 28672, 4096, 1792, 688, 640, 256])
def test_quant8_full_every_width(q, K):
    M = 2 * 148 + 7
    x = _inputs(M, K, "swiglu", K + 1)
    xq, xs = q.hadamard_quant8(x, mode="full")
    torch.cuda.synchronize()
    rows = [r for r in _rows(M) if r != 9]
    xh = x[rows].float().cpu().numpy().astype(np.float64)
    rc, rs = oquant.quantize_sym_rows(olayer.online_transform(xh, "full"), 0.9, qmax=127)
    P.assert_codes(xq[rows].cpu().numpy().astype(np.int64), rc, f"int8 FULL K={K}")
    P.assert_scales(xs[rows].cpu().numpy(), rs, f"int8 FULL K={K}")
    s9 = xs[9].item()
    assert s9 != s9 and not xq[9].any()  # non-finite row: scale NaN, codes 0
    assert xs[5].item() == 1.0 and not xq[5].any()  # zero row: scale 1, codes 0
    assert int(xq.abs().max()) <= 127


@pytest.mark.parametrize("K,hd", [(512, 128), (1024, 64), (8192, 256), (2048, 128)])
def test_quant8_across_heads_smem_shapes(q, K, hd):
    M = 41
    x = _inputs(M, K, "normal", K + hd)
    xq, xs = q.hadamard_quant8(x, mode="across_heads", head_dim=hd)
    torch.cuda.synchronize()
    rows = [r for r in _rows(M) if r != 9]
    xh = x[rows].float().cpu().numpy().astype(np.float64)
    rc, rs = oquant.quantize_sym_rows(olayer.online_transform(xh, "across_heads", hd), 0.9, qmax=127)
    P.assert_codes(xq[rows].cpu().numpy().astype(np.int64), rc, f"int8 HEADS K={K} hd={hd}")
    P.assert_scales(xs[rows].cpu().numpy(), rs, f"int8 HEADS K={K} hd={hd}")
    assert xs[9].item() != xs[9].item() and not xq[9].any()


@pytest.mark.parametrize("mode,K,group,hd", [("full", 11008, 128, 128), ("full", 28672, 128, 128),
                                             ("full", 4096, 64, 128), ("full", 13824, 256, 128),
                                             ("full", 5120, 64, 128), ("across_heads", 8192, 128, 128),
                                             ("across_heads", 4096, 64, 128), ("across_heads", 2048, 256, 64)])
def test_group_quant_after_transform(q, mode, K, group, hd):
    """Group-wise INT4 of the transformed row: codes / scales per run of `group` consecutive
    elements of y; the packed and the one-code-per-byte outputs agree exactly."""
    M = 37
    x = _inputs(M, K, "swiglu" if mode == "full" else "outlier", K + group)
    xq, xs = q.hadamard_quant_group(x, group, mode=mode, head_dim=hd)
    xq8, xs8 = q.hadamard_quant_group8(x, group, mode=mode, head_dim=hd)
    torch.cuda.synchronize()
    got = P.unpack_signed(xq.cpu().numpy())
    assert np.array_equal(got, xq8.cpu().numpy().astype(np.int64))
    assert torch.equal(torch.nan_to_num(xs, 7.0), torch.nan_to_num(xs8, 7.0))
    rows = [r for r in _rows(M) if r != 9]
    xh = x[rows].float().cpu().numpy().astype(np.float64)
    rc, rs = oquant.quantize_sym_groups(olayer.online_transform(xh, mode, hd), group)
    P.assert_codes(got[rows], rc, f"group {group} {mode} K={K}")
    P.assert_scales(xs[rows].cpu().numpy(), rs, f"group {group} {mode} K={K}")
    # the Inf element (index 3) spreads through H: FULL to every output, ACROSS_HEADS to index 3
    # of every head; exactly the groups holding such an element get scale NaN and codes 0
    idx = np.arange(K)
    hit = np.ones(K, bool) if mode == "full" else (idx % hd) == 3
    bad = hit.reshape(-1, group).any(1)
    s9 = xs[9].cpu().numpy()
    assert np.array_equal(np.isnan(s9), bad)
    assert not got[9].reshape(-1, group)[bad].any()
    assert torch.all(xs[5] == 1.0) and not xq[5].any()
    assert int(np.abs(got).max()) <= 7
