"""Token sharding on one GPU (BASELINE configs 3/5): the decoder-layer step run on
G contiguous row shards one after another — exactly what each rank of `bench.py --gpus G` runs
on its slice — reproduces the unsharded step bit for bit (layer output and KV cache), because
every kernel is row-independent and the GEMM accumulates exactly."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,T", [(8, 8 * 2048), (3, 3000)])
def test_sequential_shards_equal_unsharded_bitwise(G, T):
    from paper_2404_00456_b200 import dist as qd
    from paper_2404_00456_b200.runtime import DecoderLayerStep, QuaRotLayer
    dev = "cuda"
    S = synth.inputs.LLAMA2_70B
    dims = {"qkv": (S.qkv_out, S.hidden), "o": (S.hidden, S.hidden), "gate_up": (2 * S.ffn, S.hidden),
            "down": (S.hidden, S.ffn)}
    w = {n: (synth.packed_weight_codes(a, b, 300 + i, dev), synth.weight_scales(a, 310 + i, dev))
         for i, (n, (a, b)) in enumerate(dims.items())}
    layer = QuaRotLayer(S.hidden, S.ffn, S.n_heads, S.n_kv_heads, S.head_dim, w)
    x = synth.activations(T, S.hidden, "outlier", 320, dev) * 0.05
    z = synth.activations(T, S.hidden, "normal", 321, dev)
    full = DecoderLayerStep(layer, T, dev)
    full.run_device({"x": x, "attn_out": z})
    torch.cuda.synchronize()
    ref = {k: t.clone() for k, t in full.result_tensors().items()}
    del full
    for r0, r1 in qd.shard_plan(T, G):
        st = DecoderLayerStep(layer, r1 - r0, dev, row_offset=r0)
        st.run_device({"x": x[r0:r1].contiguous(), "attn_out": z[r0:r1].contiguous()})
        torch.cuda.synchronize()
        for k, t in st.result_tensors().items():
            assert torch.equal(t.view(torch.uint8), ref[k][r0:r1].contiguous().view(torch.uint8)), (k, r0, r1)
        del st


def test_chain_kperm_equals_natural_order_bitwise():
    """QUAROT_HAD_KPERM on the down_proj input (with the offline column permutation of W_down)
    gives the same layer output and KV cache bit for bit as the natural element order."""
    from paper_2404_00456_b200.runtime import DecoderLayerStep, QuaRotLayer
    dev = "cuda"
    S = synth.inputs.LLAMA2_70B
    T = 3000
    dims = {"qkv": (S.qkv_out, S.hidden), "o": (S.hidden, S.hidden), "gate_up": (2 * S.ffn, S.hidden),
            "down": (S.hidden, S.ffn)}
    w = {n: (synth.packed_weight_codes(a, b, 400 + i, dev), synth.weight_scales(a, 410 + i, dev))
         for i, (n, (a, b)) in enumerate(dims.items())}
    layer = QuaRotLayer(S.hidden, S.ffn, S.n_heads, S.n_kv_heads, S.head_dim, w)
    inp = {"x": synth.activations(T, S.hidden, "outlier", 420, dev) * 0.05,
           "attn_out": synth.activations(T, S.hidden, "normal", 421, dev)}
    outs = []
    for kp in (False, True):
        st = DecoderLayerStep(layer, T, dev, kperm=kp)
        st.run_device(inp)
        torch.cuda.synchronize()
        outs.append({k: t.clone() for k, t in st.result_tensors().items()})
    for k in outs[0]:
        assert torch.equal(outs[0][k].view(torch.uint8), outs[1][k].view(torch.uint8)), k


@pytest.mark.parametrize("M", [1, 37, 300])
def test_kperm_codes_are_the_natural_codes_permuted(M):
    import paper_2404_00456_b200 as q
    K = 28672
    x = synth.activations(M, K, "swiglu", M, "cuda")
    xq_n, xs_n = q.hadamard_quant(x, "full")
    xq_p, xs_p = q.hadamard_quant(x, "full", kperm=True)
    perm = q.full_kperm(K)
    assert torch.equal(xq_p, q.permute_k_packed(xq_n, perm))
    assert torch.equal(xs_p, xs_n)
