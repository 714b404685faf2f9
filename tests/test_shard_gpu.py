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
