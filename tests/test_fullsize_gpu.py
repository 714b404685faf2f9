"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

One prefill step of `runtime.PrefillStep` (the 9 launches bench.py times) runs over the whole
batch — Llama-2-7B 8 x 2048 and Llama-2-70B 64 x 2048 tokens — and sampled outputs are
checked one by one against the CPU oracle:
  * quantized activations of every linear (sampled token rows, all K);
  * int32 accumulators (bit-exact) and fp16 outputs on sampled (row, column) blocks;
  * the KV cache and rotated Q of sampled tokens;
plus properties that hold at any size on the full tensors (finite positive scales, codes in
[-7, 7], the packed nibble 0x8 never appears)."""
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

DEV = "cuda"


def _layer(shapes, device):
    from paper_2404_00456_b200.runtime import QuaRotLayer
    S = shapes
    dims = {"qkv": (S.qkv_out, S.hidden), "o": (S.hidden, S.hidden), "gate_up": (2 * S.ffn, S.hidden),
            "down": (S.hidden, S.ffn)}
    w = {name: (synth.packed_weight_codes(n, k, 1000 + i, device), synth.weight_scales(n, 1010 + i, device))
         for i, (name, (n, k)) in enumerate(dims.items())}
    return QuaRotLayer(S.hidden, S.ffn, S.n_heads, S.n_kv_heads, S.head_dim, w)


def _inputs(shapes, tokens, device):
    return {"attn_in": synth.activations(tokens, shapes.hidden, "outlier", 100, device),
            "attn_out": synth.activations(tokens, shapes.hidden, "normal", 101, device),
            "ffn_in": synth.activations(tokens, shapes.hidden, "outlier", 102, device),
            "ffn_act": synth.activations(tokens, shapes.ffn, "swiglu", 103, device)}


def _no_nibble8(packed: torch.Tensor) -> bool:
    lo = packed & 0xF
    hi = packed >> 4
    return not bool(((lo == 8) | (hi == 8)).any().item())


def test_full_m_down_gemm_blocks_bit_exact():
    """The bench's down_proj launch shape (M = 131072, N = 8192, K = 28672: 512 x 32 tiles over
    74 CTA pairs, 112 k-blocks each): whole 256-row x 256-column tile blocks at the first, a
    middle and the last M / N tiles compared element-exactly with the oracle's int64 GEMM."""
    import paper_2404_00456_b200 as q
    M, N, K = 131072, 8192, 28672

    def codes(rows, seed):  # uniform packed codes in [-7, 7] (nibble 0x8 = -8 mapped to 0x9 = -7)
        g = torch.Generator(device=DEV).manual_seed(seed)
        b = torch.randint(0, 256, (rows, K // 2), dtype=torch.uint8, device=DEV, generator=g)
        b = torch.where((b & 0xF) == 8, b + 1, b)
        return torch.where((b >> 4) == 8, b + 16, b)
    xq, wq = codes(M, 501), codes(N, 502)
    acc = q.int4_matmul_s32(xq, wq)
    torch.cuda.synchronize()
    for (m0, n0) in ((0, 0), (M // 2 + 256 * 37, N // 2 + 256 * 5), (M - 256, N - 256), (256 * 300, 0)):
        r = torch.arange(m0, m0 + 256, device=DEV)
        c = torch.arange(n0, n0 + 256, device=DEV)
        ref = ogemm.int_matmul_exact_f64(P.unpack_signed(xq[r].cpu().numpy()), P.unpack_signed(wq[c].cpu().numpy()))
        assert np.array_equal(acc[r][:, c].cpu().numpy().astype(np.int64), ref), (m0, n0)


@pytest.mark.parametrize("cfg", [1, 2])
def test_full_size_step_sampled_parity(cfg):
    import paper_2404_00456_b200 as q
    from paper_2404_00456_b200.runtime import PrefillStep
    spec = synth.CONFIGS[cfg]
    S, T = spec["shapes"], spec["tokens"]
    layer = _layer(S, DEV)
    inputs = _inputs(S, T, DEV)
    x_attn_ref = inputs["attn_in"].clone()
    step = PrefillStep(layer, T, DEV)
    rows = olayer.token_sample(T, 12)
    rows_t = torch.as_tensor(rows, device=DEV)
    rng = np.random.default_rng(cfg)
    for spec_lin, key in zip(layer.specs, ("attn_in", "attn_out", "ffn_in", "ffn_act")):
        # the step runs the four linears; re-run each quantizer + GEMM as the step does and keep
        # its quantized activations for the checks
        x = inputs[key]
        xq, xs = q.hadamard_quant(x, spec_lin.mode, layer.head_dim, layer.clip_act)
        wq, ws = layer.weights[spec_lin.name]
        y = q.int4_linear(xq, xs, wq, ws)
        cols = np.sort(rng.choice(spec_lin.n, size=min(256, spec_lin.n), replace=False))
        cols[-1] = spec_lin.n - 1  # the last N tile
        cols_t = torch.as_tensor(cols, device=DEV)
        # accumulators of the FULL-M launch (the bench's M, every tile of the grid), sampled blocks
        acc_full = q.int4_matmul_s32(xq, wq)
        acc = acc_full[rows_t][:, cols_t].contiguous()
        del acc_full
        torch.cuda.synchronize()
        # full-tensor properties
        assert torch.isfinite(xs).all() and (xs > 0).all()
        assert _no_nibble8(xq)
        # sampled rows: codes and scales vs the oracle's quantizer
        xh = x[rows_t].float().cpu().numpy().astype(np.float64)
        rc, _, rs = olayer.hadamard_quant(xh, spec_lin.mode, layer.head_dim, layer.clip_act)
        gc = P.unpack_signed(xq[rows_t].cpu().numpy())
        P.assert_codes(gc, rc, f"{S.name} {spec_lin.name} codes")
        P.assert_scales(xs[rows_t].cpu().numpy(), rs, f"{S.name} {spec_lin.name} scales")
        # sampled (row, column) block of the full launch: accumulators bit-exact, and the bench
        # launch's fp16 outputs within 2 ulp of the oracle epilogue on the same codes / scales
        cw = oquant.unpack_int4_signed(wq[cols_t].cpu().numpy())
        ref_acc = ogemm.int_matmul_exact_f64(gc, cw)
        got_acc = acc.cpu().numpy().astype(np.int64)
        assert np.array_equal(got_acc, ref_acc), f"{S.name} {spec_lin.name}: accumulators differ"
        ref_y = ogemm.dequant_epilogue(ref_acc, xs[rows_t].cpu().numpy(), ws.cpu().numpy()[cols])
        got_y = y[rows_t][:, cols_t].cpu().numpy()
        assert P.frob_rel(got_y, ref_y) <= P.FROB_REL
        assert P.max_fp16_ulp(got_y, ref_y) <= 2, f"{S.name} {spec_lin.name}: fp16 outputs"
        del xq, xs, y, acc
    # the timed step itself (same launches as bench.py) reproduces the per-call results
    step.run_device(inputs)
    torch.cuda.synchronize()
    xq, xs = q.hadamard_quant(x_attn_ref, "none", layer.head_dim, layer.clip_act)
    wq, ws = layer.weights["qkv"]
    y = q.int4_linear(xq, xs, wq, ws)
    # KV cache of the step vs the oracle on sampled tokens (the step rotated Q in place)
    d = layer.head_dim
    nq, nkv = layer.n_heads * d, layer.n_kv * d
    yh = y[rows_t].float().cpu().numpy().astype(np.float64)
    ref = okv.kv_init(yh[:, nq:nq + nkv].reshape(len(rows), -1, d), yh[:, nq + nkv:].reshape(len(rows), -1, d),
                      yh[:, :nq].reshape(len(rows), -1, d))
    for t in ("k", "v"):
        P.assert_codes(P.unpack_unsigned(step.kv[f"{t}_codes"][rows_t].cpu().numpy()),
                       P.unpack_unsigned(ref[f"{t}_codes"]), f"{t} codes")
        P.assert_scales(step.kv[f"{t}_scale"][rows_t].cpu().numpy(), ref[f"{t}_scale"], f"{t} scale")
        P.assert_codes(step.kv[f"{t}_zero"][rows_t].cpu().numpy(), ref[f"{t}_zero"], f"{t} zero")
    q_rot = step.out["qkv"][rows_t][:, :nq].cpu().numpy().reshape(len(rows), -1, d)
    assert P.max_fp16_ulp(q_rot, ref["q_rot"]) <= 1
    assert torch.equal(step.out["qkv"][:, nq:], y[:, nq:])  # K/V part of the step's QKV output
