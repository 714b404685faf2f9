"""One small invocation of every hot-path kernel family (for compute-sanitizer memcheck /
racecheck / synccheck runs): reduced-M versions of BASELINE configs 1-2 plus the
70B-width tcgen05 kernels at a few hundred rows.  python scripts/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_00456_b200 as q  # noqa: E402

dev = "cuda"
M = int(os.environ.get("SAN_M", "300"))
for K in (4096, 8192):
    q.hadamard_quant(synth.activations(M, K, "outlier", seed=1, device=dev), "none", rmsnorm=True)
    q.hadamard_quant(synth.activations(M, K, "normal", seed=2, device=dev), "across_heads", head_dim=128)
for K in (11008, 28672, 13824, 5120, 1792):
    q.hadamard_quant(synth.activations(M, K, "swiglu", seed=3, device=dev), "full")
    q.hadamard_quant8(synth.activations(M, K, "swiglu", seed=3, device=dev), mode="full")
q.hadamard_quant(synth.activations(M, 28672, "swiglu", seed=3, device=dev), "full", kperm=True)  # the chain's form
q.hadamard_quant(synth.activations(M, 28672, "swiglu", seed=3, device=dev), "full", clip_ratio=0.5, kperm=True)
for mode in ("none", "full", "across_heads"):
    q.hadamard_quant_group(synth.activations(M, 4096, "normal", seed=4, device=dev), 128, mode=mode)
for (N, K) in ((10240, 8192), (8192, 28672), (4096, 11008 + 256 - 11008 % 256)):
    xq = synth.packed_weight_codes(M, K, 5, dev)
    wq = synth.packed_weight_codes(N, K, 6, dev)
    xs = torch.rand(M, device=dev) + 0.5
    ws = synth.weight_scales(N, 7, dev)
    q.int4_linear(xq, xs, wq, ws)
    q.int4_matmul_s32(xq, wq)
    q.int4_linear(xq, xs, wq, ws, residual=torch.zeros(M, N, dtype=torch.float16, device=dev))
    wil, wsil = q.interleave_gate_up(wq, ws)
    q.int4_linear_swiglu(xq, xs, wil, wsil)
    for G in (64, 128, 256):
        q.int4_linear_group(xq, torch.rand(M, K // G, device=dev), wq, torch.rand(K // G, N, device=dev), group=G)
T, n_q, n_kv, d = M, 64, 8, 128
fused = synth.activations(T, (n_q + 2 * n_kv) * d, "normal", seed=8, device=dev)
qv = fused[:, : n_q * d].view(T, n_q, d)
kv_ = fused[:, n_q * d:(n_q + n_kv) * d].view(T, n_kv, d)
vv = fused[:, (n_q + n_kv) * d:].view(T, n_kv, d)
q.kv_quant(kv_, vv, qv)
q.kv_quant(kv_, vv, qv, rope=(0, 2048, 10000.0))
f7 = synth.activations(T, 96 * d, "normal", seed=12, device=dev)  # Llama-2-7B: 32 / 32 heads
q.kv_quant(f7[:, 32 * d:64 * d].view(T, 32, d), f7[:, 64 * d:].view(T, 32, d), f7[:, :32 * d].view(T, 32, d),
           rope=(0, 2048, 10000.0))
B, s_max = 4, 512
cache = q.kv_cache_empty(B, s_max, n_kv, d, device=dev)
pos = torch.tensor([5, 100, 511, 0], dtype=torch.int32, device=dev)
kq = synth.activations(B, n_kv * d, "normal", seed=9, device=dev).view(B, n_kv, d)
vq = synth.activations(B, n_kv * d, "normal", seed=10, device=dev).view(B, n_kv, d)
qq = synth.activations(B, n_q * d, "normal", seed=11, device=dev).view(B, n_q, d)
q.kv_append(kq, vq, qq, pos, cache)
q.kv_decode(qq, cache, pos + 1, n_kv=n_kv)
torch.cuda.synchronize()
print("sanitize_run OK")
