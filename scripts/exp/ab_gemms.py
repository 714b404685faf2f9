"""Time the four 70B chain GEMMs (131072 tokens) of the library QUAROT_LIB points at (median of ROUNDS x 5 calls each)."""
import os, statistics, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2404_00456_b200 as q
M = 131072
out = []
for name, N, K, kind in (("qkv", 10240, 8192, "plain"), ("o", 8192, 8192, "res"), ("gateup", 57344, 8192, "swiglu"),
                         ("down", 8192, 28672, "res")):
    xq = synth.packed_weight_codes(M, K, 1, "cuda"); wq = synth.packed_weight_codes(N, K, 2, "cuda")
    xs = torch.rand(M, device="cuda") + 0.5; ws = synth.weight_scales(N, 3, "cuda")
    y = torch.empty(M, N // 2 if kind == "swiglu" else N, dtype=torch.float16, device="cuda")
    r = torch.randn(M, N, device="cuda").half() if kind == "res" else None
    fn = (lambda: q.int4_linear_swiglu(xq, xs, wq, ws, act=y)) if kind == "swiglu" else (lambda: q.int4_linear(xq, xs, wq, ws, y=y, residual=r))
    ts = []
    for _ in range(int(os.environ.get("ROUNDS", 3))):
        for _ in range(2): fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5): fn()
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 5)
    ms = statistics.median(ts)
    out.append(f"{name} {ms:.3f} ms {2 * M * N * K / ms / 1e9:.0f} TOPS")
    del xq, wq, y, r; torch.cuda.empty_cache()
print(" | ".join(out), flush=True)
