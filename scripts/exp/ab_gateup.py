"""Time the gate/up SwiGLU GEMM (70B, 131072 tokens) of the library QUAROT_LIB points at: median of ROUNDS x 5 calls."""
import os, statistics, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2404_00456_b200 as q
M, N, K = 131072, 57344, 8192
xq = synth.packed_weight_codes(M, K, 1, "cuda"); wq = synth.packed_weight_codes(N, K, 2, "cuda")
xs = torch.rand(M, device="cuda") + 0.5; ws = synth.weight_scales(N, 3, "cuda")
y = torch.empty(M, N // 2, dtype=torch.float16, device="cuda")
ts = []
for _ in range(int(os.environ.get("ROUNDS", 3))):
    for _ in range(2): q.int4_linear_swiglu(xq, xs, wq, ws, act=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): q.int4_linear_swiglu(xq, xs, wq, ws, act=y)
    b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 5)
ms = statistics.median(ts)
print("gateup", round(ms, 3), "ms", round(2 * M * N * K / ms / 1e9), "TOPS", [round(t, 3) for t in ts], flush=True)
