"""Sweep the GEMM raster group (pair-rows sharing A in L2) on the chain's four GEMMs, interleaved."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_00456_b200 as q  # noqa: E402

L = q.lib()
L.quarot_debug_gemm_group_m.argtypes = [ctypes.c_int]
M = 131072
groups = [int(g) for g in os.environ.get("GROUPS", "8,16,32,64,0").split(",")]
xq_big = synth.packed_weight_codes(M, 14336 * 2, 1, "cuda")
xs = torch.rand(M, device="cuda") * 0.01
for name, N, K in (("qkv", 10240, 8192), ("o+res", 8192, 8192), ("gate_up+swiglu", 57344, 8192),
                   ("down+res", 8192, 28672)):
    xq = xq_big[:, : K // 2]
    wq = synth.packed_weight_codes(N, K, 2, "cuda")
    ws = synth.weight_scales(N, 3, "cuda")
    if name.startswith("gate_up"):
        wqi, wsi = q.interleave_gate_up(wq, ws)
        y = torch.empty(M, N // 2, dtype=torch.float16, device="cuda")
        fn = lambda: q.int4_linear_swiglu(xq, xs, wqi, wsi, act=y)
    elif "res" in name:
        r = synth.activations(M, N, "normal", 4, "cuda")
        y = torch.empty(M, N, dtype=torch.float16, device="cuda")
        fn = lambda: q.int4_linear(xq, xs, wq, ws, y=y, residual=r)
    else:
        y = torch.empty(M, N, dtype=torch.float16, device="cuda")
        fn = lambda: q.int4_linear(xq, xs, wq, ws, y=y)
    times = {g: [] for g in groups}
    for g in groups:
        L.quarot_debug_gemm_group_m(g)
        fn()
    for _ in range(5):
        for g in groups:
            L.quarot_debug_gemm_group_m(g)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            fn()
            b.record()
            torch.cuda.synchronize()
            times[g].append(a.elapsed_time(b) / 2)
    print(name, {g: round(2 * M * N * K / statistics.median(t) / 1e9) for g, t in times.items()}, flush=True)
    del wq, y
L.quarot_debug_gemm_group_m(0)
