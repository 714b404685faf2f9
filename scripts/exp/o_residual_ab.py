import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2404_00456_b200 as q
M = 131072
def timeit(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters
xq = synth.packed_weight_codes(M, 8192, 1, "cuda")
for name, N in (("qkv", 10240), ("o", 8192)):
    wq = synth.packed_weight_codes(N, 8192, 2, "cuda")
    xs = torch.rand(M, device="cuda") + 0.5
    ws = synth.weight_scales(N, 3, "cuda")
    y = torch.empty(M, N, dtype=torch.float16, device="cuda")
    r = torch.randn(M, N, device="cuda").half()
    for kind in ("plain", "resid", "inplace"):
        if kind == "plain": fn = lambda: q.int4_linear(xq, xs, wq, ws, y=y)
        elif kind == "resid": fn = lambda: q.int4_linear(xq, xs, wq, ws, y=y, residual=r)
        else: fn = lambda: q.int4_linear(xq, xs, wq, ws, y=r, residual=r)
        ms = timeit(fn)
        print(name, kind, round(ms, 3), "ms", round(2 * M * N * 8192 / ms / 1e9), "TOPS", flush=True)
