"""INT4 GEMM roofline probes at the four Llama-2-70B chain shapes (131072 tokens): mode 0 product,
1 MMA issue only, 2 no widening stores, 3 no TMA, 4 no fp16 stores, 5 no B widening stores,
6 no A TMEM stores, 7 no epilogue work.  Prints ms and TOPS per (shape, mode)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2404_00456_b200 as q
lib = q.lib()
lib.quarot_debug_gemm_mode.argtypes = [ctypes.c_int]
M = int(os.environ.get("TOKENS", 131072))
modes = [int(v) for v in os.environ.get("MODES", "0,1,2,5,6,7,4,0").split(",")]
def timeit(fn, iters=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters
for name, N, K, kind in (("qkv", 10240, 8192, "plain"), ("o", 8192, 8192, "res"), ("gateup", 57344, 8192, "swiglu"),
                         ("down", 8192, 28672, "res")):
    xq = synth.packed_weight_codes(M, K, 1, "cuda")
    wq = synth.packed_weight_codes(N, K, 2, "cuda")
    xs = torch.rand(M, device="cuda") + 0.5
    ws = synth.weight_scales(N, 3, "cuda")
    y = torch.empty(M, N // 2 if kind == "swiglu" else N, dtype=torch.float16, device="cuda")
    r = torch.randn(M, N, device="cuda").half() if kind == "res" else None
    for mode in modes:
        lib.quarot_debug_gemm_mode(mode)
        if kind == "swiglu":
            fn = lambda: q.int4_linear_swiglu(xq, xs, wq, ws, act=y)
        else:
            fn = lambda: q.int4_linear(xq, xs, wq, ws, y=y, residual=r)
        ms = timeit(fn)
        print(name, "mode", mode, round(ms, 3), "ms", round(2 * M * N * K / ms / 1e9), "TOPS", flush=True)
    lib.quarot_debug_gemm_mode(0)
    del xq, wq, y, r
    torch.cuda.empty_cache()
