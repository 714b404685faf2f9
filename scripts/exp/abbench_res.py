"""A/B of the fused-epilogue GEMM variants (residual, SwiGLU) across library builds, interleaved."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_00456_b200 import quarot  # noqa: E402

libs = {}
for name in sys.argv[1:]:
    path = quarot.LIB_PATH if name == "base" else os.path.join(os.path.dirname(quarot.LIB_PATH), "..", "_variants",
                                                                  f"libquarot_{name}.so")
    h = ctypes.CDLL(os.path.abspath(path))
    for fn in ("quarot_int4_linear_residual", "quarot_int4_linear_swiglu"):
        getattr(h, fn).argtypes = quarot._SIGS[fn]
        getattr(h, fn).restype = ctypes.c_int
    libs[name] = h
M = 131072
xq_big = synth.packed_weight_codes(M, 8192, 1, "cuda")
xs = torch.rand(M, device="cuda") * 0.01
stream = torch.cuda.current_stream().cuda_stream
for sname, N, K in (("o+res", 8192, 8192), ("gate_up+swiglu", 57344, 8192)):
    wq = synth.packed_weight_codes(N, K, 2, "cuda")
    ws = synth.weight_scales(N, 3, "cuda")
    if "res" in sname:
        y = torch.empty(M, N, dtype=torch.float16, device="cuda")
        r = synth.activations(M, N, "normal", 4, "cuda")
        call = lambda h: h.quarot_int4_linear_residual(xq_big.data_ptr(), xs.data_ptr(), M, K, xq_big.stride(0),
                                                       wq.data_ptr(), ws.data_ptr(), N, wq.stride(0), r.data_ptr(),
                                                       r.stride(0), y.data_ptr(), y.stride(0), stream)
    else:
        y = torch.empty(M, N // 2, dtype=torch.float16, device="cuda")
        call = lambda h: h.quarot_int4_linear_swiglu(xq_big.data_ptr(), xs.data_ptr(), M, K, xq_big.stride(0),
                                                     wq.data_ptr(), ws.data_ptr(), N, wq.stride(0), y.data_ptr(),
                                                     y.stride(0), stream)
    outs = {}
    for n, h in libs.items():
        assert call(h) == 0
        torch.cuda.synchronize()
        outs[n] = y.clone()
    ref = next(iter(outs.values()))
    same = {n: bool(torch.equal(o, ref)) for n, o in outs.items()}
    times = {n: [] for n in libs}
    for _ in range(6):
        for n, h in libs.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                call(h)
            b.record()
            torch.cuda.synchronize()
            times[n].append(a.elapsed_time(b) / 3)
    print(sname, "identical:", same, {n: round(2 * M * N * K / statistics.median(t) / 1e9, 1) for n, t in times.items()},
          flush=True)
    del wq, y
