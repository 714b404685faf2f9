"""A/B timing of GEMM variants in ONE process, interleaved, so clock/power drift hits every
variant alike.  Usage: abbench.py LIB [LIB ...]   ('base' = the in-tree libquarot.so)."""
import ctypes
import json
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
    f = h.quarot_int4_linear
    f.argtypes = quarot._SIGS["quarot_int4_linear"]
    f.restype = ctypes.c_int
    libs[name] = f

M = int(os.environ.get("AB_M", 131072))
shapes = [("qkv", 10240, 8192), ("gate_up", 57344, 8192), ("down", 8192, 28672)]
xq_big = synth.packed_weight_codes(M, 28672, 1, "cuda")
xs = torch.rand(M, device="cuda") + 0.5
stream = torch.cuda.current_stream().cuda_stream
res = {}
for sname, N, K in shapes:
    xq = xq_big[:, : K // 2]
    wq = synth.packed_weight_codes(N, K, 2, "cuda")
    ws = synth.weight_scales(N, 3, "cuda")
    y = torch.empty(M, N, dtype=torch.float16, device="cuda")
    times = {n: [] for n in libs}

    def call(f):
        st = f(xq.data_ptr(), xs.data_ptr(), M, K, xq.stride(0), wq.data_ptr(), ws.data_ptr(), N, wq.stride(0),
               y.data_ptr(), y.stride(0), stream)
        assert st == 0, st

    for n, f in libs.items():
        for _ in range(2):
            call(f)
    for rnd in range(int(os.environ.get("AB_ROUNDS", 6))):
        for n, f in libs.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                call(f)
            b.record()
            torch.cuda.synchronize()
            times[n].append(a.elapsed_time(b) / 3)
    for n in libs:
        ms = statistics.median(times[n])
        res[f"{sname}/{n}"] = round(2 * M * N * K / ms / 1e9, 1)
    print(sname, {n: res[f"{sname}/{n}"] for n in libs}, flush=True)
    del wq, y
print(json.dumps(res))
