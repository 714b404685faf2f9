"""A/B timing of group-wise GEMM variants (int4_group_gemm_kernel) in one process, interleaved.
Usage: abbench_group.py LIB [LIB ...]   ('base' = the in-tree libquarot.so); env AB_G (128)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2404_00456_b200 import quarot  # noqa: E402

libs = {}
for name in sys.argv[1:]:
    path = quarot.LIB_PATH if name == "base" else os.path.join(os.path.dirname(quarot.LIB_PATH), "..", "_variants",
                                                                  f"libquarot_{name}.so")
    f = ctypes.CDLL(os.path.abspath(path)).quarot_int4_linear_group
    f.argtypes = quarot._SIGS["quarot_int4_linear_group"]
    f.restype = ctypes.c_int
    libs[name] = f
M = int(os.environ.get("AB_M", 131072))
stream = torch.cuda.current_stream().cuda_stream
xq_big = torch.randint(0, 256, (M, 28672 // 2), dtype=torch.uint8, device="cuda")
for G in [int(g) for g in os.environ.get("AB_G", "128").split(",")]:
    for sname, N, K in (("o", 8192, 8192), ("gate_up", 57344, 8192)):
        xq = xq_big[:, : K // 2]
        wq = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda")
        xs = torch.rand(M, K // G, device="cuda") * 0.01 + 0.001
        ws = torch.rand(K // G, N, device="cuda") * 0.01 + 0.001
        y = torch.empty(M, N, dtype=torch.float16, device="cuda")

        def call(f):
            st = f(xq.data_ptr(), xs.data_ptr(), xs.stride(0), M, K, xq.stride(0), wq.data_ptr(), ws.data_ptr(),
                   ws.stride(0), N, wq.stride(0), G, y.data_ptr(), y.stride(0), stream)
            assert st == 0, st

        times = {n: [] for n in libs}
        for f in libs.values():
            call(f)
        for _ in range(int(os.environ.get("AB_ROUNDS", 5))):
            for n, f in libs.items():
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(2):
                    call(f)
                b.record()
                torch.cuda.synchronize()
                times[n].append(a.elapsed_time(b) / 2)
        print(f"G{G}", sname, {n: round(2 * M * N * K / statistics.median(t) / 1e9, 1) for n, t in times.items()},
              flush=True)
        del wq, y
