"""A/B of the FULL K = 28672 quantizers, interleaved over rounds (median): variant 0 =
warpgroup-per-row (natural order), 'kperm' = the same kernel writing the transform-native order,
3 = the 16-warps-per-row kernel.  Time at 131072 tokens (CUDA events, inputs > L2), algorithmic
GB/s; code agreement of kperm (un-permuted) with natural, and of variant 3 with variant 0."""
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_00456_b200 as q  # noqa: E402

M, K = int(os.environ.get("TOKENS", 131072)), 28672
lib = q.lib()
lib.quarot_debug_hq_full_variant.argtypes = [ctypes.c_int]
x = synth.activations(M, K, "swiglu", 7, "cuda")
pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
hbm = json.load(open(pk))["hbm_gbs"] if os.path.exists(pk) else 6553.6
xq = torch.empty(M, K // 2, dtype=torch.uint8, device="cuda")
xs = torch.empty(M, dtype=torch.float32, device="cuda")


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def run(name):
    if name.startswith("kperm"):  # kperm[N]: variant N writing the transform-native order
        lib.quarot_debug_hq_full_variant(int(name[5:] or 0))
        return lambda: q.hadamard_quant(x, "full", q=xq, scale=xs, kperm=True)
    lib.quarot_debug_hq_full_variant(int(name))
    return lambda: q.hadamard_quant(x, "full", q=xq, scale=xs)


names = os.environ.get("VARIANTS", "3,0,kperm").split(",")
times = {n: [] for n in names}
for _ in range(int(os.environ.get("ROUNDS", 3))):
    for n in names:
        times[n].append(timeit(run(n)))
for n in names:
    ms = statistics.median(times[n])
    gbs = M * (2.5 * K + 4) / (ms * 1e-3) / 1e9
    print(n, json.dumps({"ms": ms, "all": [round(t, 4) for t in times[n]], "gbs": gbs, "frac_hbm": gbs / hbm}),
          flush=True)
lib.quarot_debug_hq_full_variant(0)
R = 8192
nat0 = q.hadamard_quant(x[:R], "full")[0]
lib.quarot_debug_hq_full_variant(3)
nat3 = q.hadamard_quant(x[:R], "full")[0]
lib.quarot_debug_hq_full_variant(0)
kp = q.hadamard_quant(x[:R], "full", kperm=True)[0]
perm = q.full_kperm(K)
inv = torch.empty_like(perm)
inv[perm] = torch.arange(K)
print("kperm == natural after un-permuting:", torch.equal(q.permute_k_packed(kp, inv), nat0), flush=True)
print("bytes differing variant 0 vs 3:", (nat0 != nat3).sum().item(), "of", nat0.numel(), flush=True)
