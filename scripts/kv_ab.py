"""KV Init (+RoPE) on the Llama-2-70B shapes (64 Q / 8 KV heads x 128) read out of a fused QKV
output, interleaved over rounds (median): algorithmic GB/s vs MEASURED_PEAKS hbm_gbs.
  VARIANTS=rope,norope TOKENS=131072 python scripts/kv_ab.py"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_00456_b200 as q  # noqa: E402

T = int(os.environ.get("TOKENS", 131072))
pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
hbm = json.load(open(pk))["hbm_gbs"] if os.path.exists(pk) else 6553.6
fused = synth.activations(T, 10240, "normal", 6, "cuda")
qv, kv_, vv = fused[:, :8192].view(T, 64, 128), fused[:, 8192:9216].view(T, 8, 128), fused[:, 9216:].view(T, 8, 128)
out = q.kv_quant(kv_, vv, qv)
nbytes = T * (2 * 8 * (2 * 128 + 64 + 5) + 4 * 64 * 128)


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


names = os.environ.get("VARIANTS", "rope,norope").split(",")
times = {n: [] for n in names}
for _ in range(int(os.environ.get("ROUNDS", 3))):
    for n in names:
        rope = (0, 2048, 10000.0) if n == "rope" else None
        times[n].append(timeit(lambda: q.kv_quant(kv_, vv, qv, out=out, rope=rope)))
for n in names:
    ms = statistics.median(times[n])
    gbs = nbytes / (ms * 1e-3) / 1e9
    print(n, json.dumps({"ms": ms, "all": [round(t, 4) for t in times[n]], "gbs": gbs, "frac_hbm": gbs / hbm}), flush=True)
