"""KV Init (+RoPE) at the 7B (32 / 32 heads) and 70B (64 / 8) shapes and token counts: ms and % of HBM."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2404_00456_b200 as q
pk = os.path.join(os.getcwd(), "MEASURED_PEAKS.json")
HBM = json.load(open(pk))["hbm_gbs"] if os.path.exists(pk) else 6553.6
def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters
for n_q, n_kv in ((32, 32), (64, 8)):
    for T in (16384, 131072):
        W = (n_q + 2 * n_kv) * 128
        fused = synth.activations(T, W, "normal", 6, "cuda")
        qv = fused[:, :n_q * 128].view(T, n_q, 128)
        kv_ = fused[:, n_q * 128:(n_q + n_kv) * 128].view(T, n_kv, 128)
        vv = fused[:, (n_q + n_kv) * 128:].view(T, n_kv, 128)
        out = q.kv_quant(kv_, vv, qv)
        byts = T * (2 * n_kv * (2 * 128 + 64 + 5) + 4 * n_q * 128)
        for rope in (None, (0, 2048, 10000.0)):
            ms = timeit(lambda: q.kv_quant(kv_, vv, qv, out=out, rope=rope))
            print(f"nq={n_q} nkv={n_kv} T={T} rope={rope is not None} {ms:.4f} ms {byts / ms / 1e6 / HBM:.3f} of HBM", flush=True)
        del fused, out; torch.cuda.empty_cache()
