"""A/B the FULL K=28672 (MODE=full) or ACROSS_HEADS (MODE=across_heads) quantizers: tcgen05 kernel (variant 0) vs the mma.sync kernel (variant 1).
Codes/scales agreement and CUDA-event timing at 131072 tokens.  python scripts/ab_hqfull.py [M]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_00456_b200 as q

M = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
K = int(sys.argv[2]) if len(sys.argv) > 2 else 28672
MODE = os.environ.get("MODE", "full")
lib = q.lib()
setv = lib.quarot_debug_hq_full_variant if MODE == "full" else lib.quarot_debug_hq_heads_variant
setv.argtypes = [ctypes.c_int]
x = synth.activations(M, K, "swiglu" if MODE == "full" else "normal", 5, "cuda")
res = {}
outs = {}
for var in [int(v) for v in os.environ.get("VARIANTS", "1,0").split(",")]:
    setv(var)
    for _ in range(3):
        o = q.hadamard_quant(x, MODE)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 10
    for _ in range(n):
        q.hadamard_quant(x, MODE)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    outs[var] = [t.clone() for t in o]
    res[var] = {"ms": ms, "gbs": M * (2.5 * K + 4) / ms / 1e6}
    print(var, json.dumps(res[var]), flush=True)
ks = list(outs); (q1, s1), (q0, s0) = outs[ks[0]], outs[ks[-1]]
def codes(p):
    lo = (p & 0xF).to(torch.int16); hi = (p >> 4).to(torch.int16)
    lo = torch.where(lo > 7, lo - 16, lo); hi = torch.where(hi > 7, hi - 16, hi)
    return torch.stack([lo, hi], -1).reshape(p.shape[0], -1)
c1, c0 = codes(q1), codes(q0)
d = (c1 - c0).abs()
print("scale rel max", ((s1 - s0).abs() / s1.abs()).max().item())
print("code diff frac", (d > 0).float().mean().item(), "max", d.max().item())
bad = (d > 0).nonzero()[:10]
print("first diffs", bad.tolist())
setv(0)
