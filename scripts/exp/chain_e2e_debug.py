"""Where does the end-to-end chain error at 70B widths come from?  GPU chain vs oracle.decoder_layer
on 256 tokens: per-intermediate relative Frobenius / ulp, and code flips of each quantizer when the
oracle quantizes its OWN intermediate vs the GPU quantizing the GPU's."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth
from oracle import glue as oglue, layer as olayer
from tests import _parity as P
from paper_2404_00456_b200.runtime import DecoderLayerStep, QuaRotLayer
import paper_2404_00456_b200 as q
dev = "cuda"
H, F, nh, nkv, T = 8192, 28672, 64, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = {"qkv": ((nh + 2 * nkv) * 128, H), "o": (H, H), "gate_up": (2 * F, H), "down": (H, F)}
w = {n: (synth.packed_weight_codes(a, b, 2000 + i, dev), synth.weight_scales(a, 2010 + i, dev))
     for i, (n, (a, b)) in enumerate(dims.items())}
step = DecoderLayerStep(QuaRotLayer(H, F, nh, nkv, 128, w), T, dev)
x = synth.activations(T, H, "outlier", 100, dev) * 0.05
z = synth.activations(T, H, "normal", 101, dev)
step.run_device({"x": x, "attn_out": z})
gu_gpu = q.int4_linear(*q.hadamard_quant(step.o, "none", rmsnorm=True), *w["gate_up"])
torch.cuda.synchronize()
wo = {n: (P.unpack_signed(a.cpu().numpy()), b.cpu().numpy()) for n, (a, b) in w.items()}
ref = oglue.decoder_layer(x.cpu().numpy(), z.cpu().numpy(), wo, np.arange(T) % 2048,
                          {"n_heads": nh, "n_kv": nkv, "head_dim": 128, "ffn": F})
def rep(name, g, r):
    g = np.asarray(g, np.float64); r = np.asarray(r, np.float64)
    print(f"{name:8s} frob {P.frob_rel(g, r):.3e}  maxulp {P.max_fp16_ulp(g.astype(np.float16), r.astype(np.float16))}"
          f"  |r| rms {np.sqrt(np.mean(r*r)):.3e}")
rep("o", step.o.cpu().numpy(), ref["o"])
rep("gate_up", gu_gpu.cpu().numpy(), ref["gate_up"])
rep("act", step.act.cpu().numpy(), ref["act"])
rep("out", step.out.cpu().numpy(), ref["out"])
rep("out-o", step.out.cpu().numpy().astype(np.float64) - step.o.cpu().numpy(), ref["out"].astype(np.float64) - ref["o"])
# quantizer flips: GPU codes of GPU act vs oracle codes of oracle act
xq, xs = q.hadamard_quant(step.act, "full")
gc = P.unpack_signed(xq.cpu().numpy())
rc, _, rs = olayer.hadamard_quant(ref["act"].astype(np.float64), "full")
print("act codes (own inputs):", P.code_stats(gc, rc), "scale rel", np.max(np.abs(xs.cpu().numpy() / rs - 1)))
xq2, xs2 = q.hadamard_quant(step.o, "none", rmsnorm=True)
rc2, _, rs2 = oglue.rmsnorm_quant(ref["o"].astype(np.float64))
print("o codes (own inputs):", P.code_stats(P.unpack_signed(xq2.cpu().numpy()), rc2))
# per-row error of out
e = np.linalg.norm(step.out.cpu().numpy().astype(np.float64) - ref["out"], axis=1) / np.linalg.norm(ref["out"].astype(np.float64), axis=1)
print("per-row out rel err: median %.3e  p90 %.3e  max %.3e" % (np.median(e), np.percentile(e, 90), e.max()))
print("rows by err:", np.argsort(-e)[:8], e[np.argsort(-e)[:8]])
