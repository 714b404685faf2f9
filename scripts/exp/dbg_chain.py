import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_00456_b200 as q
from paper_2404_00456_b200.runtime import QuaRotLayer, DecoderLayerStep
S = {"hidden": 512, "ffn": 28 * 32, "n_heads": 4, "n_kv": 1}
S["qkv"] = (S["n_heads"] + 2 * S["n_kv"]) * 128
dims = {"qkv": (S["qkv"], S["hidden"]), "o": (S["hidden"], S["hidden"]), "gate_up": (2 * S["ffn"], S["hidden"]), "down": (S["hidden"], S["ffn"])}
w = {n: (synth.packed_weight_codes(a, b, 2000 + i, "cuda"), synth.weight_scales(a, 2010 + i, "cuda")) for i, (n, (a, b)) in enumerate(dims.items())}
layer = QuaRotLayer(S["hidden"], S["ffn"], S["n_heads"], S["n_kv"], 128, w)
T = 300
x = synth.activations(T, S["hidden"], "outlier", 100, "cuda") * 0.05
z = synth.activations(T, S["hidden"], "normal", 101, "cuda")
step = DecoderLayerStep(layer, T, "cuda")
step.run_device({"x": x, "attn_out": z})
torch.cuda.synchronize()
xq, xs = q.hadamard_quant(step.o, "none", rmsnorm=True)
act_u = q.swiglu(q.int4_linear(xq, xs, *w["gate_up"]))
act_f = q.int4_linear_swiglu(xq, xs, *q.interleave_gate_up(*w["gate_up"]))
print("fused-vs-unfused (fresh)", (act_f.float() - act_u.float()).abs().max().item())
print("step.act vs fresh fused", (step.act.float() - act_f.float()).abs().max().item(), step.act.float().abs().max().item())
il = step.gate_up_il
print("il equal", torch.equal(il[0], q.interleave_gate_up(*w["gate_up"])[0]))
import numpy as np
from oracle import glue as oglue, quant as oquant
from tests import _parity as P
F = S["ffn"]
g_o = step.o.cpu().numpy()
co, _, so = oglue.rmsnorm_quant(g_o.astype(np.float64))
fcols = np.arange(0, F, 7)
gucols = np.concatenate([fcols, F + fcols])
gct = torch.as_tensor(gucols, device="cuda")
ref = oglue.linear_swiglu(co, so, oquant.unpack_int4_signed(w["gate_up"][0][gct].cpu().numpy()), w["gate_up"][1][gct].cpu().numpy(), len(fcols))
g = step.act.cpu().numpy()[:, fcols]
print("ulp", P.max_fp16_ulp(g, ref), g[0, :5], ref[0, :5])
print("codes equal gpu", np.array_equal(P.unpack_signed(xq.cpu().numpy()), co), "scale rel", np.max(np.abs(xs.cpu().numpy()/so-1)))
