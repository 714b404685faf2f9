"""One KV-cache Init (+RoPE) launch set at T tokens (ncu target).  python scripts/one_kv.py T [rope]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
import paper_2404_00456_b200 as q
T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
rope = len(sys.argv) > 2 and sys.argv[2] == "rope"
fused = synth.activations(T, 10240, "normal", 6, "cuda")
qv, kv_, vv = fused[:, :8192].view(T, 64, 128), fused[:, 8192:9216].view(T, 8, 128), fused[:, 9216:].view(T, 8, 128)
out = q.kv_quant(kv_, vv, qv)
for _ in range(2):
    q.kv_quant(kv_, vv, qv, out=out, rope=(0, 2048, 10000.0) if rope else None)
torch.cuda.synchronize()
