"""One FULL hadamard_quant launch set (ncu target).  python scripts/exp/one_hqfull.py M K [variant] [kperm]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
import paper_2404_00456_b200 as q
M, K = int(sys.argv[1]), int(sys.argv[2])
var = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kperm = len(sys.argv) > 4 and sys.argv[4] == "kperm"
q.lib().quarot_debug_hq_full_variant.argtypes = [ctypes.c_int]
q.lib().quarot_debug_hq_full_variant(var)
x = synth.activations(M, K, "swiglu", 5, "cuda")
for _ in range(2):
    q.hadamard_quant(x, "full", kperm=kperm)
torch.cuda.synchronize()
