"""One gate/up SwiGLU INT4 linear (ncu target).  M [N2] [K]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
import paper_2404_00456_b200 as q
M = int(sys.argv[1]); N = int(sys.argv[2]) if len(sys.argv) > 2 else 57344; K = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
xq = synth.packed_weight_codes(M, K, 1, "cuda"); wq = synth.packed_weight_codes(N, K, 2, "cuda")
xs = torch.rand(M, device="cuda") + 0.5; ws = synth.weight_scales(N, 3, "cuda")
y = torch.empty(M, N // 2, dtype=torch.float16, device="cuda")
for _ in range(2): q.int4_linear_swiglu(xq, xs, wq, ws, act=y)
torch.cuda.synchronize()
