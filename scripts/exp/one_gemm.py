"""Run one INT4 linear of a given shape a few times (ncu target).  M N K [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
import paper_2404_00456_b200 as q
M, N, K = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
xq = synth.packed_weight_codes(M, K, 1, "cuda")
wq = synth.packed_weight_codes(N, K, 2, "cuda")
xs = torch.rand(M, device="cuda") + 0.5
ws = synth.weight_scales(N, 3, "cuda")
y = torch.empty(M, N, dtype=torch.float16, device="cuda")
for _ in range(reps):
    q.int4_linear(xq, xs, wq, ws, y=y)
torch.cuda.synchronize()
