"""One group-wise GEMM launch (ncu target).  python scripts/one_group_gemm.py M N K"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_00456_b200 as q
M, N, K = (int(v) for v in sys.argv[1:4])
xq = torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda")
wq = torch.randint(-7, 8, (N, K), dtype=torch.int8, device="cuda")
xs = torch.rand(M, K // 128, device="cuda") * 0.01 + 0.001
ws = torch.rand(K // 128, N, device="cuda") * 0.01 + 0.001
for _ in range(2):
    q.int4_linear_group(xq, xs, wq, ws)
torch.cuda.synchronize()
