"""One group-wise GEMM launch (ncu target).  python scripts/exp/one_group_gemm.py M N K G [packed|int8]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2404_00456_b200 as q
M, N, K, G = (int(v) for v in sys.argv[1:5])
kind = sys.argv[5] if len(sys.argv) > 5 else "packed"
xs = torch.rand(M, K // G, device="cuda") * 0.01 + 0.001
ws = torch.rand(K // G, N, device="cuda") * 0.01 + 0.001
if kind == "packed":
    xq = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda")
    wq = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda")
    fn = lambda: q.int4_linear_group(xq, xs, wq, ws, group=G)
else:
    xq = torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda")
    wq = torch.randint(-7, 8, (N, K), dtype=torch.int8, device="cuda")
    fn = lambda: q.int4_linear_group8(xq, xs, wq, ws)
for _ in range(2):
    fn()
torch.cuda.synchronize()
