import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np, synth
import paper_2404_00456_b200 as q
DEV = "cuda"
for (M, N, K) in ((300, 512, 4096), (512, 512, 4096), (256, 256, 4096), (1024, 1024, 8192)):
    xq = synth.packed_weight_codes(M, K, 1, DEV)
    wq = synth.packed_weight_codes(N, K, 2, DEV)
    xs = torch.rand(M, device=DEV) * 0.01 + 0.001
    ws = synth.weight_scales(N, 3, DEV)
    r = synth.activations(M, N, "normal", 4, DEV)
    y = q.int4_linear(xq, xs, wq, ws, residual=r)
    y0 = q.int4_linear(xq, xs, wq, ws) + r
    torch.cuda.synchronize()
    bad = (y != y0).nonzero()
    print(M, N, K, "mismatches", bad.shape[0], flush=True)
    if bad.shape[0]:
        rows = torch.unique(bad[:, 0]); cols = torch.unique(bad[:, 1])
        print(" rows", rows[:20].tolist(), "... n", rows.numel(), " cols", cols[:20].tolist(), "... n", cols.numel())
        i, j = bad[0].tolist()
        print(" e.g.", i, j, y[i, j].item(), y0[i, j].item(), "r", r[i, j].item(), "lin", (y0[i,j]-r[i,j]).item())
