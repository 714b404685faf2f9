"""Full-matrix check of the INT4 GEMM against torch._int_mm (debug probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_00456_b200 as q


def unpack(p):
    lo = (p & 0xF).to(torch.int16); hi = ((p >> 4) & 0xF).to(torch.int16)
    lo = torch.where(lo >= 8, lo - 16, lo); hi = torch.where(hi >= 8, hi - 16, hi)
    return torch.stack([lo, hi], -1).reshape(p.shape[0], -1).to(torch.int8)


K = int(os.environ.get("K", 8192))
for M, N in ((256, 8192), (2048, 8192), (16384, 8192)):
    xq = synth.packed_weight_codes(M, K, 1, "cuda")
    wq = synth.packed_weight_codes(N, K, 2, "cuda")
    ref = torch._int_mm(unpack(xq), unpack(wq).t())
    for rep in range(2):
        acc = q.int4_matmul_s32(xq, wq)
        bad = acc != ref
        nb = bad.sum().item()
        msg = f"M={M} rep={rep} bad={nb}"
        if nb:
            idx = bad.nonzero()
            r, c = idx[:, 0], idx[:, 1]
            msg += f" rows%256 hist={torch.bincount(r % 256 // 32, minlength=8).tolist()} cols%256/16={torch.bincount(c % 256 // 16, minlength=16).tolist()}"
            msg += f" mtiles={torch.unique(r // 256).tolist()[:10]} ntiles={torch.unique(c // 256).tolist()[:12]}"
            d = (acc - ref)[bad]
            msg += f" diff sample={d[:6].tolist()}"
        print(msg, flush=True)
    xs = torch.rand(M, device="cuda") * 0.01 + 0.001
    ws = synth.weight_scales(N, 3, "cuda")
    y = q.int4_linear(xq, xs, wq, ws).double()
    yr = ref.double() * xs.double()[:, None] * ws.double()[None, :]
    bad = (y - yr).abs() > 2e-3 * yr.abs() + 1e-4
    nb = bad.sum().item()
    msg = f"  fp16 M={M} bad={nb}"
    if nb:
        idx = bad.nonzero(); r, c = idx[:, 0], idx[:, 1]
        msg += f" rows%256/32={torch.bincount(r % 256 // 32, minlength=8).tolist()} cols%256/16={torch.bincount(c % 256 // 16, minlength=16).tolist()}"
        msg += f" mtiles={torch.unique(r // 256).tolist()[:10]} ntiles={torch.unique(c // 256).tolist()[:12]}"
    print(msg, flush=True)
