import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_00456_b200 as q
what = sys.argv[1]
if what == "gemm":
    xq = synth.packed_weight_codes(300, 512, 1, "cuda"); wq = synth.packed_weight_codes(776, 512, 2, "cuda")
    acc = q.int4_matmul_s32(xq, wq); torch.cuda.synchronize(); print("gemm ok", acc.shape)
elif what == "full28":
    x = synth.activations(5, 28672, "outlier", 1, "cuda")
    a, s = q.hadamard_quant(x, "full"); torch.cuda.synchronize(); print("full28 ok", s)
