import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2404_00456_b200 as q
for M in (1, 2, 3, 150, 300):
    x = synth.activations(M, 28672, "swiglu", 3, "cuda")
    xq, xs = q.hadamard_quant(x, "full")
    torch.cuda.synchronize()
    print("M", M, "ok", flush=True)
