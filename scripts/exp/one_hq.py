"""Run one hadamard_quant of a given mode / width a few times (ncu target).  MODE K [M] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_00456_b200 as q
mode, K = sys.argv[1], int(sys.argv[2])
M = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
x = synth.activations(M, K, "swiglu" if mode == "full" else "outlier", 5, "cuda")
for _ in range(reps):
    q.hadamard_quant(x, mode)
torch.cuda.synchronize()
