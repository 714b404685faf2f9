"""One append + decode at a tab:QAttention_bench shape (ncu target).  n_q n_kv B [L]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
import paper_2404_00456_b200 as q
n_q, n_kv, B = (int(v) for v in sys.argv[1:4])
L = int(sys.argv[4]) if len(sys.argv) > 4 else 2048
cache = q.kv_cache_empty(B, L, n_kv, 128)
k, v, qq = synth.kv_inputs(B, n_kv, n_q, 128, seed=1, device="cuda")
lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
for _ in range(3):
    q.kv_decode(qq, cache, lens)
torch.cuda.synchronize()
