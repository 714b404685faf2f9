import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2404_00456_b200 as q
T, n_kv, n_q, hd = 37, 8, 64, 128
k, v, qq = synth.kv_inputs(T, n_kv, n_q, hd, seed=T + 1, device="cuda")
q_f = qq.clone()
out = q.kv_quant(k, v, q_f, rope=(0, 2048, 10000.0))
q2 = qq.clone(); k2 = k.clone()
q.rope(q2, pos0=0, seq_len=2048); q.rope(k2, pos0=0, seq_len=2048)
out2 = q.kv_quant(k2, v, q2)
torch.cuda.synchronize()
d = (q_f.view(torch.int16) != q2.view(torch.int16))
print("q differ:", d.sum().item(), "of", d.numel())
idx = d.nonzero()[:20]
print(idx.tolist())
# undo H: compare RoPE'd (pre-H) values by running kv_quant without H? print a few values
for key in ("k_codes", "k_scale", "k_zero", "v_codes"):
    print(key, torch.equal(out[key], out2[key]))
