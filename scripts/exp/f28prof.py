"""Phase timing of the FULL-28672 quantizer (variant built with -DQR_F28_PROF)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["QUAROT_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "_variants", "libquarot_f28prof.so")
import numpy as np, torch, synth
import paper_2404_00456_b200 as q
M = 32768
x = synth.activations(M, 28672, "swiglu", 5, "cuda")
q.hadamard_quant(x, "full")
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (148 * 8))()
q.lib().quarot_debug_f28_prof(buf)  # reset
q.hadamard_quant(x, "full")
torch.cuda.synchronize()
q.lib().quarot_debug_f28_prof(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 8).astype(np.float64)
rows = M / 148
names = ["p1_wait_xs", "p1_wait_zempty", "p1_total", "p2_wait_zfull", "p2_total"]
for i, n in enumerate(names):
    print(f"{n:16s} cycles/row {a[:, i].mean() / rows:10.1f}")
