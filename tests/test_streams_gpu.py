"""Every entry point enqueues on the caller's stream (include/quarot.h conventions):
the hot-path calls are captured into a CUDA graph on a side stream — a launch on any other
stream (e.g. the legacy default stream) invalidates the capture — and the replay must equal
the eager result bit for bit."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    from paper_2404_00456_b200 import quarot
    quarot.lib()
    return quarot


def test_chain_captures_into_cuda_graph_and_replays_bitwise(q):
    from paper_2404_00456_b200.runtime import DecoderLayerStep, QuaRotLayer
    dev = "cuda"
    H, F, nh, nkv, T = 8192, 28672, 64, 8, 512   # 70B widths: the tcgen05 quantizers and KV kernel
    dims = {"qkv": ((nh + 2 * nkv) * 128, H), "o": (H, H), "gate_up": (2 * F, H), "down": (H, F)}
    wts = {n: (synth.packed_weight_codes(a, b, 40 + i, dev), synth.weight_scales(a, 50 + i, dev))
           for i, (n, (a, b)) in enumerate(dims.items())}
    step = DecoderLayerStep(QuaRotLayer(H, F, nh, nkv, 128, wts), T, dev)
    inp = {"x": synth.activations(T, H, "outlier", 60, dev) * 0.05, "attn_out": synth.activations(T, H, "normal", 61, dev)}
    step.run_device(inp)      # eager (also performs the one-time table uploads)
    torch.cuda.synchronize()
    eager = {k: t.clone() for k, t in step.result_tensors().items()}
    for t in step.result_tensors().values():
        t.zero_()
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        step.run_device(inp, stream=side)
    g.replay()
    torch.cuda.synchronize()
    for k, t in step.result_tensors().items():
        assert torch.equal(t, eager[k]), k


def test_side_stream_ordering(q):
    """hadamard_quant then int4_linear on a non-blocking side stream while the default stream is
    busy: the GEMM must see the quantizer's output (same stream order), equal to a default-stream run."""
    dev = "cuda"
    M, K, N = 4096, 28672, 8192
    x = synth.activations(M, K, "swiglu", 70, dev)
    wq, ws = synth.packed_weight_codes(N, K, 71, dev), synth.weight_scales(N, 72, dev)
    ref = q.int4_linear(*q.hadamard_quant(x, "full"), wq, ws)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    big = torch.empty(1 << 28, dtype=torch.float16, device=dev)
    xq = torch.empty(M, K // 2, dtype=torch.uint8, device=dev)
    xs = torch.empty(M, dtype=torch.float32, device=dev)
    for _ in range(3):
        big.normal_()          # keep the default stream busy
        xq.fill_(0x77)
        xs.fill_(float("nan"))
        s.wait_stream(torch.cuda.current_stream())
        big.mul_(2.0)
        q.hadamard_quant(x, "full", q=xq, scale=xs, stream=s)
        y = q.int4_linear(xq, xs, wq, ws, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        assert torch.equal(y, ref)


def test_prepare_then_first_call_inside_graph_capture():
    """quarot_prepare (one-time constant uploads) in a fresh process, then the FIRST quantizer and
    KV calls of that process inside a CUDA-graph capture on a side stream: no host
    synchronization happens during capture (it would invalidate it), and the replay equals an
    eager run bitwise."""
    import subprocess
    import sys
    code = r'''
import sys, torch
sys.path.insert(0, ".")
import synth
import paper_2404_00456_b200 as q
q.prepare()
x = synth.activations(300, 28672, "swiglu", 3, "cuda")
k, v, qq = synth.kv_inputs(64, 8, 64, 128, seed=2, device="cuda")
xq = torch.empty(300, 14336, dtype=torch.uint8, device="cuda")
xs = torch.empty(300, dtype=torch.float32, device="cuda")
out = {"k_codes": torch.empty(64, 8, 64, dtype=torch.uint8, device="cuda"),
       "k_scale": torch.empty(64, 8, dtype=torch.float32, device="cuda"),
       "k_zero": torch.empty(64, 8, dtype=torch.uint8, device="cuda"),
       "v_codes": torch.empty(64, 8, 64, dtype=torch.uint8, device="cuda"),
       "v_scale": torch.empty(64, 8, dtype=torch.float32, device="cuda"),
       "v_zero": torch.empty(64, 8, dtype=torch.uint8, device="cuda")}
qc = qq.clone()
side = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=side):
    q.hadamard_quant(x, "full", q=xq, scale=xs, kperm=True, stream=side)
    q.kv_quant(k, v, qc, out=out, rope=(0, 2048, 10000.0), stream=side)
g.replay()
torch.cuda.synchronize()
xq2, xs2 = q.hadamard_quant(x, "full", kperm=True)
qc2 = qq.clone()
out2 = q.kv_quant(k, v, qc2, rope=(0, 2048, 10000.0))
torch.cuda.synchronize()
assert torch.equal(xq, xq2) and torch.equal(xs, xs2)
assert torch.equal(qc, qc2) and all(torch.equal(out[n], out2[n]) for n in out)
print("OK")
'''
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
