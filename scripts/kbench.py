"""Kernel micro-benchmarks (CUDA events, warm, inputs > L2) for fast iteration on the GPU box.

  python scripts/kbench.py [gemm] [hq] [kv] [--tokens 131072]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_00456_b200 as q  # noqa: E402


def _peaks():
    """HBM GB/s and the INT8 TOPS denominator (2 x sustained bf16) from MEASURED_PEAKS.json."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), 2.0 * float(p.get("bf16_tflops_sustained", p["bf16_tflops"]))
    except (OSError, KeyError, ValueError):
        return 6650.0, 2800.0  # B200_PROFILING.md fallback (6.65 TB/s, 2 x 1.4 PF sustained bf16)


HBM_GBS, INT8_TOPS = _peaks()


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="*", default=["gemm", "hq", "kv"])
    ap.add_argument("--tokens", type=int, default=131072)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    M = a.tokens
    dev = "cuda"
    res = {}
    if "gemm_mmaonly" in a.what:
        # roofline probe: the same kernel with producers disabled (MMA issue rate only)
        import ctypes
        q.lib().quarot_debug_gemm_mode.argtypes = [ctypes.c_int]
        xq = synth.packed_weight_codes(M, 8192, 1, dev)
        N, K = 57344, 8192
        wq = synth.packed_weight_codes(N, K, 2, dev)
        xs = torch.rand(M, device=dev) + 0.5
        ws = synth.weight_scales(N, 3, dev)
        y = torch.empty(M, N, dtype=torch.float16, device=dev)
        for mode, name in ((0, "normal"), (1, "mma_only"), (2, "no_widen_stores"), (3, "no_tma")):
            q.lib().quarot_debug_gemm_mode(mode)
            ms = timeit(lambda: q.int4_linear(xq, xs, wq, ws, y=y), a.iters)
            res["gate_up_" + name] = {"ms": ms, "tops": 2 * M * N * K / ms / 1e9}
            print(name, json.dumps(res["gate_up_" + name]), flush=True)
        q.lib().quarot_debug_gemm_mode(0)
    if "ksweep" in a.what:
        # per-tile fixed cost: time(K) = tiles/pairs * (t_tile0 + t_kb * K / 256)
        import ctypes
        q.lib().quarot_debug_gemm_mode.argtypes = [ctypes.c_int]
        Ms, N = 65536, 8192
        xq_big = synth.packed_weight_codes(Ms, 32768, 1, dev)
        wq_big = synth.packed_weight_codes(N, 32768, 2, dev)
        xs = torch.rand(Ms, device=dev) + 0.5
        ws = synth.weight_scales(N, 3, dev)
        y = torch.empty(Ms, N, dtype=torch.float16, device=dev)
        for mode in [int(m) for m in os.environ.get("KSWEEP_MODES", "0,1").split(",")]:
            q.lib().quarot_debug_gemm_mode(mode)
            for K in (8192, 16384, 32768):
                xq, wq = xq_big[:, : K // 2], wq_big[:, : K // 2]
                ms = timeit(lambda: q.int4_linear(xq, xs, wq, ws, y=y), a.iters)
                tiles_per_pair = (Ms // 256) * (N // 256) / 74
                print(json.dumps({"mode": mode, "K": K, "ms": ms, "tops": 2 * Ms * N * K / ms / 1e9,
                                  "us_per_tile": ms * 1e3 / tiles_per_pair}), flush=True)
        q.lib().quarot_debug_gemm_mode(0)
        del xq_big, wq_big, y
    if "gemm" in a.what:
        xq_big = synth.packed_weight_codes(M, 28672, 1, dev)
        for name, N, K in (("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 57344, 8192), ("down", 8192, 28672)):
            xq = xq_big[:, : K // 2]
            wq = synth.packed_weight_codes(N, K, 2, dev)
            xs = torch.rand(M, device=dev) + 0.5
            ws = synth.weight_scales(N, 3, dev)
            y = torch.empty(M, N, dtype=torch.float16, device=dev)
            ms = timeit(lambda: q.int4_linear(xq, xs, wq, ws, y=y), a.iters)
            tops = 2 * M * N * K / ms / 1e9
            res[f"gemm_{name}"] = {"ms": ms, "tops": tops, "frac_int8_2x_bf16_sustained": tops / INT8_TOPS}
            print(name, json.dumps(res[f"gemm_{name}"]), flush=True)
            del wq, y
        del xq_big
    if "hq" in a.what:
        cases = [c.split(":") for c in os.environ.get("HQ_CASES", "none:8192,none_rms:8192,across_heads:8192,full:28672,full:11008,none:4096").split(",")]
        for mode, K in cases:
            K = int(K)
            x = synth.activations(M, K, "outlier", 5, dev)
            qb = torch.empty(M, K // 2, dtype=torch.uint8, device=dev)
            sb = torch.empty(M, dtype=torch.float32, device=dev)
            rms = mode == "none_rms"
            ms = timeit(lambda: q.hadamard_quant(x, "none" if rms else mode, 128, 0.9, q=qb, scale=sb, rmsnorm=rms), a.iters)
            gbs = M * (2.5 * K + 4) / ms / 1e6
            res[f"hq_{mode}_{K}"] = {"ms": ms, "gbs": gbs, "frac_hbm": gbs / HBM_GBS}
            print(mode, K, json.dumps(res[f"hq_{mode}_{K}"]), flush=True)
            del x
    if "kv" in a.what:
        fused = synth.activations(M, 10240, "normal", 6, dev)
        T, d = M, 128
        qv = fused[:, :8192].view(T, 64, d)
        kv_ = fused[:, 8192:9216].view(T, 8, d)
        vv = fused[:, 9216:].view(T, 8, d)
        out = q.kv_quant(kv_, vv, qv)
        ms = timeit(lambda: q.kv_quant(kv_, vv, qv, out=out), a.iters)
        byts = 2 * T * 8 * (2 * d + d // 2 + 5) + T * 64 * d * 4
        res["kv"] = {"ms": ms, "gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / HBM_GBS}
        print("kv", json.dumps(res["kv"]), flush=True)
        ms = timeit(lambda: q.kv_quant(kv_, vv, qv, out=out, rope=(0, 2048, 10000.0)), a.iters)
        res["kv_rope"] = {"ms": ms, "gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / HBM_GBS}
        print("kv_rope", json.dumps(res["kv_rope"]), flush=True)
        ms = timeit(lambda: q.rope(fused[:, :9216].view(T, 72, d)), a.iters)
        print("rope", json.dumps({"ms": ms}), flush=True)
    if "decode" in a.what:
        # SURVEY §8 f2 / tab:QAttention_bench: append + decode of one token per sequence on a
        # cache of 2047 rows (seq_len 2048); bytes = the INT4 cache rows read (codes + scales)
        for n_q, n_kv in ((32, 32), (40, 40), (64, 64), (64, 8)):
            for B in (1, 8, 16, 32, 64):
                L, d = 2048, 128
                cache = q.kv_cache_empty(B, L, n_kv, d)
                kn, vn, qn = synth.kv_inputs(B, n_kv, n_q, d, seed=1, device=dev)
                pos = torch.full((B,), L - 1, dtype=torch.int32, device=dev)
                lens = torch.full((B,), L, dtype=torch.int32, device=dev)
                out = torch.empty(B, n_q, d, dtype=torch.float16, device=dev)
                ws = torch.empty(q.lib().quarot_kv_decode_workspace_bytes(B, n_q, d, L) // 4, device=dev)
                qb = qn.clone()

                def step():
                    qb.copy_(qn)
                    q.kv_append(kn, vn, qb, pos, cache)
                    q.kv_decode(qb, cache, lens, out=out, workspace=ws)
                ms = timeit(step, max(a.iters, 20))
                ms_dec = timeit(lambda: q.kv_decode(qb, cache, lens, out=out, workspace=ws), max(a.iters, 20))
                byts = B * n_kv * L * (2 * d // 2 + 10)
                key = f"decode_{n_q}x{n_kv}_b{B}"
                res[key] = {"ms_append_decode": ms, "ms_decode": ms_dec, "gbs_decode": byts / ms_dec / 1e6,
                            "frac_hbm": byts / ms_dec / 1e6 / HBM_GBS}
                print(key, json.dumps(res[key]), flush=True)
                del cache
    if "gemm_group" in a.what:
        # group-wise W4A4 GEMM on packed INT4 codes (G = 64 / 128 / 256) and the
        # int8-stored-codes variant (G = 128); the Llama-2-70B linear shapes
        xq_big = torch.randint(0, 256, (M, 28672 // 2), dtype=torch.uint8, device=dev)
        xq8_big = torch.randint(-7, 8, (M, 28672), dtype=torch.int8, device=dev)
        for name, N, K in (("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 57344, 8192), ("down", 8192, 28672)):
            wq = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev)
            y = torch.empty(M, N, dtype=torch.float16, device=dev)
            for G in (64, 128, 256):
                xs = torch.rand(M, K // G, device=dev) * 0.01 + 0.001
                ws = torch.rand(K // G, N, device=dev) * 0.01 + 0.001
                ms = timeit(lambda: q.int4_linear_group(xq_big[:, :K // 2], xs, wq, ws, group=G, y=y), a.iters)
                tops = 2 * M * N * K / ms / 1e9
                res[f"gemm_group{G}_{name}"] = {"ms": ms, "tops": tops, "frac_int8_2x_bf16_sustained": tops / INT8_TOPS}
                print(f"group{G}", name, json.dumps(res[f"gemm_group{G}_{name}"]), flush=True)
            del wq
            wq8 = torch.randint(-7, 8, (N, K), dtype=torch.int8, device=dev)
            xs = torch.rand(M, K // 128, device=dev) * 0.01 + 0.001
            ws = torch.rand(K // 128, N, device=dev) * 0.01 + 0.001
            ms = timeit(lambda: q.int4_linear_group8(xq8_big[:, :K], xs, wq8, ws, y=y), a.iters)
            tops = 2 * M * N * K / ms / 1e9
            res[f"gemm_group8_{name}"] = {"ms": ms, "tops": tops}
            print("group8 (int8-stored)", name, json.dumps(res[f"gemm_group8_{name}"]), flush=True)
            del wq8, y
        del xq_big, xq8_big
    if "gemm8" in a.what:
        # A8W8: the native kind::i8 path, same shapes as the W4A4 bench; the
        # difference to "gemm" is the cost of unpacking INT4 on B200
        xq_big = torch.randint(-127, 128, (M, 28672), dtype=torch.int8, device=dev)
        for name, N, K in (("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 57344, 8192), ("down", 8192, 28672)):
            xq = xq_big[:, :K]
            wq = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
            xs = torch.rand(M, device=dev) + 0.5
            ws = synth.weight_scales(N, 3, dev)
            y = torch.empty(M, N, dtype=torch.float16, device=dev)
            ms = timeit(lambda: q.int8_linear(xq, xs, wq, ws, y=y), a.iters)
            tops = 2 * M * N * K / ms / 1e9
            res[f"gemm8_{name}"] = {"ms": ms, "tops": tops, "frac_int8_2x_bf16_sustained": tops / INT8_TOPS}
            print("a8w8", name, json.dumps(res[f"gemm8_{name}"]), flush=True)
            del wq, y
        del xq_big
    if "intmm" in a.what:
        # library INT8 reference: cuBLASLt via torch._int_mm, 8192^3 (denominator context)
        A = torch.randint(-7, 8, (8192, 8192), dtype=torch.int8, device=dev)
        B = torch.randint(-7, 8, (8192, 8192), dtype=torch.int8, device=dev)
        ms = timeit(lambda: torch._int_mm(A, B), a.iters)
        res["cublaslt_int8_8192"] = {"ms": ms, "tops": 2 * 8192**3 / ms / 1e9}
        print("intmm", json.dumps(res["cublaslt_int8_8192"]), flush=True)
        Ab = A.to(torch.bfloat16)
        Bb = B.to(torch.bfloat16)
        ms = timeit(lambda: Ab @ Bb, a.iters)
        res["cublas_bf16_8192"] = {"ms": ms, "tflops": 2 * 8192**3 / ms / 1e9}
        print("bf16", json.dumps(res["cublas_bf16_8192"]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
