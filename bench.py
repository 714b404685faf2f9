#!/usr/bin/env python
"""QuaRot hot-path benchmark (driver contract).

A step = one pass of every SURVEY §8(a) row over one batch: one Llama-2-70B decoder layer
(hidden 8192, FFN 28672 = 1024 x H_28, 64 Q / 8 KV heads x 128) prefilling 64 x 2048 = 131072
tokens per GPU, as the chain of runtime.DecoderLayerStep (attention core excluded):
RMSNorm+quantize -> INT4 QKV GEMM -> RoPE -> KV-cache Init (+Q rotation) ; Hadamard-heads +
quantize -> INT4 O GEMM + residual ; RMSNorm+quantize -> INT4 gate/up GEMM -> SwiGLU ;
Hadamard (1024 x H_28) + quantize -> INT4 down GEMM + residual (9 kernel launches, all ours).
`--step linears` times rows a1-a7 alone on independent inputs (9 launches).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 runs under torchrun, one process per GPU; each rank processes its own 64 x 2048
batch (token sharding, weak scaling, no collective on the data path); rank 0 prints one
JSON line with the whole-job tokens/s = N * tokens / max-over-ranks time.
`--impl reference` times the CPU oracle (the parity reference) on a bounded token sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "llama2-70b layer prefill tokens/s (QuaRot W4A4 hot path)"
UNIT = "tokens/s"
WORKLOAD = "llama2-70b-layer-prefill-64x2048"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16_burst": p["bf16_tflops"],
                "bf16_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_burst": 1590.0, "bf16_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def make_layer(device, seed_base=1000):
    from paper_2404_00456_b200.runtime import QuaRotLayer
    S = synth.inputs.LLAMA2_70B
    shapes = {"qkv": (S.qkv_out, S.hidden), "o": (S.hidden, S.hidden), "gate_up": (2 * S.ffn, S.hidden),
              "down": (S.hidden, S.ffn)}
    weights = {}
    for i, (name, (n, k)) in enumerate(shapes.items()):
        weights[name] = (synth.packed_weight_codes(n, k, seed_base + i, device=device),
                         synth.weight_scales(n, seed_base + 10 + i, device=device))
    return QuaRotLayer(S.hidden, S.ffn, S.n_heads, S.n_kv_heads, S.head_dim, weights)


def make_inputs(tokens, device, rank, step="chain"):
    S = synth.inputs.LLAMA2_70B
    base = 100 + 10 * rank
    if step == "chain":
        return {"x": synth.activations(tokens, S.hidden, "outlier", base + 0, device),
                "attn_out": synth.activations(tokens, S.hidden, "normal", base + 1, device)}
    return {"attn_in": synth.activations(tokens, S.hidden, "outlier", base + 0, device),
            "attn_out": synth.activations(tokens, S.hidden, "normal", base + 1, device),
            "ffn_in": synth.activations(tokens, S.hidden, "outlier", base + 2, device),
            "ffn_act": synth.activations(tokens, S.ffn, "swiglu", base + 3, device)}


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


# ----------------------------------------------------------------------------- CPU oracle

def oracle_step(host_in: dict, host_w: dict, layer_dims: dict) -> None:
    """The CPU oracle (oracle/) on host rows: the same 9 steps, fp64 / int64."""
    from oracle import kv as okv
    from oracle import layer as olayer
    from oracle import quant as oquant
    hd = layer_dims["head_dim"]
    outs = {}
    for name, key, mode in (("qkv", "attn_in", "none"), ("o", "attn_out", "across_heads"),
                            ("gate_up", "ffn_in", "none"), ("down", "ffn_act", "full")):
        x = host_in[key].astype(np.float64)
        cx, _, sx = olayer.hadamard_quant(x, mode, hd, 0.9)
        wq, ws = host_w[name]
        ys = []
        for r0 in range(0, wq.shape[0], 2048):   # weight rows in blocks to bound memory
            cw = oquant.unpack_int4_signed(wq[r0:r0 + 2048])
            ys.append(olayer.int4_linear(cx, sx, cw, ws[r0:r0 + 2048])[1])
        outs[name] = np.concatenate(ys, axis=1)
        if name == "qkv":
            y = outs["qkv"].astype(np.float64)
            T, nq, nkv = y.shape[0], layer_dims["n_heads"] * hd, layer_dims["n_kv"] * hd
            okv.kv_init(y[:, nq:nq + nkv].reshape(T, -1, hd), y[:, nq + nkv:].reshape(T, -1, hd),
                        y[:, :nq].reshape(T, -1, hd))
    return outs


def _block_linear(cx, sx, wq, ws, residual=None):
    """Oracle int4 linear with the packed weights unpacked in row blocks (memory bound)."""
    from oracle import layer as olayer
    from oracle import quant as oquant
    ys = []
    for r0 in range(0, wq.shape[0], 2048):
        cw = oquant.unpack_int4_signed(wq[r0:r0 + 2048])
        acc = olayer.int4_linear(cx, sx, cw, ws[r0:r0 + 2048])[0]
        ys.append(acc * sx.astype(np.float64)[:, None] * ws[r0:r0 + 2048].astype(np.float64)[None, :])
    y = np.concatenate(ys, axis=1)
    if residual is not None:
        y = y + residual.astype(np.float64)
    return y.astype(np.float16)


def oracle_chain_step(host_in: dict, host_w: dict, dims: dict, positions) -> dict:
    """The CPU oracle on host rows for the decoder-layer chain (oracle/glue.py pieces)."""
    from oracle import glue as oglue
    from oracle import kv as okv
    from oracle import layer as olayer
    d, nh, nkv, F = dims["head_dim"], dims["n_heads"], dims["n_kv"], dims["ffn"]
    x = host_in["x"]
    T = x.shape[0]
    cx, _, sx = oglue.rmsnorm_quant(x.astype(np.float64))
    qkv = _block_linear(cx, sx, *host_w["qkv"]).astype(np.float64)
    nq, nk = nh * d, nkv * d
    qr = oglue.rope(qkv[:, :nq].reshape(T, nh, d), positions).astype(np.float16).astype(np.float64)
    kr = oglue.rope(qkv[:, nq:nq + nk].reshape(T, nkv, d), positions).astype(np.float16).astype(np.float64)
    cache = okv.kv_init(kr, qkv[:, nq + nk:].reshape(T, nkv, d), qr)
    cz, _, sz = olayer.hadamard_quant(host_in["attn_out"].astype(np.float64), "across_heads", d)
    o = _block_linear(cz, sz, *host_w["o"], residual=x)
    co, _, so = oglue.rmsnorm_quant(o.astype(np.float64))
    wq_gu, ws_gu = host_w["gate_up"]
    acts = []
    for f0 in range(0, F, 1024):  # gate/up rows in blocks (memory bound), SwiGLU on fp64 values
        from oracle import quant as oquant
        f1 = min(F, f0 + 1024)
        rows_blk = np.concatenate([np.arange(f0, f1), F + np.arange(f0, f1)])
        acts.append(oglue.linear_swiglu(co, so, oquant.unpack_int4_signed(wq_gu[rows_blk]), ws_gu[rows_blk], f1 - f0))
    act = np.concatenate(acts, axis=1)
    ca, _, sa = olayer.hadamard_quant(act.astype(np.float64), "full", d)
    return {"out": _block_linear(ca, sa, *host_w["down"], residual=o), "cache": cache}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        blas = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        blas = 1
    return len(os.sched_getaffinity(0)), blas


def host_sample(inputs: dict, layer, sample: int):
    rows = torch.linspace(0, next(iter(inputs.values())).shape[0] - 1, sample).round().long()
    host_in = {k: v[rows.to(v.device)].cpu().numpy() for k, v in inputs.items()}
    host_w = {k: (w.cpu().numpy(), s.cpu().numpy()) for k, (w, s) in layer.weights.items()}
    return host_in, host_w, rows.numpy()


def layer_dims(layer):
    return {"head_dim": layer.head_dim, "n_heads": layer.n_heads, "n_kv": layer.n_kv, "ffn": layer.ffn}


def run_oracle(args, host_in, host_w, layer, rows):
    if args.step == "chain":
        return oracle_chain_step(host_in, host_w, layer_dims(layer), rows % 2048)
    return oracle_step(host_in, host_w, layer_dims(layer))


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on bounded token samples."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    device = "cuda" if torch.cuda.is_available() else "cpu"
    layer = make_layer(device)
    sample = args.ref_tokens
    inputs = make_inputs(sample * 16, device, 0, args.step)
    host_in, host_w, rows = host_sample(inputs, layer, sample)
    for _ in range(args.warmup):
        run_oracle(args, host_in, host_w, layer, rows)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run_oracle(args, host_in, host_w, layer, rows)
    dt = (time.perf_counter() - t0) / args.steps
    cores, blas = cpu_threads()
    value = sample / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "step": args.step, "tokens_per_step": sample,
                       "sample": f"{sample} tokens of the 64x2048 batch through the whole {args.step} step "
                                 "(full-width layer, dense fp64 Hadamard, int64 GEMM)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "blas_threads": blas,
                             "kind": "oracle", "sample": f"{sample} tokens per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- ours

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tokens", type=int, default=64 * 2048, help="tokens per GPU per step")
    ap.add_argument("--ref-tokens", type=int, default=2, help="oracle sample tokens per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--profile-steps", type=int, default=0, help="run N untimed steps and exit (ncu)")
    ap.add_argument("--step", default="chain", choices=["chain", "linears"],
                    help="chain: the decoder-layer chain (a1-a8, 9 launches); linears: a1-a7 on independent inputs")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    import paper_2404_00456_b200 as q
    from paper_2404_00456_b200 import dist as qd
    from paper_2404_00456_b200.runtime import DecoderLayerStep, HostPipeline, PrefillStep
    q.lib()
    layer = make_layer(dev)
    T = args.tokens
    inputs = make_inputs(T, dev, rank, args.step)
    step = DecoderLayerStep(layer, T, dev) if args.step == "chain" else PrefillStep(layer, T, dev)
    stream = torch.cuda.current_stream()
    if args.profile_steps:
        for _ in range(args.profile_steps):
            step.run_device(inputs, stream)
        torch.cuda.synchronize()
        return 0

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step.run_device(inputs, stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    per_kernel = {}
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        all_events = []
        t_start.record(stream)
        for _ in range(args.steps):
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            evs = [("start", ev0)]
            step.run_device(inputs, stream, events=evs)
            all_events.append(evs)
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = t_start.elapsed_time(t_end) / args.steps
    for evs in all_events:
        for (_, a), (name, b) in zip(evs[:-1], evs[1:]):
            per_kernel.setdefault(name, []).append(a.elapsed_time(b))
    kern_ms = {k: sum(v) / len(v) for k, v in per_kernel.items()}
    ms = qd.max_over_ranks(ms, dev)  # max over ranks (no-op at N = 1)
    clocks = clk.summary()

    # ---- roofline of the dominant kernel (the INT4 GEMM) and the HBM-bound kernels
    peaks = _peaks()
    int8_peak = 2.0 * peaks["bf16_sustained"]  # dense INT8 = 2 x bf16 (nominal 4.5 vs 2.25 POPS)
    gemm_ms = sum(v for k, v in kern_ms.items() if k.startswith("gemm_"))
    hq_ms = sum(v for k, v in kern_ms.items() if k.startswith("hq_"))
    gemm_tops = layer.gemm_ops(T) / (gemm_ms * 1e-3) / 1e12
    hq_gbs = layer.hq_bytes(T) / (hq_ms * 1e-3) / 1e9
    kv_gbs = layer.kv_bytes(T) / (kern_ms["kv_quant"] * 1e-3) / 1e9
    glue_bytes = {"rope": T * (layer.n_heads + layer.n_kv) * layer.head_dim * 4, "swiglu": T * layer.ffn * 6}
    if args.step == "chain" and step.fuse_swiglu:  # the gate/up GEMM writes act (F wide), not gate|up
        kernels_note = "gate/up GEMM epilogue computes SwiGLU (writes act)"
    traffic = load_traffic()
    kernels = {}
    for s in layer.specs:
        kernels[f"gemm_{s.name}"] = {"ms": kern_ms[f"gemm_{s.name}"], "tops": 2 * T * s.n * s.k / (kern_ms[f"gemm_{s.name}"] * 1e-3) / 1e12}
        kernels[f"hq_{s.name}"] = {"ms": kern_ms[f"hq_{s.name}"], "mode": s.mode,
                                   "gbs": T * (2.5 * s.k + 4) / (kern_ms[f"hq_{s.name}"] * 1e-3) / 1e9}
        kernels[f"hq_{s.name}"]["frac_hbm"] = kernels[f"hq_{s.name}"]["gbs"] / peaks["hbm_gbs"]
        kernels[f"gemm_{s.name}"]["frac_int8"] = kernels[f"gemm_{s.name}"]["tops"] / int8_peak
    kernels["kv_quant"] = {"ms": kern_ms["kv_quant"], "gbs": kv_gbs, "frac_hbm": kv_gbs / peaks["hbm_gbs"]}
    for gname, gb in glue_bytes.items():
        if gname in kern_ms:
            g_gbs = gb / (kern_ms[gname] * 1e-3) / 1e9
            kernels[gname] = {"ms": kern_ms[gname], "gbs": g_gbs, "frac_hbm": g_gbs / peaks["hbm_gbs"]}

    tokens_total = T * world
    line = {
        "metric": METRIC, "value": qd.aggregate_throughput(T, ms, world), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int4xint4->int32 (fp16 io, fp32 transform)",
        "data": "synthetic (seeded; random INT4 weight codes, Llama-2-70B shapes)",
        "config": {"workload": WORKLOAD, "step": args.step, "tokens_per_gpu": T, "global_batch": 64 * world,
                   "seq_len": 2048,
                   "hidden": layer.hidden, "ffn": layer.ffn, "heads": [layer.n_heads, layer.n_kv, layer.head_dim],
                   "parallelism": f"token-shard x{world} (no data-path collective)",
                   "l2": "inputs larger than L2 (GB-scale activations per step)",
                   "attention_core": "excluded (SURVEY §8 a8): the out_proj input is a synthetic activation"},
        "roofline": {"bound": "tensor", "kernel": "int4_gemm (tcgen05 kind::i8, 4 launches/step)",
                     "achieved": gemm_tops, "peak": int8_peak, "unit": "TFLOP/s",
                     "frac": gemm_tops / int8_peak,
                     "frac_vs_burst_peak": gemm_tops / (2.0 * peaks["bf16_burst"]),
                     "peak_note": f"dense INT8 = 2 x bf16_tflops_sustained ({peaks['source']}); the kernel is "
                                  "timed inside a ~90 ms step. ncu tensor-pipe active % (clock-independent) is "
                                  "in profiles/",
                     "traffic": traffic.get("int4_gemm")},
        "roofline_hbm": {"bound": "hbm", "kernel": "hadamard_quant (4 launches/step)", "achieved": hq_gbs,
                         "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": hq_gbs / peaks["hbm_gbs"],
                         "traffic": traffic.get("hadamard_quant")},
        "kernels": kernels,
        "gpu_launches": step.LAUNCHES * args.steps,
        "clocks": clocks,
    }

    # ---- end to end through the public API with pinned host buffers
    if not args.no_e2e:
        try:
            host_in = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in inputs.items()}
            for k in inputs:
                host_in[k].copy_(inputs[k])
            pipe = HostPipeline(step, host_in, chunks=8)
            pipe.run()
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.e2e_steps):
                pipe.run()
            e1.record()
            torch.cuda.synchronize()
            e_ms = e0.elapsed_time(e1) / args.e2e_steps
            e_ms = qd.max_over_ranks(e_ms, dev)
            line["e2e"] = {"value": qd.aggregate_throughput(T, e_ms, world), "unit": UNIT,
                           "h2d_bytes_per_step": pipe.h2d_bytes(), "d2h_bytes_per_step": pipe.d2h_bytes(),
                           "ms_per_step": e_ms, "chunks": 8, "steps": args.e2e_steps}
            del pipe, host_in
        except Exception as exc:  # noqa: BLE001
            line["e2e"] = {"value": None, "unit": UNIT, "error": repr(exc)[:200]}

    # ---- CPU oracle baseline (rank 0, N == 1 only)
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        sample = args.ref_tokens
        host_in, host_w, rows = host_sample(inputs, layer, sample)
        t0 = time.perf_counter()
        run_oracle(args, host_in, host_w, layer, rows)
        dt = time.perf_counter() - t0
        cores, blas = cpu_threads()
        line["cpu_baseline"] = {"value": sample / dt, "unit": UNIT, "cores": cores, "blas_threads": blas,
                                "kind": "oracle",
                                "sample": f"{sample} tokens (evenly spaced rows of the batch) through the whole "
                                          f"{args.step} step, {dt:.1f} s"}
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
