"""Prefill executor for one QuaRot-quantized Llama decoder layer's hot path.

One `step` = every row of SURVEY §8(a) over one batch of tokens, as the paper's per-layer
prefill uses them (Fig. ffn_quarot, Fig. attn_quarot, App. P:858-860):

  1. quantize(x_attn)                      NONE   -> INT4 QKV GEMM (+dequant) -> qkv fp16
  2. KV-cache Init on the qkv output views: per-head H on K (and Q, in place), asym INT4 K/V
  3. Hadamard-heads + quantize(attn_out)   HEADS  -> INT4 O GEMM   -> o fp16
  4. quantize(x_ffn)                       NONE   -> INT4 gate/up GEMM -> gate_up fp16
  5. Hadamard + quantize(ffn_act)          FULL   -> INT4 down GEMM -> down fp16

= 9 kernel launches through the C ABI (`PrefillStep`, rows a1-a7 with independent synthetic
inputs per linear).  `DecoderLayerStep` adds the a8 glue and chains the linears into a real
decoder layer (attention core excluded): 9 launches with every fusion on, the bench default.

`run_device` enqueues a step on one stream with inputs resident in HBM.  `run_host` is
the end-to-end path for callers whose activations live in (pinned) host memory: the
batch is split into token chunks and H2D copy, compute and D2H copy run on three streams
so transfers overlap the kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import quarot as q


@dataclass
class LinearSpec:
    name: str
    k: int
    n: int
    mode: str


class QuaRotLayer:
    """Packed INT4 weights + per-channel scales of one decoder layer's four linears."""

    def __init__(self, hidden: int, ffn: int, n_heads: int, n_kv_heads: int, head_dim: int,
                 weights: dict, clip_act: float = 0.9, clip_kv: float = 0.95):
        self.hidden, self.ffn = hidden, ffn
        self.n_heads, self.n_kv, self.head_dim = n_heads, n_kv_heads, head_dim
        self.qkv_out = (n_heads + 2 * n_kv_heads) * head_dim
        self.specs = [LinearSpec("qkv", hidden, self.qkv_out, "none"),
                      LinearSpec("o", hidden, hidden, "across_heads"),
                      LinearSpec("gate_up", hidden, 2 * ffn, "none"),
                      LinearSpec("down", ffn, hidden, "full")]
        for s in self.specs:
            wq, ws = weights[s.name]
            if tuple(wq.shape) != (s.n, s.k // 2) or tuple(ws.shape) != (s.n,):
                raise ValueError(f"weight {s.name}: expected [{s.n}, {s.k // 2}] / [{s.n}]")
        self.weights = weights
        self.clip_act, self.clip_kv = clip_act, clip_kv

    def gemm_ops(self, tokens: int) -> int:
        return sum(2 * tokens * s.n * s.k for s in self.specs)

    def hq_bytes(self, tokens: int) -> int:
        # fp16 read + packed INT4 write + fp32 scale per token (algorithmic)
        return sum(tokens * (2 * s.k + s.k // 2 + 4) for s in self.specs)

    def kv_bytes(self, tokens: int) -> int:
        d = self.head_dim
        kv = 2 * tokens * self.n_kv * (2 * d + d // 2 + 5)   # read fp16, write codes + scale + zero
        qrot = tokens * self.n_heads * d * 4                 # read + write fp16 Q
        return kv + qrot


class PrefillStep:
    """Workspaces for `tokens` rows and the 9-launch step (see module docstring)."""

    LAUNCHES = 9

    def __init__(self, layer: QuaRotLayer, tokens: int, device="cuda"):
        self.layer, self.tokens, self.device = layer, tokens, torch.device(device)
        L = layer
        max_k = max(s.k for s in L.specs)
        self.xq = torch.empty(tokens, max_k // 2, dtype=torch.uint8, device=device)
        self.xs = torch.empty(tokens, dtype=torch.float32, device=device)
        self.out = {s.name: torch.empty(tokens, s.n, dtype=torch.float16, device=device) for s in L.specs}
        d = L.head_dim
        self.kv = {
            "k_codes": torch.empty(tokens, L.n_kv, d // 2, dtype=torch.uint8, device=device),
            "k_scale": torch.empty(tokens, L.n_kv, dtype=torch.float32, device=device),
            "k_zero": torch.empty(tokens, L.n_kv, dtype=torch.uint8, device=device),
            "v_codes": torch.empty(tokens, L.n_kv, d // 2, dtype=torch.uint8, device=device),
            "v_scale": torch.empty(tokens, L.n_kv, dtype=torch.float32, device=device),
            "v_zero": torch.empty(tokens, L.n_kv, dtype=torch.uint8, device=device),
        }

    def _linear(self, spec: LinearSpec, x: torch.Tensor, r0: int, r1: int, stream, events, tag):
        L = self.layer
        xq = self.xq[r0:r1, : spec.k // 2]
        xs = self.xs[r0:r1]
        q.hadamard_quant(x, spec.mode, L.head_dim, L.clip_act, q=xq, scale=xs, stream=stream)
        if events is not None:
            events.append((f"hq_{spec.name}", torch.cuda.Event(enable_timing=True)))
            events[-1][1].record(stream)
        wq, ws = L.weights[spec.name]
        q.int4_linear(xq, xs, wq, ws, y=self.out[spec.name][r0:r1], stream=stream)
        if events is not None:
            events.append((f"gemm_{spec.name}", torch.cuda.Event(enable_timing=True)))
            events[-1][1].record(stream)

    def run_rows(self, inputs: dict, r0: int, r1: int, stream=None, events=None):
        """Enqueue the step for token rows [r0, r1) of `inputs` (device fp16 tensors
        'attn_in' [T, hidden], 'attn_out' [T, hidden], 'ffn_in' [T, hidden],
        'ffn_act' [T, ffn]); outputs land in self.out / self.kv rows [r0, r1)."""
        L = self.layer
        stream = torch.cuda.current_stream() if stream is None else stream
        qkv, o, gu, down = L.specs
        self._linear(qkv, inputs["attn_in"][r0:r1], r0, r1, stream, events, "qkv")
        y = self.out["qkv"][r0:r1]
        T, d = r1 - r0, L.head_dim
        nq, nkv = L.n_heads * d, L.n_kv * d
        qv = y[:, :nq].view(T, L.n_heads, d)
        kv_ = y[:, nq:nq + nkv].view(T, L.n_kv, d)
        vv = y[:, nq + nkv:].view(T, L.n_kv, d)
        q.kv_quant(kv_, vv, qv, flags=q.KV_ROTATE_K, clip_ratio=L.clip_kv,
                   out={k: t[r0:r1] for k, t in self.kv.items()}, stream=stream)
        if events is not None:
            events.append(("kv_quant", torch.cuda.Event(enable_timing=True)))
            events[-1][1].record(stream)
        self._linear(o, inputs["attn_out"][r0:r1], r0, r1, stream, events, "o")
        self._linear(gu, inputs["ffn_in"][r0:r1], r0, r1, stream, events, "gate_up")
        self._linear(down, inputs["ffn_act"][r0:r1], r0, r1, stream, events, "down")

    def run_device(self, inputs: dict, stream=None, events=None):
        self.run_rows(inputs, 0, self.tokens, stream, events)

    INPUTS = ("attn_in", "attn_out", "ffn_in", "ffn_act")

    def result_tensors(self) -> dict:
        return {"down": self.out["down"], **self.kv}


class HostPipeline:
    """End-to-end step from pinned host inputs to pinned host results, chunked over tokens
    so H2D (stream 1), the kernels (stream 2) and D2H (stream 3) overlap.  Results copied
    back per step: the step's `result_tensors()` (layer output and quantized KV cache)."""

    def __init__(self, step, host_inputs: dict, chunks: int = 8):
        self.step, self.host_in, self.chunks = step, host_inputs, chunks
        dev = step.device
        self.dev_in = {k: torch.empty(v.shape, dtype=v.dtype, device=dev) for k, v in host_inputs.items()}
        self.results = step.result_tensors()
        self.host_out = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for k, t in self.results.items()}
        self.s_h2d, self.s_cmp, self.s_d2h = (torch.cuda.Stream(dev) for _ in range(3))

    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.host_in.values())

    def d2h_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.host_out.values())

    def run(self):
        T = self.step.tokens
        bounds = [T * c // self.chunks for c in range(self.chunks + 1)]
        for c in range(self.chunks):
            r0, r1 = bounds[c], bounds[c + 1]
            with torch.cuda.stream(self.s_h2d):
                for k, h in self.host_in.items():
                    self.dev_in[k][r0:r1].copy_(h[r0:r1], non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(self.s_h2d)
            self.s_cmp.wait_event(e_in)
            self.step.run_rows(self.dev_in, r0, r1, stream=self.s_cmp)
            e_cmp = torch.cuda.Event()
            e_cmp.record(self.s_cmp)
            self.s_d2h.wait_event(e_cmp)
            with torch.cuda.stream(self.s_d2h):
                for k, t in self.results.items():
                    self.host_out[k][r0:r1].copy_(t[r0:r1], non_blocking=True)
        cur = torch.cuda.current_stream()
        cur.wait_stream(self.s_d2h)


class DecoderLayerStep:
    """The QuaRot decoder-layer prefill chain (BASELINE config 5) with the
    attention core excluded — the out_proj input is a supplied activation:

      1. RMSNorm + quantize(x)            (fused)         -> QKV GEMM          -> qkv
      2+3. RoPE on K and Q, per-head H on K (and Q, in place), asym INT4 K/V — one pass
         (quarot_kv_quant_rope; fuse_rope=False: quarot_rope in place, then quarot_kv_quant)
      4. Hadamard-heads + quantize(attn_out)              -> O GEMM + x        -> o
      5. RMSNorm + quantize(o)            (fused)         -> gate/up GEMM with SwiGLU fused
                                                             in its epilogue   -> act
      6. Hadamard (FULL) + quantize(act)                  -> down GEMM + o     -> out
    = 9 kernel launches (+1 with fuse_rope=False, +1 with fuse_swiglu=False: gate/up GEMM ->
    gu, then SwiGLU)."""

    def __init__(self, layer: QuaRotLayer, tokens: int, device="cuda", seq_len: int = 2048, theta: float = 10000.0,
                 fuse_swiglu: bool = True, fuse_rope: bool = True, row_offset: int = 0, kperm: bool | None = None):
        """tokens: rows this step processes; row_offset: their first row in the global batch (a
        token shard of a multi-GPU job, dist.shard_bounds): RoPE positions are
        (row_offset + t) % seq_len, so a sharded run equals the unsharded one bit for bit.
        kperm (default: on where supported, FFN = 1024 x 28): the down_proj input is quantized in
        the FULL kernel's native K order (quarot.h QUAROT_HAD_KPERM) against down_proj weights whose
        columns were permuted the same way offline — bit-identical outputs, faster stores."""
        self.layer, self.tokens, self.device = layer, tokens, torch.device(device)
        self.seq_len, self.theta, self.row_offset = seq_len, theta, row_offset
        self.fuse_swiglu, self.fuse_rope = fuse_swiglu, fuse_rope
        self.kperm = (layer.ffn == 28672) if kperm is None else kperm
        if self.kperm:  # offline: W_down columns in the native K order of the FULL quantizer
            wq, ws = layer.weights["down"]
            self.down_kperm = (q.permute_k_packed(wq, q.full_kperm(layer.ffn)), ws)
        self.LAUNCHES = 9 + (not fuse_swiglu) + (not fuse_rope)
        if fuse_swiglu:  # offline: gate/up rows interleaved in blocks of 8 for the fused epilogue
            self.gate_up_il = q.interleave_gate_up(*layer.weights["gate_up"])
        L = layer
        max_k = max(s.k for s in L.specs)
        self.xq = torch.empty(tokens, max_k // 2, dtype=torch.uint8, device=device)
        self.xs = torch.empty(tokens, dtype=torch.float32, device=device)
        self.qkv = torch.empty(tokens, L.qkv_out, dtype=torch.float16, device=device)
        self.o = torch.empty(tokens, L.hidden, dtype=torch.float16, device=device)
        self.gu = None if fuse_swiglu else torch.empty(tokens, 2 * L.ffn, dtype=torch.float16, device=device)
        self.act = torch.empty(tokens, L.ffn, dtype=torch.float16, device=device)
        self.out = torch.empty(tokens, L.hidden, dtype=torch.float16, device=device)
        d = L.head_dim
        self.kv = {
            "k_codes": torch.empty(tokens, L.n_kv, d // 2, dtype=torch.uint8, device=device),
            "k_scale": torch.empty(tokens, L.n_kv, dtype=torch.float32, device=device),
            "k_zero": torch.empty(tokens, L.n_kv, dtype=torch.uint8, device=device),
            "v_codes": torch.empty(tokens, L.n_kv, d // 2, dtype=torch.uint8, device=device),
            "v_scale": torch.empty(tokens, L.n_kv, dtype=torch.float32, device=device),
            "v_zero": torch.empty(tokens, L.n_kv, dtype=torch.uint8, device=device),
        }
        with torch.cuda.device(self.device):
            q.prepare()  # one-time constant uploads now, not inside a timed region or a graph capture

    INPUTS = ("x", "attn_out")

    def result_tensors(self) -> dict:
        """Per-step results a host caller keeps: the layer output and the quantized KV cache."""
        return {"out": self.out, **self.kv}

    def run_rows(self, inputs: dict, r0: int, r1: int, stream=None, events=None):
        """inputs: 'x' residual stream [T, hidden] fp16, 'attn_out' [T, hidden] fp16 stand-in for
        the attention core's output.  Rows [r0, r1); positions (row_offset + r0 + t) % seq_len."""
        x, attn_out = inputs["x"], inputs["attn_out"]
        L = self.layer
        stream = torch.cuda.current_stream() if stream is None else stream
        d = L.head_dim
        T = r1 - r0

        def mark(name):
            if events is not None:
                events.append((name, torch.cuda.Event(enable_timing=True)))
                events[-1][1].record(stream)

        def linear(spec, xin, rms, out, residual=None):
            xq = self.xq[r0:r1, : spec.k // 2]
            xs = self.xs[r0:r1]
            kp = self.kperm and spec.name == "down"
            q.hadamard_quant(xin, spec.mode, d, L.clip_act, q=xq, scale=xs, stream=stream, rmsnorm=rms, kperm=kp)
            mark(f"hq_{spec.name}")
            wq, ws = self.down_kperm if kp else L.weights[spec.name]
            q.int4_linear(xq, xs, wq, ws, y=out, stream=stream, residual=residual)
            mark(f"gemm_{spec.name}")

        qkv_s, o_s, gu_s, down_s = L.specs
        xr = x[r0:r1]
        qkv = self.qkv[r0:r1]
        linear(qkv_s, xr, True, qkv)
        nq, nkv = L.n_heads * d, L.n_kv * d
        if not self.fuse_rope:
            q.rope(qkv[:, : nq + nkv].view(T, L.n_heads + L.n_kv, d), pos0=self.row_offset + r0, seq_len=self.seq_len,
                   theta=self.theta, stream=stream)
            mark("rope")
        q.kv_quant(qkv[:, nq:nq + nkv].view(T, L.n_kv, d), qkv[:, nq + nkv:].view(T, L.n_kv, d),
                   qkv[:, :nq].view(T, L.n_heads, d), flags=q.KV_ROTATE_K, clip_ratio=L.clip_kv,
                   out={k: t[r0:r1] for k, t in self.kv.items()}, stream=stream,
                   rope=(self.row_offset + r0, self.seq_len, self.theta) if self.fuse_rope else None)
        mark("kv_quant")
        o = self.o[r0:r1]
        linear(o_s, attn_out[r0:r1], False, o, residual=xr)
        act = self.act[r0:r1]
        if self.fuse_swiglu:
            xq = self.xq[r0:r1, : gu_s.k // 2]
            xs = self.xs[r0:r1]
            q.hadamard_quant(o, "none", d, L.clip_act, q=xq, scale=xs, stream=stream, rmsnorm=True)
            mark("hq_gate_up")
            q.int4_linear_swiglu(xq, xs, *self.gate_up_il, act=act, stream=stream)
            mark("gemm_gate_up")
        else:
            gu = self.gu[r0:r1]
            linear(gu_s, o, True, gu)
            q.swiglu(gu, act=act, stream=stream)
            mark("swiglu")
        linear(down_s, act, False, self.out[r0:r1], residual=o)

    def run_device(self, inputs: dict, stream=None, events=None):
        self.run_rows(inputs, 0, self.tokens, stream, events)
