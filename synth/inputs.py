"""Seeded input generators (no method arithmetic).  See synth/__init__.py."""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class LayerShapes:
    """Llama-2 decoder-layer linear shapes (nn.Linear [out, in] orientation)."""
    name: str
    hidden: int
    ffn: int
    n_heads: int
    n_kv_heads: int
    head_dim: int = 128

    @property
    def qkv_out(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def linears(self):
        """(name, K, N, online mode) for the four quantized linears of one layer
        ("1 1/2 Hadamard transforms per layer")."""
        return (
            ("qkv", self.hidden, self.qkv_out, "none"),
            ("o", self.hidden, self.hidden, "across_heads"),
            ("gate_up", self.hidden, 2 * self.ffn, "none"),
            ("down", self.ffn, self.hidden, "full"),
        )


LLAMA2_7B = LayerShapes("llama2-7b", 4096, 11008, 32, 32)
LLAMA2_70B = LayerShapes("llama2-70b", 8192, 28672, 64, 8)

# BASELINE.json configs (index = position in the list)
CONFIGS = {
    0: dict(name="tiny-16x256", tokens=16, k=256, n=256),
    1: dict(name="llama2-7b-8x2048", shapes=LLAMA2_7B, tokens=8 * 2048),
    2: dict(name="llama2-70b-64x2048", shapes=LLAMA2_70B, tokens=64 * 2048),
    3: dict(name="llama2-70b-kv-64x2048", shapes=LLAMA2_70B, tokens=64 * 2048),
    4: dict(name="llama2-70b-layer-chain", shapes=LLAMA2_70B, tokens=64 * 2048),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def activations(m: int, k: int, kind: str, seed: int, device="cpu",
                n_outliers: int = 8, outlier_gain: float = 50.0) -> torch.Tensor:
    """fp16 [m, k] activation rows with the structure of the paper's linear inputs.

    kind:
      "normal"     N(0,1)                                   (out_proj input)
      "outlier"    N(0,1) with `n_outliers` channels x gain (QKV / gate-up input:
                   massive channels as in Fig. activation_dist)
      "swiglu"     silu(g) * u, g, u ~ N(0,1)               (down_proj input)
    """
    g = _gen(seed, device)
    if kind == "normal":
        x = torch.randn(m, k, generator=g, device=device, dtype=torch.float32)
    elif kind == "outlier":
        x = torch.randn(m, k, generator=g, device=device, dtype=torch.float32)
        ch = torch.randperm(k, generator=g, device=device)[:n_outliers]
        x[:, ch] *= outlier_gain
    elif kind == "swiglu":
        a = torch.randn(m, k, generator=g, device=device, dtype=torch.float32)
        b = torch.randn(m, k, generator=g, device=device, dtype=torch.float32)
        x = torch.nn.functional.silu(a) * b
    else:
        raise ValueError(f"unknown activation kind {kind!r}")
    return x.to(torch.float16)


# Two's-complement nibble for a code c in [-7, 7] (the storage format D2; not arithmetic
# of the method).  Index = c + 7.
_NIBBLE = torch.tensor([(c & 0xF) for c in range(-7, 8)], dtype=torch.uint8)


def packed_weight_codes(n: int, k: int, seed: int, device="cpu") -> torch.Tensor:
    """uint8 [n, k/2]: random INT4 weight codes in [-7, 7], two per byte, low nibble =
    even k.  Each code ~ Binomial(14, 1/2) - 7 (bell-shaped like RTN codes of a
    Gaussian, std 1.87), drawn i.i.d."""
    if k % 2:
        raise ValueError("k must be even")
    g = _gen(seed, device)
    probs = torch.full((n, k), 0.5, device=device)
    idx = torch.zeros(n, k, dtype=torch.int64, device=device)
    for _ in range(14):
        idx += torch.bernoulli(probs, generator=g).to(torch.int64)
    nib = _NIBBLE.to(device)[idx]
    return (nib[:, 0::2] | (nib[:, 1::2] << 4)).contiguous()


def weight_scales(n: int, seed: int, device="cpu") -> torch.Tensor:
    """fp32 [n] positive per-channel scales ~ U(0.5, 1.5) * 0.02."""
    g = _gen(seed, device)
    return (torch.rand(n, generator=g, device=device) + 0.5) * 0.02


def dense_weight(n: int, k: int, seed: int, device="cpu") -> torch.Tensor:
    """fp32 [n, k] ~ N(0, 1/k) full-precision weight (tiny config; the oracle rotates
    and RTN-quantizes it offline)."""
    g = _gen(seed, device)
    return torch.randn(n, k, generator=g, device=device) / (k ** 0.5)


def kv_inputs(t: int, n_kv: int, n_q: int, head_dim: int, seed: int, device="cpu",
              n_outliers: int = 2, outlier_gain: float = 20.0):
    """fp16 K, V [t, n_kv, head_dim] ~ N(0,1) with `n_outliers` planted channels x gain
    per head in K (keys carry outliers); Q [t, n_q, head_dim] ~ N(0,1)."""
    g = _gen(seed, device)
    k = torch.randn(t, n_kv, head_dim, generator=g, device=device)
    v = torch.randn(t, n_kv, head_dim, generator=g, device=device)
    for h in range(n_kv):
        ch = torch.randperm(head_dim, generator=g, device=device)[:n_outliers]
        k[:, h, ch] *= outlier_gain
    q = torch.randn(t, n_q, head_dim, generator=g, device=device) if n_q else None
    return (k.to(torch.float16), v.to(torch.float16),
            None if q is None else q.to(torch.float16))
