"""Seeded synthetic input generators shared by the oracle-side tests and the CUDA-path
bench.  This module holds NONE of the method's arithmetic (no Hadamard transform, no
quantization, no GEMM): only random draws with the shapes and value structure of the
paper's workloads (DESIGN.md §4 "Input recipe").

Every generator takes an explicit integer seed and a torch device; large tensors are
drawn on the GPU with ``torch.Generator(device)`` and sampled rows are copied to the
host bit-exactly for the oracle."""

from .inputs import (  # noqa: F401
    CONFIGS,
    LayerShapes,
    activations,
    kv_inputs,
    packed_weight_codes,
    weight_scales,
    dense_weight,
)
