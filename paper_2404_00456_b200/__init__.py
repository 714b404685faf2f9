"""B200-native (sm_100a) QuaRot online quantized-linear hot path (arXiv 2404.00456).

The compute lives in ``libquarot.so`` (hand-written CUDA, C ABI in include/quarot.h);
``quarot`` is its thin ctypes binding.  See DESIGN.md."""

from .quarot import (  # noqa: F401
    ACROSS_HEADS, FULL, NONE, RMSNORM, KPERM, EXPORTS, LIB_PATH, QuarotError,
    abi_version, base_hadamard, hadamard_quant, int4_linear, int4_matmul_s32, kv_quant,
    last_launch_count, lib, quarot_linear, rope, swiglu, interleave_gate_up, int4_linear_swiglu,
    kv_append, kv_decode, kv_cache_empty, hadamard_quant8, int8_linear, int8_matmul_s32,
    hadamard_quant_group, hadamard_quant_group8, int4_linear_group, int4_linear_group8, full_kperm, permute_k_packed,
    prepare,
)
