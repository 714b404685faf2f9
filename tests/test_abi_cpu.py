"""C-ABI library checks that need no GPU: it loads, exports every symbol include/quarot.h
declares, validates arguments before touching CUDA, and its independently built Hadamard
tables agree with the oracle's."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import hadamard as had

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "quarot.h")


@pytest.fixture(scope="module")
def q():
    from paper_2404_00456_b200 import build
    build.build()
    from paper_2404_00456_b200 import quarot
    quarot.lib()
    return quarot


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(quarot_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    syms = declared_symbols()
    for name in ("quarot_hadamard_quant", "quarot_int4_linear", "quarot_kv_quant"):
        assert name in syms


def test_library_exports_every_declared_symbol(q):
    lib = ctypes.CDLL(q.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in quarot.h but not exported"
    assert set(declared_symbols()) == set(q.EXPORTS)


def test_abi_version_and_status_strings(q):
    assert q.abi_version() == 2
    for s in range(7):
        assert q.lib().quarot_status_string(s)


@pytest.mark.parametrize("m", [20, 28, 108, 172])
def test_library_tables_match_oracle(m):
    # two independent constructions of the same instance (reading Z3) must agree exactly
    from paper_2404_00456_b200 import quarot
    got = quarot.base_hadamard(m).numpy().astype(np.int64)
    assert np.array_equal(got, had.base_matrix(m))


def test_unsupported_base_size(q):
    with pytest.raises(q.QuarotError):
        q.base_hadamard(12)


def _hq(q, x=16, M=4, K=256, ld_x=256, mode=0, hd=128, clip=0.9, qp=32, ld_q=128, sp=48):
    return q.lib().quarot_hadamard_quant(x, M, K, ld_x, mode, hd, clip, qp, ld_q, sp, None)


def test_hadamard_quant_validation_without_gpu(q):
    # All of these are rejected before any CUDA call (dummy non-null pointers are fine).
    assert _hq(q, mode=3) == 5 and _hq(q, mode=-1) == 5              # ERR_ARG
    assert _hq(q, clip=0.0) == 5 and _hq(q, clip=1.5) == 5 and _hq(q, clip=float("nan")) == 5
    assert _hq(q, K=255) == 2 and _hq(q, ld_x=100) == 2 and _hq(q, ld_q=64) == 2  # ERR_DIM
    assert _hq(q, M=-1) == 2
    assert _hq(q, M=0) == 0                                            # no-op
    assert _hq(q, x=None) == 1 and _hq(q, qp=None) == 1 and _hq(q, sp=None) == 1  # ERR_NULL
    assert _hq(q, x=16 * 7 + 2) == 4                                   # misaligned pointer
    assert _hq(q, mode=1, K=12 * 16, ld_x=12 * 16, ld_q=96) == 3       # 192 = 2^4 * 12: no H_12
    assert _hq(q, mode=2, K=256, hd=48, ld_q=128) == 2                 # K % head_dim
    assert _hq(q, mode=2, K=384, ld_x=384, hd=128, ld_q=192) == 3      # 3 heads: not 2^n
    assert _hq(q, mode=2, K=256, hd=32) == 3                           # head_dim < 64


def _hqg(q, x=16, M=4, K=256, ld_x=256, group=128, clip=0.9, qp=32, ld_q=128, sp=48, ld_s=2, mode=0, hd=128):
    return q.lib().quarot_hadamard_quant_group(x, M, K, ld_x, mode, hd, group, clip, qp, ld_q, sp, ld_s, None)


def test_hadamard_quant_group_validation_without_gpu(q):
    # quarot_hadamard_quant_group (§8 f3): every rejection happens before any CUDA call
    assert _hqg(q, group=100) == 3 and _hqg(q, group=32) == 3           # ERR_UNSUPPORTED_SIZE
    assert _hqg(q, K=192, ld_x=192, ld_q=96, group=128) == 2            # K % group
    assert _hqg(q, ld_s=1) == 2 and _hqg(q, ld_x=100) == 2 and _hqg(q, M=-1) == 2  # ERR_DIM
    assert _hqg(q, clip=0.0) == 5                                       # ERR_ARG
    assert _hqg(q, M=0) == 0                                            # no-op
    assert _hqg(q, x=None) == 1 and _hqg(q, sp=None) == 1               # ERR_NULL
    assert _hqg(q, x=16 * 7 + 2) == 4                                   # misaligned pointer
    assert _hqg(q, mode=3) == 5 and _hqg(q, mode=0x100) == 5            # bad mode / flags
    assert _hqg(q, mode=1, K=192 * 4, ld_x=768, ld_q=384, ld_s=6) == 3  # 768 = 2^6 * 12: no H_12
    assert _hqg(q, mode=1, K=65536, ld_x=65536, ld_q=32768, ld_s=512) == 3  # FULL: K <= 32768
    assert _hqg(q, mode=2, hd=96) == 2                                  # K % head_dim
    assert _hqg(q, mode=2, hd=256) == 3                                 # a single head
    assert _hqg(q, mode=1, M=0) == 0 and _hqg(q, mode=2, M=0) == 0      # no-ops


def _lin(q, M=128, K=256, N=256, ld_xq=128, ld_wq=128, ld_y=256, xp=16, wp=16, yp=16):
    return q.lib().quarot_int4_linear(xp, 16, M, K, ld_xq, wp, 16, N, ld_wq, yp, ld_y, None)


def test_gemm_validation_without_gpu(q):
    assert _lin(q, M=0) == 0
    assert _lin(q, K=192, ld_xq=96, ld_wq=96) == 4      # K % 128
    assert _lin(q, N=250, ld_y=256) == 4                # N % 8
    assert _lin(q, ld_y=100) == 2
    assert _lin(q, xp=None) == 1
    assert _lin(q, xp=8) == 4
    assert q.lib().quarot_int4_matmul_s32(16, 4, 256, 128, 16, 256, 128, 16, 258, None) == 4


def test_kv_validation_without_gpu(q):
    f = q.lib().quarot_kv_quant
    # k, ld_k, v, ld_v, T, n_kv, hd, q, ld_q, n_q, flags, clip, 6 outputs, stream
    args = [16, 1024, 16, 1024, 4, 8, 128, None, 0, 0, 1, 0.95, 16, 16, 16, 16, 16, 16, None]
    # pointers are dummies: only argument sets rejected before any CUDA call are used
    bad = list(args); bad[10] = 4
    assert f(*bad) == 5                                 # unknown flag bit
    bad = list(args); bad[11] = 0.0
    assert f(*bad) == 5
    bad = list(args); bad[6] = 96
    assert f(*bad) == 3                                 # head_dim unsupported
    bad = list(args); bad[4] = 0
    assert f(*bad) == 0                                 # T == 0: no-op
    bad = list(args); bad[0] = None
    assert f(*bad) == 1
    bad = list(args); bad[1] = 1000
    assert f(*bad) == 2                                 # ld_k < n_kv * head_dim
    bad = list(args); bad[1] = 1028
    assert f(*bad) == 4                                 # ld_k % 8


def _lg(q, xp=16, sx=16, ld_sx=2, M=4, K=256, ld_xq=128, wp=16, sw=16, ld_sw=256, N=256, ld_wq=128, group=128,
        yp=16, ld_y=256, fn="quarot_int4_linear_group"):
    return getattr(q.lib(), fn)(xp, sx, ld_sx, M, K, ld_xq, wp, sw, ld_sw, N, ld_wq, group, yp, ld_y, None)


def test_int4_linear_group_validation_without_gpu(q):
    # quarot_int4_linear_group (§8 f3, packed INT4, G = 64 / 128 / 256): rejected before any CUDA call
    assert _lg(q, group=32) == 3 and _lg(q, group=512) == 3             # ERR_UNSUPPORTED_SIZE
    assert _lg(q, K=384, ld_xq=192, ld_wq=192, ld_sx=3) == 4            # K % 256
    assert _lg(q, ld_sx=1) == 2 and _lg(q, ld_sw=100) == 2 and _lg(q, ld_y=100) == 2  # ERR_DIM
    assert _lg(q, group=64, ld_sx=3) == 2                               # K / 64 scales per row
    assert _lg(q, ld_xq=100) == 2                                       # ld_xq < K / 2
    assert _lg(q, N=260, ld_sw=260, ld_y=264) == 4                      # N % 8
    assert _lg(q, ld_sw=258) == 4                                       # ld_sw % 4
    assert _lg(q, M=0) == 0                                             # no-op
    assert _lg(q, xp=None) == 1 and _lg(q, sw=None) == 1                # ERR_NULL
    # quarot_int4_linear_group8 (int8-stored codes, G = 128 only)
    g8 = dict(fn="quarot_int4_linear_group8", ld_xq=256, ld_wq=256)
    assert _lg(q, group=64, **g8) == 3
    assert _lg(q, K=384, ld_sx=3, fn="quarot_int4_linear_group8", ld_xq=384, ld_wq=384) == 4
    assert _lg(q, M=0, **g8) == 0


def test_hadamard_quant8_validation_without_gpu(q):
    lib = q.lib()
    f = lambda mode, K, hd=128: lib.quarot_hadamard_quant8(16, 4, K, K, mode, hd, 0.9, 16, K, 16, None)
    assert f(q.FULL, 768) == 3                       # 768 = 2^6 x 12: no stored H_12
    assert f(q.FULL, 65536) == 3                     # the smem kernels take K <= 32768
    assert f(q.ACROSS_HEADS, 128) == 3               # a single head
    assert f(q.ACROSS_HEADS, 384, hd=96) == 3        # head_dim not a power of two
    assert f(q.ACROSS_HEADS, 500, hd=128) == 2       # K % head_dim
    assert f(q.FULL | q.RMSNORM, 28672) == 5         # RMSNorm only with mode NONE


# ---------------------------------------------------------------- binding marshalling

_CTYPE = {"int64_t": "c_int64", "int32_t": "c_int", "uint32_t": "c_uint", "float": "c_float"}


def declared_signatures():
    """name -> list of ctypes type names, parsed from include/quarot.h."""
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    sigs = {}
    for m in re.finditer(r"\b(?:quarot_status|int64_t|int32_t|void|const char\*)\s+(quarot_[a-z0-9_]+)\s*\(([^)]*)\)\s*;",
                         src):
        params = [p.strip() for p in m.group(2).split(",") if p.strip() and p.strip() != "void"]
        types = []
        for p in params:
            t = p.rsplit(None, 1)[0] if "*" not in p else "ptr"
            types.append("c_void_p" if t == "ptr" else _CTYPE[t.replace("const ", "").strip()])
        sigs[m.group(1)] = types
    return sigs


def test_binding_argtypes_match_header(q):
    """Every ctypes signature in quarot.py has the header's parameter count and types."""
    import ctypes as ct
    decl = declared_signatures()
    assert set(decl) == set(q.EXPORTS)
    for name, args in q._SIGS.items():
        got = [a.__name__ for a in args]
        want = decl[name]
        norm = {"c_long": "c_int64", "c_longlong": "c_int64", "c_int32": "c_int", "c_uint32": "c_uint"}
        got = [norm.get(g, g) for g in got]
        want = [norm.get(w, w) for w in want]
        assert got == want, f"{name}: binding {got} vs header {want}"
    assert ct.sizeof(ct.c_int) == 4


class _FakeLib:
    """Records calls and checks each one passes exactly the declared number of arguments
    (ctypes itself silently accepts extra trailing arguments for cdecl functions)."""

    def __init__(self, sigs):
        self.sigs, self.calls = sigs, []

    def __getattr__(self, name):
        def fn(*args):
            assert len(args) == len(self.sigs[name]), f"{name}: {len(args)} args, header has {len(self.sigs[name])}"
            self.calls.append((name, args))
            if name == "quarot_kv_decode_workspace_bytes":
                return 64
            return 0
        return fn


def test_every_wrapper_passes_declared_arity_and_stream(monkeypatch):
    """Call every Python wrapper against a fake library (CPU tensors stand in for device ones):
    each call has the header's arity and its LAST argument is the caller's stream handle."""
    import torch
    from paper_2404_00456_b200 import quarot as qq
    fake = _FakeLib(declared_signatures())
    monkeypatch.setattr(qq, "lib", lambda: fake)
    monkeypatch.setattr(qq, "_dev", lambda t, name, dtype=None: t.data_ptr())
    STREAM = 0xABC0
    u8 = lambda *s: torch.zeros(*s, dtype=torch.uint8)
    f16 = lambda *s: torch.zeros(*s, dtype=torch.float16)
    f32 = lambda *s: torch.zeros(*s, dtype=torch.float32)
    i8 = lambda *s: torch.zeros(*s, dtype=torch.int8)
    dev = torch.device("cpu")
    x = f16(4, 256)
    qq.hadamard_quant(x, "full", stream=STREAM)
    qq.hadamard_quant(x, "none", rmsnorm=True, stream=STREAM)
    xq, xs, wq, ws = u8(4, 128), f32(4), u8(16, 128), f32(16)
    qq.int4_linear(xq, xs, wq, ws, stream=STREAM)
    qq.int4_linear(xq, xs, wq, ws, residual=f16(4, 16), stream=STREAM)
    qq.int4_linear_swiglu(xq, xs, wq, ws, stream=STREAM)
    qq.int4_matmul_s32(xq, wq, stream=STREAM)
    qq.rope(f16(4, 2, 128), stream=STREAM)
    qq.swiglu(f16(4, 32), stream=STREAM)
    k, v, qh = f16(4, 2, 128), f16(4, 2, 128), f16(4, 4, 128)
    out = {n: u8(4, 2, 64) if "codes" in n else (f32(4, 2) if "scale" in n else u8(4, 2))
           for n in ("k_codes", "k_scale", "k_zero", "v_codes", "v_scale", "v_zero")}
    qq.kv_quant(k, v, qh, out=out, stream=STREAM)
    qq.kv_quant(k, v, qh, out=out, rope=(0, 2048, 1e4), stream=STREAM)
    qq.hadamard_quant_group(x, stream=STREAM)
    qq.hadamard_quant_group8(x, stream=STREAM)
    qq.int4_linear_group(u8(4, 128), f32(4, 2), u8(16, 128), f32(2, 16), stream=STREAM)
    qq.int4_linear_group8(i8(4, 256), f32(4, 2), i8(16, 256), f32(2, 16), stream=STREAM)
    qq.hadamard_quant_group(x, mode="full", stream=STREAM)
    qq.hadamard_quant8(x, mode="full", stream=STREAM)
    qq.hadamard_quant8(x, stream=STREAM)
    qq.int8_linear(i8(4, 256), f32(4), i8(16, 256), f32(16), stream=STREAM)
    qq.int8_matmul_s32(i8(4, 256), i8(16, 256), stream=STREAM)
    cache = qq.kv_cache_empty(2, 8, 2, 128, device=dev)
    pos = torch.zeros(2, dtype=torch.int32)
    monkeypatch.setattr(torch.Tensor, "device", property(lambda self: dev), raising=False)
    qq.kv_append(f16(2, 2, 128), f16(2, 2, 128), f16(2, 4, 128), pos, cache, stream=STREAM)
    qq.kv_decode(f16(2, 4, 128), cache, pos, stream=STREAM)
    launched = [c for c in fake.calls if c[0] != "quarot_kv_decode_workspace_bytes"]
    assert len(launched) >= 18
    for name, args in launched:
        assert args[-1] == STREAM, f"{name}: stream not forwarded (last arg {args[-1]!r})"


def test_full_kperm_permutation_matches_header_formula(q):
    """quarot_full_kperm (QUAROT_HAD_KPERM): a bijection, equal to the header's formula
    p(i) = (a >> 5) * 32 J + 32 j' + (a & 31) for i = a * J + j', J = K / 256."""
    K = 28672
    perm = q.full_kperm(K).numpy()
    assert np.array_equal(np.sort(perm), np.arange(K))
    J = K // 256
    i = np.arange(K)
    a, j = i // J, i % J
    p = (a >> 5) * 32 * J + 32 * j + (a & 31)
    assert np.array_equal(perm[p], i)
    with pytest.raises(q.QuarotError):
        q.full_kperm(8192)


def test_permute_k_packed_roundtrip(q):
    import torch
    rng = np.random.default_rng(0)
    K = 28672
    w = torch.from_numpy(rng.integers(0, 256, (3, K // 2), dtype=np.uint8))
    perm = q.full_kperm(K)
    wp = q.permute_k_packed(w, perm)
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(K)
    assert torch.equal(q.permute_k_packed(wp, inv), w)


def test_kperm_flag_validation_without_gpu(q):
    f = lambda mode, K, ld_q=None, qp=32: q.lib().quarot_hadamard_quant(16, 4, K, K, mode, 128, 0.9, qp,
                                                                         ld_q or K // 2, 48, None)
    assert f(q.FULL | q.KPERM, 8192) == 3                 # KPERM only at K = 1024 x 28
    assert f(q.NONE | q.KPERM, 28672) == 5                # FULL only
    assert f(q.FULL | q.KPERM, 28672, ld_q=14344) == 4    # ld_q % 16
    assert f(q.FULL | q.KPERM, 28672, qp=40) == 4         # q 16-byte aligned
