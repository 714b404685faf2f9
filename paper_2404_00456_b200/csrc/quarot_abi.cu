// quarot_abi.cu — the extern "C" boundary (include/quarot.h): argument validation and
// dispatch to the sm_100a kernels.  No torch types, no allocation, no host synchronization (except
// the one-time constant uploads, quarot_prepare).
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/quarot.h"
#include "quarot_internal.h"

namespace {
// the last launch failure, for quarot_last_cuda_error() (diagnostics only)
thread_local char g_last_cuda_error[160] = "";
quarot_status cuda_fail(cudaError_t e) {
  std::snprintf(g_last_cuda_error, sizeof g_last_cuda_error, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return QUAROT_ERR_CUDA;
}

thread_local int32_t g_last_launches = 0;

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
bool clip_ok(float c) { return c > 0.f && c <= 1.f; }  // NaN fails both

// K = 2^n * m with m in {1, 20, 28, 108, 172}; smallest admissible m (largest power of two).
bool factorize(int64_t K, int64_t& p, int& m) {
  const int cands[5] = {1, 20, 28, 108, 172};
  for (int c : cands) {
    if (K % c == 0 && pow2(K / c)) {
      p = K / c;
      m = c;
      return true;
    }
  }
  return false;
}

}  // namespace

extern "C" {

const char* quarot_status_string(int32_t s) {
  switch (s) {
    case QUAROT_OK: return "ok";
    case QUAROT_ERR_NULL: return "null pointer argument";
    case QUAROT_ERR_DIM: return "dimension error (non-positive, odd, inconsistent or ld < width)";
    case QUAROT_ERR_UNSUPPORTED_SIZE:
      return "unsupported size: FULL needs K = 2^n * m with m in {1, 20, 28, 108, 172} and 2^n >= 2; "
             "ACROSS_HEADS needs K / head_dim and head_dim powers of two (head_dim >= 64); "
             "KV needs head_dim in {64, 128, 256}";
    case QUAROT_ERR_ALIGN: return "alignment error (16-byte pointers / leading dimensions, width granularity)";
    case QUAROT_ERR_ARG: return "bad argument (clip ratio outside (0, 1], unknown mode or flags)";
    case QUAROT_ERR_CUDA: return "CUDA launch error";
    default: return "unknown status";
  }
}

int32_t quarot_abi_version(void) { return QUAROT_ABI_VERSION; }
const char* quarot_last_cuda_error(void) { return g_last_cuda_error; }

int32_t quarot_last_launch_count(void) { return g_last_launches; }

quarot_status quarot_full_kperm(int64_t K, int64_t* perm) {
  if (!perm) return QUAROT_ERR_NULL;
  if (K != 28672) return QUAROT_ERR_UNSUPPORTED_SIZE;
  const int64_t J = K / 256;  // natural element i = a * J + j', a < 256
  for (int64_t a = 0; a < 256; ++a)
    for (int64_t j = 0; j < J; ++j) perm[(a >> 5) * 32 * J + 32 * j + (a & 31)] = a * J + j;
  return QUAROT_OK;
}

quarot_status quarot_prepare(void) {
  // every lazily initialised launcher, called with zero rows: one-time setup only, no launch
  cudaError_t e = qr::ensure_device_tables();
  if (e == cudaSuccess) e = qr::launch_hq_full28_tc(nullptr, 0, 0, 0.9f, nullptr, 0, nullptr, nullptr);
  if (e == cudaSuccess) e = qr::launch_hq_full172_tc(nullptr, 0, 0, 0.9f, nullptr, 0, nullptr, nullptr);
  if (e == cudaSuccess) e = qr::launch_hq_full_small_tc(nullptr, 0, 0, 128, 108, 0.9f, nullptr, 0, nullptr, nullptr);
  if (e == cudaSuccess) e = qr::launch_hq_full_small_tc(nullptr, 0, 0, 256, 20, 0.9f, nullptr, 0, nullptr, nullptr);
  for (int nh = 16; e == cudaSuccess && nh <= 64; nh *= 2)
    e = qr::launch_hq_heads_tc(nullptr, 0, (int64_t)nh * 128, 0, 128, 0.9f, nullptr, 0, nullptr, nullptr);
  if (e == cudaSuccess)
    e = qr::launch_kv_tc(nullptr, 0, nullptr, 0, 0, 8, nullptr, 0, 64, 0.95f, false, 0, 2048, 10000.f, nullptr,
                         nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e == cudaSuccess ? QUAROT_OK : cuda_fail(e);
}

quarot_status quarot_base_hadamard(int32_t m, int8_t* out) {
  if (!out) return QUAROT_ERR_NULL;
  const int8_t* h = qr::base_hadamard_host(m);
  if (!h) return QUAROT_ERR_UNSUPPORTED_SIZE;
  std::memcpy(out, h, (size_t)m * m);
  return QUAROT_OK;
}

quarot_status quarot_hadamard_quant(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode,
                                    int32_t head_dim, float clip_ratio, uint8_t* q, int64_t ld_q, float* scale,
                                    void* stream) {
  g_last_launches = 0;
  const bool rms = (mode & QUAROT_HAD_RMSNORM) != 0;
  const bool kperm = (mode & QUAROT_HAD_KPERM) != 0;
  mode &= ~(QUAROT_HAD_RMSNORM | QUAROT_HAD_KPERM);
  if (mode < QUAROT_HAD_NONE || mode > QUAROT_HAD_ACROSS_HEADS) return QUAROT_ERR_ARG;
  if (rms && mode != QUAROT_HAD_NONE) return QUAROT_ERR_ARG;
  if (kperm && mode != QUAROT_HAD_FULL) return QUAROT_ERR_ARG;
  if (!clip_ok(clip_ratio)) return QUAROT_ERR_ARG;
  if (M < 0 || K <= 0 || (K & 1) || ld_x < K || ld_q < K / 2) return QUAROT_ERR_DIM;
  if (kperm && K != 28672) return QUAROT_ERR_UNSUPPORTED_SIZE;
  if (kperm && (ld_q % 16 || (M > 0 && q && !aligned16(q)))) return QUAROT_ERR_ALIGN;
  if (M > 0x7fffffffLL) return QUAROT_ERR_DIM;
  if (M == 0) return QUAROT_OK;
  if (!x || !q || !scale) return QUAROT_ERR_NULL;
  if (!aligned16(x) || !aligned16(q) || (ld_x % 8) || (ld_q % (mode == QUAROT_HAD_ACROSS_HEADS ? 16 : 4)))
    return QUAROT_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (mode == QUAROT_HAD_NONE) {
    if (K % 16) return QUAROT_ERR_ALIGN;
    if (K > 32768) return QUAROT_ERR_UNSUPPORTED_SIZE;
    e = qr::launch_hq_none(x, M, K, ld_x, clip_ratio, q, ld_q, scale, st, rms);
  } else if (mode == QUAROT_HAD_ACROSS_HEADS) {
    if (head_dim <= 0 || K % head_dim) return QUAROT_ERR_DIM;
    if (!pow2(head_dim) || head_dim < 64 || !pow2(K / head_dim) || K / head_dim > 512)
      return QUAROT_ERR_UNSUPPORTED_SIZE;
    if (K % 32) return QUAROT_ERR_ALIGN;
    if (!qr::hq_heads_tc_supported(K, head_dim)) {
      // CUDA-core fallback limits: (head_dim / 2) x G threads <= 256 with G = max(1, n_h / 32)
      // head groups, and the row staged in shared memory (4.5 K bytes)
      const int64_t nh = K / head_dim, G = nh > 32 ? nh / 32 : 1;
      if (head_dim / 2 * G > 256 || K > 32768) return QUAROT_ERR_UNSUPPORTED_SIZE;
    }
    e = qr::launch_hq_heads(x, M, K, ld_x, head_dim, clip_ratio, q, ld_q, scale, st);
  } else {
    int64_t p = 0;
    int m = 0;
    if (!factorize(K, p, m) || p < 2 || K > 32768) return QUAROT_ERR_UNSUPPORTED_SIZE;
    if (K % 16) return QUAROT_ERR_ALIGN;
    if (m > 1) {
      if (!qr::base_hadamard_host(m)) return QUAROT_ERR_UNSUPPORTED_SIZE;
      e = qr::ensure_device_tables();
      if (e != cudaSuccess) return cuda_fail(e);
    }
    e = kperm ? qr::launch_hq_full28_tc(x, M, ld_x, clip_ratio, q, ld_q, scale, st, false, true)
              : qr::launch_hq_full(x, M, K, ld_x, (int)p, m, clip_ratio, q, ld_q, scale, st);
  }
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

static quarot_status check_gemm(const uint8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const uint8_t* wq,
                                int64_t N, int64_t ld_wq, const void* out, int64_t ld_out, int64_t out_elems_align) {
  if (M < 0 || N <= 0 || K <= 0 || ld_xq < K / 2 || ld_wq < K / 2 || ld_out < N) return QUAROT_ERR_DIM;
  if (M > 0x7fffffffLL || N > 0x7fffffffLL) return QUAROT_ERR_DIM;
  if (M == 0) return QUAROT_OK;
  if (!xq || !wq || !out) return QUAROT_ERR_NULL;
  if (K % 128 || N % 8 || ld_xq % 16 || ld_wq % 16 || ld_out % out_elems_align) return QUAROT_ERR_ALIGN;
  if (!aligned16(xq) || !aligned16(wq) || !aligned16(out)) return QUAROT_ERR_ALIGN;
  // the MMA accumulates 256 * acc with |acc| <= 7 * 8 * K (activation codes in [-7, 7], weight
  // codes in [-8, 7]): exact in int32 for K <= 149796
  if (K > 149796) return QUAROT_ERR_UNSUPPORTED_SIZE;
  return QUAROT_OK;
}

quarot_status quarot_int4_linear(const uint8_t* xq, const float* x_scale, int64_t M, int64_t K, int64_t ld_xq,
                                 const uint8_t* wq, const float* w_scale, int64_t N, int64_t ld_wq, void* y,
                                 int64_t ld_y, void* stream) {
  g_last_launches = 0;
  quarot_status s = check_gemm(xq, M, K, ld_xq, wq, N, ld_wq, y, ld_y, 8);
  if (s != QUAROT_OK || M == 0) return s;
  if (!x_scale || !w_scale) return QUAROT_ERR_NULL;
  if (!aligned16(w_scale)) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_int4_gemm(xq, x_scale, M, K, ld_xq, wq, w_scale, N, ld_wq, y, ld_y,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_int4_linear_residual(const uint8_t* xq, const float* x_scale, int64_t M, int64_t K,
                                          int64_t ld_xq, const uint8_t* wq, const float* w_scale, int64_t N,
                                          int64_t ld_wq, const void* residual, int64_t ld_r, void* y, int64_t ld_y,
                                          void* stream) {
  g_last_launches = 0;
  quarot_status s = check_gemm(xq, M, K, ld_xq, wq, N, ld_wq, y, ld_y, 8);
  if (s != QUAROT_OK || M == 0) return s;
  if (!x_scale || !w_scale || !residual) return QUAROT_ERR_NULL;
  if (ld_r < N) return QUAROT_ERR_DIM;
  if (!aligned16(w_scale) || !aligned16(residual) || (ld_r % 8)) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_int4_gemm(xq, x_scale, M, K, ld_xq, wq, w_scale, N, ld_wq, y, ld_y,
                                       static_cast<cudaStream_t>(stream), residual, ld_r);
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_int4_linear_swiglu(const uint8_t* xq, const float* x_scale, int64_t M, int64_t K,
                                        int64_t ld_xq, const uint8_t* wq, const float* w_scale, int64_t N2,
                                        int64_t ld_wq, void* act, int64_t ld_act, void* stream) {
  g_last_launches = 0;
  if (N2 <= 0 || N2 % 16) return N2 <= 0 ? QUAROT_ERR_DIM : QUAROT_ERR_ALIGN;
  if (ld_act < N2 / 2) return QUAROT_ERR_DIM;
  quarot_status s = check_gemm(xq, M, K, ld_xq, wq, N2, ld_wq, act, N2, 8);
  if (s != QUAROT_OK || M == 0) return s;
  if (!x_scale || !w_scale) return QUAROT_ERR_NULL;
  if (!aligned16(w_scale) || (ld_act % 8)) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_int4_gemm_swiglu(xq, x_scale, M, K, ld_xq, wq, w_scale, N2, ld_wq, act, ld_act,
                                              static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_rope(void* x, int64_t T, int32_t n_heads, int32_t head_dim, int64_t ld_x, int64_t pos0,
                          int32_t seq_len, float theta, void* stream) {
  g_last_launches = 0;
  if (T < 0 || n_heads <= 0 || head_dim <= 0 || seq_len <= 0 || pos0 < 0) return QUAROT_ERR_DIM;
  if (head_dim % 16 || head_dim > 256) return QUAROT_ERR_UNSUPPORTED_SIZE;
  if (ld_x < (int64_t)n_heads * head_dim) return QUAROT_ERR_DIM;
  if (!(theta > 1.f)) return QUAROT_ERR_ARG;
  if (T == 0) return QUAROT_OK;
  if (!x) return QUAROT_ERR_NULL;
  if (!aligned16(x) || (ld_x % 8)) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_rope(x, T, n_heads, head_dim, ld_x, pos0, seq_len, theta, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_swiglu(const void* gate_up, int64_t M, int64_t F, int64_t ld_gu, void* act, int64_t ld_act,
                            void* stream) {
  g_last_launches = 0;
  if (M < 0 || F <= 0 || ld_gu < 2 * F || ld_act < F) return QUAROT_ERR_DIM;
  if (M == 0) return QUAROT_OK;
  if (!gate_up || !act) return QUAROT_ERR_NULL;
  if (F % 8 || ld_gu % 8 || ld_act % 8 || !aligned16(gate_up) || !aligned16(act)) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_swiglu(gate_up, M, F, ld_gu, act, ld_act, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_int4_matmul_s32(const uint8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const uint8_t* wq,
                                     int64_t N, int64_t ld_wq, int32_t* acc, int64_t ld_acc, void* stream) {
  g_last_launches = 0;
  quarot_status s = check_gemm(xq, M, K, ld_xq, wq, N, ld_wq, acc, ld_acc, 4);
  if (s != QUAROT_OK || M == 0) return s;
  cudaError_t e =
      qr::launch_int4_gemm_s32(xq, M, K, ld_xq, wq, N, ld_wq, acc, ld_acc, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

// ---- group-wise
static quarot_status hq_group_impl(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode, int32_t head_dim,
                                   int32_t group, float clip_ratio, uint8_t* q, int64_t ld_q, float* scale,
                                   int64_t ld_s, void* stream, bool q8) {
  g_last_launches = 0;
  if (mode < QUAROT_HAD_NONE || mode > QUAROT_HAD_ACROSS_HEADS) return QUAROT_ERR_ARG;
  if (!clip_ok(clip_ratio)) return QUAROT_ERR_ARG;
  if (!(group == 64 || group == 128 || group == 256)) return QUAROT_ERR_UNSUPPORTED_SIZE;
  if (M < 0 || K <= 0 || K % 2 || ld_x < K || ld_q < (q8 ? K : K / 2) || ld_s < K / group) return QUAROT_ERR_DIM;
  if (K % group) return QUAROT_ERR_DIM;
  if (M > 0x7fffffffLL) return QUAROT_ERR_DIM;              // rows on gridDim.x
  int64_t p = 0;
  int m = 0;
  if (mode == QUAROT_HAD_NONE) {
    if (K > 0xffffLL * 1024) return QUAROT_ERR_UNSUPPORTED_SIZE;  // 1024-element blocks on gridDim.y
  } else if (mode == QUAROT_HAD_FULL) {
    // the row is transformed in shared memory: K <= 32768, K = 2^n m
    if (!factorize(K, p, m) || p < 2 || K > 32768 || (m > 1 && !qr::base_hadamard_host(m)))
      return QUAROT_ERR_UNSUPPORTED_SIZE;
  } else {
    if (head_dim <= 0 || K % head_dim) return QUAROT_ERR_DIM;
    if (!pow2(head_dim) || !pow2(K / head_dim) || K / head_dim < 2 || K > 32768) return QUAROT_ERR_UNSUPPORTED_SIZE;
  }
  if (M == 0) return QUAROT_OK;
  if (!x || !q || !scale) return QUAROT_ERR_NULL;
  if (!aligned16(x) || !aligned16(q) || (ld_x % 8) || (ld_q % (q8 ? 8 : 4)) || (mode != QUAROT_HAD_NONE && K % 16))
    return QUAROT_ERR_ALIGN;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (mode == QUAROT_HAD_NONE) {
    e = qr::launch_hq_none_group(x, M, K, ld_x, group, clip_ratio, q, ld_q, scale, ld_s, st, q8);
  } else if (mode == QUAROT_HAD_FULL) {
    e = m > 1 ? qr::ensure_device_tables() : cudaSuccess;
    if (e == cudaSuccess)
      e = qr::launch_hq_full(x, M, K, ld_x, (int)p, m, clip_ratio, q, ld_q, scale, st, q8 ? 3 : 2, group, ld_s);
  } else {
    e = qr::launch_hq_heads_group(x, M, K, ld_x, head_dim, clip_ratio, q, ld_q, scale, ld_s, group, q8, st);
  }
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_hadamard_quant_group(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode,
                                         int32_t head_dim, int32_t group, float clip_ratio, uint8_t* q, int64_t ld_q,
                                         float* scale, int64_t ld_s, void* stream) {
  return hq_group_impl(x, M, K, ld_x, mode, head_dim, group, clip_ratio, q, ld_q, scale, ld_s, stream, false);
}

quarot_status quarot_hadamard_quant_group8(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode,
                                          int32_t head_dim, int32_t group, float clip_ratio, int8_t* q, int64_t ld_q,
                                          float* scale, int64_t ld_s, void* stream) {
  return hq_group_impl(x, M, K, ld_x, mode, head_dim, group, clip_ratio, reinterpret_cast<uint8_t*>(q), ld_q, scale,
                       ld_s, stream, true);
}

quarot_status quarot_int4_linear_group(const uint8_t* xq, const float* x_scale, int64_t ld_sx, int64_t M, int64_t K,
                                       int64_t ld_xq, const uint8_t* wq, const float* w_scale_t, int64_t ld_sw,
                                       int64_t N, int64_t ld_wq, int32_t group, void* y, int64_t ld_y, void* stream) {
  g_last_launches = 0;
  if (!(group == 64 || group == 128 || group == 256)) return QUAROT_ERR_UNSUPPORTED_SIZE;
  if (M < 0 || N <= 0 || K <= 0 || ld_xq < K / 2 || ld_wq < K / 2 || ld_y < N || ld_sx < K / group || ld_sw < N)
    return QUAROT_ERR_DIM;
  if (M > 0x7fffffffLL || N > 0x7fffffffLL) return QUAROT_ERR_DIM;
  if (M == 0) return QUAROT_OK;
  if (!xq || !x_scale || !wq || !w_scale_t || !y) return QUAROT_ERR_NULL;
  if (K % 256 || N % 8 || ld_xq % 16 || ld_wq % 16 || ld_y % 8 || ld_sw % 4 || !aligned16(xq) || !aligned16(wq) ||
      !aligned16(y) || !aligned16(w_scale_t))
    return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_int4_group_gemm(xq, x_scale, ld_sx, M, K, ld_xq, wq, w_scale_t, ld_sw, N, ld_wq, group, y,
                                             ld_y, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_int4_linear_group8(const int8_t* xq, const float* x_scale, int64_t ld_sx, int64_t M, int64_t K,
                                       int64_t ld_xq, const int8_t* wq, const float* w_scale_t, int64_t ld_sw,
                                       int64_t N, int64_t ld_wq, int32_t group, void* y, int64_t ld_y, void* stream) {
  g_last_launches = 0;
  if (group != 128) return QUAROT_ERR_UNSUPPORTED_SIZE;
  if (M < 0 || N <= 0 || K <= 0 || ld_xq < K || ld_wq < K || ld_y < N || ld_sx < K / 128 || ld_sw < N)
    return QUAROT_ERR_DIM;
  if (M == 0) return QUAROT_OK;
  if (!xq || !x_scale || !wq || !w_scale_t || !y) return QUAROT_ERR_NULL;
  if (K % 256 || N % 8 || ld_xq % 16 || ld_wq % 16 || ld_y % 8 || ld_sw % 4 || !aligned16(xq) || !aligned16(wq) ||
      !aligned16(y) || !aligned16(w_scale_t))
    return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_int8_group_gemm(xq, x_scale, ld_sx, M, K, ld_xq, wq, w_scale_t, ld_sw, N, ld_wq, y, ld_y,
                                             static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_hadamard_quant8(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode,
                                     int32_t head_dim, float clip_ratio, int8_t* q, int64_t ld_q, float* scale,
                                     void* stream) {
  g_last_launches = 0;
  const bool rms = (mode & QUAROT_HAD_RMSNORM) != 0;
  mode &= ~QUAROT_HAD_RMSNORM;
  if (mode < QUAROT_HAD_NONE || mode > QUAROT_HAD_ACROSS_HEADS) return QUAROT_ERR_ARG;
  if (rms && mode != QUAROT_HAD_NONE) return QUAROT_ERR_ARG;
  if (!clip_ok(clip_ratio)) return QUAROT_ERR_ARG;
  if (M < 0 || K <= 0 || ld_x < K || ld_q < K) return QUAROT_ERR_DIM;
  if (M > 0x7fffffffLL) return QUAROT_ERR_DIM;
  int64_t p = 0;
  int m = 0;
  if (mode == QUAROT_HAD_FULL &&
      (!factorize(K, p, m) || p < 2 || K > 32768 || (m > 1 && !qr::base_hadamard_host(m))))
    return QUAROT_ERR_UNSUPPORTED_SIZE;
  if (mode == QUAROT_HAD_ACROSS_HEADS) {
    if (head_dim <= 0 || K % head_dim) return QUAROT_ERR_DIM;
    if (!pow2(head_dim) || !pow2(K / head_dim) || K / head_dim < 2) return QUAROT_ERR_UNSUPPORTED_SIZE;
  }
  if (M == 0) return QUAROT_OK;
  if (!x || !q || !scale) return QUAROT_ERR_NULL;
  if (!aligned16(x) || !aligned16(q) || (ld_x % 8) || (ld_q % 8) || (K % 16)) return QUAROT_ERR_ALIGN;
  if (K > 32768) return QUAROT_ERR_UNSUPPORTED_SIZE;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (mode == QUAROT_HAD_NONE) {
    e = qr::launch_hq_none_q8(x, M, K, ld_x, clip_ratio, q, ld_q, scale, st, rms);
  } else {
    e = qr::ensure_device_tables();
    if (e == cudaSuccess) {
      uint8_t* qb = reinterpret_cast<uint8_t*>(q);
      if (mode == QUAROT_HAD_FULL)
        e = qr::launch_hq_full(x, M, K, ld_x, (int)p, m, clip_ratio, qb, ld_q, scale, st, 1);
      else if (qr::hq_heads_tc_supported(K, head_dim) && qr::g_hq_heads_variant != 1)
        e = qr::launch_hq_heads_tc(x, M, K, ld_x, head_dim, clip_ratio, qb, ld_q, scale, st, true);
      else
        e = qr::launch_hq_heads8(x, M, K, ld_x, head_dim, clip_ratio, qb, ld_q, scale, st);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

static quarot_status check_gemm8(const int8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const int8_t* wq, int64_t N,
                                 int64_t ld_wq, const void* out, int64_t ld_out, int64_t out_elems_align) {
  if (M < 0 || N <= 0 || K <= 0 || ld_xq < K || ld_wq < K || ld_out < N) return QUAROT_ERR_DIM;
  if (M > 0x7fffffffLL || N > 0x7fffffffLL) return QUAROT_ERR_DIM;
  if (M == 0) return QUAROT_OK;
  if (!xq || !wq || !out) return QUAROT_ERR_NULL;
  if (K % 128 || N % 8 || ld_xq % 16 || ld_wq % 16 || ld_out % out_elems_align) return QUAROT_ERR_ALIGN;
  if (!aligned16(xq) || !aligned16(wq) || !aligned16(out)) return QUAROT_ERR_ALIGN;
  if (K > 131072) return QUAROT_ERR_UNSUPPORTED_SIZE;  // 127 * 127 * K must fit int32
  return QUAROT_OK;
}

quarot_status quarot_int8_linear(const int8_t* xq, const float* x_scale, int64_t M, int64_t K, int64_t ld_xq,
                                 const int8_t* wq, const float* w_scale, int64_t N, int64_t ld_wq, void* y,
                                 int64_t ld_y, void* stream) {
  g_last_launches = 0;
  quarot_status s = check_gemm8(xq, M, K, ld_xq, wq, N, ld_wq, y, ld_y, 8);
  if (s != QUAROT_OK || M == 0) return s;
  if (!x_scale || !w_scale) return QUAROT_ERR_NULL;
  if (!aligned16(w_scale)) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_int8_gemm(xq, x_scale, M, K, ld_xq, wq, w_scale, N, ld_wq, y, ld_y,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_int8_matmul_s32(const int8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const int8_t* wq,
                                     int64_t N, int64_t ld_wq, int32_t* acc, int64_t ld_acc, void* stream) {
  g_last_launches = 0;
  quarot_status s = check_gemm8(xq, M, K, ld_xq, wq, N, ld_wq, acc, ld_acc, 4);
  if (s != QUAROT_OK || M == 0) return s;
  cudaError_t e =
      qr::launch_int8_gemm_s32(xq, M, K, ld_xq, wq, N, ld_wq, acc, ld_acc, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_kv_quant(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int32_t n_kv,
                              int32_t head_dim, void* q, int64_t ld_q, int32_t n_q, uint32_t flags, float clip_ratio,
                              uint8_t* k_codes, float* k_scale, uint8_t* k_zero, uint8_t* v_codes, float* v_scale,
                              uint8_t* v_zero, void* stream) {
  g_last_launches = 0;
  if (flags & ~3u) return QUAROT_ERR_ARG;
  if (!clip_ok(clip_ratio)) return QUAROT_ERR_ARG;
  if (T < 0 || n_kv <= 0 || n_q < 0 || head_dim <= 0) return QUAROT_ERR_DIM;
  if (!(head_dim == 64 || head_dim == 128 || head_dim == 256)) return QUAROT_ERR_UNSUPPORTED_SIZE;
  const bool has_q = q != nullptr && n_q > 0;
  if (ld_k < (int64_t)n_kv * head_dim || ld_v < (int64_t)n_kv * head_dim ||
      (has_q && ld_q < (int64_t)n_q * head_dim))
    return QUAROT_ERR_DIM;
  if (T == 0) return QUAROT_OK;
  if (!k || !v || !k_codes || !k_scale || !k_zero || !v_codes || !v_scale || !v_zero) return QUAROT_ERR_NULL;
  if (!aligned16(k) || !aligned16(v) || (has_q && !aligned16(q)) || !aligned16(k_codes) || !aligned16(v_codes))
    return QUAROT_ERR_ALIGN;
  if ((ld_k % 8) || (ld_v % 8) || (has_q && (ld_q % 8))) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_kv_quant(k, ld_k, v, ld_v, T, n_kv, head_dim, has_q ? q : nullptr, ld_q,
                                      has_q ? n_q : 0, flags, clip_ratio, k_codes, k_scale, k_zero, v_codes,
                                      v_scale, v_zero, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_kv_quant_rope(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T,
                                   int32_t n_kv, int32_t head_dim, void* q, int64_t ld_q, int32_t n_q,
                                   uint32_t flags, float clip_ratio, int64_t pos0, int32_t seq_len, float theta,
                                   uint8_t* k_codes, float* k_scale, uint8_t* k_zero, uint8_t* v_codes,
                                   float* v_scale, uint8_t* v_zero, void* stream) {
  g_last_launches = 0;
  if (flags & ~3u) return QUAROT_ERR_ARG;
  if (!clip_ok(clip_ratio)) return QUAROT_ERR_ARG;
  if (seq_len < 1 || pos0 < 0 || !(theta > 0.f)) return QUAROT_ERR_ARG;
  if (T < 0 || n_kv <= 0 || n_q < 0 || head_dim <= 0) return QUAROT_ERR_DIM;
  if (!(head_dim == 64 || head_dim == 128 || head_dim == 256)) return QUAROT_ERR_UNSUPPORTED_SIZE;
  const bool has_q = q != nullptr && n_q > 0;
  if (ld_k < (int64_t)n_kv * head_dim || ld_v < (int64_t)n_kv * head_dim ||
      (has_q && ld_q < (int64_t)n_q * head_dim))
    return QUAROT_ERR_DIM;
  if (T == 0) return QUAROT_OK;
  if (!k || !v || !k_codes || !k_scale || !k_zero || !v_codes || !v_scale || !v_zero) return QUAROT_ERR_NULL;
  if (!aligned16(k) || !aligned16(v) || (has_q && !aligned16(q)) || !aligned16(k_codes) || !aligned16(v_codes))
    return QUAROT_ERR_ALIGN;
  if ((ld_k % 8) || (ld_v % 8) || (has_q && (ld_q % 8))) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_kv_quant_rope(k, ld_k, v, ld_v, T, n_kv, head_dim, has_q ? q : nullptr, ld_q,
                                           has_q ? n_q : 0, flags, clip_ratio, pos0, seq_len, theta, k_codes,
                                           k_scale, k_zero, v_codes, v_scale, v_zero, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

quarot_status quarot_kv_append(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t B,
                               int32_t n_kv, int32_t head_dim, void* q, int64_t ld_q, int32_t n_q,
                               uint32_t flags, float clip_ratio, const int32_t* positions, float theta,
                               int64_t s_max, uint8_t* k_codes, float* k_scale, uint8_t* k_zero,
                               uint8_t* v_codes, float* v_scale, uint8_t* v_zero, void* stream) {
  g_last_launches = 0;
  if (flags & ~3u) return QUAROT_ERR_ARG;
  if (!clip_ok(clip_ratio) || !(theta > 0.f)) return QUAROT_ERR_ARG;
  if (B < 0 || n_kv <= 0 || n_q < 0 || head_dim <= 0 || s_max <= 0) return QUAROT_ERR_DIM;
  if (!(head_dim == 64 || head_dim == 128 || head_dim == 256)) return QUAROT_ERR_UNSUPPORTED_SIZE;
  const bool has_q = q != nullptr && n_q > 0;
  if (ld_k < (int64_t)n_kv * head_dim || ld_v < (int64_t)n_kv * head_dim ||
      (has_q && ld_q < (int64_t)n_q * head_dim))
    return QUAROT_ERR_DIM;
  if (B == 0) return QUAROT_OK;
  if (!k || !v || !positions || !k_codes || !k_scale || !k_zero || !v_codes || !v_scale || !v_zero)
    return QUAROT_ERR_NULL;
  if (!aligned16(k) || !aligned16(v) || (has_q && !aligned16(q)) || !aligned16(k_codes) || !aligned16(v_codes))
    return QUAROT_ERR_ALIGN;
  if ((ld_k % 8) || (ld_v % 8) || (has_q && (ld_q % 8))) return QUAROT_ERR_ALIGN;
  cudaError_t e = qr::launch_kv_quant_rope(k, ld_k, v, ld_v, B, n_kv, head_dim, has_q ? q : nullptr, ld_q,
                                           has_q ? n_q : 0, flags, clip_ratio, 0, 1, theta, k_codes, k_scale,
                                           k_zero, v_codes, v_scale, v_zero, static_cast<cudaStream_t>(stream),
                                           positions, s_max);
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = 1;
  return QUAROT_OK;
}

int64_t quarot_kv_decode_workspace_bytes(int64_t B, int32_t n_q, int32_t head_dim, int64_t s_max) {
  if (B <= 0 || n_q <= 0 || head_dim <= 0 || s_max <= 0 || B > 65535 || s_max > (1 << 30)) return 0;
  return qr::kv_decode_workspace_bytes(B, n_q, head_dim, s_max);
}

quarot_status quarot_kv_decode(const void* q, const uint8_t* k_codes, const float* k_scale,
                               const uint8_t* k_zero, const uint8_t* v_codes, const float* v_scale,
                               const uint8_t* v_zero, const int32_t* seq_lens, int64_t B, int32_t n_q,
                               int32_t n_kv, int32_t head_dim, int64_t s_max, float sm_scale, void* out,
                               float* workspace, int64_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  if (B < 0 || n_q <= 0 || n_kv <= 0 || head_dim <= 0 || s_max <= 0 || s_max > (1 << 30)) return QUAROT_ERR_DIM;
  if (B > 65535 || n_kv > 65535) return QUAROT_ERR_DIM;  // grid (split, n_kv, B)
  if (B * s_max > 0x7fffffffLL) return QUAROT_ERR_UNSUPPORTED_SIZE;  // TMA row coordinate of the cache
  if (n_q % n_kv) return QUAROT_ERR_DIM;
  const int G = n_q / n_kv;
  if (head_dim != 128 || !(G == 1 || G == 2 || G == 4 || G == 8)) return QUAROT_ERR_UNSUPPORTED_SIZE;
  if (!(sm_scale == sm_scale) || sm_scale == INFINITY || sm_scale == -INFINITY) return QUAROT_ERR_ARG;
  if (B == 0) return QUAROT_OK;
  if (!q || !k_codes || !k_scale || !k_zero || !v_codes || !v_scale || !v_zero || !seq_lens || !out || !workspace)
    return QUAROT_ERR_NULL;
  if (workspace_bytes < quarot_kv_decode_workspace_bytes(B, n_q, head_dim, s_max)) return QUAROT_ERR_ARG;
  if (!aligned16(q) || !aligned16(k_codes) || !aligned16(v_codes) || !aligned16(out) || !aligned16(workspace))
    return QUAROT_ERR_ALIGN;
  int launches = 0;
  cudaError_t e = qr::launch_kv_decode(q, k_codes, k_scale, k_zero, v_codes, v_scale, v_zero, seq_lens, (int)B, n_q,
                                       n_kv, head_dim, (int)s_max, sm_scale, out, workspace,
                                       static_cast<cudaStream_t>(stream), &launches);
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launches = launches;
  return QUAROT_OK;
}

}  // extern "C"
