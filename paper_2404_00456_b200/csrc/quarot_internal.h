// quarot_internal.h — launchers shared between the kernels and the C-ABI shim.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qr {

// int4_gemm.cu
cudaError_t launch_int4_gemm(const uint8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                             const uint8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* y,
                             int64_t ld_y, cudaStream_t stream, const void* residual = nullptr,
                             int64_t ld_r = 0);
cudaError_t launch_int4_gemm_swiglu(const uint8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                                    const uint8_t* wq, const float* ws, int64_t N2, int64_t ld_wq, void* act,
                                    int64_t ld_act, cudaStream_t stream);
cudaError_t launch_int4_gemm_s32(const uint8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const uint8_t* wq,
                                 int64_t N, int64_t ld_wq, int32_t* acc, int64_t ld_acc, cudaStream_t stream);

// hadamard_quant.cu
// group-wise symmetric INT4, mode NONE: group in {64, 128, 256}, scale [M][K/group]
cudaError_t launch_hq_none_group(const void* x, int64_t M, int64_t K, int64_t ld_x, int group, float clip,
                                 uint8_t* q, int64_t ld_q, float* scale, int64_t ld_s, cudaStream_t stream,
                                 bool q8 = false);
// group-wise W4A4 GEMM (§8 f3): codes one per int8 byte, x scales [M][ld_sx], weight scales
// transposed [K/128][ld_sw]; y fp16
cudaError_t launch_int8_group_gemm(const int8_t* xq, const float* xs, int64_t ld_sx, int64_t M, int64_t K,
                                   int64_t ld_xq, const int8_t* wq, const float* ws_t, int64_t ld_sw, int64_t N,
                                   int64_t ld_wq, void* y, int64_t ld_y, cudaStream_t stream);
// group-wise W4A4 GEMM on packed INT4 codes (§8 f3), group in {64, 128, 256}
cudaError_t launch_int4_group_gemm(const uint8_t* xq, const float* xs, int64_t ld_sx, int64_t M, int64_t K,
                                   int64_t ld_xq, const uint8_t* wq, const float* ws_t, int64_t ld_sw, int64_t N,
                                   int64_t ld_wq, int group, void* y, int64_t ld_y, cudaStream_t stream);
cudaError_t launch_hq_none(const void* x, int64_t M, int64_t K, int64_t ld_x, float clip, uint8_t* q,
                           int64_t ld_q, float* scale, cudaStream_t stream, bool rmsnorm = false);
cudaError_t launch_hq_heads(const void* x, int64_t M, int64_t K, int64_t ld_x, int head_dim, float clip,
                            uint8_t* q, int64_t ld_q, float* scale, cudaStream_t stream);
// hq_full_tc.cu: K = 1024 x 28 on the tcgen05 path (the default for that width)
// kperm: codes in the transform-native K order (quarot.h QUAROT_HAD_KPERM)
cudaError_t launch_hq_full28_tc(const void* x, int64_t M, int64_t ld_x, float clip, uint8_t* q, int64_t ld_q,
                                float* scale, cudaStream_t stream, bool q8 = false, bool kperm = false);
extern int g_hq_full_variant;
// hq_full_small_tc.cu: the Llama-2-13B widths K = 128 x 108 and 256 x 20 on the tcgen05 path
bool hq_full_small_tc_supported(int64_t pow2, int m);
cudaError_t launch_hq_full_small_tc(const void* x, int64_t M, int64_t ld_x, int64_t pow2, int m, float clip,
                                    uint8_t* q, int64_t ld_q, float* scale, cudaStream_t stream, bool q8 = false);
// hq_full172_tc.cu: K = 64 x 172 on the tcgen05 path (the default for that width)
cudaError_t launch_hq_full172_tc(const void* x, int64_t M, int64_t ld_x, float clip, uint8_t* q, int64_t ld_q,
                                 float* scale, cudaStream_t stream, bool q8 = false);
// hq_heads_tc.cu: ACROSS_HEADS on the tcgen05 path (head_dim 128, n_h in {16, 32, 64})
bool hq_heads_tc_supported(int64_t K, int head_dim);
cudaError_t launch_hq_heads_tc(const void* x, int64_t M, int64_t K, int64_t ld_x, int head_dim, float clip, uint8_t* q,
                               int64_t ld_q, float* scale, cudaStream_t stream, bool q8 = false);
// FULL, K = pow2 * m.  out: 0 INT4 per row, 1 int8 per row (A8), 2 INT4 per group (scale [M][ld_s]),
// 3 INT4 per group one code per byte.  The model widths take the tcgen05 kernels for out 0 / 1.
cudaError_t launch_hq_full(const void* x, int64_t M, int64_t K, int64_t ld_x, int pow2, int m, float clip,
                           uint8_t* q, int64_t ld_q, float* scale, cudaStream_t stream, int out = 0, int group = 0,
                           int64_t ld_s = 0);
// ACROSS_HEADS group-wise (§8 f3): y = (H_{n_h} (x) I) z, then per-group INT4 (q8: one code per byte)
cudaError_t launch_hq_heads_group(const void* x, int64_t M, int64_t K, int64_t ld_x, int head_dim, float clip,
                                  uint8_t* q, int64_t ld_q, float* scale, int64_t ld_s, int group, bool q8,
                                  cudaStream_t stream);
// ACROSS_HEADS 8-bit per row on the smem kernel (the shapes the tcgen05 kernel does not take)
cudaError_t launch_hq_heads8(const void* x, int64_t M, int64_t K, int64_t ld_x, int head_dim, float clip, uint8_t* q,
                             int64_t ld_q, float* scale, cudaStream_t stream);
extern int g_hq_heads_variant;

// kv_quant.cu
cudaError_t launch_kv_quant(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int n_kv,
                            int head_dim, void* q, int64_t ld_q, int n_q, uint32_t flags, float clip, uint8_t* k_codes, float* k_scale, uint8_t* k_zero,
                            uint8_t* v_codes, float* v_scale, uint8_t* v_zero, cudaStream_t stream);
cudaError_t launch_kv_quant_rope(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int n_kv,
                                 int head_dim, void* q, int64_t ld_q, int n_q, uint32_t flags, float clip,
                                 int64_t pos0, int seq_len, float theta, uint8_t* k_codes, float* k_scale,
                                 uint8_t* k_zero, uint8_t* v_codes, float* v_scale, uint8_t* v_zero,
                                 cudaStream_t stream, const int32_t* positions = nullptr, int64_t s_max = 0);
// kv_quant_tc.cu: KV Init (± RoPE) on the tcgen05 path (head_dim 128, n_kv power of two >= 4,
// n_q % n_kv == 0, K rotated / V not, no per-sequence positions)
bool kv_tc_supported(int n_kv, int head_dim, int n_q, uint32_t flags, const int32_t* positions);
cudaError_t launch_kv_tc(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int n_kv, void* q,
                         int64_t ld_q, int n_q, float clip, bool rope, int64_t pos0, int seq_len, float theta,
                         uint8_t* k_codes, float* k_scale, uint8_t* k_zero, uint8_t* v_codes, float* v_scale,
                         uint8_t* v_zero, cudaStream_t stream);
extern int g_kv_variant;
// A8W8: int8 per-token quantizer (mode NONE, optional RMSNorm) and the
// int8 x int8 GEMM with the same epilogues
cudaError_t launch_hq_none_q8(const void* x, int64_t M, int64_t K, int64_t ld_x, float clip, int8_t* q, int64_t ld_q,
                              float* scale, cudaStream_t stream, bool rmsnorm);
cudaError_t launch_int8_gemm(const int8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                             const int8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* y, int64_t ld_y,
                             cudaStream_t stream, const void* residual = nullptr, int64_t ld_r = 0);
cudaError_t launch_int8_gemm_s32(const int8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const int8_t* wq, int64_t N,
                                 int64_t ld_wq, int32_t* acc, int64_t ld_acc, cudaStream_t stream);
// KV Decode: split-sequence flash decoding over the INT4 cache + the combine pass.
int64_t kv_decode_workspace_bytes(int64_t B, int64_t n_q, int64_t head_dim, int64_t s_max);
cudaError_t launch_kv_decode(const void* q, const uint8_t* k_codes, const float* k_scale, const uint8_t* k_zero,
                             const uint8_t* v_codes, const float* v_scale, const uint8_t* v_zero,
                             const int32_t* seq_lens, int B, int n_q, int n_kv, int head_dim, int s_max,
                             float sm_scale, void* out, float* workspace, cudaStream_t stream,
                             int* launches = nullptr);

// glue.cu
cudaError_t launch_rope(void* x, int64_t T, int n_heads, int head_dim, int64_t ld_x, int64_t pos0, int seq_len,
                        float theta, cudaStream_t stream);
cudaError_t launch_swiglu(const void* gu, int64_t M, int64_t F, int64_t ld_gu, void* act, int64_t ld_act,
                          cudaStream_t stream);

// hadamard_tables.cu — host construction of the stored H_m (m = 28, 172), verified H H^T = m I,
// and their device-side mma.sync B-fragment tables (built once per device).
const int8_t* base_hadamard_host(int m);  // nullptr for unsupported m
cudaError_t ensure_device_tables();
const uint32_t* device_bfrag_table(int m);  // device pointer (valid after ensure_device_tables)
// H_28 as mma.sync A fragments [mt][ks][lane][4] (rows b, cols b'), for hq_full28_kernel
const uint32_t* device_afrag28();

}  // namespace qr
