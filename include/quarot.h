/* quarot.h — C ABI of the B200 (sm_100a) QuaRot online quantized-linear hot path.
 *
 * QuaRot: Outlier-Free 4-Bit Inference in Rotated LLMs (arXiv 2404.00456).
 * Citations: P:<n> = line n of the paper's LaTeX source.
 *
 * The library implements, as hand-written CUDA kernels for sm_100a:
 *   quarot_hadamard_quant   online Hadamard (FULL / ACROSS_HEADS / NONE) fused with
 *                           per-token symmetric INT4 RTN and nibble packing
 *                           (P:182-185 Stage 1b, P:204-208 Stage 1c, P:232-233 Stage 2b)
 *   quarot_int4_linear      INT4 x INT4 GEMM (tcgen05 kind::i8, int32 accumulators in
 *                           TMEM) with the fused dequantizing epilogue
 *   quarot_int4_matmul_s32  the same mainloop exporting the raw int32 accumulators
 *                           (parity only)
 *   quarot_kv_quant         KV-cache "Init": per-head Hadamard on K (and optionally Q, in
 *                           place) + asymmetric INT4 group quantization
 *                           (P:210-225 Stage 1d, P:236-237 Stage 2c)
 *   quarot_kv_quant_rope    the same with RoPE fused in front
 *   quarot_kv_append        routine "Append": one new token per sequence into the cache
 *   quarot_kv_decode        routine "Decode": attention over the INT4 cache
 *   quarot_hadamard_quant8, quarot_int8_linear   A8W8 (8-bit RTN configuration)
 *   quarot_hadamard_quant_group(8), quarot_int4_linear_group(8)   group-wise W4A4 (§8 f3)
 *
 * Conventions (all entry points)
 *  - Tensor pointers are CUDA DEVICE pointers owned by the caller.  The library never
 *    allocates device memory; its only state is immutable per-device tables in static
 *    __device__ storage: the stored Hadamard matrices H_20, H_28, H_108, H_172 (built and
 *    verified H H^T = m I on first use) and the constant MMA operand images derived from them
 *    (written once per device by a synchronous copy on the first call that needs them: make
 *    that call outside CUDA graph capture).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  All work is enqueued
 *    on it; no entry point synchronizes the host.  Calls are reentrant across streams.
 *  - Arguments are validated before any launch; a failing call launches nothing and
 *    leaves outputs untouched.  Launch failures map to QUAROT_ERR_CUDA; asynchronous
 *    faults surface at the caller's next synchronization.  Nothing throws.
 *  - Outputs must not alias inputs (except q in quarot_kv_quant[_rope], rotated in place).
 *  - Results are bitwise deterministic for identical inputs and independent of how
 *    rows are split across calls or GPUs (no atomics in any reduction).
 *  - INT4 signed codes are stored two per byte, two's complement nibbles, LOW nibble =
 *    EVEN index: byte j = (c[2j] & 0xF) | (c[2j+1] << 4)   (the "sub-byte format").
 */
#ifndef QUAROT_H_
#define QUAROT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QUAROT_ABI_VERSION 2  /* 2: mode / head_dim in the group-wise quantizers */

typedef enum {
  QUAROT_OK = 0,
  QUAROT_ERR_NULL = 1,             /* a required pointer is NULL                        */
  QUAROT_ERR_DIM = 2,              /* non-positive / inconsistent dimension, ld < width */
  QUAROT_ERR_UNSUPPORTED_SIZE = 3, /* K not 2^n * m with m in {1, 20, 28, 108, 172}; heads not 2^n */
  QUAROT_ERR_ALIGN = 4,            /* pointer / leading dimension misaligned (16 B) or a
                                      width not a multiple of the kernel granularity    */
  QUAROT_ERR_ARG = 5,              /* clip ratio outside (0, 1], bad mode or flags       */
  QUAROT_ERR_CUDA = 6              /* CUDA runtime error at launch                       */
} quarot_status;

typedef enum {
  /* QKV / gate-up input: quantize only (the global rotation Q is fused into W). */
  QUAROT_HAD_NONE = 0,
  /* down_proj input: y = H^_K x, H^_K = (H_{2^n} (x) H_m) / sqrt(K), K = 2^n m,
   * m in {1, 20, 28, 108, 172} (20 and 108 serve the Llama-2-13B widths).
   * Element i = a*m + b: H_m acts on the contiguous index b, H_{2^n} (Sylvester / natural order, Eq. 1) on a.  y_i = sum_j H^_ij x_j. */
  QUAROT_HAD_FULL = 1,
  /* out_proj input, "Hadamard heads" (Eq. 9): y = (H_{n_h} (x) I_{d_h}) z / sqrt(n_h),
   * n_h = K / head_dim; n_h and head_dim powers of two. */
  QUAROT_HAD_ACROSS_HEADS = 2
} quarot_had_mode;

/* Mode flag (OR-ed into `mode`, NONE only): RMS-normalize each row first, x <- x / sqrt(mean(x^2)
 * + 1e-5), in FP32 — the scale-free RMSNorm feeding "quantize" (Fig. ffn_quarot; reading
 * Z21).  A positive per-row scaling leaves the codes unchanged, so the kernel quantizes x and
 * divides the scale by the row RMS: one pass over x (SURVEY §8 a8 fused, f1). */
#define QUAROT_HAD_RMSNORM 0x100

/* Mode flag (OR-ed into `mode`, FULL only; K = 1024 x 28): write the codes in the transform's
 * native K order instead of the natural element order.  The FULL kernel produces output element
 * i = a * J + j' (a = the 2^n Sylvester index, j' = the H_m-side index, J = K / 256) with a warp
 * owning 32 consecutive j'; in the native order the code of element i sits at position
 *     p(i) = (a >> 5) * 32 J + 32 j' + (a & 31)
 * so every thread writes 16 contiguous bytes and a warp 512 (quarot_full_kperm returns the
 * permutation).  The INT4 GEMM's accumulator is a sum over k, so pairing these codes with
 * weights whose columns are permuted the same way offline (W'[n][p] = W[n][i(p)]) gives
 * bit-identical int32 accumulators and outputs.  Requires
 * ld_q % 16 == 0 and a 16-byte aligned q (QUAROT_ERR_ALIGN); other K: QUAROT_ERR_UNSUPPORTED_SIZE. */
#define QUAROT_HAD_KPERM 0x200

/* Rows a1|a2 + a3 of the hot path: online Hadamard + per-token symmetric INT4 RTN + pack.
 *
 *   x      fp16 [M][ld_x] row-major (K used); 16-B aligned; ld_x % 8 == 0.
 *   M      tokens (>= 0; M == 0 is a no-op).      K  width (even; see mode).
 *   mode   quarot_had_mode.  head_dim: used by ACROSS_HEADS only (power of two).
 *   clip_ratio  in (0, 1]; the paper uses 0.9.
 *   q      uint8 [M][ld_q] (K/2 bytes used), 16-B aligned; ld_q % 4 == 0 (% 16 for
 *          ACROSS_HEADS).
 *   scale  fp32 [M].
 * Per row, with y the transformed (normalized) row (fp32 arithmetic on fp16 input):
 *   a = max_k |y_k|;  a == 0 -> scale 1, codes 0;  a not finite -> scale NaN, codes 0;
 *   else scale = fp32(clip * a / 7), code_k = clamp(round_half_even(y_k / scale), -7, 7)
 *   ("dividing the maximum absolute value of each token by 7 ... round the
 *   result to its nearest integer").  x^ = code * scale approximates y.
 * Granularity / limits (QUAROT_ERR_ALIGN / QUAROT_ERR_UNSUPPORTED_SIZE otherwise):
 *   NONE: K % 16 == 0, K <= 32768.
 *   ACROSS_HEADS: K % 32 == 0; head_dim a power of two >= 64; n_h = K / head_dim a power of
 *     two.  head_dim 128 with n_h in {16, 32, 64} runs on the tensor cores; every other
 *     shape on the CUDA-core kernel, which needs (head_dim / 2) * max(1, n_h / 32) <= 256
 *     and K <= 32768.
 *   FULL: K = 2^n m with 2^n >= 2, K % 16 == 0, K <= 32768.                          */
quarot_status quarot_hadamard_quant(const void* x, int64_t M, int64_t K, int64_t ld_x,
                                    int32_t mode, int32_t head_dim, float clip_ratio,
                                    uint8_t* q, int64_t ld_q, float* scale, void* stream);

/* Rows a4 + a5: y[m][n] = fp16_rn( (fp32)acc[m][n] * x_scale[m] * w_scale[n] ),
 *   acc[m][n] = sum_k cx[m][k] * cw[n][k]   (exact int32).
 *   xq     uint8 [M][ld_xq] packed INT4 activations (output of quarot_hadamard_quant).
 *   wq     uint8 [N][ld_wq] packed INT4 weights, nn.Linear [out][in] orientation (same
 *          nibble layout along K), pre-rotated offline to pair with the online mode.
 *   x_scale fp32 [M], w_scale fp32 [N] (per output channel, "per-column").
 *   y      fp16 [M][ld_y].
 * Requirements: K % 128 == 0; N % 8 == 0; ld_xq, ld_wq % 16 == 0; ld_y % 8 == 0; all
 * pointers 16-B aligned.  Ragged M and N tails are handled.  Activation codes must lie in
 * [-7, 7] (quarot_hadamard_quant never writes -8), weight codes in [-8, 7]: the accumulator
 * is then exact for K <= 149796 (larger K: QUAROT_ERR_UNSUPPORTED_SIZE). */
quarot_status quarot_int4_linear(const uint8_t* xq, const float* x_scale, int64_t M, int64_t K,
                                 int64_t ld_xq, const uint8_t* wq, const float* w_scale,
                                 int64_t N, int64_t ld_wq, void* y, int64_t ld_y, void* stream);

/* quarot_int4_linear with the residual add of the decoder layer fused into the epilogue
 * (SURVEY §8 a8): y = fp16_rn( (fp32)fp16_rn((fp32)acc * x_scale[m] * w_scale[n]) + (fp32)residual[m][n] )
 *   — the linear output is cast to FP16 first ("immediately cast (and scale) to FP16"), then
 *   the FP16 model's residual add; bitwise equal to quarot_int4_linear followed by an fp16 add.
 *   residual fp16 [M][ld_r] (ld_r % 8 == 0, 16-B aligned); it may alias y (in-place add). */
quarot_status quarot_int4_linear_residual(const uint8_t* xq, const float* x_scale, int64_t M, int64_t K,
                                          int64_t ld_xq, const uint8_t* wq, const float* w_scale,
                                          int64_t N, int64_t ld_wq, const void* residual, int64_t ld_r,
                                          void* y, int64_t ld_y, void* stream);

/* Gate/up projection with the SwiGLU activation fused into the epilogue (SURVEY §8 a8 + f1):
 * the N2 = 2F rows of wq / w_scale are the gate and up rows interleaved in blocks of 8 —
 * row 16j + i is gate feature 8j + i and row 16j + 8 + i is up feature 8j + i (i < 8), an
 * offline layout choice (quarot.interleave_gate_up) — and the output is
 *   act[m][f] = fp16_rn( fp16_rn(silu(g)) * u ),  g = fp16_rn(acc_gate * x_scale[m] * w_scale[gate row]),
 *   u = fp16_rn(acc_up * x_scale[m] * w_scale[up row])  — the fp16 linear outputs through
 *   the FP16 model's SiLU and multiply (reading Z23); bitwise equal to quarot_int4_linear on the
 *   de-interleaved weights followed by quarot_swiglu.
 *   act fp16 [M][ld_act], ld_act >= N2/2, % 8 == 0.  N2 % 16 == 0. */
quarot_status quarot_int4_linear_swiglu(const uint8_t* xq, const float* x_scale, int64_t M, int64_t K,
                                        int64_t ld_xq, const uint8_t* wq, const float* w_scale, int64_t N2,
                                        int64_t ld_wq, void* act, int64_t ld_act, void* stream);

/* Parity only: the same tcgen05 mainloop, raw accumulators acc int32 [M][ld_acc]
 * (ld_acc % 4 == 0).  Same requirements as quarot_int4_linear. */
quarot_status quarot_int4_matmul_s32(const uint8_t* xq, int64_t M, int64_t K, int64_t ld_xq,
                                     const uint8_t* wq, int64_t N, int64_t ld_wq,
                                     int32_t* acc, int64_t ld_acc, void* stream);

/* Rows a6 + a7, KV-cache Init (P:858 routine "Init").
 *   k, v   fp16 [T][ld_k] / [T][ld_v]: token t's heads at k + t*ld_k, [n_kv][head_dim]
 *          contiguous (post-RoPE keys, values).  ld_* are in elements, >= n*head_dim,
 *          multiples of 8 — so K, V and Q can be read straight out of a fused QKV output.
 *   q      optional fp16 [T][ld_q] ([n_q][head_dim] per token), rotated IN PLACE
 *          q_h <- H^ q_h (Eq. 13), rounded to fp16; NULL or n_q == 0 skips it.
 *   flags  bit0: rotate K (Eq. 14; default set), bit1: rotate V (the paper fuses
 *          V's rotation into W_v, so bit1 is for tests only).  Other bits: ERR_ARG.
 *   clip_ratio in (0, 1]; the paper uses 0.95.  Group = head_dim (128 in the paper).
 *   *_codes uint8 [T][n_kv][head_dim/2] unsigned nibbles (low = even index);
 *   *_scale fp32 [T][n_kv]; *_zero uint8 [T][n_kv].
 * Per group g (after the optional rotation H^ = H_{head_dim} / sqrt(head_dim)):
 *   lo = clip * min(min g, 0), hi = clip * max(max g, 0);  hi == lo -> scale 1, zero 0,
 *   codes 0;  else scale = fp32((hi - lo) / 15), zero = clamp(rne(-lo / scale), 0, 15),
 *   code = clamp(rne(g / scale) + zero, 0, 15);  x^ = (code - zero) * scale.
 * Requirements: head_dim in {64, 128, 256}; T >= 0; n_kv >= 1; 16-B aligned pointers. */
quarot_status quarot_kv_quant(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T,
                              int32_t n_kv, int32_t head_dim, void* q, int64_t ld_q, int32_t n_q,
                              uint32_t flags,
                              float clip_ratio, uint8_t* k_codes, float* k_scale,
                              uint8_t* k_zero, uint8_t* v_codes, float* v_scale,
                              uint8_t* v_zero, void* stream);

/* quarot_kv_quant with RoPE fused in front ("RoPE + per-head H + KV quant"
 * in one pass).  Same arguments and outputs as quarot_kv_quant, plus the quarot_rope
 * parameters (pos0, seq_len, theta).  K and Q are read PRE-RoPE; each K / Q head gets
 *   r = fp16_rn(rope(x))  (exactly quarot_rope's arithmetic: fp64 angle table rounded to fp32,
 *   fp32 rotate-half, fp16 RNE), then the rotation / quantization of quarot_kv_quant.
 * K stays untouched in memory (only its codes are written); Q is overwritten with
 * fp16(H^ fp16(rope(q))).  V gets no RoPE.  Requirements: quarot_kv_quant's, seq_len >= 1,
 * theta > 0, pos0 >= 0. */
quarot_status quarot_kv_quant_rope(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T,
                                   int32_t n_kv, int32_t head_dim, void* q, int64_t ld_q, int32_t n_q,
                                   uint32_t flags, float clip_ratio, int64_t pos0, int32_t seq_len,
                                   float theta, uint8_t* k_codes, float* k_scale, uint8_t* k_zero,
                                   uint8_t* v_codes, float* v_scale, uint8_t* v_zero, void* stream);

/* group-wise symmetric INT4 ("group-wise quantization", group sizes 256 / 128 /
 * 64 in tab:group_wise_ablation P:392-416), after the online transform of `mode`.
 * quarot_hadamard_quant_group: y = the transformed row exactly as quarot_hadamard_quant computes it
 *   (mode NONE / FULL / ACROSS_HEADS, head_dim for ACROSS_HEADS; the normalized transform, reading
 *   Z5); then every run of `group` consecutive elements of y (natural element order) is quantized by
 *   the rule of quarot_hadamard_quant (scale = fp32(clip * max|y_g| / 7), codes RNE, clamp [-7, 7];
 *   zero group: scale 1, codes 0; non-finite group: scale NaN, codes 0).
 *   x      fp16 [M][ld_x] device, K elements used per row
 *   q      uint8 [M][ld_q] device, K/2 packed bytes (low nibble = even element)
 *   scale  fp32 [M][ld_s] device, K/group scales per row (ld_s >= K/group)
 *   group  64, 128 or 256 (QUAROT_ERR_UNSUPPORTED_SIZE otherwise); K % group == 0 (QUAROT_ERR_DIM)
 *   mode   NONE: M < 2^31, K <= 65535 * 1024.  FULL: K = 2^n m (n >= 1, m in {1, 20, 28, 108, 172}),
 *          K <= 32768, K % 16 == 0.  ACROSS_HEADS: head_dim and n_h = K / head_dim >= 2 powers of two,
 *          K <= 32768, K % 16 == 0 (QUAROT_ERR_UNSUPPORTED_SIZE / QUAROT_ERR_ALIGN otherwise).
 *          RMSNORM / KPERM flags: QUAROT_ERR_ARG.
 * Errors as quarot_hadamard_quant; x and q 16-byte aligned, ld_x % 8 == 0, ld_q % 4 == 0.
 * quarot_hadamard_quant_group8: the same codes, one per int8 byte (q int8 [M][ld_q], ld_q >= K,
 *   ld_q % 8 == 0). */
quarot_status quarot_hadamard_quant_group(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode,
                                         int32_t head_dim, int32_t group, float clip_ratio, uint8_t* q, int64_t ld_q,
                                         float* scale, int64_t ld_s, void* stream);
quarot_status quarot_hadamard_quant_group8(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode,
                                          int32_t head_dim, int32_t group, float clip_ratio, int8_t* q, int64_t ld_q,
                                          float* scale, int64_t ld_s, void* stream);
/* quarot_int4_linear_group: group-wise W4A4 linear (§8 f3), group G in {64, 128, 256}:
 *   y[m][n] = fp16( sum_g x_scale[m][g] * w_scale_t[g][n] * sum_{k in g} cx[m][k] * cw[n][k] ),
 *   the per-group integer sums exact (int32 on the tensor cores), the scaled sum in fp32.
 *   xq uint8 [M][ld_xq] and wq uint8 [N][ld_wq]: packed INT4 codes (the sub-byte format above,
 *   K/2 bytes per row; activation codes in [-7, 7], weight codes in [-8, 7]); x_scale fp32
 *   [M][ld_sx] (K/G per row, as quarot_hadamard_quant_group writes them); w_scale_t fp32
 *   [K/G][ld_sw] (transposed, prepared offline); y fp16 [M][ld_y].  K % 256 == 0, N % 8 == 0,
 *   ld_xq / ld_wq % 16 == 0, ld_y % 8 == 0, ld_sw % 4 == 0, 16-byte aligned xq / wq / y / w_scale_t
 *   (QUAROT_ERR_ALIGN); other G: QUAROT_ERR_UNSUPPORTED_SIZE.
 * quarot_int4_linear_group8: the same for G = 128 with the codes stored one per int8 byte
 *   (xq int8 [M][ld_xq], wq int8 [N][ld_wq], ld >= K; the format quarot_hadamard_quant_group8
 *   writes) on the native kind::i8 path without unpacking — the comparison point for the
 *   on-chip widening. */
quarot_status quarot_int4_linear_group(const uint8_t* xq, const float* x_scale, int64_t ld_sx, int64_t M, int64_t K,
                                       int64_t ld_xq, const uint8_t* wq, const float* w_scale_t, int64_t ld_sw,
                                       int64_t N, int64_t ld_wq, int32_t group, void* y, int64_t ld_y, void* stream);
quarot_status quarot_int4_linear_group8(const int8_t* xq, const float* x_scale, int64_t ld_sx, int64_t M, int64_t K,
                                        int64_t ld_xq, const int8_t* wq, const float* w_scale_t, int64_t ld_sw,
                                        int64_t N, int64_t ld_wq, int32_t group, void* y, int64_t ld_y, void* stream);

/* A8W8 QuaRot ("lossless" 8-bit RTN, P:6, tab:rtn_results): the native
 * kind::i8 tensor path with no unpacking, the comparison point for the INT4 unpack cost.
 * quarot_hadamard_quant8: as quarot_hadamard_quant but codes are int8 in [-127, 127], one byte
 *   per element (q int8 [M][ld_q], ld_q >= K, % 8), scale = fp32(clip * amax / 127).  Modes:
 *   NONE (optionally | QUAROT_HAD_RMSNORM), FULL for every K = 2^n m of quarot_hadamard_quant
 *   (the tcgen05 kernels at 1024 x 28, 64 x 172, 128 x 108 and 256 x 20), ACROSS_HEADS for
 *   power-of-two head_dim and n_h >= 2 (tcgen05 at head_dim 128 with 16-64 heads); K <= 32768.
 *   RMSNORM with FULL / ACROSS_HEADS returns QUAROT_ERR_ARG.
 * quarot_int8_linear: y[m,n] = fp16_rn(fp32(acc) * x_scale[m] * w_scale[n]),
 *   acc = sum_k xq[m,k] * wq[n,k] (int8 x int8 -> exact int32).  xq int8 [M][ld_xq], wq int8
 *   [N][ld_wq] (nn.Linear layout), ld % 16 == 0, K % 128 == 0, K <= 131072, N % 8 == 0.
 * quarot_int8_matmul_s32: raw accumulators (parity only). */
quarot_status quarot_hadamard_quant8(const void* x, int64_t M, int64_t K, int64_t ld_x, int32_t mode,
                                     int32_t head_dim, float clip_ratio, int8_t* q, int64_t ld_q, float* scale,
                                     void* stream);
quarot_status quarot_int8_linear(const int8_t* xq, const float* x_scale, int64_t M, int64_t K, int64_t ld_xq,
                                 const int8_t* wq, const float* w_scale, int64_t N, int64_t ld_wq, void* y,
                                 int64_t ld_y, void* stream);
quarot_status quarot_int8_matmul_s32(const int8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const int8_t* wq,
                                     int64_t N, int64_t ld_wq, int32_t* acc, int64_t ld_acc, void* stream);

/* the decoding routines of the paper's quantized attention.
 * Cache layout (one cache per sequence, s_max rows each): *_codes uint8
 * [B][s_max][n_kv][head_dim/2], *_scale fp32 [B][s_max][n_kv], *_zero uint8 [B][s_max][n_kv]
 * — i.e. quarot_kv_quant's output layout with T = B * s_max tokens (Init fills rows 0..T-1 of
 * a sequence by calling it on that sequence's slice).
 *
 * quarot_kv_append — routine 2 "Append": one new token per sequence.  k, v, q fp16
 *   [B][ld_*] (heads [n][head_dim] contiguous; PRE-RoPE k and q).  positions int32 [B]
 *   (DEVICE): the new token's row in its sequence's cache, also its RoPE position.  Applies
 *   RoPE (theta) to K and Q, then exactly quarot_kv_quant's rotation / quantization; writes the
 *   K/V groups at cache row positions[b] of sequence b and overwrites q with the rotated query
 *   fp16(H^ fp16(rope(q))) that quarot_kv_decode consumes.  positions[b] < s_max (unchecked:
 *   device data).  flags / clip_ratio as quarot_kv_quant. */
quarot_status quarot_kv_append(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t B,
                               int32_t n_kv, int32_t head_dim, void* q, int64_t ld_q, int32_t n_q,
                               uint32_t flags, float clip_ratio, const int32_t* positions, float theta,
                               int64_t s_max, uint8_t* k_codes, float* k_scale, uint8_t* k_zero,
                               uint8_t* v_codes, float* v_scale, uint8_t* v_zero, void* stream);

/* quarot_kv_decode — routine 3 "Decode": attention of one (rotated) query per sequence
 * against the INT4 cache, rows 0 .. seq_lens[b]-1 (seq_lens int32 [B], DEVICE, 1 <= seq_lens[b]
 * <= s_max, unchecked):  o = softmax(<q, k^_j> * sm_scale) . v^,  x^ = (c - z) * s,  GQA head
 * h -> KV head h / (n_q / n_kv).  q fp16 [B][n_q][head_dim] contiguous; out fp16
 * [B][n_q][head_dim] contiguous (o is in V's space: V is not rotated online).
 * workspace fp32, quarot_kv_decode_workspace_bytes(B, n_q, head_dim, s_max) bytes, caller-owned.
 * Requirements: head_dim == 128; n_q / n_kv in {1, 2, 4, 8}; B, n_kv <= 65535 (ERR_DIM);
 * B * s_max < 2^31 (ERR_UNSUPPORTED_SIZE: the cache rows are addressed by one TMA coordinate);
 * sm_scale finite (the standard
 * 1/sqrt(head_dim) is reading Z24); 16-B aligned pointers.  Two kernel launches. */
quarot_status quarot_kv_decode(const void* q, const uint8_t* k_codes, const float* k_scale,
                               const uint8_t* k_zero, const uint8_t* v_codes, const float* v_scale,
                               const uint8_t* v_zero, const int32_t* seq_lens, int64_t B, int32_t n_q,
                               int32_t n_kv, int32_t head_dim, int64_t s_max, float sm_scale, void* out,
                               float* workspace, int64_t workspace_bytes, void* stream);
int64_t quarot_kv_decode_workspace_bytes(int64_t B, int32_t n_q, int32_t head_dim, int64_t s_max);

/* Decoder-layer glue.
 * quarot_rope: Llama-2 rotary position embedding ("Pos", Eqs. 10-12), in place on
 *   x fp16 [T][ld_x] holding n_heads x head_dim per token: for pair (i, i + d/2),
 *   angle = pos * theta^(-2i/d), pos = (pos0 + t) % seq_len; fp32 math, fp16 RNE result.
 *   head_dim even and <= 256; ld_x % 8 == 0; x 16-B aligned.  Apply it to the Q|K block of a
 *   fused QKV output (n_heads = n_q + n_kv) before quarot_kv_quant.
 * quarot_swiglu: act[m][f] = fp16(fp16(silu(gu[m][f])) * gu[m][F + f]) — the gated FFN activation of
 *   Fig. ffn_orig with [gate | up] column halves; F % 8 == 0, ld % 8 == 0, 16-B aligned. */
quarot_status quarot_rope(void* x, int64_t T, int32_t n_heads, int32_t head_dim, int64_t ld_x,
                          int64_t pos0, int32_t seq_len, float theta, void* stream);
quarot_status quarot_swiglu(const void* gate_up, int64_t M, int64_t F, int64_t ld_gu, void* act,
                            int64_t ld_act, void* stream);

/* Host-side utilities (no GPU work). */
const char* quarot_status_string(int32_t status);
int32_t quarot_abi_version(void);
/* Copies the library's stored base Hadamard H_m (m in {20, 28, 108, 172}) as int8 +-1, row-major,
 * into host buffer out[m*m].  Lets tests compare the library's independently built table
 * with the oracle's.  Returns QUAROT_ERR_UNSUPPORTED_SIZE for other m. */
quarot_status quarot_base_hadamard(int32_t m, int8_t* out);
/* The QUAROT_HAD_KPERM permutation for width K (host, no GPU work): perm[p] = the natural element
 * index whose code sits at position p (perm: int64 [K], caller-owned).  K = 1024 x 28 only
 * (QUAROT_ERR_UNSUPPORTED_SIZE otherwise). */
quarot_status quarot_full_kperm(int64_t K, int64_t* perm);
/* One-time setup for the current device: uploads the library's constant operand images and
 * Hadamard tables (static __device__ memory) and sets the kernels' shared-memory attributes,
 * synchronously (it ends with a device synchronization).  Optional — every entry point does the
 * same lazily on first use — but calling it once before CUDA-graph capture or before a timed
 * region keeps the first real call free of host synchronization.  Idempotent; errors:
 * QUAROT_ERR_CUDA. */
quarot_status quarot_prepare(void);
/* Number of kernels the last successful entry point on this host thread enqueued. */
int32_t quarot_last_launch_count(void);
/* "cudaErrorName: description" of the last call on this host thread that returned
 * QUAROT_ERR_CUDA ("" if none); the buffer is owned by the library. */
const char* quarot_last_cuda_error(void);

/* Diagnostics: process-wide kernel-variant switches for A/B experiments and roofline probes
 * (not thread-safe; 0 restores the default).  quarot_debug_gemm_mode: 1 = the INT4 GEMM with its
 * producers idled (MMA issue only: the tensor-pipe probe bench.py reports as the INT8 peak), 2 =
 * no widening stores, 3 = no TMA, 4 = no output stores, 5 = no B widening stores, 6 = no A TMEM
 * stores, 7 = no epilogue work, 8 = the MMA skips the wait for the accumulator drain — probes 1-8
 * compute garbage.
 * quarot_debug_gemm_group_m: raster group override (pair-rows).  quarot_debug_hq_full_variant:
 * 1 = the mma.sync FULL-28 kernel, 2 / 3 = the 16-warps-per-row tcgen05 kernel (spin / sleep
 * waits).  quarot_debug_hq_heads_variant: 1 = the CUDA-core ACROSS_HEADS kernel for every width.
 * quarot_debug_kv_variant: 1 = the CUDA-core KV kernel for every shape. */
void quarot_debug_gemm_mode(int32_t mode);
void quarot_debug_gemm_group_m(int32_t group_m);
void quarot_debug_hq_full_variant(int32_t variant);
void quarot_debug_hq_heads_variant(int32_t variant);
void quarot_debug_kv_variant(int32_t variant);

#ifdef __cplusplus
}
#endif
#endif /* QUAROT_H_ */
