// hadamard_quant.cu — rows a1/a2 + a3 of the QuaRot hot path on sm_100a.
//
// Online Hadamard transform of fp16 activation rows (FP32 arithmetic), fused with
// per-token symmetric INT4 round-to-nearest (clip 0.9 P:249) and nibble packing
// (the "sub-byte format").  One read of x, one write of the packed codes + scale.
//
//   NONE          quantize only (QKV / gate-up inputs; global Q fused into W)
//   ACROSS_HEADS  y = (H_{n_h} (x) I_{d_h}) z   ("Hadamard heads", Eq. 9)
//   FULL          y = (H_{2^n} (x) H_m) x, m in {1, 20, 28, 108, 172}   (down_proj input)
//
// The orthonormal factor 1/sqrt(size) (reading Z5) is folded into the per-row scale: codes
// are invariant to positive scaling of y, so the kernels transform unnormalized and scale
// once per row in double precision.
#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace hq {

// RNE code in [-QMAX, QMAX] of v * inv (inv = 1 / scale, or 0 for a zero / non-finite row);
// QMAX = 7 for INT4, 127 for the 8-bit configuration (§8 f4)
template <int QMAX = 7>
QR_DEVICE int code_of(float v, float inv) {
  int c = __float2int_rn(v * inv);
  c = c > QMAX ? QMAX : c;
  c = c < -QMAX ? -QMAX : c;
  return c;
}
QR_DEVICE uint32_t nib(int c) { return (uint32_t)c & 0xFu; }

// Per-row scale from the unnormalized amax: scale = fp32(clip * amax * norm / 7);
// returns inv = norm / scale so that code = rne(y_unnorm * inv).  Zero row -> scale 1,
// inv 0 (all codes 0); non-finite -> scale NaN, inv 0.
QR_DEVICE void row_scale(float amax_u, double norm, float clip, float& scale, float& inv, double qmax = 7.0) {
  if (amax_u == 0.f) {
    scale = 1.f;
    inv = 0.f;
  } else if (!isfinite(amax_u)) {
    scale = __int_as_float(0x7fc00000);
    inv = 0.f;
  } else {
    const double s = (double)clip * (double)amax_u * norm / qmax;
    scale = (float)s;
    inv = (float)(norm / (double)scale);
  }
}

template <int NWARPS>
QR_DEVICE float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int w = 1; w < NWARPS; ++w) r = fmax_nan(r, red[w]);
  return r;
}

// ------------------------------------------------------------------ NONE
// One row per 128-thread CTA; each thread owns CPT 8-element chunks held in registers.
// kRms: the row is RMS-normalized first (scale-free RMSNorm): the codes of x / rms
// equal the codes of x, so only the scale changes (scale / rms).
template <int CPT, bool kRms, bool kQ8 = false>  // kQ8: int8 codes, one byte per element (A8, §8 f4)
__global__ void __launch_bounds__(128) hq_none_kernel(const __half* __restrict__ x, int64_t K, int64_t ld_x,
                                                      float clip, uint8_t* __restrict__ q, int64_t ld_q,
                                                      float* __restrict__ scale) {
  __shared__ float red[4];
  __shared__ float red2[4];
  const int64_t row = blockIdx.x;
  const int nchunk = (int)(K >> 3);
  const __half* xr = x + row * ld_x;
  uint4 v[CPT];
  // independent accumulator chains (the row's reductions are on the critical path of the CTA)
  float am[4] = {0.f, 0.f, 0.f, 0.f};
  float2 sq[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = threadIdx.x + i * 128;
    if (c < nchunk) {
      v[i] = ldg_nc_v4(xr + (int64_t)c * 8);
      const __half2* h = reinterpret_cast<const __half2*>(&v[i]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(h[e]);
        am[e] = fmax_nan(am[e], fmax_nan(fabsf(f.x), fabsf(f.y)));
        if (kRms) sq[e & 1] = f2fma(f, f, sq[e & 1]);
      }
    }
  }
  float amax = fmax_nan(fmax_nan(am[0], am[1]), fmax_nan(am[2], am[3]));
  float ssq = (sq[0].x + sq[0].y) + (sq[1].x + sq[1].y);
  double norm = 1.0;
  if (kRms) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
    if ((threadIdx.x & 31) == 0) red2[threadIdx.x >> 5] = ssq;
  }
  amax = block_max<4>(amax, red);  // (its __syncthreads also publishes red2)
  if (kRms) {  // fp32 ("RMSNorm ... in FP32"); 1/rms carries ~1 ulp
    const float tot = (red2[0] + red2[1]) + (red2[2] + red2[3]);
    norm = (double)rsqrtf(tot / (float)K + 1e-5f);
  }
  float s, inv;
  row_scale(amax, norm, clip, s, inv, kQ8 ? 127.0 : 7.0);
  if (threadIdx.x == 0) scale[row] = s;
  uint8_t* qr = q + row * ld_q;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = threadIdx.x + i * 128;
    if (c < nchunk) {
      const __half2* h = reinterpret_cast<const __half2*>(&v[i]);
      if constexpr (kQ8) {
        uint32_t w[2] = {0u, 0u};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(h[e]);
          w[e >> 1] |= (((uint32_t)code_of<127>(f.x, inv) & 0xFFu) | (((uint32_t)code_of<127>(f.y, inv) & 0xFFu) << 8))
                       << (16 * (e & 1));
        }
        *reinterpret_cast<uint2*>(qr + (int64_t)c * 8) = make_uint2(w[0], w[1]);
      } else {
        uint32_t packed = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(h[e]);
          packed |= (nib(code_of(f.x, inv)) | (nib(code_of(f.y, inv)) << 4)) << (8 * e);
        }
        *reinterpret_cast<uint32_t*>(qr + (int64_t)c * 4) = packed;
      }
    }
  }
}

// ------------------------------------------------------------------ NONE, group-wise (§8 f3)
// Group-wise symmetric INT4 (group size 128): every run of G consecutive elements of a
// row gets its own scale.  Thread = one 8-element chunk; a group is G/8 consecutive lanes
// (8, 16 or 32), reduced with shuffles; scale [row][K/G].
template <int LPG, bool kQ8 = false>  // lanes per group = G / 8; kQ8: int8 codes, one per byte
__global__ void __launch_bounds__(128) hq_none_group_kernel(const __half* __restrict__ x, int64_t K, int64_t ld_x,
                                                            float clip, uint8_t* __restrict__ q, int64_t ld_q,
                                                            float* __restrict__ scale, int64_t ld_s) {
  const int64_t row = blockIdx.x;  // rows on x (up to 2^31 - 1), chunk blocks on y
  const int64_t c = (int64_t)blockIdx.y * 128 + threadIdx.x;  // chunk (all lanes of a group exist: K % G == 0)
  const bool ok = c < (K >> 3);
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (ok) v = ldg_nc_v4(x + row * ld_x + c * 8);
  const __half2* h = reinterpret_cast<const __half2*>(&v);
  float f[8];
  float am = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __half22float2(h[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
    am = fmax_nan(am, fmax_nan(fabsf(t.x), fabsf(t.y)));
  }
#pragma unroll
  for (int o = 1; o < LPG; o <<= 1) am = fmax_nan(am, __shfl_xor_sync(0xffffffffu, am, o));
  float s, inv;
  row_scale(am, 1.0, clip, s, inv);
  if (!ok) return;
  if ((threadIdx.x & (LPG - 1)) == 0) scale[row * ld_s + c / LPG] = s;
  if constexpr (kQ8) {
    uint32_t w[2] = {0u, 0u};
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e >> 2] |= ((uint32_t)code_of(f[e], inv) & 0xFFu) << (8 * (e & 3));
    *reinterpret_cast<uint2*>(q + row * ld_q + c * 8) = make_uint2(w[0], w[1]);
  } else {
    uint32_t packed = 0;
#pragma unroll
    for (int e = 0; e < 8; e += 2) packed |= (nib(code_of(f[e], inv)) | (nib(code_of(f[e + 1], inv)) << 4)) << (4 * e);
    *reinterpret_cast<uint32_t*>(q + row * ld_q + c * 4) = packed;
  }
}

// ------------------------------------------------------------------ ACROSS_HEADS
// Thread (p, g): column pair j = 2p, 2p+1 of head_dim (one float2), heads h = g*HPT + r.
// Lane = g + G * p_lo: the FWHT over r runs in registers on fp32x2 pairs (FADD2), over g
// with warp shuffles (G <= 2 for the Llama head counts: at most one shuffle stage).
template <int HPT, int G>
__global__ void __launch_bounds__(128) hq_heads_kernel(const __half* __restrict__ x, int64_t K, int64_t ld_x,
                                                       int head_dim, float clip, uint8_t* __restrict__ q,
                                                       int64_t ld_q, float* __restrict__ scale) {
  extern __shared__ __align__(16) uint8_t sh_bytes[];  // K/2 packed bytes + reduction scratch
  float* red = reinterpret_cast<float*>(sh_bytes + (K >> 1));
  const int64_t row = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const int p = (threadIdx.x / 32) * (32 / G) + lane / G;  // column pair index
  const int P2 = head_dim >> 1;
  const __half* xr = x + row * ld_x;
  float2 v[HPT];
  const bool active = p < P2;
#pragma unroll
  for (int r = 0; r < HPT; ++r) {
    const int h = g * HPT + r;
    v[r] = active ? __half22float2(__ldg(reinterpret_cast<const __half2*>(xr + (int64_t)h * head_dim + 2 * p)))
                  : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int st = 1; st < HPT; st <<= 1) {
#pragma unroll
    for (int r = 0; r < HPT; ++r) {
      if (!(r & st)) {
        const float2 a = v[r], b = v[r + st];
        v[r] = f2add(a, b);
        v[r + st] = f2sub(a, b);
      }
    }
  }
#pragma unroll
  for (int st = 1; st < G; st <<= 1) {
    const float sg = (g & st) ? -1.f : 1.f;
#pragma unroll
    for (int r = 0; r < HPT; ++r) {
      const float o0 = __shfl_xor_sync(0xffffffffu, v[r].x, st);
      const float o1 = __shfl_xor_sync(0xffffffffu, v[r].y, st);
      v[r] = f2fma(make_float2(sg, sg), v[r], make_float2(o0, o1));  // lower: v + o, upper: o - v
    }
  }
  float amax = 0.f;
#pragma unroll
  for (int r = 0; r < HPT; ++r) amax = fmax_nan(amax, fmax_nan(fabsf(v[r].x), fabsf(v[r].y)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const int nwarps = blockDim.x >> 5;
  if (lane == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = red[0];
  for (int w = 1; w < nwarps; ++w) amax = fmax_nan(amax, red[w]);
  const int n_h = (int)(K / head_dim);
  float s, inv;
  row_scale(amax, rsqrt((double)n_h), clip, s, inv);
  if (threadIdx.x == 0) scale[row] = s;
  if (active) {
#pragma unroll
    for (int r = 0; r < HPT; ++r) {
      const int h = g * HPT + r;
      sh_bytes[h * P2 + p] = inv != 0.f ? (uint8_t)quant_pair(v[r], inv) : (uint8_t)0;
    }
  }
  __syncthreads();
  const int nvec = (int)(K >> 5);  // 16-byte vectors of packed output
  uint8_t* qr = q + row * ld_q;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x)
    *reinterpret_cast<uint4*>(qr + (int64_t)i * 16) = reinterpret_cast<const uint4*>(sh_bytes)[i];
}

// Persistent variant (the bench path): each CTA streams rows; the fp16 row (2K bytes) is
// bulk-copied into a double-buffered smem slot two rows ahead, so loads are asynchronous
// and overlap the butterflies / quantization of the current row.
template <int HPT, int G>
#ifndef QR_HEADS_HPT
#define QR_HEADS_HPT 32
#endif
__global__ void __launch_bounds__(QR_HEADS_HPT == 32 ? 128 : 256, QR_HEADS_HPT == 32 ? 4 : 2) hq_heads_persist_kernel(const __half* __restrict__ x, int64_t M, int64_t K,
                                                               int64_t ld_x, int head_dim, float clip,
                                                               uint8_t* __restrict__ q, int64_t ld_q,
                                                               float* __restrict__ scale) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int row_bytes = (int)(2 * K);
  uint8_t* bufs = smem;                                                // [2][row_bytes]
  uint8_t* out = smem + 2 * row_bytes;                                 // K/2 packed bytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(out + (K >> 1));        // [2]
  float* red = reinterpret_cast<float*>(bars + 2);                     // [2][4]
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const int p = (threadIdx.x / 32) * (32 / G) + lane / G;
  const int P2 = head_dim >> 1;
  const bool active = p < P2;
  const int nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int64_t row, int b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[b])), "r"(row_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(bufs + b * row_bytes)),
        "l"(x + row * ld_x), "r"(row_bytes), "r"(smem_u32(&bars[b]))
        : "memory");
  };
  if (threadIdx.x == 0) {
    if ((int64_t)blockIdx.x < M) issue(blockIdx.x, 0);
    if ((int64_t)blockIdx.x + gridDim.x < M) issue(blockIdx.x + gridDim.x, 1);
  }
  const int n_h = (int)(K / head_dim);
  const double norm = rsqrt((double)n_h);
  int it = 0;
  for (int64_t row = blockIdx.x; row < M; row += gridDim.x, ++it) {
    const int b = it & 1;
    mbar_wait_sleep(&bars[b], (it >> 1) & 1);
    const __half* xr = reinterpret_cast<const __half*>(bufs + b * row_bytes);
    float2 v[HPT];
#pragma unroll
    for (int r = 0; r < HPT; ++r) {
      const int h = g * HPT + r;
      v[r] = active ? __half22float2(*reinterpret_cast<const __half2*>(xr + h * head_dim + 2 * p))
                    : make_float2(0.f, 0.f);
    }
    __syncthreads();  // buffer b fully read: refill it two rows ahead
    if (threadIdx.x == 0 && row + 2 * (int64_t)gridDim.x < M) issue(row + 2 * (int64_t)gridDim.x, b);
#pragma unroll
    for (int st = 1; st < HPT; st <<= 1) {
#pragma unroll
      for (int r = 0; r < HPT; ++r) {
        if (!(r & st)) {
          const float2 a = v[r], c = v[r + st];
          v[r] = f2add(a, c);
          v[r + st] = f2sub(a, c);
        }
      }
    }
#pragma unroll
    for (int st = 1; st < G; st <<= 1) {
      const float sg = (g & st) ? -1.f : 1.f;
#pragma unroll
      for (int r = 0; r < HPT; ++r) {
        const float o0 = __shfl_xor_sync(0xffffffffu, v[r].x, st);
        const float o1 = __shfl_xor_sync(0xffffffffu, v[r].y, st);
        v[r] = f2fma(make_float2(sg, sg), v[r], make_float2(o0, o1));
      }
    }
    float am[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < HPT; ++r) am[r & 3] = fmax_nan(am[r & 3], fmax_nan(fabsf(v[r].x), fabsf(v[r].y)));
    float amax = fmax_nan(fmax_nan(am[0], am[1]), fmax_nan(am[2], am[3]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) red[b * 4 + (threadIdx.x >> 5)] = amax;
    __syncthreads();
    amax = red[b * 4];
    for (int w = 1; w < nwarps; ++w) amax = fmax_nan(amax, red[b * 4 + w]);
    float sc, inv;
    row_scale(amax, norm, clip, sc, inv);
    if (threadIdx.x == 0) scale[row] = sc;
    if (active) {
#pragma unroll
      for (int r = 0; r < HPT; ++r) {
        const int h = g * HPT + r;
        out[h * P2 + p] = inv != 0.f ? (uint8_t)quant_pair(v[r], inv) : (uint8_t)0;
      }
    }
    __syncthreads();
    uint8_t* qr = q + row * ld_q;
    const int nvec = (int)(K >> 5);
    for (int i = threadIdx.x; i < nvec; i += blockDim.x)
      *reinterpret_cast<uint4*>(qr + (int64_t)i * 16) = reinterpret_cast<const uint4*>(out)[i];
  }
}

// ------------------------------------------------------------------ FULL
// One row per CTA, staged in shared memory: X (fp16, K) and Z (fp32, K).
//  1) copy x -> X (m > 1) or -> Z (m == 1);
//  2) m > 1: Z[a][:] = H_m X[a][:] for every chunk a with mma.sync.m16n8k16 (fp16 in, exact
//     +-1 products, fp32 accumulation) on 16-chunk groups;
//  3) H_{2^n} along a (stride m): radix-2^r passes, 2^r values per thread in registers;
//     the last pass also tracks amax;
//  4) scale, RNE codes, pack 8 codes per 32-bit store.
template <int MB>
struct BaseDims {
  static constexpr int KS = (MB + 15) / 16;
  static constexpr int NT = (MB + 7) / 8;
};

QR_DEVICE void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int MB>
QR_DEVICE void base_transform(const uint32_t* __restrict__ X32, float* __restrict__ Z, int P,
                              const uint32_t* __restrict__ bfrag) {
  constexpr int KS = BaseDims<MB>::KS;
  constexpr int NT = BaseDims<MB>::NT;
  constexpr int MW = MB / 2;  // 32-bit words per chunk
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int ngroups = (P + 15) / 16;
  for (int grp = warp; grp < ngroups; grp += nwarps) {
    const int a_lo = grp * 16 + gq, a_hi = a_lo + 8;
    uint32_t afr[KS][4];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int w0 = ks * 8 + t, w1 = w0 + 4;  // word index within the chunk
      afr[ks][0] = (a_lo < P && w0 < MW) ? X32[a_lo * MW + w0] : 0u;
      afr[ks][1] = (a_hi < P && w0 < MW) ? X32[a_hi * MW + w0] : 0u;
      afr[ks][2] = (a_lo < P && w1 < MW) ? X32[a_lo * MW + w1] : 0u;
      afr[ks][3] = (a_hi < P && w1 < MW) ? X32[a_hi * MW + w1] : 0u;
    }
#pragma unroll 1
    for (int nt = 0; nt < NT; ++nt) {
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint2 b = __ldg(reinterpret_cast<const uint2*>(bfrag) + ((ks * NT + nt) * 32 + lane));
        mma_16816(d, afr[ks], b.x, b.y);
      }
      const int b = nt * 8 + 2 * t;
      if (b < MB) {
        if (a_lo < P) *reinterpret_cast<float2*>(Z + a_lo * MB + b) = make_float2(d[0], d[1]);
        if (a_hi < P) *reinterpret_cast<float2*>(Z + a_hi * MB + b) = make_float2(d[2], d[3]);
      }
    }
  }
}

// One radix-R pass of the Walsh-Hadamard transform along a (stride m) on bits
// [sh, sh + log2 R) of a.  Returns the thread's running amax if kAmax.
template <int R, bool kAmax>
QR_DEVICE float fwht_pass(float* __restrict__ Z, int P, int m, int sh) {
  const int items = (P / R) * m;
  float amax = 0.f;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int b = it % m;
    const int rest = it / m;
    const int lo = rest & ((1 << sh) - 1);
    const int hi = rest >> sh;
    const int a0 = hi * (R << sh) + lo;
    float v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = Z[(a0 + (j << sh)) * m + b];
#pragma unroll
    for (int st = 1; st < R; st <<= 1) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (!(j & st)) {
          const float x0 = v[j], x1 = v[j + st];
          v[j] = x0 + x1;
          v[j + st] = x0 - x1;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      Z[(a0 + (j << sh)) * m + b] = v[j];
      if (kAmax) amax = fmax_nan(amax, fabsf(v[j]));
    }
  }
  return amax;
}

template <bool kAmax>
QR_DEVICE float fwht_pass_dyn(int r, float* Z, int P, int m, int sh) {
  switch (r) {
    case 1: return fwht_pass<2, kAmax>(Z, P, m, sh);
    case 2: return fwht_pass<4, kAmax>(Z, P, m, sh);
    case 3: return fwht_pass<8, kAmax>(Z, P, m, sh);
    case 4: return fwht_pass<16, kAmax>(Z, P, m, sh);
    default: return fwht_pass<32, kAmax>(Z, P, m, sh);
  }
}

// OUT: the output format of the quantizer stage — 0 = INT4 packed, one scale per row (a3);
// 1 = int8 codes, one scale per row (A8, §8 f4); 2 = INT4 packed, one scale per run of `group`
// consecutive elements (group-wise, §8 f3); 3 = the same one code per int8 byte (the
// group-wise GEMM's operand format).  MB == 1 with stride > 1 is ACROSS_HEADS: P = n_h heads of
// `stride` = head_dim elements, y = (H_{n_h} (x) I) z (the FWHT along a at stride head_dim).
template <int OUT>
QR_DEVICE void quantize_groups(const float* __restrict__ Z, int K, int group, double norm, float clip,
                               uint8_t* __restrict__ qr, float* __restrict__ sr) {
  constexpr bool kQ8 = OUT == 3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int per = group >> 5;  // 2, 4 or 8 elements per lane
  for (int g = warp; g < K / group; g += nwarps) {
    const int e0 = g * group + lane * per;
    float v[8];
    float am = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[j] = j < per ? Z[e0 + j] : 0.f;
      am = fmax_nan(am, fabsf(v[j]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) am = fmax_nan(am, __shfl_xor_sync(0xffffffffu, am, o));
    float s, inv;
    row_scale(am, norm, clip, s, inv);
    if (lane == 0) sr[g] = s;
    if constexpr (kQ8) {
      uint32_t w[2] = {0u, 0u};
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j >> 2] |= ((uint32_t)code_of(v[j], inv) & 0xFFu) << (8 * (j & 3));
      if (per == 8) *reinterpret_cast<uint2*>(qr + e0) = make_uint2(w[0], w[1]);
      else if (per == 4) *reinterpret_cast<uint32_t*>(qr + e0) = w[0];
      else *reinterpret_cast<uint16_t*>(qr + e0) = (uint16_t)w[0];
    } else {
      uint32_t packed = 0;
#pragma unroll
      for (int j = 0; j < 8; j += 2) packed |= (nib(code_of(v[j], inv)) | (nib(code_of(v[j + 1], inv)) << 4)) << (4 * j);
      if (per == 8) *reinterpret_cast<uint32_t*>(qr + e0 / 2) = packed;
      else if (per == 4) *reinterpret_cast<uint16_t*>(qr + e0 / 2) = (uint16_t)packed;
      else qr[e0 / 2] = (uint8_t)packed;
    }
  }
}

template <int MB, int OUT = 0>
__global__ void hq_full_kernel(const __half* __restrict__ x, int64_t ld_x, int P, int stride, float clip,
                               uint8_t* __restrict__ q, int64_t ld_q, float* __restrict__ scale, int64_t ld_s,
                               int group, const uint32_t* __restrict__ bfrag) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int m = MB > 1 ? MB : stride;
  const int K = P * m;
  float* Z = reinterpret_cast<float*>(smem);
  uint32_t* X32 = reinterpret_cast<uint32_t*>(smem + (size_t)K * 4);
  float* red = reinterpret_cast<float*>(smem + (size_t)K * 4 + (MB > 1 ? (size_t)K * 2 : 0));
  const int64_t row = blockIdx.x;
  const __half* xr = x + row * ld_x;
  // 1/sqrt of the transform's order: K for FULL, n_h for ACROSS_HEADS (reading Z5)
  const double norm = rsqrt((double)P * (double)MB);

  // 1) stage the row
  const int nvec = K >> 3;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    const uint4 v = ldg_nc_v4(xr + (int64_t)i * 8);
    if (MB > 1) {
      reinterpret_cast<uint4*>(X32)[i] = v;
    } else {
      const __half2* h = reinterpret_cast<const __half2*>(&v);
      float4 f0, f1;
      float2 t0 = __half22float2(h[0]), t1 = __half22float2(h[1]), t2 = __half22float2(h[2]),
             t3 = __half22float2(h[3]);
      f0 = make_float4(t0.x, t0.y, t1.x, t1.y);
      f1 = make_float4(t2.x, t2.y, t3.x, t3.y);
      reinterpret_cast<float4*>(Z)[2 * i] = f0;
      reinterpret_cast<float4*>(Z)[2 * i + 1] = f1;
    }
  }
  __syncthreads();
  // 2) H_m on tensor cores
  if (MB > 1) {
    base_transform<MB>(X32, Z, P, bfrag);
    __syncthreads();
  }
  // 3) H_{2^n} along a
  int nbits = 0;
  while ((1 << nbits) < P) ++nbits;
  const int npass = (nbits + 4) / 5;
  float amax = 0.f;
  int sh = 0;
  for (int ps = 0; ps < npass; ++ps) {
    const int r = (nbits - sh + (npass - ps) - 1) / (npass - ps);  // balanced split
    if (ps == npass - 1 && OUT < 2) amax = fwht_pass_dyn<true>(r, Z, P, m, sh);
    else fwht_pass_dyn<false>(r, Z, P, m, sh);
    sh += r;
    __syncthreads();
  }
  if constexpr (OUT >= 2) {  // group-wise: the transformed row is complete in Z
    quantize_groups<OUT>(Z, K, group, norm, clip, q + row * ld_q, scale + row * ld_s);
    return;
  }
  if (npass == 0) {  // P == 1: amax over the base transform output
    for (int i = threadIdx.x; i < K; i += blockDim.x) amax = fmax_nan(amax, fabsf(Z[i]));
  }
  // 4) scale + codes
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) amax = fmax_nan(amax, red[w]);
  float s, inv;
  row_scale(amax, norm, clip, s, inv, OUT == 1 ? 127.0 : 7.0);
  if (threadIdx.x == 0) scale[row] = s;
  uint8_t* qr = q + row * ld_q;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    const float4 f0 = reinterpret_cast<const float4*>(Z)[2 * i];
    const float4 f1 = reinterpret_cast<const float4*>(Z)[2 * i + 1];
    if constexpr (OUT == 1) {
      const float f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
      uint32_t w[2] = {0u, 0u};
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j >> 2] |= ((uint32_t)code_of<127>(f[j], inv) & 0xFFu) << (8 * (j & 3));
      *reinterpret_cast<uint2*>(qr + (int64_t)i * 8) = make_uint2(w[0], w[1]);
    } else {
      const uint32_t packed = nib(code_of(f0.x, inv)) | (nib(code_of(f0.y, inv)) << 4) |
                              (nib(code_of(f0.z, inv)) << 8) | (nib(code_of(f0.w, inv)) << 12) |
                              (nib(code_of(f1.x, inv)) << 16) | (nib(code_of(f1.y, inv)) << 20) |
                              (nib(code_of(f1.z, inv)) << 24) | (nib(code_of(f1.w, inv)) << 28);
      *reinterpret_cast<uint32_t*>(qr + (int64_t)i * 4) = packed;
    }
  }
}


// ------------------------------------------------------------------ FULL, K = 1024 x 28
// The bench / 70B down_proj width, K = 28672: i = a*28 + b (reading Z2); Sylvester H_1024 is
// the tensor product of H_2 over the 10 bits of a (Eq. 1), so its stages can run in any order.
// Persistent CTAs (one per SM) with two warp groups working on consecutive rows, so the
// tensor-core phase of row i+1 overlaps the quantization phase of row i.  Element i = a*28 + b
// (a < 1024, b < 28); y = (H_1024 (x) H_28) x.  The 10 bits of a are split so that no
// transform stage needs a warp shuffle:
//  * P1 (4 warps, 4 units per row each; unit = a-group ag of 128 a's x m-tile mt of 16 output
//    b's): H_28 on tensor cores (mma.sync m16n8k16: A = H_28 padded to 32, B = x^T, exact
//    +-1 x fp16 products, fp32 accumulation) over 16 n-tiles, then H over the 5 a-bits the
//    accumulator fragment keeps in registers (column bit j = a1, n-tile bits = a0, a4, a5, a6)
//    with FADD/FADD2.  B column n = g <-> a bits 1-3 (a stride of 2 rows = 28 words keeps the
//    fragment loads bank-conflict-free).  Results go to Z as fp32.
//  * P2 (14 warps): thread tp = c * 14 + bp owns P1-bit combination c and b-pair bp for the 32
//    combinations p2 of the remaining bits (lane bits t = a2, a3 and ag = a7..a9): 32 LDS.64,
//    releases Z, H_32 over p2 with FADD2, row amax (NaN-propagating), RNE codes with the magic
//    add, one packed byte per p2.
// Z layout: [p2 (32)][c (32) x b (28) + 8 pad] fp32 — P2 reads are contiguous per p2, and the
// 8-word pad spreads P1's four t-lanes over distinct banks.
#ifndef QR_F28_P1W
#define QR_F28_P1W 4
#endif
#ifdef QR_F28_PROF
__device__ unsigned long long g_f28_prof[148 * 8];  // per CTA: p1_wait_x, p1_wait_z, p1_total, p2_wait, p2_total
#endif
namespace f28 {
constexpr int MB = 28, P = 1024, K = MB * P;  // (M is the row count)
constexpr int P1_WARPS = QR_F28_P1W, P2_WARPS = 14, NT = (P1_WARPS + P2_WARPS) * 32;
constexpr int UNITS = 16 / P1_WARPS;  // P1 units per warp per row
constexpr int P2_THREADS = P2_WARPS * 32;                                      // 448 = 32 * 14
constexpr int XS_BYTES = K * 2;         // 57344 per row buffer, double-buffered
constexpr int ZP = 32 * MB + 8;         // floats per p2 slice (904)
constexpr int Z_BYTES = 32 * ZP * 4;    // 115712
constexpr size_t SMEM = 2 * XS_BYTES + Z_BYTES + 256;  // 230656 of the 232448 available
}  // namespace f28

QR_DEVICE void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __launch_bounds__(f28::NT, 1)  // 18 warps: at most 5 per SM sub-partition -> 96 registers
    hq_full28_kernel(const __half* __restrict__ x, int64_t M, int64_t ld_x, float clip, uint8_t* __restrict__ q,
                     int64_t ld_q, float* __restrict__ scale, const uint32_t* __restrict__ afrag) {
  using namespace f28;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* xs0 = smem;                                              // fp16 rows [2]
  float* Z = reinterpret_cast<float*>(smem + 2 * XS_BYTES);         // fp32 after phase 1
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * XS_BYTES + Z_BYTES);
  uint64_t* xs_full = bars;       // [2]
  uint64_t* z_full = bars + 2;
  uint64_t* z_empty = bars + 3;
  float* red = reinterpret_cast<float*>(bars + 4);  // [2][16]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&xs_full[0], 1);
    mbar_init(&xs_full[1], 1);
    mbar_init(z_full, P1_WARPS * 32);
    mbar_init(z_empty, P2_THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue_row = [&](int64_t row, int buf) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&xs_full[buf])),
                 "r"(XS_BYTES)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(xs0 + buf * XS_BYTES)),
        "l"(x + row * ld_x), "r"(XS_BYTES), "r"(smem_u32(&xs_full[buf]))
        : "memory");
  };

#ifdef QR_F28_PROF
  const long long t_start = clock64();
#endif
  if (warp < P1_WARPS) {
    // ======================= P1: bulk copy + H_28 (tensor cores) + H over 5 a-bits in registers
    const int g = lane >> 2, t = lane & 3;
    if (threadIdx.x == 0) {  // prefetch the first two rows
      if ((int64_t)blockIdx.x < M) issue_row(blockIdx.x, 0);
      if ((int64_t)blockIdx.x + gridDim.x < M) issue_row(blockIdx.x + gridDim.x, 1);
    }
    int it = 0;
    for (int64_t row = blockIdx.x; row < M; row += gridDim.x, ++it) {
      const int buf = it & 1;
      const uint32_t* xw = reinterpret_cast<const uint32_t*>(xs0 + buf * XS_BYTES);
#ifdef QR_F28_PROF
      const long long t0 = clock64();
#endif
      mbar_wait_sleep(&xs_full[buf], (it >> 1) & 1);
#ifdef QR_F28_PROF
      const long long t1 = clock64();
#endif
      mbar_wait_sleep(z_empty, (it & 1) ^ 1);
#ifdef QR_F28_PROF
      if (threadIdx.x == 0) {
        atomicAdd(&g_f28_prof[blockIdx.x * 8 + 0], (unsigned long long)(t1 - t0));
        atomicAdd(&g_f28_prof[blockIdx.x * 8 + 1], (unsigned long long)(clock64() - t1));
      }
#endif
#pragma unroll 1
      for (int u = 0; u < UNITS; ++u) {
        const int unit = warp * UNITS + u;  // 0..15
        const int ag = unit >> 1, mt = unit & 1;
        uint32_t ha[2][4];  // H_28 A fragments of this m-tile (2 k-steps x 4 regs)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(afrag) + ((mt * 2 + ks) * 32 + lane));
          ha[ks][0] = v.x;
          ha[ks][1] = v.y;
          ha[ks][2] = v.z;
          ha[ks][3] = v.w;
        }
        float2 d[16][2];  // [nt][h]: output b = 16 mt + g + 8 h; (j = 0, 1) in .x / .y
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
          // B column n = g: a = ag * 128 + (nt & 1) + 2 g + 16 (nt >> 1); k = input b
          const int a = ag * 128 + (nt & 1) + 2 * g + 16 * (nt >> 1);
          const uint32_t* xa = xw + a * (MB / 2) + t;
          const uint32_t b00 = xa[0], b01 = xa[4], b10 = xa[8];
          const uint32_t b11 = (t < 2) ? xa[12] : 0u;
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          mma_16816(acc, ha[0], b00, b01);
          mma_16816(acc, ha[1], b10, b11);
          // D column n = 2 t + j <-> a bits 1-3: j = a1 lives inside the register pair
          d[nt][0] = make_float2(acc[0] + acc[1], acc[0] - acc[1]);
          d[nt][1] = make_float2(acc[2] + acc[3], acc[2] - acc[3]);
        }
#pragma unroll
        for (int st = 1; st < 16; st <<= 1) {  // n-tile bits = a0, a4, a5, a6
#pragma unroll
          for (int nt = 0; nt < 16; ++nt) {
            if (!(nt & st)) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float2 uu = d[nt][h], vv = d[nt + st][h];
                d[nt][h] = f2add(uu, vv);
                d[nt + st][h] = f2sub(uu, vv);
              }
            }
          }
        }
        // Z[p2][c][b]: p2 = t | ag << 2 (a2, a3, a7..a9); c = a0 | j << 1 | (nt >> 1) << 2
        float* zt = Z + (t | (ag << 2)) * ZP + 16 * mt + g;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c0 = (nt & 1) | ((nt >> 1) << 2);
            if (16 * mt + 8 * h + g < MB) {
              zt[c0 * MB + 8 * h] = d[nt][h].x;
              zt[(c0 | 2) * MB + 8 * h] = d[nt][h].y;
            }
          }
      }
      mbar_arrive(z_full);
      named_bar(1, P1_WARPS * 32);  // every P1 thread is done reading xs[buf]
      if (threadIdx.x == 0 && row + 2 * (int64_t)gridDim.x < M) issue_row(row + 2 * (int64_t)gridDim.x, buf);
    }
#ifdef QR_F28_PROF
    if (threadIdx.x == 0) atomicAdd(&g_f28_prof[blockIdx.x * 8 + 2], (unsigned long long)(clock64() - t_start));
#endif
  } else {
    // ======================= P2: H_32 over p2, amax, codes, packed output
    const int tp = threadIdx.x - P1_WARPS * 32;  // 0..447 = c * 14 + bp
    const int w2 = warp - P1_WARPS;
    const int c = tp / 14, bp = tp - 14 * (tp / 14);
    // element a of (c, p2): a0 = c0, a1 = c1, a2..a3 = p2 & 3, a4..a6 = c >> 2, a7..a9 = p2 >> 2
    const int a_c = (c & 3) | ((c >> 2) << 4);
    int it = 0;
    for (int64_t row = blockIdx.x; row < M; row += gridDim.x, ++it) {
#ifdef QR_F28_PROF
      const long long t2 = clock64();
#endif
      mbar_wait_sleep(z_full, it & 1);
#ifdef QR_F28_PROF
      if (threadIdx.x == P1_WARPS * 32) atomicAdd(&g_f28_prof[blockIdx.x * 8 + 3], (unsigned long long)(clock64() - t2));
#endif
      float2 v[32];
      const float2* zp = reinterpret_cast<const float2*>(Z) + tp;  // (c * 28 + 2 bp) / 2 == tp
#pragma unroll
      for (int p2 = 0; p2 < 32; ++p2) v[p2] = zp[p2 * (ZP / 2)];
      mbar_arrive(z_empty);
#pragma unroll
      for (int st = 1; st < 32; st <<= 1) {
#pragma unroll
        for (int p2 = 0; p2 < 32; ++p2) {
          if (!(p2 & st)) {
            const float2 uu = v[p2], ww = v[p2 + st];
            v[p2] = f2add(uu, ww);
            v[p2 + st] = f2sub(uu, ww);
          }
        }
      }
      float am[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent max chains
#pragma unroll
      for (int p2 = 0; p2 < 32; ++p2)
        am[p2 & 3] = fmax_nan(am[p2 & 3], fmax_nan(fabsf(v[p2].x), fabsf(v[p2].y)));
      float amax = fmax_nan(fmax_nan(am[0], am[1]), fmax_nan(am[2], am[3]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (lane == 0) red[(it & 1) * 16 + w2] = amax;  // double-buffered: no barrier needed after the read
      named_bar(2, P2_THREADS);
      amax = red[(it & 1) * 16];
#pragma unroll
      for (int w = 1; w < P2_WARPS; ++w) amax = fmax_nan(amax, red[(it & 1) * 16 + w]);
      float s, inv;
      row_scale(amax, rsqrt((double)K), clip, s, inv);
      if (tp == 0) scale[row] = s;
      // byte of (a, b-pair) at a * 14 + bp
      uint8_t* qr = q + row * ld_q + a_c * (MB / 2) + bp;
      if (inv != 0.f) {
#pragma unroll
        for (int p2 = 0; p2 < 32; ++p2)
          qr[((p2 & 3) << 2 | (p2 >> 2) << 7) * (MB / 2)] = (uint8_t)quant_pair(v[p2], inv);
      } else {
#pragma unroll
        for (int p2 = 0; p2 < 32; ++p2) qr[((p2 & 3) << 2 | (p2 >> 2) << 7) * (MB / 2)] = 0;
      }
    }
#ifdef QR_F28_PROF
    if (threadIdx.x == P1_WARPS * 32) atomicAdd(&g_f28_prof[blockIdx.x * 8 + 4], (unsigned long long)(clock64() - t_start));
#endif
  }
}

}  // namespace hq

// ------------------------------------------------------------------ launchers

cudaError_t launch_hq_none(const void* x, int64_t M, int64_t K, int64_t ld_x, float clip, uint8_t* q,
                           int64_t ld_q, float* scale, cudaStream_t stream, bool rmsnorm) {
  const int64_t nchunk = K / 8;
  const int cpt = (int)((nchunk + 127) / 128);
  const dim3 grid((unsigned)M);
  const __half* xh = static_cast<const __half*>(x);
#define QR_NONE(C)                                                                               \
  do {                                                                                           \
    if (rmsnorm) hq::hq_none_kernel<C, true><<<grid, 128, 0, stream>>>(xh, K, ld_x, clip, q, ld_q, scale);  \
    else hq::hq_none_kernel<C, false><<<grid, 128, 0, stream>>>(xh, K, ld_x, clip, q, ld_q, scale);        \
  } while (0)
  if (cpt <= 1) QR_NONE(1);
  else if (cpt <= 2) QR_NONE(2);
  else if (cpt <= 4) QR_NONE(4);
  else if (cpt <= 8) QR_NONE(8);
  else if (cpt <= 16) QR_NONE(16);
  else QR_NONE(32);
#undef QR_NONE
  return cudaPeekAtLastError();
}

cudaError_t launch_hq_none_group(const void* x, int64_t M, int64_t K, int64_t ld_x, int group, float clip,
                                 uint8_t* q, int64_t ld_q, float* scale, int64_t ld_s, cudaStream_t stream, bool q8) {
  const dim3 grid((unsigned)M, (unsigned)((K / 8 + 127) / 128));
  const __half* xh = static_cast<const __half*>(x);
#define QR_G(L)                                                                                                \
  do {                                                                                                         \
    if (q8) hq::hq_none_group_kernel<L, true><<<grid, 128, 0, stream>>>(xh, K, ld_x, clip, q, ld_q, scale, ld_s); \
    else hq::hq_none_group_kernel<L, false><<<grid, 128, 0, stream>>>(xh, K, ld_x, clip, q, ld_q, scale, ld_s);  \
  } while (0)
  if (group == 64) QR_G(8);
  else if (group == 128) QR_G(16);
  else QR_G(32);
#undef QR_G
  return cudaPeekAtLastError();
}

cudaError_t launch_hq_none_q8(const void* x, int64_t M, int64_t K, int64_t ld_x, float clip, int8_t* q, int64_t ld_q,
                              float* scale, cudaStream_t stream, bool rmsnorm) {
  const int64_t nchunk = K / 8;
  const int cpt = (int)((nchunk + 127) / 128);
  const dim3 grid((unsigned)M);
  const __half* xh = static_cast<const __half*>(x);
  uint8_t* qb = reinterpret_cast<uint8_t*>(q);
#define QR_NONE8(C)                                                                                            \
  do {                                                                                                         \
    if (rmsnorm) hq::hq_none_kernel<C, true, true><<<grid, 128, 0, stream>>>(xh, K, ld_x, clip, qb, ld_q, scale);  \
    else hq::hq_none_kernel<C, false, true><<<grid, 128, 0, stream>>>(xh, K, ld_x, clip, qb, ld_q, scale);        \
  } while (0)
  if (cpt <= 1) QR_NONE8(1);
  else if (cpt <= 2) QR_NONE8(2);
  else if (cpt <= 4) QR_NONE8(4);
  else if (cpt <= 8) QR_NONE8(8);
  else if (cpt <= 16) QR_NONE8(16);
  else QR_NONE8(32);
#undef QR_NONE8
  return cudaPeekAtLastError();
}

int g_hq_heads_variant = 0;  // debug: 1 = the CUDA-core butterfly kernel for every width

cudaError_t launch_hq_heads(const void* x, int64_t M, int64_t K, int64_t ld_x, int head_dim, float clip,
                            uint8_t* q, int64_t ld_q, float* scale, cudaStream_t stream) {
  if (g_hq_heads_variant == 0 && hq_heads_tc_supported(K, head_dim))
    return launch_hq_heads_tc(x, M, K, ld_x, head_dim, clip, q, ld_q, scale, stream);
  const int n_h = (int)(K / head_dim);
  const int P2 = head_dim / 2;
  const __half* xh = static_cast<const __half*>(x);
  // G groups of heads per column pair; HPT = n_h / G heads per thread (<= 32 in registers)
#ifndef QR_HEADS_HPT
#define QR_HEADS_HPT 32
#endif
  const int G = n_h > QR_HEADS_HPT ? n_h / QR_HEADS_HPT : 1;
  if (G > 16) return cudaErrorInvalidValue;
  const int HPT = n_h / G;
  int threads = P2 * G;
  threads = ((threads + 31) / 32) * 32;
  if (threads > 256) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(2 * 2 * K) + (size_t)(K / 2) + 64;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // persistent CTAs with a fixed row interleave: launch exactly as many as are resident, or
  // the CTAs of a second partial wave would start late and run at reduced occupancy
#define QR_HEADS(H, GG)                                                                                         \
  do {                                                                                                          \
    cudaError_t ee = cudaFuncSetAttribute(hq::hq_heads_persist_kernel<H, GG>,                                   \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
    if (ee != cudaSuccess) return ee;                                                                           \
    int per_sm = 1;                                                                                             \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hq::hq_heads_persist_kernel<H, GG>, threads, smem);  \
    const int64_t want = (int64_t)nsm * (per_sm > 0 ? per_sm : 1);                                             \
    const dim3 grid((unsigned)(M < want ? M : want));                                                           \
    hq::hq_heads_persist_kernel<H, GG><<<grid, threads, smem, stream>>>(xh, M, K, ld_x, head_dim, clip, q, ld_q, \
                                                                        scale);                                 \
  } while (0)
  switch (G) {
    case 1:
      switch (HPT) {
        case 1: QR_HEADS(1, 1); break;
        case 2: QR_HEADS(2, 1); break;
        case 4: QR_HEADS(4, 1); break;
        case 8: QR_HEADS(8, 1); break;
        case 16: QR_HEADS(16, 1); break;
        default: QR_HEADS(32, 1); break;
      }
      break;
    case 2: QR_HEADS(QR_HEADS_HPT, 2); break;
    case 4: QR_HEADS(QR_HEADS_HPT, 4); break;
    case 8: QR_HEADS(QR_HEADS_HPT, 8); break;
    default: QR_HEADS(QR_HEADS_HPT, 16); break;
  }
#undef QR_HEADS
  return cudaPeekAtLastError();
}

// The smem kernel hq_full_kernel<MB, OUT> for one (MB, OUT): the row staged in shared memory,
// H_m by mma.sync, the Sylvester factor by radix passes (every width 2^n m, and ACROSS_HEADS
// when MB == 1 and stride = head_dim).
template <int MB, int OUT>
static cudaError_t launch_generic(const __half* xh, int64_t M, int64_t K, int64_t ld_x, int P, int stride, float clip,
                                  uint8_t* q, int64_t ld_q, float* scale, int64_t ld_s, int group,
                                  cudaStream_t stream) {
  const int threads = K >= 16384 ? 512 : 256;
  const size_t smem = (size_t)K * 4 + (MB > 1 ? (size_t)K * 2 : 0) + 32 * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(hq::hq_full_kernel<MB, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  hq::hq_full_kernel<MB, OUT><<<dim3((unsigned)M), threads, smem, stream>>>(
      xh, ld_x, P, stride, clip, q, ld_q, scale, ld_s, group, MB > 1 ? device_bfrag_table(MB) : nullptr);
  return cudaPeekAtLastError();
}

template <int OUT>
static cudaError_t launch_generic_m(const __half* xh, int64_t M, int64_t K, int64_t ld_x, int P, int m, int stride,
                                    float clip, uint8_t* q, int64_t ld_q, float* scale, int64_t ld_s, int group,
                                    cudaStream_t stream) {
  switch (m) {
    case 1: return launch_generic<1, OUT>(xh, M, K, ld_x, P, stride, clip, q, ld_q, scale, ld_s, group, stream);
    case 20: return launch_generic<20, OUT>(xh, M, K, ld_x, P, 20, clip, q, ld_q, scale, ld_s, group, stream);
    case 28: return launch_generic<28, OUT>(xh, M, K, ld_x, P, 28, clip, q, ld_q, scale, ld_s, group, stream);
    case 108: return launch_generic<108, OUT>(xh, M, K, ld_x, P, 108, clip, q, ld_q, scale, ld_s, group, stream);
    case 172: return launch_generic<172, OUT>(xh, M, K, ld_x, P, 172, clip, q, ld_q, scale, ld_s, group, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_hq_full(const void* x, int64_t M, int64_t K, int64_t ld_x, int pow2, int m, float clip,
                           uint8_t* q, int64_t ld_q, float* scale, cudaStream_t stream, int out, int group,
                           int64_t ld_s) {
  const __half* xh = static_cast<const __half*>(x);
  const bool q8 = out == 1;
  if (out <= 1 && g_hq_full_variant != 1) {  // the tcgen05 kernels of the model widths
    if (m == 28 && pow2 == 1024) return launch_hq_full28_tc(x, M, ld_x, clip, q, ld_q, scale, stream, q8);
    if (hq_full_small_tc_supported(pow2, m)) return launch_hq_full_small_tc(x, M, ld_x, pow2, m, clip, q, ld_q, scale, stream, q8);
    if (m == 172 && pow2 == 64) return launch_hq_full172_tc(x, M, ld_x, clip, q, ld_q, scale, stream, q8);
  }
  if (out == 0 && m == 28 && pow2 == 1024) {  // debug variant 1: the mma.sync FULL-28 kernel
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
      cudaError_t e = cudaFuncSetAttribute(hq::hq_full28_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)hq::f28::SMEM);
      if (e != cudaSuccess) return e;
      attr[dev & 63] = true;
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)(M < nsm ? M : nsm);
    hq::hq_full28_kernel<<<grid, hq::f28::NT, hq::f28::SMEM, stream>>>(xh, M, ld_x, clip, q, ld_q, scale,
                                                                      device_afrag28());
    return cudaPeekAtLastError();
  }
  switch (out) {
    case 0: return launch_generic_m<0>(xh, M, K, ld_x, pow2, m, 1, clip, q, ld_q, scale, 1, 0, stream);
    case 1: return launch_generic_m<1>(xh, M, K, ld_x, pow2, m, 1, clip, q, ld_q, scale, 1, 0, stream);
    case 2: return launch_generic_m<2>(xh, M, K, ld_x, pow2, m, 1, clip, q, ld_q, scale, ld_s, group, stream);
    case 3: return launch_generic_m<3>(xh, M, K, ld_x, pow2, m, 1, clip, q, ld_q, scale, ld_s, group, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_hq_heads_group(const void* x, int64_t M, int64_t K, int64_t ld_x, int head_dim, float clip,
                                  uint8_t* q, int64_t ld_q, float* scale, int64_t ld_s, int group, bool q8,
                                  cudaStream_t stream) {
  const __half* xh = static_cast<const __half*>(x);
  const int nh = (int)(K / head_dim);
  return q8 ? launch_generic<1, 3>(xh, M, K, ld_x, nh, head_dim, clip, q, ld_q, scale, ld_s, group, stream)
            : launch_generic<1, 2>(xh, M, K, ld_x, nh, head_dim, clip, q, ld_q, scale, ld_s, group, stream);
}

cudaError_t launch_hq_heads8(const void* x, int64_t M, int64_t K, int64_t ld_x, int head_dim, float clip, uint8_t* q,
                             int64_t ld_q, float* scale, cudaStream_t stream) {
  return launch_generic<1, 1>(static_cast<const __half*>(x), M, K, ld_x, (int)(K / head_dim), head_dim, clip, q, ld_q,
                              scale, 1, 0, stream);
}

}  // namespace qr

extern "C" void quarot_debug_hq_heads_variant(int32_t v) { qr::g_hq_heads_variant = v; }

#ifdef QR_F28_PROF
extern "C" void quarot_debug_f28_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, qr::hq::g_f28_prof, sizeof(unsigned long long) * 148 * 8);
  cudaMemset(nullptr, 0, 0);
  static unsigned long long zero[148 * 8] = {};
  cudaMemcpyToSymbol(qr::hq::g_f28_prof, zero, sizeof(zero));
}
#endif
