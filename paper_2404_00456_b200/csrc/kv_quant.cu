// kv_quant.cu — rows a6 + a7 of the QuaRot hot path: quantized KV-cache "Init".
//
//  * Stage 1d (Eqs. 13-14): post-RoPE keys and queries are rotated head-wise,
//    k_h <- H^_{d_h} k_h, q_h <- H^_{d_h} q_h, so attention scores are unchanged.
//  * Stage 2c / Setup: the cache is quantized asymmetrically to 4 bits
//    with group size 128 (= head_dim) and clip ratio 0.95.
//
// One warp per (token, head, tensor) group; each lane holds E = head_dim/32 consecutive
// elements.  The Walsh-Hadamard butterflies run in registers over the low log2(E) index bits
// and with warp shuffles over the 5 lane bits.  V is rotated only if flags bit1 is set
// (the paper fuses V's rotation into W_v).
#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace kvq {

QR_DEVICE float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
QR_DEVICE float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int E>
QR_DEVICE void fwht_warp(float (&v)[E], int lane) {
#pragma unroll
  for (int st = 1; st < E; st <<= 1) {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (!(j & st)) {
        const float a = v[j], b = v[j + st];
        v[j] = a + b;
        v[j + st] = a - b;
      }
    }
  }
#pragma unroll
  for (int st = 1; st < 32; st <<= 1) {
    const bool upper = (lane & st) != 0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const float o = __shfl_xor_sync(0xffffffffu, v[j], st);
      v[j] = upper ? (o - v[j]) : (v[j] + o);
    }
  }
}

template <int E>
QR_DEVICE void load_half(const __half* p, float (&v)[E]) {
  if constexpr (E == 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h[e]);
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
  } else if constexpr (E == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float2 f = __half22float2(h[e]);
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
  } else {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(p));
    v[0] = f.x;
    v[1] = f.y;
  }
}

// Asymmetric 4-bit quantization of one group held by the warp (unnormalized values v,
// true values = v * norm).  Writes E/2 packed bytes per lane, scale and zero by lane 0.
template <int E>
QR_DEVICE void quant_group(const float (&v)[E], double norm, float clip, int lane, uint8_t* codes,
                           float* scale_out, uint8_t* zero_out) {
  float mn = v[0], mx = v[0];
  bool finite = true;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    mn = fminf(mn, v[j]);
    mx = fmaxf(mx, v[j]);
    finite = finite && isfinite(v[j]);
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  finite = __all_sync(0xffffffffu, finite);
  const double lo = (double)clip * (double)fminf(mn, 0.f) * norm;
  const double hi = (double)clip * (double)fmaxf(mx, 0.f) * norm;
  float s;
  int z;
  float inv;
  if (!finite) {
    s = __int_as_float(0x7fc00000);
    z = 0;
    inv = 0.f;
  } else if (hi == lo) {
    s = 1.f;
    z = 0;
    inv = 0.f;
  } else {
    s = (float)((hi - lo) / 15.0);
    const double zr = rint(-lo / (double)s);
    z = (int)(zr < 0.0 ? 0.0 : (zr > 15.0 ? 15.0 : zr));
    inv = (float)(norm / (double)s);
  }
  uint32_t packed = 0;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    int c = __float2int_rn(v[j] * inv) + z;
    c = c < 0 ? 0 : (c > 15 ? 15 : c);
    if (inv == 0.f) c = 0;
    packed |= (uint32_t)c << (4 * j);
  }
  if constexpr (E == 8) {
    *reinterpret_cast<uint32_t*>(codes + lane * 4) = packed;
  } else if constexpr (E == 4) {
    *reinterpret_cast<uint16_t*>(codes + lane * 2) = (uint16_t)packed;
  } else {
    codes[lane] = (uint8_t)packed;
  }
  if (lane == 0) {
    *scale_out = s;
    *zero_out = (uint8_t)z;
  }
}

template <int E>
__global__ void kv_quant_kernel(const __half* __restrict__ k, int64_t ld_k, const __half* __restrict__ v,
                                int64_t ld_v, __half* q, int64_t ld_q, int64_t T, int n_kv, int n_q, uint32_t flags, float clip, uint8_t* __restrict__ k_codes,
                                float* __restrict__ k_scale, uint8_t* __restrict__ k_zero,
                                uint8_t* __restrict__ v_codes, float* __restrict__ v_scale,
                                uint8_t* __restrict__ v_zero) {
  constexpr int HD = 32 * E;
  const int lane = threadIdx.x & 31;
  const int64_t per_tok = 2 * (int64_t)n_kv + n_q;
  const int64_t total = T * per_tok;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  const double rnorm = rsqrt((double)HD);
  for (int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); task < total; task += wstride) {
    const int64_t t = task / per_tok;
    const int which = (int)(task - t * per_tok);
    float x[E];
    if (which < 2 * n_kv) {
      const bool is_k = which < n_kv;
      const int h = is_k ? which : which - n_kv;
      const int64_t g = t * n_kv + h;
      load_half<E>(is_k ? (k + t * ld_k + h * HD + lane * E) : (v + t * ld_v + h * HD + lane * E), x);
      const bool rot = is_k ? (flags & 1u) : (flags & 2u);
      if (rot) fwht_warp<E>(x, lane);
      if (is_k)
        quant_group<E>(x, rot ? rnorm : 1.0, clip, lane, k_codes + g * (HD / 2), k_scale + g, k_zero + g);
      else
        quant_group<E>(x, rot ? rnorm : 1.0, clip, lane, v_codes + g * (HD / 2), v_scale + g, v_zero + g);
    } else {
      const int h = which - 2 * n_kv;
      __half* qp = q + t * ld_q + h * HD + lane * E;
      load_half<E>(qp, x);
      fwht_warp<E>(x, lane);
      const float rn = (float)rnorm;
      __half2 out[E / 2];
#pragma unroll
      for (int e = 0; e < E / 2; ++e) {
        // product in fp64 then one rounding to fp16 would need fp64; fp32 product
        // (|err| <= 2^-24 relative) then RNE to fp16 matches the oracle's fp16(H^ q) except
        // at rare fp16 ties.
        out[e] = __floats2half2_rn(x[2 * e] * rn, x[2 * e + 1] * rn);
      }
      if constexpr (E == 8) *reinterpret_cast<uint4*>(qp) = *reinterpret_cast<uint4*>(out);
      else if constexpr (E == 4) *reinterpret_cast<uint2*>(qp) = *reinterpret_cast<uint2*>(out);
      else *reinterpret_cast<__half2*>(qp) = out[0];
    }
  }
}

}  // namespace kvq

cudaError_t launch_kv_quant(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int n_kv,
                            int head_dim, void* q, int64_t ld_q, int n_q, uint32_t flags, float clip, uint8_t* k_codes, float* k_scale, uint8_t* k_zero,
                            uint8_t* v_codes, float* v_scale, uint8_t* v_zero, cudaStream_t stream) {
  const int64_t groups = T * (2 * (int64_t)n_kv + (q ? n_q : 0));
  if (groups == 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (groups + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const int nq = q ? n_q : 0;
  const __half* kh = static_cast<const __half*>(k);
  const __half* vh = static_cast<const __half*>(v);
  __half* qh = static_cast<__half*>(q);
#define QR_KV(E)                                                                                              \
  kvq::kv_quant_kernel<E><<<(unsigned)blocks, threads, 0, stream>>>(kh, ld_k, vh, ld_v, qh, ld_q, T, n_kv, nq, flags, clip,  \
                                                                     k_codes, k_scale, k_zero, v_codes,     \
                                                                     v_scale, v_zero)
  if (head_dim == 64) QR_KV(2);
  else if (head_dim == 128) QR_KV(4);
  else QR_KV(8);
#undef QR_KV
  return cudaPeekAtLastError();
}

}  // namespace qr
