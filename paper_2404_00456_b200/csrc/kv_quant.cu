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

// Layout of the work: the (token, group) pairs of one launch are flattened,
// f = t * G + g with G = 2 n_kv + n_q groups per token (K heads, V heads, Q heads); each group
// of head_dim elements is held by LPG = head_dim / 32 consecutive lanes, 32 elements per lane
// (four 16-byte loads), so a warp processes 32 / LPG groups at once.  The Walsh-Hadamard
// butterflies run on bits 0-4 of the element index in registers (fp32x2 where the pairs line
// up) and on the log2(LPG) lane bits with shuffles.
constexpr int EPL = 32;  // elements per lane

QR_DEVICE void fwht32_regs(float (&v)[EPL]) {
#pragma unroll
  for (int j = 0; j < EPL; j += 2) {  // index bit 0
    const float a = v[j], b = v[j + 1];
    v[j] = a + b;
    v[j + 1] = a - b;
  }
#pragma unroll
  for (int st = 2; st < EPL; st <<= 1) {  // index bits 1..4, as fp32x2 pairs
#pragma unroll
    for (int j = 0; j < EPL; j += 2) {
      if (!(j & st)) {
        const float2 a = make_float2(v[j], v[j + 1]), b = make_float2(v[j + st], v[j + st + 1]);
        const float2 s = f2add(a, b), d = f2sub(a, b);
        v[j] = s.x;
        v[j + 1] = s.y;
        v[j + st] = d.x;
        v[j + st + 1] = d.y;
      }
    }
  }
}

template <int LPG>
QR_DEVICE void fwht_lanes(float (&v)[EPL], int sub) {
#pragma unroll
  for (int st = 1; st < LPG; st <<= 1) {
    const float sg = (sub & st) ? -1.f : 1.f;
#pragma unroll
    for (int j = 0; j < EPL; j += 2) {
      const float o0 = __shfl_xor_sync(0xffffffffu, v[j], st);
      const float o1 = __shfl_xor_sync(0xffffffffu, v[j + 1], st);
      const float2 r = f2fma(make_float2(sg, sg), make_float2(v[j], v[j + 1]), make_float2(o0, o1));
      v[j] = r.x;
      v[j + 1] = r.y;
    }
  }
}

template <int LPG>
QR_DEVICE float group_min(float x) {
#pragma unroll
  for (int o = 1; o < LPG; o <<= 1) x = fmin_nan(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
template <int LPG>
QR_DEVICE float group_max(float x) {
#pragma unroll
  for (int o = 1; o < LPG; o <<= 1) x = fmax_nan(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// RoPE parameters of the fused variant (kRope): position = (pos0 + t) % seq_len; the cos/sin
// table of a batch of `tpb` tokens is built in smem (fp64 -> fp32, as quarot_rope does)
struct RopeArgs {
  int64_t pos0;
  int seq_len;
  float theta;
  int tpb;
  // Append (P:858 routine 2): token t is sequence t's new token at row positions[t] of its
  // cache (s_max rows per sequence); its RoPE position is positions[t].  nullptr: Init.
  const int32_t* positions;
  int64_t s_max;
};

template <int LPG, bool kRope>
__global__ void __launch_bounds__(256) kv_quant_kernel(const __half* __restrict__ k, int64_t ld_k,
                                                       const __half* __restrict__ v, int64_t ld_v, __half* q,
                                                       int64_t ld_q, int64_t T, int n_kv, int n_q, uint32_t flags,
                                                       float clip, uint8_t* __restrict__ k_codes,
                                                       float* __restrict__ k_scale, uint8_t* __restrict__ k_zero,
                                                       uint8_t* __restrict__ v_codes, float* __restrict__ v_scale,
                                                       uint8_t* __restrict__ v_zero, RopeArgs ra) {
  extern __shared__ float2 rope_cs[];  // kRope: [tpb][HD / 2] (cos, sin)
  constexpr int HD = 32 * LPG;
  constexpr int GPW = 32 / LPG;  // groups per warp
  const int lane = threadIdx.x & 31;
  const int sub = lane % LPG;
  const int G = 2 * n_kv + n_q;
  const int64_t total = T * G;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const double rnorm = rsqrt((double)HD);
  // one (token, group) item per LPG lanes; warp-uniform control flow around the shuffles
  auto item = [&](const int64_t t, const int which, const bool ok, const int tt) {
    const bool is_k = which < n_kv, is_v = !is_k && which < 2 * n_kv, is_q = which >= 2 * n_kv;
    const __half* src = is_k ? k + t * ld_k + which * HD
                             : (is_v ? v + t * ld_v + (which - n_kv) * HD : q + t * ld_q + (which - 2 * n_kv) * HD);
    src += sub * EPL;
    float x[EPL];
    uint32_t raw[EPL / 2];  // the lane's 32 fp16 inputs as 16 packed words
    if (ok) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(src) + c);
        raw[4 * c] = u.x;
        raw[4 * c + 1] = u.y;
        raw[4 * c + 2] = u.z;
        raw[4 * c + 3] = u.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < EPL / 2; ++j) raw[j] = 0u;
    }
#pragma unroll
    for (int j = 0; j < EPL / 2; ++j) {
      const float2 ff = __half22float2(*reinterpret_cast<const __half2*>(&raw[j]));
      x[2 * j] = ff.x;
      x[2 * j + 1] = ff.y;
    }
    if constexpr (kRope) {
      // RoPE on K and Q (rotate-half pairs (i, i + HD/2)): the partner half lives
      // LPG/2 lanes away (exchanged as packed fp16 words); the result is rounded to fp16 as
      // the unfused path stores it (Z22)
      constexpr int HALF = HD / 2;
      const bool first = sub < LPG / 2;
      const float2* cs = rope_cs + tt * HALF + (sub % (LPG / 2)) * EPL;
      const bool do_rope = is_k || is_q;
#pragma unroll
      for (int j = 0; j < EPL / 2; ++j) {
        const uint32_t ow = __shfl_xor_sync(0xffffffffu, raw[j], LPG / 2);
        const float2 o = __half22float2(*reinterpret_cast<const __half2*>(&ow));
        const float4 c2 = *reinterpret_cast<const float4*>(cs + 2 * j);  // (cos, sin) of 2 pairs
        const float r0 = first ? rope_first(x[2 * j], o.x, c2.x, c2.y) : rope_second(o.x, x[2 * j], c2.x, c2.y);
        const float r1 =
            first ? rope_first(x[2 * j + 1], o.y, c2.z, c2.w) : rope_second(o.y, x[2 * j + 1], c2.z, c2.w);
        if (do_rope) {
          x[2 * j] = __half2float(__float2half_rn(r0));
          x[2 * j + 1] = __half2float(__float2half_rn(r1));
        }
      }
    }
    const bool rot = is_q || (is_k && (flags & 1u)) || (is_v && (flags & 2u));
    // rotation is group-uniform; shuffles need the whole warp, so every lane runs the
    // butterflies and non-rotated groups discard the result
    float y[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) y[j] = x[j];
    fwht32_regs(y);
    fwht_lanes<LPG>(y, sub);
    if (rot) {
#pragma unroll
      for (int j = 0; j < EPL; ++j) x[j] = y[j];
    }
    // ---- K / V: asymmetric 4-bit group quantization (Z14), scale / zero per group
    // NaN-propagating min / max in four independent chains (a serial 32-deep chain put the
    // reduction on the item's critical path); a NaN or +-Inf in the group makes mn or mx
    // non-finite, which is the group's non-finite test
    float mn4[4] = {x[0], x[1], x[2], x[3]}, mx4[4] = {x[0], x[1], x[2], x[3]};
#pragma unroll
    for (int j = 4; j < EPL; ++j) {
      mn4[j & 3] = fmin_nan(mn4[j & 3], x[j]);
      mx4[j & 3] = fmax_nan(mx4[j & 3], x[j]);
    }
    float mn = fmin_nan(fmin_nan(mn4[0], mn4[1]), fmin_nan(mn4[2], mn4[3]));
    float mx = fmax_nan(fmax_nan(mx4[0], mx4[1]), fmax_nan(mx4[2], mx4[3]));
    mn = group_min<LPG>(mn);
    mx = group_max<LPG>(mx);
    const bool finite = isfinite(mn) && isfinite(mx);
    if (!ok) return;
    if (!is_q) {
      const double norm = rot ? rnorm : 1.0;
      const double lo = (double)clip * (double)fminf(mn, 0.f) * norm;
      const double hi = (double)clip * (double)fmaxf(mx, 0.f) * norm;
      float s = 1.f, inv = 0.f;
      int z = 0;
      if (!finite) {
        s = __int_as_float(0x7fc00000);
      } else if (hi != lo) {
        s = (float)((hi - lo) / 15.0);
        const double zr = rint(-lo / (double)s);
        z = (int)(zr < 0.0 ? 0.0 : (zr > 15.0 ? 15.0 : zr));
        inv = (float)(norm / (double)s);
      }
      uint32_t w[4] = {0u, 0u, 0u, 0u};
      if (inv != 0.f) {
        const float zf = (float)z;
#pragma unroll
        for (int j = 0; j < EPL; j += 2) {
          // rne(x * inv) + z == rne(x * inv + z) (z integral); clamp to [0, 15]; magic-add RNE
          float2 m = f2fma(make_float2(x[j], x[j + 1]), make_float2(inv, inv), make_float2(zf, zf));
          m.x = fminf(fmaxf(m.x, 0.f), 15.f);
          m.y = fminf(fmaxf(m.y, 0.f), 15.f);
          m = f2add(m, make_float2(12582912.f, 12582912.f));
          const uint32_t byte = (__float_as_uint(m.x) & 0xFu) | ((__float_as_uint(m.y) & 0xFu) << 4);
          w[j >> 3] |= byte << (8 * ((j >> 1) & 3));
        }
      }
      const int h = is_k ? which : which - n_kv;
      const int64_t row = (kRope && ra.positions) ? t * ra.s_max + __ldg(ra.positions + t) : t;
      const int64_t gi = row * n_kv + h;
      uint8_t* codes = (is_k ? k_codes : v_codes) + gi * (HD / 2) + sub * (EPL / 2);
      *reinterpret_cast<uint4*>(codes) = make_uint4(w[0], w[1], w[2], w[3]);
      if (sub == 0) {
        (is_k ? k_scale : v_scale)[gi] = s;
        (is_k ? k_zero : v_zero)[gi] = (uint8_t)z;
      }
    } else {
      // ---- Q: rotated in place, rounded to fp16 (Eq. 13)
      const float rn = (float)rnorm;
      __half* dst = const_cast<__half*>(src);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 u;
        __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = __floats2half2_rn(x[8 * c + 2 * e] * rn, x[8 * c + 2 * e + 1] * rn);
        reinterpret_cast<uint4*>(dst)[c] = u;
      }
    }
  };
  if constexpr (!kRope) {
    for (int64_t f0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * GPW; f0 < total;
         f0 += nwarps * GPW) {
      const int64_t f = f0 + lane / LPG;
      const bool ok = f < total;
      const int64_t t = ok ? f / G : 0;
      item(t, ok ? (int)(f - t * G) : 0, ok, 0);
    }
  } else {
    // a block takes tpb tokens at a time: their cos/sin tables, then tpb * G items over its warps
    constexpr int HALF = HD / 2;
    const int units = ra.tpb * G;
    const int bw = (int)(blockDim.x >> 5), w = (int)(threadIdx.x >> 5);
    double* inv_freq = reinterpret_cast<double*>(rope_cs + 2 * ra.tpb * HALF);  // [HALF], after 2 tables
    for (int i = threadIdx.x; i < HALF; i += blockDim.x)
      inv_freq[i] = pow((double)ra.theta, -2.0 * (double)i / (double)HD);
    __syncthreads();
    int buf = 0;
    for (int64_t t0 = (int64_t)blockIdx.x * ra.tpb; t0 < T; t0 += (int64_t)gridDim.x * ra.tpb, buf ^= 1) {
      // double-buffered table: the batch before last is no longer read once this sync passes
      float2* tab = rope_cs + buf * ra.tpb * HALF;
      for (int i = threadIdx.x; i < ra.tpb * HALF; i += blockDim.x) {
        const int tt = i / HALF, ii = i - tt * HALF;
        const int64_t pos = ra.positions ? (t0 + tt < T ? (int64_t)__ldg(ra.positions + t0 + tt) : 0)
                                         : (ra.pos0 + t0 + tt) % ra.seq_len;
        double sn, cn;
        sincos((double)pos * inv_freq[ii], &sn, &cn);  // == pos * theta^(-2 ii / d), as quarot_rope
        tab[i] = make_float2((float)cn, (float)sn);
      }
      __syncthreads();
      for (int u0 = w * GPW; u0 < units; u0 += bw * GPW) {
        const int u = u0 + lane / LPG;
        const int tt = u < units ? u / G : 0;
        const bool ok = u < units && t0 + tt < T;
        item(t0 + tt, ok ? u - tt * G : 0, ok, tt + buf * ra.tpb);
      }
    }
  }
}

}  // namespace kvq

int g_kv_variant = 0;  // debug: 1 = the CUDA-core kernel for every shape

cudaError_t launch_kv_quant(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int n_kv,
                            int head_dim, void* q, int64_t ld_q, int n_q, uint32_t flags, float clip,
                            uint8_t* k_codes, float* k_scale, uint8_t* k_zero, uint8_t* v_codes, float* v_scale,
                            uint8_t* v_zero, cudaStream_t stream) {
  const int nq = q ? n_q : 0;
  const int64_t groups = T * (2 * (int64_t)n_kv + nq);
  if (groups == 0) return cudaSuccess;
  if (g_kv_variant == 0 && kv_tc_supported(n_kv, head_dim, nq, flags, nullptr))
    return launch_kv_tc(k, ld_k, v, ld_v, T, n_kv, q, ld_q, nq, clip, false, 0, 1, 0.f, k_codes, k_scale, k_zero,
                        v_codes, v_scale, v_zero, stream);
  const int threads = 256;
  const int lpg = head_dim / 32;
  const int64_t warps_needed = (groups + (32 / lpg) - 1) / (32 / lpg);
  int64_t blocks = (warps_needed + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const __half* kh = static_cast<const __half*>(k);
  const __half* vh = static_cast<const __half*>(v);
  __half* qh = static_cast<__half*>(q);
#define QR_KV(L)                                                                                                \
  kvq::kv_quant_kernel<L, false><<<(unsigned)blocks, threads, 0, stream>>>(kh, ld_k, vh, ld_v, qh, ld_q, T, n_kv,  \
                                                                          nq, flags, clip, k_codes, k_scale,      \
                                                                          k_zero, v_codes, v_scale, v_zero,       \
                                                                          kvq::RopeArgs{0, 1, 0.f, 0, nullptr, 0})
  if (head_dim == 64) QR_KV(2);
  else if (head_dim == 128) QR_KV(4);
  else QR_KV(8);
#undef QR_KV
  return cudaPeekAtLastError();
}

cudaError_t launch_kv_quant_rope(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int n_kv,
                                 int head_dim, void* q, int64_t ld_q, int n_q, uint32_t flags, float clip,
                                 int64_t pos0, int seq_len, float theta, uint8_t* k_codes, float* k_scale,
                                 uint8_t* k_zero, uint8_t* v_codes, float* v_scale, uint8_t* v_zero,
                                 cudaStream_t stream, const int32_t* positions, int64_t s_max) {
  const int nq = q ? n_q : 0;
  const int G = 2 * n_kv + nq;
  if (T == 0 || G == 0) return cudaSuccess;
  if (g_kv_variant == 0 && kv_tc_supported(n_kv, head_dim, nq, flags, positions))
    return launch_kv_tc(k, ld_k, v, ld_v, T, n_kv, q, ld_q, nq, clip, true, pos0, seq_len, theta, k_codes, k_scale,
                        k_zero, v_codes, v_scale, v_zero, stream);
  const int threads = 256;
  const int lpg = head_dim / 32;
  const int gpb = (threads / 32) * (32 / lpg);  // items one pass of the block covers
  // tokens per block batch: a whole number of passes when possible (G = 80, 64 items -> 4)
  int tpb = 1;
  while (tpb < 16 && (tpb * G) % gpb) tpb *= 2;
  if (tpb < 8 && T >= 8 * 148) tpb = 8;  // fewer table builds / barriers per item
  int64_t blocks = (T + tpb - 1) / tpb;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const size_t smem = (size_t)2 * tpb * (head_dim / 2) * sizeof(float2) + (head_dim / 2) * sizeof(double);
  const kvq::RopeArgs ra{pos0, seq_len, theta, tpb, positions, s_max};
  const __half* kh = static_cast<const __half*>(k);
  const __half* vh = static_cast<const __half*>(v);
  __half* qh = static_cast<__half*>(q);
#define QR_KVR(L)                                                                                              \
  kvq::kv_quant_kernel<L, true><<<(unsigned)blocks, threads, smem, stream>>>(kh, ld_k, vh, ld_v, qh, ld_q, T,    \
                                                                            n_kv, nq, flags, clip, k_codes,    \
                                                                            k_scale, k_zero, v_codes, v_scale, \
                                                                            v_zero, ra)
  if (head_dim == 64) QR_KVR(2);
  else if (head_dim == 128) QR_KVR(4);
  else QR_KVR(8);
#undef QR_KVR
  return cudaPeekAtLastError();
}

}  // namespace qr

extern "C" void quarot_debug_kv_variant(int32_t v) { qr::g_kv_variant = v; }
