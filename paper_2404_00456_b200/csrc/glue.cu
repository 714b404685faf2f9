// glue.cu — decoder-layer glue of SURVEY §8 row a8: RoPE and SwiGLU (RMSNorm is fused into
// the NONE quantizer, the residual add into the GEMM epilogue).
//
// RoPE ("Pos", Eqs. 10-12): Llama-2 rotate-half form, pair (i, i + d/2) rotated by
// pos * theta^(-2i/d).  One CTA iteration per token: the d/2 (cos, sin) values are computed once
// in double precision into smem and reused by every head of the token.
// SwiGLU (Fig. ffn_orig): act = fp16(fp16(silu(gate)) * up) over [gate | up] column halves.
#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace glue {

constexpr int MAX_HALF = 128;

__global__ void __launch_bounds__(256) rope_kernel(__half* __restrict__ x, int64_t T, int n_heads, int head_dim,
                                                   int64_t ld_x, int64_t pos0, int seq_len, float theta) {
  __shared__ float2 cs[MAX_HALF];
  const int half = head_dim >> 1;
  const int vec_per_head = half / 8;        // 8 pairs per work item (16-byte loads of each half)
  const int items = n_heads * vec_per_head;
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const int64_t pos = (pos0 + t) % seq_len;
    __syncthreads();  // previous token's table fully used
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
      const double a = (double)pos * pow((double)theta, -2.0 * (double)i / (double)head_dim);
      double sn, cn;
      sincos(a, &sn, &cn);
      cs[i] = make_float2((float)cn, (float)sn);
    }
    __syncthreads();
    __half* xt = x + t * ld_x;
    for (int w = threadIdx.x; w < items; w += blockDim.x) {
      const int h = w / vec_per_head, v = w - h * vec_per_head;
      __half* p1 = xt + h * head_dim + v * 8;
      __half* p2 = p1 + half;
      uint4 u1 = *reinterpret_cast<const uint4*>(p1);
      uint4 u2 = *reinterpret_cast<const uint4*>(p2);
      __half2* a1 = reinterpret_cast<__half2*>(&u1);
      __half2* a2 = reinterpret_cast<__half2*>(&u2);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x1 = __half22float2(a1[e]), x2 = __half22float2(a2[e]);
        const float2 c0 = cs[v * 8 + 2 * e], c1 = cs[v * 8 + 2 * e + 1];
        a1[e] = __floats2half2_rn(rope_first(x1.x, x2.x, c0.x, c0.y), rope_first(x1.y, x2.y, c1.x, c1.y));
        a2[e] = __floats2half2_rn(rope_second(x1.x, x2.x, c0.x, c0.y), rope_second(x1.y, x2.y, c1.x, c1.y));
      }
      *reinterpret_cast<uint4*>(p1) = u1;
      *reinterpret_cast<uint4*>(p2) = u2;
    }
  }
}

__global__ void __launch_bounds__(256) swiglu_kernel(const __half* __restrict__ gu, int64_t M, int64_t F,
                                                     int64_t ld_gu, __half* __restrict__ act, int64_t ld_act) {
  const int64_t vpr = F / 8;  // 16-byte vectors per row
  const int64_t total = M * vpr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vpr, c = (i - m * vpr) * 8;
    const uint4 gv = ldg_nc_v4(gu + m * ld_gu + c);
    const uint4 uv = ldg_nc_v4(gu + m * ld_gu + F + c);
    const __half2* g2 = reinterpret_cast<const __half2*>(&gv);
    const __half2* u2 = reinterpret_cast<const __half2*>(&uv);
    uint4 o;
    __half2* o2 = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 g = __half22float2(g2[e]), u = __half22float2(u2[e]);
      // the FP16 model's ops (reading Z23): fp16(silu(g)), then fp16(that * u)
      const float sx = __half2float(__float2half_rn(silu_f32(g.x)));
      const float sy = __half2float(__float2half_rn(silu_f32(g.y)));
      o2[e] = __floats2half2_rn(sx * u.x, sy * u.y);
    }
    *reinterpret_cast<uint4*>(act + m * ld_act + c) = o;
  }
}

}  // namespace glue

static int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

cudaError_t launch_rope(void* x, int64_t T, int n_heads, int head_dim, int64_t ld_x, int64_t pos0, int seq_len,
                        float theta, cudaStream_t stream) {
  if (T == 0) return cudaSuccess;
  const int64_t grid = T < (int64_t)sm_count() * 16 ? T : (int64_t)sm_count() * 16;
  glue::rope_kernel<<<(unsigned)grid, 256, 0, stream>>>(static_cast<__half*>(x), T, n_heads, head_dim, ld_x, pos0,
                                                        seq_len, theta);
  return cudaPeekAtLastError();
}

cudaError_t launch_swiglu(const void* gu, int64_t M, int64_t F, int64_t ld_gu, void* act, int64_t ld_act,
                          cudaStream_t stream) {
  if (M == 0) return cudaSuccess;
  const int64_t total = M * (F / 8);
  int64_t grid = (total + 255) / 256;
  if (grid > (int64_t)sm_count() * 8) grid = (int64_t)sm_count() * 8;
  glue::swiglu_kernel<<<(unsigned)grid, 256, 0, stream>>>(static_cast<const __half*>(gu), M, F, ld_gu,
                                                          static_cast<__half*>(act), ld_act);
  return cudaPeekAtLastError();
}

}  // namespace qr
