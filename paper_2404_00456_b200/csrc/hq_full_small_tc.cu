// hq_full_small_tc.cu — rows a1 + a3 for the Llama-2-13B widths on the tcgen05
// path: K = 128 x 108 (FFN 13824) and 256 x 20 (hidden 5120), element i = a*m + b (reading Z2).
//
// Split a = a_hi * 2^L + a_lo so that the contraction j = a_lo*m + b has a 16-byte-multiple
// pitch (216 / 80 elements = 432 / 160 B) and a_hi leaves 64 columns:
//     y[a'_hi*J + j'] = sum_{a_hi} H_64[a'_hi][a_hi] D[j'][a_hi],
//     D[j'][a_hi] = sum_j (H_{2^L} (x) H_m)[j'][j] x[a_hi*J + j],   J = 2^L m.
// The row is TMA'd by a 3-D map [row][a_hi][j] straight into the K-major SW128 operand (j past J
// zero-filled); D = MT M=128 kind::f16 MMAs (N = 64, K = 64 * KATOMS) into TMEM; H_64 over the 64
// columns in registers exactly as hq_full172_tc.cu (bits 1-5 packed, bit 0 within the pair);
// 16 epilogue warps in groups of 4 * MT (one row per group at a time).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace hqs {

constexpr int NA = 64;  // a_hi columns
// producer warps at the highest ids (the schedulers prefer them), as in the other FULL kernels
#ifndef QR_SMALL_PROD_HIGH
#define QR_SMALL_PROD_HIGH 1
#endif
constexpr int NUM_EPI = 16, EPI_WARP0 = QR_SMALL_PROD_HIGH ? 0 : 4, CTL_WARP0 = QR_SMALL_PROD_HIGH ? 16 : 0;
constexpr int TMA_WARP = CTL_WARP0, MMA_WARP = CTL_WARP0 + 1;
constexpr int NUM_THREADS = (4 + NUM_EPI) * 32;  // 640
constexpr uint32_t TMEM_COLS = 512;

template <int MB, int LLO>
struct Cfg {
  static constexpr int J = MB << LLO;
  static constexpr int P = NA << LLO;
  static constexpr int K = MB * P;
  static constexpr int KATOMS = (J + 63) / 64;
  static constexpr int MT = (J + 127) / 128;
  static constexpr int A_BYTES = MT * KATOMS * 16384;
  static constexpr int B_BYTES = KATOMS * NA * 128;
  static constexpr int STAGES_FIT = (232448 - 1024 - 512 - A_BYTES) / B_BYTES;
  static constexpr int STAGES = STAGES_FIT > 4 ? 4 : STAGES_FIT;
  static constexpr size_t SMEM = 1024 + (size_t)A_BYTES + (size_t)STAGES * B_BYTES + 512;
  static constexpr int GW = 4 * MT;         // epilogue warps per row group
  static constexpr int NG = NUM_EPI / GW;   // row groups
  static constexpr int TBUF = (int)(TMEM_COLS / (MT * NA));
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(NA >> 3) << 17) | ((128u >> 4) << 24);
  static_assert(STAGES >= 2 && SMEM <= 232448, "smem");
  static_assert(TBUF >= 2 * NG, "TMEM buffers per group");
};

QR_DEVICE void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(id), "r"(acc));
}
QR_DEVICE void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
QR_DEVICE bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(p));
  return p != 0;
}
QR_DEVICE void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
QR_DEVICE void bfly(float2& u, float2& v) {
  const float2 s = f2add(u, v), d = f2sub(u, v);
  u = s;
  v = d;
}
QR_DEVICE uint32_t code_word(float2 a, float2 b, float inv) {
  const float2 i2 = make_float2(inv, inv), mg = make_float2(12582912.f, 12582912.f);
  const float2 ma = f2fma(a, i2, mg), mb = f2fma(b, i2, mg);
  uint32_t lo = __byte_perm(__float_as_uint(ma.x), __float_as_uint(ma.y), 0x5410);
  uint32_t hi = __byte_perm(__float_as_uint(mb.x), __float_as_uint(mb.y), 0x5410);
  lo = __vmaxs2(__vmins2(lo, 0x00070007u), 0xFFF9FFF9u);
  hi = __vmaxs2(__vmins2(hi, 0x00070007u), 0xFFF9FFF9u);
  return __byte_perm(lo, hi, 0x6420);
}

template <int MB, int LLO, bool kQ8>  // kQ8: int8 codes in [-127, 127], one byte per element (§8 f4)
__global__ void __launch_bounds__(NUM_THREADS, 1)
    hq_full_small_tc_kernel(const __grid_constant__ CUtensorMap tmX, int64_t M, float clip, uint8_t* __restrict__ q,
                            int64_t ld_q, float* __restrict__ scale, const uint4* __restrict__ a_img) {
  using C = Cfg<MB, LLO>;
  constexpr int J = C::J, K = C::K, MT = C::MT, KATOMS = C::KATOMS, STAGES = C::STAGES, GW = C::GW, NG = C::NG,
                TBUF = C::TBUF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* t_full = empty + STAGES;  // [TBUF]
  uint64_t* t_empty = t_full + TBUF;  // [TBUF]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + TBUF);
  __shared__ float red[4][2][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < C::A_BYTES / 16; i += NUM_THREADS) reinterpret_cast<uint4*>(sA)[i] = __ldg(a_img + i);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < TBUF; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], GW);
    }
    fence_barrier_init();
  }
  if (warp == MMA_WARP) {
    tmem_alloc(tmem_holder, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int64_t nrows = M > (int64_t)blockIdx.x ? (M - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;

  if (warp >= CTL_WARP0 && warp < CTL_WARP0 + 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");  // 128 x 56 + 512 x 104 <= 640 x 96
    if (warp == TMA_WARP) {
      if (lane == 0) {
        for (int64_t it = 0; it < nrows; ++it) {
          const int s = (int)(it % STAGES);
          mbar_wait_sleep(&empty[s], (uint32_t)((it / STAGES) & 1) ^ 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                       "r"(C::B_BYTES)
                       : "memory");
          const int row = (int)((int64_t)blockIdx.x + it * gridDim.x);
          const uint32_t dst = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
          for (int t = 0; t < KATOMS; ++t) tma_load_3d(dst + t * NA * 128, &tmX, 64 * t, 0, row, &full[s]);
        }
      }
    } else if (warp == MMA_WARP) {
      const uint32_t sa = smem_u32(sA), sb = smem_u32(sB);
      for (int64_t it = 0; it < nrows; ++it) {
        const int s = (int)(it % STAGES), tb = (int)(it % TBUF);
        mbar_wait_sleep(&t_empty[tb], (uint32_t)((it / TBUF) & 1) ^ 1u);
        mbar_wait_sleep(&full[s], (uint32_t)((it / STAGES) & 1));
        tc_fence_after();
        const uint64_t b_desc = umma_desc_sw128(sb + (uint32_t)(s * C::B_BYTES));
        const uint32_t d0 = tmem_base + (uint32_t)(tb * MT * NA);
        if (elect_one()) {
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const uint64_t a_desc = umma_desc_sw128(sa + (uint32_t)(mt * KATOMS * 16384));
#pragma unroll
            for (int kk = 0; kk < KATOMS * 4; ++kk) {  // atom kk/4 (A: +16 KB, B: +8 KB), +32 B per K = 16
              const uint64_t koff = (uint64_t)(2 * (kk & 3));
              mma_f16(d0 + (uint32_t)(mt * NA), a_desc + (uint64_t)((kk >> 2) * (16384 >> 4)) + koff,
                      b_desc + (uint64_t)((kk >> 2) * (NA * 128 >> 4)) + koff, C::IDESC, kk > 0 ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          mma_commit(&t_full[tb]);
        }
        __syncwarp();
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
    const int e = warp - EPI_WARP0;  // 0..15
    const int g = e / GW;            // row group
    const int qd = warp & 3;         // TMEM lane quarter
    const int mh = (e % GW) >> 2;    // M-tile
    const int jp = mh * 128 + qd * 32 + lane;  // output j'
    const bool warp_ok = mh * 128 + qd * 32 < J;
    const bool lane_ok = jp < J;
    const bool odd = (lane & 1) != 0;
    const uint32_t t_lane = tmem_base + ((uint32_t)(qd * 32) << 16) + (uint32_t)(mh * NA);
    const float norm_f = (float)rsqrt((double)K);
    const float c0 = (float)((double)clip * rsqrt((double)K) / (kQ8 ? 127.0 : 7.0));
    const uint32_t sh_keep = odd ? 4u : 0u, sh_recv = odd ? 0u : 4u;
    const uint32_t keep_mask = odd ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
    // byte (a_hi, p = j'/2) at a_hi * J/2 + p; even lane writes a_hi < 32, odd lane a_hi >= 32
    uint8_t* const qlane = q + (jp >> 1) + (int64_t)(odd ? 32 : 0) * (J / 2);
    for (int64_t it = g; it < nrows; it += NG) {
      const int tb = (int)(it % TBUF), pb = (int)((it / NG) & 1);
      const int64_t row = (int64_t)blockIdx.x + it * gridDim.x;
      mbar_wait_sleep(&t_full[tb], (uint32_t)((it / TBUF) & 1));
      tc_fence_after();
      float2 v[32];
      float amax = 0.f;
      if (warp_ok) {
        uint32_t r[2][32];
        QR_TMEM_LD32(t_lane + (uint32_t)(tb * MT * NA), r[0]);
        QR_TMEM_LD32(t_lane + (uint32_t)(tb * MT * NA + 32), r[1]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          v[c] = make_float2(__uint_as_float(r[0][2 * c]), __uint_as_float(r[0][2 * c + 1]));
          v[16 + c] = make_float2(__uint_as_float(r[1][2 * c]), __uint_as_float(r[1][2 * c + 1]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[tb]);
      if (warp_ok) {
#pragma unroll
        for (int st = 1; st < 32; st <<= 1)  // a bits 1-5
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (!(c & st)) bfly(v[c], v[c + st]);
        float am[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 32; ++c) {  // a bit 0: within the register pair
          v[c] = pair_bfly(v[c]);
          am[c & 3] = fmax_nan(am[c & 3], fmax_nan(fabsf(v[c].x), fabsf(v[c].y)));
        }
        amax = lane_ok ? fmax_nan(fmax_nan(am[0], am[1]), fmax_nan(am[2], am[3])) : 0.f;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (lane == 0) red[g][pb][e % GW] = amax;
      bar_named(1 + g, GW * 32);
      amax = red[g][pb][0];
#pragma unroll
      for (int w = 1; w < GW; ++w) amax = fmax_nan(amax, red[g][pb][w]);
      float sc = 1.f, inv = 0.f;
      if (!isfinite(amax)) {
        sc = __int_as_float(0x7fc00000);
      } else if (amax != 0.f) {
        sc = c0 * amax;
        inv = __fdiv_rn(norm_f, sc);
      }
      if (e == g * GW && lane == 0) scale[row] = sc;
      if (!warp_ok) continue;
      if (inv == 0.f) {
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = make_float2(0.f, 0.f);
      }
      if constexpr (kQ8) {  // element (a, j') at byte a * J + j': a warp store covers 32 bytes
        if (lane_ok) {
          int8_t* const q8 = reinterpret_cast<int8_t*>(q) + row * ld_q + jp;
#pragma unroll
          for (int c = 0; c < 32; ++c) {  // v[c] = (a = 2c, 2c + 1)
            const float2 mq = f2fma(v[c], make_float2(inv, inv), make_float2(12582912.f, 12582912.f));
            const uint32_t w = __vmaxs2(__vmins2(__byte_perm(__float_as_uint(mq.x), __float_as_uint(mq.y), 0x5410),
                                                 0x007F007Fu), 0xFF81FF81u);
            q8[(int64_t)(2 * c) * J] = (int8_t)(w & 0xFFu);
            q8[(int64_t)(2 * c + 1) * J] = (int8_t)((w >> 16) & 0xFFu);
          }
        }
        continue;
      }
      uint32_t out[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {  // codes of a = 4m..4m+3 (even lane keeps) / 32 + 4m.. (odd)
        const uint32_t w0 = code_word(v[2 * m], v[2 * m + 1], inv);
        const uint32_t w1 = code_word(v[16 + 2 * m], v[16 + 2 * m + 1], inv);
        const uint32_t got = __shfl_xor_sync(0xffffffffu, odd ? w0 : w1, 1);
        const uint32_t keep = odd ? w1 : w0;
        out[m] = ((keep << sh_keep) & keep_mask) | ((got << sh_recv) & ~keep_mask);
      }
      if (lane_ok) {
        uint8_t* const qr = qlane + row * ld_q;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          uint8_t* dst = qr + (int64_t)(4 * m) * (J / 2);
          const uint32_t o = out[m];
          dst[0] = (uint8_t)o;
          dst[J / 2] = (uint8_t)(o >> 8);
          dst[J] = (uint8_t)(o >> 16);
          dst[3 * J / 2] = (uint8_t)(o >> 24);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace hqs

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_small() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult res;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &res) == cudaSuccess &&
        res == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// (H_{2^L} (x) H_m)[j'][j] (j' = a'_lo*m + b', j = a_lo*m + b; row i of H dotted with x, Z4),
// zero-padded to MT*128 x KATOMS*64 as [M-tile][atom][128 rows][128 B] K-major SW128 images
template <int MB, int LLO>
std::vector<uint16_t> a_image_small(const int8_t* h) {
  using C = hqs::Cfg<MB, LLO>;
  std::vector<uint16_t> img(C::A_BYTES / 2, 0);
  for (int m = 0; m < C::MT * 128; ++m)
    for (int k = 0; k < C::KATOMS * 64; ++k) {
      int v = 0;
      if (m < C::J && k < C::J) {
        const int alo_o = m / MB, bo = m % MB, alo_i = k / MB, bi = k % MB;
        v = ((__builtin_popcount(alo_o & alo_i) & 1) ? -1 : 1) * h[bo * MB + bi];
      }
      const int mt = m >> 7, r = m & 127, kc = k / 64, c = (k % 64) / 8, within = k % 8;
      const size_t off = (size_t)(mt * C::KATOMS + kc) * 16384 + (size_t)(r >> 3) * 1024 + (size_t)(r & 7) * 128 +
                         (size_t)((c ^ (r & 7)) << 4) + (size_t)within * 2;
      img[off / 2] = v > 0 ? 0x3C00 : (v < 0 ? 0xBC00 : 0);
    }
  return img;
}

std::mutex g_mu_small;
void* g_img_small[64][2];
// the constant A images live in static device memory (the library allocates none)
__device__ uint4 g_small_img108[hqs::Cfg<108, 1>::A_BYTES / 16];
__device__ uint4 g_small_img20[hqs::Cfg<20, 2>::A_BYTES / 16];

template <int MB, int LLO>
cudaError_t launch_small(const void* x, int64_t M, int64_t ld_x, float clip, uint8_t* q, int64_t ld_q, float* scale,
                         cudaStream_t stream, int slot, bool q8) {
  using C = hqs::Cfg<MB, LLO>;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  void* img = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu_small);
    if (!g_img_small[dev & 63][slot]) {
      const int8_t* h = base_hadamard_host(MB);
      if (!h) return cudaErrorInvalidValue;
      auto host = a_image_small<MB, LLO>(h);
      void* d = nullptr;
      e = MB == 108 ? cudaGetSymbolAddress(&d, g_small_img108) : cudaGetSymbolAddress(&d, g_small_img20);
      if (e != cudaSuccess) return e;
      e = cudaMemcpy(d, host.data(), host.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return e;
      e = cudaDeviceSynchronize();  // one-time: the image is complete before any stream reads it
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(hqs::hq_full_small_tc_kernel<MB, LLO, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)C::SMEM);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(hqs::hq_full_small_tc_kernel<MB, LLO, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)C::SMEM);
      if (e != cudaSuccess) return e;
      g_img_small[dev & 63][slot] = d;
    }
    img = g_img_small[dev & 63][slot];
  }
  if (M == 0) return cudaSuccess;  // quarot_prepare: one-time setup only
  auto fn = encode_fn_small();
  if (!fn) return cudaErrorInvalidValue;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)C::J, (cuuint64_t)hqs::NA, (cuuint64_t)M};
  cuuint64_t strides[2] = {(cuuint64_t)C::J * 2, (cuuint64_t)ld_x * 2};
  cuuint32_t box[3] = {64u, (cuuint32_t)hqs::NA, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(x), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(M < nsm ? M : nsm);
  auto kern = q8 ? hqs::hq_full_small_tc_kernel<MB, LLO, true> : hqs::hq_full_small_tc_kernel<MB, LLO, false>;
  kern<<<grid, hqs::NUM_THREADS, C::SMEM, stream>>>(
      map, M, clip, q, ld_q, scale, static_cast<const uint4*>(img));
  return cudaPeekAtLastError();
}

}  // namespace

bool hq_full_small_tc_supported(int64_t pow2, int m) { return (m == 108 && pow2 == 128) || (m == 20 && pow2 == 256); }

cudaError_t launch_hq_full_small_tc(const void* x, int64_t M, int64_t ld_x, int64_t pow2, int m, float clip,
                                    uint8_t* q, int64_t ld_q, float* scale, cudaStream_t stream, bool q8) {
  if (m == 108 && pow2 == 128) return launch_small<108, 1>(x, M, ld_x, clip, q, ld_q, scale, stream, 0, q8);
  if (m == 20 && pow2 == 256) return launch_small<20, 2>(x, M, ld_x, clip, q, ld_q, scale, stream, 1, q8);
  return cudaErrorInvalidValue;
}

}  // namespace qr
