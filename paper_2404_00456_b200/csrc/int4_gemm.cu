// int4_gemm.cu — rows a4 + a5 of the QuaRot hot path on sm_100a tensor cores.
//
// acc[m][n] = sum_k cx[m][k] * cw[n][k] (exact int32, "INT4 ... on a TensorCore is
// INT32"), y = fp16(acc * s_x[m] * s_w[n]) (P:233 dequantization with row and column
// scales), fused in the epilogue instead of the paper's separate kernel.
//
// sm_100 tcgen05 has no s4 kind, so packed INT4 operands are widened to INT8 on the way
// into shared memory and multiplied with tcgen05.mma kind::i8 into TMEM int32 accumulators.
//
// Design:
//  * persistent CTAs (one per SM), grouped-M tile raster for L2 reuse, tile 128 x 256,
//    k-block 128 (one 128-byte SWIZZLE_128B atom row per operand row), 4-stage smem ring;
//  * 8 producer warps: LDG.128 the packed tiles straight into registers (one k-block of
//    prefetch), widen with the "x16 nibble trick" (int8 = code*16 = byte & 0xF0 for the
//    high nibble, (byte << 4) & 0xF0 for the low nibble: 3 ALU ops per 8 codes, no sign
//    extension), STS.128 into the canonical K-major SW128 layout.  Each 32-code packed chunk
//    becomes [16 low-nibble codes | 16 high-nibble codes]: the SAME permutation of k for A
//    and B, so the dot product is unchanged.  The MMA accumulates 256*acc (|256*acc| <=
//    256*49*K < 2^31 for K <= 171196), the epilogue shifts right by 8 exactly;
//  * 1 MMA warp: a single thread issues 4 x tcgen05.mma (M128 N256 K32) per k-block and
//    tcgen05.commit's the stage back to the producers;
//  * 4 epilogue warps: tcgen05.ld 32x32b.x32 from TMEM (double-buffered 2 x 256 columns so
//    the next tile's mainloop overlaps this tile's epilogue), scale, round to fp16, store.
#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace gemm {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 128;           // int8 elements per k-block
constexpr int BKP = BK / 2;       // packed bytes per row per k-block
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;  // 16 KB
constexpr int B_BYTES = BN * BK;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_EPI_WARPS = 4;
constexpr int NUM_PROD_WARPS = 8;
constexpr int PROD_THREADS = NUM_PROD_WARPS * 32;
constexpr int MMA_WARP = NUM_EPI_WARPS + NUM_PROD_WARPS;  // warp 12
constexpr int NUM_THREADS = (MMA_WARP + 1) * 32;          // 416
constexpr int CHUNKS = (BM + BN) * (BKP / 16);            // 1536 x 16-byte packed chunks
constexpr int CPT = CHUNKS / PROD_THREADS;                // 6 per producer thread
constexpr int TMEM_COLS = 512;                            // 2 accumulators x 256 columns
constexpr int GROUP_M = 16;
constexpr uint32_t IDESC = idesc_i8(BM, BN);
constexpr size_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

static_assert(CHUNKS % PROD_THREADS == 0, "chunk split");

struct Params {
  const uint8_t* xq;
  const uint8_t* wq;
  const float* x_scale;
  const float* w_scale;
  void* out;  // fp16 y or int32 acc
  int64_t M, N, K, ld_xq, ld_wq, ld_out;
  int num_m, num_n, num_kb, num_tiles;
};

QR_DEVICE void tile_coords(const Params& p, int t, int& mb, int& nb) {
  const int per_group = GROUP_M * p.num_n;
  const int group = t / per_group;
  const int first_m = group * GROUP_M;
  const int gm = min(p.num_m - first_m, GROUP_M);
  const int within = t - group * per_group;
  mb = first_m + within % gm;
  nb = within / gm;
}

QR_DEVICE uint32_t lo_nib16(uint32_t w) { return (w << 4) & 0xF0F0F0F0u; }
QR_DEVICE uint32_t hi_nib16(uint32_t w) { return w & 0xF0F0F0F0u; }

template <bool kS32>
__global__ void __launch_bounds__(NUM_THREADS, 1) int4_gemm_kernel(const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full_bar = bars;                       // [STAGES] producers -> MMA
  uint64_t* empty_bar = bars + STAGES;             // [STAGES] MMA commit -> producers
  uint64_t* tfull_bar = bars + 2 * STAGES;         // [2] MMA commit -> epilogue
  uint64_t* tempty_bar = bars + 2 * STAGES + 2;    // [2] epilogue -> MMA
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], NUM_PROD_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], NUM_EPI_WARPS);
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

  const int my_tiles = (p.num_tiles > (int)blockIdx.x)
                           ? (p.num_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1
                           : 0;

  if (warp >= NUM_EPI_WARPS && warp < MMA_WARP) {
    // ===================== producers: LDG packed -> widen -> STS =====================
    const int pt = threadIdx.x - NUM_EPI_WARPS * 32;
    const int total = my_tiles * p.num_kb;
    uint4 nxt[CPT];
    auto load = [&](int it, uint4 (&dst)[CPT]) {
      const int tl = it / p.num_kb;
      const int kb = it - tl * p.num_kb;
      int mb, nb;
      tile_coords(p, (int)blockIdx.x + tl * (int)gridDim.x, mb, nb);
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int c = pt + i * PROD_THREADS;
        const int r = c >> 2;
        const int q = c & 3;
        const uint8_t* src;
        bool ok;
        if (r < BM) {
          const int64_t row = (int64_t)mb * BM + r;
          ok = row < p.M;
          src = p.xq + row * p.ld_xq + (int64_t)kb * BKP + q * 16;
        } else {
          const int64_t row = (int64_t)nb * BN + (r - BM);
          ok = row < p.N;
          src = p.wq + row * p.ld_wq + (int64_t)kb * BKP + q * 16;
        }
        dst[i] = ok ? ldg_nc_v4(src) : make_uint4(0, 0, 0, 0);
      }
    };
    if (total > 0) load(0, nxt);
    for (int it = 0; it < total; ++it) {
      const int stage = it % STAGES;
      const uint32_t phase = (it / STAGES) & 1;
      uint4 cur[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) cur[i] = nxt[i];
      if (it + 1 < total) load(it + 1, nxt);
      mbar_wait(&empty_bar[stage], phase ^ 1);
      const uint32_t sbase = smem_u32(smem + stage * STAGE_BYTES);
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int c = pt + i * PROD_THREADS;
        const int r = c >> 2;
        const int q = c & 3;
        const uint32_t obase = (r < BM) ? sbase + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 128u
                                        : sbase + A_BYTES + (uint32_t)((r - BM) >> 3) * 1024u +
                                              (uint32_t)((r - BM) & 7) * 128u;
        const uint32_t sw = (uint32_t)(r & 7);  // (r - BM) & 7 == r & 7 since BM % 8 == 0
        const uint4 w = cur[i];
        const uint4 lo = make_uint4(lo_nib16(w.x), lo_nib16(w.y), lo_nib16(w.z), lo_nib16(w.w));
        const uint4 hi = make_uint4(hi_nib16(w.x), hi_nib16(w.y), hi_nib16(w.z), hi_nib16(w.w));
        sts_v4(obase + ((((uint32_t)(2 * q)) ^ sw) << 4), lo);
        sts_v4(obase + ((((uint32_t)(2 * q + 1)) ^ sw) << 4), hi);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[stage]);
    }
  } else if (warp == MMA_WARP) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      int it = 0;
      for (int tl = 0; tl < my_tiles; ++tl) {
        const int acc = tl & 1;
        const uint32_t acc_phase = (tl >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint64_t a_desc = umma_desc_sw128(a_addr);
          const uint64_t b_desc = umma_desc_sw128(a_addr + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            // advance 32 bytes along K inside the 128-byte swizzle atom: +2 in 16-byte units
            mma_i8_ss(d_tmem, a_desc + (uint64_t)(2 * k), b_desc + (uint64_t)(2 * k), IDESC,
                      (kb | k) != 0 ? 1u : 0u);
          }
          mma_commit(&empty_bar[stage]);
        }
        mma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue warps 0..3 =====================
    const int row_in_tile = warp * 32 + lane;
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int acc = tl & 1;
      const uint32_t acc_phase = (tl >> 1) & 1;
      int mb, nb;
      tile_coords(p, (int)blockIdx.x + tl * (int)gridDim.x, mb, nb);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int64_t m = (int64_t)mb * BM + row_in_tile;
      const bool row_ok = m < p.M;
      float sx = 0.f;
      if (!kS32 && row_ok) sx = __ldg(p.x_scale + m);
      const uint32_t taddr = tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t r[32];
        QR_TMEM_LD32(taddr + (uint32_t)(cc * 32), r);
        tmem_ld_wait();
        const int64_t n0 = (int64_t)nb * BN + cc * 32;
        if (row_ok) {
          if constexpr (kS32) {
            int32_t* dst = reinterpret_cast<int32_t*>(p.out) + m * p.ld_out + n0;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              if (n0 + g * 4 < p.N) {
                int4 v = make_int4((int32_t)r[4 * g] >> 8, (int32_t)r[4 * g + 1] >> 8,
                                   (int32_t)r[4 * g + 2] >> 8, (int32_t)r[4 * g + 3] >> 8);
                *reinterpret_cast<int4*>(dst + g * 4) = v;
              }
            }
          } else {
            __half* dst = reinterpret_cast<__half*>(p.out) + m * p.ld_out + n0;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              if (n0 + g * 8 < p.N) {
                const float4 s0 = __ldg(reinterpret_cast<const float4*>(p.w_scale + n0 + g * 8));
                const float4 s1 = __ldg(reinterpret_cast<const float4*>(p.w_scale + n0 + g * 8 + 4));
                const float sw[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
                uint32_t h[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float v0 = ((float)((int32_t)r[8 * g + 2 * e] >> 8) * sx) * sw[2 * e];
                  const float v1 = ((float)((int32_t)r[8 * g + 2 * e + 1] >> 8) * sx) * sw[2 * e + 1];
                  __half2 hv = __floats2half2_rn(v0, v1);
                  h[e] = *reinterpret_cast<uint32_t*>(&hv);
                }
                *reinterpret_cast<uint4*>(dst + g * 8) = make_uint4(h[0], h[1], h[2], h[3]);
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace gemm

static int g_num_sms[64];

static int num_sms_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!g_num_sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev] = v > 0 ? v : 148;
  }
  return g_num_sms[dev];
}

template <bool kS32>
static cudaError_t launch_gemm_impl(const uint8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                                    const uint8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* out,
                                    int64_t ld_out, cudaStream_t stream) {
  using namespace gemm;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(int4_gemm_kernel<kS32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  Params p;
  p.xq = xq;
  p.wq = wq;
  p.x_scale = xs;
  p.w_scale = ws;
  p.out = out;
  p.M = M;
  p.N = N;
  p.K = K;
  p.ld_xq = ld_xq;
  p.ld_wq = ld_wq;
  p.ld_out = ld_out;
  p.num_m = (int)((M + BM - 1) / BM);
  p.num_n = (int)((N + BN - 1) / BN);
  p.num_kb = (int)(K / BK);
  p.num_tiles = p.num_m * p.num_n;
  const int grid = p.num_tiles < num_sms_current() ? p.num_tiles : num_sms_current();
  int4_gemm_kernel<kS32><<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(p);
  return cudaPeekAtLastError();
}

cudaError_t launch_int4_gemm(const uint8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                             const uint8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* y,
                             int64_t ld_y, cudaStream_t stream) {
  return launch_gemm_impl<false>(xq, xs, M, K, ld_xq, wq, ws, N, ld_wq, y, ld_y, stream);
}

cudaError_t launch_int4_gemm_s32(const uint8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const uint8_t* wq,
                                 int64_t N, int64_t ld_wq, int32_t* acc, int64_t ld_acc, cudaStream_t stream) {
  return launch_gemm_impl<true>(xq, nullptr, M, K, ld_xq, wq, nullptr, N, ld_wq, acc, ld_acc, stream);
}

}  // namespace qr
