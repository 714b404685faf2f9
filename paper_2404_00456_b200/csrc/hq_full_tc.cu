// hq_full_tc.cu — rows a1 + a3 for K = 1024 x 28 (the Llama-2-70B down_proj input, P:182-185,
// P:67) with the first Kronecker factors on the tcgen05 tensor path.
//
// y = (H_1024 (x) H_28) x per token row (Sylvester H_1024, element i = a*28 + b, reading Z2).
// Split a = a_hi*4 + a_lo (a_hi < 256, a_lo < 4): Sylvester gives H_1024 = H_256 (x) H_4, so
//
//     y[a'_hi*112 + j'] = sum_{a_hi} H_256[a'_hi][a_hi] * D[j'][a_hi],
//     D[j'][a_hi]      = sum_j (H_4 (x) H_28)[j'][j] * x[a_hi*112 + j],   j = a_lo*28 + b.
//
//  * D is ONE dense fp16 contraction per row: tcgen05.mma kind::f16, M = 128 (j', 112 real rows
//    of the constant A = H_4 (x) H_28, zero-padded), N = 256 (a_hi), K = 112 (7 MMAs of K = 16).
//    +-1 x fp16 products are exact; the accumulation is fp32 (the paper's FP32 Hadamard).
//    The row is TMA'd straight into the K-major SWIZZLE_128B operand layout by a 3-D tensor map
//    [row][a_hi][j] (two 64-wide j boxes; j >= 112 is zero-filled), 3-stage ring.
//  * D lands in TMEM (fp32, lane = j', column = a_hi), double-buffered (2 x 256 columns), so the
//    MMA of row r+1 overlaps the epilogue of row r.
//  * H_256 over the columns runs in registers with packed fp32x2 butterflies (FADD2): 16
//    epilogue warps, four per TMEM lane quarter (g = 0..3).  Pass 1: each thread loads the 64
//    columns with a_hi bits 6-7 = g and transforms bits 1-5 (pairs = adjacent columns), then
//    stores them back to TMEM; pass 2 (after the lane's other three threads): the 64 columns
//    with bits 4-5 = g, bits 6, 7 and 0 (within the register pair).  Every bit exactly once.
//  * Rows are software-pipelined with split-phase mbarriers: pass1(r+1), then the quantization of
//    row r once all 16 warps posted their partial amax (its values parked in TMEM), then pass2(r+1).
//  * Scale (1/sqrt(K) folded in, reading Z5), RNE
//    INT4 codes with the magic add; the two nibbles of a byte are adjacent j' = adjacent TMEM
//    lanes, merged with one shuffle per code word.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace hqtc {

constexpr int MB = 28, P = 1024, K = MB * P;
constexpr int J = 4 * MB;                    // 112: contraction (a_lo, b) per a_hi
constexpr int NA = P / 4;                    // 256 a_hi columns
constexpr int A_BYTES = 128 * 128 * 2;       // (H_4 (x) H_28) padded to 128 x 128 fp16, SW128 K-major
constexpr int BOX_BYTES = NA * 128;          // 256 a_hi rows x 64 j (128 B)
constexpr int STAGE_BYTES = 2 * BOX_BYTES;   // 64 KB per token row
constexpr int STAGES = 3;
constexpr int TMA_WARP = 0, MMA_WARP = 1, EPI_WARP0 = 4, NUM_EPI = 16;  // warps 2-3 idle (warpgroup 0)
constexpr int TPL = NUM_EPI / 4;  // epilogue threads per TMEM lane
constexpr int NUM_THREADS = (EPI_WARP0 + NUM_EPI) * 32;
constexpr uint32_t TMEM_COLS = 512;
constexpr size_t SMEM = 1024 + A_BYTES + (size_t)STAGES * STAGE_BYTES + 256;  // + barriers
static_assert(SMEM <= 232448, "227 KB dynamic smem");
// kind::f16: D f32 (bits 4-5 = 1), A = B = f16 (0), both K-major, N/8 at 17, M/16 at 24
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(NA >> 3) << 17) | ((128u >> 4) << 24);

QR_DEVICE void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}
QR_DEVICE void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
QR_DEVICE void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
QR_DEVICE bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(p));
  return p != 0;
}
QR_DEVICE void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

#define QR_TMEM_ST16(taddr, r)                                                                          \
  asm volatile(                                                                                         \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr), \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),  \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]))
#define QR_TMEM_ST32(taddr, r)                                                                          \
  asm volatile(                                                                                         \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                   \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),  \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),      \
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),     \
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))
#define QR_TMEM_LD8(taddr, r)                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                 \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
                 "=r"(r[7])                                                                             \
               : "r"(taddr))
#define QR_TMEM_ST8(taddr, r)                                                                           \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),    \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]))
QR_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

QR_DEVICE void bfly(float2& u, float2& v) {
  const float2 s = f2add(u, v), d = f2sub(u, v);
  u = s;
  v = d;
}

// 4 codes (low nibble of each byte; the byte is the two's-complement code) of a.x, a.y, b.x, b.y:
// RNE by the 1.5 * 2^23 magic add (|v * inv| <= 7 / 0.9 < 2^22), whose low 16 bits are the
// integer; clamp to [-7, 7] on two 16-bit lanes at a time (VIMNMX), then gather the low bytes.
// kClamp = false: the caller guarantees |v * inv| < 7.5 for every lane (RNE then lands in [-7, 7])
template <bool kClamp = true>
QR_DEVICE uint32_t code_word(float2 a, float2 b, float inv) {
  const float2 i2 = make_float2(inv, inv), mg = make_float2(12582912.f, 12582912.f);
  const float2 ma = f2add(f2mul(a, i2), mg), mb = f2add(f2mul(b, i2), mg);
  uint32_t lo = __byte_perm(__float_as_uint(ma.x), __float_as_uint(ma.y), 0x5410);
  uint32_t hi = __byte_perm(__float_as_uint(mb.x), __float_as_uint(mb.y), 0x5410);
  if constexpr (kClamp) {
    lo = __vmaxs2(__vmins2(lo, 0x00070007u), 0xFFF9FFF9u);
    hi = __vmaxs2(__vmins2(hi, 0x00070007u), 0xFFF9FFF9u);
  }
  return __byte_perm(lo, hi, 0x6420);
}

// kSpin: epilogue waits spin on try_wait (true) or with a suspend-time hint; kQ8: int8 codes in
// [-127, 127], one byte per element (A8, §8 f4)
template <bool kSpin, bool kQ8 = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    hq_full28_tc_kernel(const __grid_constant__ CUtensorMap tmX, int64_t M, float clip, uint8_t* __restrict__ q,
                        int64_t ld_q, float* __restrict__ scale, const uint4* __restrict__ a_img) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * STAGE_BYTES);  // [STAGES] TMA landed
  uint64_t* empty = full + STAGES;                                           // [STAGES] MMA done reading
  uint64_t* t_full = empty + STAGES;                                         // [2] D ready
  uint64_t* t_empty = t_full + 2;                                            // [2] epilogue done reading D
  uint64_t* pair_done = t_empty + 2;                                         // [4 quarters][2] pass 1 done
  uint64_t* amax_done = pair_done + 8;                                       // [2] row partial amax posted
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(amax_done + 2);
  __shared__ float red[2][NUM_EPI];                                          // per-warp partial amax
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < A_BYTES / 16; i += NUM_THREADS) reinterpret_cast<uint4*>(sA)[i] = __ldg(a_img + i);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], NUM_EPI);
      mbar_init(&amax_done[b], NUM_EPI);
    }
    for (int i = 0; i < 8; ++i) mbar_init(&pair_done[i], TPL);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) {
    tmem_alloc(tmem_holder, TMEM_COLS);
    tmem_relinquish();
  }
  if (warp == TMA_WARP && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int64_t nrows = M > (int64_t)blockIdx.x ? (M - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;

  if (warp < EPI_WARP0) {
    // register budget = launch bound (96) x 640 threads: 128 x 32 + 512 x 112 (an inc beyond the
    // CTA's allocation would block forever)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
    if (warp == TMA_WARP) {
      if (lane == 0) {
        for (int64_t it = 0; it < nrows; ++it) {
          const int s = (int)(it % STAGES);
          mbar_wait_sleep(&empty[s], (uint32_t)((it / STAGES) & 1) ^ 1u);
          expect_tx(&full[s], STAGE_BYTES);
          const int row = (int)((int64_t)blockIdx.x + it * gridDim.x);
          const uint32_t dst = smem_u32(sB + s * STAGE_BYTES);
          tma_load_3d(dst, &tmX, 0, 0, row, &full[s]);
          tma_load_3d(dst + BOX_BYTES, &tmX, 64, 0, row, &full[s]);
        }
      }
    } else if (warp == MMA_WARP) {
      // the whole warp runs the loop (warp-uniform descriptors); one elected lane issues
      const uint64_t a_desc = umma_desc_sw128(smem_u32(sA));
      const uint32_t sb = smem_u32(sB);
      for (int64_t it = 0; it < nrows; ++it) {
        const int s = (int)(it % STAGES), buf = (int)(it & 1);
        mbar_wait_sleep(&t_empty[buf], (uint32_t)((it >> 1) & 1) ^ 1u);
        mbar_wait_sleep(&full[s], (uint32_t)((it / STAGES) & 1));
        tc_fence_after();
        const uint64_t b_desc = umma_desc_sw128(sb + (uint32_t)(s * STAGE_BYTES));
        const uint32_t d_tmem = tmem_base + (uint32_t)(buf * NA);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < J / 16; ++kk) {  // atom kk/4 (A: +16 KB, B: +32 KB), +32 B per K = 16
            const uint64_t koff = (uint64_t)(2 * (kk & 3));
            mma_f16(d_tmem, a_desc + (uint64_t)((kk >> 2) * (16384 >> 4)) + koff,
                    b_desc + (uint64_t)((kk >> 2) * (BOX_BYTES >> 4)) + koff, IDESC, kk > 0 ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          mma_commit(&t_full[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    // Software pipeline over rows (split-phase barriers, so no warp idles at a barrier):
    //   pass1(r + 1) | quant(r) [after every warp posted its amax of row r] | pass2(r + 1)
    // The pass-2 values of a row are parked in its TMEM buffer between pass 2 and quant.
    auto epi_wait = [](uint64_t* bar, uint32_t parity) {
      if (kSpin) mbar_wait(bar, parity);
      else mbar_wait_sleep(bar, parity);
    };
    const int e = warp - EPI_WARP0;  // 0..15
    const int qd = warp & 3;         // TMEM lane quarter this warp may access
    const int g = e >> 2;            // which of the TPL = 4 threads of the lane
    const int L = qd * 32 + lane;    // TMEM lane = output j'
    const bool lane_ok = L < J;
    const bool odd = (lane & 1) != 0;
    const uint32_t t_lane = tmem_base + ((uint32_t)(qd * 32) << 16);
    const float norm_f = (float)rsqrt((double)K);
    const float c0 = (float)((double)clip * rsqrt((double)K) / (kQ8 ? 127.0 : 7.0));  // scale = c0 * amax
    // merged byte of j' = 2p (low nibble, even lane) and 2p + 1 (high nibble, odd lane)
    const uint32_t sh_keep = odd ? 4u : 0u, sh_recv = odd ? 0u : 4u;
    const uint32_t keep_mask = odd ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
    // even lanes write the a_hi bit 7 = 0 half of the pair's bytes, odd lanes the other half
    uint8_t* const qlane = q + (L >> 1) + (int64_t)(16 * g + 128 * (odd ? 1 : 0)) * (J / 2);

    // pass 1: columns 64 g + 32 i + c; a_hi bits 0-4 = c, 5 = i, 6-7 = g; transforms bits 1-5
    auto pass1 = [&](int64_t it) {
      const int buf = (int)(it & 1);
      epi_wait(&t_full[buf], (uint32_t)((it >> 1) & 1));
      tc_fence_after();
      const uint32_t tb = t_lane + (uint32_t)(buf * NA + 64 * g);
      uint32_t r[2][32];
      QR_TMEM_LD32(tb, r[0]);
      QR_TMEM_LD32(tb + 32u, r[1]);
      tmem_ld_wait();
      float2 P[2][16];  // P[i][c'] = columns (2c', 2c' + 1): adjacent registers of the load
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int c = 0; c < 16; ++c) P[i][c] = make_float2(__uint_as_float(r[i][2 * c]), __uint_as_float(r[i][2 * c + 1]));
#pragma unroll
      for (int st = 1; st < 16; st <<= 1)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (!(c & st)) bfly(P[i][c], P[i][c + st]);
#pragma unroll
      for (int c = 0; c < 16; ++c) bfly(P[0][c], P[1][c]);  // bit 5
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          r[i][2 * c] = __float_as_uint(P[i][c].x);
          r[i][2 * c + 1] = __float_as_uint(P[i][c].y);
        }
      QR_TMEM_ST32(tb, r[0]);
      QR_TMEM_ST32(tb + 32u, r[1]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pair_done[qd * 2 + buf]);
    };
    // pass 2: columns 64 i + 16 g + c; a_hi bits 0-3 = c, 4-5 = g, 6-7 = i; transforms bits 6, 7
    // and 0 (within the register pair), posts the partial amax, parks the values
    auto pass2 = [&](int64_t it) {
      const int buf = (int)(it & 1);
      epi_wait(&pair_done[qd * 2 + buf], (uint32_t)((it >> 1) & 1));  // the lane's pass 1
      tc_fence_after();
      const uint32_t tb = t_lane + (uint32_t)(buf * NA + 16 * g);
      uint32_t u[4][16];
#pragma unroll
      for (int i = 0; i < 4; ++i) QR_TMEM_LD16(tb + 64u * i, u[i]);
      tmem_ld_wait();
      float am[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float2 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = make_float2(__uint_as_float(u[i][2 * c]), __uint_as_float(u[i][2 * c + 1]));
        bfly(v[0], v[1]);  // bit 6
        bfly(v[2], v[3]);
        bfly(v[0], v[2]);  // bit 7
        bfly(v[1], v[3]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          v[i] = pair_bfly(v[i]);  // bit 0
          am[i] = fmax_nan(am[i], fmax_nan(fabsf(v[i].x), fabsf(v[i].y)));
          u[i][2 * c] = __float_as_uint(v[i].x);
          u[i][2 * c + 1] = __float_as_uint(v[i].y);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) QR_TMEM_ST16(tb + 64u * i, u[i]);
      float amax = lane_ok ? fmax_nan(fmax_nan(am[0], am[1]), fmax_nan(am[2], am[3])) : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (lane == 0) red[buf][e] = amax;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&amax_done[buf]);
    };
    // quant: row scale from the partial amax values, reload the parked values, release the TMEM
    // buffer, RNE codes, merge the nibble pairs across adjacent lanes, store
    auto quant = [&](int64_t it) {
      const int buf = (int)(it & 1);
      const int64_t row = (int64_t)blockIdx.x + it * gridDim.x;
      epi_wait(&amax_done[buf], (uint32_t)((it >> 1) & 1));
      tc_fence_after();
      const uint32_t tb = t_lane + (uint32_t)(buf * NA + 16 * g);
      uint32_t u[4][16];
#pragma unroll
      for (int i = 0; i < 4; ++i) QR_TMEM_LD16(tb + 64u * i, u[i]);
      float amax = red[buf][0];
#pragma unroll
      for (int w = 1; w < NUM_EPI; ++w) amax = fmax_nan(amax, red[buf][w]);
      // scale = fp32(clip * amax / (7 sqrt(K))) (readings Z5, Z9); zero row -> 1, non-finite -> NaN
      float sc = 1.f, inv = 0.f;
      if (!isfinite(amax)) {
        sc = __int_as_float(0x7fc00000);
      } else if (amax != 0.f) {
        sc = c0 * amax;
        inv = __fdiv_rn(norm_f, sc);
      }
      if (e == 0 && lane == 0) scale[row] = sc;
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[buf]);  // D[buf] may be overwritten by row it + 2
      if (inv == 0.f) {  // zero or non-finite row: all codes 0
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < 16; ++c) u[i][c] = 0u;
      }
      if constexpr (kQ8) {  // element (a_hi, j') at byte a_hi * 112 + j': a warp store covers 32 bytes
        if (lane_ok) {
          int8_t* const q8 = reinterpret_cast<int8_t*>(q) + row * ld_q + L;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 16; c += 2) {
              const float2 m = f2fma(make_float2(__uint_as_float(u[i][c]), __uint_as_float(u[i][c + 1])),
                                     make_float2(inv, inv), make_float2(12582912.f, 12582912.f));
              const uint32_t w = __vmaxs2(__vmins2(__byte_perm(__float_as_uint(m.x), __float_as_uint(m.y), 0x5410),
                                                   0x007F007Fu), 0xFF81FF81u);
              const int a = 64 * i + 16 * g + c;
              q8[(int64_t)a * J] = (int8_t)(w & 0xFFu);
              q8[(int64_t)(a + 1) * J] = (int8_t)((w >> 16) & 0xFFu);
            }
        }
        return;
      }
      uint32_t out[2][4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {  // codes of a_hi = 64 i + 16 g + 4m .. +3
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          w[i] = code_word(make_float2(__uint_as_float(u[i][4 * m]), __uint_as_float(u[i][4 * m + 1])),
                           make_float2(__uint_as_float(u[i][4 * m + 2]), __uint_as_float(u[i][4 * m + 3])), inv);
#pragma unroll
        for (int ii = 0; ii < 2; ++ii) {  // even lane keeps i = ii (bit 7 = 0), odd lane i = ii + 2
          const uint32_t got = __shfl_xor_sync(0xffffffffu, odd ? w[ii] : w[ii + 2], 1);
          const uint32_t keep = odd ? w[ii + 2] : w[ii];
          out[ii][m] = ((keep << sh_keep) & keep_mask) | ((got << sh_recv) & ~keep_mask);
        }
      }
      if (lane_ok) {
        uint8_t* const qr = qlane + row * ld_q;
#pragma unroll
        for (int ii = 0; ii < 2; ++ii)
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            uint8_t* dst = qr + (int64_t)(64 * ii + 4 * m) * (J / 2);
            const uint32_t o = out[ii][m];
            dst[0] = (uint8_t)o;
            dst[J / 2] = (uint8_t)(o >> 8);
            dst[J] = (uint8_t)(o >> 16);
            dst[3 * J / 2] = (uint8_t)(o >> 24);
          }
      }
    };
    if (nrows > 0) {
      pass1(0);
      pass2(0);
    }
    for (int64_t it = 0; it < nrows; ++it) {
      if (it + 1 < nrows) pass1(it + 1);
      quant(it);
      if (it + 1 < nrows) pass2(it + 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace hqtc

// ============================================================================ warpgroup pair per row
// hq_full28_wg_kernel: the same transform (MMA of H_4 (x) H_28 per row into TMEM, H_256 over the
// a_hi columns on CUDA cores) with each of the two TMEM row buffers owned by its own pair of
// epilogue warpgroups (8 warps), so the two rows in flight never wait on each other, and with
// hardware named barriers (no mbarrier polling) for the two intra-row dependencies.  Round-1
// ncu: the 16-warps-share-every-row design spent ~1.9 instructions per element polling
// mbarriers.  Per row, thread (lane L = j', g = its warpgroup within the pair):
//   pass A: quarters g and g + 2 (64 columns each), bits 0-5 in registers;
//   [named barrier, the 2 warps sharing the lanes]
//   pass B: bits 6 and 7 over the 4-tuples (c, c + 64, c + 128, c + 192), c in [32 g, 32 g + 32),
//           + amax; parked in TMEM;
//   [named barrier, the 8 warps: the row's amax]
//   quant:  exactly pass B's columns, 32 at a time (so the thread's pass-B amax tells the warp
//           whether the clamp can be skipped); each loaded chunk releases one quarter (8 arrivals).
// The MMA runs per 64-column quarter (N = 64), one MMA warp per buffer, so a quarter of the next
// row is multiplied as soon as all 8 warps' quant loaded it; the MMA warp also reloads the stage
// its row freed (TMA of row it + 3).  The producer warps have the highest warp ids (the
// schedulers prefer them).  Bit 0 (within a register pair) uses one FFMA2 (pair_bfly), so all 8
// stages cost 0.5 instructions / element.
// kPerm: codes in the transform-native K order (quarot.h QUAROT_HAD_KPERM): position
//   p = (a_hi >> 5) * 3584 + j' * 32 + (a_hi & 31) — 32 consecutive a_hi of a lane are 16
//   contiguous bytes (one 16-byte store; a warp writes 512 contiguous bytes); otherwise the
//   natural element order a_hi * 112 + j' (adjacent lanes merged into bytes, byte stores).
namespace hqwg {
using hqtc::A_BYTES;
using hqtc::BOX_BYTES;
using hqtc::J;
using hqtc::K;
using hqtc::NA;
using hqtc::STAGE_BYTES;
constexpr int NH = NA / 2;  // 128 columns per half (a_hi bit 7)
constexpr int NQ = NA / 4;  // 64 columns per quarter: the MMA / release granularity
constexpr int STAGES = 3;
// the producer warps take the highest ids (the schedulers prefer the highest-id eligible warp:
// the next row's MMA issue is latency-critical for the epilogue warps waiting on it)
#ifndef QR_WG_PROD_HIGH
#define QR_WG_PROD_HIGH 1
#endif
constexpr int NUM_EPI = 16, EPI_WARP0 = QR_WG_PROD_HIGH ? 0 : 4, CTL_WARP0 = QR_WG_PROD_HIGH ? 16 : 0;
constexpr int TMA_WARP = CTL_WARP0, MMA_WARP0 = CTL_WARP0 + 1;  // MMA warps: one per buffer
constexpr int NUM_THREADS = (4 + NUM_EPI) * 32;                  // 640
constexpr uint32_t TMEM_COLS = 512;
#ifndef QR_WG_BACKOFF
#define QR_WG_BACKOFF 64  // ns between the MMA warps' barrier polls (the next row's MMA is latency-critical)
#endif
#ifndef QR_WG_TMA_IN_MMA
#define QR_WG_TMA_IN_MMA 1  // the MMA warps reload the stage their row freed (no polling TMA warp)
#endif
#ifndef QR_WG_MMA_SLEEP
#define QR_WG_MMA_SLEEP 0  // 1: the MMA warps wait with try_wait's suspend hint instead of back-off polls
#endif
#ifndef QR_WG_TMA_BACKOFF
#define QR_WG_TMA_BACKOFF 512  // ns between the TMA warp's polls (three stages of slack)
#endif
constexpr size_t SMEM = 1024 + A_BYTES + (size_t)STAGES * STAGE_BYTES + 256;
static_assert(SMEM <= 232448, "227 KB dynamic smem");
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(NQ >> 3) << 17) | ((128u >> 4) << 24);

// 8 codes -> one 32-bit word of the KPERM layout: byte t = c[2t] | c[2t+1] << 4 (a..d = pairs)
QR_DEVICE uint32_t code_word8(float2 a, float2 b, float2 c, float2 d, float inv) {
  const float2 i2 = make_float2(inv, inv), mg = make_float2(12582912.f, 12582912.f);
  const float2 ma = f2fma(a, i2, mg), mb = f2fma(b, i2, mg), mc = f2fma(c, i2, mg), md = f2fma(d, i2, mg);
  // 16-bit lanes: even codes (c0, c2) / odd codes (c1, c3) of each group of four, clamped to [-7, 7]
  uint32_t e0 = __byte_perm(__float_as_uint(ma.x), __float_as_uint(mb.x), 0x5410);
  uint32_t o0 = __byte_perm(__float_as_uint(ma.y), __float_as_uint(mb.y), 0x5410);
  uint32_t e1 = __byte_perm(__float_as_uint(mc.x), __float_as_uint(md.x), 0x5410);
  uint32_t o1 = __byte_perm(__float_as_uint(mc.y), __float_as_uint(md.y), 0x5410);
  e0 = __vmaxs2(__vmins2(e0, 0x00070007u), 0xFFF9FFF9u);
  o0 = __vmaxs2(__vmins2(o0, 0x00070007u), 0xFFF9FFF9u);
  e1 = __vmaxs2(__vmins2(e1, 0x00070007u), 0xFFF9FFF9u);
  o1 = __vmaxs2(__vmins2(o1, 0x00070007u), 0xFFF9FFF9u);
  // bytes at bits 0-7, 16-23 (the shifts as SHF: ALU pipe rather than IMAD.SHL on the FMA pipe)
  const uint32_t w0 = (e0 & 0x000F000Fu) | __funnelshift_l(0u, o0 & 0x000F000Fu, 4);
  const uint32_t w1 = (e1 & 0x000F000Fu) | __funnelshift_l(0u, o1 & 0x000F000Fu, 4);
  return __byte_perm(w0, w1, 0x6420);
}

// code_word8 without the clamp, for threads none of whose elements can reach |v * inv| >= 7.5
// (then RNE already lands in [-7, 7]): the low byte of each magic-added float is its
// two's-complement code; gather the even / odd codes' low bytes (3 PRMT each) and merge the
// nibbles with one shift and one bit-select LOP3 — 8 ALU instructions per 8 codes instead of 17.
QR_DEVICE uint32_t code_word8_nc(float2 a, float2 b, float2 c, float2 d, float inv) {
  const float2 i2 = make_float2(inv, inv), mg = make_float2(12582912.f, 12582912.f);
  const float2 ma = f2fma(a, i2, mg), mb = f2fma(b, i2, mg), mc = f2fma(c, i2, mg), md = f2fma(d, i2, mg);
  const uint32_t e = __byte_perm(__byte_perm(__float_as_uint(ma.x), __float_as_uint(mb.x), 0x0040),
                                 __byte_perm(__float_as_uint(mc.x), __float_as_uint(md.x), 0x0040), 0x5410);
  const uint32_t o = __byte_perm(__byte_perm(__float_as_uint(ma.y), __float_as_uint(mb.y), 0x0040),
                                 __byte_perm(__float_as_uint(mc.y), __float_as_uint(md.y), 0x0040), 0x5410);
  const uint32_t os = __funnelshift_l(0u, o, 4);  // o << 4 as SHF (ALU pipe; a plain shift became IMAD.SHL on the busier FMA pipe)
  uint32_t w;  // (e & 0x0F0F0F0F) | (os & 0xF0F0F0F0): LUT 0xE4 = c ? a : b over (a = e, b = os, c = mask)
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(w) : "r"(e), "r"(os), "r"(0x0F0F0F0Fu));
  return w;
}

template <bool kPerm>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    hq_full28_wg_kernel(const __grid_constant__ CUtensorMap tmX, int64_t M, float clip, uint8_t* __restrict__ q,
                        int64_t ld_q, float* __restrict__ scale, const uint4* __restrict__ a_img) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * STAGE_BYTES);  // [STAGES] TMA landed
  uint64_t* empty = full + STAGES;                                           // [STAGES] MMA done reading
  uint64_t* t_full = empty + STAGES;                                         // [buf][quarter] D ready
  uint64_t* t_empty = t_full + 8;                                            // [buf][quarter] D consumed
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 8);
  __shared__ float red[2][2][8];                                             // [buf][row parity][warp]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < A_BYTES / 16; i += NUM_THREADS) reinterpret_cast<uint4*>(sA)[i] = __ldg(a_img + i);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 8; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 8);  // the 4 lane-quarter warps of both halves
    }
    fence_barrier_init();
  }
  if (warp == MMA_WARP0) {
    tmem_alloc(tmem_holder, TMEM_COLS);
    tmem_relinquish();
  }
  if (warp == TMA_WARP && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int64_t nrows = M > (int64_t)blockIdx.x ? (M - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;

  if (warp >= CTL_WARP0 && warp < CTL_WARP0 + 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");  // 128 x 64 + 512 x 104 = 640 x 96
    auto issue_tma = [&](int64_t it) {  // local row it into stage it % STAGES (one thread)
      const int s = (int)(it % STAGES);
      hqtc::expect_tx(&full[s], STAGE_BYTES);
      const int row = (int)((int64_t)blockIdx.x + it * gridDim.x);
      const uint32_t dst = smem_u32(sB + s * STAGE_BYTES);
      hqtc::tma_load_3d(dst, &tmX, 0, 0, row, &full[s]);
      hqtc::tma_load_3d(dst + BOX_BYTES, &tmX, 64, 0, row, &full[s]);
    };
#if QR_WG_TMA_IN_MMA
    // the MMA warps issue the TMA: after row it's last quarter the warp waits for its MMAs to
    // complete (a few hundred cycles) and reloads the freed stage with row it + STAGES (a separate
    // TMA warp polled the stage's mbarrier ~130 times per row: NANOSLEEP wakes early)
    if (warp == TMA_WARP) {
      if (lane == 0)
        for (int64_t it = 0; it < nrows && it < STAGES; ++it) issue_tma(it);
    } else
#else
    if (warp == TMA_WARP) {
      if (lane == 0) {
        for (int64_t it = 0; it < nrows; ++it) {
          mbar_wait_backoff<QR_WG_TMA_BACKOFF>(&empty[it % STAGES], (uint32_t)((it / STAGES) & 1) ^ 1u);
          issue_tma(it);
        }
      }
    } else
#endif
    if (warp < MMA_WARP0 + 2) {
      // MMA warp b issues the rows of buffer b (it % 2 == b)
      const int b = warp - MMA_WARP0;
      const uint64_t a_desc = umma_desc_sw128(smem_u32(sA));
      const uint32_t sb = smem_u32(sB);
      for (int64_t it = b; it < nrows; it += 2) {
        const int s = (int)(it % STAGES);
        const uint32_t n_par = (uint32_t)((it >> 1) & 1);
        mbar_wait_backoff<QR_WG_BACKOFF>(&full[s], (uint32_t)((it / STAGES) & 1));
#pragma unroll 1
        for (int h = 0; h < 4; ++h) {  // quarter h: a_hi 64 h .. 64 h + 63 (N = 64)
#if QR_WG_MMA_SLEEP
          mbar_wait_sleep(&t_empty[4 * b + h], n_par ^ 1u);
#else
          mbar_wait_backoff<QR_WG_BACKOFF>(&t_empty[4 * b + h], n_par ^ 1u);
#endif
          tc_fence_after();
          const uint64_t b_desc = umma_desc_sw128(sb + (uint32_t)(s * STAGE_BYTES + h * (NQ * 128)));
          const uint32_t d_tmem = tmem_base + (uint32_t)(b * NA + h * NQ);
          if (hqtc::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < J / 16; ++kk) {  // atom kk/4 (A: +16 KB, B: +32 KB), +32 B per K = 16
              const uint64_t koff = (uint64_t)(2 * (kk & 3));
              hqtc::mma_f16(d_tmem, a_desc + (uint64_t)((kk >> 2) * (16384 >> 4)) + koff,
                            b_desc + (uint64_t)((kk >> 2) * (BOX_BYTES >> 4)) + koff, IDESC, kk > 0 ? 1u : 0u);
            }
            mma_commit(&t_full[4 * b + h]);
            if (h == 3) mma_commit(&empty[s]);
          }
          __syncwarp();
        }
#if QR_WG_TMA_IN_MMA
        if (it + STAGES < nrows) {
          mbar_wait_backoff<32>(&empty[s], (uint32_t)((it / STAGES) & 1));
          if (lane == 0) issue_tma(it + STAGES);
          __syncwarp();
        }
#endif
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
    const int e = warp - EPI_WARP0;   // 0..15
    const int b = e >> 3;             // row buffer (rows it % 2 == b)
    const int g = (e >> 2) & 1;       // half of the row this warp's pass A / quant own
    const int qd = warp & 3;          // TMEM lane quarter
    const int w8 = e & 7;             // warp index within the buffer's 8
    const int L = qd * 32 + lane;     // TMEM lane = output j'
    const bool lane_ok = L < J;
    const bool odd = (lane & 1) != 0;
    const uint32_t t_lane = tmem_base + ((uint32_t)(qd * 32) << 16) + (uint32_t)(b * NA);
    const int bar_lanes = 1 + 4 * b + qd, bar_row = 9 + b;  // named barriers (0 = __syncthreads)
    const float norm_f = (float)rsqrt((double)K);
    const float c0 = (float)((double)clip * rsqrt((double)K) / 7.0);  // scale = c0 * amax
    for (int64_t it = b; it < nrows; it += 2) {
      const uint32_t par = (uint32_t)((it >> 1) & 1);
      const int64_t row = (int64_t)blockIdx.x + it * gridDim.x;
      // ---- pass A: quarters g and g + 2 (64 columns each, as soon as its MMA landed),
      //      bits 0-5 (pair i = columns 2i, 2i+1)
#pragma unroll 1
      for (int k = 0; k < 2; ++k) {
        const int qh = 2 * k + g;
        mbar_wait(&t_full[4 * b + qh], par);
        tc_fence_after();
        uint32_t r[2][32];
        QR_TMEM_LD32(t_lane + 64u * qh, r[0]);
        QR_TMEM_LD32(t_lane + 64u * qh + 32u, r[1]);
        tmem_ld_wait();
        float2 P[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          P[i] = make_float2(__uint_as_float(r[i >> 4][2 * (i & 15)]), __uint_as_float(r[i >> 4][2 * (i & 15) + 1]));
#pragma unroll
        for (int st = 1; st < 32; st <<= 1)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (!(i & st)) hqtc::bfly(P[i], P[i + st]);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          P[i] = pair_bfly(P[i]);  // bit 0
          r[i >> 4][2 * (i & 15)] = __float_as_uint(P[i].x);
          r[i >> 4][2 * (i & 15) + 1] = __float_as_uint(P[i].y);
        }
        QR_TMEM_ST32(t_lane + 64u * qh, r[0]);
        QR_TMEM_ST32(t_lane + 64u * qh + 32u, r[1]);
      }
      hqtc::tmem_st_wait();
      tc_fence_before();
      hqtc::bar_named(bar_lanes, 64);  // both halves of these lanes done with pass A
      tc_fence_after();
      // ---- pass B: bits 6, 7 over (c, c + 64, c + 128, c + 192), c in [32 g, 32 g + 32); amax
      float am = 0.f;
      const uint32_t tB = t_lane + (uint32_t)(32 * g);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // unrolled: TMEM addresses are immediate offsets
        const uint32_t tc0 = tB + (uint32_t)(8 * k);
        uint32_t u[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) QR_TMEM_LD8(tc0 + 64u * i, u[i]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float2 v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = make_float2(__uint_as_float(u[i][2 * c]), __uint_as_float(u[i][2 * c + 1]));
          hqtc::bfly(v[0], v[1]);  // bit 6
          hqtc::bfly(v[2], v[3]);
          hqtc::bfly(v[0], v[2]);  // bit 7
          hqtc::bfly(v[1], v[3]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            am = fmax_nan(am, fmax_nan(fabsf(v[i].x), fabsf(v[i].y)));
            u[i][2 * c] = __float_as_uint(v[i].x);
            u[i][2 * c + 1] = __float_as_uint(v[i].y);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) QR_TMEM_ST8(tc0 + 64u * i, u[i]);
      }
      float amax = lane_ok ? am : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (lane == 0) red[b][par][w8] = amax;
      hqtc::tmem_st_wait();
      tc_fence_before();
      hqtc::bar_named(bar_row, 256);  // the row's amax; pass B's TMEM stores of all 8 warps done
      tc_fence_after();
      amax = red[b][par][0];
#pragma unroll
      for (int w = 1; w < 8; ++w) amax = fmax_nan(amax, red[b][par][w]);
      // scale = fp32(clip * amax / (7 sqrt(K))) (readings Z5, Z9); zero row -> 1, non-finite -> NaN, codes 0
      float sc = 1.f, inv = 0.f;
      if (!isfinite(amax)) {
        sc = __int_as_float(0x7fc00000);
      } else if (amax != 0.f) {
        sc = c0 * amax;
        inv = __fdiv_rn(norm_f, sc);
      }
      if (w8 == 0 && lane == 0) scale[row] = sc;
      const bool zero = !isfinite(amax);  // non-finite row: all codes 0 (a zero row has inv = 0: codes 0)
      // am covers exactly the elements this thread quantizes below: if no lane of the warp can
      // reach |v * inv| >= 7.5 (fp32 rounding is monotone and 7.5 is exact), RNE lands in
      // [-7, 7] and the clamp is skipped (with clip 0.9 only the ~1-2 lanes of a row holding
      // elements above 0.964 amax take the clamping path)
      const bool clamp = __any_sync(0xffffffffu, am * inv >= 7.5f);
      uint8_t* const qrow = q + row * ld_q;
      // KPERM: chunk cc of lane L at byte (cc * J * 32 + L * 32) / 2; cc = g + 2 ch
      uint8_t* const qk = qrow + (int64_t)(g * J * 16 + L * 16);
      // ---- quant: the columns pass B produced, 32 columns (chunk cc = g + 2 ch: a_hi = 32 cc + r)
      //      at a time; each loaded chunk releases quarter ch of this warp's lanes to the MMA of row
      //      it + 2 (8 arrivals: both halves of the 4 lane quarters)
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const int cc = g + 2 * ch;
        uint32_t r[32];
        QR_TMEM_LD32(t_lane + 32u * cc, r);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[4 * b + ch]);
        float2 V[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) V[i] = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
        if constexpr (kPerm) {
          uint32_t w[4];
          if (clamp) {
#pragma unroll
            for (int t = 0; t < 4; ++t) w[t] = code_word8(V[4 * t], V[4 * t + 1], V[4 * t + 2], V[4 * t + 3], inv);
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) w[t] = code_word8_nc(V[4 * t], V[4 * t + 1], V[4 * t + 2], V[4 * t + 3], inv);
          }
          if (zero) w[0] = w[1] = w[2] = w[3] = 0u;
          if (lane_ok) *reinterpret_cast<uint4*>(qk + (int64_t)ch * (J * 32)) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
          // natural order: element (a_hi, j') at a_hi * 112 + j'; the byte of j' = 2p, 2p + 1 at
          // a_hi * 56 + p — even lanes keep words 0..3 (a_hi + 0..15), odd lanes 4..7 (+16..31)
          uint32_t w[8];
          if (clamp) {
#pragma unroll
            for (int m = 0; m < 8; ++m) w[m] = hqtc::code_word<true>(V[2 * m], V[2 * m + 1], inv);
          } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) w[m] = hqtc::code_word<false>(V[2 * m], V[2 * m + 1], inv);
          }
#pragma unroll
          for (int m = 0; m < 8; ++m)
            if (zero) w[m] = 0u;
          const uint32_t keep_mask = odd ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
          uint8_t* const qb = qrow + (L >> 1) + (int64_t)(32 * cc + (odd ? 16 : 0)) * (J / 2);
#pragma unroll
          for (int mm = 0; mm < 4; ++mm) {
            const uint32_t got = __shfl_xor_sync(0xffffffffu, odd ? w[mm] : w[mm + 4], 1);
            const uint32_t keep = odd ? w[mm + 4] : w[mm];
            const uint32_t o = odd ? (((keep << 4) & keep_mask) | (got & 0x0F0F0F0Fu))
                                   : ((keep & keep_mask) | ((got << 4) & 0xF0F0F0F0u));
            if (lane_ok) {
              uint8_t* dst = qb + (int64_t)(4 * mm) * (J / 2);
              dst[0] = (uint8_t)o;
              dst[J / 2] = (uint8_t)(o >> 8);
              dst[J] = (uint8_t)(o >> 16);
              dst[3 * J / 2] = (uint8_t)(o >> 24);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}
}  // namespace hqwg

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_hq() {
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

// (H_4 (x) H_28)[j'][j] (j' = a'_lo*28 + b' rows, j = a_lo*28 + b columns; row i of H_28
// dotted with x, reading Z4), zero-padded to 128 x 128 fp16 and laid out as the UMMA K-major
// SWIZZLE_128B image: atom column k/64 at 16 KB, 8-row groups at 1024 B, 128 B rows, 16-byte
// chunk c of row r at chunk c ^ (r & 7).
std::vector<uint16_t> a_image_28(const int8_t* h28) {
  std::vector<uint16_t> img(128 * 128, 0);
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < 128; ++k) {
      int v = 0;
      if (m < hqtc::J && k < hqtc::J) {
        const int alo_o = m / 28, bo = m % 28, alo_i = k / 28, bi = k % 28;
        const int sgn = (__builtin_popcount(alo_o & alo_i) & 1) ? -1 : 1;
        v = sgn * h28[bo * 28 + bi];
      }
      const int kc = k / 64, kk = k % 64, chunk = kk / 8, within = kk % 8;
      const size_t off = (size_t)kc * 16384 + (size_t)(m / 8) * 1024 + (size_t)(m % 8) * 128 +
                         (size_t)((chunk ^ (m % 8)) * 16) + (size_t)within * 2;
      img[off / 2] = v > 0 ? 0x3C00 : (v < 0 ? 0xBC00 : 0);
    }
  return img;
}

std::mutex g_img_mu;
void* g_img[64];
// the constant A image lives in static device memory (the library allocates none)
__device__ uint4 g_a28_img[hqtc::A_BYTES / 16];

}  // namespace

int g_hq_full_variant = 0;  // debug: 1 = the mma.sync kernel (hq_full28_kernel), 2 = spinning epilogue waits,
                            // 3 = the 16-warps-per-row tcgen05 kernel (hq_full28_tc_kernel)

namespace {
// the (H_4 (x) H_28) operand image in device memory (uploaded once per device) and the
// kernels' shared-memory attributes
cudaError_t a28_image(const void** img_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_img_mu);
  if (!g_img[dev & 63]) {
    const int8_t* h28 = base_hadamard_host(28);
    if (!h28) return cudaErrorInvalidValue;
    auto host = a_image_28(h28);
    void* d = nullptr;
    e = cudaGetSymbolAddress(&d, g_a28_img);
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(d, host.data(), host.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    e = cudaDeviceSynchronize();  // one-time: the image is complete before any stream reads it
    if (e != cudaSuccess) return e;
    for (auto kern : {hqtc::hq_full28_tc_kernel<false>, hqtc::hq_full28_tc_kernel<true>,
                      hqtc::hq_full28_tc_kernel<false, true>}) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hqtc::SMEM);
      if (e != cudaSuccess) return e;
    }
    for (auto kern : {hqwg::hq_full28_wg_kernel<false>, hqwg::hq_full28_wg_kernel<true>}) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hqwg::SMEM);
      if (e != cudaSuccess) return e;
    }
    g_img[dev & 63] = d;
  }
  *img_out = g_img[dev & 63];
  return cudaSuccess;
}

cudaError_t x_map_28(const void* x, int64_t M, int64_t ld_x, CUtensorMap* map) {
  auto fn = encode_fn_hq();
  if (!fn) return cudaErrorInvalidValue;
  cuuint64_t dims[3] = {(cuuint64_t)hqtc::J, (cuuint64_t)hqtc::NA, (cuuint64_t)M};
  cuuint64_t strides[2] = {(cuuint64_t)hqtc::J * 2, (cuuint64_t)ld_x * 2};
  cuuint32_t box[3] = {64u, (cuuint32_t)hqtc::NA, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(x), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_hq_full28_tc(const void* x, int64_t M, int64_t ld_x, float clip, uint8_t* q, int64_t ld_q,
                                float* scale, cudaStream_t stream, bool q8, bool kperm) {
  const void* img = nullptr;
  cudaError_t e = a28_image(&img);
  if (e != cudaSuccess) return e;
  if (M == 0) return cudaSuccess;  // quarot_prepare: one-time setup only
  CUtensorMap map;
  e = x_map_28(x, M, ld_x, &map);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(M < nsm ? M : nsm);
  const uint4* a = static_cast<const uint4*>(img);
  if (!q8 && (kperm || (g_hq_full_variant != 2 && g_hq_full_variant != 3))) {
    auto kern = kperm ? hqwg::hq_full28_wg_kernel<true> : hqwg::hq_full28_wg_kernel<false>;
    kern<<<grid, hqwg::NUM_THREADS, hqwg::SMEM, stream>>>(map, M, clip, q, ld_q, scale, a);
    return cudaPeekAtLastError();
  }
  auto kern = q8 ? hqtc::hq_full28_tc_kernel<false, true>
                 : (g_hq_full_variant == 2 ? hqtc::hq_full28_tc_kernel<true> : hqtc::hq_full28_tc_kernel<false>);
  kern<<<grid, hqtc::NUM_THREADS, hqtc::SMEM, stream>>>(map, M, clip, q, ld_q, scale, a);
  return cudaPeekAtLastError();
}

}  // namespace qr

extern "C" void quarot_debug_hq_full_variant(int32_t v) { qr::g_hq_full_variant = v; }
