// kv_quant_tc.cu — rows a6 + a7 (KV-cache Init) with the per-head Hadamard on the
// tcgen05 tensor path, for head_dim 128, n_kv in {4, 8, 16, 32, 64, 128}, n_q a multiple of
// n_kv, K rotated and V not (flags = KV_ROTATE_K), optionally with RoPE fused in front (§8 f1).
//
// Per-head H_128 (Eqs. 13-14) on a head vector is a row times H^T; 128 head vectors
// at once are one kind::f16 MMA: A = the rows (M = 128, K = d), B = H_128 (N = 128), D = fp32
// in TMEM (lane = row, column = d').  The inputs are fp16 (post-RoPE rounded to fp16, reading
// Z22), so the +-1 products are exact and the sums fp32, like the butterflies they replace.
//  * Work = token blocks of B_t = 128 / n_kv tokens: n_q / n_kv Q tiles, one K tile and one V
//    tile of 128 rows each (V is not rotated: the epilogue reads it straight from the stage).
//  * A TMA warp loads each tile (3-D maps [token][head][d], two 64-wide d boxes) straight into
//    the K-major SWIZZLE_128B operand layout, 3-stage ring.  With RoPE fused, eight warps rotate
//    the Q / K rows in place in shared memory (two threads per row) from a per-block cos/sin table
//    (fp64 sincos rounded to fp32, as quarot_rope; two table warps build it a block ahead into a
//    double buffer) and round to fp16; otherwise they only hand the stage to the MMA.
//  * Epilogue warps (thread = TMEM lane = row): Q rows scaled by 1/sqrt(128), rounded to fp16,
//    written into the (consumed) stage in the operand's SW128 layout and TMA-stored back in place
//    (the bulk tensor store writes whole lines; per-thread 16-byte row stores at a 256-byte lane
//    stride touched 32 half-used sectors per instruction); K / V rows quantized asymmetrically
//    (clip 0.95, group = the row, reading Z14) entirely in-thread: min / max, scale / zero, 64
//    code bytes in four 16-byte stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace kvtc {

constexpr int HD = 128;
constexpr int TILE_BYTES = 128 * HD * 2;  // 32 KB: 128 rows x 128 fp16, two SW128 atoms
#ifndef QR_KV_STAGES
#define QR_KV_STAGES 5  // 5 x 32 KB stages: +1% with RoPE (the RoPE pass holds a stage longer)
#endif
constexpr int STAGES = QR_KV_STAGES;
constexpr int NUM_EPI = 4, NUM_PROD = 8;  // two RoPE threads per tile row
constexpr int EPI_WARP0 = 0, PROD_WARP0 = 4, MMA_WARP = 12, TMA_WARP = 13, TAB_WARP0 = 14, NUM_TAB = 2;
constexpr int NUM_THREADS = 16 * 32;
constexpr int TBUF = 4;
constexpr uint32_t TMEM_COLS = 512;
constexpr int MAX_BT = 32;                                 // tokens per block (n_kv >= 4)
constexpr int TAB_BYTES = MAX_BT * (HD / 2) * 8;           // (cos, sin) per token and pair
constexpr size_t SMEM = 1024 + TILE_BYTES + (size_t)STAGES * TILE_BYTES + 2 * TAB_BYTES + 512 + (HD / 2) * 8;
static_assert(SMEM <= 232448, "227 KB dynamic smem");
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(HD >> 3) << 17) | ((128u >> 4) << 24);

struct Args {
  const __half* k;
  int64_t ld_k;
  const __half* v;
  int64_t ld_v;
  __half* q;
  int64_t ld_q;
  int64_t T;
  int n_kv, n_q;
  float clip;
  uint8_t *k_codes, *k_zero, *v_codes, *v_zero;
  float *k_scale, *v_scale;
  int64_t pos0;
  int seq_len;
  float theta;
};

QR_DEVICE void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(id), "r"(acc));
}
QR_DEVICE bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(p));
  return p != 0;
}
QR_DEVICE void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
QR_DEVICE void tma_store_3d(const CUtensorMap* map, int x, int y, int z, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z), "r"(src)
               : "memory");
}
QR_DEVICE void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
QR_DEVICE uint32_t sw128(int row, int d) {  // byte offset of element d of tile row `row`
  const int atom = d >> 6, chunk = (d & 63) >> 3;
  return (uint32_t)(atom * 16384 + (row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4) + (d & 7) * 2);
}

// tile j of a token block: 0 .. nQ-1 = Q tiles, nQ = K tile, nQ + 1 = V tile
struct TileInfo {
  int type;  // 0 Q, 1 K, 2 V
  int row0;  // first row within the block's rows of that type
};
QR_DEVICE TileInfo tile_info(int j, int nQ) {
  if (j < nQ) return {0, j * 128};
  return {j == nQ ? 1 : 2, 0};
}

template <bool kRope>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    kv_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const Args a, const uint4* __restrict__ b_img) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;                   // H_128 K-major SW128 image
  uint8_t* sA = sB + TILE_BYTES;        // [STAGES] tiles
  float2* tab = reinterpret_cast<float2*>(sA + STAGES * TILE_BYTES);  // [2][B_t][64] (cos, sin)
  uint64_t* a_full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tab) + 2 * TAB_BYTES);
  uint64_t* a_empty = a_full + STAGES;
  uint64_t* x_full = a_empty + STAGES;  // [STAGES] TMA landed
  uint64_t* t_full = x_full + STAGES;
  uint64_t* t_empty = t_full + TBUF;
  uint64_t* tab_full = t_empty + TBUF;  // [2] table warps -> RoPE warps
  uint64_t* tab_empty = tab_full + 2;   // [2] RoPE warps -> table warps
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tab_empty + 2);
  double* inv_freq = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(a_full) + 512);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BT = 128 / a.n_kv;          // tokens per block
  const int nQ = a.n_q / a.n_kv;        // Q tiles per block
  const int tpb = nQ + 2;               // tiles per block
  const int64_t nblocks = (a.T + BT - 1) / BT;
  const int64_t my_blocks = nblocks > (int64_t)blockIdx.x ? (nblocks - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t ntiles = my_blocks * tpb;

  for (int i = threadIdx.x; i < TILE_BYTES / 16; i += NUM_THREADS) reinterpret_cast<uint4*>(sB)[i] = __ldg(b_img + i);
  if (kRope)
    for (int i = threadIdx.x; i < HD / 2; i += NUM_THREADS) inv_freq[i] = pow((double)a.theta, -2.0 * (double)i / (double)HD);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&a_full[s], NUM_PROD);
      mbar_init(&a_empty[s], 1);
      mbar_init(&x_full[s], 1);
    }
    for (int b = 0; b < TBUF; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], NUM_EPI);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tab_full[b], NUM_TAB);
      mbar_init(&tab_empty[b], NUM_PROD);
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

  if (warp == TMA_WARP) {
    // ---------------------------------------------------------------- TMA: tile -> operand layout
    if (lane == 0) {
      for (int64_t it = 0; it < ntiles; ++it) {
        const int s = (int)(it % STAGES);
        const int64_t bi = it / tpb;
        const TileInfo ti = tile_info((int)(it % tpb), nQ);
        const int nh = ti.type == 0 ? a.n_q : a.n_kv;
        const int tok = (int)(((int64_t)blockIdx.x + bi * gridDim.x) * BT + ti.row0 / nh);
        const CUtensorMap* map = ti.type == 0 ? &tmQ : (ti.type == 1 ? &tmK : &tmV);
        mbar_wait_sleep(&a_empty[s], (uint32_t)((it / STAGES) & 1) ^ 1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&x_full[s])),
                     "r"(TILE_BYTES)
                     : "memory");
        const uint32_t dst = smem_u32(sA + s * TILE_BYTES);
        tma_load_3d(dst, map, 0, 0, tok, &x_full[s]);
        tma_load_3d(dst + 16384, map, 64, 0, tok, &x_full[s]);
      }
    }
  } else if (warp >= PROD_WARP0 && warp < PROD_WARP0 + NUM_PROD) {
    // ---------------------------------------------------------------- RoPE in place (Q, K rows)
    const int pt = (warp - PROD_WARP0) * 32 + lane;
    const int r = pt & 127, half = pt >> 7;  // tile row; pairs (i, i + 64) with i in [32 half, 32 half + 32)
    int64_t it = 0;
    for (int64_t bi = 0; bi < my_blocks; ++bi) {
      const int64_t t0 = ((int64_t)blockIdx.x + bi * gridDim.x) * BT;
      const float2* btab = tab + (bi & 1) * (TAB_BYTES / 8);  // this block's cos/sin table
      if (kRope) mbar_wait(&tab_full[bi & 1], (uint32_t)((bi >> 1) & 1));
      for (int j = 0; j < tpb; ++j, ++it) {
        const int s = (int)(it % STAGES);
        const TileInfo ti = tile_info(j, nQ);
        mbar_wait(&x_full[s], (uint32_t)((it / STAGES) & 1));
        if (kRope && ti.type != 2) {
          // RoPE rotate-half pairs (i, i + 64), rounded to fp16 (reading Z22)
          const int nh = ti.type == 0 ? a.n_q : a.n_kv;
          const int tl = (ti.row0 + r) / nh;  // token within the block
          const uint32_t cs = smem_u32(btab + tl * (HD / 2));  // ld.shared (a generic load takes the L1 tag path)
          const uint32_t row = smem_u32(sA + s * TILE_BYTES);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c = 4 * half + cc;
            const uint32_t plo = row + sw128(r, 8 * c), phi = row + sw128(r, 64 + 8 * c);
            uint4 lo4, hi4;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(lo4.x), "=r"(lo4.y), "=r"(lo4.z), "=r"(lo4.w) : "r"(plo));
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(hi4.x), "=r"(hi4.y), "=r"(hi4.z), "=r"(hi4.w) : "r"(phi));
            __half2* lo = reinterpret_cast<__half2*>(&lo4);
            __half2* hi = reinterpret_cast<__half2*>(&hi4);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 x1 = __half22float2(lo[e]), x2 = __half22float2(hi[e]);
              float4 c2;  // (cos, sin) of pairs i, i + 1
              asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                           : "=f"(c2.x), "=f"(c2.y), "=f"(c2.z), "=f"(c2.w)
                           : "r"(cs + (uint32_t)((8 * c + 2 * e) * 8)));
              // pairs i, i + 1 at once: c2 = (cos_i, cos_i+1, sin_i, sin_i+1); the packed forms are
              // rope_first / rope_second elementwise, bitwise quarot_rope's
              const float2 cv = make_float2(c2.x, c2.y), sv = make_float2(c2.z, c2.w);
              const float2 f = rope_first2(x1, x2, cv, sv);
              const float2 g = rope_second2(x1, x2, cv, sv);
              lo[e] = __floats2half2_rn(f.x, f.y);
              hi[e] = __floats2half2_rn(g.x, g.y);
            }
            sts_v4(plo, lo4);
            sts_v4(phi, hi4);
          }
          fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[s]);
      }
      if (kRope && lane == 0) mbar_arrive(&tab_empty[bi & 1]);  // this warp is done with the table
    }
  } else if (warp >= TAB_WARP0 && warp < TAB_WARP0 + NUM_TAB) {
    // ---------------------------------------------------------------- cos/sin tables, a block ahead
    if (kRope) {
      const int tt0 = (warp - TAB_WARP0) * 32 + lane;
      for (int64_t bi = 0; bi < my_blocks; ++bi) {
        const int64_t t0 = ((int64_t)blockIdx.x + bi * gridDim.x) * BT;
        float2* btab = tab + (bi & 1) * (TAB_BYTES / 8);
        mbar_wait_sleep(&tab_empty[bi & 1], (uint32_t)((bi >> 1) & 1) ^ 1u);
        for (int i = tt0; i < BT * (HD / 2); i += NUM_TAB * 32) {
          const int tt = i / (HD / 2), ii = i - tt * (HD / 2);
          const int64_t pos = (a.pos0 + t0 + tt) % a.seq_len;
          double sn, cn;
          sincos((double)pos * inv_freq[ii], &sn, &cn);  // == quarot_rope's table
          // layout per two pairs (2k, 2k + 1): (cos_2k, cos_2k+1, sin_2k, sin_2k+1) — the RoPE warps'
          // packed fp32x2 operands
          reinterpret_cast<float*>(btab)[tt * HD + (ii & ~1) * 2 + (ii & 1)] = (float)cn;
          reinterpret_cast<float*>(btab)[tt * HD + (ii & ~1) * 2 + 2 + (ii & 1)] = (float)sn;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tab_full[bi & 1]);
      }
    }
  } else if (warp == MMA_WARP) {
    // ---------------------------------------------------------------- MMA: D = rows x H^T (Q, K tiles)
    const uint32_t sa = smem_u32(sA), sb = smem_u32(sB);
    int64_t mt = 0;  // MMA tiles issued (the TMEM buffer ring)
    for (int64_t it = 0; it < ntiles; ++it) {
      const TileInfo ti = tile_info((int)(it % tpb), nQ);
      if (ti.type == 2) continue;  // V: not rotated, the epilogue reads the stage directly
      const int s = (int)(it % STAGES), tb = (int)(mt % TBUF);
      mbar_wait(&t_empty[tb], (uint32_t)((mt / TBUF) & 1) ^ 1u);
      mbar_wait(&a_full[s], (uint32_t)((it / STAGES) & 1));
      tc_fence_after();
      const uint64_t a_desc = umma_desc_sw128(sa + (uint32_t)(s * TILE_BYTES));
      const uint64_t b_desc = umma_desc_sw128(sb);
      const uint32_t d_tmem = tmem_base + (uint32_t)(tb * HD);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {  // atom kk/4 at +16 KB, +32 B per K = 16
          const uint64_t koff = (uint64_t)((kk >> 2) * (16384 >> 4) + 2 * (kk & 3));
          mma_f16(d_tmem, a_desc + koff, b_desc + koff, IDESC, kk > 0 ? 1u : 0u);
        }
        if (ti.type == 1) mma_commit(&a_empty[s]);  // K: the stage is free once read; Q: the
        mma_commit(&t_full[tb]);                     // epilogue reuses it for the TMA store
      }
      __syncwarp();
      ++mt;
    }
  } else if (warp < EPI_WARP0 + NUM_EPI) {
    // ---------------------------------------------------------------- epilogue: thread = row
    const int r = warp * 32 + lane;
    const uint32_t t_lane = tmem_base + ((uint32_t)(warp * 32) << 16);
    const double rnorm = rsqrt((double)HD);
    const float rn = (float)rnorm;
    int64_t mt = 0;  // MMA tiles consumed (the TMEM buffer ring)
    for (int64_t it = 0; it < ntiles; ++it) {
      const int s = (int)(it % STAGES);
      const int64_t bi = it / tpb;
      const TileInfo ti = tile_info((int)(it % tpb), nQ);
      const int64_t t0 = ((int64_t)blockIdx.x + bi * gridDim.x) * BT;
      const int nh = ti.type == 0 ? a.n_q : a.n_kv;
      const int rr = ti.row0 + r;
      const int tl = rr / nh, h = rr - tl * nh;
      const int64_t t = t0 + tl;
      const bool ok = t < a.T;
      const uint32_t stage = smem_u32(sA + s * TILE_BYTES);
      uint32_t u[HD / 2];  // one 64-column half of the row at a time (register budget)
      if (ti.type == 0) {  // Q: rotated, rounded to fp16 (Eq. 13), TMA-stored back in place
        const int tb = (int)(mt % TBUF);
        mbar_wait_sleep(&t_full[tb], (uint32_t)((mt / TBUF) & 1));
        tc_fence_after();
        const uint32_t tcol = t_lane + (uint32_t)(tb * HD);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          QR_TMEM_LD32(tcol + 64u * hf, u);
          QR_TMEM_LD32(tcol + 64u * hf + 32u, (u + 32));
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint4 w;
            __half2* hw = reinterpret_cast<__half2*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              hw[e] = __floats2half2_rn(__uint_as_float(u[8 * c + 2 * e]) * rn, __uint_as_float(u[8 * c + 2 * e + 1]) * rn);
            sts_v4(stage + sw128(r, 64 * hf + 8 * c), w);  // the MMA has read the stage (t_full)
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[tb]);
        ++mt;
        fence_proxy_async_smem();  // the rows' generic stores -> the TMA store (async proxy)
        bar_named(1, NUM_EPI * 32);
        if (threadIdx.x == EPI_WARP0 * 32) {
          const int tok = (int)(t0 + ti.row0 / nh);  // rows past T are clipped by the tensor map
          tma_store_3d(&tmQ, 0, 0, tok, stage);
          tma_store_3d(&tmQ, 64, 0, tok, stage + 16384);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read: the stage is free
          mbar_arrive(&a_empty[s]);
        }
        continue;
      }
      if (ti.type == 2) {
        // V: the row (128 fp16) is copied to registers as 64 packed half2 and the stage released
        // at once — the MHA shapes quantize two of every three tiles, and holding the V stage
        // through the whole quantization starved the TMA ring.  Asymmetric 4-bit quantization of
        // the row exactly as for K below (fp16 -> fp32 is exact), with norm = 1 (V not rotated).
        mbar_wait(&a_full[s], (uint32_t)((it / STAGES) & 1));  // landed (no RoPE on V)
        uint32_t hv[HD / 2];
#pragma unroll
        for (int c = 0; c < HD / 8; ++c)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(hv[4 * c]), "=r"(hv[4 * c + 1]), "=r"(hv[4 * c + 2]), "=r"(hv[4 * c + 3])
                       : "r"(stage + sw128(r, 8 * c)));
        bar_named(1, NUM_EPI * 32);  // every row of the V stage is in registers: release it
        if (threadIdx.x == EPI_WARP0 * 32) mbar_arrive(&a_empty[s]);
        auto h2 = [&](int k) { return *reinterpret_cast<const __half2*>(&hv[k]); };
        __half2 mn2[4] = {h2(0), h2(1), h2(2), h2(3)}, mx2[4] = {h2(0), h2(1), h2(2), h2(3)};
#pragma unroll
        for (int k = 4; k < HD / 2; ++k) {
          mn2[k & 3] = __hmin2_nan(mn2[k & 3], h2(k));
          mx2[k & 3] = __hmax2_nan(mx2[k & 3], h2(k));
        }
        const __half2 mnh = __hmin2_nan(__hmin2_nan(mn2[0], mn2[1]), __hmin2_nan(mn2[2], mn2[3]));
        const __half2 mxh = __hmax2_nan(__hmax2_nan(mx2[0], mx2[1]), __hmax2_nan(mx2[2], mx2[3]));
        const float mn = fmin_nan(__low2float(mnh), __high2float(mnh));
        const float mx = fmax_nan(__low2float(mxh), __high2float(mxh));
        const double lo = (double)a.clip * (double)fminf(mn, 0.f);
        const double hi = (double)a.clip * (double)fmaxf(mx, 0.f);
        float sc = 1.f, inv = 0.f;
        int z = 0;
        if (!(isfinite(mn) && isfinite(mx))) {
          sc = __int_as_float(0x7fc00000);
        } else if (hi != lo) {
          sc = (float)((hi - lo) / 15.0);
          const double zr = rint(-lo / (double)sc);
          z = (int)(zr < 0.0 ? 0.0 : (zr > 15.0 ? 15.0 : zr));
          inv = (float)(1.0 / (double)sc);
        }
        const int64_t gi = t * a.n_kv + h;
        const float zf = (float)z;
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = 0u;
        if (inv != 0.f) {
#pragma unroll
          for (int k = 0; k < HD / 2; ++k) {  // elements 2k, 2k + 1: one code byte
            float2 m = f2fma(__half22float2(h2(k)), make_float2(inv, inv), make_float2(zf, zf));
            m.x = fminf(fmaxf(m.x, 0.f), 15.f);
            m.y = fminf(fmaxf(m.y, 0.f), 15.f);
            m = f2add(m, make_float2(12582912.f, 12582912.f));
            const uint32_t byte = (__float_as_uint(m.x) & 0xFu) | ((__float_as_uint(m.y) & 0xFu) << 4);
            w[k >> 2] |= byte << (8 * (k & 3));
          }
        }
        if (ok) {
          uint4* codes = reinterpret_cast<uint4*>(a.v_codes + gi * (HD / 2));
#pragma unroll
          for (int c = 0; c < 4; ++c) codes[c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
          a.v_scale[gi] = sc;
          a.v_zero[gi] = (uint8_t)z;
        }
        continue;
      }
      // K: asymmetric 4-bit quantization of the row (group = head_dim, reading Z14) from TMEM
      // (rotated); the V branches below are no longer taken (V is handled above)
      int tb = 0;
      uint32_t tcol = 0;
      if (ti.type == 1) {
        tb = (int)(mt % TBUF);
        mbar_wait_sleep(&t_full[tb], (uint32_t)((mt / TBUF) & 1));
        tc_fence_after();
        tcol = t_lane + (uint32_t)(tb * HD);
      } else {
        mbar_wait(&a_full[s], (uint32_t)((it / STAGES) & 1));  // landed (no RoPE on V)
      }
      auto load_half = [&](int hf) {
        if (ti.type == 1) {
          QR_TMEM_LD32(tcol + 64u * hf, u);
          QR_TMEM_LD32(tcol + 64u * hf + 32u, (u + 32));
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint4 w;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                         : "r"(stage + sw128(r, 64 * hf + 8 * c)));
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ws[e]));
              u[8 * c + 2 * e] = __float_as_uint(f.x);
              u[8 * c + 2 * e + 1] = __float_as_uint(f.y);
            }
          }
        }
      };
      float mn4[4], mx4[4];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        load_half(hf);
        if (hf == 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) mn4[j] = mx4[j] = __uint_as_float(u[j]);
        }
#pragma unroll
        for (int j = 0; j < HD / 2; ++j) {
          mn4[j & 3] = fmin_nan(mn4[j & 3], __uint_as_float(u[j]));
          mx4[j & 3] = fmax_nan(mx4[j & 3], __uint_as_float(u[j]));
        }
      }
      const float mn = fmin_nan(fmin_nan(mn4[0], mn4[1]), fmin_nan(mn4[2], mn4[3]));
      const float mx = fmax_nan(fmax_nan(mx4[0], mx4[1]), fmax_nan(mx4[2], mx4[3]));
      const double norm = ti.type == 1 ? rnorm : 1.0;
      const double lo = (double)a.clip * (double)fminf(mn, 0.f) * norm;
      const double hi = (double)a.clip * (double)fmaxf(mx, 0.f) * norm;
      float sc = 1.f, inv = 0.f;
      int z = 0;
      if (!(isfinite(mn) && isfinite(mx))) {
        sc = __int_as_float(0x7fc00000);
      } else if (hi != lo) {
        sc = (float)((hi - lo) / 15.0);
        const double zr = rint(-lo / (double)sc);
        z = (int)(zr < 0.0 ? 0.0 : (zr > 15.0 ? 15.0 : zr));
        inv = (float)(norm / (double)sc);
      }
      const int64_t gi = t * a.n_kv + h;
      uint8_t* codes = (ti.type == 1 ? a.k_codes : a.v_codes) + gi * (HD / 2);
      const float zf = (float)z;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // the first half is reloaded (TMEM / smem reads are cheap)
        load_half(hf);
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = 0u;
        if (inv != 0.f) {
#pragma unroll
          for (int j = 0; j < HD / 2; j += 2) {
            // rne(x * inv) + z == rne(x * inv + z) (z integral); clamp to [0, 15]; magic-add RNE
            float2 m = f2fma(make_float2(__uint_as_float(u[j]), __uint_as_float(u[j + 1])), make_float2(inv, inv),
                             make_float2(zf, zf));
            m.x = fminf(fmaxf(m.x, 0.f), 15.f);
            m.y = fminf(fmaxf(m.y, 0.f), 15.f);
            m = f2add(m, make_float2(12582912.f, 12582912.f));
            const uint32_t byte = (__float_as_uint(m.x) & 0xFu) | ((__float_as_uint(m.y) & 0xFu) << 4);
            w[j >> 3] |= byte << (8 * ((j >> 1) & 3));
          }
        }
        if (ok) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
            reinterpret_cast<uint4*>(codes)[2 * hf + c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
        }
      }
      if (ti.type == 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[tb]);
        ++mt;
      } else {
        bar_named(1, NUM_EPI * 32);  // every row of the V stage read: release it
        if (threadIdx.x == EPI_WARP0 * 32) mbar_arrive(&a_empty[s]);
      }
      if (ok) {
        (ti.type == 1 ? a.k_scale : a.v_scale)[gi] = sc;
        (ti.type == 1 ? a.k_zero : a.v_zero)[gi] = (uint8_t)z;
      }
    }
    if (threadIdx.x == EPI_WARP0 * 32) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace kvtc

namespace {

// H_128 as the K-major SWIZZLE_128B image (rows = output d', K = input d): two atoms of
// 64 columns per matrix, 16-byte chunk c of row r at chunk c ^ (r & 7)
std::vector<uint16_t> b_images() {
  std::vector<uint16_t> img(kvtc::TILE_BYTES / 2, 0);
  for (int which = 0; which < 1; ++which)
    for (int r = 0; r < kvtc::HD; ++r)
      for (int k = 0; k < kvtc::HD; ++k) {
        const int v = which == 0 ? ((__builtin_popcount(r & k) & 1) ? -1 : 1) : (r == k ? 1 : 0);
        const int atom = k >> 6, chunk = (k & 63) >> 3;
        const size_t off = (size_t)which * kvtc::TILE_BYTES + (size_t)atom * 16384 + (size_t)(r >> 3) * 1024 +
                           (size_t)(r & 7) * 128 + (size_t)((chunk ^ (r & 7)) << 4) + (size_t)(k & 7) * 2;
        img[off / 2] = v > 0 ? 0x3C00 : (v < 0 ? 0xBC00 : 0);
      }
  return img;
}

std::mutex g_mu;
void* g_bimg[64];
// the constant B images live in static device memory (the library allocates none)
__device__ uint4 g_kv_bimg[kvtc::TILE_BYTES / 16];

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_kv() {
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

}  // namespace

bool kv_tc_supported(int n_kv, int head_dim, int n_q, uint32_t flags, const int32_t* positions) {
  auto p2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  return head_dim == kvtc::HD && n_kv >= 4 && n_kv <= 128 && p2(n_kv) && (n_q == 0 || (p2(n_q) && n_q <= 128)) &&
         n_q % n_kv == 0 && flags == 1u && positions == nullptr;
}

cudaError_t launch_kv_tc(const void* k, int64_t ld_k, const void* v, int64_t ld_v, int64_t T, int n_kv, void* q,
                         int64_t ld_q, int n_q, float clip, bool rope, int64_t pos0, int seq_len, float theta,
                         uint8_t* k_codes, float* k_scale, uint8_t* k_zero, uint8_t* v_codes, float* v_scale,
                         uint8_t* v_zero, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  void* img = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_bimg[dev & 63]) {
      auto host = b_images();
      void* d = nullptr;
      e = cudaGetSymbolAddress(&d, g_kv_bimg);
      if (e != cudaSuccess) return e;
      e = cudaMemcpy(d, host.data(), host.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return e;
      e = cudaDeviceSynchronize();  // one-time: the image is complete before any stream reads it
      if (e != cudaSuccess) return e;
      for (auto kern : {kvtc::kv_tc_kernel<false>, kvtc::kv_tc_kernel<true>}) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kvtc::SMEM);
        if (e != cudaSuccess) return e;
      }
      g_bimg[dev & 63] = d;
    }
    img = g_bimg[dev & 63];
  }
  if (T == 0) return cudaSuccess;  // quarot_prepare: one-time setup only
  kvtc::Args a;
  a.k = static_cast<const __half*>(k);
  a.ld_k = ld_k;
  a.v = static_cast<const __half*>(v);
  a.ld_v = ld_v;
  a.q = static_cast<__half*>(q);
  a.ld_q = ld_q;
  a.T = T;
  a.n_kv = n_kv;
  a.n_q = q ? n_q : 0;
  a.clip = clip;
  a.k_codes = k_codes;
  a.k_scale = k_scale;
  a.k_zero = k_zero;
  a.v_codes = v_codes;
  a.v_scale = v_scale;
  a.v_zero = v_zero;
  a.pos0 = pos0;
  a.seq_len = seq_len;
  a.theta = theta;
  auto fn = encode_fn_kv();
  if (!fn) return cudaErrorInvalidValue;
  // 3-D maps [token][head][d] (token stride ld, head stride 256 B), box {64 d, heads, tokens}
  auto make = [&](CUtensorMap* m, const void* base, int nh, int64_t ld) -> bool {
    const int nh_eff = nh > 0 ? nh : 1;
    cuuint64_t dims[3] = {(cuuint64_t)kvtc::HD, (cuuint64_t)nh_eff, (cuuint64_t)T};
    cuuint64_t strides[2] = {(cuuint64_t)kvtc::HD * 2, (cuuint64_t)(ld > 0 ? ld : kvtc::HD) * 2};
    cuuint32_t box[3] = {64u, (cuuint32_t)nh_eff, (cuuint32_t)(128 / nh_eff)};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  CUtensorMap mq, mk, mv;
  if (!make(&mk, k, n_kv, ld_k) || !make(&mv, v, n_kv, ld_v) || !make(&mq, q ? q : k, q ? n_q : n_kv, q ? ld_q : ld_k))
    return cudaErrorInvalidValue;
  const int BT = 128 / n_kv;
  const int64_t nblocks = (T + BT - 1) / BT;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(nblocks < nsm ? nblocks : nsm);
  if (grid == 0) return cudaSuccess;
  auto kern = rope ? kvtc::kv_tc_kernel<true> : kvtc::kv_tc_kernel<false>;
  kern<<<grid, kvtc::NUM_THREADS, kvtc::SMEM, stream>>>(mq, mk, mv, a, static_cast<const uint4*>(img));
  return cudaPeekAtLastError();
}

}  // namespace qr
