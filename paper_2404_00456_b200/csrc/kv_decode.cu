// kv_decode.cu — SURVEY §8 f2: routine 3 "Decode" of the paper's quantized attention:
// "computes the attention output using a quantized implementation of flash attention which can
// load the quantized cache and compute the final value vector" — one new query per sequence
// against the INT4 K/V cache (asymmetric, group = head_dim, x^ = (c - z) * s; Z14), with
// grouped-query attention (query head h reads KV head h / (n_q / n_kv)).
//
// Split-sequence flash decoding.  Grid (split, kv head, sequence); a CTA (4 warps) takes a
// chunk of 256 cache rows for one KV head and all G = n_q / n_kv query heads of its group;
// each warp takes 64 rows:
//  * scores on the INT8 tensor path: S[G x 8 rows] = Q[G x 128] . C^T with mma.sync m16n8k32
//    (A = the query as two int8 limbs, B = the codes as unsigned bytes, s32 accumulators);
//    the zero point and the scales are applied per row afterwards:
//    <q, k^> = s_k * (<q, c> - z * sum(q)).  The head dimension is permuted identically on both
//    operands so lane t of the fragment reads the 16 contiguous code bytes 16t .. 16t + 15 of
//    its row (one 16-byte load per row, 4 byte-permutes per 8 codes);
//  * online softmax per head (exp2, NaN-free masking of rows past the sequence length);
//  * P.V on the fp16 tensor path (mma.sync m16n8k16, fp32 accumulation): the score fragment of
//    two n-tiles IS the A fragment of one k-step (rows of the k-step = the 16 cache rows, the
//    FlashAttention-2 register reuse), holding p' = fp16(p * s_v); B = the V codes as exact fp16
//    1024 + c built in registers (PRMT + LOP3 per two codes) from 8-byte row chunks read straight
//    from global memory — lane g covers dims 16 g .. 16 g + 15 of every row, so n-tile j at
//    position g is dim 16 g + j; the zero point and the 1024 bias leave exactly as
//    sum_j p'_j (1024 + z_j), subtracted per head;
//  * the 4 warps merge in smem and the CTA writes one partial (m, l, o[128]) per query head;
//    kv_decode_combine merges the splits of a sequence (log-sum-exp) into fp16.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "quarot_internal.h"

#ifndef QR_DEC_CTAS_PER_SM
#define QR_DEC_CTAS_PER_SM 4  // target CTAs per SM of the split-sequence grid
#endif

namespace qr {
namespace kvd {

constexpr int HD = 128;             // head_dim (the paper's: 128 for every Llama-2 size)
constexpr int WARPS = 8;
constexpr int ROWS_PER_WARP = 32;
constexpr int CHUNK = WARPS * ROWS_PER_WARP;  // cache rows per chunk (one ring stage)
constexpr int STAGES = 3;
constexpr int STAGE_BYTES = 2 * CHUNK * 64;   // K and V codes of a chunk: 32 KB
// the ring, then (after the last chunk, aliased onto it) the warps' merge records; barriers and
// the query fragments behind it
template <int G>
constexpr size_t smem_bytes() {
  static_assert((size_t)WARPS * G * (HD + 4) * 4 <= (size_t)STAGES * STAGE_BYTES, "merge records fit the ring");
  return (size_t)STAGES * STAGE_BYTES + 2 * STAGES * 8 + 32 * 20 * 4;  // ring, full[], done[], qfrag
}
constexpr float LOG2E = 1.4426950408889634f;

QR_DEVICE void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// D (s32) += A (s8, 16 x 32) . B (u8, 32 x 8)
QR_DEVICE void imma16832(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// fp16_rn(lo) | fp16_rn(hi) << 16
QR_DEVICE uint32_t pack_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// byte i of the word pair (lo4, hi4) -> fp16x2 (lo nibble - 8, hi nibble - 8), exact
QR_DEVICE uint32_t nib2half2(uint32_t lo4, uint32_t hi4, int i) {
  const uint32_t m = __byte_perm(lo4, hi4, (uint32_t)i | ((uint32_t)(4 + i) << 8));
  uint32_t h = (m & 0x00FF00FFu) | 0x64006400u;  // fp16 1024 + c
  const uint32_t bias = 0x64086408u;             // fp16 1032
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(h) : "r"(h), "r"(bias));
  return h;
}

struct Args {
  const __half* q;  // [B][n_q][HD], rotated (Eq. 13)
  const uint8_t* kc;
  const float* ks;
  const uint8_t* kz;
  const uint8_t* vc;
  const float* vs;
  const uint8_t* vz;
  const int32_t* seq_lens;
  int n_q, n_kv, s_max, nsplit, chunks_per_cta;  // nsplit = CTAs per (sequence, KV head)
  float sm_scale_log2;  // sm_scale * log2(e)
  float* ws;            // [B][n_q][nsplit][HD + 2]: o (HD), m, l
  __half* out;          // [B][n_q][HD]: written directly when nsplit == 1 (no combine pass)
};

// Barriers of the chunk ring (static smem so the kernel needs no dynamic-smem attribute games)
QR_DEVICE void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <int G>
__global__ void __launch_bounds__(WARPS * 32, 2)
    kv_decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Args a) {
  static_assert(G <= 8, "query heads per KV head: the fragments hold 8");
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int L = __ldg(a.seq_lens + b);
  // this CTA's chunks of CHUNK rows: [c0, c1), clipped to the sequence length
  const int nch_all = (L + CHUNK - 1) / CHUNK;
  const int c0 = split * a.chunks_per_cta, c1 = min(nch_all, c0 + a.chunks_per_cta);
  const int nch = max(0, c1 - c0);
  const int64_t grp0 = ((int64_t)b * a.s_max) * a.n_kv + kvh;  // group index of row 0
  const int64_t kvrow_stride = (int64_t)a.n_kv;

  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* ring = dsm;                                            // [STAGES][K 16 KB | V 16 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + STAGES * STAGE_BYTES);
  uint32_t* done = reinterpret_cast<uint32_t*>(full + STAGES);                         // [STAGES] warps done
  uint32_t (*qfrag_s)[20] = reinterpret_cast<uint32_t (*)[20]>(full + 2 * STAGES);    // [32][20]
  float (*mrg_s)[G][HD + 4] = reinterpret_cast<float (*)[G][HD + 4]>(dsm);           // [WARPS][G][HD + 4], after the loop

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0u;
    }
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
  }
  __syncthreads();
  // producer: chunk j -> stage j % STAGES.  Chunks 0 .. STAGES-1 are issued by thread 0 up front;
  // chunk j + STAGES by the LAST warp to finish chunk j (a shared counter per stage), so no warp
  // ever waits for another to free a stage
  auto produce = [&](int j) {
    const int s = j % STAGES;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"((uint32_t)STAGE_BYTES)
                 : "memory");
    const int row = (int)((int64_t)b * a.s_max + (int64_t)(c0 + j) * CHUNK);
    tma_load_3d(smem_u32(ring + s * STAGE_BYTES), &tmK, 0, kvh, row, &full[s]);
    tma_load_3d(smem_u32(ring + s * STAGE_BYTES + CHUNK * 64), &tmV, 0, kvh, row, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int j = 0; j < min(nch, STAGES); ++j) produce(j);

  // ---- query fragments: IMMA rows g = head g's high limb, rows g + 8 = its low limb.  The fp16
  // query is split into two int8 limbs, q ~= s_q (q_hi + q_lo / 256) with s_q = max|q| / 127
  // (error <= s_q / 512 per element, ~2^-16 relative), so one m16n8k32 IMMA gives both limbs' dot
  // products with the codes (unsigned bytes) and the scores run on the INT8 tensor path; dims
  // permuted as in the header.  Warp 0 builds them once per CTA; every warp reads its lane's copy.
  if (warp == 0) {
    float f[32];
    if (g < G) {
      const uint4* src = reinterpret_cast<const uint4*>(a.q + ((int64_t)b * a.n_q + kvh * G + g) * HD + 32 * t);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 u = __ldg(src + c);
        const uint32_t uw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 ff = __half22float2(*reinterpret_cast<const __half2*>(&uw[e]));
          f[8 * c + 2 * e] = ff.x;
          f[8 * c + 2 * e + 1] = ff.y;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) f[e] = 0.f;
    }
    float mx = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e) mx = fmaxf(mx, fabsf(f[e]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float sq = mx > 0.f ? mx / 127.f : 1.f;
    const float inv = 1.f / sq;
    int sum_hi = 0, sum_lo = 0;
    uint32_t fr[16];
#pragma unroll
    for (int w4 = 0; w4 < 8; ++w4) {  // 4 dims per register: dims 32t + 4 w4 .. + 3
      uint32_t hw = 0, lw = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = f[4 * w4 + e];
        const int h = __float2int_rn(x * inv);
        int l = __float2int_rn((x - (float)h * sq) * inv * 256.f);
        l = max(-127, min(127, l));
        sum_hi += h;
        sum_lo += l;
        hw |= (uint32_t)(h & 0xFF) << (8 * e);
        lw |= (uint32_t)(l & 0xFF) << (8 * e);
      }
      // k-step ks = w4 / 2: a0 / a1 (rows g / g + 8) hold k 4t..4t+3 (dims 32t + 8 ks + 0..3),
      // a2 / a3 hold k 16 + 4t .. (dims 32t + 8 ks + 4..7)
      fr[4 * (w4 >> 1) + 2 * (w4 & 1)] = hw;
      fr[4 * (w4 >> 1) + 2 * (w4 & 1) + 1] = lw;
    }
    float sm = (float)sum_hi + (float)sum_lo * (1.f / 256.f);
    sm += __shfl_xor_sync(0xffffffffu, sm, 1);
    sm += __shfl_xor_sync(0xffffffffu, sm, 2);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<uint4*>(&qfrag_s[lane][4 * i]) = make_uint4(fr[4 * i], fr[4 * i + 1], fr[4 * i + 2], fr[4 * i + 3]);
    qfrag_s[lane][16] = __float_as_uint(sq);
    qfrag_s[lane][17] = __float_as_uint(sm);  // in units of s_q
  }
  __syncthreads();  // qfrag_s
  uint32_t qa[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 v = *reinterpret_cast<const uint4*>(&qfrag_s[lane][4 * i]);
    qa[i][0] = v.x, qa[i][1] = v.y, qa[i][2] = v.z, qa[i][3] = v.w;
  }
  const float qs = __uint_as_float(qfrag_s[lane][16]), qsum = __uint_as_float(qfrag_s[lane][17]);

  // per-row scales / zero points of lane = row (warp * 32 + lane) of a chunk, loaded one chunk
  // ahead and converted only when used (the conversion would wait for the load)
  struct RowRaw {
    float ks, vs;
    uint32_t kz, vz;
  };
  auto ld_rowp = [&](int j) {
    const int row = (c0 + j) * CHUNK + warp * ROWS_PER_WARP + lane;
    RowRaw r{0.f, 0.f, 8u, 0u};
    if (j < nch && row < L) {
      const int64_t gi = grp0 + (int64_t)row * kvrow_stride;
      r.ks = __ldg(a.ks + gi);
      r.kz = __ldg(a.kz + gi);
      r.vs = __ldg(a.vs + gi);
      r.vz = __ldg(a.vz + gi);
    }
    return r;
  };
  RowRaw rp_next = ld_rowp(0);

  // running online-softmax state of this warp: head g's (m, l, zsum); o^T fragments (heads 2t, 2t+1)
  float m_run = -INFINITY, l_run = 0.f, z_run = 0.f;
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

  for (int j = 0; j < nch; ++j) {
    const float4 rp_mine = make_float4(rp_next.ks * a.sm_scale_log2, (float)rp_next.kz, rp_next.vs, (float)rp_next.vz);
    rp_next = ld_rowp(j + 1);
    const int s = j % STAGES;
    const int row0 = (c0 + j) * CHUNK + warp * ROWS_PER_WARP;  // this warp's first row of the chunk
    mbar_wait(&full[s], (uint32_t)((j / STAGES) & 1));
    const uint8_t* kst = ring + s * STAGE_BYTES + warp * ROWS_PER_WARP * 64;  // [32 rows][64 B] K codes
    const uint8_t* vst = kst + CHUNK * 64;                                    // V codes
    // ---- scores: 4 n-tiles of 8 rows; head g (fragment row g), rows 8 nt + 2t + jj
    float sc[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const uint4 kw = *reinterpret_cast<const uint4*>(kst + (nt * 8 + g) * 64 + 16 * t);
      const uint32_t wv[4] = {kw.x, kw.y, kw.z, kw.w};
      int acc[4] = {0, 0, 0, 0};  // rows g: <q_hi, c>, rows g + 8: <q_lo, c>
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        // the lane's code bytes 4 ks .. 4 ks + 3 = dims 32t + 8 ks + 0..7, split into unsigned
        // bytes [lo, hi, lo, hi]: b0 = dims +0..3 (bytes 4ks, 4ks+1), b1 = dims +4..7
        const uint32_t lo4 = wv[ks] & 0x0F0F0F0Fu, hi4 = (wv[ks] >> 4) & 0x0F0F0F0Fu;
        const uint32_t b0 = __byte_perm(lo4, hi4, 0x5140), b1 = __byte_perm(lo4, hi4, 0x7362);
        imma16832(acc, qa[ks], b0, b1);
      }
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int rl = nt * 8 + 2 * t + jj;
        const float sk = __shfl_sync(0xffffffffu, rp_mine.x, rl), zk = __shfl_sync(0xffffffffu, rp_mine.y, rl);
        const float dot = (float)acc[jj] + (float)acc[2 + jj] * (1.f / 256.f);
        sc[nt][jj] = row0 + rl < L ? (dot - zk * qsum) * (qs * sk) : -INFINITY;
      }
    }
    // ---- online softmax for head g
    float mc = m_run;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) mc = fmaxf(mc, fmaxf(sc[nt][0], sc[nt][1]));
    mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 1));
    mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, 2));
    const float alpha = (mc == -INFINITY) ? 1.f : exp2f(m_run - mc);  // m_run = -inf -> 0
    m_run = mc;
    float lc = 0.f, zc = 0.f;
    uint32_t pb[2][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      float pv[2];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int rl = nt * 8 + 2 * t + jj;
        const float sv = __shfl_sync(0xffffffffu, rp_mine.z, rl), zv = __shfl_sync(0xffffffffu, rp_mine.w, rl);
        const float p = (mc == -INFINITY) ? 0.f : exp2f(sc[nt][jj] - mc);
        lc += p;
        const float ph = __half2float(__float2half_rn(p * sv));
        zc += ph * (zv + 1024.f);
        pv[jj] = ph;
      }
      pb[nt >> 1][nt & 1] = pack_h2(pv[0], pv[1]);
    }
    lc += __shfl_xor_sync(0xffffffffu, lc, 1);
    lc += __shfl_xor_sync(0xffffffffu, lc, 2);
    zc += __shfl_xor_sync(0xffffffffu, zc, 1);
    zc += __shfl_xor_sync(0xffffffffu, zc, 2);
    l_run = l_run * alpha + lc;
    z_run = z_run * alpha + zc;
    // rescale o^T: its columns are heads 2t, 2t+1, whose alpha lives in lanes g = 2t, 2t+1
    const float a0 = __shfl_sync(0xffffffffu, alpha, 4 * ((2 * t) & 7)),
                a1 = __shfl_sync(0xffffffffu, alpha, 4 * ((2 * t + 1) & 7));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i][0] *= a0, o[i][2] *= a0;
      o[i][1] *= a1, o[i][3] *= a1;
    }
    // ---- P.V as O^T = V^T P^T: 2 k-steps x 8 m-tiles of mma.sync m16n8k16.  m-tile i rows g /
    // g + 8 are dims 16 g + 2 i / 16 g + 2 i + 1 (the two nibbles of byte i of the lane's chunk);
    // D element (i, c) of lane (g, t) is dim 16 g + 2 i + (c >= 2), head 2 t + (c & 1)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      uint32_t lo[4][2], hi[4][2];  // [row r][word]: nibble planes of rows 16 kk + {2t, 2t+1, 2t+8, 2t+9}
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int rl = 16 * kk + 2 * t + (r & 1) + 8 * (r >> 1);
        const uint2 vw = *reinterpret_cast<const uint2*>(vst + rl * 64 + 8 * g);
        lo[r][0] = vw.x & 0x0F0F0F0Fu, hi[r][0] = (vw.x >> 4) & 0x0F0F0F0Fu;
        lo[r][1] = vw.y & 0x0F0F0F0Fu, hi[r][1] = (vw.y >> 4) & 0x0F0F0F0Fu;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int w = i >> 2, by = i & 3;
        const uint32_t sel = (uint32_t)by | ((uint32_t)(4 + by) << 8);
        // a0 = (dim 16g+2i, rows 2t, 2t+1), a1 = (dim +1, rows 2t, 2t+1), a2 / a3 = rows 2t+8, 2t+9;
        // fp16 1024 + c, exact
        uint32_t af[4];
        af[0] = (__byte_perm(lo[0][w], lo[1][w], sel) & 0x000F000Fu) | 0x64006400u;
        af[1] = (__byte_perm(hi[0][w], hi[1][w], sel) & 0x000F000Fu) | 0x64006400u;
        af[2] = (__byte_perm(lo[2][w], lo[3][w], sel) & 0x000F000Fu) | 0x64006400u;
        af[3] = (__byte_perm(hi[2][w], hi[3][w], sel) & 0x000F000Fu) | 0x64006400u;
        mma16816(o[i], af, pb[kk][0], pb[kk][1]);
      }
    }
    __syncwarp();
    if (lane == 0) {  // this warp is done with the stage; the last one refills it with chunk j + STAGES
      const uint32_t n = atomicAdd(&done[s], 1u);
      if (n == (uint32_t)(WARPS * (j / STAGES + 1) - 1) && j + STAGES < nch) produce(j + STAGES);
    }
  }
  // ---- merge the warps: each writes (o - zsum, m, l) per head into its record (over the ring:
  // every warp must be done with its last chunk first); head 2t + e's zsum lives in the lanes
  // with g = 2t + e
  float zs[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) zs[e] = __shfl_sync(0xffffffffu, z_run, 4 * ((2 * t + e) & 7));
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int r = 2 * t + e;
    if (r < G) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mrg_s[warp][r][16 * g + 2 * i] = o[i][e] - zs[e];
        mrg_s[warp][r][16 * g + 2 * i + 1] = o[i][2 + e] - zs[e];
      }
    }
  }
  if (t == 0 && g < G) {
    mrg_s[warp][g][HD] = m_run;
    mrg_s[warp][g][HD + 1] = l_run;
  }
  __syncthreads();
  // thread = (head r, dim d): 256 threads cover two heads per pass
  for (int rr = 0; rr < G; rr += WARPS * 32 / HD) {
    const int r = rr + (int)(threadIdx.x / HD), d = (int)(threadIdx.x % HD);
    if (r >= G) break;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, mrg_s[w][r][HD]);
    float O = 0.f, Ls = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float mw = mrg_s[w][r][HD];
      const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      O += f * mrg_s[w][r][d];
      Ls += f * mrg_s[w][r][HD + 1];
    }
    if (a.nsplit == 1) {  // one CTA per (sequence, KV head): the combine pass's arithmetic, here
      a.out[((int64_t)b * a.n_q + kvh * G + r) * HD + d] = __float2half_rn(O / Ls);
      continue;
    }
    float* dst = a.ws + (((int64_t)b * a.n_q + kvh * G + r) * a.nsplit + split) * (HD + 2);
    dst[d] = O;
    if (d == 0) {
      dst[HD] = M;
      dst[HD + 1] = Ls;
    }
  }
}

// one CTA per (sequence, query head), thread = dim: merge the splits, apply the value
// scale (already in p * s_v) and round to fp16
__global__ void __launch_bounds__(HD) kv_decode_combine(const float* __restrict__ ws, int nsplit, int n_q,
                                                        __half* __restrict__ out) {
  const int64_t bh = blockIdx.x;  // b * n_q + h
  const float* src = ws + bh * nsplit * (HD + 2);
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, src[s * (HD + 2) + HD]);
  float O = 0.f, Ls = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float ms = src[s * (HD + 2) + HD];
    const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
    O += f * src[s * (HD + 2) + threadIdx.x];
    Ls += f * src[s * (HD + 2) + HD + 1];
  }
  out[bh * HD + threadIdx.x] = __float2half_rn(O / Ls);
}

}  // namespace kvd

int64_t kv_decode_workspace_bytes(int64_t B, int64_t n_q, int64_t head_dim, int64_t s_max) {
  const int64_t nsplit = (s_max + kvd::CHUNK - 1) / kvd::CHUNK;
  return B * n_q * nsplit * (head_dim + 2) * (int64_t)sizeof(float);
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_dec() {
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
// the cache's codes as [B * s_max rows][n_kv][64 B]; box = one chunk of one KV head (256 x 64 B)
bool cache_map(CUtensorMap* m, const uint8_t* codes, int64_t rows, int n_kv) {
  auto fn = encode_fn_dec();
  if (!fn) return false;
  cuuint64_t dims[3] = {64u, (cuuint64_t)n_kv, (cuuint64_t)rows};
  cuuint64_t strides[2] = {64u, (cuuint64_t)n_kv * 64u};
  cuuint32_t box[3] = {64u, 1u, (cuuint32_t)kvd::CHUNK};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(codes), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <int G>
cudaError_t launch_g(dim3 grid, const CUtensorMap& mk, const CUtensorMap& mv, const kvd::Args& a, cudaStream_t st) {
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kvd::kv_decode_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kvd::smem_bytes<G>());
    if (e != cudaSuccess) return e;
    attr[dev & 63] = true;
  }
  kvd::kv_decode_kernel<G><<<grid, kvd::WARPS * 32, kvd::smem_bytes<G>(), st>>>(mk, mv, a);
  return cudaSuccess;
}
}  // namespace

cudaError_t launch_kv_decode(const void* q, const uint8_t* k_codes, const float* k_scale, const uint8_t* k_zero,
                             const uint8_t* v_codes, const float* v_scale, const uint8_t* v_zero,
                             const int32_t* seq_lens, int B, int n_q, int n_kv, int head_dim, int s_max,
                             float sm_scale, void* out, float* workspace, cudaStream_t stream, int* launches) {
  if (B == 0) return cudaSuccess;
  CUtensorMap mk, mv;
  const int64_t rows = (int64_t)B * s_max;
  if (!cache_map(&mk, k_codes, rows, n_kv) || !cache_map(&mv, v_codes, rows, n_kv)) return cudaErrorInvalidValue;
  kvd::Args a;
  a.q = static_cast<const __half*>(q);
  a.kc = k_codes;
  a.ks = k_scale;
  a.kz = k_zero;
  a.vc = v_codes;
  a.vs = v_scale;
  a.vz = v_zero;
  a.seq_lens = seq_lens;
  a.n_q = n_q;
  a.n_kv = n_kv;
  a.s_max = s_max;
  // CTAs per (sequence, KV head): enough CTAs for ~4 per SM, each streaming >= 1 chunk
  const int nchunks = (s_max + kvd::CHUNK - 1) / kvd::CHUNK;
  int nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pairs = (int64_t)B * n_kv;
  // target CTAs per SM: when there are already >= 2 (sequence, KV head) pairs per SM, 2 (fewer,
  // longer CTAs: the 70B GQA batch-64 shape runs one CTA per pair, 0.064 -> 0.060 ms); otherwise
  // QR_DEC_CTAS_PER_SM (4: small batches need the split for parallelism)
  const int64_t target = pairs >= 2 * (int64_t)nsm ? 2 : QR_DEC_CTAS_PER_SM;
  int per = (int)((target * nsm + pairs - 1) / pairs);
  per = per < 1 ? 1 : (per > nchunks ? nchunks : per);
  a.chunks_per_cta = (nchunks + per - 1) / per;
  a.nsplit = (nchunks + a.chunks_per_cta - 1) / a.chunks_per_cta;
  a.sm_scale_log2 = sm_scale * kvd::LOG2E;
  a.ws = workspace;
  a.out = static_cast<__half*>(out);
  const dim3 grid(a.nsplit, n_kv, B);
  const int G = n_q / n_kv;
  cudaError_t e;
  switch (G) {
    case 1: e = launch_g<1>(grid, mk, mv, a, stream); break;
    case 2: e = launch_g<2>(grid, mk, mv, a, stream); break;
    case 4: e = launch_g<4>(grid, mk, mv, a, stream); break;
    case 8: e = launch_g<8>(grid, mk, mv, a, stream); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  if (launches) *launches = a.nsplit > 1 ? 2 : 1;
  if (a.nsplit == 1) return cudaSuccess;  // the decode kernel wrote the output
  kvd::kv_decode_combine<<<(unsigned)((int64_t)B * n_q), kvd::HD, 0, stream>>>(workspace, a.nsplit, n_q,
                                                                              static_cast<__half*>(out));
  return cudaPeekAtLastError();
}

}  // namespace qr
