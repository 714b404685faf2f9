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
//  * P.V on CUDA cores: lane owns 4 dimensions; o += (p * s_v) * c per row, and the zero point
//    enters once per head as sum_j (p_j s_vj) z_vj;
//  * the 4 warps merge in smem and the CTA writes one partial (m, l, o[128]) per query head;
//    kv_decode_combine merges the splits of a sequence (log-sum-exp) into fp16.
#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace kvd {

constexpr int HD = 128;             // head_dim (the paper's: 128 for every Llama-2 size)
constexpr int WARPS = 4;
constexpr int ROWS_PER_WARP = 64;
constexpr int CHUNK = WARPS * ROWS_PER_WARP;  // cache rows per CTA
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
  int n_q, n_kv, s_max, nsplit;
  float sm_scale_log2;  // sm_scale * log2(e)
  float* ws;            // [B][n_q][nsplit][HD + 2]: o (HD), m, l
};

template <int G>
__global__ void __launch_bounds__(WARPS * 32) kv_decode_kernel(Args a) {
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int L = __ldg(a.seq_lens + b);
  const int row0 = split * CHUNK + warp * ROWS_PER_WARP;
  const int64_t kvrow_stride = (int64_t)a.n_kv;  // rows of one sequence are s_max * n_kv groups
  const int64_t grp0 = ((int64_t)b * a.s_max) * a.n_kv + kvh;  // group index of row 0

  // per-warp buffer: the warp's V code rows [64][HD/2] and p * s_v [64][G] during the warp's
  // own work, then (aliased) its merge record o[G][HD + 4] (+ m, l) for the CTA combine
  constexpr int VC_BYTES = ROWS_PER_WARP * (HD / 2);
  constexpr int WB_WORK = VC_BYTES + ROWS_PER_WARP * G * 4, WB_MRG = G * (HD + 4) * 4;
  constexpr int WB = WB_WORK > WB_MRG ? WB_WORK : WB_MRG;
  __shared__ __align__(16) uint8_t wbuf[WARPS][WB];
  __shared__ float4 rowp_s[WARPS][ROWS_PER_WARP];      // (s_k * sm_scale_log2, z_k, s_v, z_v) per row
  uint8_t (*vcode_w)[HD / 2] = reinterpret_cast<uint8_t (*)[HD / 2]>(wbuf[warp]);
  float (*p_w)[G] = reinterpret_cast<float (*)[G]>(wbuf[warp] + VC_BYTES);
  auto mrg = [&](int w, int r) -> float* { return reinterpret_cast<float*>(wbuf[w]) + r * (HD + 4); };

  // ---- prologue: every load of the warp's 64 rows is issued before any is consumed
  //  V codes: 16-byte cp.async chunks (row = lane / 4 + 8 i, part = lane % 4), zero-filled
  //  past the sequence; per-row scales / zeros into smem; K code chunks into registers
  {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rl = (lane >> 2) + 8 * i, row = row0 + rl;
      const bool ok = row < L;
      const uint8_t* src = a.vc + (grp0 + (int64_t)(ok ? row : 0) * kvrow_stride) * (HD / 2) + 16 * (lane & 3);
      const uint32_t dst = smem_u32(&vcode_w[rl][16 * (lane & 3)]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int rl = lane + 32 * i, row = row0 + rl;
      float4 rp = make_float4(0.f, 8.f, 0.f, 0.f);
      if (row < L) {
        const int64_t gi = grp0 + (int64_t)row * kvrow_stride;
        rp = make_float4(__ldg(a.ks + gi) * a.sm_scale_log2, (float)__ldg(a.kz + gi), __ldg(a.vs + gi),
                         (float)__ldg(a.vz + gi));
      }
      rowp_s[warp][rl] = rp;
    }
  }
  uint4 kw_all[8];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int rowB = row0 + nt * 8 + g;  // the row this lane feeds into the B fragment
    kw_all[nt] = make_uint4(0, 0, 0, 0);
    if (rowB < L)
      kw_all[nt] = __ldg(reinterpret_cast<const uint4*>(a.kc + (grp0 + (int64_t)rowB * kvrow_stride) * (HD / 2)) + t);
  }

  // ---- query fragments (rows r = g, g + 8 of the head group; dims permuted, see header).
  // The fp16 query is split into two int8 limbs, q ~= s_q (q_hi + q_lo / 256) with
  // s_q = max|q| / 127 (error <= s_q / 512 per element, ~2^-16 relative), so the scores run on
  // the INT8 tensor path with the codes as unsigned bytes (no per-code fp16 conversion).
  // warp 0 builds the fragments once for the CTA; every warp then reads its lane's copy
  __shared__ __align__(16) uint32_t qfrag_s[32][36];  // [lane]: qhi 16 | qlo 16 | qs 2 | qsum 2
  uint32_t qhi[4][4], qlo[4][4];  // [k-step][a0..a3]
  float qs[2], qsum[2];           // s_q and sum(q~) of rows g, g + 8
  if (warp == 0) {
  #pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int r = g + 8 * hh;
      float f[32];
      if (r < G) {
        const uint4* src = reinterpret_cast<const uint4*>(a.q + ((int64_t)b * a.n_q + kvh * G + r) * HD + 32 * t);
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
        // k-step ks = w4 / 2: a0 / a1 hold k 4t..4t+3 (dims 32t + 8 ks + 0..3), a2 / a3 hold
        // k 16 + 4t .. (dims 32t + 8 ks + 4..7)
        qhi[w4 >> 1][(w4 & 1) * 2 + hh] = hw;
        qlo[w4 >> 1][(w4 & 1) * 2 + hh] = lw;
      }
      float sm = (float)sum_hi + (float)sum_lo * (1.f / 256.f);
      sm += __shfl_xor_sync(0xffffffffu, sm, 1);
      sm += __shfl_xor_sync(0xffffffffu, sm, 2);
      qs[hh] = sq;
      qsum[hh] = sm;  // in units of s_q
    }

#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      *reinterpret_cast<uint4*>(&qfrag_s[lane][4 * ks]) = make_uint4(qhi[ks][0], qhi[ks][1], qhi[ks][2], qhi[ks][3]);
      *reinterpret_cast<uint4*>(&qfrag_s[lane][16 + 4 * ks]) =
          make_uint4(qlo[ks][0], qlo[ks][1], qlo[ks][2], qlo[ks][3]);
    }
    *reinterpret_cast<uint4*>(&qfrag_s[lane][32]) = make_uint4(__float_as_uint(qs[0]), __float_as_uint(qs[1]),
                                                                __float_as_uint(qsum[0]), __float_as_uint(qsum[1]));
  }
  __syncthreads();
  if (warp != 0) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const uint4 h4 = *reinterpret_cast<const uint4*>(&qfrag_s[lane][4 * ks]);
      const uint4 l4 = *reinterpret_cast<const uint4*>(&qfrag_s[lane][16 + 4 * ks]);
      qhi[ks][0] = h4.x, qhi[ks][1] = h4.y, qhi[ks][2] = h4.z, qhi[ks][3] = h4.w;
      qlo[ks][0] = l4.x, qlo[ks][1] = l4.y, qlo[ks][2] = l4.z, qlo[ks][3] = l4.w;
    }
    const uint4 sq4 = *reinterpret_cast<const uint4*>(&qfrag_s[lane][32]);
    qs[0] = __uint_as_float(sq4.x), qs[1] = __uint_as_float(sq4.y);
    qsum[0] = __uint_as_float(sq4.z), qsum[1] = __uint_as_float(sq4.w);
  }

  // ---- scores for the warp's 64 rows: 8 n-tiles of 8 rows (rowp_s is visible: __syncthreads above)
  float sc[8][4];  // [nt][c]: rows (heads) g, g+8 x cache rows 2t, 2t+1
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const uint4 kw = kw_all[nt];
    const uint32_t wv[4] = {kw.x, kw.y, kw.z, kw.w};
    int ah[4] = {0, 0, 0, 0}, al[4] = {0, 0, 0, 0};
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      // the lane's code bytes 4 ks .. 4 ks + 3 = dims 32t + 8 ks + 0..7, split into unsigned
      // bytes [lo, hi, lo, hi]: b0 = dims +0..3 (bytes 4ks, 4ks+1), b1 = dims +4..7
      const uint32_t lo4 = wv[ks] & 0x0F0F0F0Fu, hi4 = (wv[ks] >> 4) & 0x0F0F0F0Fu;
      const uint32_t b0 = __byte_perm(lo4, hi4, 0x5140), b1 = __byte_perm(lo4, hi4, 0x7362);
      imma16832(ah, qhi[ks], b0, b1);
      imma16832(al, qlo[ks], b0, b1);
    }
    // per cache row: s_k * s_q * (<q~, c> - z * sum(q~)) * sm_scale, in log2 units; -inf past L
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int row = row0 + nt * 8 + 2 * t + j;
      const float4 rp = rowp_s[warp][nt * 8 + 2 * t + j];
      const float sk = rp.x, zk = rp.y;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const float dot = (float)ah[2 * hh + j] + (float)al[2 * hh + j] * (1.f / 256.f);
        const float v = (dot - zk * qsum[hh]) * (qs[hh] * sk);
        sc[nt][2 * hh + j] = row < L ? v : -INFINITY;
      }
    }
  }
  // ---- softmax over the warp's rows, per head (rows g and g + 8)
  float m[2], l[2];
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(sc[nt][2 * hh], sc[nt][2 * hh + 1]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    m[hh] = mx;
    l[hh] = 0.f;
  }
  float zsum[2] = {0.f, 0.f};
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int rl = nt * 8 + 2 * t + j;  // row within the warp's 64
      const float4 rp = rowp_s[warp][rl];
      const float sv = rp.z, zv = rp.w;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const float p = (m[hh] == -INFINITY) ? 0.f : exp2f(sc[nt][2 * hh + j] - m[hh]);
        l[hh] += p;
        const float pv = p * sv;
        zsum[hh] += pv * zv;
        const int r = g + 8 * hh;
        if (r < G) p_w[rl][r] = pv;
      }
    }
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 1);
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 2);
    zsum[hh] += __shfl_xor_sync(0xffffffffu, zsum[hh], 1);
    zsum[hh] += __shfl_xor_sync(0xffffffffu, zsum[hh], 2);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  // ---- P.V: lane owns dims 4 lane .. 4 lane + 3 (code bytes 2 lane, 2 lane + 1)
  // codes -> floats by the magic-number trick (0x4B0000cc = 2^23 + c), 2 codes per FADD2;
  // accumulation with FFMA2 on dim pairs
  float2 o2[G][2];
#pragma unroll
  for (int r = 0; r < G; ++r) o2[r][0] = o2[r][1] = make_float2(0.f, 0.f);
  const int nrows = min(ROWS_PER_WARP, L - row0);
  const float2 two23 = make_float2(8388608.f, 8388608.f);
#pragma unroll 8
  for (int rl = 0; rl < nrows; ++rl) {
    const uint32_t cw = *reinterpret_cast<const unsigned short*>(&vcode_w[rl][2 * lane]);
    const uint32_t lo = cw & 0x0F0Fu, hi = (cw >> 4) & 0x0F0Fu;  // (c0, c2), (c1, c3)
    const float2 c01 = f2sub(make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7540)),
                                         __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7540))), two23);
    const float2 c23 = f2sub(make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7541)),
                                         __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7541))), two23);
    if constexpr (G % 4 == 0) {  // the row's p of four heads in one 16-byte load
#pragma unroll
      for (int r4 = 0; r4 < G; r4 += 4) {
        const float4 p4 = *reinterpret_cast<const float4*>(&p_w[rl][r4]);
        const float pp[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          o2[r4 + e][0] = f2fma(make_float2(pp[e], pp[e]), c01, o2[r4 + e][0]);
          o2[r4 + e][1] = f2fma(make_float2(pp[e], pp[e]), c23, o2[r4 + e][1]);
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < G; ++r) {
        const float pv = p_w[rl][r];
        o2[r][0] = f2fma(make_float2(pv, pv), c01, o2[r][0]);
        o2[r][1] = f2fma(make_float2(pv, pv), c23, o2[r][1]);
      }
    }
  }
  // ---- merge the 4 warps: each writes (o - zsum, m, l) per head over its own (now idle)
  // buffer; lanes with t = 0 hold head g's m / l / zsum: broadcast from lane 4 (r & 7)
  float mv[G], lv[G], zv_[G];
#pragma unroll
  for (int r = 0; r < G; ++r) {
    const int src = 4 * (r & 7);
    mv[r] = __shfl_sync(0xffffffffu, r < 8 ? m[0] : m[1], src);
    lv[r] = __shfl_sync(0xffffffffu, r < 8 ? l[0] : l[1], src);
    zv_[r] = __shfl_sync(0xffffffffu, r < 8 ? zsum[0] : zsum[1], src);
  }
  __syncwarp();  // every lane is done reading the warp's codes / p before they are overwritten
#pragma unroll
  for (int r = 0; r < G; ++r) {
    float* mr = mrg(warp, r);
    *reinterpret_cast<float4*>(mr + 4 * lane) =
        make_float4(o2[r][0].x - zv_[r], o2[r][0].y - zv_[r], o2[r][1].x - zv_[r], o2[r][1].y - zv_[r]);
    if (lane == 0) {
      mr[HD] = mv[r];
      mr[HD + 1] = lv[r];
    }
  }
  __syncthreads();
  // thread = (head r, dim d) pairs; 128 threads cover HD dims of one head per pass
  for (int r = 0; r < G; ++r) {
    const int d = threadIdx.x;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, mrg(w, r)[HD]);
    float O = 0.f, Ls = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float* mw_ = mrg(w, r);
      const float mw = mw_[HD];
      const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      O += f * mw_[d];
      Ls += f * mw_[HD + 1];
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

cudaError_t launch_kv_decode(const void* q, const uint8_t* k_codes, const float* k_scale, const uint8_t* k_zero,
                             const uint8_t* v_codes, const float* v_scale, const uint8_t* v_zero,
                             const int32_t* seq_lens, int B, int n_q, int n_kv, int head_dim, int s_max,
                             float sm_scale, void* out, float* workspace, cudaStream_t stream) {
  if (B == 0) return cudaSuccess;
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
  a.nsplit = (s_max + kvd::CHUNK - 1) / kvd::CHUNK;
  a.sm_scale_log2 = sm_scale * kvd::LOG2E;
  a.ws = workspace;
  const dim3 grid(a.nsplit, n_kv, B);
  const int G = n_q / n_kv;
  switch (G) {
    case 1: kvd::kv_decode_kernel<1><<<grid, kvd::WARPS * 32, 0, stream>>>(a); break;
    case 2: kvd::kv_decode_kernel<2><<<grid, kvd::WARPS * 32, 0, stream>>>(a); break;
    case 4: kvd::kv_decode_kernel<4><<<grid, kvd::WARPS * 32, 0, stream>>>(a); break;
    case 8: kvd::kv_decode_kernel<8><<<grid, kvd::WARPS * 32, 0, stream>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  kvd::kv_decode_combine<<<(unsigned)((int64_t)B * n_q), kvd::HD, 0, stream>>>(workspace, a.nsplit, n_q,
                                                                              static_cast<__half*>(out));
  return cudaPeekAtLastError();
}

}  // namespace qr
