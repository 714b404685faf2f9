// int4_gemm.cu — rows a4 + a5 of the QuaRot hot path on sm_100a tensor cores.
//
// acc[m][n] = sum_k cx[m][k] * cw[n][k] (exact int32, "INT4 ... on a TensorCore is
// INT32"), y = fp16(acc * s_x[m] * s_w[n]) (P:233 dequantization with row and column
// scales), fused in the epilogue instead of the paper's separate kernel.
//
// sm_100 tcgen05 has no s4 kind, so the packed INT4 operands are widened to INT8 on chip and
// multiplied with tcgen05.mma kind::i8 into TMEM int32 accumulators.
//
// Design — a CTA pair (cluster 2x1) computes a 256 x 256 output tile with
// tcgen05.mma.cta_group::2 (M256 N256 K32); CTA r owns A rows [128r, 128r+128) and B rows
// [128r, 128r+128) of the tile:
//  * TMA warp: cp.async.bulk.tensor loads the PACKED A and B k-blocks (128 rows x 64 B each,
//    SWIZZLE_64B) into an 8-stage staging ring — asynchronous, no registers in flight;
//  * 4 A-widen warps (thread = row): LDS the row's 64 packed bytes, widen to 128 int8 with the
//    "x16 nibble trick" (int8 = code*16 = byte & 0xF0 for the high nibble, (byte << 4) & 0xF0
//    for the low nibble), tcgen05.st them into a TMEM A stage: the MMA takes A from TMEM
//    (TS form), so widened A never goes back through shared memory;
//  * 4 B-widen warps: LDS packed B, widen, STS.128 into a 4-stage K-major SWIZZLE_128B ring;
//  * every packed 32-code chunk becomes [16 low-nibble codes | 16 high-nibble codes]: the
//    SAME permutation of k for A and B, so the dot product is unchanged.  The MMA
//    accumulates 256*acc (|256*acc| <= 256*49*K < 2^31 for K <= 171196); the epilogue shifts
//    right by 8, exactly;
//  * MMA warp (leader CTA, one thread): 4 x tcgen05.mma per k-block; tcgen05.commit
//    multicasts the stage release to both CTAs;
//  * 8 epilogue warps per CTA (2 per TMEM lane quarter, one column half each): tcgen05.ld
//    32x32b.x32 (next chunk in flight while the current one is stored), scale, fp16, store.
// Shared-memory traffic per CTA per k-block: 16 KB TMA + 16 KB LDS + 16 KB STS + 16 KB MMA
// read = 64 KB per 512 MMA cycles (125 B/clk at the full tensor rate, vs ~128 B/clk).
// No thread ever holds a global load in flight across the proxy fence (whose MEMBAR would
// wait for it), which is what capped the register-prefetch design at ~40% of peak.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "quarot_internal.h"

namespace qr {
namespace gemm {

constexpr int BM = 256;            // pair tile rows (128 per CTA)
constexpr int BMC = 128;
constexpr int BN = 256;            // pair tile cols (128 B rows per CTA)
constexpr int BNC = 128;
constexpr int BK = 256;            // int8 elements per k-block (8 MMAs of K = 32)
constexpr int BKP = BK / 2;        // packed bytes per row per k-block (128 B: one TMA SWIZZLE_128B row)
constexpr int CPR = BKP / 16;      // 16-byte packed chunks per row per k-block
constexpr int KATOMS = BK / 128;   // 128-byte K-major swizzle atoms per widened row
#ifndef QR_GEMM_SSTAGES
#define QR_GEMM_SSTAGES 4
#endif
#ifndef QR_GEMM_OSTAGES
#define QR_GEMM_OSTAGES 3
#endif
#ifndef QR_OPWAIT
#define QR_OPWAIT mbar_wait_sleep
#endif
#ifndef QR_EPIWAIT  // the epilogue's wait for a finished accumulator (experiments: mbar_wait, mbar_wait_backoff<32>)
#define QR_EPIWAIT mbar_wait_sleep
#endif
constexpr int SSTAGES = QR_GEMM_SSTAGES;  // packed staging ring (TMA destination)
// the two B-widen groups take alternate k-blocks: with an even ring each staging slot is always
// read by the same group, so no waiter can run two phases ahead of a slot (parity aliasing)
static_assert(QR_GEMM_SSTAGES % 2 == 0, "staging ring must be even");
constexpr int OSTAGES = QR_GEMM_OSTAGES;  // widened operand ring (TMEM A: 64 columns + smem B each)
constexpr int A_COLS = BK / 4;                      // TMEM columns per A stage (4 int8 per column)
constexpr int SA_BYTES = BMC * BKP;                 // 16 KB packed A
constexpr int SB_BYTES = BNC * BKP;                 // 16 KB packed B
constexpr int SSTAGE_BYTES = SA_BYTES + SB_BYTES;   // 32 KB
constexpr int OB_BYTES = BNC * BK;                  // 32 KB widened B: KATOMS x [128 rows][128 B] SW128
static_assert(256 + OSTAGES * A_COLS <= 512, "TMEM budget");
constexpr int NUM_EPI_WARPS = 8;                    // warps 0..7: TMEM lane quarter w % 4, column half w / 4
constexpr int A_WARP0 = 8;                          // warps 8..11
constexpr int B_WARP0 = 12;                         // warps 12..19: two groups of 4, alternating k-blocks
constexpr int TMA_WARP = 20;
constexpr int MMA_WARP = 21;
constexpr int NUM_THREADS = 24 * 32;                // warps 22, 23 only pad warpgroup 5
// per-role register budgets (setmaxnreg; the launch gives every warp 80): warpgroup 5 (TMA,
// MMA, 2 idle) and the B-widen warpgroups give registers to the epilogue, which holds three
// 32-column accumulator chunks at once.  6144 + 6144 freed = 12288 = 256 x (128 - 80).
constexpr int EPI_REGS = 128;
constexpr int BW_REGS = 56;
constexpr int CTL_REGS = 32;
constexpr int TMEM_COLS = 512;
constexpr int ACC_COL = 0;                          // accumulator: columns [0, 256)
constexpr int A_COL0 = 256;                         // A stages: A_COLS columns each
constexpr uint32_t IDESC = idesc_i8(BM, BN);
constexpr size_t SMEM_BYTES = SSTAGES * SSTAGE_BYTES + OSTAGES * OB_BYTES + 1024 + 512 + BN * 4;
static_assert(SMEM_BYTES <= 232448, "227 KB dynamic smem");

struct Params {
  const float* x_scale;
  const float* w_scale;
  void* out;  // fp16 y or int32 acc
  const __half* residual;  // optional fp16 residual added in the epilogue (decoder layer, a8)
  int swiglu;              // 1: rows of W interleaved [8 gate | 8 up]; out = silu(gate) * up, N/2 wide
  int64_t M, N, K, ld_out, ld_r;
  int num_m, num_n, num_kb, num_tiles;  // num_m in 256-row pair tiles
  int group_m;  // raster: pair-rows per group (tiles walk m fastest inside a group, then n)
};

QR_DEVICE void tile_coords(const Params& p, int t, int& mb, int& nb) {
  const int per_group = p.group_m * p.num_n;
  const int group = t / per_group;
  const int first_m = group * p.group_m;
  const int gm = min(p.num_m - first_m, p.group_m);
  const int within = t - group * per_group;
  mb = first_m + within % gm;
  nb = within / gm;
}

QR_DEVICE uint32_t lo_nib16(uint32_t w) { return (w << 4) & 0xF0F0F0F0u; }
QR_DEVICE uint32_t hi_nib16(uint32_t w) { return w & 0xF0F0F0F0u; }

// fp16_rn(lo) | fp16_rn(hi) << 16 in a register
QR_DEVICE uint32_t pack_half2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// named barrier over the 8 epilogue warps (id 1; id 0 is __syncthreads)
QR_DEVICE void epi_bar_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
#define QR_SETMAXNREG_INC(n) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(n))
#define QR_SETMAXNREG_DEC(n) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(n))
QR_DEVICE uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
QR_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
QR_DEVICE uint32_t map_to_rank(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
// Arrive on a barrier by shared::cluster address (default .release.cta, as CUTLASS's
// ClusterBarrier::arrive(cta_id)).
QR_DEVICE void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
QR_DEVICE void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
QR_DEVICE void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
QR_DEVICE uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::i8, CTA pair
QR_DEVICE void mma_i8_ts_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}
QR_DEVICE void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
#define QR_TMEM_ST32(taddr, r)                                                                             \
  asm volatile(                                                                                            \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                     \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),     \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),          \
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),         \
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                      \
      : "memory")

// tcgen05.st of 8 registers into 8 consecutive columns of the warp's 32 lanes (STTM takes a
// contiguous register range, so a constant fill keeps 8 registers, not 32, live)
#define QR_TMEM_ST8(taddr, r)                                                                               \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),        \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])         \
               : "memory")

// Converts and stores one 32-column accumulator chunk of one row (columns n0 .. n0 + 31;
// wsc = their 32 weight scales in smem).  fp16: y = fp16_rn(fp32(acc) * s_x * s_w); with a
// residual, fp16_rn(fp32(y) + fp32(r)); s32: raw accumulators; SwiGLU: the chunk is
// [8 gate | 8 up] x 2 (interleaved weight rows) and 16 act = fp16_rn(fp16_rn(silu(g)) * u)
// values go to column n0 / 2, g and u the fp16 linear outputs (the FP16 model's ops, Z23).  The INT32 result is "immediately cast (and
// scale[d]) to FP16" before any further op, so the fused epilogues equal the unfused
// GEMM -> fp16 -> residual add / quarot_swiglu chain bit for bit.
// kEpi: the epilogue variant as a compile-time choice (0 = read p.residual / p.swiglu at run time,
// 1 = plain, 2 = + residual, 3 = SwiGLU): a specialized kernel keeps only its own code and registers
template <int kEpi>
QR_DEVICE bool epi_residual(const Params& p) { return kEpi == 0 ? p.residual != nullptr : kEpi == 2; }
template <int kEpi>
QR_DEVICE bool epi_swiglu(const Params& p) { return kEpi == 0 ? p.swiglu != 0 : kEpi == 3; }

template <bool kS32, int kDbg, int kShift = 8, int kEpi = 0>  // kShift: the x16 nibble scaling of both operands (A4W4)
QR_DEVICE void epi_chunk(const Params& p, const uint32_t (&rc)[32], int64_t m, bool row_ok, int64_t n0, float sx,
                         const float* wsc) {
  if (!row_ok) return;
  // the accumulator is 2^kShift x the integer dot product (exactly: both operands carry the x16
  // nibble scaling), and |dot| < 2^24, so fp32(acc) * (s_x 2^-kShift) rounds exactly like
  // fp32(acc >> kShift) * s_x (no shift per element; 2^-kShift s_x only loses bits when s_x <
  // 2^-118, where every output rounds to fp16 zero either way)
  const float sxs = sx * (1.f / (float)(1 << kShift));
  if constexpr (kS32) {
    int32_t* dst = reinterpret_cast<int32_t*>(p.out) + m * p.ld_out + n0;
#pragma unroll
    for (int g = 0; g < 8; ++g)
      if (n0 + g * 4 < p.N)
        *reinterpret_cast<int4*>(dst + g * 4) =
            make_int4((int32_t)rc[4 * g] >> kShift, (int32_t)rc[4 * g + 1] >> kShift,
                      (int32_t)rc[4 * g + 2] >> kShift, (int32_t)rc[4 * g + 3] >> kShift);
  } else if (epi_swiglu<kEpi>(p)) {
#pragma unroll
    for (int hgrp = 0; hgrp < 2; ++hgrp) {
      const int64_t nn = n0 + 16 * hgrp;
      if (nn < p.N) {
        const float* sg = wsc + 16 * hgrp;
        uint32_t h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // two act outputs (columns c, c + 1) per packed half2
          const int c = 2 * e;
          const __half2 gh = __floats2half2_rn(((float)(int32_t)rc[16 * hgrp + c] * sxs) * sg[c],
                                               ((float)(int32_t)rc[16 * hgrp + c + 1] * sxs) * sg[c + 1]);
          const __half2 uh = __floats2half2_rn(((float)(int32_t)rc[16 * hgrp + 8 + c] * sxs) * sg[8 + c],
                                               ((float)(int32_t)rc[16 * hgrp + 9 + c] * sxs) * sg[9 + c]);
          const float2 gf = __half22float2(gh);
          const __half2 sh = __floats2half2_rn(silu_f32(gf.x), silu_f32(gf.y));  // fp16(silu(g))
          // fp16(fp16(silu(g)) * u): the product of two fp16 values is exact in fp32, so one
          // fp16 multiply (RN) gives the same bits as the fp32 multiply rounded to fp16
          const __half2 act = __hmul2(sh, uh);
          h[e] = *reinterpret_cast<const uint32_t*>(&act);
        }
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.out) + m * p.ld_out + (nn >> 1)) =
            make_uint4(h[0], h[1], h[2], h[3]);
      }
    }
  } else {
    __half* dst = reinterpret_cast<__half*>(p.out) + m * p.ld_out + n0;
    uint4 rres0 = make_uint4(0, 0, 0, 0), rres1 = rres0, rres2 = rres0, rres3 = rres0;
    if (epi_residual<kEpi>(p)) {  // all four loads in flight at once
      const __half* rrow = p.residual + m * p.ld_r + n0;
      if (n0 < p.N) rres0 = *reinterpret_cast<const uint4*>(rrow);
      if (n0 + 8 < p.N) rres1 = *reinterpret_cast<const uint4*>(rrow + 8);
      if (n0 + 16 < p.N) rres2 = *reinterpret_cast<const uint4*>(rrow + 16);
      if (n0 + 24 < p.N) rres3 = *reinterpret_cast<const uint4*>(rrow + 24);
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (n0 + g * 8 < p.N) {
        const float4 s0 = *reinterpret_cast<const float4*>(wsc + g * 8);
        const float4 s1 = *reinterpret_cast<const float4*>(wsc + g * 8 + 4);
        const float swv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        const uint4 rr = g == 0 ? rres0 : g == 1 ? rres1 : g == 2 ? rres2 : rres3;
        const uint32_t rw[4] = {rr.x, rr.y, rr.z, rr.w};
        uint32_t h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v0 = ((float)(int32_t)rc[8 * g + 2 * e] * sxs) * swv[2 * e];
          float v1 = ((float)(int32_t)rc[8 * g + 2 * e + 1] * sxs) * swv[2 * e + 1];
          if (epi_residual<kEpi>(p)) {  // the linear output is fp16 before the residual add
            v0 = __half2float(__float2half_rn(v0)) + __half2float(__ushort_as_half((unsigned short)(rw[e] & 0xFFFFu)));
            v1 = __half2float(__float2half_rn(v1)) + __half2float(__ushort_as_half((unsigned short)(rw[e] >> 16)));
          }
          h[e] = pack_half2(v0, v1);
        }
        if (kDbg != 4 || (h[0] == 0x7c017c01u && h[1] == 0x7c017c01u))  // probe 4: no stores
          *reinterpret_cast<uint4*>(dst + g * 8) = make_uint4(h[0], h[1], h[2], h[3]);
      }
    }
  }
}

// The residual chunk from the warp's TMA-staged box (32 rows x 64 fp16, SWIZZLE_128B: 16-byte
// chunk c of row r at r * 128 + ((c ^ (r & 7)) << 4)); half = which 32 columns of the box.
// Same arithmetic as epi_chunk's residual path: y = fp16(fp16(acc * s_x * s_w) + r).
QR_DEVICE void epi_chunk_res(const Params& p, const uint32_t (&rc)[32], int64_t m, bool row_ok, int64_t n0, float sx,
                             const float* wsc, const uint8_t* box, int half) {
  if (!row_ok) return;
  const int r = threadIdx.x & 31;
  const uint32_t rowb = smem_u32(box) + (uint32_t)r * 128u;
  const float sxs = sx * (1.f / 256.f);  // as epi_chunk: fp32(acc) * s_x / 256 == fp32(acc >> 8) * s_x
  __half* dst = reinterpret_cast<__half*>(p.out) + m * p.ld_out + n0;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (n0 + g * 8 < p.N) {
      const uint4 rr = lds_v4(rowb + ((uint32_t)((4 * half + g) ^ (r & 7)) << 4));
      const float4 s0 = *reinterpret_cast<const float4*>(wsc + g * 8);
      const float4 s1 = *reinterpret_cast<const float4*>(wsc + g * 8 + 4);
      const float swv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      const uint32_t rw[4] = {rr.x, rr.y, rr.z, rr.w};
      uint32_t h[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v0 = ((float)(int32_t)rc[8 * g + 2 * e] * sxs) * swv[2 * e];
        float v1 = ((float)(int32_t)rc[8 * g + 2 * e + 1] * sxs) * swv[2 * e + 1];
        v0 = __half2float(__float2half_rn(v0)) + __half2float(__ushort_as_half((unsigned short)(rw[e] & 0xFFFFu)));
        v1 = __half2float(__float2half_rn(v1)) + __half2float(__ushort_as_half((unsigned short)(rw[e] >> 16)));
        h[e] = pack_half2(v0, v1);
      }
      *reinterpret_cast<uint4*>(dst + g * 8) = make_uint4(h[0], h[1], h[2], h[3]);
    }
  }
}

template <bool kS32, int kDbg = 0, int kEpi = 0>  // kDbg: 0 normal; roofline probes: 1 MMA only, 2 no widening, 3 no TMA, 4 no fp16 stores,
                                                   // 5 no B widening stores, 6 no A TMEM stores, 7 no epilogue work,
                                                   // 8 the MMA does not wait for the accumulator drain
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    int4_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmR, const Params p) {
  // the residual variant gives one operand stage to a per-warp residual staging area (8 x 4 KB,
  // TMA-loaded [32 rows x 64 cols] boxes): the residual rows then reach the epilogue through the
  // async proxy instead of 32-row uncoalesced loads on the L1 path the widening LDS/STS need
  constexpr bool kResTma = kEpi == 2 && !kS32;
  constexpr int kOst = kResTma ? OSTAGES - 1 : OSTAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_smem = smem;                                  // [SSTAGES][A 8 KB | B 8 KB]
  uint8_t* opb_smem = smem + SSTAGES * SSTAGE_BYTES;           // [kOst][32 KB]
  uint8_t* res_smem = opb_smem + kOst * OB_BYTES;              // kResTma: [8 warps][32 rows][128 B] SW128
  uint64_t* bars = reinterpret_cast<uint64_t*>(opb_smem + OSTAGES * OB_BYTES);
  uint64_t* st_full = bars;                          // [SSTAGES] TMA -> widen warps
  uint64_t* st_empty = st_full + SSTAGES;            // [SSTAGES] widen warps -> TMA (8 warps)
  uint64_t* op_full = st_empty + SSTAGES;            // [OSTAGES] widen warps of both CTAs -> leader MMA
  uint64_t* op_empty = op_full + OSTAGES;            // [OSTAGES] MMA commit -> widen warps
  uint64_t* t_full = op_empty + OSTAGES;             // MMA commit -> epilogue
  uint64_t* t_empty = t_full + 1;                    // epilogues of both CTAs -> leader MMA
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 1);
  uint64_t* res_bar = bars + 24;                     // kResTma: [8 warps] residual box landed
  float* ws_smem = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);  // [BN] tile's w_scale

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = (int)blockIdx.x >> 1;
  const int num_pairs = (int)gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SSTAGES; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], 8);
    }
    for (int s = 0; s < kOst; ++s) {
      mbar_init(&op_full[s], 2 * 8);
      mbar_init(&op_empty[s], 1);
    }
    mbar_init(t_full, 1);
    mbar_init(t_empty, 2 * NUM_EPI_WARPS);
    if (kResTma)
      for (int w = 0; w < NUM_EPI_WARPS; ++w) mbar_init(&res_bar[w], 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == TMA_WARP && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (kResTma) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmR)) : "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int my_tiles = (p.num_tiles > pair) ? (p.num_tiles - 1 - pair) / num_pairs + 1 : 0;
  const int total = my_tiles * p.num_kb;

  constexpr bool kMmaOnly = kDbg == 1;
  // roles by warpgroup (setmaxnreg is warpgroup-wide); kMmaOnly (probe 1) idles the producers
  if (warp >= TMA_WARP) {
    QR_SETMAXNREG_DEC(CTL_REGS);
    if (warp == TMA_WARP && !kMmaOnly) {
      // ===================== TMA producer: packed k-blocks -> staging ring =====================
      if (lane == 0) {
        for (int it = 0; it < total; ++it) {
          const int tl = it / p.num_kb;
          const int kb = it - tl * p.num_kb;
          int mb, nb;
          tile_coords(p, pair + tl * num_pairs, mb, nb);
          const int s = it % SSTAGES;
          mbar_wait_sleep(&st_empty[s], ((it / SSTAGES) & 1) ^ 1);
          if (kDbg == 3) {
            mbar_arrive(&st_full[s]);
          } else {
            mbar_expect_tx(&st_full[s], SSTAGE_BYTES);
            const uint32_t dst = smem_u32(stage_smem + s * SSTAGE_BYTES);
            tma_load_2d(dst, &tmA, kb * BKP, mb * BM + (int)rank * BMC, &st_full[s]);
            tma_load_2d(dst + SA_BYTES, &tmB, kb * BKP, nb * BN + (int)rank * BNC, &st_full[s]);
          }
        }
      }
    } else if (warp == MMA_WARP) {
      // ===================== MMA issuer (leader CTA, one thread) =====================
      if (rank == 0 && lane == 0) {
        int it = 0;
        for (int tl = 0; tl < my_tiles; ++tl) {
          if (kDbg != 8) mbar_wait(t_empty, (tl & 1) ^ 1);  // probe 8: no wait for the drain
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + ACC_COL;
          for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
            const int o = kMmaOnly ? 0 : it % kOst;
            if (!kMmaOnly) mbar_wait(&op_full[o], (it / kOst) & 1);
            tc_fence_after();
            const uint64_t b_desc = umma_desc_sw128(smem_u32(opb_smem + o * OB_BYTES));
            const uint32_t a_tmem = tmem_base + (uint32_t)(A_COL0 + A_COLS * o);
  #pragma unroll
            for (int k = 0; k < BK / 32; ++k)  // atom k/4 at +16 KB, 32 bytes along K within it
              mma_i8_ts_2sm(d_tmem, a_tmem + (uint32_t)(8 * k),
                            b_desc + (uint64_t)((k >> 2) * (BNC * 128 / 16) + 2 * (k & 3)), IDESC,
                            (kb | k) != 0 ? 1u : 0u);
            if (!kMmaOnly) mma_commit_pair(&op_empty[o]);
          }
          mma_commit_pair(t_full);
        }
      }
      __syncwarp();
    }
  } else if (warp >= B_WARP0) {
    QR_SETMAXNREG_DEC(BW_REGS);
    if (!kMmaOnly) {
      // ===================== B widen: packed smem -> int8 SW128 smem =====================
      // two groups of 4 warps take alternate k-blocks, so one group's proxy fence (a MEMBAR
      // that drains its STS) overlaps the other group's loads and stores
      const int grp = (warp - B_WARP0) >> 2;
      const int t = threadIdx.x - (B_WARP0 + 4 * grp) * 32;  // 0..127
      // thread t owns packed chunk q = t % 8 of rows t / 8 + 16 i (i < CPT_B): the swizzle phase
      // (row & 7) and the chunk are the same for all i, so every address is a base + immediate.
      // Widened: chunk q -> K atom q / 4, int8 chunks 2 (q % 4) (lo nibbles) and +1 (hi nibbles)
      // of a [8-row x 128 B] SW128 group; row r at (r / 8) * 1024 + (r % 8) * 128.
      constexpr int CPT_B = BNC * CPR / 128;  // packed chunks per thread
      static_assert(CPR == 8 && BNC % 16 == 0, "B widen mapping assumes 8 chunks per row");
      const uint32_t rr0 = (uint32_t)t >> 3, q = (uint32_t)t & 7u, swz = rr0 & 7u;
      const uint32_t src_off = rr0 * BKP + ((q ^ swz) << 4);
      const uint32_t atom = q >> 2, qa = q & 3u, odd = atom & 1u;
      const uint32_t dst_row = atom * (BNC * 128u) + (rr0 >> 3) * 1024u + swz * 128u;
      // lanes 8j..8j+7 share a row and form one 128-byte store phase: atom-0 lanes store their lo
      // chunk first and atom-1 lanes their hi chunk, so each phase covers all 8 chunk slots of
      // the bank window (the same order for both atoms is a 2-way bank conflict)
      const uint32_t d0 = ((2u * qa + odd) ^ swz) << 4, d1 = ((2u * qa + (odd ^ 1u)) ^ swz) << 4;
      const uint32_t sh0 = odd ? 0u : 4u, sh1 = odd ? 4u : 0u;  // lo = (w << 4) & F0.., hi = w & F0..
      const uint32_t opfull_leader = map_to_rank(&op_full[0], 0);
      for (int it = grp; it < total; it += 2) {
        const int s = it % SSTAGES;
        const int o = it % kOst;
        mbar_wait_sleep(&st_full[s], (it / SSTAGES) & 1);
        const uint32_t src = smem_u32(stage_smem + s * SSTAGE_BYTES) + SA_BYTES + src_off;
        uint4 w[CPT_B];
  #pragma unroll
        for (int i = 0; i < CPT_B; ++i) w[i] = lds_v4(src + (uint32_t)i * (16u * BKP));
        QR_OPWAIT(&op_empty[o], ((it / kOst) & 1) ^ 1);
        const uint32_t dst = smem_u32(opb_smem + o * OB_BYTES) + dst_row;
  #pragma unroll
        for (int i = 0; i < (kDbg == 2 || kDbg == 5 ? 0 : CPT_B); ++i) {
          const uint4 v = w[i];
          sts_v4(dst + (uint32_t)i * 2048u + d0,
                 make_uint4((v.x << sh0) & 0xF0F0F0F0u, (v.y << sh0) & 0xF0F0F0F0u, (v.z << sh0) & 0xF0F0F0F0u,
                            (v.w << sh0) & 0xF0F0F0F0u));
          sts_v4(dst + (uint32_t)i * 2048u + d1,
                 make_uint4((v.x << sh1) & 0xF0F0F0F0u, (v.y << sh1) & 0xF0F0F0F0u, (v.z << sh1) & 0xF0F0F0F0u,
                            (v.w << sh1) & 0xF0F0F0F0u));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&st_empty[s]);  // after the STS consumed the loaded registers (see A widen)
          mbar_arrive_cluster(opfull_leader + (uint32_t)o * 8u);
        }
      }
    }
  } else if (warp >= A_WARP0) {
    if (!kMmaOnly) {
      // ===================== A widen: thread = row, packed smem -> int8 TMEM =====================
      const int row = (warp - A_WARP0) * 32 + lane;            // == TMEM lane (warp % 4 quarter)
      const uint32_t sw = (uint32_t)(row & 7);                  // TMA SWIZZLE_128B chunk xor
      const uint32_t opfull_leader = map_to_rank(&op_full[0], 0);
      const uint32_t tlane = (uint32_t)((warp - A_WARP0) * 32) << 16;
      for (int it = 0; it < total; ++it) {
        const int s = it % SSTAGES;
        const int o = it % kOst;
        mbar_wait_sleep(&st_full[s], (it / SSTAGES) & 1);
        const uint32_t src = smem_u32(stage_smem + s * SSTAGE_BYTES) + (uint32_t)row * BKP;
        uint4 w[CPR];
  #pragma unroll
        for (int c = 0; c < CPR; ++c) w[c] = lds_v4(src + (((uint32_t)c ^ sw) << 4));
        QR_OPWAIT(&op_empty[o], ((it / kOst) & 1) ^ 1);
        tc_fence_after();
  #pragma unroll
        for (int half = 0; half < CPR / 4; ++half) {
          uint32_t r[32];
  #pragma unroll
          for (int cc = 0; cc < 4; ++cc) {  // packed chunk c -> MMA k-step c: [16 lo | 16 hi] int8
            const uint4 v = w[4 * half + cc];
            r[8 * cc + 0] = lo_nib16(v.x);
            r[8 * cc + 1] = lo_nib16(v.y);
            r[8 * cc + 2] = lo_nib16(v.z);
            r[8 * cc + 3] = lo_nib16(v.w);
            r[8 * cc + 4] = hi_nib16(v.x);
            r[8 * cc + 5] = hi_nib16(v.y);
            r[8 * cc + 6] = hi_nib16(v.z);
            r[8 * cc + 7] = hi_nib16(v.w);
          }
          if (kDbg != 2 && kDbg != 6) QR_TMEM_ST32(tmem_base + tlane + (uint32_t)(A_COL0 + A_COLS * o + 32 * half), r);
        }
        // the staging slot is released only once every lane has consumed its loads (the stores
        // above read the registers): an arrive does not wait for in-flight LDS, so releasing
        // right after issuing them lets the next TMA write overtake the reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&st_empty[s]);
        if (kDbg != 2 && kDbg != 6) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(opfull_leader + (uint32_t)o * 8u);
      }
    }
  } else {
    // ===================== epilogue warps 0..7 (each CTA: its 128 rows) =====================
    // warp w owns TMEM lanes 32 (w % 4) .. +31 (its rows) and columns 128 (w / 4) .. +127, in
    // four 32-column chunks.  The accumulator gates the next tile's MMAs, so it is drained
    // first: chunks 0-2 are loaded together, chunk 0 is converted and stored, chunk 3 is
    // loaded into its registers and the accumulator is released; the remaining three chunks
    // are converted and stored while the next tile's MMAs already run.
    QR_SETMAXNREG_INC(EPI_REGS);
    const uint32_t tempty_leader = map_to_rank(t_empty, 0);
    const int quarter = warp & 3, chalf = warp >> 2;
    const int row_in_tile = (int)rank * BMC + quarter * 32 + lane;
    const int et = threadIdx.x;  // 0..255: epilogue warps are warps 0..7
    // kResTma: this warp's staging box and its TMA load (expect 4 KB on res_bar[warp])
    uint8_t* res_w = res_smem + warp * 4096;
    uint32_t res_par = 0u;
    auto res_load = [&](int64_t col, int row) {
      mbar_expect_tx(&res_bar[warp], 4096u);
      tma_load_2d(smem_u32(res_w), &tmR, (int)col, row, &res_bar[warp]);
    };
    for (int tl = 0; tl < my_tiles; ++tl) {
      int mb, nb;
      tile_coords(p, pair + tl * num_pairs, mb, nb);
      const int64_t m = (int64_t)mb * BM + row_in_tile;
      const bool row_ok = m < p.M;
      const int64_t ncol0 = (int64_t)nb * BN + chalf * 128;  // this warp's first column
      // scales (and the residual row segment, into L2) are fetched while the accumulator is
      // still being computed, so the drain never waits on DRAM
      float sx = 0.f;
      if (!kS32) {
        if (row_ok) sx = __ldg(p.x_scale + m);
        const int64_t n = (int64_t)nb * BN + et;
        ws_smem[et] = n < p.N ? __ldg(p.w_scale + n) : 0.f;
        if (epi_residual<kEpi>(p) && !kResTma && row_ok) {
          const __half* rrow = p.residual + m * p.ld_r + ncol0;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rrow));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rrow + 64));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rrow + 127));
        }
        epi_bar_sync();
      }
      if constexpr (kResTma) {  // residual box 0 (the warp's 32 rows x columns ncol0 .. +63)
        if (lane == 0) res_load(ncol0, (int)(m - lane));
      }
      QR_EPIWAIT(t_full, tl & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + ACC_COL + (uint32_t)(chalf * 128);
      if constexpr (kResTma) {
        uint32_t ra[32], rb[32], rc[32];
        const float* wsc = ws_smem + chalf * 128;
        QR_TMEM_LD32(taddr, ra);
        QR_TMEM_LD32(taddr + 32u, rb);
        QR_TMEM_LD32(taddr + 64u, rc);
        tmem_ld_wait();
        mbar_wait(&res_bar[warp], res_par);
        res_par ^= 1u;
        epi_chunk_res(p, ra, m, row_ok, ncol0, sx, wsc, res_w, 0);
        QR_TMEM_LD32(taddr + 96u, ra);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader);
        epi_chunk_res(p, rb, m, row_ok, ncol0 + 32, sx, wsc + 32, res_w, 1);
        __syncwarp();  // every lane is done reading box 0
        if (lane == 0) res_load(ncol0 + 64, (int)(m - lane));
        mbar_wait(&res_bar[warp], res_par);
        res_par ^= 1u;
        epi_chunk_res(p, rc, m, row_ok, ncol0 + 64, sx, wsc + 64, res_w, 0);
        epi_chunk_res(p, ra, m, row_ok, ncol0 + 96, sx, wsc + 96, res_w, 1);
        __syncwarp();  // box 1 read by every lane before the next tile's box 0 lands
        epi_bar_sync();
        continue;
      }
      if constexpr (kDbg == 7) {  // probe: hand the accumulator straight back
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader);
        if (!kS32) epi_bar_sync();
        continue;
      }
      uint32_t ra[32], rb[32], rc[32];
      QR_TMEM_LD32(taddr, ra);
      QR_TMEM_LD32(taddr + 32u, rb);
      QR_TMEM_LD32(taddr + 64u, rc);
      tmem_ld_wait();
      epi_chunk<kS32, kDbg, 8, kEpi>(p, ra, m, row_ok, ncol0, sx, ws_smem + chalf * 128);
      QR_TMEM_LD32(taddr + 96u, ra);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader);
      epi_chunk<kS32, kDbg, 8, kEpi>(p, rb, m, row_ok, ncol0 + 32, sx, ws_smem + chalf * 128 + 32);
      epi_chunk<kS32, kDbg, 8, kEpi>(p, rc, m, row_ok, ncol0 + 64, sx, ws_smem + chalf * 128 + 64);
      epi_chunk<kS32, kDbg, 8, kEpi>(p, ra, m, row_ok, ncol0 + 96, sx, ws_smem + chalf * 128 + 96);
      if (!kS32) epi_bar_sync();  // every warp is done with ws_smem before the next tile's fill
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ============================================================================ A8W8 (§8 f4)
// INT8 x INT8 -> INT32 (QuaRot's 8-bit RTN configuration, P:6, tab:rtn_results): the native
// kind::i8 tensor path with no unpacking — the comparison point for the INT4 unpack cost.
// Both operands are TMA'd straight into the UMMA SW128 K-major layout (two 128-byte swizzle
// atoms per 256-wide k-block), the MMA reads both from smem (SS form), and with no A stages in
// TMEM the accumulator is double-buffered (2 x 256 columns): the epilogue of tile t overlaps
// the mainloop of tile t + 1.  Warps per CTA: 0-7 epilogue, 8 TMA, 9 relay (its CTA's stage
// landed -> the leader's "ready" barrier), 10 MMA issuer (leader CTA).
namespace i8 {
constexpr int STAGES = 3;
constexpr int A_BYTES = BMC * BK;              // 32 KB: 128 rows x 256 int8
constexpr int B_BYTES = BNC * BK;              // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 64 KB
constexpr int TMA_WARP = 8, RELAY_WARP = 9, MMA_WARP = 10;
constexpr int NUM_THREADS = 12 * 32;
constexpr size_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 512 + BN * 4;
static_assert(SMEM_BYTES <= 232448, "227 KB dynamic smem");
}  // namespace i8

QR_DEVICE void mma_i8_ss_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <bool kS32>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(i8::NUM_THREADS, 1)
    int8_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + i8::STAGES * i8::STAGE_BYTES);
  uint64_t* full = bars;                 // [i8::STAGES] local TMA complete
  uint64_t* ready = full + i8::STAGES;       // [i8::STAGES] leader: both CTAs' stage landed (2 arrivals)
  uint64_t* empty = ready + i8::STAGES;      // [i8::STAGES] MMA commit (multicast) -> TMA
  uint64_t* t_full = empty + i8::STAGES;     // [2] MMA commit (multicast) -> epilogue
  uint64_t* t_empty = t_full + 2;        // [2] leader: epilogues of both CTAs
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 2);
  float* ws_smem = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = (int)blockIdx.x >> 1;
  const int num_pairs = (int)gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < i8::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], 2 * NUM_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == i8::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == i8::TMA_WARP && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int my_tiles = (p.num_tiles > pair) ? (p.num_tiles - 1 - pair) / num_pairs + 1 : 0;
  const int total = my_tiles * p.num_kb;

  if (warp == i8::TMA_WARP) {
    if (lane == 0) {
      for (int it = 0; it < total; ++it) {
        const int tl = it / p.num_kb, kb = it - tl * p.num_kb;
        int mb, nb;
        tile_coords(p, pair + tl * num_pairs, mb, nb);
        const int s = it % i8::STAGES;
        mbar_wait_sleep(&empty[s], ((it / i8::STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[s], i8::STAGE_BYTES);
        const uint32_t dst = smem_u32(smem + s * i8::STAGE_BYTES);
        const int ya = mb * BM + (int)rank * BMC, yb = nb * BN + (int)rank * BNC;
        tma_load_2d(dst, &tmA, kb * BK, ya, &full[s]);
        tma_load_2d(dst + BMC * 128, &tmA, kb * BK + 128, ya, &full[s]);
        tma_load_2d(dst + i8::A_BYTES, &tmB, kb * BK, yb, &full[s]);
        tma_load_2d(dst + i8::A_BYTES + BNC * 128, &tmB, kb * BK + 128, yb, &full[s]);
      }
    }
  } else if (warp == i8::RELAY_WARP) {
    if (lane == 0) {
      const uint32_t ready_leader = map_to_rank(&ready[0], 0);
      for (int it = 0; it < total; ++it) {
        const int s = it % i8::STAGES;
        mbar_wait(&full[s], (it / i8::STAGES) & 1);
        mbar_arrive_cluster(ready_leader + (uint32_t)s * 8u);
      }
    }
  } else if (warp == i8::MMA_WARP) {
    if (rank == 0 && lane == 0) {
      int it = 0;
      for (int tl = 0; tl < my_tiles; ++tl) {
        const int ab = tl & 1;
        mbar_wait(&t_empty[ab], ((tl >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(ab * BN);
        for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
          const int s = it % i8::STAGES;
          mbar_wait(&ready[s], (it / i8::STAGES) & 1);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + s * i8::STAGE_BYTES);
          const uint64_t a_desc = umma_desc_sw128(base), b_desc = umma_desc_sw128(base + i8::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {  // atom k/4 at +16 KB, 32 bytes along K within it
            const uint64_t off = (uint64_t)((k >> 2) * (BMC * 128 / 16) + 2 * (k & 3));
            mma_i8_ss_2sm(d_tmem, a_desc + off, b_desc + off, IDESC, (kb | k) != 0 ? 1u : 0u);
          }
          mma_commit_pair(&empty[s]);
        }
        mma_commit_pair(&t_full[ab]);
      }
    }
    __syncwarp();
  } else if (warp < NUM_EPI_WARPS) {
    const uint32_t tempty_leader = map_to_rank(&t_empty[0], 0);
    const int quarter = warp & 3, chalf = warp >> 2;
    const int row_in_tile = (int)rank * BMC + quarter * 32 + lane;
    const int et = threadIdx.x;
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int ab = tl & 1;
      int mb, nb;
      tile_coords(p, pair + tl * num_pairs, mb, nb);
      const int64_t m = (int64_t)mb * BM + row_in_tile;
      const bool row_ok = m < p.M;
      const int64_t ncol0 = (int64_t)nb * BN + chalf * 128;
      float sx = 0.f;
      if (!kS32) {
        if (row_ok) sx = __ldg(p.x_scale + m);
        const int64_t n = (int64_t)nb * BN + et;
        ws_smem[et] = n < p.N ? __ldg(p.w_scale + n) : 0.f;
        if (p.residual && row_ok) {
          const __half* rrow = p.residual + m * p.ld_r + ncol0;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rrow));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rrow + 64));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rrow + 127));
        }
        epi_bar_sync();
      }
      mbar_wait_sleep(&t_full[ab], (tl >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr =
          tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(ab * BN) + (uint32_t)(chalf * 128);
      uint32_t ra[32], rb[32], rc[32];
      QR_TMEM_LD32(taddr, ra);
      QR_TMEM_LD32(taddr + 32u, rb);
      QR_TMEM_LD32(taddr + 64u, rc);
      tmem_ld_wait();
      epi_chunk<kS32, 0, 0>(p, ra, m, row_ok, ncol0, sx, ws_smem + chalf * 128);
      QR_TMEM_LD32(taddr + 96u, ra);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)ab * 8u);
      epi_chunk<kS32, 0, 0>(p, rb, m, row_ok, ncol0 + 32, sx, ws_smem + chalf * 128 + 32);
      epi_chunk<kS32, 0, 0>(p, rc, m, row_ok, ncol0 + 64, sx, ws_smem + chalf * 128 + 64);
      epi_chunk<kS32, 0, 0>(p, ra, m, row_ok, ncol0 + 96, sx, ws_smem + chalf * 128 + 96);
      if (!kS32) epi_bar_sync();
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == i8::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}


// ============================================================================ group-wise (§8 f3)
// W4A4 with one scale per 128-k group on both operands (tab:group_wise_ablation):
//   y[m, n] = fp16( sum_g sx[m, g] sw[n, g] acc_g[m, n] ),  acc_g = sum_{k in g} cx cw (exact int32).
// Codes are stored one per int8 byte (values in [-7, 7]), so both operands take the A8W8 TMA /
// SS-MMA path unchanged; the MMA warp starts a fresh accumulator for every group (4 MMAs of
// K = 32) in alternating TMEM buffers, and the epilogue folds each group into fp32 registers
// (128 accumulators per thread) with the group's row scale and the tile's 256 column scales,
// staged per group in smem from the transposed weight-scale layout [K/G][N] (coalesced).
namespace gq {
constexpr int G = 128;
constexpr size_t SMEM_BYTES = i8::STAGES * i8::STAGE_BYTES + 1024 + 512 + NUM_EPI_WARPS * 2 * 128 * 4;
static_assert(SMEM_BYTES <= 232448, "227 KB dynamic smem");
}  // namespace gq

struct GParams {
  uint32_t bias[8];        // int4_group_gemm_kernel: the TMEM accumulator bias (gq4::BIAS) x 8
  const float* x_scale;    // [M][ld_sx], K / G per row
  const float* w_scale_t;  // [K / G][ld_sw]
  __half* out;
  int64_t M, N, K, ld_out, ld_sx, ld_sw;
  int num_m, num_n, num_kb, num_tiles, group_m;
};

QR_DEVICE void gtile_coords(const GParams& p, int t, int& mb, int& nb) {
  const int per_group = p.group_m * p.num_n;
  const int group = t / per_group;
  const int first_m = group * p.group_m;
  const int gm = min(p.num_m - first_m, p.group_m);
  const int within = t - group * per_group;
  mb = first_m + within % gm;
  nb = within / gm;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(i8::NUM_THREADS, 1)
    int8_group_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const GParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + i8::STAGES * i8::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* ready = full + i8::STAGES;
  uint64_t* empty = ready + i8::STAGES;
  uint64_t* t_full = empty + i8::STAGES;  // [2]
  uint64_t* t_empty = t_full + 2;         // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 2);
  float* ws_smem = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);  // [warp][2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = (int)blockIdx.x >> 1;
  const int num_pairs = (int)gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < i8::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], 2 * NUM_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == i8::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int my_tiles = (p.num_tiles > pair) ? (p.num_tiles - 1 - pair) / num_pairs + 1 : 0;
  const int total = my_tiles * p.num_kb;
  const int ngroups = (int)(p.K / gq::G);

  if (warp >= NUM_EPI_WARPS) {
    QR_SETMAXNREG_DEC(56);  // 128 x 56 + 256 x 224 = 384 x 168
    if (warp == i8::TMA_WARP) {
      if (lane == 0) {
        for (int it = 0; it < total; ++it) {
          const int tl = it / p.num_kb, kb = it - tl * p.num_kb;
          int mb, nb;
          gtile_coords(p, pair + tl * num_pairs, mb, nb);
          const int s = it % i8::STAGES;
          mbar_wait_sleep(&empty[s], ((it / i8::STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], i8::STAGE_BYTES);
          const uint32_t dst = smem_u32(smem + s * i8::STAGE_BYTES);
          const int ya = mb * BM + (int)rank * BMC, yb = nb * BN + (int)rank * BNC;
          tma_load_2d(dst, &tmA, kb * BK, ya, &full[s]);
          tma_load_2d(dst + BMC * 128, &tmA, kb * BK + 128, ya, &full[s]);
          tma_load_2d(dst + i8::A_BYTES, &tmB, kb * BK, yb, &full[s]);
          tma_load_2d(dst + i8::A_BYTES + BNC * 128, &tmB, kb * BK + 128, yb, &full[s]);
        }
      }
    } else if (warp == i8::RELAY_WARP) {
      if (lane == 0) {
        const uint32_t ready_leader = map_to_rank(&ready[0], 0);
        for (int it = 0; it < total; ++it) {
          const int s = it % i8::STAGES;
          mbar_wait_sleep(&full[s], (it / i8::STAGES) & 1);
          mbar_arrive_cluster(ready_leader + (uint32_t)s * 8u);
        }
      }
    } else if (warp == i8::MMA_WARP) {
      if (rank == 0 && lane == 0) {
        int it = 0, gc = 0;
        for (int tl = 0; tl < my_tiles; ++tl) {
          for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
            const int s = it % i8::STAGES;
            mbar_wait_sleep(&ready[s], (it / i8::STAGES) & 1);
            tc_fence_after();
            const uint32_t base = smem_u32(smem + s * i8::STAGE_BYTES);
            const uint64_t a_desc = umma_desc_sw128(base), b_desc = umma_desc_sw128(base + i8::A_BYTES);
#pragma unroll
            for (int hg = 0; hg < BK / gq::G; ++hg, ++gc) {  // a fresh accumulator per 128-k group
              const int ab = gc & 1;
              mbar_wait_sleep(&t_empty[ab], ((gc >> 1) & 1) ^ 1);
              tc_fence_after();
              const uint32_t d_tmem = tmem_base + (uint32_t)(ab * BN);
#pragma unroll
              for (int k = 4 * hg; k < 4 * hg + 4; ++k) {  // atom k/4 at +16 KB, 32 bytes along K within it
                const uint64_t off = (uint64_t)((k >> 2) * (BMC * 128 / 16) + 2 * (k & 3));
                mma_i8_ss_2sm(d_tmem, a_desc + off, b_desc + off, IDESC, k != 4 * hg ? 1u : 0u);
              }
              mma_commit_pair(&t_full[ab]);
            }
            mma_commit_pair(&empty[s]);
          }
        }
      }
      __syncwarp();
    }
  } else {
    QR_SETMAXNREG_INC(224);
    const uint32_t tempty_leader = map_to_rank(&t_empty[0], 0);
    const int quarter = warp & 3, chalf = warp >> 2;
    const int row_in_tile = (int)rank * BMC + quarter * 32 + lane;
    int gc = 0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      int mb, nb;
      gtile_coords(p, pair + tl * num_pairs, mb, nb);
      const int64_t m = (int64_t)mb * BM + row_in_tile;
      const bool row_ok = m < p.M;
      float2 acc[64];  // columns (2c, 2c + 1) of the thread's 128
#pragma unroll
      for (int c = 0; c < 64; ++c) acc[c] = make_float2(0.f, 0.f);
      // the scales of group g + 1 are loaded while group g is folded (their L2 latency would
      // otherwise sit on every group's critical path); each warp stages its own 128 column
      // scales in a private smem slice (no block-wide barrier per group)
      const int64_t n4 = (int64_t)nb * BN + chalf * 128 + 4 * lane;
      auto ld_ws = [&](int g) {
        return n4 < p.N ? __ldg(reinterpret_cast<const float4*>(p.w_scale_t + (int64_t)g * p.ld_sw + n4))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      float4 ws_next = ld_ws(0);
      float sx_next = row_ok ? __ldg(p.x_scale + m * p.ld_sx) : 0.f;
      for (int g = 0; g < ngroups; ++g, ++gc) {
        const int ab = gc & 1;
        float* wsw = ws_smem + (warp * 2 + ab) * 128;
        reinterpret_cast<float4*>(wsw)[lane] = ws_next;
        const float sx = sx_next;
        if (g + 1 < ngroups) {
          ws_next = ld_ws(g + 1);
          sx_next = row_ok ? __ldg(p.x_scale + m * p.ld_sx + g + 1) : 0.f;
        }
        __syncwarp();
        mbar_wait(&t_full[ab], (gc >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(ab * BN) + (uint32_t)(chalf * 128);
        const float* wsc = wsw;
        const float2 sx2 = make_float2(sx, sx), mg = make_float2(-12582912.f, -12582912.f);
#pragma unroll
        for (int cc = 0; cc < 4; cc += 2) {  // two 32-column chunks per TMEM round trip
          uint32_t rc[2][32];
          QR_TMEM_LD32(taddr + 32u * cc, rc[0]);
          QR_TMEM_LD32(taddr + 32u * cc + 32u, rc[1]);
          tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(wsc + 32 * (cc + h) + c);
              // int32 -> fp32 exactly by the 1.5 * 2^23 magic (|acc_g| <= 128 * 49 < 2^22): an
              // integer add and a packed add instead of the quarter-rate I2F
              const float2 d0 = f2add(make_float2(__int_as_float((int)rc[h][c] + 0x4B400000),
                                                  __int_as_float((int)rc[h][c + 1] + 0x4B400000)), mg);
              const float2 d1 = f2add(make_float2(__int_as_float((int)rc[h][c + 2] + 0x4B400000),
                                                  __int_as_float((int)rc[h][c + 3] + 0x4B400000)), mg);
              const int j = (32 * (cc + h) + c) >> 1;
              acc[j] = f2fma(d0, f2mul(sx2, make_float2(w4.x, w4.y)), acc[j]);
              acc[j + 1] = f2fma(d1, f2mul(sx2, make_float2(w4.z, w4.w)), acc[j + 1]);
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)ab * 8u);
      }
      if (row_ok) {
        __half* dst = p.out + m * p.ld_out + (int64_t)nb * BN + chalf * 128;
        const int64_t n0 = (int64_t)nb * BN + chalf * 128;
#pragma unroll
        for (int c = 0; c < 128; c += 8) {
          if (n0 + c < p.N)
            *reinterpret_cast<uint4*>(dst + c) =
                make_uint4(pack_half2(acc[c / 2].x, acc[c / 2].y), pack_half2(acc[c / 2 + 1].x, acc[c / 2 + 1].y),
                           pack_half2(acc[c / 2 + 2].x, acc[c / 2 + 2].y), pack_half2(acc[c / 2 + 3].x, acc[c / 2 + 3].y));
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == i8::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}


// ============================================================ group-wise W4A4, packed INT4 (§8 f3)
// The same computation as int8_group_gemm_kernel with the codes kept in the paper's 4-bit storage
// (two per byte) and group sizes G = 64, 128, 256 (tab:group_wise_ablation):
//  * TMA loads the PACKED A and B k-blocks (128 rows x 128 B each per CTA) into a 2-stage
//    staging ring; two pairs of widen warps take alternate k-blocks and write the operands
//    widened (the x16 nibble trick of int4_gemm_kernel, [16 lo | 16 hi] per 32-code chunk — the
//    same permutation of k on both sides, inside one group) into a 2-stage SW128 int8 ring;
//  * the MMA warp (leader CTA) runs G / 32 SS MMAs (cta_group::2, M256 N256 K32) per group into
//    one of two 256-column TMEM buffers and commits the buffer to the epilogue;
//  * the buffers hold the bias 0x4B400000 (the fp32 bits of 1.5 * 2^23) when a group starts and
//    every MMA accumulates onto it, so the epilogue reads fp32(1.5 * 2^23 + 256 acc_g) directly
//    (|256 acc_g| <= 256 * 49 * 256 < 2^22): one packed subtract recovers 256 acc_g exactly, one
//    packed multiply forms s_x s_w / 256 and one packed FMA folds the group into the fp32 sums —
//    1.5 issue slots per output element per group; the epilogue then rewrites the bias.
#ifndef QR_GQ_ABL  // timing ablations (scripts/exp/abbench_group.py); 0 = the product kernel
#define QR_GQ_ABL 0
#endif
#ifndef QR_GQ_TWAIT  // the MMA warp's wait for a drained accumulator buffer
#define QR_GQ_TWAIT mbar_wait_sleep
#endif
#ifndef QR_GQ_EWAIT  // the epilogue's wait for a finished group
#define QR_GQ_EWAIT mbar_wait_sleep
#endif
#ifndef QR_GQ_OWAIT  // the MMA warp's wait for a widened operand stage
#define QR_GQ_OWAIT mbar_wait_sleep
#endif
namespace gq4 {
constexpr int SSTAGES = 2, OSTAGES = 2;
constexpr int SSTAGE_BYTES = SA_BYTES + SB_BYTES;  // 32 KB packed
constexpr int OA_BYTES = BMC * BK, OB4_BYTES = BNC * BK;  // 32 KB + 32 KB widened
constexpr int OSTAGE_BYTES = OA_BYTES + OB4_BYTES;
// 16 warps = 512 threads: 0-7 epilogue (216 registers: the 128 fp32 sums + two 16-column chunks),
// warpgroups 2-3 (40 registers) = 8 TMA, 9 MMA, 10-13 widen (two pairs on alternate k-blocks; in a
// pair one warp widens A, the other B), 14-15 idle
constexpr int EPI_WARPS = 8, TMA_WARP = 8, MMA_WARP = 9, W_WARP0 = 10, NUM_W = 4;
constexpr int NUM_THREADS = 16 * 32;
constexpr int WS_BYTES = EPI_WARPS * 2 * 128 * 4;  // per epilogue warp, per buffer: 128 column scales
constexpr size_t SMEM_BYTES = 1024 + SSTAGES * SSTAGE_BYTES + OSTAGES * OSTAGE_BYTES + 512 + WS_BYTES;
static_assert(SMEM_BYTES <= 232448, "227 KB dynamic smem");
constexpr uint32_t BIAS = 0x4B400000u;
}  // namespace gq4

template <int G>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gq4::NUM_THREADS, 1)
    int4_group_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const GParams p) {
  static_assert(G == 64 || G == 128 || G == 256, "group size");
  constexpr int GPK = BK / G;       // groups per k-block
  constexpr int MPG = G / 32;       // MMAs per group
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_smem = smem;                                        // [SSTAGES][A 16 KB | B 16 KB] packed
  uint8_t* op_smem = smem + gq4::SSTAGES * gq4::SSTAGE_BYTES;         // [OSTAGES][A 32 KB | B 32 KB] int8 SW128
  uint64_t* bars = reinterpret_cast<uint64_t*>(op_smem + gq4::OSTAGES * gq4::OSTAGE_BYTES);
  uint64_t* st_full = bars;                         // [SSTAGES] TMA -> widen group
  uint64_t* st_empty = st_full + gq4::SSTAGES;      // [SSTAGES] widen pair -> TMA
  uint64_t* op_full = st_empty + gq4::SSTAGES;      // [OSTAGES] widen warps of both CTAs -> leader MMA
  uint64_t* op_empty = op_full + gq4::OSTAGES;      // [OSTAGES] MMA commit -> widen warps
  uint64_t* t_full = op_empty + gq4::OSTAGES;       // [2] MMA commit -> epilogue
  uint64_t* t_empty = t_full + 2;                   // [2] epilogues of both CTAs -> leader MMA
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 2);
  float* ws_smem = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = (int)blockIdx.x >> 1;
  const int num_pairs = (int)gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < gq4::SSTAGES; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], 2);
    }
    for (int s = 0; s < gq4::OSTAGES; ++s) {
      mbar_init(&op_full[s], 2 * 2);
      mbar_init(&op_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], 2 * gq4::EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == gq4::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == gq4::TMA_WARP && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (warp < gq4::EPI_WARPS) {  // both accumulator buffers start at the bias (this CTA's lanes)
    const int quarter = warp & 3, chalf = warp >> 2;
    uint32_t bias8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) bias8[i] = gq4::BIAS;
#pragma unroll 1
    for (int c = 0; c < 32; ++c)
      QR_TMEM_ST8(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)((c >> 4) * BN + chalf * 128 + 8 * (c & 15)),
                  bias8);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const int my_tiles = (p.num_tiles > pair) ? (p.num_tiles - 1 - pair) / num_pairs + 1 : 0;
  const int total = my_tiles * p.num_kb;
  const int ngroups = (int)(p.K / G);

  // register budgets per role (setmaxnreg is warpgroup-wide: warps 8-15 are warpgroups 2-3).  An
  // increase draws only on what this CTA's decreases released: 256 x (128 - 40) = 256 x (216 - 128)
  if (warp >= gq4::TMA_WARP) {
    QR_SETMAXNREG_DEC(40);  // one instruction per warpgroup (.sync.aligned)
  }
  if (warp == gq4::TMA_WARP || warp == gq4::MMA_WARP) {
    if (warp == gq4::TMA_WARP) {
      if (lane == 0) {
        for (int it = 0; it < total; ++it) {
          const int tl = it / p.num_kb, kb = it - tl * p.num_kb;
          int mb, nb;
          gtile_coords(p, pair + tl * num_pairs, mb, nb);
          const int s = it % gq4::SSTAGES;
          mbar_wait_sleep(&st_empty[s], ((it / gq4::SSTAGES) & 1) ^ 1);
          mbar_expect_tx(&st_full[s], gq4::SSTAGE_BYTES);
          const uint32_t dst = smem_u32(stage_smem + s * gq4::SSTAGE_BYTES);
          tma_load_2d(dst, &tmA, kb * BKP, mb * BM + (int)rank * BMC, &st_full[s]);
          tma_load_2d(dst + SA_BYTES, &tmB, kb * BKP, nb * BN + (int)rank * BNC, &st_full[s]);
        }
      }
    } else if (warp == gq4::MMA_WARP) {
      if (rank == 0 && lane == 0) {
        int it = 0, gc = 0;
        for (int tl = 0; tl < my_tiles; ++tl) {
          for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
            const int o = it % gq4::OSTAGES;
            QR_GQ_OWAIT(&op_full[o], (it / gq4::OSTAGES) & 1);
            tc_fence_after();
            const uint32_t base = smem_u32(op_smem + o * gq4::OSTAGE_BYTES);
            const uint64_t a_desc = umma_desc_sw128(base), b_desc = umma_desc_sw128(base + gq4::OA_BYTES);
#pragma unroll
            for (int hg = 0; hg < GPK; ++hg, ++gc) {
              const int ab = gc & 1;
              QR_GQ_TWAIT(&t_empty[ab], ((gc >> 1) & 1) ^ 1);
              tc_fence_after();
              const uint32_t d_tmem = tmem_base + (uint32_t)(ab * BN);
#pragma unroll
              for (int k = MPG * hg; k < MPG * hg + MPG; ++k) {  // atom k/4 at +16 KB, 32 bytes along K within it
                const uint64_t off = (uint64_t)((k >> 2) * (BMC * 128 / 16) + 2 * (k & 3));
                mma_i8_ss_2sm(d_tmem, a_desc + off, b_desc + off, IDESC, 1u);  // onto the bias
              }
              mma_commit_pair(&t_full[ab]);
            }
            mma_commit_pair(&op_empty[o]);
          }
        }
      }
      __syncwarp();
    }
  } else if (warp >= gq4::W_WARP0 && warp < gq4::W_WARP0 + gq4::NUM_W) {
    // ===================== widen A or B: packed smem -> int8 SW128 smem =====================
    // lane t owns packed chunk qc = t % 8 of rows rr0 + 4 i (rr0 = t / 8 < 4, i < 32): the swizzle
    // phase of row r = rr0 + 8 i2 + 4 h is rr0 + 4 h, and r / 8 = i2, so both variants are
    // precomputed.  Widened: chunk qc -> K atom qc / 4, int8 chunks 2 (qc % 4) (lo nibbles) and +1
    // (hi nibbles) of the row's 128-byte line; each 8-lane store phase covers all 8 chunk slots.
    const int wi = (warp - gq4::W_WARP0) >> 1;    // the pair takes k-blocks it == wi (mod 2)
    const int opnd = (warp - gq4::W_WARP0) & 1;   // 0: A, 1: B
    const uint32_t t = (uint32_t)lane;
    const uint32_t rr0 = t >> 3, qc = t & 7u;
    const uint32_t atom = qc >> 2, qa = qc & 3u, odd = atom & 1u;
    const uint32_t sh0 = odd ? 0u : 4u, sh1 = odd ? 4u : 0u;
    uint32_t src_off[2], dst_off[2], d0[2], d1[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t swz = rr0 + 4u * h;
      src_off[h] = swz * BKP + ((qc ^ swz) << 4);
      dst_off[h] = atom * (BNC * 128u) + swz * 128u;
      d0[h] = ((2u * qa + odd) ^ swz) << 4;
      d1[h] = ((2u * qa + (odd ^ 1u)) ^ swz) << 4;
    }
    const uint32_t opfull_leader = map_to_rank(&op_full[0], 0);
    for (int it = wi; it < total; it += 2) {
      const int s = it % gq4::SSTAGES;
      const int o = it % gq4::OSTAGES;
      mbar_wait_sleep(&st_full[s], (it / gq4::SSTAGES) & 1);
      QR_OPWAIT(&op_empty[o], ((it / gq4::OSTAGES) & 1) ^ 1);
      {
        const uint32_t src = smem_u32(stage_smem + s * gq4::SSTAGE_BYTES) + (opnd ? SA_BYTES : 0);
        const uint32_t dst = smem_u32(op_smem + o * gq4::OSTAGE_BYTES) + (opnd ? gq4::OA_BYTES : 0);
#pragma unroll 1
        for (int i0 = 0; i0 < ((QR_GQ_ABL & 4) ? 0 : 16); i0 += 2) {  // row octets i0, i0 + 1 (two rows per lane each)
          uint4 w[2][2];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) w[i][h] = lds_v4(src + (uint32_t)(i0 + i) * 1024u + src_off[h]);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint4 v = w[i][h];
              const uint32_t base = dst + (uint32_t)(i0 + i) * 1024u + dst_off[h];
              sts_v4(base + d0[h], make_uint4((v.x << sh0) & 0xF0F0F0F0u, (v.y << sh0) & 0xF0F0F0F0u,
                                              (v.z << sh0) & 0xF0F0F0F0u, (v.w << sh0) & 0xF0F0F0F0u));
              sts_v4(base + d1[h], make_uint4((v.x << sh1) & 0xF0F0F0F0u, (v.y << sh1) & 0xF0F0F0F0u,
                                              (v.z << sh1) & 0xF0F0F0F0u, (v.w << sh1) & 0xF0F0F0F0u));
            }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&st_empty[s]);
        mbar_arrive_cluster(opfull_leader + (uint32_t)o * 8u);
      }
    }
  } else if (warp < gq4::EPI_WARPS) {
    QR_SETMAXNREG_INC(216);
    // ===================== epilogue warps 0..7: fold every group into fp32 sums =====================
    const uint32_t tempty_leader = map_to_rank(&t_empty[0], 0);
    const int quarter = warp & 3, chalf = warp >> 2;
    const int row_in_tile = (int)rank * BMC + quarter * 32 + lane;
    // the bias block is read from kernel parameters, so the compiler keeps it in one register
    // block instead of re-materializing the constant before every store
    uint32_t bias8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) bias8[i] = p.bias[i];
    int gc = 0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      int mb, nb;
      gtile_coords(p, pair + tl * num_pairs, mb, nb);
      const int64_t m = (int64_t)mb * BM + row_in_tile;
      const bool row_ok = m < p.M;
      float2 acc[64];  // columns (2c, 2c + 1) of the thread's 128
#pragma unroll
      for (int c = 0; c < 64; ++c) acc[c] = make_float2(0.f, 0.f);
      const int64_t n4 = (int64_t)nb * BN + chalf * 128 + 4 * lane;
      auto ld_ws = [&](int g) {
        return n4 < p.N ? __ldg(reinterpret_cast<const float4*>(p.w_scale_t + (int64_t)g * p.ld_sw + n4))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      float4 ws_next = ld_ws(0);
      float sx_next = row_ok ? __ldg(p.x_scale + m * p.ld_sx) : 0.f;
      for (int g = 0; g < ngroups; ++g, ++gc) {
        const int ab = gc & 1;
        float* wsw = ws_smem + (warp * 2 + ab) * 128;
        reinterpret_cast<float4*>(wsw)[lane] = ws_next;
        const float sx = sx_next * (1.f / 256.f);  // the x16 nibble scaling of both operands
        if (g + 1 < ngroups) {
          ws_next = ld_ws(g + 1);
          sx_next = row_ok ? __ldg(p.x_scale + m * p.ld_sx + g + 1) : 0.f;
        }
        __syncwarp();
        QR_GQ_EWAIT(&t_full[ab], (gc >> 1) & 1);  // sleeping, not spinning: the widen warps share these schedulers
        tc_fence_after();
        const uint32_t taddr =
            tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(ab * BN) + (uint32_t)(chalf * 128);
        const float2 sx2 = make_float2(sx, sx), mg = make_float2(-12582912.f, -12582912.f);
        // 16-column chunks, software-pipelined: the load of chunk c + 1 is in flight while chunk c
        // is folded (tcgen05.wait::ld waits for every outstanding load, so one wait per chunk)
        uint32_t rc[2][16];
        float4 wsc[2][4];  // the chunk's 16 column scales, loaded one chunk ahead
        const uint32_t wsa = smem_u32(wsw);
        auto ld_wsc = [&](int cc, float4(&w)[4]) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(w[i].x), "=f"(w[i].y), "=f"(w[i].z), "=f"(w[i].w)
                         : "r"(wsa + (uint32_t)(64 * cc + 16 * i)));
        };
        ld_wsc(0, wsc[0]);
        QR_TMEM_LD16(taddr, rc[0]);
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          uint32_t(&cur)[16] = rc[cc & 1];
          const float4(&w)[4] = wsc[cc & 1];
          if (!(QR_GQ_ABL & 2)) {
            QR_TMEM_ST8(taddr + 16u * cc, bias8);  // the next group of this buffer starts at the bias
            QR_TMEM_ST8(taddr + 16u * cc + 8u, bias8);
          }
          if (cc + 1 < 8) {
            QR_TMEM_LD16(taddr + 16u * (cc + 1), rc[(cc + 1) & 1]);
            if (!(QR_GQ_ABL & 8)) ld_wsc(cc + 1, wsc[(cc + 1) & 1]);
          }
          if (QR_GQ_ABL & 1) {
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[(16 * cc + c) >> 1].x += __uint_as_float(cur[c]);
          } else
#pragma unroll
          for (int c = 0; c < 16; c += 4) {
            const float4 w4 = w[c >> 2];
            const float2 d0 = f2add(make_float2(__uint_as_float(cur[c]), __uint_as_float(cur[c + 1])), mg);
            const float2 d1 = f2add(make_float2(__uint_as_float(cur[c + 2]), __uint_as_float(cur[c + 3])), mg);
            const int j = (16 * cc + c) >> 1;
            acc[j] = f2fma(d0, f2mul(sx2, make_float2(w4.x, w4.y)), acc[j]);
            acc[j + 1] = f2fma(d1, f2mul(sx2, make_float2(w4.z, w4.w)), acc[j + 1]);
          }
          if (cc + 1 < 8) tmem_ld_wait();
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)ab * 8u);
      }
      if (row_ok) {
        __half* dst = p.out + m * p.ld_out + (int64_t)nb * BN + chalf * 128;
        const int64_t n0 = (int64_t)nb * BN + chalf * 128;
#pragma unroll
        for (int c = 0; c < 128; c += 8) {
          if (n0 + c < p.N)
            *reinterpret_cast<uint4*>(dst + c) =
                make_uint4(pack_half2(acc[c / 2].x, acc[c / 2].y), pack_half2(acc[c / 2 + 1].x, acc[c / 2 + 1].y),
                           pack_half2(acc[c / 2 + 2].x, acc[c / 2 + 2].y), pack_half2(acc[c / 2 + 3].x, acc[c / 2 + 3].y));
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == gq4::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

}  // namespace gemm

namespace {

int g_num_sms[64];

int num_sms_current() {
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D map over packed INT4 rows: [rows][K/2 bytes] with row pitch ld bytes; box 128 B x 128
// rows, SWIZZLE_128B (16-byte chunk c of row r lands at chunk c ^ (r & 7)); rows past the end
// are zero-filled.
bool make_packed_map(CUtensorMap* map, const uint8_t* base, int64_t rows, int64_t kbytes, int64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kbytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)gemm::BKP, 128u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// residual fp16 [rows][ld] as a 2-D map, box 64 columns (128 B) x 32 rows, SWIZZLE_128B (the
// residual epilogue's per-warp staging box); OOB rows / columns are zero-filled
bool make_res_map(CUtensorMap* map, const __half* base, int64_t rows, int64_t cols, int64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64u, 32u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

int g_gemm_debug_mode = 0;
int g_gemm_group_m = 0;  // debug override of the raster group (0 = automatic)

template <bool kS32>
static cudaError_t launch_gemm_impl(const uint8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                                    const uint8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* out,
                                    int64_t ld_out, cudaStream_t stream, const void* residual = nullptr,
                                    int64_t ld_r = 0, int swiglu = 0) {
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
  CUtensorMap ma, mb, mr;
  if (!make_packed_map(&ma, xq, M, K / 2, ld_xq) || !make_packed_map(&mb, wq, N, K / 2, ld_wq))
    return cudaErrorInvalidValue;
  if (residual && !kS32) {
    if (!make_res_map(&mr, static_cast<const __half*>(residual), M, N, ld_r)) return cudaErrorInvalidValue;
  } else {
    mr = mb;  // unused
  }
  Params p;
  p.x_scale = xs;
  p.w_scale = ws;
  p.out = out;
  p.residual = static_cast<const __half*>(residual);
  p.ld_r = ld_r;
  p.swiglu = swiglu;
  p.M = M;
  p.N = N;
  p.K = K;
  p.ld_out = ld_out;
  p.num_m = (int)((M + BM - 1) / BM);
  p.num_n = (int)((N + BN - 1) / BN);
  p.num_kb = (int)((K + BK - 1) / BK);  // a K % 256 == 128 tail is zero-filled by the TMA
  p.num_tiles = p.num_m * p.num_n;
  // Raster group: the ~74 concurrently running tiles share the A rows of group_m pair-rows,
  // which stay in L2 while the group walks across N, so B is re-read from DRAM num_m / group_m
  // times.  ~64 MB of A per group, 8..32 pair-rows (measured best on the Llama-2-70B linears:
  // 32 at K = 8192, 16 at K = 28672; within 3% across 8..64).
  {
    const int64_t a_tile_bytes = (int64_t)BM * (K / 2);
    int g = (int)((64ll << 20) / (a_tile_bytes > 0 ? a_tile_bytes : 1));
    g = g < 8 ? 8 : (g > 32 ? 32 : g);
    if (g_gemm_group_m > 0) g = g_gemm_group_m;
    p.group_m = g < 1 ? 1 : (g > p.num_m ? p.num_m : g);
  }
  const int max_pairs = num_sms_current() / 2;
  const int pairs = p.num_tiles < max_pairs ? p.num_tiles : max_pairs;
  if (g_gemm_debug_mode >= 1 && g_gemm_debug_mode <= 8) {
    auto kern = g_gemm_debug_mode == 1   ? int4_gemm_kernel<kS32, 1>
                : g_gemm_debug_mode == 2 ? int4_gemm_kernel<kS32, 2>
                : g_gemm_debug_mode == 3 ? int4_gemm_kernel<kS32, 3>
                : g_gemm_debug_mode == 4 ? int4_gemm_kernel<kS32, 4>
                : g_gemm_debug_mode == 5 ? int4_gemm_kernel<kS32, 5>
                : g_gemm_debug_mode == 6 ? int4_gemm_kernel<kS32, 6>
                : g_gemm_debug_mode == 7 ? int4_gemm_kernel<kS32, 7>
                                         : int4_gemm_kernel<kS32, 8>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<2 * pairs, NUM_THREADS, SMEM_BYTES, stream>>>(ma, mb, mr, p);
  } else {
    const int epi = kS32 ? 0 : (swiglu ? 3 : (residual ? 2 : 1));
    auto kern = epi == 1 ? int4_gemm_kernel<kS32, 0, 1> : epi == 2 ? int4_gemm_kernel<kS32, 0, 2>
              : epi == 3 ? int4_gemm_kernel<kS32, 0, 3> : int4_gemm_kernel<kS32, 0, 0>;
    static bool attr_epi[64][4] = {};
    if (!attr_epi[dev & 63][epi]) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
      if (e != cudaSuccess) return e;
      attr_epi[dev & 63][epi] = true;
    }
    kern<<<2 * pairs, NUM_THREADS, SMEM_BYTES, stream>>>(ma, mb, mr, p);
  }
  return cudaPeekAtLastError();
}

// A8W8: int8 rows [rows][K] (ld bytes), box 128 B x 128 rows, SWIZZLE_128B (one UMMA atom)
static bool make_i8_map(CUtensorMap* map, const uint8_t* base, int64_t rows, int64_t K, int64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {128u, 128u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool kS32>
static cudaError_t launch_i8_impl(const int8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                                  const int8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* out,
                                  int64_t ld_out, cudaStream_t stream, const void* residual, int64_t ld_r) {
  using namespace gemm;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(int8_gemm_kernel<kS32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)i8::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  CUtensorMap ma, mb;
  if (!make_i8_map(&ma, reinterpret_cast<const uint8_t*>(xq), M, K, ld_xq) ||
      !make_i8_map(&mb, reinterpret_cast<const uint8_t*>(wq), N, K, ld_wq))
    return cudaErrorInvalidValue;
  Params p;
  p.x_scale = xs;
  p.w_scale = ws;
  p.out = out;
  p.residual = static_cast<const __half*>(residual);
  p.ld_r = ld_r;
  p.swiglu = 0;
  p.M = M;
  p.N = N;
  p.K = K;
  p.ld_out = ld_out;
  p.num_m = (int)((M + BM - 1) / BM);
  p.num_n = (int)((N + BN - 1) / BN);
  p.num_kb = (int)((K + BK - 1) / BK);
  p.num_tiles = p.num_m * p.num_n;
  {
    const int64_t a_tile_bytes = (int64_t)BM * K;
    int g = (int)((64ll << 20) / (a_tile_bytes > 0 ? a_tile_bytes : 1));
    g = g < 8 ? 8 : (g > 32 ? 32 : g);
    p.group_m = g > p.num_m ? p.num_m : g;
  }
  const int max_pairs = num_sms_current() / 2;
  const int pairs = p.num_tiles < max_pairs ? p.num_tiles : max_pairs;
  int8_gemm_kernel<kS32><<<2 * pairs, i8::NUM_THREADS, i8::SMEM_BYTES, stream>>>(ma, mb, p);
  return cudaPeekAtLastError();
}

cudaError_t launch_int8_gemm(const int8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                             const int8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* y, int64_t ld_y,
                             cudaStream_t stream, const void* residual, int64_t ld_r) {
  return launch_i8_impl<false>(xq, xs, M, K, ld_xq, wq, ws, N, ld_wq, y, ld_y, stream, residual, ld_r);
}

cudaError_t launch_int8_gemm_s32(const int8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const int8_t* wq, int64_t N,
                                 int64_t ld_wq, int32_t* acc, int64_t ld_acc, cudaStream_t stream) {
  return launch_i8_impl<true>(xq, nullptr, M, K, ld_xq, wq, nullptr, N, ld_wq, acc, ld_acc, stream, nullptr, 0);
}


cudaError_t launch_int8_group_gemm(const int8_t* xq, const float* xs, int64_t ld_sx, int64_t M, int64_t K,
                                   int64_t ld_xq, const int8_t* wq, const float* ws_t, int64_t ld_sw, int64_t N,
                                   int64_t ld_wq, void* y, int64_t ld_y, cudaStream_t stream) {
  using namespace gemm;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(int8_group_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)gq::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  CUtensorMap ma, mb;
  if (!make_i8_map(&ma, reinterpret_cast<const uint8_t*>(xq), M, K, ld_xq) ||
      !make_i8_map(&mb, reinterpret_cast<const uint8_t*>(wq), N, K, ld_wq))
    return cudaErrorInvalidValue;
  GParams p;
  p.x_scale = xs;
  p.w_scale_t = ws_t;
  p.out = static_cast<__half*>(y);
  p.M = M;
  p.N = N;
  p.K = K;
  p.ld_out = ld_y;
  p.ld_sx = ld_sx;
  p.ld_sw = ld_sw;
  p.num_m = (int)((M + BM - 1) / BM);
  p.num_n = (int)((N + BN - 1) / BN);
  p.num_kb = (int)(K / BK);
  p.num_tiles = p.num_m * p.num_n;
  {
    const int64_t a_tile_bytes = (int64_t)BM * K;
    int g = (int)((64ll << 20) / (a_tile_bytes > 0 ? a_tile_bytes : 1));
    g = g < 8 ? 8 : (g > 32 ? 32 : g);
    p.group_m = g > p.num_m ? p.num_m : g;
  }
  const int max_pairs = num_sms_current() / 2;
  const int pairs = p.num_tiles < max_pairs ? p.num_tiles : max_pairs;
  int8_group_gemm_kernel<<<2 * pairs, i8::NUM_THREADS, gq::SMEM_BYTES, stream>>>(ma, mb, p);
  return cudaPeekAtLastError();
}

cudaError_t launch_int4_group_gemm(const uint8_t* xq, const float* xs, int64_t ld_sx, int64_t M, int64_t K,
                                   int64_t ld_xq, const uint8_t* wq, const float* ws_t, int64_t ld_sw, int64_t N,
                                   int64_t ld_wq, int group, void* y, int64_t ld_y, cudaStream_t stream) {
  using namespace gemm;
  auto kern = group == 64 ? int4_group_gemm_kernel<64> : group == 128 ? int4_group_gemm_kernel<128>
                                                                       : int4_group_gemm_kernel<256>;
  static bool attr_set[64][3] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int gi = group == 64 ? 0 : group == 128 ? 1 : 2;
  if (!attr_set[dev & 63][gi]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gq4::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63][gi] = true;
  }
  CUtensorMap ma, mb;
  if (!make_packed_map(&ma, xq, M, K / 2, ld_xq) || !make_packed_map(&mb, wq, N, K / 2, ld_wq))
    return cudaErrorInvalidValue;
  GParams p;
  for (int i = 0; i < 8; ++i) p.bias[i] = gq4::BIAS;
  p.x_scale = xs;
  p.w_scale_t = ws_t;
  p.out = static_cast<__half*>(y);
  p.M = M;
  p.N = N;
  p.K = K;
  p.ld_out = ld_y;
  p.ld_sx = ld_sx;
  p.ld_sw = ld_sw;
  p.num_m = (int)((M + BM - 1) / BM);
  p.num_n = (int)((N + BN - 1) / BN);
  p.num_kb = (int)(K / BK);
  p.num_tiles = p.num_m * p.num_n;
  {
    const int64_t a_tile_bytes = (int64_t)BM * (K / 2);
    int g = (int)((64ll << 20) / (a_tile_bytes > 0 ? a_tile_bytes : 1));
    g = g < 8 ? 8 : (g > 32 ? 32 : g);
    p.group_m = g > p.num_m ? p.num_m : g;
  }
  const int max_pairs = num_sms_current() / 2;
  const int pairs = p.num_tiles < max_pairs ? p.num_tiles : max_pairs;
  kern<<<2 * pairs, gq4::NUM_THREADS, gq4::SMEM_BYTES, stream>>>(ma, mb, p);
  return cudaPeekAtLastError();
}

// Debug / roofline probe (not in the public header): mode 1 = MMA issue only.
extern "C" void quarot_debug_gemm_mode(int32_t mode) { g_gemm_debug_mode = mode; }
extern "C" void quarot_debug_gemm_group_m(int32_t g) { g_gemm_group_m = g; }

cudaError_t launch_int4_gemm(const uint8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                             const uint8_t* wq, const float* ws, int64_t N, int64_t ld_wq, void* y,
                             int64_t ld_y, cudaStream_t stream, const void* residual, int64_t ld_r) {
  return launch_gemm_impl<false>(xq, xs, M, K, ld_xq, wq, ws, N, ld_wq, y, ld_y, stream, residual, ld_r);
}

cudaError_t launch_int4_gemm_swiglu(const uint8_t* xq, const float* xs, int64_t M, int64_t K, int64_t ld_xq,
                                    const uint8_t* wq, const float* ws, int64_t N2, int64_t ld_wq, void* act,
                                    int64_t ld_act, cudaStream_t stream) {
  return launch_gemm_impl<false>(xq, xs, M, K, ld_xq, wq, ws, N2, ld_wq, act, ld_act, stream, nullptr, 0, 1);
}

cudaError_t launch_int4_gemm_s32(const uint8_t* xq, int64_t M, int64_t K, int64_t ld_xq, const uint8_t* wq,
                                 int64_t N, int64_t ld_wq, int32_t* acc, int64_t ld_acc, cudaStream_t stream) {
  return launch_gemm_impl<true>(xq, nullptr, M, K, ld_xq, wq, nullptr, N, ld_wq, acc, ld_acc, stream);
}

}  // namespace qr
