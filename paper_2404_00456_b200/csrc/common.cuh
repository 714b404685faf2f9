// common.cuh — sm_100a PTX helpers shared by the QuaRot kernels (mbarrier, tcgen05, fences).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define QR_DEVICE __device__ __forceinline__

namespace qr {

QR_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
QR_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
QR_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
QR_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
QR_DEVICE bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
QR_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  while (!mbar_try_wait(addr, parity)) {
  }
}
// try_wait with a suspend-time hint: the waiting warp sleeps (until the phase completes or the
// hint elapses) instead of spinning, so idle roles do not steal issue slots from busy ones.
QR_DEVICE bool mbar_try_wait_sleep(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// try_wait + an explicit back-off: for producer warps whose waits are long (a row of epilogue
// work), so their retries do not take issue slots from the epilogue warps on the same SMSP
// (try_wait's suspend hint wakes on every barrier event of the CTA)
template <int kNs>
QR_DEVICE void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  while (!mbar_try_wait(addr, parity)) __nanosleep(kNs);
}
QR_DEVICE void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  while (!mbar_try_wait_sleep(addr, parity)) {
  }
}

// silu(g) = g / (1 + e^-g) in fp32 with the fast reciprocal division (MUFU.RCP + FMUL, <= 2 ulp;
// the IEEE division was ~8 instructions and a slow-path branch per element of the SwiGLU epilogue).
// The GEMM's fused SwiGLU epilogue and the standalone quarot_swiglu kernel both use this, so the
// fused and unfused chains stay bitwise equal; fp16(silu) then rounds away the fp32 difference
// except within ~2^-21 of an fp16 rounding boundary.
// e^-g as __expf(-g) computes it (ex2.approx of -g * log2(e) in fp32), with .ftz: only a subnormal
// e^-g differs (flushed to 0), and 1 + subnormal == 1 in fp32, so silu is bitwise unchanged while
// the non-ftz form's subnormal range fix-up (a compare and two predicated multiplies) disappears.
QR_DEVICE float silu_f32(float g) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(g * -1.44269502162933349609375f));
  return __fdividef(g, 1.f + e);
}

// RoPE rotate-half of one pair in fp32 with one fixed rounding sequence, so every
// kernel that applies it (the standalone RoPE kernel and the RoPE fused into the KV passes) agrees
// bitwise: x1 c - x2 s = fma(x1, c, -rn(x2 s)) and x2 c + x1 s = fma(x2, c, rn(x1 s)).  (The
// fma form, because ptxas contracts packed mul.rn.f32x2 + sub.rn.f32x2 into FFMA2 even with the
// explicit rounding modifier; the packed forms below state the same arithmetic explicitly.)
QR_DEVICE float rope_first(float x1, float x2, float c, float s) { return __fmaf_rn(x1, c, -__fmul_rn(x2, s)); }
QR_DEVICE float rope_second(float x1, float x2, float c, float s) { return __fmaf_rn(x2, c, __fmul_rn(x1, s)); }

// ---------------------------------------------------------------- proxy fences
// generic-proxy st.shared -> async-proxy (tcgen05.mma operand) visibility
QR_DEVICE void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05 / TMEM
QR_DEVICE void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
}
QR_DEVICE void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
QR_DEVICE void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
QR_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
QR_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem desc] * B[smem desc]^T, kind::i8 (s8 x s8 -> s32), one CTA.
QR_DEVICE void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
QR_DEVICE void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets lane (base+i).
#define QR_TMEM_LD32(taddr, r)                                                                        \
  asm volatile(                                                                                       \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                     \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),           \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),    \
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),    \
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                             \
      : "r"(taddr))
#define QR_TMEM_LD16(taddr, r)                                                                        \
  asm volatile(                                                                                       \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),           \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
        "=r"(r[14]), "=r"(r[15])                                                                       \
      : "r"(taddr))
QR_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B canonical layout:
// 8-row x 128-byte swizzle atoms stacked along M/N at 1024 B (SBO); LBO unused (=1).
QR_DEVICE uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);        // start address  [0,14)
  d |= (uint64_t)1 << 16;                             // LBO (ignored for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                   // SBO = 1024 B  [32,46)
  d |= (uint64_t)1 << 46;                             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                             // layout type SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::i8: s8 x s8 -> s32, A and B K-major, shape M x N.
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
  return (2u << 4)            // D format S32
         | (1u << 7)          // A signed 8-bit
         | (1u << 10)         // B signed 8-bit
         | ((N >> 3) << 17)   // N / 8
         | ((M >> 4) << 24);  // M / 16
}

// ---------------------------------------------------------------- misc
QR_DEVICE float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

QR_DEVICE float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

QR_DEVICE uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

QR_DEVICE void sts_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------- packed fp32x2 (sm_100)
QR_DEVICE float2 f2add(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0,%1}, rc;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
QR_DEVICE float2 f2sub(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "sub.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0,%1}, rc;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
QR_DEVICE float2 f2fma(float2 a, float2 b, float2 cc) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(cc.x), "f"(cc.y));
  return r;
}
QR_DEVICE float2 f2mul(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mul.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0,%1}, rc;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// rope_first / rope_second on two pairs at once (packed fp32x2, the same roundings)
QR_DEVICE float2 rope_first2(float2 x1, float2 x2, float2 c, float2 sn) {
  const float2 t = f2mul(x2, sn);
  return f2fma(x1, c, make_float2(-t.x, -t.y));
}
QR_DEVICE float2 rope_second2(float2 x1, float2 x2, float2 c, float2 sn) { return f2fma(x2, c, f2mul(x1, sn)); }
// (x + y, x - y) of the pair held in one float2: ONE FFMA2, p * (1, -1) + swap(p) — SASS
// `FFMA2 d, p, UR.F32x2, p.F32x2.LO_HI`, the constant read from a uniform register pair (the
// broadcast form y * (1, -1) + x made ptxas re-materialise the 1.0 before every FFMA2: +1 MOV
// per pair).  The multiply by +-1 is exact, so d = (fl(x + y), fl(x - y)) bitwise.
QR_DEVICE float2 pair_bfly(float2 p) { return f2fma(p, make_float2(1.f, -1.f), make_float2(p.y, p.x)); }
// the broadcast form y * (1, -1) + x (same results); the K = 11008 kernel schedules better with it
// (measured: 1.17 vs 1.24 ms at 131072 tokens)
QR_DEVICE float2 pair_bfly_bc(float2 p) {
  return f2fma(make_float2(p.y, p.y), make_float2(1.f, -1.f), make_float2(p.x, p.x));
}
// byte = nib(rne(clamp(v.x * inv))) | nib(rne(clamp(v.y * inv))) << 4; RNE via 1.5 * 2^23
QR_DEVICE uint32_t quant_pair(float2 v, float inv) {
  float2 m = f2mul(v, make_float2(inv, inv));
  m.x = fminf(fmaxf(m.x, -7.f), 7.f);
  m.y = fminf(fmaxf(m.y, -7.f), 7.f);
  m = f2add(m, make_float2(12582912.f, 12582912.f));
  return (__float_as_uint(m.x) & 0xFu) | ((__float_as_uint(m.y) & 0xFu) << 4);
}

}  // namespace qr
