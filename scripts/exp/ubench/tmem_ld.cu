// TMEM load throughput micro-benchmark: cycles per tcgen05.ld per SM for several shapes, with and
// without .pack::16b (does packing two 16-bit halves halve the TMEM read cost?).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD32(SHAPE, r, a)                                                                                   \
  asm volatile("tcgen05.ld.sync.aligned." SHAPE ".b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                     \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),      \
                 "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),   \
                 "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),   \
                 "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                           \
               : "r"(a))

template <int V>
__global__ void __launch_bounds__(512, 1) k(int iters, int nwarps, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = holder + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      const uint32_t a = base + (uint32_t)((i & 1) * 256);
      if (V == 0) LD32("32x32b.x32", r, a);             // 32 columns, 32 regs
      if (V == 1) LD32("32x32b.x32.pack::16b", r, a);   // 64 columns (low halves), 32 regs
      if (V == 2) LD32("16x256b.x8", r, a);             // 16 lanes x 256 bit x 8
      if (V == 3) LD32("16x128b.x16", r, a);
      if (V == 4) {  // store throughput: 32x32b.x32 of 32 registers
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = acc + j;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                     :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                     "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
                     "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
                     "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        r[0] = i; r[31] = 0; r[17] = 0;
      } else
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= r[0] ^ r[31] ^ r[17];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 4096);
  const char* names[] = {"32x32b.x32", "32x32b.x32.pack16", "16x256b.x8", "16x128b.x16", "st 32x32b.x32"};
  const int iters = 20000;
  for (int nw : {4, 8, 12, 16}) {
    for (int v = 0; v < 5; ++v) {
      auto f = v == 0 ? k<0> : v == 1 ? k<1> : v == 2 ? k<2> : v == 3 ? k<3> : k<4>;
      f<<<148, 512>>>(iters, nw, cyc, sink);
      f<<<148, 512>>>(iters, nw, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      double c = (double)h[0] / iters;  // cycles per iteration (all warps)
      // register bytes per SM per iteration: nw warps x 32 lanes x 32 regs x 4 B
      const double rbytes = nw * 32.0 * 32 * 4;
      printf("%-20s warps %2d: %7.1f cyc/iter  %6.1f reg-B/cyc/SM  err=%s\n", names[v], nw, c, rbytes / c,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
