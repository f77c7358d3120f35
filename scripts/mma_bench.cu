// Microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::f16 (M=128, K=16)
// back to back into 8 TMEM accumulators, vs N; A operand SWIZZLE_NONE (SW=0) or
// SWIZZLE_32B (SW=1, the conv's halo layout), B SWIZZLE_NONE K-major.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint64_t desc_sw32(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46) |
         (6ull << 61);
}
template <int N, int SW>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (w == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su(&tb))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int R = 512 / N > 8 ? 8 : 512 / N;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a0 = su(sm), b0 = su(sm + 64 * 1024);
    t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int r = 0; r < R; ++r) {
        uint64_t ad = SW ? desc_sw32(a0 + r * 4352 + (it % 3) * 32)
                         : desc(a0 + r * 2080 + (it % 3) * 16, 20800, 128);
        uint64_t bd = desc(b0, N * 16, 128);
        uint32_t acc = it > 0;
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                     :: "r"(tb + r * N), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su(&bar)));
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su(&bar)));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
}
template <int N, int SW> void run() {
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k<N, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  k<N, SW><<<148, 128, 100 * 1024>>>(d, iters);
  long long h[148]; cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  const int R = 512 / N > 8 ? 8 : 512 / N;
  printf("SW=%d N=%3d: %.1f cycles per MMA (M=128,K=16), %d MMAs; ideal 128*N/256 = %d; err=%s\n", SW, N,
         (double)h[0] / (iters * R), iters * R, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<16, 0>(); run<32, 0>(); run<64, 0>(); run<96, 0>(); run<128, 0>(); run<256, 0>();
  run<16, 1>(); run<32, 1>(); run<64, 1>(); run<96, 1>(); run<128, 1>(); run<256, 1>();
  return 0;
}
