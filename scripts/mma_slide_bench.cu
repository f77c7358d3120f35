// Microbenchmark: the conv's sliding MMA pattern (N = 2*Cout; per halo row h and
// kx one tcgen05.mma with the ky blocks stacked along N), A = SWIZZLE_32B halo rows
// of 136 px (4352 B) shifted by kx*32 B, B = no-swizzle K-major [k8][3N][8].
// Prints cycles per MMA back to back (one CTA per SM, no other warps busy).
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
__device__ __forceinline__ uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
// MODE 0: sliding (N<=64), 1: plain 9 taps x R rows, 2: sliding but A not shifted (kx ignored),
// 3: sliding + 5 tcgen05.commit per 30 MMAs (the conv's per-slot signals), 4: sliding + one
// no-swizzle N=256 bias MMA per tile, 5: 3 and 4, 6: sliding with h outer / kx inner
template <int N, int MODE>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar, bar2;
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar2))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (w == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su(&tb))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  constexpr int R = 512 / (2 * N) > 8 ? 8 : 512 / (2 * N);
  long long n_mma = 0;
  if (threadIdx.x == 0) {
    const uint32_t a0 = su(sm), b0 = su(sm + 160 * 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t dcol = tb + (it & 1) * R * N;
      if (MODE == 4 || MODE == 5) {
        mma(dcol, desc(a0, 2048, 128), desc(b0, 4096, 128), idesc(128, 256), 0u);
        ++n_mma;
      }
      if (MODE == 6) {
#pragma unroll 1
        for (int h = 0; h < R + 2; ++h) {
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
            const int kymax = h < 2 ? h : 2;
            const int kymin = h - (R - 1) > 0 ? h - (R - 1) : 0;
            const int nb = kymax - kymin + 1;
            const uint64_t bd = desc(b0 + kx * 3 * N * 32 + (2 - kymax) * N * 16, 3 * N * 16, 128);
            const uint64_t ad = desc_sw32(a0 + h * 4352 + kx * 32);
            mma(dcol + (h - kymax) * N, ad, bd, idesc(128, nb * N), 1u);
            ++n_mma;
          }
        }
      } else if (MODE != 1) {
#pragma unroll 1
        for (int kx = 0; kx < 3; ++kx) {
#pragma unroll
          for (int h = 0; h < R + 2; ++h) {
            const int kymax = h < 2 ? h : 2;
            const int kymin = h - (R - 1) > 0 ? h - (R - 1) : 0;
            const int nb = kymax - kymin + 1;
            const uint64_t bd = desc(b0 + kx * 3 * N * 32 + (2 - kymax) * N * 16, 3 * N * 16, 128);
            const uint64_t ad = desc_sw32(a0 + h * 4352 + (MODE == 2 ? 0 : kx * 32));
            mma(dcol + (h - kymax) * N, ad, bd, idesc(128, nb * N), 1u);
            ++n_mma;
          }
          if ((MODE == 3 || MODE == 5) && kx == 2)
            for (int c = 0; c < 5; ++c)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su(&bar2)));
        }
      } else {
#pragma unroll 1
        for (int tap = 0; tap < 9; ++tap) {
          const int ky = tap / 3, kx = tap % 3;
          const uint64_t bd = desc(b0 + tap * N * 32, N * 16, 128);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            mma(dcol + r * N, desc_sw32(a0 + (r + ky) * 4352 + kx * 32), bd, idesc(128, N), 1u);
            ++n_mma;
          }
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su(&bar)));
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su(&bar)));
    out[2 * blockIdx.x] = clock64() - t0;
    out[2 * blockIdx.x + 1] = n_mma;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
}
template <int N, int MODE> void run(const char* what) {
  long long* d; cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  k<N, MODE><<<148, 128, 210 * 1024>>>(d, 400);
  long long h[296]; cudaMemcpy(h, d, 148 * 16, cudaMemcpyDeviceToHost);
  constexpr int R = 512 / (2 * N) > 8 ? 8 : 512 / (2 * N);
  const double per = (double)h[0] / h[1];
  const double macs = MODE == 1 ? 128.0 * N * 16 : 128.0 * N * 16 * 3 * R / (R + 2);
  printf("%-28s N=%3d R=%d: %6.1f cycles/MMA, %5.0f useful MAC/clk (peak ~4096)  err=%s\n", what, N, R, per,
         macs / per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  run<32, 0>("slide (conv)"); run<32, 2>("slide, A unshifted"); run<32, 1>("plain 9 taps");
  run<32, 3>("slide + 5 commits/tile"); run<32, 4>("slide + bias MMA"); run<32, 5>("slide + both");
  run<32, 6>("slide, h outer"); run<64, 3>("slide + 5 commits/tile"); run<64, 5>("slide + both");
  run<64, 0>("slide (conv)"); run<64, 2>("slide, A unshifted"); run<64, 1>("plain 9 taps");
  run<128, 1>("plain 9 taps"); run<256, 1>("plain 9 taps");
  return 0;
}
