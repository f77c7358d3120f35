// TMA tensor-load throughput for the gated conv's halo boxes (research tool).
// A (H, W, C) bf16 NHWC tensor; every CTA streams (tile, chunk) halo boxes into
// a 3-stage ring and only waits for completion.  Variants:
//   0: two boxes {8 ch, 130 px, R+2 rows}   (current no-swizzle K-major slabs)
//   1: one box  {16 ch, 130 px, R+2 rows}   (32-byte inner dimension)
//   2: one box  {8 ch, 130 px, R+2 rows}    (half the bytes of variant 0)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void tma_kernel(const __grid_constant__ CUtensorMap m, int variant, int tiles_x,
                           int n_tiles, int rows, int chunks) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int S = 3, STAGE = 48 * 1024;
  __shared__ uint64_t bar[S];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t box = variant == 0 ? 2u * 8 * 130 * 2 * rows
                                    : (variant == 1 ? 16u * 130 * 2 * rows : 8u * 130 * 2 * rows);
  int it = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int y0 = (tile / tiles_x) * (rows - 2), x0 = (tile % tiles_x) * 128;
    for (int q = 0; q < chunks; ++q, ++it) {
      const int s = it % S;
      if (it >= S) {  // wait for the previous use of this stage
        const uint32_t ph = (uint32_t)((it / S) - 1) & 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra W;\n\t}" ::"r"(su32(&bar[s])),
            "r"(ph));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])),
                   "r"(box));
      uint8_t* dst = smem + s * STAGE;
      const int c = 16 * q;
      if (variant == 1) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst)),
            "l"(&m), "r"(c), "r"(x0 - 1), "r"(y0 - 1), "r"(su32(&bar[s]))
            : "memory");
      } else {
        for (int k = 0; k < (variant == 0 ? 2 : 1); ++k)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst + k * 24 * 1024)),
              "l"(&m), "r"(c + 8 * k), "r"(x0 - 1), "r"(y0 - 1), "r"(su32(&bar[s]))
              : "memory");
      }
    }
  }
  for (int j = it - S; j < it; ++j) {
    if (j < 0) continue;
    const int s = j % S;
    const uint32_t ph = (uint32_t)(j / S) & 1u;
    asm volatile(
        "{\n\t.reg .pred p;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W2;\n\t}" ::"r"(su32(&bar[s])),
        "r"(ph));
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int H = 1088, W = 1920;
  for (int C : {16, 32, 64}) {
    void* buf;
    cudaMalloc(&buf, (size_t)H * W * C * 2);
    cudaMemset(buf, 0, (size_t)H * W * C * 2);
    for (int rows : {3, 4, 6, 10}) {
      for (int variant = 0; variant < 3; ++variant) {
        CUtensorMap m;
        cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H};
        cuuint64_t strides[2] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * W};
        cuuint32_t boxd[3] = {(cuuint32_t)(variant == 1 ? 16 : 8), 130, (cuuint32_t)rows};
        cuuint32_t es[3] = {1, 1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, boxd, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
          printf("encode failed\n");
          return 1;
        }
        const int tiles_x = (W + 127) / 128, tiles_y = (H + rows - 3) / (rows - 2);
        const int n_tiles = tiles_x * tiles_y, chunks = C / 16;
        cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 48 * 1024);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(e0);
          tma_kernel<<<148, 32, 3 * 48 * 1024>>>(m, variant, tiles_x, n_tiles, rows, chunks);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double boxes = (double)n_tiles * chunks;
        const double bytes = boxes * (variant == 2 ? 8 : 16) * 130 * 2 * rows;
        printf("C=%2d rows=%2d variant=%d  %.1f us  %.0f GB/s  %.2f ns per 16B-row per SM  err=%s\n",
               C, rows, variant, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
               ms * 1e6 / (bytes / 16 / 148), cudaGetErrorString(cudaGetLastError()));
      }
    }
    cudaFree(buf);
  }
  return 0;
}
