// morton.cu -- 63-bit Morton (z-order) keys of a device point cloud
// (pkg/src/nar/geometry/morton.py:9-46), bit-identical to the reference:
//   scaled = ((double)p - lo) / extent * 2^21   (IEEE f64, same op order)
//   q = clip(floor(scaled), 0, 2^21 - 1); key = spread(qx) | spread(qy)<<1 | spread(qz)<<2
// The reorder itself is a stable sort of the keys (host side, torch.sort).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "nar_b200.h"

namespace nar {

__device__ __forceinline__ uint64_t spread21(uint64_t x) {
  x &= 0x1FFFFFull;
  x = (x | (x << 32)) & 0x1F00000000FFFFull;
  x = (x | (x << 16)) & 0x1F0000FF0000FFull;
  x = (x | (x << 8)) & 0x100F00F00F00F00Full;
  x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

struct MortonBox {
  double lo[3], ext[3];
};

__device__ __forceinline__ uint64_t quant21(float p, double lo, double ext) {
  const double scaled = __dmul_rn(__ddiv_rn(__dsub_rn((double)p, lo), ext), 2097152.0);
  double f = floor(scaled);
  // np.floor(...).astype(int64) then clip to [0, 2^21 - 1]: NaN and |f| >= 2^63 convert
  // to INT64_MIN on x86 and clip to 0; other negatives clip to 0, large values to 2^21 - 1
  if (!(f >= 0.0) || f >= 9223372036854775808.0) f = 0.0;
  else if (f > 2097151.0) f = 2097151.0;
  return (uint64_t)f;
}

__global__ void morton_kernel(const float* __restrict__ pos, int64_t n, const MortonBox box,
                              uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t qx = quant21(pos[3 * i], box.lo[0], box.ext[0]);
    const uint64_t qy = quant21(pos[3 * i + 1], box.lo[1], box.ext[1]);
    const uint64_t qz = quant21(pos[3 * i + 2], box.lo[2], box.ext[2]);
    keys[i] = spread21(qx) | (spread21(qy) << 1) | (spread21(qz) << 2);
  }
}

}  // namespace nar

extern "C" int nar_morton_keys(const float* positions_dev, int64_t n, const double* lo,
                               const double* hi, uint64_t* keys_dev, void* stream) {
  if (n < 0 || !lo || !hi || (n > 0 && (!positions_dev || !keys_dev)))
    return nar::set_error(NAR_ERR_INVALID, "bad morton arguments");
  if (n == 0) return NAR_OK;
  nar::MortonBox b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = lo[a];
    b.ext[a] = hi[a] > lo[a] ? hi[a] - lo[a] : 1.0;  // morton.py:25
  }
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  nar::count_launch();
  nar::morton_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(positions_dev, n, b,
                                                                        keys_dev);
  return nar::check_launch("morton_keys");
}
