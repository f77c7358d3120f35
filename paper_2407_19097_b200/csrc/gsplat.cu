// Tile-binned, depth-ordered Gaussian splat blending on the GPU.
//
// Reference: splat_blend_image's CSR binning (pkg/src/nar/_kernels/__init__.py:97-166)
// and the native per-tile blend splat_blend_tiles (_kernels/_native.pyx:80-159).
// The splats arrive depth-sorted (id order = blend order).  Binning builds
// (tile << 32 | splat) pair keys, sorts them with a device radix sort (so each
// tile's list is in ascending splat id, exactly the reference's stable sort),
// and finds every tile's range.  The blend runs one CTA per tile, one thread
// per pixel: batches of the tile's splats are staged in shared memory and
// every thread walks them in order with the reference's f64 arithmetic
// (-fmad=false, same association), skipping pixels whose transmittance fell
// below 1/255; the CTA stops once no pixel of the tile is still active (the
// reference's `done == tile_px` break).  Only exp() differs in the last ulp
// from libm.

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "nar_b200.h"

namespace nar {

constexpr double kMinTransmittance = 1.0 / 255.0;  // _native.pyx:29

__device__ __forceinline__ void splat_tiles(const int32_t* boxes, int64_t s, int ts, int& tx0,
                                            int& tx1, int& ty0, int& ty1) {
  tx0 = boxes[4 * s] / ts;
  tx1 = boxes[4 * s + 1] / ts;
  ty0 = boxes[4 * s + 2] / ts;
  ty1 = boxes[4 * s + 3] / ts;
}

__global__ void splat_count_kernel(const int32_t* __restrict__ boxes, int64_t n, int ts,
                                   int64_t* __restrict__ counts) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  int tx0, tx1, ty0, ty1;
  splat_tiles(boxes, s, ts, tx0, tx1, ty0, ty1);
  counts[s] = (int64_t)(tx1 - tx0 + 1) * (ty1 - ty0 + 1);
}

__global__ void splat_emit_kernel(const int32_t* __restrict__ boxes, int64_t n, int ts,
                                  int tiles_x, const int64_t* __restrict__ offs,
                                  uint64_t* __restrict__ keys) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  int tx0, tx1, ty0, ty1;
  splat_tiles(boxes, s, ts, tx0, tx1, ty0, ty1);
  int64_t o = offs[s];
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx)
      keys[o++] = ((uint64_t)(ty * tiles_x + tx) << 32) | (uint64_t)s;
}

__global__ void tile_range_kernel(const uint64_t* __restrict__ keys, int64_t m,
                                  int64_t* __restrict__ tstart, int64_t* __restrict__ tend) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t t = (uint32_t)(keys[i] >> 32);
  if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) tstart[t] = i;
  if (i == m - 1 || (uint32_t)(keys[i + 1] >> 32) != t) tend[t] = i + 1;
}

struct SplatArgs {
  const double* mu;       // (n, 2)
  const double* inv_abc;  // (n, 3): a, b, c of the inverse 2D covariance
  const int32_t* boxes;   // (n, 4): x0, x1, y0, y1, image-clipped
  const double* color;    // (n, 3)
  const double* opacity;  // (n,)
  const uint64_t* keys;   // sorted (tile << 32 | splat)
  const int64_t* tstart;
  const int64_t* tend;
  int32_t width, height, ts, tiles_x;
  double* rgb;            // (H, W, 3) f64 out
};

constexpr int kSplatBatch = 256;

__global__ void __launch_bounds__(1024) splat_blend_kernel(const SplatArgs a) {
  __shared__ double s_mx[kSplatBatch], s_my[kSplatBatch], s_a[kSplatBatch], s_b[kSplatBatch],
      s_c[kSplatBatch], s_r[kSplatBatch], s_g[kSplatBatch], s_bl[kSplatBatch], s_op[kSplatBatch];
  __shared__ int4 s_box[kSplatBatch];
  const int t = blockIdx.x;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int lx = threadIdx.x % a.ts, ly = threadIdx.x / a.ts;
  const int x = tx * a.ts + lx, y = ty * a.ts + ly;
  const bool inside = x < a.width && y < a.height;
  double r = 0.0, g = 0.0, b = 0.0, tr = 1.0;
  bool active = inside;
  const int64_t lo = a.tstart[t], hi = a.tend[t];
  const int nthreads = blockDim.x;
  for (int64_t base = lo; base < hi; base += kSplatBatch) {
    if (__syncthreads_count(active) == 0) break;  // every pixel of the tile is done
    const int cnt = (int)(hi - base < kSplatBatch ? hi - base : kSplatBatch);
    for (int i = threadIdx.x; i < cnt; i += nthreads) {
      const int64_t s = (int64_t)(a.keys[base + i] & 0xFFFFFFFFull);
      s_mx[i] = a.mu[2 * s];
      s_my[i] = a.mu[2 * s + 1];
      s_a[i] = a.inv_abc[3 * s];
      s_b[i] = a.inv_abc[3 * s + 1];
      s_c[i] = a.inv_abc[3 * s + 2];
      s_r[i] = a.color[3 * s];
      s_g[i] = a.color[3 * s + 1];
      s_bl[i] = a.color[3 * s + 2];
      s_op[i] = a.opacity[s];
      s_box[i] = make_int4(a.boxes[4 * s], a.boxes[4 * s + 1], a.boxes[4 * s + 2],
                           a.boxes[4 * s + 3]);
    }
    __syncthreads();
    if (active) {
      for (int k = 0; k < cnt; ++k) {
        const int4 bx = s_box[k];
        if (x < bx.x || x > bx.y || y < bx.z || y > bx.w) continue;
        // _native.pyx:141-157, same association
        const double dy = (double)y - s_my[k];
        const double dx = (double)x - s_mx[k];
        const double q = s_a[k] * (dx * dx) + (2.0 * s_b[k] * dy) * dx + s_c[k] * (dy * dy);
        const double alpha = s_op[k] * exp(-0.5 * q);
        const double contrib = alpha * tr;
        r += contrib * s_r[k];
        g += contrib * s_g[k];
        b += contrib * s_bl[k];
        tr = tr * (1.0 - alpha);
        if (tr < kMinTransmittance) {
          active = false;
          break;
        }
      }
    }
    __syncthreads();
  }
  if (inside) {
    double* o = a.rgb + ((int64_t)y * a.width + x) * 3;
    o[0] = r;
    o[1] = g;
    o[2] = b;
  }
}

}  // namespace nar

using namespace nar;

extern "C" {

int nar_splat_blend(const double* mu, const double* inv_abc, const int32_t* boxes,
                    const double* color, const double* opacity, int64_t n, int32_t width,
                    int32_t height, int32_t tile_size, double* rgb_out, void* stream) {
  if (width <= 0 || height <= 0 || !rgb_out) return set_error(NAR_ERR_INVALID, "bad image");
  if (tile_size < 1 || tile_size > 32)
    return set_error(NAR_ERR_INVALID, "tile_size must be in [1, 32]");
  if (n < 0 || n >= ((int64_t)1 << 32)) return set_error(NAR_ERR_INVALID, "bad splat count");
  if (n > 0 && (!mu || !inv_abc || !boxes || !color || !opacity))
    return set_error(NAR_ERR_INVALID, "NULL splat array");
  cudaStream_t st = (cudaStream_t)stream;
  nar::keep_pool_memory();
  const int tiles_x = (width + tile_size - 1) / tile_size;
  const int tiles_y = (height + tile_size - 1) / tile_size;
  const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
  if (n_tiles >= ((int64_t)1 << 31)) return set_error(NAR_ERR_INVALID, "too many tiles");
  int64_t *counts = nullptr, *offs = nullptr, *tstart = nullptr, *tend = nullptr;
  uint64_t *keys = nullptr, *keys_sorted = nullptr;
  void* tmp = nullptr;
  int rc = NAR_OK;
  int64_t m = 0;
  auto fail = [&](int code, const char* msg) {
    if (!rc) rc = set_error(code, msg);
  };
  const unsigned gn = (unsigned)((n + 255) / 256);
  if (cudaMallocAsync(reinterpret_cast<void**>(&tstart), (size_t)n_tiles * 8, st) ||
      cudaMallocAsync(reinterpret_cast<void**>(&tend), (size_t)n_tiles * 8, st))
    fail(NAR_ERR_NOMEM, "cudaMallocAsync of tile ranges failed");
  if (!rc) {
    cudaMemsetAsync(tstart, 0, (size_t)n_tiles * 8, st);
    cudaMemsetAsync(tend, 0, (size_t)n_tiles * 8, st);
  }
  if (!rc && n > 0) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&counts), (size_t)n * 8, st) ||
        cudaMallocAsync(reinterpret_cast<void**>(&offs), (size_t)n * 8, st))
      fail(NAR_ERR_NOMEM, "cudaMallocAsync of splat counts failed");
  }
  if (!rc && n > 0) {
    nar::count_launch();
    splat_count_kernel<<<gn, 256, 0, st>>>(boxes, n, tile_size, counts);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, offs, n, st);
    if (cudaMallocAsync(&tmp, tb, st)) fail(NAR_ERR_NOMEM, "scan scratch");
    if (!rc) {
      cub::DeviceScan::ExclusiveSum(tmp, tb, counts, offs, n, st);
      cudaFreeAsync(tmp, st);
      tmp = nullptr;
      int64_t last_off = 0, last_cnt = 0;
      cudaMemcpyAsync(&last_off, offs + n - 1, 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(&last_cnt, counts + n - 1, 8, cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) fail(NAR_ERR_CUDA, "splat binning failed");
      m = last_off + last_cnt;
    }
  }
  if (!rc && m > 0) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&keys), (size_t)m * 8, st) ||
        cudaMallocAsync(reinterpret_cast<void**>(&keys_sorted), (size_t)m * 8, st))
      fail(NAR_ERR_NOMEM, "cudaMallocAsync of tile pairs failed");
    if (!rc) {
      nar::count_launch();
      splat_emit_kernel<<<gn, 256, 0, st>>>(boxes, n, tile_size, tiles_x, offs, keys);
      int end_bit = 32;
      while (end_bit < 64 && ((uint64_t)(n_tiles - 1) >> (end_bit - 32))) ++end_bit;
      size_t tb = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys_sorted, (int64_t)m, 0, end_bit, st);
      if (cudaMallocAsync(&tmp, tb, st)) fail(NAR_ERR_NOMEM, "sort scratch");
      if (!rc) {
        cub::DeviceRadixSort::SortKeys(tmp, tb, keys, keys_sorted, (int64_t)m, 0, end_bit, st);
        nar::count_launch();
        tile_range_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(keys_sorted, m, tstart,
                                                                        tend);
      }
    }
  }
  if (!rc) {
    SplatArgs a;
    a.mu = mu;
    a.inv_abc = inv_abc;
    a.boxes = boxes;
    a.color = color;
    a.opacity = opacity;
    a.keys = keys_sorted;
    a.tstart = tstart;
    a.tend = tend;
    a.width = width;
    a.height = height;
    a.ts = tile_size;
    a.tiles_x = tiles_x;
    a.rgb = rgb_out;
    nar::count_launch();
    splat_blend_kernel<<<(unsigned)n_tiles, tile_size * tile_size, 0, st>>>(a);
  }
  for (void* p : {(void*)counts, (void*)offs, (void*)keys, (void*)keys_sorted, tmp,
                  (void*)tstart, (void*)tend})
    if (p) cudaFreeAsync(p, st);
  if (!rc) rc = check_launch("splat_blend");
  return rc;
}

}  // extern "C"
