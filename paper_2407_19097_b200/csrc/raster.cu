// raster.cu -- MSR render (project + cull + packed-key early-z) and resolve
// kernels for sm_100a, plus their C-ABI entry points (include/nar_b200.h).
//
// Render follows pkg/src/nar/_kernels/_native.pyx:56-77 operation for
// operation in IEEE f64 with explicit round-to-nearest intrinsics (no FMA
// contraction; the reference builds with -ffp-contract=off, setup.py:23-25),
// so the packed keys are bit-identical to the CPU oracle.  Non-finite
// projections are culled as in python_impl.py:43-47.
//
// Data layout in HBM:
//   positions : f32 AoS (n, 3), 12 B/point, streamed once per frame by TMA
//               bulk copies (cp.async.bulk) into a 4-stage smem ring;
//   keybuf    : u64 (H*W,) row-major, L2-resident (16.6 MB at 1080p);
//               key = f32bits(depth) << 32 | (index & 0xFFFFFFFF).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>

#include "nar_b200.h"
#include "common.cuh"

namespace nar {

// ----------------------------------------------------------------------------
// camera in kernel-parameter form
// ----------------------------------------------------------------------------
struct DevCam {
  double r[9];
  double c[3];
  double f, cx, cy, nr, fr;
  double wd, hd;
  int32_t w, h;
};

static DevCam make_devcam(const nar_camera& cam) {
  DevCam k;
  for (int i = 0; i < 9; ++i) k.r[i] = cam.R[i];
  for (int i = 0; i < 3; ++i) k.c[i] = cam.campos[i];
  k.f = cam.f;
  k.cx = cam.cx;
  k.cy = cam.cy;
  k.nr = cam.near_;
  k.fr = cam.far_;
  k.wd = (double)cam.width;
  k.hd = (double)cam.height;
  k.w = cam.width;
  k.h = cam.height;
  return k;
}

// Projection of one point, _native.pyx:58-73 in the same f64 op order:
//   w = (double)p - c;  uz = (w0*r20 + w1*r21) + w2*r22  (ux, uy alike)
//   px = floor((cx + f*(ux/uz)) + 0.5)
// Returns false for culled points; otherwise the pixel and f32 depth bits.
__device__ __forceinline__ bool project_point(float x, float y, float z, const DevCam& k,
                                              uint32_t& pix, uint32_t& dbits) {
  const double w0 = __dsub_rn((double)x, k.c[0]);
  const double w1 = __dsub_rn((double)y, k.c[1]);
  const double w2 = __dsub_rn((double)z, k.c[2]);
  const double uz =
      __dadd_rn(__dadd_rn(__dmul_rn(w0, k.r[6]), __dmul_rn(w1, k.r[7])), __dmul_rn(w2, k.r[8]));
  // python_impl.py:43 ok = (uz > near) & (uz < far): NaN is culled.
  if (!(uz > k.nr && uz < k.fr)) return false;
  const double ux =
      __dadd_rn(__dadd_rn(__dmul_rn(w0, k.r[0]), __dmul_rn(w1, k.r[1])), __dmul_rn(w2, k.r[2]));
  const double uy =
      __dadd_rn(__dadd_rn(__dmul_rn(w0, k.r[3]), __dmul_rn(w1, k.r[4])), __dmul_rn(w2, k.r[5]));
  const double px = floor(__dadd_rn(__dadd_rn(k.cx, __dmul_rn(k.f, __ddiv_rn(ux, uz))), 0.5));
  const double py = floor(__dadd_rn(__dadd_rn(k.cy, __dmul_rn(k.f, __ddiv_rn(uy, uz))), 0.5));
  if (!(px >= 0.0 && px < k.wd && py >= 0.0 && py < k.hd)) return false;
  pix = (uint32_t)(int32_t)py * (uint32_t)k.w + (uint32_t)(int32_t)px;
  dbits = __float_as_uint(__double2float_rn(uz));
  return true;
}

template <bool kSigned>
__device__ __forceinline__ void fold_key(uint64_t* keybuf, uint32_t pix, uint64_t key) {
  if (kSigned) {
    const long long k = (long long)(key ^ NAR_SIGN_FLIP);
    long long* p = reinterpret_cast<long long*>(keybuf) + pix;
    if (k < (long long)__ldcg(reinterpret_cast<const unsigned long long*>(p))) atomicMin(p, k);
  } else {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(keybuf) + pix;
    if (key < __ldcg(p)) atomicMin(p, (unsigned long long)key);
  }
}

// ----------------------------------------------------------------------------
// render: persistent CTAs, TMA bulk-copy ring of point tiles in smem
// ----------------------------------------------------------------------------
constexpr int kRenderThreads = 256;
constexpr int kPtsPerThread = 4;
constexpr int kTilePts = kRenderThreads * kPtsPerThread;  // 1024 points
constexpr int kTileBytes = kTilePts * 12;                 // 12 KB
constexpr int kStages = 4;
constexpr int kRenderSmem = kStages * kTileBytes + 64;

template <bool kSigned>
__global__ void __launch_bounds__(kRenderThreads, 4)
    render_tma_kernel(uint64_t* __restrict__ keybuf, const float* __restrict__ pos,
                      int64_t n_tiles, uint64_t base_index, const DevCam cam) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* ring = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kTileBytes);
  const int tid = threadIdx.x;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t first = blockIdx.x;
  const int64_t stride = gridDim.x;
  // prologue: fill the ring
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int64_t t = first + (int64_t)s * stride;
      if (t < n_tiles) {
        mbar_expect_tx(&full[s], kTileBytes);
        bulk_g2s(ring + s * (kTilePts * 3), pos + t * (int64_t)(kTilePts * 3), kTileBytes,
                 &full[s]);
      }
    }
  }

  int it = 0;
  for (int64_t t = first; t < n_tiles; t += stride, ++it) {
    const int s = it % kStages;
    const uint32_t phase = (uint32_t)(it / kStages) & 1u;
    mbar_wait(&full[s], phase);
    const float* tile = ring + s * (kTilePts * 3);
    const uint64_t tile_base = base_index + (uint64_t)t * kTilePts;

    uint32_t pix[kPtsPerThread];
    uint64_t key[kPtsPerThread];
    bool ok[kPtsPerThread];
#pragma unroll
    for (int j = 0; j < kPtsPerThread; ++j) {
      const int p = j * kRenderThreads + tid;
      uint32_t db = 0;
      ok[j] = project_point(tile[3 * p], tile[3 * p + 1], tile[3 * p + 2], cam, pix[j], db);
      key[j] = ((uint64_t)db << 32) | ((tile_base + (uint64_t)p) & 0xFFFFFFFFull);
    }
    __syncthreads();  // everyone is done reading stage s
    if (tid == 0) {
      const int64_t nt = t + (int64_t)kStages * stride;
      if (nt < n_tiles) {
        mbar_expect_tx(&full[s], kTileBytes);
        bulk_g2s(ring + s * (kTilePts * 3), pos + nt * (int64_t)(kTilePts * 3), kTileBytes,
                 &full[s]);
      }
    }
#pragma unroll
    for (int j = 0; j < kPtsPerThread; ++j)
      if (ok[j]) fold_key<kSigned>(keybuf, pix[j], key[j]);
  }
}

// Plain-load variant for unaligned inputs and the < 1 tile tail.
template <bool kSigned>
__global__ void __launch_bounds__(256)
    render_simple_kernel(uint64_t* __restrict__ keybuf, const float* __restrict__ pos,
                         int64_t n, uint64_t base_index, const DevCam cam) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t pix, db;
    if (project_point(__ldg(pos + 3 * i), __ldg(pos + 3 * i + 1), __ldg(pos + 3 * i + 2), cam,
                      pix, db)) {
      const uint64_t key = ((uint64_t)db << 32) | ((base_index + (uint64_t)i) & 0xFFFFFFFFull);
      fold_key<kSigned>(keybuf, pix, key);
    }
  }
}

__global__ void fill_u64_kernel(uint64_t* __restrict__ p, int64_t n, uint64_t v) {
  const int64_t n2 = n / 2;
  ulonglong2 vv = make_ulonglong2(v, v);
  ulonglong2* p2 = reinterpret_cast<ulonglong2*>(p);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x)
    p2[i] = vv;
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[n - 1] = v;
}

// ----------------------------------------------------------------------------
// resolve: one thread per output pixel (rasterizer.py:140-178)
// ----------------------------------------------------------------------------
struct ResolveParams {
  nar_selection sel;
  nar_segment seg[NAR_MAX_SEGMENTS];
  int32_t nseg;
  DevCam cam;
  float near_f;
  float* data;
  uint8_t* coverage;
  int64_t* index_plane;
  float* depth;
  int32_t C, data_h, data_w;
  int32_t owner_only, clear;
};

__device__ __forceinline__ float stream_value(const void* base, int32_t fmt, int32_t arity,
                                              int64_t row, int32_t col) {
  // rasterizer.py:116-120 _stream_as_float: u8 -> f32(u8) / 255 (IEEE f32 divide)
  if (fmt == NAR_FMT_U8) {
    const uint8_t v = __ldg(static_cast<const uint8_t*>(base) + row * arity + col);
    return __fdiv_rn((float)v, 255.0f);
  }
  return __ldg(static_cast<const float*>(base) + row * arity + col);
}

template <bool kSigned>
__global__ void __launch_bounds__(256)
    resolve_kernel(uint64_t* __restrict__ keybuf, const ResolveParams P) {
  const int32_t W = P.cam.w, H = P.cam.h;
  const int64_t npix_out = (int64_t)P.data_h * P.data_w;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= npix_out) return;
  const int32_t y = (int32_t)(gid / P.data_w);
  const int32_t x = (int32_t)(gid - (int64_t)y * P.data_w);
  float ch[NAR_MAX_CHANNELS];
#pragma unroll
  for (int c = 0; c < NAR_MAX_CHANNELS; ++c) ch[c] = 0.0f;

  if (y < H && x < W) {
    const int64_t pix = (int64_t)y * W + x;
    uint64_t key = keybuf[pix];
    if (kSigned) key ^= NAR_SIGN_FLIP;
    if (P.clear) keybuf[pix] = kSigned ? (NAR_EMPTY_KEY ^ NAR_SIGN_FLIP) : NAR_EMPTY_KEY;
    const bool covered = key != NAR_EMPTY_KEY;
    const int64_t idx = covered ? (int64_t)(key & 0xFFFFFFFFull) : -1;
    const float dep = covered ? __uint_as_float((uint32_t)(key >> 32)) : 0.0f;
    if (P.coverage) P.coverage[pix] = covered ? 1 : 0;
    if (P.index_plane) P.index_plane[pix] = idx;
    if (P.depth) P.depth[pix] = dep;

    int s = -1;
    if (covered) {
      for (int k = 0; k < P.nseg; ++k)
        if (idx >= P.seg[k].begin && idx < P.seg[k].begin + P.seg[k].count) s = k;
    }
    const bool owner = s >= 0;
    const nar_selection& sel = P.sel;
    int col = 0;
    if (owner) {
      const nar_segment& sg = P.seg[s];
      const int64_t row = idx - sg.begin;
      if (sel.rgb) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
          ch[c] = stream_value(sg.rgb, sel.rgb_format, sel.rgb_arity, row,
                               sel.rgb_arity == 1 ? 0 : c);
        col += 3;
      }
      if (sel.depth) {
        // rasterizer.py:156-157 f32(near) / depth, clipped to [0, 1]
        float d = __fdiv_rn(P.near_f, dep);
        d = fminf(fmaxf(d, 0.0f), 1.0f);
        ch[col++] = d;
      }
      if (sel.vel2d || sel.vel3d) {
        double v[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
          v[c] = (double)stream_value(sg.velocity, sel.vel_format, sel.vel_arity, row, c);
        const double scale = sel.velocity_scale;
        if (sel.vel2d) {
          // velocity.py:26-48 + camera.py:154-166, f64 (BLAS order: <= 1 f32 ulp)
          const DevCam& k = P.cam;
          const double w0 = (double)__ldg(sg.positions + 3 * row) - k.c[0];
          const double w1 = (double)__ldg(sg.positions + 3 * row + 1) - k.c[1];
          const double w2 = (double)__ldg(sg.positions + 3 * row + 2) - k.c[2];
          const double ux = w0 * k.r[0] + w1 * k.r[1] + w2 * k.r[2];
          const double uy = w0 * k.r[3] + w1 * k.r[4] + w2 * k.r[5];
          const double uz = w0 * k.r[6] + w1 * k.r[7] + w2 * k.r[8];
          const double sc = k.f / (uz * uz);
          double vp0 = 0.0, vp1 = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double j0 = (uz * k.r[j] - ux * k.r[6 + j]) * sc;
            const double j1 = (uz * k.r[3 + j] - uy * k.r[6 + j]) * sc;
            vp0 += j0 * v[j];
            vp1 += j1 * v[j];
          }
          const double mag = hypot(vp0, vp1);
          const double theta = mag < 1e-9 ? 0.0 : atan2(-vp1, vp0);
          ch[col++] = (float)(vp0 / scale);
          ch[col++] = (float)(vp1 / scale);
          ch[col++] = (float)theta;
          ch[col++] = (float)(mag / scale);
        }
        if (sel.vel3d) {
          // velocity.py:17-23
          const double nrm = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
          ch[col++] = (float)(v[0] / scale);
          ch[col++] = (float)(v[1] / scale);
          ch[col++] = (float)(v[2] / scale);
          ch[col++] = (float)(nrm / scale);
        }
      }
      for (int q = 0; q < sel.n_scalars; ++q) {
        const int32_t ar = sel.scalar_arity[q];
        for (int c = 0; c < ar && col < NAR_MAX_CHANNELS; ++c)
          ch[col++] = stream_value(sg.scalars[q], sel.scalar_format[q], ar, row, c);
      }
      if (sel.coverage_channel && col < NAR_MAX_CHANNELS) ch[col++] = 1.0f;
    } else if (covered && !P.owner_only) {
      // winner outside every segment: only possible for inconsistent inputs;
      // keep zeros (the host validated the index ranges).
    }
  }
  if (P.data) {
    float* dst = P.data + gid * P.C;
    // channel count is small (<= 16); vectorise when 4-aligned
    if ((P.C & 3) == 0) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int c = 0; c < NAR_MAX_CHANNELS / 4; ++c)
        if (4 * c < P.C) d4[c] = make_float4(ch[4 * c], ch[4 * c + 1], ch[4 * c + 2], ch[4 * c + 3]);
    } else {
#pragma unroll
      for (int c = 0; c < NAR_MAX_CHANNELS; ++c)
        if (c < P.C) dst[c] = ch[c];
    }
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
static int g_num_sms = 0;
static int g_render_blocks_per_sm = 0;
static std::once_flag g_init_once;

static int device_init() {
  int err = 0;
  std::call_once(g_init_once, [&]() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { err = 1; return; }
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(render_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRenderSmem);
    cudaFuncSetAttribute(render_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRenderSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_render_blocks_per_sm,
                                                  render_tma_kernel<false>, kRenderThreads,
                                                  kRenderSmem);
    if (g_render_blocks_per_sm < 1) g_render_blocks_per_sm = 1;
  });
  if (err || g_num_sms == 0) return set_error(NAR_ERR_CUDA, "no CUDA device");
  return NAR_OK;
}

static int launch_render(uint64_t* keybuf, const float* pos, int64_t n, uint64_t base,
                         const DevCam& cam, bool sgn, cudaStream_t st) {
  if (n <= 0) return NAR_OK;
  int rc = device_init();
  if (rc) return rc;
  int64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(pos) & 15) == 0) {
    const int64_t n_tiles = n / kTilePts;
    if (n_tiles > 0) {
      const int64_t cap = (int64_t)g_num_sms * g_render_blocks_per_sm;
      const int grid = (int)(n_tiles < cap ? n_tiles : cap);
      if (sgn)
        render_tma_kernel<true><<<grid, kRenderThreads, kRenderSmem, st>>>(keybuf, pos, n_tiles,
                                                                           base, cam);
      else
        render_tma_kernel<false><<<grid, kRenderThreads, kRenderSmem, st>>>(keybuf, pos, n_tiles,
                                                                            base, cam);
      done = n_tiles * kTilePts;
    }
  }
  const int64_t rest = n - done;
  if (rest > 0) {
    int64_t blocks = (rest + 255) / 256;
    const int64_t cap = (int64_t)(g_num_sms > 0 ? g_num_sms : 148) * 8;
    if (blocks > cap) blocks = cap;
    if (sgn)
      render_simple_kernel<true><<<(int)blocks, 256, 0, st>>>(keybuf, pos + 3 * done, rest,
                                                             base + (uint64_t)done, cam);
    else
      render_simple_kernel<false><<<(int)blocks, 256, 0, st>>>(keybuf, pos + 3 * done, rest,
                                                              base + (uint64_t)done, cam);
  }
  return check_launch("render");
}

static int validate_camera(const nar_camera* cam) {
  if (!cam) return set_error(NAR_ERR_INVALID, "camera is NULL");
  if (cam->width <= 0 || cam->height <= 0)
    return set_error(NAR_ERR_INVALID, "width and height must be positive");
  if ((int64_t)cam->width * cam->height >= (int64_t)1 << 32)
    return set_error(NAR_ERR_INVALID, "framebuffer exceeds 2^32 pixels");
  return NAR_OK;
}

static int render_host_impl(uint64_t* keybuf_dev, const float* pos_host, int64_t n,
                            uint64_t base, const DevCam& cam, bool sgn, cudaStream_t st) {
  if (n <= 0) return NAR_OK;
  const int64_t kChunk = (int64_t)1 << 23;  // 8 Mi points = 96 MiB per buffer
  const int64_t chunk = n < kChunk ? ((n + kTilePts - 1) / kTilePts) * kTilePts : kChunk;
  const int nbuf = n > chunk ? 2 : 1;
  float* dbuf[2] = {nullptr, nullptr};
  cudaStream_t cp = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  int rc = NAR_OK;
  for (int b = 0; b < nbuf; ++b) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&dbuf[b]), (size_t)chunk * 12, st) != cudaSuccess) {
      rc = set_error(NAR_ERR_NOMEM, "cudaMallocAsync of point chunk failed");
      break;
    }
  }
  if (!rc && cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking) != cudaSuccess)
    rc = set_error(NAR_ERR_CUDA, "stream creation failed");
  for (int b = 0; b < 2 && !rc; ++b) {
    cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
  }
  if (!rc) {
    // the chunk buffers were allocated on `st`; make the copy stream wait
    cudaEventRecord(done[0], st);
    cudaStreamWaitEvent(cp, done[0], 0);
    for (int64_t off = 0, k = 0; off < n && !rc; off += chunk, ++k) {
      const int b = (int)(k % nbuf);
      const int64_t cnt = (n - off) < chunk ? (n - off) : chunk;
      if (k >= nbuf) cudaStreamWaitEvent(cp, done[b], 0);
      if (cudaMemcpyAsync(dbuf[b], pos_host + 3 * off, (size_t)cnt * 12, cudaMemcpyHostToDevice,
                          cp) != cudaSuccess) {
        rc = set_error(NAR_ERR_CUDA, "H2D copy of points failed");
        break;
      }
      cudaEventRecord(copied[b], cp);
      cudaStreamWaitEvent(st, copied[b], 0);
      rc = launch_render(keybuf_dev, dbuf[b], cnt, base + (uint64_t)off, cam, sgn, st);
      cudaEventRecord(done[b], st);
    }
  }
  for (int b = 0; b < nbuf; ++b)
    if (dbuf[b]) cudaFreeAsync(dbuf[b], st);
  for (int b = 0; b < 2; ++b) {
    if (copied[b]) cudaEventDestroy(copied[b]);
    if (done[b]) cudaEventDestroy(done[b]);
  }
  if (cp) cudaStreamDestroy(cp);
  if (!rc) rc = check_launch("render_host");
  return rc;
}

}  // namespace nar

using namespace nar;

extern "C" {

int nar_keybuf_fill(uint64_t* keybuf_dev, int64_t npix, uint64_t value, void* stream) {
  if (npix < 0 || (npix > 0 && !keybuf_dev)) return set_error(NAR_ERR_INVALID, "bad keybuf");
  if (npix == 0) return NAR_OK;
  int rc = device_init();
  if (rc) return rc;
  int64_t blocks = (npix / 2 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > (int64_t)g_num_sms * 16) blocks = (int64_t)g_num_sms * 16;
  fill_u64_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(keybuf_dev, npix, value);
  return check_launch("keybuf_fill");
}

int nar_render(uint64_t* keybuf_dev, const float* positions_dev, int64_t n, uint64_t base_index,
               const nar_camera* cam, int32_t key_domain, void* stream) {
  int rc = validate_camera(cam);
  if (rc) return rc;
  if (n < 0) return set_error(NAR_ERR_INVALID, "negative point count");
  if (n > 0 && (!keybuf_dev || !positions_dev)) return set_error(NAR_ERR_INVALID, "NULL buffer");
  return launch_render(keybuf_dev, positions_dev, n, base_index, make_devcam(*cam),
                       key_domain == NAR_KEYS_SIGNED, (cudaStream_t)stream);
}

int nar_render_host(uint64_t* keybuf_dev, const float* positions_host, int64_t n,
                    uint64_t base_index, const nar_camera* cam, int32_t key_domain,
                    void* stream) {
  int rc = validate_camera(cam);
  if (rc) return rc;
  if (n < 0) return set_error(NAR_ERR_INVALID, "negative point count");
  if (n > 0 && (!keybuf_dev || !positions_host)) return set_error(NAR_ERR_INVALID, "NULL buffer");
  rc = device_init();
  if (rc) return rc;
  return render_host_impl(keybuf_dev, positions_host, n, base_index, make_devcam(*cam),
                          key_domain == NAR_KEYS_SIGNED, (cudaStream_t)stream);
}

int nar_zbuffer_accumulate(uint64_t* keybuf, const float* positions, int64_t n,
                           uint64_t base_index, const double* R, const double* campos, double f,
                           double cx, double cy, double near_, double far_, int32_t width,
                           int32_t height) {
  if (!keybuf || !R || !campos) return set_error(NAR_ERR_INVALID, "NULL argument");
  nar_camera cam;
  memcpy(cam.R, R, sizeof(cam.R));
  memcpy(cam.campos, campos, sizeof(cam.campos));
  cam.f = f;
  cam.cx = cx;
  cam.cy = cy;
  cam.near_ = near_;
  cam.far_ = far_;
  cam.width = width;
  cam.height = height;
  int rc = validate_camera(&cam);
  if (rc) return rc;
  if (n < 0 || (n > 0 && !positions)) return set_error(NAR_ERR_INVALID, "bad positions");
  rc = device_init();
  if (rc) return rc;
  const int64_t npix = (int64_t)width * height;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
    return set_error(NAR_ERR_CUDA, "stream creation failed");
  uint64_t* dkey = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&dkey), (size_t)npix * 8, st) != cudaSuccess) {
    cudaStreamDestroy(st);
    return set_error(NAR_ERR_NOMEM, "cudaMallocAsync of keybuf failed");
  }
  // keybuf is folded in place: start from the caller's contents
  if (cudaMemcpyAsync(dkey, keybuf, (size_t)npix * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
    rc = set_error(NAR_ERR_CUDA, "H2D copy of keybuf failed");
  if (!rc) rc = render_host_impl(dkey, positions, n, base_index, make_devcam(cam), false, st);
  if (!rc && cudaMemcpyAsync(keybuf, dkey, (size_t)npix * 8, cudaMemcpyDeviceToHost, st) !=
                 cudaSuccess)
    rc = set_error(NAR_ERR_CUDA, "D2H copy of keybuf failed");
  cudaFreeAsync(dkey, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !rc)
    rc = set_error(NAR_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  cudaStreamDestroy(st);
  return rc;
}

int nar_resolve(uint64_t* keybuf_dev, const nar_camera* cam, int32_t key_domain,
                const nar_selection* sel, const nar_segment* segments, int32_t n_segments,
                const nar_resolve_out* out, void* stream) {
  int rc = validate_camera(cam);
  if (rc) return rc;
  if (!keybuf_dev || !sel || !out) return set_error(NAR_ERR_INVALID, "NULL argument");
  if (n_segments < 0 || n_segments > NAR_MAX_SEGMENTS || (n_segments > 0 && !segments))
    return set_error(NAR_ERR_INVALID, "bad segment table");
  if (sel->n_scalars < 0 || sel->n_scalars > NAR_MAX_SCALARS)
    return set_error(NAR_ERR_CONFIG, "too many scalar streams");
  int C = (sel->rgb ? 3 : 0) + (sel->depth ? 1 : 0) + (sel->vel2d ? 4 : 0) +
          (sel->vel3d ? 4 : 0) + (sel->coverage_channel ? 1 : 0);
  for (int q = 0; q < sel->n_scalars; ++q) C += sel->scalar_arity[q];
  if (C > NAR_MAX_CHANNELS) return set_error(NAR_ERR_CONFIG, "more than 16 channels");
  if (sel->rgb && !(sel->rgb_arity == 1 || sel->rgb_arity >= 3))
    return set_error(NAR_ERR_CONFIG, "rgb stream needs arity 1 or >= 3");
  if ((sel->vel2d || sel->vel3d) && sel->vel_arity < 3)
    return set_error(NAR_ERR_CONFIG, "velocity stream needs arity >= 3");
  if ((sel->vel2d || sel->vel3d) && sel->velocity_scale == 0.0)
    return set_error(NAR_ERR_CONFIG, "velocity_scale must be non-zero");
  rc = device_init();
  if (rc) return rc;
  ResolveParams P;
  memset(&P, 0, sizeof(P));
  P.sel = *sel;
  for (int k = 0; k < n_segments; ++k) {
    P.seg[k] = segments[k];
    if (sel->rgb && !segments[k].rgb && segments[k].count > 0)
      return set_error(NAR_ERR_CONFIG, "segment lacks the rgb stream");
    if ((sel->vel2d || sel->vel3d) && !segments[k].velocity && segments[k].count > 0)
      return set_error(NAR_ERR_CONFIG, "segment lacks the velocity stream");
    if (sel->vel2d && !segments[k].positions && segments[k].count > 0)
      return set_error(NAR_ERR_CONFIG, "vel2d needs segment positions");
    for (int q = 0; q < sel->n_scalars; ++q)
      if (!segments[k].scalars[q] && segments[k].count > 0)
        return set_error(NAR_ERR_CONFIG, "segment lacks a scalar stream");
  }
  P.nseg = n_segments;
  P.cam = make_devcam(*cam);
  P.near_f = (float)cam->near_;
  P.data = out->data;
  P.coverage = out->coverage;
  P.index_plane = out->index_plane;
  P.depth = out->depth;
  P.C = C;
  P.data_h = out->data_h > 0 ? out->data_h : cam->height;
  P.data_w = out->data_w > 0 ? out->data_w : cam->width;
  if (P.data_h < cam->height || P.data_w < cam->width)
    return set_error(NAR_ERR_INVALID, "padded data extent smaller than the image");
  P.owner_only = out->owner_only;
  P.clear = out->clear_keybuf;
  const int64_t n_out = (int64_t)P.data_h * P.data_w;
  const int64_t blocks = (n_out + 255) / 256;
  if (key_domain == NAR_KEYS_SIGNED)
    resolve_kernel<true><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(keybuf_dev, P);
  else
    resolve_kernel<false><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(keybuf_dev, P);
  return check_launch("resolve");
}

}  // extern "C"
