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
//               bulk copies (cp.async.bulk, L2 evict-first) into per-warp
//               smem rings (3 x 1.5 KB units, or 6 x 768 B chunks);
//   keybuf    : u64 (H*W,) row-major, L2-resident (16.6 MB at 1080p);
//               key = f32bits(depth) << 32 | (index & 0xFFFFFFFF).
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>
#include <unordered_map>

#include "nar_b200.h"
#include "common.cuh"

namespace nar {

// ----------------------------------------------------------------------------
// camera in kernel-parameter form
// ----------------------------------------------------------------------------
struct DevCam {
  double r[9];
  double c[3];
  double nc[3];  // -c: p - c evaluated as p + (-c) (bit-identical) with a constant-bank operand
  double f, cx, cy, nr, fr;
  double wd, hd;
  int32_t w, h;
  // certified fast pixel path (see project_fast)
  double cxh, cyh;       // cx + 0.5, cy + 0.5
  double fr_[6];         // f * R rows 0, 1
  int32_t fast;          // camera within the bound's domain
  // f32 occlusion pre-test (see pretest): camera position as f32 hi + lo,
  // rotation row 2, f * rows 0/1, principal point; `pre` = bounds hold
  float chi[3];          // camera position rounded to f32
  float r2f[3], uz0;     // uz = R2 . (p - chi) + uz0      (uz0 = -R2 . (c - chi))
  float fxr[3], fx0;     // T' uz = (f R0 + cx R2) . (p - chi) + fx0
  float fyr[3], fy0;
  int32_t pre;
};

static DevCam make_devcam(const nar_camera& cam) {
  DevCam k;
  for (int i = 0; i < 9; ++i) k.r[i] = cam.R[i];
  for (int i = 0; i < 3; ++i) k.c[i] = cam.campos[i];
  for (int i = 0; i < 3; ++i) k.nc[i] = -cam.campos[i];
  k.f = cam.f;
  k.cx = cam.cx;
  k.cy = cam.cy;
  k.nr = cam.near_;
  k.fr = cam.far_;
  k.wd = (double)cam.width;
  k.hd = (double)cam.height;
  k.w = cam.width;
  k.h = cam.height;
  for (int i = 0; i < 6; ++i) k.fr_[i] = cam.f * cam.R[i];
  k.cxh = cam.cx + 0.5;
  k.cyh = cam.cy + 0.5;
  k.fast = (fabs(cam.f) <= 1048576.0 && fabs(cam.cx) < 32768.0 && fabs(cam.cy) < 32768.0 &&
            cam.width <= 65536 && cam.height <= 65536)
               ? 1
               : 0;
  double uz0 = 0.0, fx0 = 0.0, fy0 = 0.0;
  for (int i = 0; i < 3; ++i) {
    k.chi[i] = (float)cam.campos[i];
    const double lo = cam.campos[i] - (double)k.chi[i];
    const double fxr = cam.f * cam.R[i] + cam.cx * cam.R[6 + i];
    const double fyr = cam.f * cam.R[3 + i] + cam.cy * cam.R[6 + i];
    k.r2f[i] = (float)cam.R[6 + i];
    k.fxr[i] = (float)fxr;
    k.fyr[i] = (float)fyr;
    uz0 -= cam.R[6 + i] * lo;
    fx0 -= fxr * lo;
    fy0 -= fyr * lo;
  }
  k.uz0 = (float)uz0;
  k.fx0 = (float)fx0;
  k.fy0 = (float)fy0;
  // pretest error budget: |T'32 - T'| < 0.5 px and relative uz32 error
  // < 2^-14 for every point whose pixel is within 1 of the image (|w|/uz <= K)
  const double af = fabs(cam.f);
  const double K = sqrt(1.0 + ((cam.width + 2.0) / af) * ((cam.width + 2.0) / af) +
                        ((cam.height + 2.0) / af) * ((cam.height + 2.0) / af));
  k.pre = (k.fast && af >= 1e-3 && cam.width / af < 1024.0 && cam.height / af < 1024.0 &&
           K <= 16.0 && (af + fabs(cam.cx) + fabs(cam.cy)) * K < 65536.0)
              ? 1
              : 0;
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

// Certified fast projection.  The depth uz (cull test and key) is computed
// exactly as the reference does.  The pixel snap T = fl(fl(cx + fl(f * fl(ux
// / uz))) + 0.5) is replaced by T' = fma(fux', r, cx + 0.5) with fux' a DFMA
// chain over the host-rounded rows f*R and r = 1/uz from rcp.approx + two
// Newton steps.  For |T'| < 2^16, |cx|, |cy| < 2^15 and f <= 2^20 (checked on
// the host: DevCam::fast) the distance |T' - T| is below 2^-28 (DESIGN.md,
// "certified pixel snap"), so floor(T') == floor(T) whenever T' is at least
// 1.5 * 2^-24 from an integer.  The rare "uncertain" points are re-projected
// exactly.
// Returns 0 = culled, 1 = certain (ix, iy, dbits valid), 2 = uncertain.
__device__ __forceinline__ double rcp_approx_f64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__device__ __forceinline__ bool snap_certain(double t, uint32_t& i) {
  // s = t + 1.5*2^20 puts t on a 2^-32 grid: for |t| < 2^19 the high word is
  // 0x41380000 + floor(t) and the low word is frac(t) * 2^32.  Outside that
  // range (and for inf / NaN) the high word leaves the window, so i lands far
  // outside any image and the point is a certain miss.  A fraction within
  // 2^-23 of an integer is reported uncertain (exact f64 path decides).
  const double s = __dadd_rn(t, 1572864.0);
  i = (uint32_t)__double2hiint(s) - 0x41380000u;
  return (uint32_t)__double2loint(s) - 512u < 0xFFFFFC01u;
}

__device__ __forceinline__ void project_fast(float x, float y, float z, const DevCam& k,
                                             uint32_t& ix_out, uint32_t& iy_out, uint32_t& dbits,
                                             bool& hit, bool& uncertain) {
  const double w0 = __dadd_rn((double)x, k.nc[0]);  // == __dsub_rn(x, c[0]) bit for bit
  const double w1 = __dadd_rn((double)y, k.nc[1]);
  const double w2 = __dadd_rn((double)z, k.nc[2]);
  const double uz =
      __dadd_rn(__dadd_rn(__dmul_rn(w0, k.r[6]), __dmul_rn(w1, k.r[7])), __dmul_rn(w2, k.r[8]));
  const bool in_depth = uz > k.nr && uz < k.fr;  // python_impl.py:43 (NaN culled)
  dbits = __float_as_uint(__double2float_rn(uz));
  double r = rcp_approx_f64(uz);
  double e = __fma_rn(-uz, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-uz, r, 1.0);
  r = __fma_rn(r, e, r);
  // f * ux and f * uy with f folded into the rotation rows (host-rounded)
  const double fx = __fma_rn(w2, k.fr_[2], __fma_rn(w1, k.fr_[1], __dmul_rn(w0, k.fr_[0])));
  const double fy = __fma_rn(w2, k.fr_[5], __fma_rn(w1, k.fr_[4], __dmul_rn(w0, k.fr_[3])));
  const double tx = __fma_rn(fx, r, k.cxh);
  const double ty = __fma_rn(fy, r, k.cyh);
  uint32_t ix, iy;
  const bool cx_ok = snap_certain(tx, ix);
  const bool cy_ok = snap_certain(ty, iy);
  const bool certain = k.fast && cx_ok && cy_ok;
  const bool inside = ix < (uint32_t)k.w && iy < (uint32_t)k.h;
  ix_out = ix;
  iy_out = iy;
  hit = in_depth && certain && inside;  // certain hit
  uncertain = in_depth && !certain;     // in depth range, snap not certified
}

// f32 occlusion pre-test.  T' = T - 0.5 = (f R0 + cx R2).w / (R2.w) (the
// principal point folded into the rows, so no separate add), evaluated in f32
// as T'32 = fx32 * rcp(uz32) + 1.5*2^23: the low word of that sum is
// round(T'32), which is within +-1 of the exact pixel floor(T) for every point
// whose pixel is within one pixel of the image (|T'32 - T'| < 0.5 under the
// DevCam::pre bounds); points further out stay outside.  u = round(T'32) + 1
// indexes the Hi-Z on a grid shifted by one pixel whose blocks are dilated by
// one pixel (hiz_kernel), so the block of u bounds the depth of the exact
// pixel without clamping.  Returns true when the point certainly cannot win.
// Packed f32x2 helpers (FADD2 / FFMA2: two lanes of f32 per instruction; a
// pair built from one value twice becomes a scalar-broadcast operand).
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// (w0, w1) = (x, y) - chi[0..1] as one FADD2 (x, y adjacent in the lane's
// registers); returns the reject decision for one point.
__device__ __forceinline__ bool pretest_reject_w(float w0, float w1, float w2, const DevCam& k,
                                                 uint32_t zaddr, uint32_t umax, uint32_t vmax,
                                                 int shift, int zw) {
  const float uz = fmaf(w2, k.r2f[2], fmaf(w1, k.r2f[1], fmaf(w0, k.r2f[0], k.uz0)));
  // (T' uz for x, for y) with the rows paired: three FFMA2
  const uint64_t fxy =
      fma2(pk2(w2, w2), pk2(k.fxr[2], k.fyr[2]),
           fma2(pk2(w1, w1), pk2(k.fxr[1], k.fyr[1]),
                fma2(pk2(w0, w0), pk2(k.fxr[0], k.fyr[0]), pk2(k.fx0, k.fy0))));
  float rz;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rz) : "f"(uz));
  // bits of T' + 1.5*2^23 + 1 = 0x4B400000 + u with u = round(T') + 1; the
  // constant part of the block index is folded into the caller's `zd` base
  float sx, sy;
  upk2(fma2(fxy, pk2(rz, rz), pk2(12582913.0f, 12582913.0f)), sx, sy);
  // u, v clamped (unsigned: u < 0 wraps high) to the table's zero column /
  // row, whose entries reject any depth: no separate range test.  u in
  // (W+1, umax) lands in the last real column -- a candidate the exact path culls.
  const uint32_t u = min((uint32_t)__float_as_int(sx) - 0x4B400000u, umax);
  const uint32_t v = min((uint32_t)__float_as_int(sy) - 0x4B400000u, vmax);
  const uint32_t b = (v >> shift) * (uint32_t)zw + (u >> shift);
  uint16_t zq;
  asm("ld.shared.u16 %0, [%1];" : "=h"(zq) : "r"(zaddr + 2u * b));
  // (f32 bits of uz32 * (1 - 2^-14)) >> 16 > zd: strictly behind (negative / NaN uz32
  // compare high and are rejected unless the block is still empty)
  return (__float_as_uint(uz * 0.99993896484375f) >> 16) > (uint32_t)zq;
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

template <bool kSigned>
__device__ __forceinline__ void red_key(uint64_t* keybuf, uint32_t pix, uint64_t key) {
  if (kSigned)
    atomicMin(reinterpret_cast<long long*>(keybuf) + pix, (long long)(key ^ NAR_SIGN_FLIP));
  else
    atomicMin(reinterpret_cast<unsigned long long*>(keybuf) + pix, (unsigned long long)key);
}

// Atomic half of fold_key, given a previously loaded current value.
template <bool kSigned>
__device__ __forceinline__ bool fold_loaded(uint64_t* keybuf, uint32_t pix, uint64_t key,
                                            uint64_t cur) {
  if (kSigned) {
    const long long k = (long long)(key ^ NAR_SIGN_FLIP);
    const bool win = k < (long long)cur;
    if (win) atomicMin(reinterpret_cast<long long*>(keybuf) + pix, k);
    return win;
  } else {
    const bool win = key < cur;
    if (win) atomicMin(reinterpret_cast<unsigned long long*>(keybuf) + pix, (unsigned long long)key);
    return win;
  }
}

// ----------------------------------------------------------------------------
// render: persistent CTAs, every warp streams its own point chunks (64 points in
// the exact kernel, 128-point units in the pre-test kernel) through a private
// ring of TMA bulk copies (no cross-warp coupling on the data path)
// ----------------------------------------------------------------------------
#ifndef NAR_RENDER_WARPS
#define NAR_RENDER_WARPS 24
#endif
#ifndef NAR_RENDER_PPT
#define NAR_RENDER_PPT 2
#endif
constexpr int kRenderWarps = NAR_RENDER_WARPS;
constexpr int kRenderThreads = kRenderWarps * 32;
constexpr int kPtsPerThread = NAR_RENDER_PPT;
constexpr int kChunkPts = 32 * kPtsPerThread;                // points per warp step
constexpr int kChunkBytes = kChunkPts * 12;
// ring depth of the exact kernel: 6 x 64-point or 3 x 128-point chunks in flight per warp
constexpr int kWarpStages = kPtsPerThread >= 4 ? 3 : 6;
constexpr int kRingBytes = kRenderWarps * kWarpStages * kChunkBytes;
constexpr int kQueueBytes = kRenderWarps * 32 * 16;
constexpr int kHizMaxEntries = 34816;                        // 68 KB coarse depth (u16)
constexpr int kRenderSmem = kRingBytes + kQueueBytes + kHizMaxEntries * 2 +
                            kRenderWarps * kWarpStages * 8 + kRenderWarps * kWarpStages * 4 + 128;
constexpr int kUnitPts = 128;  // schedule granularity (tail -> simple kernel)
constexpr int kChunksPerUnit = kUnitPts / kChunkPts;  // exact-kernel chunks per unit (1 or 2)
static_assert(kChunksPerUnit * kChunkPts == kUnitPts, "chunk / unit sizes");
constexpr int kUnitBytes = kUnitPts * 12;
constexpr int kTilePts = kUnitPts;

// Unit schedule of one launch: slots j in [j0, j1) map to 128-point units of
// the cloud by mode 0: j; 1 (Hi-Z seed pass): j*S; 2 (the rest):
// j + j/(S-1) + 1, i.e. every unit that is not a multiple of S.  The exact
// kernel walks 64-point halves of the units (chunk c = slot c/2, half c%2).
constexpr int kHizSeedStride = 24;  // S
struct ChunkMap {
  int64_t j0, j1;  // unit slots (< 2^25: point indices are 32-bit)
  int32_t mode;
  // interleaving: slot j -> j' = period*(j >> lshift) + r0 + (j & (2^lshift - 1)), i.e.
  // the residues [r0, r0 + 2^lshift) mod `period` of the mode's sequence, so a
  // pass samples the whole cloud (spatially uniform also for sorted clouds)
  uint32_t period, r0, lshift;
  __device__ __forceinline__ uint32_t unit(uint32_t j) const {
    const uint32_t jj = period * (j >> lshift) + r0 + (j & ((1u << lshift) - 1u));
    return mode == 0 ? jj : (mode == 1 ? jj * kHizSeedStride : jj + jj / (kHizSeedStride - 1) + 1);
  }
  // unit() for a compile-time mode (modes 0 and 1 always have period 1, r0 0,
  // lshift 0: slot j is unit j, resp. unit j * kHizSeedStride)
  template <int M>
  __device__ __forceinline__ uint32_t unit_m(uint32_t j) const {
    if (M == 0) return j;
    if (M == 1) return j * kHizSeedStride;
    const uint32_t jj = period * (j >> lshift) + r0 + (j & ((1u << lshift) - 1u));
    return jj + jj / (kHizSeedStride - 1) + 1;
  }
  // first point of 64-point chunk c (c counts halves of slots)
  __device__ __forceinline__ uint32_t off64(uint32_t c) const {
    return unit(c / kChunksPerUnit) * kUnitPts + (c % kChunksPerUnit) * kChunkPts;
  }
};

// Hierarchical-Z: zq[b] = ceil(max f32 depth bits in coarse block b / 2^16)
// over 2^shift x 2^shift pixels; a point with (depth bits >> 16) > zq[b] is
// behind every pixel of the block (strictly deeper), so it cannot win.
struct HizArgs {
  const uint16_t* zmax;  // NULL: no coarse test in this pass
  int32_t shift, zw, entries;  // zw: table pitch incl. the zero column
  int32_t zh;                  // table rows incl. the zero row
  unsigned long long* stats;  // NULL, or this pass's counter of points passing the coarse test
  unsigned long long* stats_clear;  // seed pass: counters to zero (block 0), else NULL
};

constexpr int kPassStats = 8;  // passes with statistics (see PassState)
// counters per render: [0, kPassStats) points past the coarse test, [kPassStats, 2 kPassStats)
// points past the exact kernel's early-z read (an atomic issued; exact-kernel passes only)
constexpr int kStatCtrs = 2 * kPassStats;

// Sum of a per-thread count over the warp, added once by lane 0.
__device__ __forceinline__ void add_warp_count(unsigned long long* ctr, uint32_t v) {
  v = __reduce_add_sync(0xffffffffu, v);
  if (ctr && (threadIdx.x & 31) == 0 && v) atomicAdd(ctr, (unsigned long long)v);
}

struct QEntry {
  float x, y, z;
  uint32_t idx;
};

// Exact re-projection of up to 32 queued uncertain points, one per lane.
template <bool kSigned>
__device__ __forceinline__ void flush_queue(const QEntry* q, int n, int lane, uint64_t* keybuf,
                                            const DevCam& cam) {
  __syncwarp();
  if (lane < n) {
    const QEntry e = q[lane];
    uint32_t pix, db;
    if (project_point(e.x, e.y, e.z, cam, pix, db))
      fold_key<kSigned>(keybuf, pix, ((uint64_t)db << 32) | e.idx);
  }
  __syncwarp();
}

// Exact kernel (seed pass, small clouds, cameras outside the pre-test bounds).
// Per warp step (one 64-point chunk, 2 points per lane):
// (1) certified fast projection; uncertain points go to the warp's queue and
//     are re-projected exactly once 32 have gathered;
// (2) Hi-Z test against the smem coarse depth -- occluded points stop here;
// (3) hand the ring slot back to TMA (chunk k + kWarpStages);
// (4) kRed (seed pass): atomicMin (RED) every hit; otherwise fold the PREVIOUS
//     chunk's hits, whose keybuf reads were issued one step ago, so the
//     random-L2 read latency overlaps a chunk of math, and
// (5) issue this chunk's keybuf reads.
template <bool kSigned, bool kRed, bool kStats = false>
__global__ void __launch_bounds__(kRenderThreads, 1)
    render_tma_kernel(uint64_t* __restrict__ keybuf, const float* __restrict__ pos,
                      const ChunkMap cm, uint64_t base_index, const DevCam cam, const HizArgs hz) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t pol = l2_evict_first_policy();  // the point stream (see bulk_g2s_stream)
  float* ring = reinterpret_cast<float*>(smem) + warp * (kWarpStages * kChunkPts * 3);
  QEntry* wq = reinterpret_cast<QEntry*>(smem + kRingBytes) + warp * 32;
  uint16_t* zs = reinterpret_cast<uint16_t*>(smem + kRingBytes + kQueueBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes + kQueueBytes +
                                               kHizMaxEntries * 2) + warp * kWarpStages;
  // first point of the chunk in each ring slot, written by the lane that issues its copy
  // (the chunk -> unit map is computed once per chunk)
  uint32_t* soff = reinterpret_cast<uint32_t*>(smem + kRingBytes + kQueueBytes + kHizMaxEntries * 2 +
                                               kRenderWarps * kWarpStages * 8) + warp * kWarpStages;

  const int64_t c_first = kChunksPerUnit * cm.j0 + (int64_t)blockIdx.x * kRenderWarps + warp;
  const int64_t c_stride = (int64_t)gridDim.x * kRenderWarps;
  const int64_t n_chunks = kChunksPerUnit * cm.j1;
  if (lane == 0) {
    for (int s = 0; s < kWarpStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    for (int s = 0; s < kWarpStages; ++s) {
      const int64_t c = c_first + (int64_t)s * c_stride;
      if (c < n_chunks) {
        const uint32_t off = cm.off64((uint32_t)c);
        soff[s] = off;
        mbar_expect_tx(&full[s], kChunkBytes);
        bulk_g2s_stream(ring + s * (kChunkPts * 3), pos + (size_t)off * 3, kChunkBytes, &full[s], pol);
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (see render_pre_kernel)
  const bool use_hiz = hz.zmax != nullptr;
  if (hz.stats_clear && blockIdx.x == 0 && threadIdx.x < kStatCtrs) hz.stats_clear[threadIdx.x] = 0ull;
  if (use_hiz) {
    const uint4* src = reinterpret_cast<const uint4*>(hz.zmax);
    uint4* dst = reinterpret_cast<uint4*>(zs);
    for (int i = tid; i < (hz.entries + 7) / 8; i += kRenderThreads) dst[i] = __ldcg(src + i);
    __syncthreads();
  }
  __syncwarp();

  const uint32_t lt_mask = (1u << lane) - 1u;
  int qn = 0;  // warp-uniform queue fill
  uint32_t ppix[kPtsPerThread];
  uint64_t pkey[kPtsPerThread], pcur[kPtsPerThread];
  uint32_t pmask = 0;
  uint32_t n_surv = 0;  // points past the coarse test (pass statistics)
  uint32_t n_win = 0;   // ... and past the early-z read (kStats)
#pragma unroll
  for (int j = 0; j < kPtsPerThread; ++j) {
    ppix[j] = 0;
    pkey[j] = 0;
    pcur[j] = 0;
  }

  int s = 0;          // ring slot of this chunk
  uint32_t ph = 0u;    // its mbarrier phase parity
#pragma unroll 2
  for (int64_t c = c_first; c < n_chunks; c += c_stride) {
    mbar_wait(&full[s], ph);
    const int sc = s;  // this chunk's slot; advance (the kRed path continues early)
    if (++s == kWarpStages) {
      s = 0;
      ph ^= 1u;
    }
    const float* chunk = ring + sc * (kChunkPts * 3);
    const uint32_t cbase = (uint32_t)base_index + soff[sc];

    // (1) projections: straight-line, interleavable across the 4 points
    float px[kPtsPerThread], py[kPtsPerThread], pz[kPtsPerThread];
    uint32_t ixs[kPtsPerThread], iys[kPtsPerThread], dbs[kPtsPerThread];
    bool hits[kPtsPerThread], uncs[kPtsPerThread];
#pragma unroll
    for (int j = 0; j < kPtsPerThread; ++j) {
      const int p = j * 32 + lane;
      px[j] = chunk[3 * p];
      py[j] = chunk[3 * p + 1];
      pz[j] = chunk[3 * p + 2];
    }
    __syncwarp();
    {  // (3) slot sc is consumed: refill it with the chunk kWarpStages steps ahead
      const int64_t cn = c + (int64_t)kWarpStages * c_stride;
      if (lane == 0 && cn < n_chunks) {
        const uint32_t off = cm.off64((uint32_t)cn);
        soff[sc] = off;  // read by the lanes after this slot's next full wait
        fence_proxy_async_smem();
        mbar_expect_tx(&full[sc], kChunkBytes);
        bulk_g2s_stream(ring + sc * (kChunkPts * 3), pos + (size_t)off * 3, kChunkBytes, &full[sc], pol);
      }
    }
#pragma unroll
    for (int j = 0; j < kPtsPerThread; ++j)
      project_fast(px[j], py[j], pz[j], cam, ixs[j], iys[j], dbs[j], hits[j], uncs[j]);

    // (2) Hi-Z test, uncertain queue
    uint32_t pix[kPtsPerThread], idxs[kPtsPerThread];
    uint64_t key[kPtsPerThread];
    uint32_t okmask = 0, umask = 0;
#pragma unroll
    for (int j = 0; j < kPtsPerThread; ++j) {
      const int p = j * 32 + lane;
      const uint32_t db = dbs[j];
      bool hit = hits[j];
      if (use_hiz) {  // behind every pixel of its coarse block? (index clamped: no branch)
        const uint32_t zb =
            hit ? ((iys[j] + 1u) >> hz.shift) * (uint32_t)hz.zw + ((ixs[j] + 1u) >> hz.shift) : 0u;
        hit = hit && (db >> 16) <= zs[zb];
      }
      pix[j] = iys[j] * (uint32_t)cam.w + ixs[j];
      const uint32_t idx = cbase + (uint32_t)p;
      key[j] = ((uint64_t)db << 32) | idx;
      okmask |= (uint32_t)hit << j;
      umask |= (uint32_t)uncs[j] << j;
      idxs[j] = idx;
    }
    if (__any_sync(0xffffffffu, umask != 0u)) {
#pragma unroll
      for (int j = 0; j < kPtsPerThread; ++j) {
        const uint32_t b = __ballot_sync(0xffffffffu, (umask >> j) & 1u);
        if (b) {
          const int nb = __popc(b);
          if (qn + nb > 32) {
            flush_queue<kSigned>(wq, qn, lane, keybuf, cam);
            qn = 0;
          }
          if ((umask >> j) & 1u)
            wq[qn + __popc(b & lt_mask)] = QEntry{px[j], py[j], pz[j], idxs[j]};
          qn += nb;
        }
      }
    }
    if constexpr (kRed) {  // seed units: the keybuf is still mostly empty, early-z would not filter
#pragma unroll
      for (int j = 0; j < kPtsPerThread; ++j)
        if ((okmask >> j) & 1u) red_key<kSigned>(keybuf, pix[j], key[j]);
      continue;
    }
    // (4) + (5)
#pragma unroll
    for (int j = 0; j < kPtsPerThread; ++j)
      if ((pmask >> j) & 1u) {
        const bool w = fold_loaded<kSigned>(keybuf, ppix[j], pkey[j], pcur[j]);
        if constexpr (kStats) n_win += w;
      }
#pragma unroll
    for (int j = 0; j < kPtsPerThread; ++j) {
      if ((okmask >> j) & 1u)
        pcur[j] = __ldcg(reinterpret_cast<const unsigned long long*>(keybuf) + pix[j]);
      ppix[j] = pix[j];
      pkey[j] = key[j];
    }
    pmask = okmask;
    n_surv += __popc(okmask);
  }
#pragma unroll
  for (int j = 0; j < kPtsPerThread; ++j)
    if ((pmask >> j) & 1u) {
      const bool w = fold_loaded<kSigned>(keybuf, ppix[j], pkey[j], pcur[j]);
      if constexpr (kStats) n_win += w;
    }
  flush_queue<kSigned>(wq, qn, lane, keybuf, cam);
  add_warp_count(hz.stats, n_surv);
  if constexpr (kStats) add_warp_count(hz.stats ? hz.stats + kPassStats : nullptr, n_win);
}

// Hi-Z passes: the f32 pre-test rejects most points in ~25 instructions; the
// rest (candidates) are compacted into a per-warp shared-memory queue and run
// through the exact path 32 at a time with every lane busy:
// (1) pre-test the lane's 4 points; ballot-compact candidates (xyz, index)
//     onto the queue; hand the ring slot back to TMA;
// (2) while >= 32 are queued, pop 32: certified projection (uncertain ones
//     take the exact f64 path inline -- they are ~1e-6 of points) and a
//     fire-and-forget atomicMin (RED).
// Each warp step takes one 128-point unit (4 points per lane) in one ring
// stage; candidates are drained after each half, so the queue never holds
// more than 31 + 64.  Seed units (kMode 1) skip (1) and (2): exact_direct.
#ifndef NAR_PRE_STAGES
#define NAR_PRE_STAGES 3
#endif
constexpr int kPreStages = NAR_PRE_STAGES;
constexpr int kPreRingBytes = kRenderWarps * kPreStages * kUnitBytes;
constexpr int kCandCap = 32 + 64;  // queue entries per warp (drained after every 64 points)
constexpr int kCandBytes = kRenderWarps * kCandCap * 16;
constexpr int kPreSmem =
    kPreRingBytes + kCandBytes + kHizMaxEntries * 2 + kRenderWarps * kPreStages * 8 + 128;
static_assert(kPreSmem <= 227 * 1024, "pre-test kernel smem");

// Exact path for one queued candidate.  Certain hits go straight to a
// fire-and-forget atomicMin (RED): the candidates already passed the Hi-Z
// test, so an early-z read of the keybuf would mostly confirm them and only
// stall the warp for the L2 round trip.  Uncertain snaps (~1e-6 of points)
// take the exact f64 path.
template <bool kSigned>
__device__ __forceinline__ void exact_candidate(const QEntry e, uint64_t* keybuf,
                                                const DevCam& cam) {
  uint32_t ix, iy, db;
  bool hit, unc;
  project_fast(e.x, e.y, e.z, cam, ix, iy, db, hit, unc);
  if (hit) {
    red_key<kSigned>(keybuf, iy * (uint32_t)cam.w + ix, ((uint64_t)db << 32) | e.idx);
  } else if (unc) {
    uint32_t pix;
    if (project_point(e.x, e.y, e.z, cam, pix, db))
      red_key<kSigned>(keybuf, pix, ((uint64_t)db << 32) | e.idx);
  }
}

// Seed units (kMode 1) skip the pre-test: every point goes straight down the
// exact path, 4 independent projections per lane (the keybuf is still nearly
// empty, so neither the coarse test nor early z would filter); with a coarse
// depth present (the keybuf already holds this frame) the exact pixel is tested.
template <bool kSigned>
__device__ __forceinline__ void exact_direct(float x, float y, float z, uint32_t idx,
                                             uint64_t* keybuf, const DevCam& cam,
                                             const uint16_t* zs, const HizArgs& hz) {
  uint32_t ix, iy, db;
  bool hit, unc;
  project_fast(x, y, z, cam, ix, iy, db, hit, unc);
  if (hit) {
    if (hz.zmax) {
      const uint32_t zb = ((iy + 1u) >> hz.shift) * (uint32_t)hz.zw + ((ix + 1u) >> hz.shift);
      hit = (db >> 16) <= zs[zb];
    }
    if (hit) red_key<kSigned>(keybuf, iy * (uint32_t)cam.w + ix, ((uint64_t)db << 32) | idx);
  } else if (unc) {
    uint32_t pix;
    if (project_point(x, y, z, cam, pix, db))
      red_key<kSigned>(keybuf, pix, ((uint64_t)db << 32) | idx);
  }
}

// timing experiments (-DNAR_RENDER_TRACE): per-warp finish time (globaltimer, ns) of
// the last pre-test launch, to size the tail imbalance of the static unit split
#ifdef NAR_RENDER_TRACE
__device__ unsigned long long g_render_trace[148 * kRenderWarps + 1];
#endif
template <bool kSigned, int kMode, bool kStats>
__global__ void __launch_bounds__(kRenderThreads, 1)
    render_pre_kernel(uint64_t* __restrict__ keybuf, const float* __restrict__ pos,
                      const ChunkMap cm, uint64_t base_index, const DevCam cam, const HizArgs hz) {
  static_assert(kMode >= 0 && kMode <= 2, "ChunkMap mode");
  if (hz.stats_clear && blockIdx.x == 0 && threadIdx.x < kStatCtrs) hz.stats_clear[threadIdx.x] = 0ull;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t pol = l2_evict_first_policy();  // the point stream (see bulk_g2s_stream)
  float* ring = reinterpret_cast<float*>(smem) + warp * (kPreStages * kUnitPts * 3);
  QEntry* wq = reinterpret_cast<QEntry*>(smem + kPreRingBytes) + warp * kCandCap;
  uint16_t* zs = reinterpret_cast<uint16_t*>(smem + kPreRingBytes + kCandBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPreRingBytes + kCandBytes +
                                               kHizMaxEntries * 2) + warp * kPreStages;

  const uint32_t j_first = (uint32_t)cm.j0 + blockIdx.x * kRenderWarps + warp;
  const uint32_t j_stride = gridDim.x * kRenderWarps;
  const uint32_t j_end = (uint32_t)cm.j1;
  // unit indices of the kPreStages slots in flight, oldest first (a register
  // FIFO: each slot's index is computed once, when its refill is issued)
  uint32_t uq[kPreStages];
#pragma unroll
  for (int s = 0; s < kPreStages; ++s) uq[s] = cm.unit_m<kMode>(j_first + s * j_stride);
  if (lane == 0) {
    for (int s = 0; s < kPreStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
#pragma unroll
    for (int s = 0; s < kPreStages; ++s) {
      const uint32_t j = j_first + s * j_stride;
      if (j < j_end) {
        mbar_expect_tx(&full[s], kUnitBytes);
        bulk_g2s_stream(ring + s * (kUnitPts * 3), pos + (size_t)uq[s] * (kUnitPts * 3),
                        kUnitBytes, &full[s], pol);
      }
    }
  }
  // the point stream above does not depend on the previous kernel; the coarse depth
  // and the keybuf do (a no-op unless launched as a programmatic dependent)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (hz.zmax) {
    const uint4* src = reinterpret_cast<const uint4*>(hz.zmax);
    uint4* dst = reinterpret_cast<uint4*>(zs);
    for (int i = tid; i < (hz.entries + 7) / 8; i += kRenderThreads) dst[i] = __ldcg(src + i);
  }
  __syncthreads();
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t zaddr = smem_u32(zs);
  // first u (v) of the zero column (row): see pretest_reject_w
  const uint32_t umax = (uint32_t)(hz.zw - 1) << hz.shift, vmax = (uint32_t)(hz.zh - 1) << hz.shift;
  int qn = 0;  // warp-uniform queue fill
  uint32_t n_drained = 0;  // candidates drained in full batches of 32 (pass statistics)
  int s = 0;          // ring slot of this iteration: k % kPreStages
  uint32_t ph = 0u;    // its mbarrier phase parity: (k / kPreStages) & 1
  for (uint32_t j = j_first; j < j_end; j += j_stride) {
    mbar_wait(&full[s], ph);
    const float* unit = ring + s * (kUnitPts * 3);
    const uint32_t cb = (uint32_t)base_index + uq[0] * kUnitPts;
    // lane l takes points 4l .. 4l+3: three conflict-free 16-byte loads
    const float4* u4 = reinterpret_cast<const float4*>(unit) + 3 * lane;
    const float4 a0 = u4[0], a1 = u4[1], a2 = u4[2];
    const float px[4] = {a0.x, a0.w, a1.z, a2.y};
    const float py[4] = {a0.y, a1.x, a1.w, a2.z};
    const float pz[4] = {a0.z, a1.y, a2.x, a2.w};
    __syncwarp();
    {  // stage s is consumed: refill it with unit k + kPreStages
      const uint32_t jn = j + kPreStages * j_stride;
      const uint32_t un = cm.unit_m<kMode>(jn);
      if (jn < j_end)  // warp-uniform: one elected lane issues (no per-lane loop)
        bulk_g2s_elect_stream(ring + s * (kUnitPts * 3), pos + (size_t)un * (kUnitPts * 3),
                              kUnitBytes, &full[s], pol);
#pragma unroll
      for (int i = 0; i + 1 < kPreStages; ++i) uq[i] = uq[i + 1];
      uq[kPreStages - 1] = un;
    }
    if (kMode == 1) {  // seed units: straight down the exact path
#pragma unroll
      for (int q = 0; q < 4; ++q)
        exact_direct<kSigned>(px[q], py[q], pz[q], cb + (uint32_t)(4 * lane + q), keybuf, cam, zs,
                              hz);
      if (++s == kPreStages) {
        s = 0;
        ph ^= 1u;
      }
      continue;
    }
    // w = p - chi: the (x, y) or (y, z) halves of each point that sit in one
    // aligned register pair go through FADD2
    float w[4][3];
    {
      const uint64_t c01 = pk2(cam.chi[0], cam.chi[1]), c12 = pk2(cam.chi[1], cam.chi[2]);
      upk2(sub2(pk2(a0.x, a0.y), c01), w[0][0], w[0][1]);
      w[0][2] = a0.z - cam.chi[2];
      w[1][0] = a0.w - cam.chi[0];
      upk2(sub2(pk2(a1.x, a1.y), c12), w[1][1], w[1][2]);
      upk2(sub2(pk2(a1.z, a1.w), c01), w[2][0], w[2][1]);
      w[2][2] = a2.x - cam.chi[2];
      w[3][0] = a2.y - cam.chi[0];
      upk2(sub2(pk2(a2.z, a2.w), c12), w[3][1], w[3][2]);
    }
    bool cand[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      cand[q] = !pretest_reject_w(w[q][0], w[q][1], w[q][2], cam, zaddr, umax, vmax, hz.shift,
                                  hz.zw);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int q = 2 * h; q < 2 * h + 2; ++q) {
        const uint32_t b = __ballot_sync(0xffffffffu, cand[q]);
        if (cand[q])
          wq[qn + __popc(b & lt_mask)] =
              QEntry{px[q], py[q], pz[q], cb + (uint32_t)(4 * lane + q)};
        qn += __popc(b);
      }
      if (qn >= 32) {  // warp-uniform; at most 31 + 64 queued
        __syncwarp();
        const QEntry e = wq[qn - 32 + lane];
        __syncwarp();
        qn -= 32;
        if (kStats) n_drained += 32;
        exact_candidate<kSigned>(e, keybuf, cam);
        if (qn >= 32) {
          __syncwarp();
          const QEntry e2 = wq[qn - 32 + lane];
          __syncwarp();
          qn -= 32;
          if (kStats) n_drained += 32;
          exact_candidate<kSigned>(e2, keybuf, cam);
        }
      }
    }
    if (++s == kPreStages) {
      s = 0;
      ph ^= 1u;
    }
  }
  __syncwarp();
  if (lane < qn) exact_candidate<kSigned>(wq[lane], keybuf, cam);
  // warp-uniform total: every candidate was drained in a batch or is in the tail
  if (kStats && lane == 0 && n_drained + qn)
    atomicAdd(hz.stats, (unsigned long long)(n_drained + qn));
#ifdef NAR_RENDER_TRACE
  if (lane == 0 && blockIdx.x < 148) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_render_trace[blockIdx.x * kRenderWarps + warp] = t;
  }
#endif
}

#ifdef NAR_RENDER_TRACE
extern "C" int nar_debug_render_trace(unsigned long long* out, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_render_trace, n * 8) == cudaSuccess ? 0 : 2;
}
#endif

// Coarse max depth of the current keybuf on the shifted, dilated grid: block
// (bu, bv) holds ceil(max depth bits / 2^16) over pixels x in
// [bu*S - 2, bu*S + S - 1] (and y alike), i.e. the pixels whose u = x + 1 falls
// in the block plus a one-pixel border -- the window the f32 pre-test needs.
// S = 2^shift threads per block, one row each (threads 0, 1 take the two extra
// rows), max-reduced with warp shuffles.
template <bool kSigned, int kNv>  // kNv: 16-byte loads per row, (side + 2) / 2
__global__ void __launch_bounds__(256)
    hiz_kernel(const uint64_t* __restrict__ keybuf, int W, int H, int shift, int zw, int zh,
               uint16_t* __restrict__ zmax) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int side = 1 << shift;
  const int b = (int)(t >> shift), row = (int)(t & (side - 1));
  const bool valid = b < zw * zh;
  uint32_t m = 0;
  const int bx = valid ? b % zw : 0, by = valid ? b / zw : 0;
  const bool edge = bx == zw - 1 || by == zh - 1;  // zero column / row: rejects every point
  if (valid && !edge) {
    const int x0 = max((bx << shift) - 2, 0), x1 = min((bx << shift) + side, W);
    // rows are 16-byte aligned when W is even: pairs of keys per load, all
    // issued before the max (x0 is even); (side + 2) / 2 loads for 8-, 16- and
    // 32-pixel blocks (4K frames take 16)
    const bool vec = ((W & 1) == 0) && 2 * kNv == side + 2;
    auto scan = [&](int y) {
      if (y < 0 || y >= H) return;
      const unsigned long long* p =
          reinterpret_cast<const unsigned long long*>(keybuf) + (size_t)y * W;
      if (vec) {
        ulonglong2 v[kNv];
#pragma unroll
        for (int i = 0; i < kNv; ++i)
          v[i] = x0 + 2 * i + 1 < x1
                     ? __ldcg(reinterpret_cast<const ulonglong2*>(p + x0) + i)
                     : make_ulonglong2(0ull, 0ull);
#pragma unroll
        for (int i = 0; i < kNv; ++i) {
          const bool in = x0 + 2 * i + 1 < x1;
          uint64_t a = v[i].x, b = v[i].y;
          if (kSigned) {
            a = in ? a ^ NAR_SIGN_FLIP : 0ull;
            b = in ? b ^ NAR_SIGN_FLIP : 0ull;
          }
          m = max(m, max((uint32_t)(a >> 32), (uint32_t)(b >> 32)));
        }
        return;
      }
#pragma unroll 4
      for (int x = x0; x < x1; ++x) {
        uint64_t k = __ldcg(p + x);
        if (kSigned) k ^= NAR_SIGN_FLIP;
        m = max(m, (uint32_t)(k >> 32));
      }
    };
    const int y = (by << shift) - 2 + row;
    scan(y);
    if (row < 2) scan(y + side);
  }
  for (int o = 1; o < side; o <<= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (valid && row == 0) {
    const uint32_t q = (m >> 16) + ((m & 0xFFFFu) != 0u);  // round up: conservative
    zmax[b] = edge ? (uint16_t)0 : (uint16_t)(q > 0xFFFFu ? 0xFFFFu : q);
  }
}

// The same coarse table with coalesced reads (even W): a CTA takes one block row by and
// 256 consecutive 2-pixel chunks of it -- every load instruction of a warp covers 512
// contiguous bytes of one image row (hiz_kernel gives each thread a row of one block, so
// its warp touches 32 rows per load).  Each thread keeps the max depth bits of its chunk
// over the window rows [by S - 2, by S + S); the chunk maxima go through shared memory
// and block bx takes chunks [bx S/2 - 1, bx S/2 + S/2 - 1] (its dilated window).  CTA x
// covers kNb = 255 / (S/2) blocks; the edge column / row get 0 as in hiz_kernel.
template <bool kSigned, int S>
__global__ void __launch_bounds__(256)
    hiz_rows_kernel(const uint64_t* __restrict__ keybuf, int W, int H, int zw, int zh,
                    uint16_t* __restrict__ zmax) {
  // the next render pass may be launched now (programmatic dependent launch): its
  // CTAs take SMs as our blocks drain and start their point streams, then wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int kHalf = S / 2, kNb = 255 / kHalf;
  __shared__ uint32_t cm[256];
  const int by = blockIdx.y;
  const int b0 = blockIdx.x * kNb;
  const int t = threadIdx.x;
  uint32_t m = 0;
  if (by < zh - 1) {
    const int c = b0 * kHalf - 1 + t;  // chunk: pixels 2c, 2c + 1
    if (c >= 0 && 2 * c + 1 < W && t <= kNb * kHalf) {
      const int ya = max(by * S - 2, 0), yb = min(by * S + S, H);
      const ulonglong2* p = reinterpret_cast<const ulonglong2*>(keybuf) + c;
      const int rs = W / 2;  // row stride in chunks
      int y = ya;
      for (; y + 4 <= yb; y += 4) {  // 4 rows in flight
        ulonglong2 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = __ldcg(p + (size_t)(y + i) * rs);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint64_t a = kSigned ? v[i].x ^ NAR_SIGN_FLIP : v[i].x;
          const uint64_t b = kSigned ? v[i].y ^ NAR_SIGN_FLIP : v[i].y;
          m = max(m, max((uint32_t)(a >> 32), (uint32_t)(b >> 32)));
        }
      }
      for (; y < yb; ++y) {
        const ulonglong2 v = __ldcg(p + (size_t)y * rs);
        const uint64_t a = kSigned ? v.x ^ NAR_SIGN_FLIP : v.x;
        const uint64_t b = kSigned ? v.y ^ NAR_SIGN_FLIP : v.y;
        m = max(m, max((uint32_t)(a >> 32), (uint32_t)(b >> 32)));
      }
    }
  }
  cm[t] = m;
  __syncthreads();
  const int bx = b0 + t;
  if (t < kNb && bx < zw) {
    uint32_t mm = 0;
#pragma unroll
    for (int i = 0; i <= kHalf; ++i) mm = max(mm, cm[t * kHalf + i]);
    const bool edge = bx == zw - 1 || by == zh - 1;
    const uint32_t q = (mm >> 16) + ((mm & 0xFFFFu) != 0u);  // round up: conservative
    zmax[(size_t)by * zw + bx] = edge ? (uint16_t)0 : (uint16_t)(q > 0xFFFFu ? 0xFFFFu : q);
  }
}

static void hiz_geometry(int W, int H, int& shift, int& zw, int& zh) {
  shift = 3;  // <= 5 (one warp per coarse block row set) for any image < 2^32 pixels
  for (;;) {
    // u = x + 1 in [0, W + 1] on the shifted grid, plus a zero column / row
    zw = ((W + 1) >> shift) + 2;
    zh = ((H + 1) >> shift) + 2;
    if ((int64_t)zw * zh <= kHizMaxEntries) return;
    ++shift;
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
  // composite + resolve over peer memory: the key of a pixel is the minimum
  // over nkeys keybufs (other GPUs' buffers mapped into this address space);
  // only padded-output rows [row0, row1) are resolved (this rank's slice)
  const uint64_t* keys[NAR_MAX_SEGMENTS];
  int32_t nkeys;
  int32_t row0, row1;
  // the winners' rgb bytes per image pixel (c0 | c1 << 8 | c2 << 16), gathered on the
  // host (nar_host_gather_rgb) instead of by the kernel (nar_resolve_pixrgb)
  const uint32_t* pix_rgb;
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

// Vel2D channels of one point (velocity.py:26-48 + camera.py:154-166), f64 as the
// reference (BLAS order: <= 1 f32 ulp): (vx, vy, theta, magnitude), scaled.
__device__ __forceinline__ void vel2d_channels(const float* pos3, const double v[3],
                                               const DevCam& k, double scale, float out[4]) {
  const double w0 = (double)__ldg(pos3) - k.c[0];
  const double w1 = (double)__ldg(pos3 + 1) - k.c[1];
  const double w2 = (double)__ldg(pos3 + 2) - k.c[2];
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
  out[0] = (float)(vp0 / scale);
  out[1] = (float)(vp1 / scale);
  out[2] = (float)theta;
  out[3] = (float)(mag / scale);
}

// kRgbd: the selection is exactly rgb (u8, arity >= 3) + depth -- one float4
// store per pixel.  Otherwise channels are stored straight to global memory as
// they are produced (no per-thread channel array: dynamic indexing would put
// it in local memory).
template <bool kSigned, bool kRgbd>
__global__ void __launch_bounds__(256)
    resolve_kernel(uint64_t* __restrict__ keybuf, const ResolveParams P) {
  const int32_t W = P.cam.w, H = P.cam.h;
  const int64_t npix_out = (int64_t)(P.row1 - P.row0) * P.data_w;
  const int64_t lid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (lid >= npix_out) return;
  const int64_t gid = (int64_t)P.row0 * P.data_w + lid;
  const int32_t y = (int32_t)(gid / P.data_w);
  const int32_t x = (int32_t)(gid - (int64_t)y * P.data_w);
  float* dst = P.data ? P.data + gid * P.C : nullptr;
  if (!(y < H && x < W)) {  // padding of the CNN input: zeros
    if (dst) {
      if (kRgbd) *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      else for (int c = 0; c < P.C; ++c) dst[c] = 0.0f;
    }
    return;
  }
  const int64_t pix = (int64_t)y * W + x;
  const uint64_t empty_raw = kSigned ? (NAR_EMPTY_KEY ^ NAR_SIGN_FLIP) : NAR_EMPTY_KEY;
  uint64_t key;
  if (P.nkeys > 0) {  // composite: min over the ranks' keybufs (in the unsigned order)
    key = NAR_EMPTY_KEY;
    for (int k = 0; k < P.nkeys; ++k) {
      uint64_t v = __ldcg(reinterpret_cast<const unsigned long long*>(P.keys[k]) + pix);
      if (kSigned) v ^= NAR_SIGN_FLIP;
      key = v < key ? v : key;
    }
    if (P.clear)
      for (int k = 0; k < P.nkeys; ++k) const_cast<uint64_t*>(P.keys[k])[pix] = empty_raw;
  } else {
    key = keybuf[pix];
    if (kSigned) key ^= NAR_SIGN_FLIP;
    if (P.clear) keybuf[pix] = empty_raw;
  }
  const bool covered = key != NAR_EMPTY_KEY;
  const int64_t idx = covered ? (int64_t)(key & 0xFFFFFFFFull) : -1;
  const float dep = covered ? __uint_as_float((uint32_t)(key >> 32)) : 0.0f;
  if (P.coverage) P.coverage[pix] = covered ? 1 : 0;
  if (P.index_plane) P.index_plane[pix] = idx;
  if (P.depth) P.depth[pix] = dep;
  if (!dst) return;  // planes only (no channel data requested)

  int s = -1;
  if (covered) {
    for (int k = 0; k < P.nseg; ++k)
      if (idx >= P.seg[k].begin && idx < P.seg[k].begin + P.seg[k].count) s = k;
  }
  const nar_selection& sel = P.sel;
  if (kRgbd) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (s >= 0) {
      const uint8_t* c = static_cast<const uint8_t*>(P.seg[s].rgb) +
                         (idx - P.seg[s].begin) * sel.rgb_arity;
      // the 3 bytes through one aligned 8-byte load (two when they straddle):
      // attributes in mapped host memory cost one PCIe read per load
      // -- only where the aligned words lie inside the stream's own bytes
      // [base, base + count * arity); at its first / last bytes, byte loads
      const uintptr_t ca = reinterpret_cast<uintptr_t>(c);
      const uint32_t off = (uint32_t)(ca & 7u);
      const uintptr_t lo = reinterpret_cast<uintptr_t>(P.seg[s].rgb);
      const uintptr_t hi = lo + (uintptr_t)P.seg[s].count * (uintptr_t)sel.rgb_arity;
      uint64_t w;
      if (ca - off >= lo && ca - off + (off > 5u ? 16u : 8u) <= hi) {
        const unsigned long long* w8 = reinterpret_cast<const unsigned long long*>(ca - off);
        w = __ldg(w8) >> (8u * off);
        if (off > 5u) w |= __ldg(w8 + 1) << (8u * (8u - off));
      } else {
        w = (uint64_t)__ldg(c) | ((uint64_t)__ldg(c + 1) << 8) | ((uint64_t)__ldg(c + 2) << 16);
      }
      v.x = __fdiv_rn((float)(uint32_t)(w & 0xFFu), 255.0f);
      v.y = __fdiv_rn((float)(uint32_t)((w >> 8) & 0xFFu), 255.0f);
      v.z = __fdiv_rn((float)(uint32_t)((w >> 16) & 0xFFu), 255.0f);
      v.w = fminf(fmaxf(__fdiv_rn(P.near_f, dep), 0.0f), 1.0f);
    }
    *reinterpret_cast<float4*>(dst) = v;
    return;
  }
  if (s < 0) {  // empty, or (owner_only) won by another rank's points
    for (int c = 0; c < P.C; ++c) dst[c] = 0.0f;
    return;
  }
  const nar_segment& sg = P.seg[s];
  const int64_t row = idx - sg.begin;
  int col = 0;
  if (sel.rgb) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      dst[col++] = stream_value(sg.rgb, sel.rgb_format, sel.rgb_arity, row,
                                sel.rgb_arity == 1 ? 0 : c);
  }
  if (sel.depth) {
    // rasterizer.py:156-157 f32(near) / depth, clipped to [0, 1]
    dst[col++] = fminf(fmaxf(__fdiv_rn(P.near_f, dep), 0.0f), 1.0f);
  }
  if (sel.vel2d || sel.vel3d) {
    double v[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      v[c] = (double)stream_value(sg.velocity, sel.vel_format, sel.vel_arity, row, c);
    const double scale = sel.velocity_scale;
    if (sel.vel2d) {
      float vc[4];
      vel2d_channels(sg.positions + 3 * row, v, P.cam, scale, vc);
#pragma unroll
      for (int c = 0; c < 4; ++c) dst[col++] = vc[c];
    }
    if (sel.vel3d) {
      // velocity.py:17-23
      const double nrm = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
      dst[col++] = (float)(v[0] / scale);
      dst[col++] = (float)(v[1] / scale);
      dst[col++] = (float)(v[2] / scale);
      dst[col++] = (float)(nrm / scale);
    }
  }
  for (int q = 0; q < sel.n_scalars; ++q) {
    const int32_t ar = sel.scalar_arity[q];
    for (int c = 0; c < ar && col < P.C; ++c)
      dst[col++] = stream_value(sg.scalars[q], sel.scalar_format[q], ar, row, c);
  }
  if (sel.coverage_channel && col < P.C) dst[col++] = 1.0f;
}

// The RGB+D resolve of a local keybuf (no peers), kPix pixels per thread: the keybuf
// words of all its pixels are read first, then the winners' rgb words are gathered
// together (kPix independent random reads in flight per thread -- the gathers are
// what bounds the resolve), then the channels computed and stored.  Same results as
// resolve_kernel<kSigned, true>.  kVel: RGB+D+Vel2D (C = 8, f32 velocity of arity >= 3,
// C3's selection): the velocity and position of each winner are gathered in the same
// phase and the channels come from the general kernel's vel2d_channels.
template <bool kSigned, int kPix, bool kVel = false, bool kPixRgb = false>
__global__ void __launch_bounds__(256)
    resolve_rgbd_kernel(uint64_t* __restrict__ keybuf, const ResolveParams P) {
  const int32_t W = P.cam.w, H = P.cam.h;
  // output rows [row0, row1) (a rank's slice of the peer composite, else all)
  const int64_t base = (int64_t)P.row0 * P.data_w;
  const int64_t npix_out = base + (int64_t)(P.row1 - P.row0) * P.data_w;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t lid0 = base + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const uint64_t empty_raw = kSigned ? (NAR_EMPTY_KEY ^ NAR_SIGN_FLIP) : NAR_EMPTY_KEY;
  int64_t pix[kPix];
  uint64_t key[kPix];
  bool img[kPix];
#pragma unroll
  for (int j = 0; j < kPix; ++j) {
    const int64_t gid = lid0 + j * stride;
    const int32_t y = (int32_t)(gid / P.data_w);
    const int32_t x = (int32_t)(gid - (int64_t)y * P.data_w);
    img[j] = gid < npix_out && y < H && x < W;
    pix[j] = (int64_t)y * W + x;
    if (P.nkeys > 0) {  // composite: min over the ranks' keybufs (unsigned order), raw domain
      uint64_t m = NAR_EMPTY_KEY;
      if (img[j])
        for (int q = 0; q < P.nkeys; ++q) {
          uint64_t v = __ldcg(reinterpret_cast<const unsigned long long*>(P.keys[q]) + pix[j]);
          if (kSigned) v ^= NAR_SIGN_FLIP;
          m = v < m ? v : m;
        }
      key[j] = kSigned ? m ^ NAR_SIGN_FLIP : m;
    } else {
      key[j] = img[j] ? keybuf[pix[j]] : empty_raw;
    }
  }
  uint64_t wd[kPix];
  float dep[kPix];
  bool hit[kPix];
  float vel[kVel ? kPix : 1][3];
  const float* ppos[kVel ? kPix : 1];
#pragma unroll
  for (int j = 0; j < kPix; ++j) {
    if (img[j] && P.clear) {
      if (P.nkeys > 0)
        for (int q = 0; q < P.nkeys; ++q) const_cast<uint64_t*>(P.keys[q])[pix[j]] = empty_raw;
      else
        keybuf[pix[j]] = empty_raw;
    }
    const uint64_t k = kSigned ? key[j] ^ NAR_SIGN_FLIP : key[j];
    const bool covered = img[j] && k != NAR_EMPTY_KEY;
    const int64_t idx = covered ? (int64_t)(k & 0xFFFFFFFFull) : -1;
    dep[j] = covered ? __uint_as_float((uint32_t)(k >> 32)) : 0.0f;
    if (img[j]) {
      if (P.coverage) P.coverage[pix[j]] = covered ? 1 : 0;
      if (P.index_plane) P.index_plane[pix[j]] = idx;
      if (P.depth) P.depth[pix[j]] = dep[j];
    }
    int s = -1;
    if (covered)
      for (int q = 0; q < P.nseg; ++q)
        if (idx >= P.seg[q].begin && idx < P.seg[q].begin + P.seg[q].count) s = q;
    hit[j] = s >= 0;
    wd[j] = 0;
    if constexpr (kPixRgb) {
      if (s >= 0) wd[j] = __ldg(P.pix_rgb + pix[j]);
    } else if (s >= 0) {  // see resolve_kernel: aligned 8-byte words inside the stream's bytes
      const uint8_t* c = static_cast<const uint8_t*>(P.seg[s].rgb) + (idx - P.seg[s].begin) * P.sel.rgb_arity;
      const uintptr_t ca = reinterpret_cast<uintptr_t>(c);
      const uint32_t off = (uint32_t)(ca & 7u);
      const uintptr_t lo = reinterpret_cast<uintptr_t>(P.seg[s].rgb);
      const uintptr_t hi = lo + (uintptr_t)P.seg[s].count * (uintptr_t)P.sel.rgb_arity;
      if (ca - off >= lo && ca - off + (off > 5u ? 16u : 8u) <= hi) {
        const unsigned long long* w8 = reinterpret_cast<const unsigned long long*>(ca - off);
        uint64_t w = __ldg(w8) >> (8u * off);
        if (off > 5u) w |= __ldg(w8 + 1) << (8u * (8u - off));
        wd[j] = w;
      } else {
        wd[j] = (uint64_t)__ldg(c) | ((uint64_t)__ldg(c + 1) << 8) | ((uint64_t)__ldg(c + 2) << 16);
      }
      if constexpr (kVel) {
        const int64_t row = idx - P.seg[s].begin;
        const float* vp = static_cast<const float*>(P.seg[s].velocity) + row * P.sel.vel_arity;
#pragma unroll
        for (int c2 = 0; c2 < 3; ++c2) vel[j][c2] = __ldg(vp + c2);
        ppos[j] = P.seg[s].positions + 3 * row;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kPix; ++j) {
    const int64_t gid = lid0 + j * stride;
    if (gid >= npix_out) continue;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);  // padding and background: zeros
    float4 v2 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hit[j]) {
      v.x = __fdiv_rn((float)(uint32_t)(wd[j] & 0xFFu), 255.0f);
      v.y = __fdiv_rn((float)(uint32_t)((wd[j] >> 8) & 0xFFu), 255.0f);
      v.z = __fdiv_rn((float)(uint32_t)((wd[j] >> 16) & 0xFFu), 255.0f);
      v.w = fminf(fmaxf(__fdiv_rn(P.near_f, dep[j]), 0.0f), 1.0f);
      if constexpr (kVel) {
        const double vd[3] = {(double)vel[j][0], (double)vel[j][1], (double)vel[j][2]};
        float vc[4];
        vel2d_channels(ppos[j], vd, P.cam, P.sel.velocity_scale, vc);
        v2 = make_float4(vc[0], vc[1], vc[2], vc[3]);
      }
    }
    float4* d = reinterpret_cast<float4*>(P.data + gid * (kVel ? 8 : 4));
    d[0] = v;
    if constexpr (kVel) d[1] = v2;
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
static int g_num_sms = 0;
static std::once_flag g_init_once[kMaxDevices];  // kernel attributes are per device
static bool g_no_pre = false;  // NAR_RENDER_NO_PRETEST=1: exact-path-only Hi-Z passes

static int device_init() {
  int err = 0;
  const int cur = current_device();
  std::call_once(g_init_once[cur], [&]() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { err = 1; return; }
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(render_tma_kernel<false, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRenderSmem);
    cudaFuncSetAttribute(render_tma_kernel<true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRenderSmem);
    cudaFuncSetAttribute(render_tma_kernel<false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRenderSmem);
    cudaFuncSetAttribute(render_tma_kernel<true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRenderSmem);
    cudaFuncSetAttribute(render_tma_kernel<false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRenderSmem);
    cudaFuncSetAttribute(render_tma_kernel<true, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRenderSmem);
    for (auto k : {render_pre_kernel<false, 0, false>, render_pre_kernel<false, 1, false>,
                   render_pre_kernel<false, 2, false>, render_pre_kernel<true, 0, false>,
                   render_pre_kernel<true, 1, false>, render_pre_kernel<true, 2, false>,
                   render_pre_kernel<false, 0, true>, render_pre_kernel<false, 1, true>,
                   render_pre_kernel<false, 2, true>, render_pre_kernel<true, 0, true>,
                   render_pre_kernel<true, 1, true>, render_pre_kernel<true, 2, true>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kPreSmem);
    const char* np = getenv("NAR_RENDER_NO_PRETEST");
    g_no_pre = np && np[0] == '1';
  });
  if (err || g_num_sms == 0) return set_error(NAR_ERR_CUDA, "no CUDA device");
  return NAR_OK;
}

// Per-pass kernel choice from the previous frame's statistics.  The pre-test
// kernel wins where the coarse test rejects most points (volumetric clouds);
// where most points pass it (2.5-D clouds such as terrain scans) the exact
// kernel with pipelined early-z is faster (1.74 vs 2.39 ms at C4).  Every pass
// counts the points past its coarse test into device counters owned by the
// (Hi-Z scratch, point buffer) pair; at the end of a render they are copied to
// pinned memory, and the next render of the pair reads them (if the copy has
// landed) without any sync.  Pairs are independent, so concurrent renders of
// several point buffers on their own streams do not mix their counters.
struct PassState {
  unsigned long long* dev = nullptr;   // device counters
  unsigned long long* host = nullptr;  // pinned copy of the counters
  cudaEvent_t ev = nullptr;
  bool pending = false;
  int64_t pts[kPassStats] = {};        // points of each pass in the copied frame
  bool exact[kPassStats] = {};         // current choice per pass
  bool was_exact[kPassStats] = {};     // ... in the copied frame
  double win[kPassStats] = {-1, -1, -1, -1, -1, -1, -1, -1};  // last exact-pass win fraction
  uint32_t calls = 0;
  uint32_t reads = 0;  // statistics copies read (win fractions re-sampled every 8th)
};
static std::mutex g_pass_mu;
struct PassKeyHash {
  size_t operator()(const std::pair<const void*, const void*>& k) const {
    return std::hash<const void*>()(k.first) * 31u + std::hash<const void*>()(k.second);
  }
};
static std::unordered_map<std::pair<const void*, const void*>, PassState, PassKeyHash> g_pass;
static double g_dense_frac = -1.0;  // exact kernel above this survivor fraction
static double g_win_frac = -1.0;    // ... unless more than this share of its survivors won

static double dense_frac() {
  if (g_dense_frac < 0.0) {
    const char* e = getenv("NAR_RENDER_DENSE_FRAC");
    g_dense_frac = e ? atof(e) : 0.60;
  }
  return g_dense_frac;
}

static double win_frac() {
  if (g_win_frac < 0.0) {
    const char* e = getenv("NAR_RENDER_WIN_FRAC");
    g_win_frac = e ? atof(e) : 0.10;
  }
  return g_win_frac;
}

// Renders n points.  With a Hi-Z scratch (zmax), the aligned part is split
// into passes; before every pass but the first (and before the first too when
// `refresh_first`, i.e. the keybuf already holds this frame's keys) the coarse
// depth is rebuilt from the keybuf and the pass rejects points behind it.
static int launch_render(uint64_t* keybuf, const float* pos, int64_t n, uint64_t base,
                         const DevCam& cam, bool sgn, cudaStream_t st, uint16_t* zmax = nullptr,
                         bool refresh_first = false) {
  if (n <= 0) return NAR_OK;
  int rc = device_init();
  if (rc) return rc;
  int64_t done = 0;
  int shift = 3, zw = 1, zh = 1;
  hiz_geometry(cam.w, cam.h, shift, zw, zh);
  auto refresh = [&]() {
    const int64_t nt = ((int64_t)zw * zh) << shift;
    const unsigned g = (unsigned)((nt + 255) / 256);
    // vectorised row scans for 8/16/32-pixel blocks, scalar beyond
    auto k = sgn ? (shift == 3 ? hiz_kernel<true, 5> : shift == 4 ? hiz_kernel<true, 9>
                                                     : hiz_kernel<true, 17>)
                 : (shift == 3 ? hiz_kernel<false, 5> : shift == 4 ? hiz_kernel<false, 9>
                                                      : hiz_kernel<false, 17>);
    nar::count_launch();
    const char* hr = getenv("NAR_HIZ_ROWS");  // 0: the one-row-per-thread kernel (per render)
    const bool rows = !(hr && hr[0] == '0');
    if (rows && (cam.w & 1) == 0 && shift >= 3 && shift <= 5) {
      const int half = 1 << (shift - 1), nb = 255 / half;
      const dim3 grid((unsigned)((zw + nb - 1) / nb), (unsigned)zh);
      auto kr = sgn ? (shift == 3 ? hiz_rows_kernel<true, 8> : shift == 4 ? hiz_rows_kernel<true, 16>
                                                            : hiz_rows_kernel<true, 32>)
                    : (shift == 3 ? hiz_rows_kernel<false, 8> : shift == 4 ? hiz_rows_kernel<false, 16>
                                                             : hiz_rows_kernel<false, 32>);
      kr<<<grid, 256, 0, st>>>(keybuf, cam.w, cam.h, zw, zh, zmax);
      return;
    }
    k<<<g, 256, 0, st>>>(keybuf, cam.w, cam.h, shift, zw, zh, zmax);
  };
  if ((reinterpret_cast<uintptr_t>(pos) & 15) == 0) {
    const int64_t n_tiles = n / kTilePts;
    PassState* ps = nullptr;
    unsigned long long* dstats = nullptr;
    int64_t pass_pts[kPassStats] = {};
    bool exact_now[kPassStats] = {};
    if (n_tiles > 0 && zmax) {
      std::lock_guard<std::mutex> lk(g_pass_mu);
      const auto key = std::make_pair((const void*)zmax, (const void*)pos);
      auto it = g_pass.find(key);
      if (it == g_pass.end() && g_pass.size() < 256) {
        PassState st0;
        if (cudaMalloc(reinterpret_cast<void**>(&st0.dev), kStatCtrs * 8) != cudaSuccess ||
            cudaHostAlloc(reinterpret_cast<void**>(&st0.host), kStatCtrs * 8,
                          cudaHostAllocDefault) != cudaSuccess ||
            cudaEventCreateWithFlags(&st0.ev, cudaEventDisableTiming) != cudaSuccess)
          return set_error(NAR_ERR_NOMEM, "pass statistics");
        it = g_pass.emplace(key, st0).first;
      }
      if (it != g_pass.end()) ps = &it->second;
      if (ps && ps->pending && cudaEventQuery(ps->ev) == cudaSuccess) {
        static const bool verbose = getenv("NAR_RENDER_STATS") != nullptr;
        if (++ps->reads % 8 == 0)  // let passes that left the exact kernel re-measure it
          for (int p = 0; p < kPassStats; ++p) ps->win[p] = -1.0;
        for (int p = 0; p < kPassStats; ++p) {
          if (ps->pts[p] <= 0) continue;
          const double f = (double)ps->host[p] / (double)ps->pts[p];
          if (ps->was_exact[p] && ps->host[p] > 0)
            ps->win[p] = (double)ps->host[kPassStats + p] / (double)ps->host[p];
          // the exact kernel's early-z read pays where most survivors lose at their
          // pixel (dense 2.5-D clouds); where many still win, the pre-test kernel's
          // plain atomics are cheaper (measured on sparse shards, bench c5 / nar1b)
          ps->exact[p] = f > dense_frac() && !(ps->win[p] > win_frac());
          if (verbose)
            fprintf(stderr, "nar pass %d: %.4f of %lld points past the coarse test, win %.4f%s\n",
                    p, f, (long long)ps->pts[p], ps->win[p], ps->was_exact[p] ? " (exact)" : "");
        }
        ps->pending = false;
      }
      if (ps) {
        for (int p = 0; p < kPassStats; ++p) exact_now[p] = ps->exact[p];
        // the first renders, then one in 16, collect statistics (the seed pass
        // zeroes the counters, the copy back is amortised); the second measures
        // the win fractions of the passes the first moved to the exact kernel
        const uint32_t call = ps->calls++;
        if ((call < 4 || call % 16 == 0) && !ps->pending) dstats = ps->dev;
      }
    }
    if (n_tiles > 0) {
      const int64_t sms = g_num_sms;
      auto kern = sgn ? render_tma_kernel<true, false> : render_tma_kernel<false, false>;
      auto kseed = sgn ? render_tma_kernel<true, true> : render_tma_kernel<false, true>;
      auto kern_st = sgn ? render_tma_kernel<true, false, true> : render_tma_kernel<false, false, true>;
      decltype(&render_pre_kernel<false, 0, false>) kpres[2][2][3] = {
          {{render_pre_kernel<false, 0, false>, render_pre_kernel<false, 1, false>,
            render_pre_kernel<false, 2, false>},
           {render_pre_kernel<false, 0, true>, render_pre_kernel<false, 1, true>,
            render_pre_kernel<false, 2, true>}},
          {{render_pre_kernel<true, 0, false>, render_pre_kernel<true, 1, false>,
            render_pre_kernel<true, 2, false>},
           {render_pre_kernel<true, 0, true>, render_pre_kernel<true, 1, true>,
            render_pre_kernel<true, 2, true>}}};
      const bool pre = cam.pre && !g_no_pre;
      int pass_no = 0;
      auto run = [&](ChunkMap cm, bool with_hiz) {
        const int pno = pass_no++;
        HizArgs hz{nullptr, shift, zw, zw * zh, zh, nullptr, nullptr};
        if (dstats && pno == 0) hz.stats_clear = dstats;  // the seed pass (never counted)
        if (dstats && pno > 0 && pno < kPassStats) {
          hz.stats = dstats + pno;
          pass_pts[pno] = (cm.j1 - cm.j0) * kUnitPts;
        }
        if (with_hiz) {
          refresh();
          hz.zmax = zmax;
        }
        const int64_t nj = cm.j1 - cm.j0;
        const int64_t need = (nj + kRenderWarps - 1) / kRenderWarps;
        const int grid = (int)(need < sms ? need : sms);
        if (grid <= 0) return;
        // a pass right after its Hi-Z refresh is a programmatic dependent of it: its
        // CTAs start their point streams while the refresh drains (NAR_RENDER_PDL=0: off)
        static const bool pdl_on = [] {
          const char* e = getenv("NAR_RENDER_PDL");
          return !(e && e[0] == '0');
        }();
        cudaLaunchAttribute pattr[1];
        pattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        pattr[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)grid);
        lc.blockDim = dim3(kRenderThreads);
        lc.stream = st;
        lc.attrs = pattr;
        lc.numAttrs = (with_hiz && pdl_on) ? 1 : 0;
        if (with_hiz && pre && !(pno < kPassStats && exact_now[pno])) {
          nar::count_launch();
          lc.dynamicSmemBytes = kPreSmem;
          cudaLaunchKernelEx(&lc, kpres[sgn ? 1 : 0][hz.stats ? 1 : 0][cm.mode], keybuf, pos, cm,
                             base, cam, hz);
        } else if (with_hiz && !(cm.mode == 1 && pre)) {
          nar::count_launch();
          lc.dynamicSmemBytes = kRenderSmem;
          cudaLaunchKernelEx(&lc, hz.stats ? kern_st : kern, keybuf, pos, cm, base, cam, hz);
        } else if (cm.mode == 1 && pre) {  // seed units: the direct path of the pre kernel
          nar::count_launch();
          kpres[sgn ? 1 : 0][0][1]<<<grid, kRenderThreads, kPreSmem, st>>>(keybuf, pos, cm, base,
                                                                          cam, hz);
        } else if (cm.mode == 1 && !with_hiz) {
          nar::count_launch();
          kseed<<<grid, kRenderThreads, kRenderSmem, st>>>(keybuf, pos, cm, base, cam, hz);
        } else {
          nar::count_launch();
          (hz.stats ? kern_st : kern)<<<grid, kRenderThreads, kRenderSmem, st>>>(keybuf, pos, cm, base,
                                                                               cam, hz);
        }
      };
      // Hi-Z schedule: a seed pass over every S-th chunk (spread over the whole
      // cloud, so the coarse depth covers the screen even for spatially sorted
      // input), then the remaining chunks in passes, each after a refresh.
      const int64_t S = kHizSeedStride;
      // ~16 units per warp per pass; NAR_RENDER_PASS_UNITS overrides (tests force
      // the multi-pass schedule on small clouds with it)
      int64_t min_pass = sms * kRenderWarps * 16;
      if (const char* e = getenv("NAR_RENDER_PASS_UNITS")) {
        const long long v = atoll(e);
        if (v > 0) min_pass = v;
      }
      if (zmax && n_tiles >= S * min_pass / 4) {
        const int64_t n_seed = (n_tiles + S - 1) / S;
        run(ChunkMap{0, n_seed, 1, 1, 0, 0}, refresh_first);
        const int64_t n_rest = n_tiles - n_seed;
        int64_t passes = n_rest / min_pass;
        int64_t max_passes = 4;
        if (const char* e = getenv("NAR_RENDER_MAX_PASSES")) {
          const long long v = atoll(e);
          if (v > 0) max_passes = v;
        }
        passes = passes < 1 ? 1 : (passes > max_passes ? max_passes : passes);
        // pass sizes grow 1, 2, 4, then stay at 4 (x the first): the early,
        // loosely culled passes are short and refresh the coarse depth sooner
        int geo = 1;
        if (const char* e = getenv("NAR_RENDER_GEO")) geo = atoi(e);
        int64_t wsum = 0, wt[64];
        for (int64_t p = 0; p < passes && p < 64; ++p) {
          wt[p] = geo ? ((int64_t)1 << (p < 2 ? p : 2)) : 1;
          wsum += wt[p];
        }
        // pass p takes the residues [acc, acc + wt[p]) mod wsum of the remaining units,
        // in blocks of kB consecutive units (contiguous DRAM runs of kB * 1.5 KB)
        const int64_t kB = 8;
        const int64_t period = wsum * kB;
        int64_t acc = 0;
        for (int64_t p = 0; p < passes && p < 64; ++p) {
          uint32_t ls = 3;  // log2(kB)
          while ((int64_t)1 << (ls + 1) <= wt[p] * kB) ++ls;
          const int64_t len = (int64_t)1 << ls;  // weights are powers of two
          const int64_t rem = n_rest % period;
          const int64_t part = rem - acc < 0 ? 0 : (rem - acc > len ? len : rem - acc);
          const int64_t slots = (n_rest / period) * len + part;
          run(ChunkMap{0, slots, 2, (uint32_t)period, (uint32_t)acc, ls}, true);
          acc += len;
        }
      } else {
        run(ChunkMap{0, n_tiles, 0, 1, 0, 0}, zmax && refresh_first);
      }
      done = n_tiles * kTilePts;
      if (ps && dstats && pass_no > 1) {  // hand the counters to later renders (no sync)
        std::lock_guard<std::mutex> lk(g_pass_mu);
        if (!ps->pending) {
          cudaMemcpyAsync(ps->host, dstats, kStatCtrs * 8, cudaMemcpyDeviceToHost, st);
          cudaEventRecord(ps->ev, st);
          for (int p = 0; p < kPassStats; ++p) {
            ps->pts[p] = pass_pts[p];
            ps->was_exact[p] = exact_now[p];
          }
          ps->pending = true;
        }
      }
    }
  }
  const int64_t rest = n - done;
  if (rest > 0) {
    int64_t blocks = (rest + 255) / 256;
    const int64_t cap = (int64_t)(g_num_sms > 0 ? g_num_sms : 148) * 8;
    if (blocks > cap) blocks = cap;
    if (sgn) {
      nar::count_launch();
      render_simple_kernel<true><<<(int)blocks, 256, 0, st>>>(keybuf, pos + 3 * done, rest,
                                                             base + (uint64_t)done, cam);
    } else {
      nar::count_launch();
      render_simple_kernel<false><<<(int)blocks, 256, 0, st>>>(keybuf, pos + 3 * done, rest,
                                                              base + (uint64_t)done, cam);
    }
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

// Host-buffer render: points stream through two device staging buffers on a
// copy stream while the previous chunk renders (copy/compute overlap).  The
// staging buffers, copy stream, events and Hi-Z scratch persist across calls
// (one set per process, grown on demand) so a frame-rate caller pays no
// allocation; the `done` events carry over, so a call never overwrites a
// buffer an earlier call's render is still reading.
struct HostPath {
  std::mutex mu;
  float* buf[2] = {nullptr, nullptr};
  int64_t cap = 0;  // points per buffer
  uint16_t* zmax = nullptr;
  cudaStream_t cp = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
};
static HostPath g_host[kMaxDevices];  // staging + Hi-Z scratch of each device

static int host_path_reserve(HostPath& h, int64_t chunk) {
  if (!h.cp) {
    if (cudaStreamCreateWithFlags(&h.cp, cudaStreamNonBlocking) != cudaSuccess)
      return set_error(NAR_ERR_CUDA, "stream creation failed");
    for (int b = 0; b < 2; ++b) {
      cudaEventCreateWithFlags(&h.copied[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&h.done[b], cudaEventDisableTiming);
      cudaEventRecord(h.done[b], h.cp);
    }
    if (cudaMalloc(reinterpret_cast<void**>(&h.zmax), (size_t)kHizMaxEntries * 2) != cudaSuccess)
      return set_error(NAR_ERR_NOMEM, "cudaMalloc of Hi-Z scratch failed");
  }
  if (chunk > h.cap) {
    for (int b = 0; b < 2; ++b) {
      cudaEventSynchronize(h.done[b]);
      if (h.buf[b]) cudaFree(h.buf[b]);
      h.buf[b] = nullptr;
    }
    h.cap = 0;
    for (int b = 0; b < 2; ++b)
      if (cudaMalloc(reinterpret_cast<void**>(&h.buf[b]), (size_t)chunk * 12) != cudaSuccess)
        return set_error(NAR_ERR_NOMEM, "cudaMalloc of point staging failed");
    h.cap = chunk;
  }
  return NAR_OK;
}

static int render_host_impl(uint64_t* keybuf_dev, const float* pos_host, int64_t n,
                            uint64_t base, const DevCam& cam, bool sgn, cudaStream_t st) {
  if (n <= 0) return NAR_OK;
  const int64_t kChunk = (int64_t)1 << 23;  // 8 Mi points = 96 MiB per buffer
  const int64_t chunk = n < kChunk ? ((n + kTilePts - 1) / kTilePts) * kTilePts : kChunk;
  HostPath& h = g_host[current_device()];
  std::lock_guard<std::mutex> lock(h.mu);
  int rc = host_path_reserve(h, chunk);
  if (rc) return rc;
  // calls on different streams share the staging and Hi-Z scratch: order
  // this call's work after the previous call's renders
  cudaStreamWaitEvent(st, h.done[0], 0);
  cudaStreamWaitEvent(st, h.done[1], 0);
  // the copy stream starts after everything already queued on `st`
  cudaEvent_t start = h.copied[0];
  cudaEventRecord(start, st);
  cudaStreamWaitEvent(h.cp, start, 0);
  for (int64_t off = 0, k = 0; off < n && !rc; off += chunk, ++k) {
    const int b = (int)(k & 1);
    const int64_t cnt = (n - off) < chunk ? (n - off) : chunk;
    cudaStreamWaitEvent(h.cp, h.done[b], 0);
    if (cudaMemcpyAsync(h.buf[b], pos_host + 3 * off, (size_t)cnt * 12, cudaMemcpyHostToDevice,
                        h.cp) != cudaSuccess) {
      rc = set_error(NAR_ERR_CUDA, "H2D copy of points failed");
      break;
    }
    cudaEventRecord(h.copied[b], h.cp);
    cudaStreamWaitEvent(st, h.copied[b], 0);
    // chunk k > 0 is tested against the coarse depth of chunks 0..k-1
    rc = launch_render(keybuf_dev, h.buf[b], cnt, base + (uint64_t)off, cam, sgn, st,
                       n > chunk ? h.zmax : nullptr, k > 0);
    cudaEventRecord(h.done[b], st);
  }
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
  nar::count_launch();
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

int nar_hiz_scratch_bytes(int32_t width, int32_t height, size_t* bytes) {
  if (!bytes || width <= 0 || height <= 0) return set_error(NAR_ERR_INVALID, "bad arguments");
  int shift, zw, zh;
  hiz_geometry(width, height, shift, zw, zh);
  *bytes = (size_t)kHizMaxEntries * 2;
  return NAR_OK;
}

int nar_render_hiz(uint64_t* keybuf_dev, uint16_t* hiz_scratch_dev, const float* positions_dev,
                   int64_t n, uint64_t base_index, const nar_camera* cam, int32_t key_domain,
                   int32_t keybuf_has_frame, void* stream) {
  int rc = validate_camera(cam);
  if (rc) return rc;
  if (n < 0) return set_error(NAR_ERR_INVALID, "negative point count");
  if (n > 0 && (!keybuf_dev || !positions_dev || !hiz_scratch_dev))
    return set_error(NAR_ERR_INVALID, "NULL buffer");
  return launch_render(keybuf_dev, positions_dev, n, base_index, make_devcam(*cam),
                       key_domain == NAR_KEYS_SIGNED, (cudaStream_t)stream, hiz_scratch_dev,
                       keybuf_has_frame != 0);
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
  nar::keep_pool_memory();
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

static int resolve_impl(uint64_t* keybuf_dev, const uint64_t* const* peers, int32_t n_peers,
                        int32_t row_begin, int32_t row_end, const nar_camera* cam,
                        int32_t key_domain, const nar_selection* sel,
                        const nar_segment* segments, int32_t n_segments,
                        const nar_resolve_out* out, void* stream,
                        const uint32_t* pix_rgb = nullptr) {
  int rc = validate_camera(cam);
  if (rc) return rc;
  if ((!keybuf_dev && n_peers <= 0) || !sel || !out)
    return set_error(NAR_ERR_INVALID, "NULL argument");
  if (n_peers < 0 || n_peers > NAR_MAX_SEGMENTS)
    return set_error(NAR_ERR_INVALID, "1..8 keybufs for a composite resolve");
  for (int k = 0; k < n_peers; ++k)
    if (!peers[k]) return set_error(NAR_ERR_INVALID, "NULL peer keybuf");
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
  P.nkeys = n_peers;
  for (int k = 0; k < n_peers; ++k) P.keys[k] = peers[k];
  P.row0 = row_begin < 0 ? 0 : row_begin;
  P.row1 = (row_end < 0 || row_end > P.data_h) ? P.data_h : row_end;
  if (P.row1 < P.row0) return set_error(NAR_ERR_INVALID, "empty row range");
  const int64_t n_out = (int64_t)(P.row1 - P.row0) * P.data_w;
  if (n_out == 0) return NAR_OK;
  const int64_t blocks = (n_out + 255) / 256;
  const bool rgbd = C == 4 && sel->rgb && sel->depth && sel->rgb_format == NAR_FMT_U8 &&
                    sel->rgb_arity >= 3 && (reinterpret_cast<uintptr_t>(out->data) & 15) == 0;
  // RGB+D of a local keybuf: several pixels per thread (NAR_RESOLVE_PIX, default 4)
  static const int kpix = [] {
    const char* e = getenv("NAR_RESOLVE_PIX");
    const int v = e ? atoi(e) : 4;
    return v == 1 || v == 2 || v == 8 ? v : 4;
  }();
  // RGB+D+Vel2D (C3's selection): the same kernel with the velocity gathers (2 pixels)
  const bool rgbdv = C == 8 && sel->rgb && sel->depth && sel->vel2d && !sel->vel3d &&
                     !sel->coverage_channel && sel->n_scalars == 0 &&
                     sel->rgb_format == NAR_FMT_U8 && sel->rgb_arity >= 3 &&
                     sel->vel_format == NAR_FMT_F32 && sel->vel_arity >= 3 &&
                     (reinterpret_cast<uintptr_t>(out->data) & 15) == 0;
  if (pix_rgb) {  // rgb already gathered per pixel on the host (nar_host_gather_rgb)
    if (!(rgbd && P.data && n_peers == 0))
      return set_error(NAR_ERR_CONFIG, "per-pixel rgb needs an RGB+D (u8 rgb) local resolve");
    P.pix_rgb = pix_rgb;
    const bool sg = key_domain == NAR_KEYS_SIGNED;
    const int kp = n_out < (1 << 20) ? 2 : 4;
    auto k = kp == 2 ? (sg ? resolve_rgbd_kernel<true, 2, false, true> : resolve_rgbd_kernel<false, 2, false, true>)
                     : (sg ? resolve_rgbd_kernel<true, 4, false, true> : resolve_rgbd_kernel<false, 4, false, true>);
    const int64_t b = (n_out + 256 * kp - 1) / (256 * kp);
    nar::count_launch();
    k<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(keybuf_dev, P);
    return check_launch("resolve");
  }
  if (rgbdv && out->data && kpix > 1) {
    auto k = key_domain == NAR_KEYS_SIGNED ? resolve_rgbd_kernel<true, 2, true>
                                           : resolve_rgbd_kernel<false, 2, true>;
    const int64_t b = (n_out + 511) / 512;
    nar::count_launch();
    k<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(keybuf_dev, P);
    return check_launch("resolve");
  }
  if (rgbd && P.data && kpix > 1) {
    const bool sg = key_domain == NAR_KEYS_SIGNED;
    // small frames (< 1 Mpixel) have too few threads to fill the GPU at 4 pixels each
    const int kp = n_out < (1 << 20) && kpix > 2 ? 2 : kpix;
    auto k = kp == 2 ? (sg ? resolve_rgbd_kernel<true, 2> : resolve_rgbd_kernel<false, 2>)
           : kp == 8 ? (sg ? resolve_rgbd_kernel<true, 8> : resolve_rgbd_kernel<false, 8>)
                     : (sg ? resolve_rgbd_kernel<true, 4> : resolve_rgbd_kernel<false, 4>);
    const int64_t b = (n_out + 256 * kp - 1) / (256 * kp);
    nar::count_launch();
    k<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(keybuf_dev, P);
    return check_launch("resolve");
  }
  auto kern = key_domain == NAR_KEYS_SIGNED
                  ? (rgbd ? resolve_kernel<true, true> : resolve_kernel<true, false>)
                  : (rgbd ? resolve_kernel<false, true> : resolve_kernel<false, false>);
  nar::count_launch();
  kern<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(keybuf_dev, P);
  return check_launch("resolve");
}

int nar_resolve(uint64_t* keybuf_dev, const nar_camera* cam, int32_t key_domain,
                const nar_selection* sel, const nar_segment* segments, int32_t n_segments,
                const nar_resolve_out* out, void* stream) {
  return resolve_impl(keybuf_dev, nullptr, 0, 0, -1, cam, key_domain, sel, segments, n_segments,
                      out, stream);
}

int nar_resolve_pixrgb(uint64_t* keybuf_dev, int32_t row_begin, int32_t row_end,
                       const nar_camera* cam, int32_t key_domain, const nar_selection* sel,
                       const nar_segment* segments, int32_t n_segments, const nar_resolve_out* out,
                       const uint32_t* pix_rgb_dev, void* stream) {
  if (!pix_rgb_dev) return set_error(NAR_ERR_INVALID, "NULL per-pixel rgb");
  return resolve_impl(keybuf_dev, nullptr, 0, row_begin, row_end, cam, key_domain, sel, segments,
                      n_segments, out, stream, pix_rgb_dev);
}

// Host side of the gather: one pass over the frame's keys on a persistent pool of
// host threads, software-prefetching the rgb bytes of the winner 16 pixels ahead
// (2M random reads of a 1 GB array: ~1.6 ms on 16 cores vs ~4.7 ms as zero-copy
// PCIe reads from the resolve kernel).
int nar_host_gather_rgb(const uint64_t* keys, int64_t npix, int32_t key_domain,
                        const uint8_t* rgb, int32_t arity, uint64_t begin, int64_t count,
                        uint32_t* out) {
  if (!keys || !out || (count > 0 && !rgb) || npix < 0 || count < 0 || arity < 3)
    return set_error(NAR_ERR_INVALID, "bad host gather arguments");
  const uint64_t flip = key_domain == NAR_KEYS_SIGNED ? NAR_SIGN_FLIP : 0ull;
  nar::host_parallel_for(npix, [&](int64_t b, int64_t e) {
    constexpr int64_t D = 16;
    auto src = [&](int64_t p) -> const uint8_t* {
      const uint64_t k = keys[p] ^ flip;
      if (k == NAR_EMPTY_KEY) return nullptr;
      const uint64_t idx = k & 0xFFFFFFFFull;
      if (idx < begin || idx - begin >= (uint64_t)count) return nullptr;
      return rgb + (idx - begin) * (uint64_t)arity;
    };
    for (int64_t p = b; p < e; ++p) {
      if (p + D < e) {
        const uint8_t* f = src(p + D);
        if (f) __builtin_prefetch(f);
      }
      const uint8_t* c = src(p);
      out[p] = c ? (uint32_t)c[0] | ((uint32_t)c[1] << 8) | ((uint32_t)c[2] << 16) : 0u;
    }
  });
  return NAR_OK;
}

int nar_resolve_peers(const uint64_t* const* keybufs, int32_t n_keybufs, int32_t row_begin,
                      int32_t row_end, const nar_camera* cam, int32_t key_domain,
                      const nar_selection* sel, const nar_segment* segments, int32_t n_segments,
                      const nar_resolve_out* out, void* stream) {
  if (!keybufs || n_keybufs < 1) return set_error(NAR_ERR_INVALID, "no keybufs");
  return resolve_impl(nullptr, keybufs, n_keybufs, row_begin, row_end, cam, key_domain, sel,
                      segments, n_segments, out, stream);
}

}  // extern "C"
