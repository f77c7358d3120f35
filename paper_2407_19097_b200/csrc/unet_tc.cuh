// unet_tc.cuh -- tcgen05 / TMEM implicit-GEMM gated 3x3 convolution (sm_100a).
//
// One launch computes  out = elu(conv(x, Wf) + bf) * sigmoid(conv(x, Wg) + bg)
// (model.py:158-163) for x = concat(srcA or up2(srcA), srcB) with zero "same"
// padding (autodiff.py:267-288), as a GEMM with
//   M = pixels (tiles of R image rows x 128 pixels),  N = 2*Coutp (f | g),
//   K = 9 taps x input channels (16-channel chunks).
//
// CTA roles (288 threads, 1 CTA per SM, persistent over tiles):
//   warps 0-3  producer: per (tile, 16-channel chunk) stage, cp.async gathers
//              the (R+2) x 130 pixel halo of the chunk into shared memory in
//              the UMMA no-swizzle K-major layout [row][k8][px][16 B] (zero
//              fill for padding, address math for concat / up2); thread 0
//              streams the chunk's pre-packed weights with a TMA bulk copy.
//   warp 8     MMA issuer (one elected thread) + TMEM owner: for each of the
//              9 taps and R rows one tcgen05.mma (M=128, N, K=16) whose A
//              descriptor is the halo row shifted by the tap (a 16-byte start
//              address offset: pixels are contiguous 16 B rows, SBO = 128 B).
//   warps 4-7  epilogue: tcgen05.ld the f and g accumulators of their TMEM
//              lane quarter, apply the gate, store bf16 NHWC.
// Accumulators are double buffered in TMEM (2 x R x N <= 512 columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace nar {

struct ConvArgs {
  const __nv_bfloat16* src_a;  // NHWC, channel stride ca_stride (multiple of 16)
  const __nv_bfloat16* src_b;  // NHWC, channel stride cb_stride, or NULL
  int ca, cb, ca_stride, cb_stride, a_up2;
  int H, W;                    // output (and src_b) resolution
  int cout, cout_stride;       // real output channels, output channel stride
  const float* wf32;           // SIMT path: HWIO f32
  const float* wg32;
  const float* bias_f;
  const float* bias_g;
  const __nv_bfloat16* wtc;    // tcgen05 path: packed (see tc_pack_weights)
  __nv_bfloat16* out;
};

constexpr int kTcThreads = 288;
constexpr int kHaloPx = 130;
constexpr int kHaloRowBytes = 2 * kHaloPx * 16;  // two 8-channel slabs

__host__ __device__ constexpr int tc_rows(int N) { return N >= 256 ? 1 : (256 / N > 8 ? 8 : 256 / N); }
__host__ __device__ constexpr int tc_a_bytes(int N) { return (tc_rows(N) + 2) * kHaloRowBytes; }
__host__ __device__ constexpr int tc_b_bytes(int N) { return 9 * N * 32; }
__host__ __device__ constexpr int tc_stage_bytes(int N) { return tc_a_bytes(N) + tc_b_bytes(N); }
__host__ __device__ constexpr int tc_stages(int N) {
  return (200 * 1024) / tc_stage_bytes(N) > 4 ? 4 : (200 * 1024) / tc_stage_bytes(N);
}
__host__ __device__ constexpr int tc_smem(int N) { return tc_stages(N) * tc_stage_bytes(N) + 256; }

// Host: pack HWIO f32 weights into bf16 [chunk q][tap][k8][n][8] where
// n < Coutp indexes f outputs and n >= Coutp g outputs (zero padded).
inline void tc_pack_weights(const std::vector<float>& wf, const std::vector<float>& wg, int ca,
                            int cb, int cout, std::vector<uint16_t>& packed) {
  const int coutp = (cout + 7) / 8 * 8, N = 2 * coutp;
  const int nqa = (ca + 15) / 16, nqb = (cb + 15) / 16, nq = nqa + nqb, cin = ca + cb;
  packed.assign((size_t)nq * 9 * 2 * N * 8, 0);
  auto bf16 = [](float v) -> uint16_t {
    uint32_t u;
    memcpy(&u, &v, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
    return (uint16_t)(u >> 16);
  };
  for (int q = 0; q < nq; ++q)
    for (int tap = 0; tap < 9; ++tap)
      for (int k8 = 0; k8 < 2; ++k8)
        for (int n = 0; n < N; ++n)
          for (int e = 0; e < 8; ++e) {
            const int cl = 16 * (q < nqa ? q : q - nqa) + 8 * k8 + e;  // channel within source
            const bool in_a = q < nqa;
            if ((in_a && cl >= ca) || (!in_a && cl >= cb)) continue;
            const int ci = in_a ? cl : ca + cl;
            const bool is_g = n >= coutp;
            const int j = is_g ? n - coutp : n;
            if (j >= cout) continue;
            const float v = (is_g ? wg : wf)[((size_t)tap * cin + ci) * cout + j];
            packed[((((size_t)q * 9 + tap) * 2 + k8) * N + n) * 8 + e] = bf16(v);
          }
}

// ---------------------------------------------------------------------------
// device helpers (tcgen05 / TMEM / cp.async)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SWIZZLE_NONE K-major: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
  // version 1 at [46,48), layout type 0 at [61,64).
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  // c_format F32 (1) at [4,6); a/b BF16 (1) at [7,10) / [10,13); K-major both;
  // N>>3 at [17,23); M>>4 at [24,29).
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float gate(float f, float g) {
  const float e = f > 0.0f ? f : __expf(f) - 1.0f;        // elu (autodiff.py:186-194)
  const float s = fmaf(0.5f, tanh_approx(0.5f * g), 0.5f); // sigmoid (autodiff.py:197-203)
  return e * s;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(kTcThreads, 1) gated_conv_tc(const ConvArgs a) {
  constexpr int R = tc_rows(N);
  constexpr int S = tc_stages(N);
  constexpr int A_BYTES = tc_a_bytes(N);
  constexpr int B_BYTES = tc_b_bytes(N);
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int COUTP = N / 2;
  constexpr uint32_t IDESC = umma_idesc_bf16(128, N);
  static_assert(2 * R * N <= 512, "TMEM budget");

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tbase_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_x = (a.W + 127) / 128;
  const int tiles_y = (a.H + R - 1) / R;
  const int n_tiles = tiles_x * tiles_y;
  const int nqa = (a.ca + 15) / 16, nqb = (a.cb + 15) / 16, nq = nqa + nqb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 129);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tbase_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_slot;

  if (warp < 4) {
    // ------------------------------ producer ------------------------------
    const int t = threadIdx.x;
    int it = 0;
    int pending = -1;  // stage whose cp.async group is still in flight
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int y0 = (tile / tiles_x) * R, x0 = (tile % tiles_x) * 128;
      for (int q = 0; q < nq; ++q, ++it) {
        const int s = it % S;
        const uint32_t ph = (uint32_t)(it / S) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* stA = smem + s * STAGE;
        if (t == 0) {
          mbar_expect_tx(&full[s], B_BYTES);
          bulk_g2s(stA + A_BYTES, a.wtc + (size_t)q * (B_BYTES / 2), B_BYTES, &full[s]);
        }
        const bool in_a = q < nqa;
        const __nv_bfloat16* src = in_a ? a.src_a : a.src_b;
        const int cst = in_a ? a.ca_stride : a.cb_stride;
        const int cbase = 16 * (in_a ? q : q - nqa);
        const bool up2 = in_a && a.a_up2;
        const int ws = up2 ? a.W / 2 : a.W;
        const uint32_t dst0 = smem_u32(stA);
        constexpr int ITEMS = (R + 2) * kHaloPx * 2;
        for (int i = t; i < ITEMS; i += 128) {
          const int k8 = i & 1;
          const int j = (i >> 1) % kHaloPx;
          const int row = (i >> 1) / kHaloPx;
          const int y = y0 - 1 + row, x = x0 - 1 + j;
          const bool ok = y >= 0 && y < a.H && x >= 0 && x < a.W;
          const int ys = up2 ? (y >> 1) : y, xs = up2 ? (x >> 1) : x;
          const __nv_bfloat16* g =
              src + ((size_t)(ok ? ys : 0) * ws + (ok ? xs : 0)) * cst + cbase + 8 * k8;
          cp_async16(dst0 + row * kHaloRowBytes + k8 * (kHaloPx * 16) + j * 16, g, ok);
        }
        cp_async_commit();
        if (pending >= 0) {
          cp_async_wait<1>();
          fence_proxy_async();
          mbar_arrive(&full[pending]);
        }
        pending = s;
      }
    }
    if (pending >= 0) {
      cp_async_wait<0>();
      fence_proxy_async();
      mbar_arrive(&full[pending]);
    }
  } else if (warp == 8) {
    // ------------------------------ MMA issuer -----------------------------
    int it = 0, tl = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tl) {
      const int b = tl & 1;
      mbar_wait(&tempty[b], (((uint32_t)tl >> 1) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t dcol = tbase + (uint32_t)(b * R * N);
      for (int q = 0; q < nq; ++q, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (uint32_t)(it / S) & 1u);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + s * STAGE);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll 1
          for (int tap = 0; tap < 9; ++tap) {
            const int ky = tap / 3, kx = tap % 3;
            const uint64_t bdesc = umma_desc(sb + tap * (N * 32), N * 16, 128);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const uint64_t adesc =
                  umma_desc(sa + (r + ky) * kHaloRowBytes + kx * 16, kHaloPx * 16, 128);
              umma_bf16(dcol + r * N, adesc, bdesc, IDESC, (q > 0 || tap > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
          if (q == nq - 1) umma_commit(&tfull[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------ epilogue -------------------------------
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const int m = quarter * 32 + lane;
    int tl = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tl) {
      const int b = tl & 1;
      const int y0 = (tile / tiles_x) * R, x0 = (tile % tiles_x) * 128;
      mbar_wait(&tfull[b], ((uint32_t)tl >> 1) & 1u);
      tc_fence_after();
      const int x = x0 + m;
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        const uint32_t col = tbase + (uint32_t)(b * R * N + r * N) + ((uint32_t)(quarter * 32) << 16);
        __nv_bfloat16* dst = a.out + ((size_t)y * a.W + x) * a.cout_stride;
        const bool ok = y < a.H && x < a.W;
#pragma unroll 1
        for (int c8 = 0; c8 < a.cout_stride / 8; ++c8) {
          float f[8], g[8];
          if (c8 * 8 < COUTP) {
            tmem_ld8(col + c8 * 8, f);
            tmem_ld8(col + COUTP + c8 * 8, g);
            tmem_wait_ld();
          }
          uint4 pk;
          uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const int j = c8 * 8 + e;
            float o0 = 0.0f, o1 = 0.0f;
            if (j < a.cout) o0 = gate(f[e] + __ldg(a.bias_f + j), g[e] + __ldg(a.bias_g + j));
            if (j + 1 < a.cout)
              o1 = gate(f[e + 1] + __ldg(a.bias_f + j + 1), g[e + 1] + __ldg(a.bias_g + j + 1));
            __nv_bfloat162 h = __floats2bfloat162_rn(o0, o1);
            pw[e / 2] = *reinterpret_cast<uint32_t*>(&h);
          }
          if (ok) *reinterpret_cast<uint4*>(dst + c8 * 8) = pk;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase)
                 : "memory");
  }
}

template <int N>
static int tc_launch_n(const ConvArgs& a, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    if (cudaFuncSetAttribute(gated_conv_tc<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             tc_smem(N)) != cudaSuccess)
      return set_error(NAR_ERR_CUDA, "cannot set conv smem size");
    attr_done = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int R = tc_rows(N);
  const int tiles = ((a.W + 127) / 128) * ((a.H + R - 1) / R);
  const int grid = tiles < sms ? tiles : sms;
  gated_conv_tc<N><<<grid, kTcThreads, tc_smem(N), st>>>(a);
  return check_launch("gated_conv_tc");
}

inline int tc_launch_gated_conv(const ConvArgs& a, cudaStream_t st) {
  const int coutp = (a.cout + 7) / 8 * 8;
  if (a.cout_stride % 8 || a.cout_stride < coutp)
    return set_error(NAR_ERR_CONFIG, "conv output stride must be a multiple of 8 >= Coutp");
  if (a.ca_stride % 16 || (a.cb && a.cb_stride % 16))
    return set_error(NAR_ERR_CONFIG, "conv input strides must be multiples of 16");
  switch (2 * coutp) {
    case 16: return tc_launch_n<16>(a, st);
    case 32: return tc_launch_n<32>(a, st);
    case 48: return tc_launch_n<48>(a, st);
    case 64: return tc_launch_n<64>(a, st);
    case 96: return tc_launch_n<96>(a, st);
    case 128: return tc_launch_n<128>(a, st);
    case 192: return tc_launch_n<192>(a, st);
    case 256: return tc_launch_n<256>(a, st);
    default: return set_error(NAR_ERR_CONFIG, "unsupported conv width");
  }
}

}  // namespace nar
