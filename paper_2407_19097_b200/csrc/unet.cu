// unet.cu -- gated U-Net forward (pkg/src/nar/neural/model.py:135-204) on B200.
//
// Plan (all activations NHWC bf16, channel counts padded to multiples of 8 so
// every pixel row is a whole number of 16-byte chunks):
//   head      : f32 in (H,W,Cin) -> y = x @ head.w + head.b (f32)  [model.py:135-143]
//   pyramid   : 4 x 2x2 average pools of the f32 head output        [model.py:146-155]
//   enc k     : a = gated(concat(pool(skip_{k-1}), pyr_k)); skip_k = gated(a)
//   dec k     : a = gated(concat(up2(x), skip_k));     x = gated(a) [model.py:174-191]
//   out       : sigmoid(x @ out.w + out.b) -> f32 (H,W,out)
// A gated conv is one implicit GEMM with N = 2*Cout (f and g branches side by
// side) and the elu(f + bf) * sigmoid(g + bg) epilogue fused; the operand
// producer resolves concat / up2 / zero padding by address arithmetic.
//
// conv kernels: gated_conv_tc (tcgen05 + TMEM, unet_tc.cuh) is the hot path;
// gated_conv_simt below is the CUDA-core version kept for on-device
// cross-checking of the tensor-core kernel (NAR_UNET_SIMT=1).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "nar_b200.h"
#include "unet_tc.cuh"

namespace nar {

static inline int rup(int x, int m) { return (x + m - 1) / m * m; }

// ----------------------------------------------------------------------------
// small kernels: head + level-0 pack, pyramid pool, encoder pool, out head
// ----------------------------------------------------------------------------
// Descriptor head + feature pyramid in one pass (model.py:135-155): one CTA
// per (T x T) level-0 tile, T = 2^(levels-1).  Each thread applies the
// per-pixel affine head y = x @ W + b in f32; the pyramid levels are 2x2
// averages of the previous level computed in f32 in shared memory (the
// reference pools the f32 head output), and every level is written once as
// bf16 NHWC padded to cp channels (zeros in the padding).
struct PyrOut {
  __nv_bfloat16* lvl[8];
  // bf16 levels: row pitch (W >> k) + pad pixels; the pad pixels of every row are
  // written as zeros (the conv's overlapping tensor map reads 16 bytes past a row's last
  // pixel, which must not be the next row's first; 2 keep rows 32-byte aligned)
  int pad;
  float* lvlf[8];  // standalone API (nar_head_pyramid): f32 (H>>k, W>>k, cin) levels instead
};

// Zero the pad pixels of the pyramid rows a CTA covers (level k: rows0 >> k rows from
// ty * (rows0 >> k), rows0 = the CTA's level-0 rows); called by the last tile column.
__device__ __forceinline__ void pyr_zero_pads(const PyrOut& out, int W, int ty, int rows0,
                                              int levels, int cp, int t) {
  for (int k = 0; k < levels; ++k) {
    const int rows = rows0 >> k, Wk = W >> k;
    for (int i = t; i < rows * out.pad; i += blockDim.x) {
      __nv_bfloat16* o =
          out.lvl[k] + ((size_t)(ty * rows + i / out.pad) * (Wk + out.pad) + Wk + i % out.pad) * cp;
      for (int c8 = 0; c8 < cp; c8 += 8) *reinterpret_cast<uint4*>(o + c8) = make_uint4(0u, 0u, 0u, 0u);
    }
  }
}

// CIN: compile-time upper bound of cin (4, 8 or 16) so the per-pixel channel
// arrays stay in registers at high occupancy.
template <int CIN>
__global__ void __launch_bounds__(256, 4)
    head_pyramid_kernel(const float* __restrict__ x, int H, int W, int cin, int cp,
                        const float* __restrict__ hw, const float* __restrict__ hb, int use_head,
                        int levels, PyrOut out) {
  extern __shared__ float tile[];  // level k-1 values of this CTA, (T*T) x cin floats, reused
  const int T = 1 << (levels - 1);
  const int tx = blockIdx.x, ty = blockIdx.y;
  const int t = threadIdx.x;
  // level 0: one thread per pixel of the T x T tile (blockDim = T*T <= 256)
  const int ly = t / T, lx = t % T;
  const int y = ty * T + ly, xx = tx * T + lx;
  float v[CIN], hv[CIN];
  const float* px = x + ((size_t)y * W + xx) * cin;
  if (CIN == 4 && cin == 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(px));
    v[0] = q.x; v[1] = q.y; v[2 % CIN] = q.z; v[3 % CIN] = q.w;
  } else {
#pragma unroll
    for (int c = 0; c < CIN; ++c) v[c] = c < cin ? __ldg(px + c) : 0.f;
  }
#pragma unroll
  for (int j = 0; j < CIN; ++j) {
    float acc = 0.f;
    if (j < cin) {
      if (use_head) {
        acc = __ldg(hb + j);
#pragma unroll
        for (int c = 0; c < CIN; ++c)
          if (c < cin) acc = fmaf(v[c], __ldg(hw + c * cin + j), acc);
      } else {
        acc = v[j];
      }
      tile[t * cin + j] = acc;
    }
    hv[j] = acc;
  }
  if (out.lvlf[0]) {  // f32 levels for the standalone API
    float* f0 = out.lvlf[0] + ((size_t)y * W + xx) * cin;
#pragma unroll
    for (int j = 0; j < CIN; ++j)
      if (j < cin) f0[j] = hv[j];
  } else {
  // bf16 level 0, padded to cp channels, 16-byte stores
  __nv_bfloat16* o0 = out.lvl[0] + ((size_t)y * (W + out.pad) + xx) * cp;
#pragma unroll
  for (int c8 = 0; c8 < 16; c8 += 8) {
    if (c8 >= cp) break;
    uint4 pk;
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float a0 = (c8 + e < CIN) ? hv[(c8 + e) % CIN] : 0.f;
      const float a1 = (c8 + e + 1 < CIN) ? hv[(c8 + e + 1) % CIN] : 0.f;
      __nv_bfloat162 h2 = __floats2bfloat162_rn(a0, a1);
      (&pk.x)[e / 2] = *reinterpret_cast<uint32_t*>(&h2);
    }
    *reinterpret_cast<uint4*>(o0 + c8) = pk;
  }
  }
  __syncthreads();
  // levels 1..L-1: 2x2 averages in f32, in place in shared memory
  int side = T;
#pragma unroll
  for (int k = 1; k < 5; ++k) {  // unrolled: out.lvl[k] stays a parameter (no local copy)
    if (k >= levels) break;
    const int ns = side >> 1;
    float m[CIN];
    const bool act = t < ns * ns;
    const int qy = act ? t / ns : 0, qx = act ? t % ns : 0;
#pragma unroll
    for (int c = 0; c < CIN; ++c) m[c] = 0.f;
    if (act) {
      const float* a0 = tile + ((2 * qy) * side + 2 * qx) * cin;
#pragma unroll
      for (int c = 0; c < CIN; ++c)
        if (c < cin)
          m[c] = ((a0[c] + a0[cin + c]) + (a0[side * cin + c] + a0[side * cin + cin + c])) * 0.25f;
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int c = 0; c < CIN; ++c)
        if (c < cin) tile[t * cin + c] = m[c];
      const int Wk = W >> k;
      if (out.lvlf[k]) {
        float* fk = out.lvlf[k] + ((size_t)(ty * ns + qy) * Wk + (tx * ns + qx)) * cin;
#pragma unroll
        for (int c = 0; c < CIN; ++c)
          if (c < cin) fk[c] = m[c];
      } else {
        __nv_bfloat16* ok = out.lvl[k] + ((size_t)(ty * ns + qy) * (Wk + out.pad) + (tx * ns + qx)) * cp;
#pragma unroll
        for (int c8 = 0; c8 < 16; c8 += 8) {
          if (c8 >= cp) break;
          uint4 pk;
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const int c = c8 + e;
            __nv_bfloat162 h2 = __floats2bfloat162_rn(
                c < CIN && c < cin ? m[c % CIN] : 0.f, c + 1 < CIN && c + 1 < cin ? m[(c + 1) % CIN] : 0.f);
            (&pk.x)[e / 2] = *reinterpret_cast<uint32_t*>(&h2);
          }
          *reinterpret_cast<uint4*>(ok + c8) = pk;
        }
      }
    }
    __syncthreads();
    side = ns;
  }
  if (out.pad && !out.lvlf[0] && tx == gridDim.x - 1) pyr_zero_pads(out, W, ty, T, levels, cp, t);
}

// Same result for the common case -- 4 input channels (16-byte aligned), levels
// <= 5, W and H multiples of 32 -- with a 2x2 pixel quad per thread: a CTA of
// 256 threads covers a 32 x 32 tile, level 1 comes straight from the quad's
// registers, and only levels 2.. go through shared memory.  4x fewer CTAs and
// barriers per pixel than head_pyramid_kernel.
__device__ __forceinline__ uint4 pack8_bf16(const float* v4, int cin) {
  uint4 pk;
  __nv_bfloat162 h0 = __floats2bfloat162_rn(v4[0], cin > 1 ? v4[1] : 0.f);
  __nv_bfloat162 h1 = __floats2bfloat162_rn(cin > 2 ? v4[2] : 0.f, cin > 3 ? v4[3] : 0.f);
  pk.x = *reinterpret_cast<uint32_t*>(&h0);
  pk.y = *reinterpret_cast<uint32_t*>(&h1);
  pk.z = 0u;
  pk.w = 0u;
  return pk;
}

// 8 bf16 of a pixel's 8 head outputs
__device__ __forceinline__ uint4 pack8f_bf16(const float* v8) {
  uint4 pk;
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(v8[e], v8[e + 1]);
    (&pk.x)[e / 2] = *reinterpret_cast<uint32_t*>(&h2);
  }
  return pk;
}

// CIN = 4 or 8 input channels (the pyramid stride cp is 8): 32 x 32 pixels per CTA,
// 2x2 quads per thread (two with 4 channels, 128 threads; one with 8, 256 threads),
// all of a thread's float4 loads issued before any is used; level 0 written as one
// 32-byte store per quad row (rows 32-byte aligned: pitch W + 2), level 1 from
// registers, levels 2-4 through shared memory.
template <int CIN>
__global__ void __launch_bounds__(CIN == 4 ? 128 : 256)
    head_pyramid_quad_kernel(const float* __restrict__ x, int H, int W, int cin, int cp,
                             const float* __restrict__ hw, const float* __restrict__ hb,
                             int use_head, int levels, PyrOut out) {
  constexpr int QPT = CIN == 4 ? 2 : 1;   // quads per thread
  constexpr int QROWS = 16 / QPT;         // quad rows per pass of the CTA's threads
  constexpr int NV = CIN / 4;             // float4 per pixel
  __shared__ float tile[16 * 16 * CIN];  // level-1 values of the CTA (16 x 16 x CIN)
  // let the first conv (a programmatic dependent) get scheduled early
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int t = threadIdx.x;
  const int qx = t & 15, qy0 = t >> 4;
  float wgt[CIN * CIN], bias[CIN];
#pragma unroll
  for (int i = 0; i < CIN * CIN; ++i)
    wgt[i] = (use_head && i / CIN < cin && i % CIN < cin) ? __ldg(hw + (i / CIN) * cin + (i % CIN)) : 0.f;
#pragma unroll
  for (int j = 0; j < CIN; ++j) bias[j] = (use_head && j < cin) ? __ldg(hb + j) : 0.f;
  float4 in[QPT][4][NV];
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    const int y0 = blockIdx.y * 32 + 2 * (qy0 + QROWS * u), x0 = blockIdx.x * 32 + 2 * qx;
#pragma unroll
    for (int d = 0; d < 4; ++d)
#pragma unroll
      for (int v = 0; v < NV; ++v)
        in[u][d][v] = __ldg(reinterpret_cast<const float4*>(
                              x + ((size_t)(y0 + (d >> 1)) * W + x0 + (d & 1)) * CIN) + v);
  }
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    const int qy = qy0 + QROWS * u;
    const int y0 = blockIdx.y * 32 + 2 * qy, x0 = blockIdx.x * 32 + 2 * qx;
    float hq[4][CIN];  // head outputs of the quad: TL, TR, BL, BR
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      float v[CIN];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        v[4 * q] = in[u][d][q].x;
        v[4 * q + 1] = in[u][d][q].y;
        v[4 * q + 2] = in[u][d][q].z;
        v[4 * q + 3] = in[u][d][q].w;
      }
#pragma unroll
      for (int j = 0; j < CIN; ++j) {
        float acc = v[j];
        if (use_head) {
          acc = bias[j];
#pragma unroll
          for (int c = 0; c < CIN; ++c) acc = fmaf(v[c], wgt[c * CIN + j], acc);
        }
        hq[d][j] = j < cin ? acc : 0.f;
      }
    }
    // the quad's two pixels of each row in one 32-byte store (full sectors)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 a = CIN == 4 ? pack8_bf16(hq[2 * h], cin) : pack8f_bf16(hq[2 * h]);
      const uint4 b = CIN == 4 ? pack8_bf16(hq[2 * h + 1], cin) : pack8f_bf16(hq[2 * h + 1]);
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      __nv_bfloat16* o = out.lvl[0] + ((size_t)(y0 + h) * (W + out.pad) + x0) * 8;
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o), "r"(w[0]),
                   "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                   : "memory");
    }
    float sum[CIN];  // the reference's 2x2 mean: ((TL + TR) + (BL + BR)) * 0.25
#pragma unroll
    for (int j = 0; j < CIN; ++j) sum[j] = ((hq[0][j] + hq[1][j]) + (hq[2][j] + hq[3][j])) * 0.25f;
    // level 1 from registers
    if (levels > 1) {
      const int W1 = W >> 1;
      __nv_bfloat16* o = out.lvl[1] + ((size_t)(blockIdx.y * 16 + qy) * (W1 + out.pad) + blockIdx.x * 16 + qx) * 8;
      *reinterpret_cast<uint4*>(o) = CIN == 4 ? pack8_bf16(sum, cin) : pack8f_bf16(sum);
    }
#pragma unroll
    for (int j = 0; j < CIN; ++j) tile[(qy * 16 + qx) * CIN + j] = sum[j];
  }
  __syncthreads();
  int side = 16;
#pragma unroll
  for (int k = 2; k < 5; ++k) {
    if (k >= levels) break;
    const int ns = side >> 1;
    float m[CIN];
#pragma unroll
    for (int c = 0; c < CIN; ++c) m[c] = 0.f;
    const bool act = t < ns * ns;
    const int py = act ? t / ns : 0, pxx = act ? t % ns : 0;
    if (act) {
      const float* a0 = tile + ((2 * py) * side + 2 * pxx) * CIN;
#pragma unroll
      for (int c = 0; c < CIN; ++c)
        m[c] = ((a0[c] + a0[CIN + c]) + (a0[side * CIN + c] + a0[side * CIN + CIN + c])) * 0.25f;
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int c = 0; c < CIN; ++c) tile[t * CIN + c] = m[c];
      const int Wk = W >> k;
      __nv_bfloat16* o = out.lvl[k] + ((size_t)(blockIdx.y * ns + py) * (Wk + out.pad) + blockIdx.x * ns + pxx) * 8;
      *reinterpret_cast<uint4*>(o) = CIN == 4 ? pack8_bf16(m, cin) : pack8f_bf16(m);
    }
    __syncthreads();
    side = ns;
  }
  if (out.pad && blockIdx.x == gridDim.x - 1) pyr_zero_pads(out, W, blockIdx.y, 32, levels, cp, t);
}

// 2x2 average of a bf16 (H,W,C) map into bf16 (H/2,W/2,C), 8 channels per thread.
__global__ void pool_bf16_kernel(const __nv_bfloat16* __restrict__ src, int H, int W, int C,
                                 __nv_bfloat16* __restrict__ dst) {
  const int Ho = H / 2, Wo = W / 2, c8n = C / 8;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)Ho * Wo * c8n) return;
  const int c8 = (int)(t % c8n);
  const int64_t p = t / c8n;
  const int y = (int)(p / Wo), x = (int)(p % Wo);
  const __nv_bfloat16* a = src + ((int64_t)(2 * y) * W + 2 * x) * C + c8 * 8;
  uint4 q[4];
  q[0] = *reinterpret_cast<const uint4*>(a);
  q[1] = *reinterpret_cast<const uint4*>(a + C);
  q[2] = *reinterpret_cast<const uint4*>(a + (int64_t)W * C);
  q[3] = *reinterpret_cast<const uint4*>(a + (int64_t)W * C + C);
  uint4 o;
  uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
  for (int i = 0; i < 4; ++i) {
    float2 s = make_float2(0.f, 0.f);
    float2 v[4];
    for (int j = 0; j < 4; ++j)
      v[j] = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&q[j])[i]);
    s.x = ((v[0].x + v[1].x) + (v[2].x + v[3].x)) * 0.25f;
    s.y = ((v[0].y + v[1].y) + (v[2].y + v[3].y)) * 0.25f;
    __nv_bfloat162 r = __float22bfloat162_rn(s);
    ow[i] = *reinterpret_cast<uint32_t*>(&r);
  }
  *reinterpret_cast<uint4*>(dst + p * C + c8 * 8) = o;
}

// logits = x @ out.w + out.b, sigmoid (model.py:189-191), f32 out (SIMT path).
__global__ void out_head_kernel(const __nv_bfloat16* __restrict__ x, int64_t npix, int C,
                                int cstride, const float* __restrict__ ow,
                                const float* __restrict__ ob, int cout, float* __restrict__ out) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const __nv_bfloat16* xp = x + p * cstride;
  for (int j = 0; j < cout; ++j) {
    float acc = ob[j];
    for (int c = 0; c < C; ++c) acc = fmaf(__bfloat162float(xp[c]), ow[c * cout + j], acc);
    out[p * cout + j] = 1.0f / (1.0f + expf(-acc));
  }
}

// ----------------------------------------------------------------------------
// CUDA-core gated conv (cross-check path)
// ----------------------------------------------------------------------------
__device__ __forceinline__ float elu_f(float x) { return x > 0.0f ? x : expm1f(x); }
__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }

// One thread per (pixel, output channel j): f_j and g_j over 9 taps x cin.
// Weights: wf/wg f32 [tap][cin_total][cout] (HWIO); bias f32.
__global__ void gated_conv_simt(ConvArgs a) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t npix = (int64_t)a.H * a.W;
  if (t >= npix * a.cout) return;
  const int j = (int)(t % a.cout);
  const int64_t p = t / a.cout;
  const int y = (int)(p / a.W), x = (int)(p % a.W);
  const int cin = a.ca + a.cb;
  float f = a.bias_f[j], g = a.bias_g[j];
  for (int ky = 0; ky < 3; ++ky) {
    const int yy = y + ky - 1;
    if (yy < 0 || yy >= a.H) continue;
    for (int kx = 0; kx < 3; ++kx) {
      const int xx = x + kx - 1;
      if (xx < 0 || xx >= a.W) continue;
      const int tap = ky * 3 + kx;
      const __nv_bfloat16* pa;
      if (a.a_up2)
        pa = a.src_a + ((int64_t)(yy / 2) * (a.W / 2) + xx / 2) * a.ca_stride;
      else
        pa = a.src_a + ((int64_t)yy * (a.a_pitch ? a.a_pitch : a.W) + xx) * a.ca_stride;
      const float* wf = a.wf32 + ((int64_t)tap * cin) * a.cout + j;
      const float* wg = a.wg32 + ((int64_t)tap * cin) * a.cout + j;
      for (int c = 0; c < a.ca; ++c) {
        const float v = __bfloat162float(pa[c]);
        f = fmaf(v, wf[(int64_t)c * a.cout], f);
        g = fmaf(v, wg[(int64_t)c * a.cout], g);
      }
      if (a.cb) {
        const __nv_bfloat16* pb = a.src_b + ((int64_t)yy * (a.b_pitch ? a.b_pitch : a.W) + xx) * a.cb_stride;
        for (int c = 0; c < a.cb; ++c) {
          const float v = __bfloat162float(pb[c]);
          f = fmaf(v, wf[(int64_t)(a.ca + c) * a.cout], f);
          g = fmaf(v, wg[(int64_t)(a.ca + c) * a.cout], g);
        }
      }
    }
  }
  a.out[p * a.cout_stride + j] = __float2bfloat16_rn(elu_f(f) * sigmoid_f(g));
  if (j == 0)  // zero the channel padding so tensor-core consumers read zeros
    for (int c = a.cout; c < a.cout_stride; ++c) a.out[p * a.cout_stride + c] = __float2bfloat16_rn(0.f);
}

// ----------------------------------------------------------------------------
// network object
// ----------------------------------------------------------------------------
struct Layer {
  std::string name;
  int ca, cb;   // real input channels from source A / source B
  int cout;
  // device weights
  float* wf32 = nullptr;  // [9][ca+cb][cout]
  float* wg32 = nullptr;
  float* bf = nullptr;
  float* bg = nullptr;
  uint16_t* wtc = nullptr;  // tcgen05-packed bf16 weights (unet_tc.cuh layout)
  bool up2 = false;         // source A is the nearest-upsampled lower level (decoder "a")
  bool pairs = false;       // packed with paired up2 chunks (tc_pack_weights)
  size_t wtc_bytes = 0;
  std::vector<float> hf, hg, hbf, hbg;  // host staging (HWIO)
  bool set_f = false, set_g = false, set_bf = false, set_bg = false;
};

}  // namespace nar

struct nar_unet {
  nar_unet_config cfg;
  std::vector<nar::Layer> layers;  // enc0a, enc0b, ..., enc4b, dec3a, ..., dec0b
  std::map<std::string, int> index;
  std::vector<float> head_w, head_b, out_w, out_b;
  float *d_head_w = nullptr, *d_head_b = nullptr, *d_out_w = nullptr, *d_out_b = nullptr;
  bool uploaded = false;
  bool simt = false;
};

namespace nar {

static int width_of(const nar_unet_config& c, int k) {
  long w = c.base_channels;
  for (int i = 0; i < k; ++i) w *= c.channel_multiplier;
  return (int)(w < c.max_channels ? w : c.max_channels);
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// channel stride of level-k activations (multiple of 16: whole K=16 MMA steps)
static int stride_of(const nar_unet_config& c, int k) { return rup(width_of(c, k), 16); }

// workspace carve-up for one (H, W)
struct Plan {
  int L;
  int H[8], W[8];
  int cinp;             // padded input channel count
  size_t off_pyr16[8], off_skip[8], off_pool[8], off_tmp[8], off_x[8];
  size_t total;
};

static Plan make_plan(const nar_unet& n, int H, int W) {
  Plan p;
  p.L = n.cfg.levels;
  // pyramid levels at an 8-channel stride when the input has <= 8 channels: 16-byte
  // pixels, written with full-sector stores and no zero padding; the conv reads them
  // through an overlapping tensor map (tc_make_map) whose channels 8..15 are the
  // next pixel's (their weights are zero)
  p.cinp = rup(n.cfg.input_channels, 8);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  for (int k = 0; k < p.L; ++k) {
    p.H[k] = H >> k;
    p.W[k] = W >> k;
    const size_t px = (size_t)p.H[k] * p.W[k];
    const int w = stride_of(n.cfg, k);
    p.off_pyr16[k] = take((px + 2 * p.H[k]) * p.cinp * 2);  // rows of W + 2 pixels (PyrOut::pad)
    // off_x[k] (k >= 1) and the bottleneck off_skip[L-1] feed an up2 and are
    // written wide (H, 2W) on the tensor-core path
    p.off_skip[k] = take(px * w * 2 * (k + 1 == p.L ? 2 : 1));
    p.off_tmp[k] = take(px * w * 2);
    p.off_x[k] = take(px * w * 2 * (k > 0 ? 2 : 1));
    p.off_pool[k] = k + 1 < p.L ? take(px / 4 * w * 2) : 0;
  }
  p.total = off + 256;
  return p;
}

// Device copies of the parameters; re-run after any nar_unet_set_param.  The
// previous copies are released first (cudaFree waits for in-flight work that
// may still read them); set_param must not race a forward on another thread.
static int upload(nar_unet* n) {
  if (n->uploaded) return NAR_OK;
  auto release = [](auto*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  release(n->d_head_w);
  release(n->d_head_b);
  release(n->d_out_w);
  release(n->d_out_b);
  for (auto& l : n->layers) {
    release(l.wf32);
    release(l.wg32);
    release(l.bf);
    release(l.bg);
    release(l.wtc);
  }
  auto dup = [](const std::vector<float>& v, float** d) -> int {
    if (cudaMalloc(d, v.size() * 4 + 4) != cudaSuccess) return 1;
    cudaMemcpy(*d, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
    return 0;
  };
  const int cin = n->cfg.input_channels;
  if (n->cfg.use_descriptor_head) {
    if (n->head_w.size() != (size_t)cin * cin || n->head_b.size() != (size_t)cin)
      return set_error(NAR_ERR_CONFIG, "head parameters not set");
    if (dup(n->head_w, &n->d_head_w) || dup(n->head_b, &n->d_head_b))
      return set_error(NAR_ERR_NOMEM, "weight upload failed");
  }
  if (n->out_w.empty() || n->out_b.empty())
    return set_error(NAR_ERR_CONFIG, "out parameters not set");
  if (dup(n->out_w, &n->d_out_w) || dup(n->out_b, &n->d_out_b))
    return set_error(NAR_ERR_NOMEM, "weight upload failed");
  for (auto& l : n->layers) {
    if (!(l.set_f && l.set_g && l.set_bf && l.set_bg)) {
      std::string m = "parameters of " + l.name + " not set";
      return set_error(NAR_ERR_CONFIG, m.c_str());
    }
    if (dup(l.hf, &l.wf32) || dup(l.hg, &l.wg32) || dup(l.hbf, &l.bf) || dup(l.hbg, &l.bg))
      return set_error(NAR_ERR_NOMEM, "weight upload failed");
    std::vector<uint16_t> packed;
    {
      const int N = 2 * tc_coutp(l.cout);
      // sliding layers with an even row tile, and plain layers up to N = 128 (R = 2 or 4)
      l.pairs = !n->simt && l.up2 && N <= 128 && (!tc_slide(N) || tc_rows(N, 2) % 2 == 0) &&
                !(getenv("NAR_TC_UP2PAIR") && getenv("NAR_TC_UP2PAIR")[0] == '0');
    }
    tc_pack_weights(l.hf, l.hg, l.ca, l.cb, l.cout, packed, l.pairs);
    l.wtc_bytes = packed.size() * 2;
    if (cudaMalloc(&l.wtc, l.wtc_bytes) != cudaSuccess)
      return set_error(NAR_ERR_NOMEM, "weight upload failed");
    cudaMemcpy(l.wtc, packed.data(), l.wtc_bytes, cudaMemcpyHostToDevice);
  }
  if (cudaGetLastError() != cudaSuccess) return set_error(NAR_ERR_CUDA, "weight upload failed");
  n->uploaded = true;
  return NAR_OK;
}

// One gated conv.  pool_out (optional): also write the 2x2 average pool of
// the output; head_out (optional): write sigmoid(out @ out.w + out.b) in f32
// (model.py:189-191) -- on the tensor-core path both are fused into the
// epilogue (out may then be NULL), on the SIMT path they run as kernels.
static int run_conv(nar_unet* n, Layer& l, const __nv_bfloat16* src_a, int ca_stride, int a_up2,
                    const __nv_bfloat16* src_b, int cb_stride, int H, int W,
                    __nv_bfloat16* out, cudaStream_t st, __nv_bfloat16* pool_out = nullptr,
                    float* head_out = nullptr, __nv_bfloat16* scratch = nullptr,
                    int out_wide = 0, int a_pitch = 0, int b_pitch = 0) {
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.a_pitch = a_pitch;
  a.b_pitch = b_pitch;
  a.src_a = src_a;
  a.src_b = src_b;
  a.ca = l.ca;
  a.cb = l.cb;
  a.ca_stride = ca_stride;
  a.cb_stride = cb_stride;
  a.a_up2 = a_up2;
  a.out_wide = out_wide;
  a.H = H;
  a.W = W;
  a.cout = l.cout;
  a.cout_stride = rup(l.cout, 16);
  a.wf32 = l.wf32;
  a.wg32 = l.wg32;
  a.bias_f = l.bf;
  a.bias_g = l.bg;
  a.wtc = reinterpret_cast<const __nv_bfloat16*>(l.wtc);
  a.up2pair = l.pairs && a_up2 == 2;
  a.out = out;
  const int cst = a.cout_stride;
  auto pool_kernel = [&](const __nv_bfloat16* src) {
    const int64_t t = (int64_t)(H / 2) * (W / 2) * (cst / 8);
    nar::count_launch();
    pool_bf16_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(src, H, W, cst, pool_out);
  };
  auto head_kernel = [&](const __nv_bfloat16* src) {
    const int64_t np = (int64_t)H * W;
    nar::count_launch();
    out_head_kernel<<<(unsigned)((np + 127) / 128), 128, 0, st>>>(
        src, np, l.cout, cst, n->d_out_w, n->d_out_b, n->cfg.output_channels, head_out);
  };
  if (n->simt) {
    if (!a.out) a.out = scratch;
    const int64_t tot = (int64_t)H * W * l.cout;
    nar::count_launch();
    gated_conv_simt<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(a);
    if (pool_out) pool_kernel(a.out);
    if (head_out) head_kernel(a.out);
    return check_launch(l.name.c_str());
  }
  const bool fuse_pool =
      pool_out && (tc_rows_for(l.cout, H, W, (l.ca + 15) / 16 + (l.cb + 15) / 16) % 2 == 0);
  if (fuse_pool) a.pool_out = pool_out;
  if (head_out) {
    a.head_out = head_out;
    a.head_w = n->d_out_w;
    a.head_b = n->d_out_b;
    a.head_n = n->cfg.output_channels;
    for (int c = 0; c < 32; ++c)
      for (int k = 0; k < 4; ++k)
        a.head_wv[c * 4 + k] =
            (c < l.cout && k < a.head_n) ? n->out_w[(size_t)c * a.head_n + k] : 0.0f;
    for (int k = 0; k < 4; ++k) a.head_bv[k] = k < a.head_n ? n->out_b[k] : 0.0f;
    if (a.head_n > 4 || l.cout > 32) {  // beyond the fused epilogue's budget
      a.head_out = nullptr;
      if (!a.out) a.out = scratch;
    }
  }
  static const int dbg = [] {
    const char* e = getenv("NAR_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  a.debug = dbg;
  static const int sblk = [] {
    const char* e = getenv("NAR_TC_SLIDE_BLOCKS");
    const int v = e ? atoi(e) : 1;
    return v < 1 ? 1 : (v > 4 ? 4 : v);
  }();
  a.slide_blocks = sblk;
  int rc = tc_launch_gated_conv(a, st);
  if (rc) return rc;
  if (pool_out && !fuse_pool) pool_kernel(a.out);
  if (head_out && !a.head_out) head_kernel(a.out);
  return check_launch(l.name.c_str());
}

}  // namespace nar

using namespace nar;

extern "C" {

int nar_unet_create(const nar_unet_config* cfg, nar_unet** out) {
  if (!cfg || !out) return set_error(NAR_ERR_INVALID, "NULL argument");
  if (cfg->input_channels < 1 || cfg->input_channels > NAR_MAX_CHANNELS)
    return set_error(NAR_ERR_CONFIG, "input_channels must be in [1, 16]");
  if (cfg->levels < 1 || cfg->levels > 7) return set_error(NAR_ERR_CONFIG, "levels out of range");
  if (cfg->output_channels < 1 || cfg->output_channels > 16)
    return set_error(NAR_ERR_CONFIG, "output_channels out of range");
  nar_unet* n = new nar_unet();
  n->cfg = *cfg;
  const char* env = getenv("NAR_UNET_SIMT");
  n->simt = env && env[0] == '1';
  const int cin = cfg->input_channels;
  for (int k = 0; k < cfg->levels; ++k) {
    const int w = width_of(*cfg, k);
    if (w < 1 || w > 128) {
      delete n;
      return set_error(NAR_ERR_CONFIG, "level widths must be in [1, 128]");
    }
    Layer a;
    a.name = "enc" + std::to_string(k) + "a";
    a.ca = k == 0 ? cin : width_of(*cfg, k - 1);
    a.cb = k == 0 ? 0 : cin;
    a.cout = w;
    Layer b;
    b.name = "enc" + std::to_string(k) + "b";
    b.ca = w;
    b.cb = 0;
    b.cout = w;
    n->layers.push_back(a);
    n->layers.push_back(b);
  }
  for (int k = cfg->levels - 2; k >= 0; --k) {
    const int w = width_of(*cfg, k);
    Layer a;
    a.name = "dec" + std::to_string(k) + "a";
    a.up2 = true;
    a.ca = width_of(*cfg, k + 1);
    a.cb = w;
    a.cout = w;
    Layer b;
    b.name = "dec" + std::to_string(k) + "b";
    b.ca = w;
    b.cb = 0;
    b.cout = w;
    n->layers.push_back(a);
    n->layers.push_back(b);
  }
  for (size_t i = 0; i < n->layers.size(); ++i) n->index[n->layers[i].name] = (int)i;
  *out = n;
  return NAR_OK;
}

int nar_unet_destroy(nar_unet* n) {
  if (!n) return NAR_OK;
  cudaFree(n->d_head_w);
  cudaFree(n->d_head_b);
  cudaFree(n->d_out_w);
  cudaFree(n->d_out_b);
  for (auto& l : n->layers) {
    cudaFree(l.wf32);
    cudaFree(l.wg32);
    cudaFree(l.bf);
    cudaFree(l.bg);
    cudaFree(l.wtc);
  }
  delete n;
  return NAR_OK;
}

int nar_unet_set_param(nar_unet* n, const char* name, const float* host, int64_t numel) {
  if (!n || !name || (!host && numel)) return set_error(NAR_ERR_INVALID, "NULL argument");
  std::string s(name);
  const int cin = n->cfg.input_channels;
  auto want = [&](int64_t expect) -> int {
    if (numel != expect) {
      std::string m = "parameter " + s + " has " + std::to_string(numel) + " values, expected " +
                      std::to_string(expect);
      return set_error(NAR_ERR_CONFIG, m.c_str());
    }
    return NAR_OK;
  };
  int rc;
  n->uploaded = false;
  if (s == "head.w") {
    if ((rc = want((int64_t)cin * cin))) return rc;
    n->head_w.assign(host, host + numel);
    return NAR_OK;
  }
  if (s == "head.b") {
    if ((rc = want(cin))) return rc;
    n->head_b.assign(host, host + numel);
    return NAR_OK;
  }
  const int w0 = width_of(n->cfg, 0);
  if (s == "out.w") {
    if ((rc = want((int64_t)w0 * n->cfg.output_channels))) return rc;
    n->out_w.assign(host, host + numel);
    return NAR_OK;
  }
  if (s == "out.b") {
    if ((rc = want(n->cfg.output_channels))) return rc;
    n->out_b.assign(host, host + numel);
    return NAR_OK;
  }
  const size_t dot = s.find('.');
  if (dot == std::string::npos || !n->index.count(s.substr(0, dot))) {
    std::string m = "unknown parameter " + s;
    return set_error(NAR_ERR_CONFIG, m.c_str());
  }
  Layer& l = n->layers[n->index[s.substr(0, dot)]];
  const std::string field = s.substr(dot + 1);
  const int64_t wn = (int64_t)9 * (l.ca + l.cb) * l.cout;
  if (field == "f_w") {
    if ((rc = want(wn))) return rc;
    l.hf.assign(host, host + numel);
    l.set_f = true;
  } else if (field == "g_w") {
    if ((rc = want(wn))) return rc;
    l.hg.assign(host, host + numel);
    l.set_g = true;
  } else if (field == "f_b") {
    if ((rc = want(l.cout))) return rc;
    l.hbf.assign(host, host + numel);
    l.set_bf = true;
  } else if (field == "g_b") {
    if ((rc = want(l.cout))) return rc;
    l.hbg.assign(host, host + numel);
    l.set_bg = true;
  } else {
    std::string m = "unknown parameter " + s;
    return set_error(NAR_ERR_CONFIG, m.c_str());
  }
  return NAR_OK;
}

// timing experiments: the clock64() stamps of the last conv launched with
// NAR_TC_DEBUG bit 3 (see TC_TRACE in unet_tc.cuh); not part of the public header
int nar_debug_tc_trace(unsigned long long* out, int n) {
  if (!out || n > kTraceTiles * kTraceSlots) return set_error(NAR_ERR_INVALID, "trace");
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_tc_trace, n * sizeof(unsigned long long)) == cudaSuccess
             ? NAR_OK
             : set_error(NAR_ERR_CUDA, "trace copy");
}

int nar_unet_workspace_bytes(const nar_unet* n, int32_t height, int32_t width, size_t* bytes) {
  if (!n || !bytes) return set_error(NAR_ERR_INVALID, "NULL argument");
  const int div = 1 << (n->cfg.levels - 1);
  if (height <= 0 || width <= 0 || height % div || width % div)
    return set_error(NAR_ERR_INVALID, "spatial dims not divisible by 2^(levels-1)");
  *bytes = make_plan(*n, height, width).total;
  return NAR_OK;
}

int nar_unet_forward(nar_unet* n, const float* in, int32_t H, int32_t W, float* out, void* ws,
                     size_t ws_bytes, void* stream) {
  if (!n || !in || !out || !ws) return set_error(NAR_ERR_INVALID, "NULL argument");
  const int div = 1 << (n->cfg.levels - 1);
  if (H <= 0 || W <= 0 || H % div || W % div)
    return set_error(NAR_ERR_INVALID, "spatial dims not divisible by 2^(levels-1)");
  const Plan p = make_plan(*n, H, W);
  if (ws_bytes < p.total) return set_error(NAR_ERR_INVALID, "workspace too small");
  int rc = upload(n);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* base = static_cast<uint8_t*>(ws);
  auto bf = [&](size_t off) { return reinterpret_cast<__nv_bfloat16*>(base + off); };
  const int cin = n->cfg.input_channels, L = p.L;

  {
    const int T = 1 << (L - 1);
    PyrOut po;
    memset(&po, 0, sizeof(po));
    for (int k = 0; k < L; ++k) po.lvl[k] = bf(p.off_pyr16[k]);
    po.pad = 2;  // zero pixels per row: the overlap read needs one, the second keeps rows 32-B aligned
    const size_t sm = (size_t)T * T * cin * 4;
    if (T * T > 256) return set_error(NAR_ERR_CONFIG, "at most 5 pyramid levels supported");
    auto kern = cin <= 4 ? head_pyramid_kernel<4>
                         : (cin <= 8 ? head_pyramid_kernel<8> : head_pyramid_kernel<16>);
    const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    if (cin == 4 && !aligned) kern = head_pyramid_kernel<8>;  // no float4 loads
    nar::count_launch();
    const bool quad = (cin == 4 || cin == 8) && p.cinp == 8 && aligned && L <= 5 &&
                      W % 32 == 0 && H % 32 == 0;
    if (quad && cin == 4)
      head_pyramid_quad_kernel<4><<<dim3(W / 32, H / 32), 128, 0, st>>>(
          in, H, W, cin, p.cinp, n->d_head_w, n->d_head_b, n->cfg.use_descriptor_head, L, po);
    else if (quad)
      head_pyramid_quad_kernel<8><<<dim3(W / 32, H / 32), 256, 0, st>>>(
          in, H, W, cin, p.cinp, n->d_head_w, n->d_head_b, n->cfg.use_descriptor_head, L, po);
    else
      kern<<<dim3(W / T, H / T), T * T, sm, st>>>(in, H, W, cin, p.cinp, n->d_head_w,
                                                 n->d_head_b, n->cfg.use_descriptor_head, L, po);
    if ((rc = check_launch("head_pyramid"))) return rc;
  }

  const bool wide = !n->simt;  // up2 sources written pre-repeated (see ConvArgs::a_up2)
  int li = 0;
  for (int k = 0; k < L; ++k) {
    Layer& la = n->layers[li++];
    Layer& lb = n->layers[li++];
    if (k == 0) {
      rc = run_conv(n, la, bf(p.off_pyr16[0]), p.cinp, 0, nullptr, 0, p.H[0], p.W[0],
                    bf(p.off_tmp[0]), st, nullptr, nullptr, nullptr, 0, p.W[0] + 2);
    } else {
      rc = run_conv(n, la, bf(p.off_pool[k - 1]), stride_of(n->cfg, k - 1), 0,
                    bf(p.off_pyr16[k]), p.cinp, p.H[k], p.W[k], bf(p.off_tmp[k]), st, nullptr,
                    nullptr, nullptr, 0, 0, p.W[k] + 2);
    }
    if (rc) return rc;
    const bool last = L == 1;
    rc = run_conv(n, lb, bf(p.off_tmp[k]), stride_of(n->cfg, k), 0, nullptr, 0, p.H[k], p.W[k],
                  last ? nullptr : bf(p.off_skip[k]), st,
                  k + 1 < L ? bf(p.off_pool[k]) : nullptr, last ? out : nullptr,
                  bf(p.off_skip[k]), wide && !last && k + 1 == L);
    if (rc) return rc;
  }
  const __nv_bfloat16* x = bf(p.off_skip[L - 1]);
  for (int k = L - 2; k >= 0; --k) {
    Layer& la = n->layers[li++];
    Layer& lb = n->layers[li++];
    rc = run_conv(n, la, x, stride_of(n->cfg, k + 1), wide ? 2 : 1, bf(p.off_skip[k]),
                  stride_of(n->cfg, k), p.H[k], p.W[k], bf(p.off_tmp[k]), st);
    if (rc) return rc;
    // dec0b: the out head (1x1 conv + sigmoid) is fused into the epilogue
    rc = run_conv(n, lb, bf(p.off_tmp[k]), stride_of(n->cfg, k), 0, nullptr, 0, p.H[k], p.W[k],
                  k == 0 ? nullptr : bf(p.off_x[k]), st, nullptr, k == 0 ? out : nullptr,
                  bf(p.off_x[k]), wide && k > 0);
    if (rc) return rc;
    x = bf(p.off_x[k]);
  }
  return NAR_OK;
}

// ---- standalone ops (model.py:135-163), f32 in/out on device ---------------------

static __global__ void pack_bf16_kernel(const float* __restrict__ in, int64_t npx, int cin,
                                        int cinp, __nv_bfloat16* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= npx * cinp) return;
  const int64_t p = t / cinp;
  const int c = (int)(t - p * cinp);
  out[t] = __float2bfloat16_rn(c < cin ? in[p * cin + c] : 0.0f);
}

static __global__ void unpack_f32_kernel(const __nv_bfloat16* __restrict__ in, int64_t npx,
                                         int cout, int cs, float* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= npx * cout) return;
  const int64_t p = t / cout;
  out[t] = __bfloat162float(in[p * cs + (t - p * cout)]);
}

int nar_head_pyramid(const float* in, int32_t H, int32_t W, int32_t C, const float* head_w,
                     const float* head_b, int32_t use_head, int32_t levels, float* const* out,
                     void* stream) {
  if (!in || !out || (use_head && (!head_w || !head_b)))
    return set_error(NAR_ERR_INVALID, "NULL argument");
  if (C < 1 || C > 16) return set_error(NAR_ERR_CONFIG, "1..16 channels");
  if (levels < 1 || levels > 5) return set_error(NAR_ERR_CONFIG, "1..5 pyramid levels");
  const int T = 1 << (levels - 1);
  if (H <= 0 || W <= 0 || H % T || W % T)
    return set_error(NAR_ERR_INVALID, "spatial dims not divisible by 2^(levels-1)");
  PyrOut po;
  memset(&po, 0, sizeof(po));
  for (int k = 0; k < levels; ++k) {
    if (!out[k]) return set_error(NAR_ERR_INVALID, "NULL pyramid level");
    po.lvlf[k] = out[k];
  }
  auto kern = C <= 4 ? head_pyramid_kernel<4> : (C <= 8 ? head_pyramid_kernel<8> : head_pyramid_kernel<16>);
  if (C == 4 && (reinterpret_cast<uintptr_t>(in) & 15)) kern = head_pyramid_kernel<8>;
  nar::count_launch();
  kern<<<dim3(W / T, H / T), T * T, (size_t)T * T * C * 4, (cudaStream_t)stream>>>(
      in, H, W, C, rup(C, 16), head_w, head_b, use_head, levels, po);
  return check_launch("head_pyramid");
}

int nar_gated_conv(const float* in, int32_t H, int32_t W, int32_t cin, const float* f_w,
                   const float* f_b, const float* g_w, const float* g_b, int32_t cout, float* out,
                   void* stream) {
  if (!in || !out || !f_w || !f_b || !g_w || !g_b) return set_error(NAR_ERR_INVALID, "NULL argument");
  if (H <= 0 || W <= 0 || cin < 1 || cout < 1 || cout > 128 || cin > 2048)
    return set_error(NAR_ERR_CONFIG, "unsupported gated conv shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int cinp = rup(cin, 16), cs = rup(cout, 16);
  const int64_t npx = (int64_t)H * W;
  std::vector<float> wf(f_w, f_w + (size_t)9 * cin * cout), wg(g_w, g_w + (size_t)9 * cin * cout);
  std::vector<uint16_t> packed;
  tc_pack_weights(wf, wg, cin, 0, cout, packed);
  __nv_bfloat16 *x = nullptr, *y = nullptr, *w = nullptr;
  float *bf = nullptr, *bg = nullptr;
  int rc = NAR_OK;
  nar::keep_pool_memory();
  if (cudaMallocAsync(reinterpret_cast<void**>(&x), (size_t)npx * cinp * 2, st) ||
      cudaMallocAsync(reinterpret_cast<void**>(&y), (size_t)npx * cs * 2, st) ||
      cudaMallocAsync(reinterpret_cast<void**>(&w), packed.size() * 2, st) ||
      cudaMallocAsync(reinterpret_cast<void**>(&bf), (size_t)cout * 4, st) ||
      cudaMallocAsync(reinterpret_cast<void**>(&bg), (size_t)cout * 4, st))
    rc = set_error(NAR_ERR_NOMEM, "gated conv scratch");
  if (!rc) {
    cudaMemcpyAsync(w, packed.data(), packed.size() * 2, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(bf, f_b, (size_t)cout * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(bg, g_b, (size_t)cout * 4, cudaMemcpyHostToDevice, st);
    nar::count_launch();
    pack_bf16_kernel<<<(unsigned)((npx * cinp + 255) / 256), 256, 0, st>>>(in, npx, cin, cinp, x);
    ConvArgs a;
    memset(&a, 0, sizeof(a));
    a.src_a = x;
    a.ca = cin;
    a.ca_stride = cinp;
    a.H = H;
    a.W = W;
    a.cout = cout;
    a.cout_stride = cs;
    a.bias_f = bf;
    a.bias_g = bg;
    a.wtc = w;
    a.out = y;
    const char* dbg = getenv("NAR_TC_DEBUG");  // timing experiments only
    a.debug = dbg ? atoi(dbg) : 0;
    rc = tc_launch_gated_conv(a, st);
    if (!rc) {
      nar::count_launch();
      unpack_f32_kernel<<<(unsigned)((npx * cout + 255) / 256), 256, 0, st>>>(y, npx, cout, cs, out);
    }
    // the host weight copy is stream-ordered: keep `packed` alive until it ran
    cudaStreamSynchronize(st);
  }
  for (void* p : {(void*)x, (void*)y, (void*)w, (void*)bf, (void*)bg})
    if (p) cudaFreeAsync(p, st);
  if (!rc) rc = check_launch("gated_conv");
  return rc;
}

}  // extern "C"
