// unet_tc.cuh -- tcgen05 / TMEM implicit-GEMM gated 3x3 convolution (sm_100a).
//
// One launch computes  out = elu(conv(x, Wf) + bf) * sigmoid(conv(x, Wg) + bg)
// (model.py:158-163) for x = concat(srcA or up2(srcA), srcB) with zero "same"
// padding (autodiff.py:267-288), as a GEMM with
//   M = pixels (tiles of R image rows x 128 pixels),  N = 2*Coutp (f | g),
//   K = 9 taps x input channels (16-channel chunks).
//
// CTA roles (576 threads, 1 CTA per SM, persistent over tiles):
//   warp 0     producer.  One lane issues, per (tile, 16-channel chunk)
//              stage, one TMA tensor load of the (R+2) x 136 pixel halo
//              (32 B per pixel) straight into the UMMA SWIZZLE_32B K-major
//              layout [row][px][32 B]; TMA zero-fills the image
//              border ("same" padding) and the concat is just a second tensor
//              map.  The decoder's up2(srcA) chunks come from a "wide" tensor
//              (the previous layer stored every pixel twice, ConvArgs::a_up2 = 2),
//              so they are plain TMA boxes of the LR low-res rows; the vertical
//              repeat is the MMA's row addressing.  A TMA bulk copy streams the
//              chunk's pre-packed weights.
//   warp 17    MMA issuer (one thread) + TMEM owner: tcgen05.mma (M=128, N,
//              K=16) whose A descriptor is a halo row shifted by the tap (a
//              16-byte start-address offset: pixels are contiguous 16 B rows,
//              SBO = 128 B); narrow layers slide (see tc_slide).
//   warps 1-16 epilogue: tcgen05.ld the f and g accumulators of their TMEM
//              lane quarter, apply the gate; store bf16 NHWC (or wide), and
//              optionally the 2x2 average pool of the output (encoder skips
//              feeding the next level) and/or the final 1x1 out head + sigmoid
//              (model.py:189-191) in f32 instead of the bf16 activation.
// Accumulators are double buffered in TMEM (2 x R x N <= 512 columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1 -- except for wide layers,
// which take a single buffer of twice the rows (see tc_bufs_for).  Within a
// tile the MMAs run row by row in the last channel chunk and each epilogue row
// slot is signalled as soon as its rows are complete (tc_epi_*), so the
// epilogue of the first rows also overlaps the MMAs of the last ones.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>
#include <utility>
#include <vector>

#include "common.cuh"

namespace nar {

struct ConvArgs {
  const __nv_bfloat16* src_a;  // NHWC, channel stride ca_stride (multiple of 8)
  const __nv_bfloat16* src_b;  // NHWC, channel stride cb_stride, or NULL
  int ca, cb, ca_stride, cb_stride;
  // a_up2: srcA is nearest-upsampled 2x.  1 = srcA is (H/2, W/2) (SIMT path);
  // 2 = srcA is "wide" (H/2, W): its producer already repeated every pixel
  // horizontally (out_wide), so the tensor-core path TMA-loads it directly and
  // resolves the vertical repeat by descriptor row addressing.
  int a_up2;
  int H, W;                    // output (and src_b) resolution
  int out_wide;                // tensor-core path: write out as (H, 2W), each pixel twice
  int a_pitch, b_pitch;        // row pitch of src_a / src_b in pixels (0: W); pyramid
                               // levels have W + 2 (zero pad pixels per row)
  int cout, cout_stride;       // real output channels, output channel stride
  const float* wf32;           // SIMT path: HWIO f32
  const float* wg32;
  const float* bias_f;
  const float* bias_g;
  const __nv_bfloat16* wtc;    // tcgen05 path: packed (see tc_pack_weights)
  __nv_bfloat16* out;          // bf16 output, or NULL (out head only)
  __nv_bfloat16* pool_out;     // 2x2-average-pooled output (H/2, W/2, cout_stride), or NULL
  const float* head_w;         // fused out head: (cout, head_n) f32, or NULL
  const float* head_b;
  float* head_out;             // (H, W, head_n) f32
  int head_n;
  // the same head weights by value (kernel-parameter constant bank): [c][4] and [4],
  // zero padded, so the fused head's FMAs take constant operands (cout <= 32)
  float head_wv[32 * 4];
  float head_bv[4];
  // timing experiments only (NAR_TC_DEBUG, wrong results): bit 0 = epilogue
  // skips the gate math and stores, bit 1 = no MMAs are issued, bit 2 = no
  // operand loads
  int debug;
  // sliding layers: halo-row blocks of the last chunk, each followed by the
  // signal of the epilogue row slots it completes (1 = signal at the tile end)
  int slide_blocks;
  // paired up2 chunks (sliding layers with a wide up2 source, R even): the packed weights
  // hold 4 stacked ky blocks per kx for source-A chunks (tc_pack_weights, pairs = true)
  int up2pair;
};

constexpr int kProdWarps = 1;   // TMA issue (one lane)
constexpr int kProdThreads = kProdWarps * 32;
constexpr int kEpiGroups = 4;   // epilogue warps per TMEM lane quarter
constexpr int kMmaWarp = kProdWarps + 4 * kEpiGroups;
constexpr int kTcThreads = (kMmaWarp + 1) * 32;  // 1 producer + 16 epilogue + 1 MMA warps
constexpr int kHaloPx = 130;                 // pixels a tile row reads (128 + 2 halo)
#ifndef NAR_TC_HALO_PITCH
#define NAR_TC_HALO_PITCH 136
#endif
constexpr int kHaloPitch = NAR_TC_HALO_PITCH;  // loaded per row: 136 x 32 B = 17 swizzle atoms
constexpr int kHaloRowBytes = kHaloPitch * 32;  // one 16-channel halo row, SWIZZLE_32B

// NB = TMEM accumulator buffers.  2: the epilogue of tile i overlaps the MMAs
// of tile i+1.  1 (N = 256 layers with enough tiles, see tc_bufs_for): twice
// the rows per tile instead, which halves how often the weights (9*N*32 B per
// 16-channel chunk, the bulk of such a layer's L2->SM traffic) are streamed.
__host__ __device__ constexpr int tc_rows(int N, int NB) {
  return 512 / (NB * N) > 8 ? 8 : 512 / (NB * N);
}
__host__ __device__ constexpr int tc_low_rows(int N, int NB) { return tc_rows(N, NB) / 2 + 2; }
// TMA tensor-load destinations must be 128-byte aligned: slabs are padded.
__host__ __device__ constexpr int tc_r128(int x) { return (x + 127) / 128 * 128; }
__host__ __device__ constexpr int tc_r1024(int x) { return (x + 1023) / 1024 * 1024; }
__host__ __device__ constexpr int tc_a_bytes(int N, int NB) {
  return tc_r1024((tc_rows(N, NB) + 2) * kHaloRowBytes);
}
// B slot of a stage: 9 taps x N rows x 32 B; layers that can take paired up2 chunks
// (N <= 128, see tc_pack_weights) reserve 3 kx x 4N rows -- 4/3 of the plain size
__host__ __device__ constexpr int tc_b_bytes(int N) { return N <= 128 ? 12 * N * 32 : 9 * N * 32; }
__host__ __device__ constexpr int tc_b3_bytes(int N) { return 9 * N * 32; }   // a plain chunk
__host__ __device__ constexpr int tc_b4_bytes(int N) { return 12 * N * 32; }  // a paired chunk
__host__ __device__ constexpr int tc_stage_bytes(int N, int NB) {
  return tc_r1024(tc_a_bytes(N, NB) + tc_b_bytes(N));
}
constexpr int kTcParamFloats = 128 * 4 + 4;  // head_w, head_b
// Narrow layers (N <= 48) use "sliding" MMAs: one MMA per (halo row, kx) with
// the three ky weight blocks stacked along N (N' = 3N) accumulates into three
// consecutive output rows at once -- (R+2)*3 MMAs per chunk instead of 9*R,
// which matters because an M=128, K=16 MMA costs ~55 cycles for any N <= 64.
__host__ __device__ constexpr bool tc_slide(int N) { return N <= 64; }
// Bias in the accumulator: every tile starts with one MMA (two for 512-column
// tiles) of a "ones" A operand (k = 0, 1 -> 1.0) against a bias B operand
// (row n: k = 0 -> hi, k = 1 -> lo bf16 halves of the packed bias of column
// n % N), so the accumulators begin at the bias (to ~2^-16 relative) and the
// epilogue reads conv + bias directly.  No-swizzle K-major, 8-row core
// matrices: A = 128 rows (LBO 2048), B = 256 rows (LBO 4096).
constexpr int kTcOnesBytes = 128 * 32;
constexpr int kTcBiasBytes = 256 * 32;
// Epilogue row slots: the kEpiGroups warp groups split a tile's rows into
// contiguous slots of whole units (a unit = one row, or a row pair when the
// output is 2x2-pooled); with fewer units than groups the groups also split
// the channel chunks.  Slot s ends at row tc_epi_last_row(s, ...).
__host__ __device__ constexpr int tc_epi_rgroups(int units) {
  return units < kEpiGroups ? (units > 0 ? units : 1) : kEpiGroups;
}
__host__ __device__ constexpr int tc_epi_first_unit(int s, int units, int rg) {
  return s * units / rg;
}
__host__ __device__ constexpr int tc_epi_last_row(int s, int units, int rg, int rstep) {
  return tc_epi_first_unit(s + 1, units, rg) * rstep - 1;
}
// Every tcgen05.commit is a bubble in the tensor pipe (~60 cycles, scripts/
// mma_slide_bench.cu), so slots completing together share one signal: the barrier
// of the first slot of their group.  Sliding layers complete all slots at the tile
// end, or (two blocks) the slots ending by row R/2-1 after the first block and
// the rest at the end; plain layers signal each slot as its last row completes.
__host__ __device__ constexpr int tc_epi_signal(int s, bool slide, int nblk, int units, int rg,
                                                int rstep, int R) {
  if (!slide) return s;
  if (nblk < 2) return 0;
  int s1 = 0;  // slots complete after the first block (rows < R/2)
  while (s1 < rg && tc_epi_last_row(s1, units, rg, rstep) <= R / 2 - 1) ++s1;
  return s < s1 ? 0 : s1;
}
__host__ __device__ constexpr int tc_fixed_smem(int N) {
  return 512 + kTcOnesBytes + kTcBiasBytes + kTcParamFloats * 4;
}
// stages: as many (<= NAR_TC_MAX_STAGES) as fit the 227 KB opt-in shared memory
#ifndef NAR_TC_WEIGHT_PREFETCH
#define NAR_TC_WEIGHT_PREFETCH 1
#endif
#ifndef NAR_TC_LD64
#define NAR_TC_LD64 1
#endif
#ifndef NAR_TC_ACOLL
#define NAR_TC_ACOLL 1
#endif
#ifndef NAR_TC_MAX_STAGES
#define NAR_TC_MAX_STAGES 3
#endif
__host__ __device__ constexpr int tc_stages(int N, int NB) {
  return (227 * 1024 - tc_fixed_smem(N)) / tc_stage_bytes(N, NB) > NAR_TC_MAX_STAGES
             ? NAR_TC_MAX_STAGES
             : (227 * 1024 - tc_fixed_smem(N)) / tc_stage_bytes(N, NB);
}
__host__ __device__ constexpr int tc_smem(int N, int NB) {
  return tc_stages(N, NB) * tc_stage_bytes(N, NB) + tc_fixed_smem(N);
}

// Padded output width of the f (and g) half: the kernel is instantiated for
// N = 2 * {8, 16, 24, 32, 48, 64, 96, 128}; other widths round up to the next
// one (the extra columns carry zero weights and bias, so they gate to 0).
__host__ __device__ constexpr int tc_coutp(int cout) {
  return cout <= 32 ? (cout + 7) / 8 * 8 : cout <= 48 ? 48 : cout <= 64 ? 64 : cout <= 96 ? 96 : 128;
}

// Host: pack HWIO f32 weights into bf16 [chunk q][tap][k8][n][8] where
// n < Coutp indexes f outputs and n >= Coutp g outputs (zero padded).  All
// weights (and, in the kernel, biases) are scaled by 1/2 -- exact in bf16 --
// so the accumulators hold f/2 and g/2, the operands of the epilogue's
// elu(f)/2 and tanh(g/2) (see gate_h).
// Sliding layers (tc_slide(N)): [chunk q][kx][k8][n' = (2 - ky) * N + n][8].
//
// Paired up2 chunks (pairs = true: a sliding layer whose source A is nearest-upsampled
// 2x): consecutive halo rows 2j-1, 2j read the same low-res row, so their two sliding
// MMAs merge into one with 4 stacked blocks per kx, [W2; W1+W2; W0+W1; W0] (n' = b*N + n,
// the sums in f32 before the bf16 rounding) feeding output rows 2j-3 .. 2j: source-A
// chunks are [chunk q][kx][k8][4N][8] (tc_b4_bytes), source-B chunks as above.  Plain
// layers (N = 96, 128) use the same blocks per output row pair (2p, 2p+1): blocks 1-2
// [W1+W2 | W0+W1] on low-res row p+1 in one N' = 2N MMA, W0 (block 3) on row p for
// row 2p and W2 (block 0) on row p+2 for row 2p+1 -- 3 MMAs per kx instead of 6.
inline void tc_pack_weights(const std::vector<float>& wf, const std::vector<float>& wg, int ca,
                            int cb, int cout, std::vector<uint16_t>& packed, bool pairs = false) {
  const int coutp = tc_coutp(cout), N = 2 * coutp;
  const bool slide = tc_slide(N);
  pairs = pairs && N <= 128;
  const int nqa = (ca + 15) / 16, nqb = (cb + 15) / 16, nq = nqa + nqb, cin = ca + cb;
  const size_t e3 = (size_t)9 * 2 * N * 8;      // elements of a plain chunk
  const size_t q4 = (size_t)3 * 2 * 4 * N * 8;  // ... of a paired chunk
  packed.assign(pairs ? nqa * q4 + nqb * e3 : (size_t)nq * e3, 0);
  // first element of chunk q
  auto chunk0 = [&](int q) { return pairs ? (q < nqa ? q * q4 : nqa * q4 + (q - nqa) * e3) : q * e3; };
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
            const float v = 0.5f * (is_g ? wg : wf)[((size_t)tap * cin + ci) * cout + j];
            if (pairs && in_a) continue;  // paired blocks: below
            if (slide) {
              const int ky = tap / 3, kx = tap % 3;
              const size_t np = (size_t)(2 - ky) * N + n;
              packed[chunk0(q) + (((size_t)kx * 2 + k8) * (3 * N) + np) * 8 + e] = bf16(v);
            } else {
              packed[chunk0(q) + (((size_t)tap * 2 + k8) * N + n) * 8 + e] = bf16(v);
            }
          }
  if (!pairs) return;
  for (int q = 0; q < nqa; ++q)
    for (int kx = 0; kx < 3; ++kx)
      for (int k8 = 0; k8 < 2; ++k8)
        for (int n = 0; n < N; ++n)
          for (int e = 0; e < 8; ++e) {
            const int ci = 16 * q + 8 * k8 + e;
            const bool is_g = n >= coutp;
            const int j = is_g ? n - coutp : n;
            if (ci >= ca || j >= cout) continue;
            const float* w = is_g ? wg.data() : wf.data();
            auto W = [&](int ky) { return w[((size_t)(ky * 3 + kx) * cin + ci) * cout + j]; };
            const float blk[4] = {W(2), W(1) + W(2), W(0) + W(1), W(0)};
            for (int b = 0; b < 4; ++b)
              packed[((((size_t)q * 3 + kx) * 2 + k8) * (4 * N) + (size_t)b * N + n) * 8 + e] =
                  bf16(0.5f * blk[b]);
          }
}

// ---------------------------------------------------------------------------
// device helpers (tcgen05 / TMEM / TMA)
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

// SWIZZLE_32B K-major (the TMA-written halo): rows of 32 B (K = 16 bf16),
// 8-row atoms of 256 B (SBO), LBO unused, layout type 6 at [61,64).  The start
// may sit at any 32-byte row: the XOR pattern follows absolute address bits.
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  // c_format F32 (1) at [4,6); a/b BF16 (1) at [7,10) / [10,13); K-major both;
  // N>>3 at [17,23); M>>4 at [24,29).
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// descriptor + byte offset: the start-address field is addr >> 4 in bits [0,14),
// and every shared-memory address < 256 KB fits it, so adding offset >> 4 never
// carries out of the field (one integer add instead of re-encoding the address)
__device__ __forceinline__ uint64_t desc_add(uint64_t d, uint32_t bytes) {
  return d + (uint64_t)(bytes >> 4);
}

// MMA issue and commit: called by one lane -- the one elect_one() picked (ptxas then
// knows a single thread issues and emits the UTCHMMAs back to back; behind a lane-0
// branch, or with elect.sync inside every asm, each MMA carried its own uniform loop or
// collective sequence)
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(e));
  return e != 0;
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

// The same MMA with an A-collector hint: 1 = fill (keep A for the next MMA), 2 = use
// (reuse the kept A, keep it), 3 = lastuse (reuse, then release) -- consecutive MMAs on
// the same A tile read it from shared memory once (A_KEEP / A_REUSE in SASS)
template <int kColl>
__device__ __forceinline__ void umma_bf16_c(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc) {
  static_assert(kColl >= 0 && kColl <= 3, "collector op");
#define NAR_UMMA_COLL(OP)                                                                  \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"                          \
               "tcgen05.mma.cta_group::1.kind::f16" OP " [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d), \
               "l"(adesc), "l"(bdesc), "r"(idesc)                                          \
               : "memory")
  if constexpr (kColl == 0) umma_bf16(tmem_d, adesc, bdesc, idesc, 1u);
  else if constexpr (kColl == 1) NAR_UMMA_COLL(".collector::a::fill");
  else if constexpr (kColl == 2) NAR_UMMA_COLL(".collector::a::use");
  else NAR_UMMA_COLL(".collector::a::lastuse");
#undef NAR_UMMA_COLL
}

// compile-time loop: f(integral_constant<int, I>) for I in [I0, I1)
template <int I0, int I1, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I0 < I1) {
    f(std::integral_constant<int, I0>{});
    static_for<I0 + 1, I1>(f);
  }
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// x64: two consecutive rows of an N = 32 layer ([f16 g16] x 2) in one load -- one
// instruction, so both rows' TMEM latency is paid once (ptxas sinks separate loads)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

// 32-byte global store (sm_100 STG.256): one full sector per lane
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t* w) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 3-D TMA tensor load (tile mode) into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// elu(f) * sigmoid(g) (autodiff.py:186-203) from the accumulators fh = f/2,
// gh = g/2 (bias included): with e = elu(f)/2 (fh, or (e^f - 1)/2 via ex2) and
// sigmoid(g) = (1 + tanh(g/2))/2, the gate is e + e*tanh(gh) -- 2 MUFU + 4
// FMA-pipe ops per output.
__device__ __forceinline__ float gate_h(float fh, float gh) {
#if defined(NAR_TC_GATE_MUFU0)  // timing experiments only (wrong numerics)
  return fmaf(fh, gh, fh);
#elif defined(NAR_TC_GATE_MUFU1)
  return fmaf(fh, tanh_approx(gh), fh);
#endif
  const float ex = ex2_approx(fh * 2.88539008177792681f);  // 2^(2 fh log2 e) = e^f
  const float e = fh > 0.0f ? fh : fmaf(0.5f, ex, -0.5f);
  const float t = tanh_approx(gh);
  return fmaf(e, t, e);
}


// timing experiments (build with -DNAR_TC_TRACE, run with NAR_TC_DEBUG bit 3): CTA 0 records clock64() stamps of its
// first kTraceTiles tiles -- [tile][0] MMA before the TMEM-empty wait, [1] after
// it, [2+2q]/[3+2q] after chunk q's full wait / after its MMAs are issued,
// [10]/[11] epilogue warp 1 after the TMEM-full wait / at the end of the tile,
// [12]/[13] producer before / after the empty wait of the tile's first chunk
constexpr int kTraceTiles = 16, kTraceSlots = 16;
__device__ unsigned long long g_tc_trace[kTraceTiles * kTraceSlots];
// (compiled in only with -DNAR_TC_TRACE: even dead, the checks cost the hot loops)
#ifdef NAR_TC_TRACE
#define TC_TRACE(tl, slot)                                                          \
  do {                                                                              \
    if ((a.debug & 8) && blockIdx.x == 0 && (tl) < kTraceTiles)                     \
      g_tc_trace[(tl) * kTraceSlots + (slot)] = clock64();                          \
  } while (0)
#else
#define TC_TRACE(tl, slot) \
  do {                     \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int N, bool kHead, int NB>
__global__ void __maxnreg__(96)
    gated_conv_tc(const ConvArgs a, const __grid_constant__ CUtensorMap tma_a,
                  const __grid_constant__ CUtensorMap tma_b) {
  constexpr int R = tc_rows(N, NB);
  constexpr int LR = tc_low_rows(N, NB);
  constexpr int S = tc_stages(N, NB);
  constexpr int A_BYTES = tc_a_bytes(N, NB);
  constexpr int B_BYTES = tc_b_bytes(N);
  constexpr int STAGE = tc_stage_bytes(N, NB);
  static_assert(A_BYTES % 128 == 0 && B_BYTES % 128 == 0, "align");
  constexpr uint32_t A_TX = (R + 2) * kHaloRowBytes;  // bytes of a direct halo box
  constexpr uint32_t UP_TX = LR * kHaloRowBytes;      // ... of a wide up2 halo box
  constexpr int COUTP = N / 2;
  constexpr uint32_t IDESC = umma_idesc_bf16(128, N);
  static_assert(NB * R * N <= 512, "TMEM budget");
  static_assert(S >= 2, "pipeline depth");

  // Programmatic dependent launch: the next layer's CTAs may be scheduled as soon
  // as every CTA of this one is running (they take an SM once ours leaves it, run
  // their prologue and wait in griddepcontrol.wait below for this grid to finish).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* fixed = smem + S * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(fixed);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;       // [buffer][row slot]
  uint64_t* tempty = tfull + 2 * kEpiGroups;
  uint32_t* tbase_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* sones = fixed + 512;                 // bias MMA operands (kTcOnesBytes)
  uint8_t* sbiasm = sones + kTcOnesBytes;       // (kTcBiasBytes)
  float* shead_w = reinterpret_cast<float*>(sbiasm + kTcBiasBytes);
  float* shead_b = shead_w + 512;
  constexpr bool SLIDE = tc_slide(N);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_x = (a.W + 127) / 128;
  const int tiles_y = (a.H + R - 1) / R;
  const int n_tiles = tiles_x * tiles_y;
  const int nqa = (a.ca + 15) / 16, nqb = (a.cb + 15) / 16, nq = nqa + nqb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      for (int g = 0; g < kEpiGroups; ++g) mbar_init(&tfull[b * kEpiGroups + g], 1);
      mbar_init(&tempty[b], 4 * kEpiGroups);
    }
    fence_mbar_init();
    prefetch_tmap(&tma_a);
    if (nqb) prefetch_tmap(&tma_b);
  }
  // bias MMA operands; columns beyond cout get bias 0, so their gate is
  // elu(0) * sigmoid(0) = 0 (padded output channels stay exact zeros)
  for (int i = threadIdx.x; i < (kTcOnesBytes + kTcBiasBytes) / 16; i += kTcThreads) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (i < 128) {
      v.x = 0x3F803F80u;  // A row i, k = 0, 1: 1.0
    } else if (i >= kTcOnesBytes / 16 && i < kTcOnesBytes / 16 + 256) {
      const int n = (i - kTcOnesBytes / 16) % N;  // B row -> accumulator column
      const int j = n < COUTP ? n : n - COUTP;
      const float b = j < a.cout ? 0.5f * (n < COUTP ? a.bias_f[j] : a.bias_g[j]) : 0.0f;
      const __nv_bfloat16 hi = __float2bfloat16_rn(b);
      const __nv_bfloat16 lo = __float2bfloat16_rn(b - __bfloat162float(hi));
      v.x = (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(lo) << 16);
    }
    reinterpret_cast<uint4*>(sones)[i] = v;
  }
  fence_proxy_async_smem();  // generic-proxy writes, read by the tensor core
  if (a.head_out)
    for (int i = threadIdx.x; i < a.cout * a.head_n; i += kTcThreads) shead_w[i] = a.head_w[i];
  if (a.head_out && threadIdx.x < a.head_n) shead_b[threadIdx.x] = a.head_b[threadIdx.x];
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tbase_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_slot;
  if (tbase != 0u) __trap();  // a 512-column allocation is always column 0 (the MMA issuer relies on it)
  // chunk q's packed weights: paired up2 chunks (4 stacked blocks) first
  constexpr uint32_t B3 = tc_b3_bytes(N), B4 = tc_b4_bytes(N);
  auto wchunk = [&](int q, size_t& boff) -> uint32_t {
    const bool in_a = q < nqa;
    boff = a.up2pair ? (in_a ? (size_t)q * B4 : (size_t)nqa * B4 + (size_t)(q - nqa) * B3)
                     : (size_t)q * B3;
    return a.up2pair && in_a ? B4 : B3;
  };
  // The weights do not depend on the previous layer: the first stages' weight
  // copies go out before the grid dependency wait (expect_tx without arrival; the
  // stage's arrive.expect_tx for its halo follows in the producer loop).
  int n_pre = 0;
  if (warp == 0 && lane == 0 && !(a.debug & 4) && NAR_TC_WEIGHT_PREFETCH) {
    const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    n_pre = my_tiles * nq < S ? my_tiles * nq : S;
    for (int it = 0; it < n_pre; ++it) {
      size_t boff;
      const uint32_t bbytes = wchunk(it % nq, boff);
      mbar_expect_tx_only(&full[it], bbytes);
      bulk_g2s(smem + it * STAGE + A_BYTES, reinterpret_cast<const uint8_t*>(a.wtc) + boff, bbytes,
               &full[it]);
    }
  }
  // Everything above touches only this launch's constant parameters; the
  // activations are the previous layer's output (and our output may still be
  // read by an earlier layer): wait for the prerequisite grid to complete.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp < kProdWarps) {
    // ------------------------------ producer ------------------------------
    // Stage `it` = (tile, 16-channel chunk q).  One lane TMA-loads the halo
    // straight into the UMMA SWIZZLE_32B layout [row][px][32 B] -- (R+2) x 136
    // pixels of a direct source (one box: 32-byte rows cost the TMA unit half
    // the row operations of two 16-byte slabs), or for a
    // wide up2 source the LR low-res rows behind them (already repeated
    // horizontally, so 130 wide pixels per row) -- plus the chunk's weights.
    if (lane == 0) {
      const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      const int n_it = my_tiles * nq;
      for (int it = 0; it < n_it; ++it) {
        const int tile = blockIdx.x + (it / nq) * gridDim.x, q = it % nq;
        const int y0 = (tile / tiles_x) * R, x0 = (tile % tiles_x) * 128;
        const int s = it % S;
        uint8_t* stA = smem + s * STAGE;
        const bool in_a = q < nqa;
        const bool up = in_a && a.a_up2;
        const int cbase = 16 * (in_a ? q : q - nqa);
        const CUtensorMap* map = in_a ? &tma_a : &tma_b;
        const int yr = up ? (y0 - 1) >> 1 : y0 - 1;  // arithmetic shift: row -1 stays OOB
        if (q == 0) TC_TRACE(it / nq, 12);
        mbar_wait(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
        if (q == 0) TC_TRACE(it / nq, 13);
        if (a.debug & 4) {  // timing experiment: no loads
          mbar_arrive(&full[s]);
          continue;
        }
        size_t boff;
        const uint32_t bbytes = wchunk(q, boff);
        const bool pre = it < n_pre;  // weights already in flight (before the grid wait)
        mbar_expect_tx(&full[s], (up ? UP_TX : A_TX) + (pre ? 0u : bbytes));
        tma_load_3d(stA, map, cbase, x0 - 1, yr, &full[s]);
        if (!pre)
          bulk_g2s(stA + A_BYTES, reinterpret_cast<const uint8_t*>(a.wtc) + boff, bbytes, &full[s]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------ MMA issuer -----------------------------
    // epilogue row slots (see tc_epi_rgroups): signalled in the last chunk -- sliding layers
    // with one commit per completion group (tc_epi_signal), plain layers row by row
    const int rstep = (!kHead && a.pool_out != nullptr) ? 2 : 1;
    const int units = R / rstep, rg = tc_epi_rgroups(units);
    int it = 0, tl = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tl) {
      const int b = tl % NB;
      uint64_t* tf = tfull + b * kEpiGroups;
      if (lane == 0) TC_TRACE(tl, 0);
      mbar_wait(&tempty[b], (((uint32_t)(tl / NB)) & 1u) ^ 1u);
      tc_fence_after();
      if (lane == 0) TC_TRACE(tl, 1);
      // one CTA per SM allocates all 512 TMEM columns, so the allocation is column 0
      // (checked at allocation): a compile-time base keeps the D addresses uniform
      const uint32_t dcol = (uint32_t)(b * R * N);
      const int y0 = (tile / tiles_x) * R;
      for (int q = 0; q < nq; ++q, ++it) {
        // halo row h -> smem row (h + par) >> sh: a wide up2 chunk holds each
        // low-res row once, and image row y0-1+h reads low-res row (y0-1+h) >> 1
        const bool up = a.a_up2 && q < nqa;
        const int sh = up ? 1 : 0, par = up ? ((y0 - 1) & 1) : 0;
        const int s = it % S;
        const bool last = q == nq - 1;
        mbar_wait(&full[s], (uint32_t)(it / S) & 1u);
        tc_fence_after();
        if (lane == 0 && q < 4) TC_TRACE(tl, 2 + 2 * q);
        if (!elect_one()) {
          // the other lanes only follow the loop (waits above, __syncwarp below)
        } else if (a.debug & 2) {
          umma_commit(&empty[s]);
          if (last)
            for (int g = 0; g < rg; ++g) umma_commit(&tf[g]);  // (all barriers: timing mode)
        } else {  // one elected lane issues this chunk's MMAs and commits
          const uint32_t sa = smem_u32(smem + s * STAGE);
          const uint32_t sb = sa + A_BYTES;
          if (q == 0) {  // this tile's R*N accumulator columns start at the bias
            const uint64_t ad = umma_desc(smem_u32(sones), 2048, 128);
            const uint64_t bd = umma_desc(smem_u32(sbiasm), 4096, 128);
#pragma unroll
            for (int c = 0; c < R * N; c += 256)
              umma_bf16(dcol + c, ad, bd, umma_idesc_bf16(128, R * N - c < 256 ? R * N - c : 256), 0u);
          }
          int slot = 0;  // next row slot to signal (last chunk)
          if constexpr (SLIDE) {
            // halo row h feeds output rows h-2..h (ky = 2, 1, 0): after h, rows <= h-2 are
            // complete.  kx outer, h inner and unrolled: consecutive MMAs share the B
            // block (h outer costs 75 vs 57 cycles per MMA, scripts/mma_slide_bench.cu).
            // With a.slide_blocks > 1 the last chunk runs its halo rows in two blocks and
            // signals the slots the first completes (default 1: one signal at the end --
            // every commit is a ~60-cycle bubble in the tensor pipe).
            auto rows = [&](auto h0c, auto h1c) {
              constexpr int H0 = decltype(h0c)::value, H1 = decltype(h1c)::value;
#pragma unroll 1
              for (int kx = 0; kx < 3; ++kx) {
                // [k8][3N][8]: LBO = 3N*16; descriptors encoded once, offsets added
                const uint64_t bk = umma_desc(sb + kx * (3 * N * 32), 3 * N * 16, 128);
                const uint64_t ak = umma_desc_sw32(sa + kx * 32);
#pragma unroll
                for (int h = H0; h < H1; ++h) {
                  const int kymax = h < 2 ? h : 2;
                  const int kymin = h - (R - 1) > 0 ? h - (R - 1) : 0;
                  const int nb = kymax - kymin + 1;
                  const uint64_t bdesc = desc_add(bk, (2 - kymax) * N * 16);
                  const uint64_t adesc =
                      desc_add(ak, (sh ? ((h + par) >> 1) : h) * kHaloRowBytes);
                  umma_bf16(dcol + (h - kymax) * N, adesc, bdesc, umma_idesc_bf16(128, nb * N), 1u);
                }
              }
              if (last) {  // one signal for all slots this block completed
                const int s0 = slot;
                while (slot < rg && H1 - 1 >= tc_epi_last_row(slot, units, rg, rstep) + 2) ++slot;
                if (slot > s0) umma_commit(&tf[s0]);
              }
            };
            constexpr int HM = R / 2 + 2;  // rows < R/2 are complete after halo row HM-1
            bool paired = false;
            if constexpr (R % 2 == 0) paired = a.up2pair && up;
            if (paired) {
              // paired up2 chunk (tc_pack_weights): halo rows 2g-1, 2g read low-res row g, one
              // MMA with blocks [W2; W1+W2; W0+W1; W0] covers output rows 2g-3 .. 2g (clipped
              // to the tile); halo rows 0 and R+1 stay single (W0 -> row 0, W2 -> row R-1)
#pragma unroll 1
              for (int kx = 0; kx < 3; ++kx) {
                // [k8][4N][8]: LBO = 4N*16
                const uint64_t bk = umma_desc(sb + kx * (4 * N * 32), 4 * N * 16, 128);
                const uint64_t ak = umma_desc_sw32(sa + kx * 32);
#pragma unroll
                for (int g = 0; g < R / 2 + 2; ++g) {
                  const int blk0 = g == 0 ? 3 : (3 - 2 * g > 0 ? 3 - 2 * g : 0);
                  const int blk1 = g == R / 2 + 1 ? 0 : (R + 2 - 2 * g < 3 ? R + 2 - 2 * g : 3);
                  const int drow = g == 0 ? 0 : (g == R / 2 + 1 ? R - 1 : 2 * g - 3 + blk0);
                  const uint64_t bdesc = desc_add(bk, blk0 * N * 16);
                  const uint64_t adesc = desc_add(ak, g * kHaloRowBytes);
                  umma_bf16(dcol + drow * N, adesc, bdesc, umma_idesc_bf16(128, (blk1 - blk0 + 1) * N), 1u);
                }
              }
              if (last) {  // (decoder layers end with the skip chunk; kept for completeness)
                const int nb = (a.slide_blocks > 1 && R >= 2) ? 2 : 1;
                for (int g = 0; g < rg; ++g)
                  if (tc_epi_signal(g, true, nb, units, rg, rstep, R) == g) umma_commit(&tf[g]);
                slot = rg;
              }
            } else if (last && a.slide_blocks > 1 && R >= 2) {
              rows(std::integral_constant<int, 0>{}, std::integral_constant<int, HM>{});
              rows(std::integral_constant<int, HM>{}, std::integral_constant<int, R + 2>{});
            } else {
              rows(std::integral_constant<int, 0>{}, std::integral_constant<int, R + 2>{});
            }
          } else if (R % 2 == 0 && a.up2pair && up) {
            // paired up2 chunk, plain layer (tc_pack_weights): per output row pair and kx
            // one N' = 2N MMA on the shared low-res row and two N MMAs for the outer taps
#pragma unroll 1
            for (int kx = 0; kx < 3; ++kx) {
              const uint32_t bk = sb + kx * (4 * N * 32);  // [k8][4N][8]: LBO = 4N*16
              const uint64_t b12 = umma_desc(bk + 1 * N * 16, 4 * N * 16, 128);
              const uint64_t b3 = umma_desc(bk + 3 * N * 16, 4 * N * 16, 128);
              const uint64_t b0 = umma_desc(bk, 4 * N * 16, 128);
              const uint64_t ax = umma_desc_sw32(sa + kx * 32);
#if NAR_TC_ACOLL
              // low-res row g outer: its (up to) three MMAs -- W0 into row 2g, W1+W2 into
              // rows 2g-2 / 2g-1, W2 into row 2g-3 -- reuse one A read (A collector)
              static_for<0, R / 2 + 2>([&](auto gc) {
                constexpr int G = decltype(gc)::value;
                constexpr bool U3 = G < R / 2, U12 = G >= 1 && G <= R / 2, U0 = G >= 2;
                constexpr int NU = (U3 ? 1 : 0) + (U12 ? 1 : 0) + (U0 ? 1 : 0);
                const uint64_t ag = desc_add(ax, G * kHaloRowBytes);
                constexpr int C3 = NU == 1 ? 0 : 1;
                constexpr int C12 = NU == 1 ? 0 : (U3 ? (U0 ? 2 : 3) : 1);
                constexpr int C0 = NU == 1 ? 0 : 3;
                if constexpr (U3) umma_bf16_c<C3>(dcol + 2 * G * N, ag, b3, IDESC);
                if constexpr (U12)
                  umma_bf16_c<C12>(dcol + 2 * (G - 1) * N, ag, b12, umma_idesc_bf16(128, 2 * N));
                if constexpr (U0) umma_bf16_c<C0>(dcol + (2 * (G - 2) + 1) * N, ag, b0, IDESC);
              });
#else
#pragma unroll
              for (int pr = 0; pr < R / 2; ++pr) {
                umma_bf16(dcol + 2 * pr * N, desc_add(ax, (pr + 1) * kHaloRowBytes), b12,
                          umma_idesc_bf16(128, 2 * N), 1u);
                umma_bf16(dcol + 2 * pr * N, desc_add(ax, pr * kHaloRowBytes), b3, IDESC, 1u);
                umma_bf16(dcol + (2 * pr + 1) * N, desc_add(ax, (pr + 2) * kHaloRowBytes), b0, IDESC,
                          1u);
              }
#endif
            }
            if (last) {  // (decoder layers end with the skip chunk; kept for completeness)
              for (int g = 0; g < rg; ++g) umma_commit(&tf[g]);
              slot = rg;
            }
          } else {
            const uint64_t b0 = umma_desc(sb, N * 16, 128);
            const uint64_t a0 = umma_desc_sw32(sa);
#if NAR_TC_ACOLL
            if (!up) {
              // halo row hr and shift kx outer, the output rows r = hr - ky it feeds inner:
              // each A tile is read from shared memory once per (hr, kx) (A collector)
              auto hrow = [&](auto hc) {
                constexpr int HR = decltype(hc)::value;
                constexpr int KYLO = HR - (R - 1) > 0 ? HR - (R - 1) : 0;
                constexpr int KYHI = HR < 2 ? HR : 2;
#pragma unroll
                for (int kx = 0; kx < 3; ++kx) {
                  const uint64_t adesc = desc_add(a0, HR * kHaloRowBytes + kx * 32);
                  auto one = [&](auto kyc) {
                    constexpr int KY = decltype(kyc)::value;
                    constexpr int C = KYLO == KYHI ? 0 : (KY == KYLO ? 1 : (KY == KYHI ? 3 : 2));
                    umma_bf16_c<C>(dcol + (HR - KY) * N, adesc,
                                   desc_add(b0, (3 * KY + kx) * (N * 32)), IDESC);
                  };
                  if constexpr (KYLO <= 0 && 0 <= KYHI) one(std::integral_constant<int, 0>{});
                  if constexpr (KYLO <= 1 && 1 <= KYHI) one(std::integral_constant<int, 1>{});
                  if constexpr (KYLO <= 2 && 2 <= KYHI) one(std::integral_constant<int, 2>{});
                }
                if (last)  // rows <= HR - 2 are complete
                  while (slot < rg && HR - 2 >= tc_epi_last_row(slot, units, rg, rstep))
                    umma_commit(&tf[slot++]);
              };
              static_for<0, R + 2>(hrow);
              if (last)
                while (slot < rg) umma_commit(&tf[slot++]);
            } else
#endif
#pragma unroll 1
            for (int r = 0; r < R; ++r) {
#pragma unroll
              for (int tap = 0; tap < 9; ++tap) {
                const int ky = tap / 3, kx = tap % 3;
                const uint64_t bdesc = desc_add(b0, tap * (N * 32));
                const uint64_t adesc =
                    desc_add(a0, ((r + ky + par) >> sh) * kHaloRowBytes + kx * 32);
                umma_bf16(dcol + r * N, adesc, bdesc, IDESC, 1u);
              }
              if (last)
                while (slot < rg && r >= tc_epi_last_row(slot, units, rg, rstep))
                  umma_commit(&tf[slot++]);
            }
          }
          umma_commit(&empty[s]);
          if (q < 4) TC_TRACE(tl, 3 + 2 * q);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------ epilogue -------------------------------
    // 16 warps: warp w covers TMEM lanes 32*(w%4)..+31 (pixels) and the row
    // groups g with g % 4 == (w-4)/4 (a group is one row, or two for pooling).
    // Channels are processed 8 at a time: one x8 TMEM load per branch and row,
    // one wait; padded channels come out as exact zeros.
    const int quarter = warp & 3;
    const int grp = (warp - kProdWarps) >> 2;
    const int m = quarter * 32 + lane;
    // kHead (the last layer): fused 1x1 out head, never pooled (host-checked)
    const bool do_pool = !kHead && a.pool_out != nullptr;  // requires R even (host-checked)
    constexpr bool do_head = kHead;
    const int rstep = do_pool ? 2 : 1;
    constexpr int RPW = (R + kEpiGroups - 1) / kEpiGroups;  // rows per warp, upper bound
    // With fewer row slots than groups (small R, or pooled row pairs) the
    // groups also split the channel chunks, so all 16 warps stay busy; the
    // head layer keeps whole channel ranges per warp (its logits sum them).
    const int units = R / rstep, rgroups = tc_epi_rgroups(units);
    const int cgroups = kEpiGroups / rgroups;
    const int rslot = grp % rgroups, cslot = grp / rgroups;
    // this warp's rows: units [u0, u1) of the tile (contiguous, see tc_epi_rgroups)
    const int u0 = tc_epi_first_unit(rslot, units, rgroups);
    const int u1 = tc_epi_first_unit(rslot + 1, units, rgroups);
    const int sig = tc_epi_signal(rslot, SLIDE, (a.slide_blocks > 1 && R >= 2) ? 2 : 1, units,
                                  rgroups, rstep, R);
    const int nc8 = a.cout_stride / 8;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int tl = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tl) {
      const int b = tl % NB;
      const int y0 = (tile / tiles_x) * R, x0 = (tile % tiles_x) * 128;
      mbar_wait(&tfull[b * kEpiGroups + sig], ((uint32_t)(tl / NB)) & 1u);
      tc_fence_after();
      if (warp == 1 && lane == 0) TC_TRACE(tl, 10);
      if (a.debug & 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        continue;
      }
      const int x = x0 + m;
      const bool xok = x < a.W;
      float logit[kHead ? RPW : 1][4];
      if (do_head) {
#pragma unroll
        for (int i = 0; i < RPW; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k) logit[i][k] = 0.0f;
      }
      if constexpr (kHead && COUTP % 16 == 0) {
        // fused out head (the last layer, <= 32 channels): rows one at a time, 16
        // channels per x16 TMEM load; the logits take the head weights from the
        // parameter bank (zero beyond cout / head_n, so no per-channel guards)
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          if (u0 + i >= u1) break;
          const int y = y0 + u0 + i;
          const bool ok = y < a.H && xok;
          float lg[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int c16 = 0; c16 < COUTP / 16; ++c16) {
            const int c0 = c16 * 16;
            float f[16], g[16], o[16];
            const uint32_t col = tbase + (uint32_t)(b * R * N + (u0 + i) * N + c0) + lane_off;
            tmem_ld16(col, f);
            tmem_ld16(col + COUTP, g);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = gate_h(f[e], g[e]);
            if (a.out != nullptr && ok) {
              uint32_t pw[8];
#pragma unroll
              for (int e = 0; e < 16; e += 2) {
                __nv_bfloat162 hh = __floats2bfloat162_rn(o[e], o[e + 1]);
                pw[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
              }
              st_global_v8(a.out + ((size_t)y * a.W + x) * a.cout_stride + c0, pw);
            }
#pragma unroll
            for (int e = 0; e < 16; ++e)
#pragma unroll
              for (int k = 0; k < 4; ++k) lg[k] = fmaf(o[e], a.head_wv[(c0 + e) * 4 + k], lg[k]);
          }
          if (ok) {
            float* dst = a.head_out + ((size_t)y * a.W + x) * a.head_n;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (k < a.head_n)
                dst[k] = fmaf(0.5f, tanh_approx(0.5f * (lg[k] + a.head_bv[k])), 0.5f);  // sigmoid
          }
        }
      } else if constexpr (!kHead && N == 32 && R == 8 && NAR_TC_LD64) {
        // N = 32 (16 channels): every warp owns two consecutive rows (4 row slots of
        // 8 rows, or of 4 pooled pairs); both rows' f and g come in one x64 load
        const int r0 = u0 * rstep;
        float v[64];
        tmem_ld64(tbase + (uint32_t)(b * R * N + r0 * N) + lane_off, v);
        tmem_wait_ld();
        float pacc[16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float o[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) o[e] = gate_h(v[32 * h + e], v[32 * h + 16 + e]);
          const int y = y0 + r0 + h;
          if (a.out != nullptr && y < a.H && xok) {
            uint32_t pw[8];
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              __nv_bfloat162 hh = __floats2bfloat162_rn(o[e], o[e + 1]);
              pw[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
            }
            const int wsh = a.out_wide;
            __nv_bfloat16* d = a.out + (((size_t)y * a.W + x) << wsh) * a.cout_stride;
            st_global_v8(d, pw);
            if (wsh) st_global_v8(d + a.cout_stride, pw);
          }
          if (do_pool) {
#pragma unroll
            for (int e = 0; e < 16; ++e) pacc[e] = h == 0 ? o[e] : pacc[e] + o[e];
          }
        }
        if (do_pool) {
#pragma unroll
          for (int e = 0; e < 16; ++e) pacc[e] += __shfl_xor_sync(0xffffffffu, pacc[e], 1);
          const int y = y0 + r0;
          if ((m & 1) == 0 && y < a.H && xok) {
            uint32_t pw[8];
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              __nv_bfloat162 hh = __floats2bfloat162_rn(0.25f * pacc[e], 0.25f * pacc[e + 1]);
              pw[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
            }
            st_global_v8(a.pool_out + ((size_t)(y >> 1) * (a.W >> 1) + (x >> 1)) * a.cout_stride, pw);
          }
        }
      } else if constexpr (!kHead && COUTP % 16 == 0) {
        // 16 channels at a time: one x16 TMEM load per branch, one 32-byte store
        // per lane (a full sector: 16-byte stores at the 32-byte pixel pitch of a
        // 16-channel layer left every sector half written); rows one at a time
        const int nc16 = a.cout_stride / 16;
        for (int c16 = cslot; c16 < nc16; c16 += cgroups) {
          const int c0 = c16 * 16;
          const bool have = c0 < COUTP;
#pragma unroll
          for (int i = 0; i < RPW; ++i) {
            if (u0 + i >= u1) break;
            const int r = (u0 + i) * rstep;
            float pacc[16];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h == 1 && !do_pool) break;
              float o[16];
              if (have) {
                float f[16], g[16];
                const uint32_t col = tbase + (uint32_t)(b * R * N + (r + h) * N + c0) + lane_off;
                tmem_ld16(col, f);
                tmem_ld16(col + COUTP, g);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e) o[e] = gate_h(f[e], g[e]);
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) o[e] = 0.0f;
              }
              const int y = y0 + r + h;
              if (a.out != nullptr && y < a.H && xok) {
                uint32_t pw[8];
#pragma unroll
                for (int e = 0; e < 16; e += 2) {
                  __nv_bfloat162 hh = __floats2bfloat162_rn(o[e], o[e + 1]);
                  pw[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
                }
                const int wsh = a.out_wide;  // wide (H, 2W) output: each pixel twice
                __nv_bfloat16* d = a.out + (((size_t)y * a.W + x) << wsh) * a.cout_stride + c0;
                st_global_v8(d, pw);
                if (wsh) st_global_v8(d + a.cout_stride, pw);
              }
              if (do_pool) {
#pragma unroll
                for (int e = 0; e < 16; ++e) pacc[e] = h == 0 ? o[e] : pacc[e] + o[e];
              }
            }
            if (do_pool) {
              // 2x2 average of the f32 outputs: rows r, r+1 here, columns m, m+1 via shuffle
#pragma unroll
              for (int e = 0; e < 16; ++e) pacc[e] += __shfl_xor_sync(0xffffffffu, pacc[e], 1);
              const int y = y0 + r;
              if ((m & 1) == 0 && y < a.H && xok) {
                uint32_t pw[8];
#pragma unroll
                for (int e = 0; e < 16; e += 2) {
                  __nv_bfloat162 hh = __floats2bfloat162_rn(0.25f * pacc[e], 0.25f * pacc[e + 1]);
                  pw[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
                }
                st_global_v8(a.pool_out + ((size_t)(y >> 1) * (a.W >> 1) + (x >> 1)) * a.cout_stride + c0,
                             pw);
              }
            }
          }
        }
      } else {
      // kHead: channel chunks unrolled (<= 4) so head weights index the
      // parameter bank with compile-time offsets
      constexpr int NC8_HEAD = 2 * ((COUTP + 15) / 16);
#pragma unroll
      for (int c8 = kHead ? 0 : cslot; c8 < (kHead ? NC8_HEAD : 1 << 20);
           c8 += (kHead ? 1 : cgroups)) {
        if (c8 >= nc8) break;
        const int c0 = c8 * 8;
        const bool have = c0 < COUTP;
        // rows of this warp: r = grp*rstep + i*4*rstep; unrolled so `slot`
        // (the logit row) is a compile-time index (registers, not local memory)
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          if (u0 + i >= u1) break;
          const int r = (u0 + i) * rstep;
          float o[2][8];
          float f[2][8], g[2][8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !do_pool) break;
            if (have) {
              const uint32_t col = tbase + (uint32_t)(b * R * N + (r + h) * N + c0) + lane_off;
              tmem_ld8(col, f[h]);
              tmem_ld8(col + COUTP, g[h]);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) f[h][e] = g[h][e] = 0.0f;
            }
          }
          if (have) tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !do_pool) break;
#pragma unroll
            for (int e = 0; e < 8; ++e) o[h][e] = gate_h(f[h][e], g[h][e]);
            const int y = y0 + r + h;
            const bool ok = y < a.H && xok;
            if (a.out != nullptr && ok) {
              uint4 pk;
              uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                __nv_bfloat162 hh = __floats2bfloat162_rn(o[h][e], o[h][e + 1]);
                pw[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
              }
              // wide (H, 2W) output: the consumer's horizontal up2 repeat
              const int wsh = a.out_wide;
              uint4* d = reinterpret_cast<uint4*>(
                  a.out + (((size_t)y * a.W + x) << wsh) * a.cout_stride + c0);
              *d = pk;
              if (wsh) d[a.cout_stride / 8] = pk;
            }
            if (do_head) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (c0 + e < a.cout)
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    if (k < a.head_n)
                      logit[kHead ? i : 0][k] =
                          fmaf(o[h][e], a.head_wv[((c0 + e) & 31) * 4 + k], logit[kHead ? i : 0][k]);
            }
          }
          if (do_pool) {
            // 2x2 average of the f32 outputs: rows r, r+1 here, columns m, m+1 via shuffle
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              v[e] = o[0][e] + o[1][e];
              v[e] += __shfl_xor_sync(0xffffffffu, v[e], 1);
            }
            const int y = y0 + r;
            if ((m & 1) == 0 && y < a.H && xok) {
              uint4 pk;
              uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                __nv_bfloat162 hh = __floats2bfloat162_rn(0.25f * v[e], 0.25f * v[e + 1]);
                pw[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
              }
              *reinterpret_cast<uint4*>(a.pool_out +
                                        ((size_t)(y >> 1) * (a.W >> 1) + (x >> 1)) * a.cout_stride +
                                        c0) = pk;
            }
          }
        }
      }
      }  // 8-channel chunks
      if (do_head && COUTP % 16 != 0) {  // (the 16-channel head path stored its own)
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          if (u0 + i >= u1) break;
          const int r = (u0 + i) * rstep;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !do_pool) break;
            const int y = y0 + r + h;
            if (y < a.H && xok) {
              float* dst = a.head_out + ((size_t)y * a.W + x) * a.head_n;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (k < a.head_n)
                  dst[k] = fmaf(0.5f, tanh_approx(0.5f * (logit[kHead ? i : 0][k] + a.head_bv[k])),
                                0.5f);  // sigmoid
            }
          }
        }
      }
      if (warp == 1 && lane == 0) TC_TRACE(tl, 11);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// host launch
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// NHWC bf16 tensor (h, w, cs) -> 3-D map over (channel, x, y), box {bc, bw, bh}.
static int tc_make_map(CUtensorMap* m, const void* base, int cs, int w, int h, int bc, int bw,
                       int bh, int pitch = 0) {
  auto fn = tc_encode_fn();
  if (!fn) return set_error(NAR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  // cs = 8 (a pyramid level): the 16-channel box still reads 32 bytes per pixel --
  // channels 8..15 overlap the next pixel (their weights are zero), so every box row
  // is in bounds (an out-of-bounds channel half makes TMA ~20 % slower); the last
  // pixel of a row reads the row's zero pad pixel (pitch = W + 2), never the next row
  cuuint64_t dims[3] = {(cuuint64_t)(cs < bc ? bc : cs), (cuuint64_t)w, (cuuint64_t)h};
  cuuint64_t strides[2] = {(cuuint64_t)cs * 2, (cuuint64_t)cs * 2 * (cuuint64_t)(pitch ? pitch : w)};
  cuuint32_t box[3] = {(cuuint32_t)bc, (cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(NAR_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return NAR_OK;
}

// Single TMEM buffer (twice the rows) only for weight-heavy layers where the
// bigger tile costs no extra wave; the rest keep double buffering's overlap.
inline int tc_sm_count() {
  static int sms[kMaxDevices] = {};
  const int dev = current_device();
  if (!sms[dev] && cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms[dev] = 148;
  return sms[dev];
}
inline int tc_bufs_for(int N, int H, int W, int nq) {
  // weight-heavy: N = 256 always; N = 128 from 8 chunks (decoder concat layers)
  if (N < 128 || (N < 256 && nq < 8)) return 2;
  const int R1 = tc_rows(N, 1), R2 = tc_rows(N, 2), sms = tc_sm_count();
  const int w1 = (((W + 127) / 128) * ((H + R1 - 1) / R1) + sms - 1) / sms;  // waves of tiles
  const int w2 = (((W + 127) / 128) * ((H + R2 - 1) / R2) + sms - 1) / sms;
  return w1 * R1 <= w2 * R2 ? 1 : 2;  // no more row-waves with the bigger tile
}
inline int tc_rows_for(int cout, int H, int W, int nq) {
  const int N = 2 * tc_coutp(cout);
  return tc_rows(N, tc_bufs_for(N, H, W, nq));
}

template <int N, bool kHead, int NB>
static int tc_launch_nhb(const ConvArgs& a, cudaStream_t st) {
  // kernel attributes are per device: set once on each device used
  static bool attr_done[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr_done[dev]) {
    const cudaError_t e =
        cudaFuncSetAttribute(gated_conv_tc<N, kHead, NB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(N, NB));
    if (e != cudaSuccess) {
      char msg[160];
      snprintf(msg, sizeof(msg), "cannot set conv smem size %d: %s", tc_smem(N, NB),
               cudaGetErrorString(e));
      return set_error(NAR_ERR_CUDA, msg);
    }
    attr_done[dev] = true;
  }
  constexpr int R = tc_rows(N, NB);
  if (a.pool_out && (R & 1)) return set_error(NAR_ERR_CONFIG, "fused pool needs an even row tile");
  CUtensorMap ma, mb;
  int rc;
  if (a.a_up2 == 1) return set_error(NAR_ERR_CONFIG, "tensor-core up2 needs a wide source");
  if (a.out_wide && (a.pool_out || a.head_out))
    return set_error(NAR_ERR_CONFIG, "wide output cannot be pooled or headed");
  if (a.a_up2)  // wide (H/2, W) source: LR low-res rows, 136 wide pixels
    rc = tc_make_map(&ma, a.src_a, a.ca_stride, a.W, a.H / 2, 16, kHaloPitch, tc_low_rows(N, NB));
  else
    rc = tc_make_map(&ma, a.src_a, a.ca_stride, a.W, a.H, 16, kHaloPitch, R + 2, a.a_pitch);
  if (rc) return rc;
  if (a.cb) {
    rc = tc_make_map(&mb, a.src_b, a.cb_stride, a.W, a.H, 16, kHaloPitch, R + 2, a.b_pitch);
    if (rc) return rc;
  } else {
    mb = ma;
  }
  const int sms = tc_sm_count();
  const int tiles = ((a.W + 127) / 128) * ((a.H + R - 1) / R);
  const int grid = tiles < sms ? tiles : sms;
  nar::count_launch();
  // launched as a programmatic dependent of the previous kernel on the stream
  // (NAR_TC_PDL=0 turns it off for timing comparisons)
  static const bool pdl = [] {
    const char* e = getenv("NAR_TC_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = tc_smem(N, NB);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, gated_conv_tc<N, kHead, NB>, a, ma, mb);
  if (e != cudaSuccess) return set_error(NAR_ERR_CUDA, cudaGetErrorString(e));
  return check_launch("gated_conv_tc");
}

template <int N, bool kHead>
static int tc_launch_nh(const ConvArgs& a, cudaStream_t st) {
  if constexpr (N == 128 || N == 256) {
    const int nq = (a.ca + 15) / 16 + (a.cb + 15) / 16;
    if (tc_bufs_for(N, a.H, a.W, nq) == 1) return tc_launch_nhb<N, kHead, 1>(a, st);
  }
  return tc_launch_nhb<N, kHead, 2>(a, st);
}

template <int N>
static int tc_launch_n(const ConvArgs& a, cudaStream_t st) {
  if (!a.head_out) return tc_launch_nh<N, false>(a, st);
  if constexpr (N <= 64) {
    if (a.pool_out) return set_error(NAR_ERR_CONFIG, "fused out head cannot be pooled");
    return tc_launch_nh<N, true>(a, st);
  } else {
    return set_error(NAR_ERR_CONFIG, "fused out head needs a layer of <= 32 channels");
  }
}

inline int tc_launch_gated_conv(const ConvArgs& a, cudaStream_t st) {
  if (a.cout < 1 || a.cout > 128) return set_error(NAR_ERR_CONFIG, "conv width must be 1..128");
  const int coutp = tc_coutp(a.cout);
  if (a.cout_stride % 8 || a.cout_stride < (a.cout + 7) / 8 * 8)
    return set_error(NAR_ERR_CONFIG, "conv output stride must be a multiple of 8 >= Cout");
  // (stride 8 < the 16-channel box: see tc_make_map -- rows need a zero pad pixel)
  if (a.ca_stride % 8 || (a.cb && a.cb_stride % 8))
    return set_error(NAR_ERR_CONFIG, "conv input strides must be multiples of 8");
  if ((a.ca_stride < 16 && a.a_pitch <= a.W) || (a.cb && a.cb_stride < 16 && a.b_pitch <= a.W))
    return set_error(NAR_ERR_CONFIG, "8-channel conv inputs need a zero pad pixel per row");
  if (a.head_out && (a.head_n < 1 || a.head_n > 4))
    return set_error(NAR_ERR_CONFIG, "fused out head supports 1..4 outputs");
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
