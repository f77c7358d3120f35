// Microbenchmark: MUFU throughput per SM for the gate's transcendental forms
// (f32 ex2 / tanh, packed f16x2 ex2 / tanh, bf16x2 tanh).  16 warps per SM,
// 8 independent chains per thread; prints element results per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float x[8];
  uint32_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = -0.001f * (threadIdx.x + i);
    __half2 t = __floats2half2_rn(x[i], x[i] * 0.5f);
    h[i] = *reinterpret_cast<uint32_t*>(&t);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 1) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      if (OP == 3) asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(h[i]));
      if (OP == 4) asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(h[i]));
      if (OP == 5) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 6) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %0;" : "+r"(h[i]) : "f"(x[i]));
      if (OP == 7) asm volatile("cvt.rn.f16x2.f32 %0, %1, %0;" : "+r"(h[i]) : "f"(x[i]));
      if (OP == 8) {  // MUFU and the bf16 pack interleaved: one pipe or two?
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %0;" : "+r"(h[i]) : "f"(x[i ^ 1]));
      }
      if (OP == 9) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x[i]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + __uint_as_float(h[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8);
  const char* names[] = {"ex2.f32", "tanh.f32", "ex2.f16x2", "tanh.f16x2", "tanh.bf16x2", "rcp.f32",
                         "cvt.bf16x2", "cvt.f16x2", "ex2+cvt.bf16x2", "ffma"};
  const int iters = 4096;
  for (int op = 0; op < 10; ++op) {
    void (*ks[])(float*, int, long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>};
    auto f = ks[op];
    f<<<sms, 512>>>(out, iters, cyc);
    f<<<sms, 512>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = 512.0 * iters * 8;  // instructions' lanes per SM
    const double elems = ops * (op >= 2 && op <= 4 ? 2 : op == 8 ? 2 : 1);
    printf("%-12s %6.2f lane-ops/clk/SM  %6.2f elements/clk/SM  (%lld cycles)\n", names[op], ops / c,
           elems / c, c);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
