// Measures the max relative error of rcp.approx.ftz.f64 (MUFU.RCP64H) over
// [0.1, 2e5] -- the input domain of the render kernel's reciprocal.
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, int n) {
  double worst = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    // log-uniform sweep of [0.1, 2e5]
    double x = 0.1 * exp(14.5087 * ((i + 0.5) / n));
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double t = __drcp_rn(x);
    double rel = fabs(y - t) / t;
    worst = fmax(worst, rel);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = worst;
}
int main() {
  const int threads = 256, blocks = 592, n = 1 << 26;
  double* d; cudaMalloc(&d, threads * blocks * 8);
  k<<<blocks, threads>>>(d, n);
  double* h = new double[threads * blocks];
  cudaMemcpy(h, d, threads * blocks * 8, cudaMemcpyDeviceToHost);
  double w = 0; for (int i = 0; i < threads * blocks; ++i) w = w > h[i] ? w : h[i];
  printf("rcp.approx.ftz.f64 max rel err = %.3e (2^%.2f)\n", w, log2(w));
  return 0;
}
