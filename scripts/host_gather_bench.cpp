// Host gather microbenchmark: 2M random 3-byte rgb reads from a 1.05 GB array with T
// threads (software prefetch D ahead), as a host-side alternative to the resolve's
// zero-copy PCIe gathers.  g++ -O3 -pthread host_gather_bench.cpp
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t n = 350000000, m = 2073600;
  uint8_t* rgb = (uint8_t*)aligned_alloc(4096, n * 3);
  memset(rgb, 7, n * 3);
  std::vector<uint32_t> idx(m);
  uint64_t s = 88172645463325252ull;
  for (size_t i = 0; i < m; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; idx[i] = (uint32_t)(s % n); }
  std::vector<uint32_t> out(m);
  const unsigned hw = std::thread::hardware_concurrency();
  printf("hardware threads %u\n", hw);
  for (int T : {1, 4, 8, 16, 32, 64}) {
    if ((unsigned)T > hw) break;
    for (int D : {0, 16, 32, 64}) {
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
          th.emplace_back([&, t] {
            const size_t b = m * t / T, e = m * (t + 1) / T;
            for (size_t i = b; i < e; ++i) {
              if (D && i + D < e) __builtin_prefetch(rgb + (size_t)idx[i + D] * 3);
              const uint8_t* c = rgb + (size_t)idx[i] * 3;
              out[i] = c[0] | (c[1] << 8) | (c[2] << 16);
            }
          });
        for (auto& x : th) x.join();
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms < best) best = ms;
      }
      printf("T=%2d prefetch=%2d  %.2f ms\n", T, D, best);
    }
  }
  uint64_t sum = 0;
  for (auto v : out) sum += v;
  printf("checksum %llu\n", (unsigned long long)sum);
}
