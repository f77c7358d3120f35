// capi.cu -- library-level C ABI: versioning, error reporting, pinned host
// memory.  Errors never cross the ABI as exceptions: every entry point
// returns a status and leaves a thread-local message (nar_last_error).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "nar_b200.h"

namespace nar {

static thread_local std::string g_last_error;

int set_error(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return NAR_OK;
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_error(NAR_ERR_CUDA, m.c_str());
}

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_total() { return g_launches.load(std::memory_order_relaxed); }

// Scratch from cudaMallocAsync stays mapped in the device's default pool (its
// release threshold is 0 by default, so every synchronisation would hand the
// memory back and the next call would map it again).
void keep_pool_memory() {
  static std::once_flag once[kMaxDevices];
  std::call_once(once[current_device()], [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

// A persistent pool of host threads for host-side passes over a frame (the
// attribute gather of nar_host_gather_rgb): the calling thread works too, and a
// call returns once every range is done.  Calls are serialised.
namespace {
struct HostPool {
  std::mutex mu, call_mu;
  std::condition_variable cv, done_cv;
  std::vector<std::thread> workers;
  const std::function<void(int64_t, int64_t)>* fn = nullptr;
  int64_t n = 0, chunk = 1;
  std::atomic<int64_t> next{0};
  int active = 0;
  uint64_t gen = 0;
  bool stop = false;

  explicit HostPool(int nt) {
    for (int t = 0; t < nt; ++t) workers.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& w : workers) w.join();
  }
  void work() {
    for (;;) {
      const int64_t b = next.fetch_add(chunk);
      if (b >= n) return;
      (*fn)(b, b + chunk < n ? b + chunk : n);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return stop || gen != seen; });
      if (stop) return;
      seen = gen;
      lk.unlock();
      work();
      lk.lock();
      if (--active == 0) done_cv.notify_all();
    }
  }
  void run(int64_t count, const std::function<void(int64_t, int64_t)>& f) {
    std::lock_guard<std::mutex> call(call_mu);
    {
      std::lock_guard<std::mutex> lk(mu);
      fn = &f;
      n = count;
      const int64_t parts = 8 * (int64_t)(workers.size() + 1);
      chunk = count / parts > 4096 ? count / parts : 4096;
      next.store(0);
      active = (int)workers.size();
      ++gen;
    }
    cv.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return active == 0; });
    fn = nullptr;
  }
};
}  // namespace

void host_parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& f) {
  if (n <= 0) return;
  static HostPool pool([] {
    const char* e = getenv("NAR_HOST_THREADS");
    const int hw = (int)std::thread::hardware_concurrency();
    const int t = e ? atoi(e) : (hw > 0 ? hw : 1);
    return (t > 64 ? 64 : (t < 1 ? 1 : t)) - 1;  // + the calling thread
  }());
  // small passes inline; after a fork the pool's threads do not exist in the child
  static const pid_t owner = getpid();
  if (n < 65536 || getpid() != owner) {
    f(0, n);
    return;
  }
  pool.run(n, f);
}

}  // namespace nar

extern "C" {

const char* nar_version(void) { return "nar_b200 0.1.0 (sm_100a)"; }

const char* nar_last_error(void) { return nar::g_last_error.c_str(); }

int nar_device_count(int32_t* count) {
  if (!count) return nar::set_error(NAR_ERR_INVALID, "NULL count");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return NAR_OK;
  }
  *count = n;
  return NAR_OK;
}

int nar_host_alloc(void** ptr, size_t bytes) {
  if (!ptr) return nar::set_error(NAR_ERR_INVALID, "NULL out pointer");
  if (cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nar::set_error(NAR_ERR_NOMEM, "cudaHostAlloc failed");
  }
  return NAR_OK;
}

int nar_host_free(void* ptr) {
  if (ptr && cudaFreeHost(ptr) != cudaSuccess) {
    cudaGetLastError();
    return nar::set_error(NAR_ERR_CUDA, "cudaFreeHost failed");
  }
  return NAR_OK;
}

uint64_t nar_launch_count(void) { return nar::launch_total(); }

int nar_host_mapped_pointer(const void* host, void** dev) {
  if (!host || !dev) return nar::set_error(NAR_ERR_INVALID, "NULL argument");
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError();
    return nar::set_error(NAR_ERR_INVALID, "pointer is not CUDA host memory");
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer)
    return nar::set_error(NAR_ERR_INVALID, "pointer is not mapped pinned host memory");
  *dev = a.devicePointer;
  return NAR_OK;
}

int nar_host_register(void* host, size_t bytes) {
  if (!host || !bytes) return nar::set_error(NAR_ERR_INVALID, "NULL or empty range");
  const cudaError_t e =
      cudaHostRegister(host, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    std::string m = std::string("cudaHostRegister failed: ") + cudaGetErrorString(e);
    return nar::set_error(NAR_ERR_INVALID, m.c_str());
  }
  return NAR_OK;
}

int nar_host_unregister(void* host) {
  if (!host) return nar::set_error(NAR_ERR_INVALID, "NULL pointer");
  if (cudaHostUnregister(host) != cudaSuccess) {
    cudaGetLastError();
    return nar::set_error(NAR_ERR_INVALID, "range was not registered");
  }
  return NAR_OK;
}

}  // extern "C"
