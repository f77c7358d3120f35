// capi.cu -- library-level C ABI: versioning, error reporting, pinned host
// memory.  Errors never cross the ABI as exceptions: every entry point
// returns a status and leaves a thread-local message (nar_last_error).
#include <cuda_runtime.h>
#include <stdio.h>

#include <atomic>
#include <mutex>
#include <string>

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
