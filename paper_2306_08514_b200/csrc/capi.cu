// C-ABI housekeeping: error strings, launch counter, version.
#include <atomic>
#include <string.h>

#include "frontend_warp.cuh"

namespace srpgpu {

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};
static std::atomic<int> g_frontend_kernel{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

int frontend_kernel_choice() { return g_frontend_kernel.load(std::memory_order_relaxed); }

}  // namespace srpgpu

extern "C" const char* srpgpu_last_error(void) { return srpgpu::g_err; }

extern "C" int srpgpu_abi_version(void) { return SRPGPU_ABI_VERSION; }

extern "C" uint64_t srpgpu_launch_count(void) {
  return (uint64_t)srpgpu::g_launches.load(std::memory_order_relaxed);
}

extern "C" int srpgpu_device_sync(void) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    srpgpu::set_error("device sync: %s", cudaGetErrorString(e));
    return SRPGPU_ERR_LAUNCH;
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_set_frontend_kernel(int32_t which) {
  if (which < 0 || which > 3) {
    srpgpu::set_error("frontend kernel choice %d not in 0..3", which);
    return SRPGPU_ERR_VALUE;
  }
  srpgpu::g_frontend_kernel.store(which, std::memory_order_relaxed);
  return SRPGPU_OK;
}
