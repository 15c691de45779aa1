// Library plumbing for libdm_moe.so: error strings, device queries, the TMA
// encoder entry point and the launch counter. No kernels live here.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
#include <map>
#include <tuple>
#include <mutex>
#include <utility>

#include "dm_internal.h"

namespace dm {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(cudaError_t err, const char* what) {
  snprintf(g_err, sizeof(g_err), "%s: %s (%d)", what, cudaGetErrorString(err), (int)err);
  return (int)err;
}

int num_sms_current() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int ensure_smem_attr(const void* func, int bytes, const char* what) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;   // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error(e, what);
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(func, dev);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return DM_OK;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return set_cuda_error(e, what);
  done[key] = bytes;
  return DM_OK;
}

int max_active_blocks(const void* func, int threads, size_t smem) {
  static std::mutex mu;
  // (kernel, device, threads, dynamic smem) -> blocks per SM. Query after the kernel's
  // dynamic-smem attribute is raised (ensure_smem_attr): above 48 KB the query fails before.
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(func, dev, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, func, threads, smem) != cudaSuccess || n < 1) n = 1;
  cache[key] = n;
  return n;
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace dm

extern "C" {

int dm_version(void) { return DM_ABI_VERSION; }

const char* dm_last_error_string(void) { return dm::g_err; }

int dm_num_sms(int device) {
  int n = 0;
  cudaError_t e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return -dm::set_cuda_error(e, "cudaDeviceGetAttribute");
  return n;
}

long long dm_launch_count(void) { return dm::g_launches.load(); }

int dm_capacity_rows_fn(int T, int E, int k) { return dm_capacity_rows(T, E, k); }

size_t dm_route_workspace_size_fn(int T, int H, int E, int k) { return dm_route_workspace_size(T, H, E, k); }

size_t dm_router_wgrad_workspace_size_fn(int T, int H, int E) { return dm_router_wgrad_workspace_size(T, H, E); }

}  // extern "C"
