// pf_runtime.cu — error plumbing and device queries behind the C ABI.
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "pf_common.cuh"

namespace pf {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return static_cast<int>(e);
  }
  return 0;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

// Occupancy and dynamic-smem attributes are cached per (device, kernel,
// shape): the driver queries cost tens of microseconds of host time, which
// the GPU would otherwise idle through in front of short launches.
namespace {
std::mutex g_cache_mu;
std::map<std::tuple<int, const void *, int, size_t>, int> g_occ;
std::map<std::pair<int, const void *>, size_t> g_smem;
}  // namespace

int occupancy(const void *kernel, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, kernel, threads, smem);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
  }
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, smem) !=
          cudaSuccess ||
      blocks <= 0) {
    cudaGetLastError();
    return 1;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_occ[key] = blocks;
  return blocks;
}

int ensure_smem(const void *kernel, size_t smem) {
  if (smem <= 48 * 1024) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(dev, kernel);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_smem.find(key);
  if (it != g_smem.end() && it->second >= smem) return 0;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
  if (e != cudaSuccess)
    return fail(static_cast<int>(e), "dynamic smem %zu B: %s", smem, cudaGetErrorString(e));
  g_smem[key] = smem;
  return 0;
}

}  // namespace pf

extern "C" {

int pf_version(void) { return 1; }

const char *pf_last_error(void) { return pf::g_err; }

int pf_sm_count(void) { return pf::sm_count(); }

}  // extern "C"
