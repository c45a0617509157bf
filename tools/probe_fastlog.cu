// Standalone probe (not part of the product): the branch-free FP64 division
// and log of the K7 fixup (pf_common.cuh fast_div_rn / fast_log) against
// CUDA's __ddiv_rn and log on random inputs of the fixup's domain.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I include tools/probe_fastlog.cu -o tools/probe_fastlog.bin
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1708_02845_b200/csrc/pf_common.cuh"

__device__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull; x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull; return x ^ (x >> 31);
}

__global__ void check(int64_t n, unsigned long long *hist_div, unsigned long long *hist_log,
                      unsigned long long *worst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = mix(2 * i), b = mix(2 * i + 1);
    // t, q in [1e-300, 1]: log-uniform mostly, plus q ~ t pairs (ratios near 1)
    const double ea = -(double)(a % 1000000) / 1000000.0 * 690.0;
    const double t = exp(ea);
    double q;
    if (b & 1) q = exp(-(double)((b >> 1) % 1000000) / 1000000.0 * 690.0);
    else q = t * (1.0 + ((double)((b >> 1) % 2000001) - 1000000.0) * 1e-12);
    const double r0 = __ddiv_rn(t, q), r1 = pf::fast_div_rn(t, q);
    const long long dd = llabs(__double_as_longlong(r0) - __double_as_longlong(r1));
    atomicAdd(&hist_div[dd > 3 ? 3 : dd], 1ull);
    const double l0 = log(r0), l1 = pf::fast_log(r0);
    const long long dl = llabs(__double_as_longlong(l0) - __double_as_longlong(l1));
    atomicAdd(&hist_log[dl > 3 ? 3 : dl], 1ull);
    atomicMax(worst, (unsigned long long)dl);
  }
}

int main() {
  unsigned long long *h; cudaMalloc(&h, 9 * 8); cudaMemset(h, 0, 9 * 8);
  const int64_t n = 1ll << 28;
  check<<<148 * 8, 256>>>(n, h, h + 4, h + 8);
  std::vector<unsigned long long> v(9); cudaMemcpy(v.data(), h, 72, cudaMemcpyDeviceToHost);
  printf("{\"n\": %lld, \"div_ulp_0_1_2_3+\": [%llu, %llu, %llu, %llu], "
         "\"log_ulp_vs_cuda_0_1_2_3+\": [%llu, %llu, %llu, %llu], \"log_worst_ulp\": %llu}\n",
         (long long)n, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8]);
  return 0;
}
