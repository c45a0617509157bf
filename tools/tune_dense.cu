// Standalone tuner for the dense field kernels (not part of the product).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        tools/tune_dense.cu -o build/tune_dense
// Times KL/TV template variants and a pure streaming-read ceiling on
// synthetic P of the C2 shape (rows x k FP64, ld = round_up(k,16)).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>

#include "../paper_1708_02845_b200/csrc/pf_runtime.cu"
#include "../paper_1708_02845_b200/csrc/dense.cu"

using namespace pf;



__global__ void fill_kernel(double *P, int64_t rows, int64_t k, int64_t ld) {
  int64_t n = rows * ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = i % ld;
    uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    P[i] = (c == 0 || c >= k) ? 0.0 : u / (double)k;
  }
}

// pure read ceiling: sum of every element, warp per row, same layout
template <int U>
__global__ void __launch_bounds__(256) read_kernel(const double *P, int64_t ld, int64_t rows,
                                                   int64_t k, double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t npair = k >> 1;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const double2 *row = reinterpret_cast<const double2 *>(P + r * ld);
    double a = 0;
    for (int64_t j0 = 0; j0 < npair; j0 += 32 * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int64_t j = j0 + lane + 32 * u;
        v[u] = j < npair ? ldg_stream2(row + j) : make_double2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) a += v[u].x + v[u].y;
    }
    a = warp_sum(a);
    if (lane == 0) out[r] = a;
  }
}

template <typename F>
float time_ms(F f, int reps = 10) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> ts;
  for (int i = 0; i < 3; ++i) f();
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main(int argc, char **argv) {
  int64_t rows = argc > 1 ? atoll(argv[1]) : 102104;
  int64_t k = argc > 2 ? atoll(argv[2]) : 4250;
  int64_t ld = round_up(k, 16), k_pad = round_up(k, 2), m_pad = round_up(k, 16);
  double *P, *H, *out, *tgt, *logt;
  uint8_t *tmask;
  uint32_t *flags;
  cudaMalloc(&P, rows * ld * 8);
  cudaMalloc(&H, rows * 8);
  cudaMalloc(&out, rows * 8);
  cudaMalloc(&tgt, k_pad * 8);
  cudaMalloc(&logt, k_pad * 8);
  cudaMalloc(&tmask, m_pad);
  cudaMalloc(&flags, 16);
  fill_kernel<<<4096, 256>>>(P, rows, k, ld);
  pf_row_negentropy_f64(P, ld, rows, k, 1e-300, H, nullptr, 0);
  pf_target_prep_f64(P + (rows / 3) * ld, k, 1e-300, tgt, logt, tmask, flags, 0);
  cudaDeviceSynchronize();
  const double bytes_kl = rows * (8.0 * k + 16) + 8.0 * k;
  const double bytes_tv = rows * (8.0 * k + 8) + 8.0 * k;
  const double bytes_rd = rows * (8.0 * k + 8);
  int sms = sm_count();
  printf("rows=%lld k=%lld sms=%d\n", (long long)rows, (long long)k, sms);

  auto run_read = [&](auto kern, const char *name) {
    int occ = occupancy((const void *)kern, 256, 0);
    int grid = sms * occ;
    float ms = time_ms([&] { kern<<<grid, 256>>>(P, ld, rows, k, out); });
    printf("%-28s occ=%d %8.4f ms %8.1f GB/s\n", name, occ, ms, bytes_rd / ms / 1e6);
  };
  run_read(read_kernel<2>, "read<2>");
  run_read(read_kernel<4>, "read<4>");
  run_read(read_kernel<8>, "read<8>");

  size_t smem = staged_smem_bytes(k_pad, m_pad);
  auto run_kl = [&](auto kern, const char *name) {
    int grid = 0;
    launch_cfg(kern, smem, rows, &grid);
    int occ = grid / sms;
    float ms = time_ms([&] {
      kern<<<grid, 256, smem>>>(P, ld, rows, k, k_pad, m_pad, H, tgt, logt, tmask, 1e-300,
                                1e-3, 0, rows / 3, nullptr, out, flags);
    });
    printf("%-28s occ=%d %8.4f ms %8.1f GB/s\n", name, occ, ms, bytes_kl / ms / 1e6);
  };
  run_kl(dense_kl_kernel<2, 1>, "kl<2,1>");
  run_kl(dense_kl_kernel<4, 1>, "kl<4,1>");
  run_kl(dense_kl_kernel<8, 1>, "kl<8,1>");
  run_kl(dense_kl_kernel<4, 5>, "kl<4,5>");
  run_kl(dense_kl_kernel<2, 5>, "kl<2,5>");
  {
    size_t keep = smem;
    smem = 0;
    run_kl(dense_kl_kernel<4, 5, false>, "kl<4,5,L1>");
    run_kl(dense_kl_kernel<4, 6, false>, "kl<4,6,L1>");
    run_kl(dense_kl_kernel<4, 8, false>, "kl<4,8,L1>");
    run_kl(dense_kl_kernel<2, 8, false>, "kl<2,8,L1>");
    run_kl(dense_kl_kernel<8, 4, false>, "kl<8,4,L1>");
    run_kl(dense_kl_kernel<6, 5, false>, "kl<6,5,L1>");
    smem = keep;
  }
  auto run_tv = [&](auto kern, const char *name) {
    int grid = 0;
    launch_cfg(kern, smem, rows, &grid);
    int occ = grid / sms;
    float ms = time_ms([&] {
      kern<<<grid, 256, smem>>>(P, ld, rows, k, k_pad, m_pad, tgt, tmask, 1e-150, 0, rows / 3,
                                nullptr, out, flags);
    });
    printf("%-28s occ=%d %8.4f ms %8.1f GB/s\n", name, occ, ms, bytes_tv / ms / 1e6);
  };
  run_tv(dense_tv_kernel<2, 1>, "tv<2,1>");
  run_tv(dense_tv_kernel<4, 1>, "tv<4,1>");
  run_tv(dense_tv_kernel<8, 1>, "tv<8,1>");
  run_tv(dense_tv_kernel<4, 5>, "tv<4,5>");
  {
    size_t keep = smem;
    smem = 0;
    run_tv(dense_tv_kernel<4, 5, false>, "tv<4,5,L1>");
    run_tv(dense_tv_kernel<4, 6, false>, "tv<4,6,L1>");
    run_tv(dense_tv_kernel<4, 8, false>, "tv<4,8,L1>");
    run_tv(dense_tv_kernel<2, 8, false>, "tv<2,8,L1>");
    run_tv(dense_tv_kernel<8, 4, false>, "tv<8,4,L1>");
    smem = keep;
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
