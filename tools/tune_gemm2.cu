// Tile-shape sweep for the K7 DMMA GEMM (not part of the product).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/tune_gemm2.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>
#include "../paper_1708_02845_b200/csrc/pf_runtime.cu"
#include "../paper_1708_02845_b200/csrc/batched.cu"
using namespace pf;

template <int WM, int WN, int MI, int NJ, int STAGES, int MINB>
__global__ void __launch_bounds__(WM * WN * 32, MINB) dmma_t(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k,
    const double *__restrict__ H, const double *__restrict__ L, int64_t ldl, int64_t T,
    const int64_t *__restrict__ targets, double clamp, double tau, int64_t row0,
    double *__restrict__ out, int64_t ldo) {
  constexpr int NT = WM * WN * 32, BM = WM * MI * 8, BN = WN * NJ * 8, S = kBK + 4;
  constexpr int SA = BM * S, SB = BN * S;
  extern __shared__ __align__(128) unsigned char smem[];
  double *As = reinterpret_cast<double *>(smem);
  double *Bs = As + STAGES * SA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t nkt = (k + kBK - 1) / kBK;
  const int fr = lane >> 2, fc = lane & 3;
  auto issue = [&](int64_t kt) {
    if (kt < nkt) {
      const int st = static_cast<int>(kt % STAGES);
      double *as = As + st * SA, *bs = Bs + st * SB;
      const int64_t k0 = kt * kBK;
      for (int e = tid; e < BM * 8; e += NT) {
        const int row = e >> 3, ch = e & 7;
        const int64_t q = q0 + row;
        const bool ok = q < rows;
        cp_async16(as + row * S + 2 * ch, P + (ok ? q : 0) * ld + k0 + 2 * ch, ok);
      }
      for (int e = tid; e < BN * 8; e += NT) {
        const int row = e >> 3, ch = e & 7;
        const int64_t t = t0 + row;
        const bool ok = t < T;
        cp_async16(bs + row * S + 2 * ch, L + (ok ? t : 0) * ldl + k0 + 2 * ch, ok);
      }
    }
    cp_async_commit();
  };
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(s);
  for (int64_t kt = 0; kt < nkt; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue(kt + STAGES - 1);
    const int st = static_cast<int>(kt % STAGES);
    const double *as = As + st * SA + (wm * MI * 8 + fr) * S + fc;
    const double *bs = Bs + st * SB + (wn * NJ * 8 + fr) * S + fc;
#pragma unroll
    for (int ks = 0; ks < kBK; ks += 4) {
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = fmax(as[8 * i * S + ks], clamp);
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = bs[8 * j * S + ks];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t q = q0 + wm * MI * 8 + 8 * i + fr;
    if (q >= rows) continue;
    const double h = H[q];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t t = t0 + wn * NJ * 8 + 8 * j + 2 * fc + c;
        if (t >= T) continue;
        const double cross = acc[i][j][c];
        double val = h - cross;
        const bool is_t = (row0 + q == targets[t]);
        if (!is_t && fabs(val) < tau * (fabs(h) + fabs(cross)))
          val = __longlong_as_double(static_cast<long long>(kBatchGuard));
        else
          val = is_t ? 0.0 : settle(val);
        out[q * ldo + t] = val;
      }
  }
}

__global__ void fill(double *P, int64_t n, int64_t ld, int64_t k, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * ld;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (i + seed) * 0x9E3779B97F4A7C15ull; h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    P[i] = (i % ld) < k ? (double)(h >> 11) * (1.0 / 9007199254740992.0) / k : 0.0;
  }
}

int main(int argc, char **argv) {
  int64_t rows = argc > 1 ? atoll(argv[1]) : 131072, k = argc > 2 ? atoll(argv[2]) : 4102,
          T = argc > 3 ? atoll(argv[3]) : 1024;
  int64_t ld = round_up(k, 16), ldl = ld;
  double *P, *H, *L, *out, *ref; int64_t *tg;
  cudaMalloc(&P, rows * ld * 8); cudaMalloc(&H, rows * 8); cudaMalloc(&L, T * ldl * 8);
  cudaMalloc(&out, rows * T * 8); cudaMalloc(&ref, rows * T * 8); cudaMalloc(&tg, T * 8);
  fill<<<4096, 256>>>(P, rows, ld, k, 1); fill<<<1024, 256>>>(L, T, ldl, k, 7);
  cudaMemset(H, 0, rows * 8);
  std::vector<int64_t> th(T); for (int64_t i = 0; i < T; ++i) th[i] = (i * 997) % rows;
  cudaMemcpy(tg, th.data(), T * 8, cudaMemcpyHostToDevice);
  const double flops = 2.0 * rows * k * T;
  pf_batched_kl_f64(P, ld, rows, k, H, L, L, ldl, T, tg, 1e-300, 0.0, 0, ref, T, nullptr, 0);
  cudaDeviceSynchronize();
  std::vector<double> a(rows * T), b(rows * T);
  cudaMemcpy(a.data(), ref, rows * T * 8, cudaMemcpyDeviceToHost);
  auto run = [&](auto kern, int NT, int BM, int BN, size_t smem, const char *name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((T + BN - 1) / BN, (rows + BM - 1) / BM);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<grid, NT, smem>>>(P, ld, rows, k, H, L, ldl, T, tg, 1e-300, 0.0, 0, out, T);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r)
      kern<<<grid, NT, smem>>>(P, ld, rows, k, H, L, ldl, T, tg, 1e-300, 0.0, 0, out, T);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
    cudaMemcpy(b.data(), out, rows * T * 8, cudaMemcpyDeviceToHost);
    bool same = a == b;
    printf("%-34s %8.3f ms %6.2f TFLOP/s occ=%d bitwise=%d (%s)\n", name, ms, flops / ms / 1e9,
           occupancy((const void *)kern, NT, smem), same, cudaGetErrorString(cudaGetLastError()));
  };
#define V(WM, WN, MI, NJ, ST, MB)                                                          \
  run(dmma_t<WM, WN, MI, NJ, ST, MB>, WM * WN * 32, WM * MI * 8, WN * NJ * 8,              \
      (size_t)ST * (WM * MI * 8 + WN * NJ * 8) * (kBK + 4) * 8,                          \
      "W" #WM "x" #WN " T" #MI "x" #NJ " S" #ST " B" #MB);
  V(4, 2, 4, 4, 3, 2)   // product shape
  V(4, 2, 4, 4, 4, 1)
  V(4, 2, 4, 8, 3, 1)
  V(2, 4, 8, 4, 3, 1)
  V(4, 2, 4, 8, 4, 1)
  V(8, 2, 4, 4, 3, 1)
  V(4, 4, 4, 4, 3, 1)
  V(2, 2, 4, 4, 4, 3)
  V(2, 2, 8, 4, 3, 2)
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
