// Standalone tuner for K7 (not part of the product): DFMA vs DMMA batched-KL GEMM,
// plus the DFMA probe.  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Iinclude
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>
#include "../paper_1708_02845_b200/csrc/pf_runtime.cu"
#include "../paper_1708_02845_b200/csrc/batched.cu"
using namespace pf;

// ---- variants measured and replaced by batched_kl_dmma2_kernel (kept for the record)
namespace pf {
constexpr int kBM = 128, kBN = 128;
constexpr int kApad = kBM + 1, kBpad = kBN + 1;
constexpr int kDS = kBM + 8;
__global__ void __launch_bounds__(kGemmThreads, 1) batched_kl_gemm_kernel(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k,
    const double *__restrict__ H, const double *__restrict__ L, int64_t ldl, int64_t T,
    const int64_t *__restrict__ targets, double clamp, double tau, int64_t row0,
    double *__restrict__ out, int64_t ldo) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *As = reinterpret_cast<double *>(smem);      // [2][kBK][kApad]
  double *Bs = As + 2 * kBK * kApad;                   // [2][kBK][kBpad]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kBN;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * kBM;
  const int64_t nkt = (k + kBK - 1) / kBK;

  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

  double2 ra[4], rb[4];
  auto load_tile = [&](int64_t kt) {
    const int64_t k0 = kt * kBK;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + kGemmThreads * u;  // 0..1023
      const int row = e >> 3, kp = (e & 7) * 2;
      const int64_t q = q0 + row, kk = k0 + kp;
      // raw load only: the clamp is applied at store time so that no math
      // waits on this load before the current tile's FMAs (long-scoreboard)
      double2 a = make_double2(0.0, 0.0);
      if (q < rows && kk < k) a = *reinterpret_cast<const double2 *>(P + q * ld + kk);
      ra[u] = a;
      const int64_t t = t0 + row;
      double2 b = make_double2(0.0, 0.0);
      if (t < T) b = *reinterpret_cast<const double2 *>(L + t * ldl + kk);  // zero-padded
      rb[u] = b;
    }
  };
  auto store_tile = [&](int buf, int64_t kt) {
    double *as = As + buf * kBK * kApad, *bs = Bs + buf * kBK * kBpad;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + kGemmThreads * u;
      const int row = e >> 3, kp = (e & 7) * 2;
      const int64_t kk = kt * kBK + kp;
      const bool okr = q0 + row < rows;
      as[kp * kApad + row] = (okr && kk < k) ? fmax(ra[u].x, clamp) : 0.0;
      as[(kp + 1) * kApad + row] = (okr && kk + 1 < k) ? fmax(ra[u].y, clamp) : 0.0;
      bs[kp * kBpad + row] = rb[u].x;
      bs[(kp + 1) * kBpad + row] = rb[u].y;
    }
  };

  load_tile(0);
  store_tile(0, 0);
  __syncthreads();
  for (int64_t kt = 0; kt < nkt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nkt) load_tile(kt + 1);
    const double *as = As + buf * kBK * kApad, *bs = Bs + buf * kBK * kBpad;
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      double a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = as[kk * kApad + ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = bs[kk * kBpad + tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nkt) store_tile(buf ^ 1, kt + 1);
    __syncthreads();
  }

  // fused epilogue: H - cross, guard, settle, zero at the target
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t q = q0 + ty + 16 * i;
    if (q >= rows) continue;
    const double h = H[q];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t t = t0 + tx + 16 * j;
      if (t >= T) continue;
      const double cross = acc[i][j];
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

// ---------------------------------------------------------------------------
// DMMA variant: the same contraction on the FP64 tensor-core path
// (mma.sync.aligned.m8n8k4.f64, SASS DMMA): 256 FMAs per warp instruction
// instead of 32, so operand staging no longer competes with math for issue
// slots.  Block tile 128 x 128, 8 warps as 2 (m) x 4 (n), warp tile 64 x 32 =
// 8 x 4 mma tiles (64 FP64 accumulators per thread), k-tiles of 16 in
// double-buffered k-major shared memory (row stride 136 doubles: each
// fragment load is the minimal 2 wavefronts).

__global__ void __launch_bounds__(kGemmThreads, 1) batched_kl_dmma_kernel(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k,
    const double *__restrict__ H, const double *__restrict__ L, int64_t ldl, int64_t T,
    const int64_t *__restrict__ targets, double clamp, double tau, int64_t row0,
    double *__restrict__ out, int64_t ldo) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *As = reinterpret_cast<double *>(smem);  // [2][kBK][kDS]
  double *Bs = As + 2 * kBK * kDS;                 // [2][kBK][kDS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;          // 2 x 4 warps
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kBN;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * kBM;
  const int64_t nkt = (k + kBK - 1) / kBK;
  const int fr = lane >> 2, fc = lane & 3;          // fragment row / k index

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double2 ra[4], rb[4];
  auto load_tile = [&](int64_t kt) {
    const int64_t k0 = kt * kBK;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + kGemmThreads * u;
      const int row = e >> 3, kp = (e & 7) * 2;
      const int64_t q = q0 + row, kk = k0 + kp;
      // raw load only: the clamp is applied at store time so that no math
      // waits on this load before the current tile's FMAs (long-scoreboard)
      double2 a = make_double2(0.0, 0.0);
      if (q < rows && kk < k) a = *reinterpret_cast<const double2 *>(P + q * ld + kk);
      ra[u] = a;
      const int64_t t = t0 + row;
      double2 b = make_double2(0.0, 0.0);
      if (t < T) b = *reinterpret_cast<const double2 *>(L + t * ldl + kk);
      rb[u] = b;
    }
  };
  auto store_tile = [&](int buf, int64_t kt) {
    double *as = As + buf * kBK * kDS, *bs = Bs + buf * kBK * kDS;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + kGemmThreads * u;
      const int row = e >> 3, kp = (e & 7) * 2;
      const int64_t kk = kt * kBK + kp;
      const bool okr = q0 + row < rows;
      as[kp * kDS + row] = (okr && kk < k) ? fmax(ra[u].x, clamp) : 0.0;
      as[(kp + 1) * kDS + row] = (okr && kk + 1 < k) ? fmax(ra[u].y, clamp) : 0.0;
      bs[kp * kDS + row] = rb[u].x;
      bs[(kp + 1) * kDS + row] = rb[u].y;
    }
  };

  load_tile(0);
  store_tile(0, 0);
  __syncthreads();
  for (int64_t kt = 0; kt < nkt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nkt) load_tile(kt + 1);
    const double *as = As + buf * kBK * kDS + wm * 64 + fr;
    const double *bs = Bs + buf * kBK * kDS + wn * 32 + fr;
#pragma unroll
    for (int ks = 0; ks < kBK; ks += 4) {
      double a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = as[(ks + fc) * kDS + 8 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[(ks + fc) * kDS + 8 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (kt + 1 < nkt) store_tile(buf ^ 1, kt + 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t q = q0 + wm * 64 + 8 * i + fr;
    if (q >= rows) continue;
    const double h = H[q];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t t = t0 + wn * 32 + 8 * j + 2 * fc + c;
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
}

}  // namespace pf


__global__ void fill(double *P, int64_t n, int64_t ld, int64_t k, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * ld;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (i + seed) * 0x9E3779B97F4A7C15ull; h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    P[i] = (i % ld) < k ? (double)(h >> 11) * (1.0 / 9007199254740992.0) / k : 0.0;
  }
}

template <typename F> float time_ms(F f, int reps = 3) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int i = 0; i < reps; ++i) f(); cudaEventRecord(b);
  cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}

int main(int argc, char **argv) {
  int64_t rows = argc > 1 ? atoll(argv[1]) : 131072, k = argc > 2 ? atoll(argv[2]) : 4102,
          T = argc > 3 ? atoll(argv[3]) : 1024;
  int64_t ld = round_up(k, 16), ldl = ld;
  double *P, *H, *L, *out, *out2; int64_t *tg;
  cudaMalloc(&P, rows * ld * 8); cudaMalloc(&H, rows * 8); cudaMalloc(&L, T * ldl * 8);
  cudaMalloc(&out, rows * T * 8); cudaMalloc(&out2, rows * T * 8); cudaMalloc(&tg, T * 8);
  fill<<<4096, 256>>>(P, rows, ld, k, 1); fill<<<1024, 256>>>(L, T, ldl, k, 7);
  cudaMemset(H, 0, rows * 8);
  std::vector<int64_t> th(T); for (int64_t i = 0; i < T; ++i) th[i] = (i * 997) % rows;
  cudaMemcpy(tg, th.data(), T * 8, cudaMemcpyHostToDevice);
  const double flops = 2.0 * rows * k * T;
  const size_t s1 = 2 * kBK * (kApad + kBpad) * 8, s2 = 2 * 2 * kBK * kDS * 8;
  cudaFuncSetAttribute(batched_kl_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  cudaFuncSetAttribute(batched_kl_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  dim3 grid((T + kBN - 1) / kBN, (rows + kBM - 1) / kBM);
  float m1 = time_ms([&] { batched_kl_gemm_kernel<<<grid, 256, s1>>>(P, ld, rows, k, H, L, ldl, T, tg, 1e-300, 0.0, 0, out, T); });
  float m2 = time_ms([&] { batched_kl_dmma_kernel<<<grid, 256, s2>>>(P, ld, rows, k, H, L, ldl, T, tg, 1e-300, 0.0, 0, out2, T); });
  const size_t s3 = (size_t)kV2Stages * (kV2StageA + kV2StageB) * 8;
  cudaFuncSetAttribute(batched_kl_dmma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s3);
  double *out3; cudaMalloc(&out3, rows * T * 8);
  dim3 grid3((T + kV2BN - 1) / kV2BN, (rows + kV2BM - 1) / kV2BM);
  float m3 = time_ms([&] { batched_kl_dmma2_kernel<<<grid3, 256, s3>>>(P, ld, rows, k, H, L, ldl, T, tg, 1e-300, 0.0, 0, out3, T); });
  printf("dmma2 gemm %8.3f ms %6.2f TFLOP/s (%s)\n", m3, flops / m3 / 1e9, cudaGetErrorString(cudaGetLastError()));
  {
    std::vector<double> a(rows * T), c(rows * T);
    cudaMemcpy(a.data(), out, rows * T * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(c.data(), out3, rows * T * 8, cudaMemcpyDeviceToHost);
    double w = 0; for (size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a[i] - c[i]) / std::max(1e-300, std::abs(a[i])));
    printf("max rel diff dfma vs dmma2 %.3e\n", w);
  }
  int64_t fl = 0; double *o; cudaMalloc(&o, 8);
  pf_probe_dfma_f64(1 << 14, &fl, o, 0);
  float mp = time_ms([&] { pf_probe_dfma_f64(1 << 16, &fl, o, 0); });
  printf("rows=%lld k=%lld T=%lld\n", (long long)rows, (long long)k, (long long)T);
  printf("dfma gemm %8.3f ms %6.2f TFLOP/s\n", m1, flops / m1 / 1e9);
  printf("dmma gemm %8.3f ms %6.2f TFLOP/s\n", m2, flops / m2 / 1e9);
  printf("dfma probe %6.2f TFLOP/s\n", fl / mp / 1e9);
  std::vector<double> a(rows * T), b(rows * T);
  cudaMemcpy(a.data(), out, rows * T * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), out2, rows * T * 8, cudaMemcpyDeviceToHost);
  double worst = 0; for (size_t i = 0; i < a.size(); ++i) worst = std::max(worst, std::abs(a[i] - b[i]) / std::max(1e-300, std::abs(a[i])));
  printf("max rel diff dfma vs dmma %.3e  status %s\n", worst, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
