// Standalone probe (not part of the product): tcgen05.mma kind::i8 on sm_100a.
//  1) correctness of the hand-built shared-memory / instruction descriptors
//     (SWIZZLE_128B K-major operands, u8 x u8 and u8 x s8, S32 accumulators in
//     TMEM read back with tcgen05.ld) against a host GEMM;
//  2) issue-rate throughput of back-to-back M=128 MMAs at N = 64/128/256 with
//     operands resident in shared memory (no global traffic), all SMs.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tune_umma.cu -o /tmp/tu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row x 128 B atoms
// stacked every 1024 B (SBO), version 1.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO
  d |= static_cast<uint64_t>(1) << 46;                 // version
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor kind::i8: S32 accumulators, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(n));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(bar)),
      "r"(phase)
      : "memory");
}

// byte offset of (row r, k-byte b) inside a SW128 K-major tile
__host__ __device__ inline uint32_t sw128_off(int r, int b) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((((b >> 4) ^ (r & 7)) & 7) << 4) + (b & 15);
}

// ---- correctness: D[m][n] = sum_k A[m][k] B[n][k], K = 128 (4 MMAs of K=32)
template <int N>
__global__ void __launch_bounds__(128, 1) umma_check_kernel(const uint8_t *A, const uint8_t *B,
                                                            int b_signed, int32_t *D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *sa = smem;                  // 128 x 128 B
  uint8_t *sb = smem + 128 * 128;      // N x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 128; i += 128) sa[sw128_off(i / 128, i % 128)] = A[i];
  for (int i = tid; i < N * 128; i += 128) sb[sw128_off(i / 128, i % 128)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) mbar_init(&bar, 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N, false, b_signed != 0);
    for (int ks = 0; ks < 4; ++ks)
      mma_i8(tm, sdesc_sw128(su32(sa) + 32 * ks), sdesc_sw128(su32(sb) + 32 * ks), id, ks > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads lanes 32w..32w+31, 8 columns at a time
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + ((32u * warp) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[tid * N + c + j] = static_cast<int32_t>(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(512));
}

// ---- throughput: ITERS x (NACC accumulators x 4 K-steps) MMAs from smem
template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) umma_rate_kernel(int iters, int32_t *sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *sa = smem;
  uint8_t *sb = smem + 128 * 128 * 2;  // two A tiles, two B tiles
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (2 * 128 * 128 + 2 * N * 128) / 4; i += 128)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u * (i & 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) mbar_init(&bar, 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N, false, false);
    for (int it = 0; it < iters; ++it) {
      const int buf = it & 1;
      const uint32_t a0 = su32(sa) + buf * 128 * 128, b0 = su32(sb) + buf * N * 128;
#pragma unroll
      for (int acc = 0; acc < NACC; ++acc)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_i8(tm + acc * N, sdesc_sw128(a0 + 32 * ks), sdesc_sw128(b0 + 32 * ks), id,
                 (it | ks) != 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + ((32u * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (v == 0x12345) sink[0] = v;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(512));
}

template <int N>
bool check(bool b_signed) {
  std::vector<uint8_t> A(128 * 128), B(N * 128);
  uint32_t s = 12345u + N;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return static_cast<uint8_t>(s >> 24); };
  for (auto &x : A) x = rnd();
  for (auto &x : B) x = rnd();
  uint8_t *dA, *dB;
  int32_t *dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const int smem = 128 * 128 + N * 128;
  CK(cudaFuncSetAttribute(umma_check_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  umma_check_kernel<N><<<1, 128, smem>>>(dA, dB, b_signed, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> D(128 * N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      int64_t r = 0;
      for (int k = 0; k < 128; ++k)
        r += static_cast<int64_t>(A[m * 128 + k]) *
             (b_signed ? static_cast<int64_t>(static_cast<int8_t>(B[n * 128 + k]))
                       : static_cast<int64_t>(B[n * 128 + k]));
      if (r != D[m * N + n] && bad++ < 5)
        printf("  mismatch N=%d m=%d n=%d got %d want %lld\n", N, m, n, D[m * N + n], (long long)r);
    }
  printf("check N=%d b_signed=%d: %s\n", N, (int)b_signed, bad ? "FAIL" : "ok");
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad == 0;
}

template <int N, int NACC>
void rate(int sms) {
  const int smem = 2 * 128 * 128 + 2 * N * 128;
  CK(cudaFuncSetAttribute(umma_rate_kernel<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          smem));
  int32_t *sink;
  CK(cudaMalloc(&sink, 4));
  const int iters = 4000;
  umma_rate_kernel<N, NACC><<<sms, 128, smem>>>(10, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  umma_rate_kernel<N, NACC><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 128 * N * 128 * NACC * (double)iters * sms;
  printf("rate N=%3d NACC=%d: %.3f ms  %.1f TOPS  (%.1f cycles/MMA/SM at 1.965 GHz)\n", N, NACC,
         ms, ops / ms / 1e9, ms * 1e-3 * 1.965e9 / (4.0 * NACC * iters));
  cudaFree(sink);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  bool ok = check<64>(false) && check<64>(true) && check<128>(false) && check<256>(true);
  if (!ok) return 1;
  rate<64, 7>(sms);
  rate<64, 7>(sms);
  rate<128, 4>(sms);
  rate<256, 2>(sms);
  rate<256, 1>(sms);
  return 0;
}
