// Standalone probe (not part of the product): is the CSR field stream's
// ~5.6 TB/s a DRAM access-pattern limit?  Streams ~500 MB laid out like C3
// (rows of ~487 entries: 8-byte data + 2-byte columns), warp per row, rows
// strided over the warps as in csr_kl_kernel, 8 pairs per lane in flight:
//   mode 0: data and columns as two arrays (the product layout)
//   mode 1: data only (no column stream)
//   mode 2: one packed array, per 8 entries 64 B data + 16 B columns
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probe_csr_stream.cu -o tools/probe_csr_stream.bin
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_1708_02845_b200/csrc/pf_common.cuh"
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int MODE>
__global__ void __launch_bounds__(256, 4) stream_kernel(const int64_t *__restrict__ ptr,
                                                        const double *__restrict__ data,
                                                        const uint16_t *__restrict__ idx,
                                                        const uint8_t *__restrict__ packed,
                                                        const int64_t *__restrict__ pptr,
                                                        int64_t rows, double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    double a = 0.0;
    if (MODE < 2) {
      const int64_t lo = ptr[r], hi = ptr[r + 1];
      const int64_t np = (hi - lo) >> 1;   // lo even by construction
      const double2 *d2 = reinterpret_cast<const double2 *>(data + lo);
      const ushort2 *i2 = reinterpret_cast<const ushort2 *>(idx + lo);
      for (int64_t j0 = 0; j0 < np; j0 += 256) {
        double2 v[8];
        ushort2 c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          int64_t j = j0 + lane + 32 * u;
          j = j < np ? j : np - 1;
          v[u] = __ldg(d2 + j);
          if (MODE == 0) c[u] = __ldg(i2 + j);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool in = j0 + lane + 32 * u < np;
          a += in ? v[u].x + v[u].y : 0.0;
          if (MODE == 0) a += in ? double(c[u].x + c[u].y) : 0.0;
        }
      }
    } else {
      const int64_t lo = pptr[r], hi = pptr[r + 1];   // in 80-byte blocks
      const int64_t nb = hi - lo;
      const uint4 *b = reinterpret_cast<const uint4 *>(packed) + lo * 5;
      for (int64_t j0 = 0; j0 < nb; j0 += 64) {
        uint4 w[2][5];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          int64_t j = j0 + lane + 32 * u;
          j = j < nb ? j : nb - 1;
#pragma unroll
          for (int q = 0; q < 5; ++q) w[u][q] = __ldg(b + j * 5 + q);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const bool in = j0 + lane + 32 * u < nb;
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q) s += __longlong_as_double(((long long)w[u][q].y << 32) | w[u][q].x) +
                                           __longlong_as_double(((long long)w[u][q].w << 32) | w[u][q].z);
          s += double(w[u][4].x & 0xffff) + double(w[u][4].w >> 16);
          a += in ? s : 0.0;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) out[r] = a;
  }
}


// mode 3: extent of the next row prefetched (the product's loop); mode 4: + the
// next row's data / column lines prefetched to L2 while this row streams;
// mode 5: two rows per warp iteration (both rows' loads in flight together)
template <int MODE, int U = 8>
__global__ void __launch_bounds__(256, MODE == 5 ? 3 : 4) stream2_kernel(const int64_t *__restrict__ ptr,
                                                        const double *__restrict__ data,
                                                        const uint16_t *__restrict__ idx,
                                                        int64_t rows, double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int R = MODE == 5 ? 2 : 1;
  int64_t r = warp * R;
  int64_t lo = r < rows ? ptr[r] : 0, hi = r < rows ? ptr[r + R < rows ? r + R : rows] : 0;
  while (r < rows) {
    const int64_t r2 = r + nwarps * R;
    const int64_t lo2 = r2 < rows ? ptr[r2] : 0, hi2 = r2 < rows ? ptr[r2 + R < rows ? r2 + R : rows] : 0;
    if (MODE == 4 && r2 < rows) {
      for (int64_t b = (lo2 * 8) / 128 * 128 + lane * 128; b < hi2 * 8; b += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char *>(data) + b));
      for (int64_t b = (lo2 * 2) / 128 * 128 + lane * 128; b < hi2 * 2; b += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char *>(idx) + b));
    }
    // R rows visited as one segment [lo, hi) (consecutive rows are contiguous)
    double a[R];
    for (int q = 0; q < R; ++q) a[q] = 0.0;
    const int64_t np = (hi - lo) >> 1;
    const int64_t mid = R == 2 ? ((r + 1 < rows ? ptr[r + 1] : hi) - lo) >> 1 : np;
    const double2 *d2 = reinterpret_cast<const double2 *>(data + lo);
    const ushort2 *i2 = reinterpret_cast<const ushort2 *>(idx + lo);
    for (int64_t j0 = 0; j0 < np; j0 += 32 * U * R) {
      double2 v[U * R];
      ushort2 c[U * R];
#pragma unroll
      for (int u = 0; u < U * R; ++u) {
        int64_t j = j0 + lane + 32 * u;
        j = j < np ? j : np - 1;
        v[u] = __ldg(d2 + j);
        c[u] = __ldg(i2 + j);
      }
#pragma unroll
      for (int u = 0; u < U * R; ++u) {
        const int64_t j = j0 + lane + 32 * u;
        const bool in = j < np;
        const double x = in ? v[u].x + v[u].y + double(c[u].x + c[u].y) : 0.0;
        if (R == 2 && j >= mid) a[R - 1] += x; else a[0] += x;
      }
    }
    for (int q = 0; q < R; ++q) {
      double t = a[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0 && r + q < rows) out[r + q] = t;
    }
    r = r2; lo = lo2; hi = hi2;
  }
}

// The product loop's extras on top of mode 3: STAGE = each CTA bulk-copies the
// 34 KB target vector into shared memory and waits before its first row
// (EARLY: the first row's loads are issued before the wait); GATHER = per entry
// an FMA with the staged vector at the entry's column.
template <bool STAGE, bool GATHER, bool EARLY>
__global__ void __launch_bounds__(256, 4) prod_kernel(const int64_t *__restrict__ ptr,
                                                      const double *__restrict__ data,
                                                      const uint16_t *__restrict__ idx,
                                                      const double *__restrict__ vec, int64_t k,
                                                      int64_t rows, double *__restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  double *lt = reinterpret_cast<double *>(smem + 16);
  if (STAGE) {
    if (threadIdx.x == 0) pf::mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      pf::mbar_expect_tx(bar, static_cast<uint32_t>(k * 8));
      pf::bulk_g2s(lt, vec, static_cast<uint32_t>(k * 8), bar);
    }
    if (!EARLY) pf::mbar_wait(bar, 0);
  }
  bool waited = !STAGE || !EARLY;
  int64_t r = warp;
  int64_t lo = r < rows ? ptr[r] : 0, hi = r < rows ? ptr[r + 1] : 0;
  while (r < rows) {
    const int64_t r2 = r + nwarps;
    const int64_t lo2 = r2 < rows ? ptr[r2] : 0, hi2 = r2 < rows ? ptr[r2 + 1] : 0;
    double a0 = 0.0, a1 = 0.0;
    const int64_t np = (hi - lo) >> 1;
    const double2 *d2 = reinterpret_cast<const double2 *>(data + lo);
    const ushort2 *i2 = reinterpret_cast<const ushort2 *>(idx + lo);
    for (int64_t j0 = 0; j0 < np; j0 += 128) {
      double2 v[4];
      ushort2 c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int64_t j = j0 + lane + 32 * u;
        j = j < np ? j : np - 1;
        v[u] = __ldg(d2 + j);
        c[u] = __ldg(i2 + j);
      }
      if (!waited) { pf::mbar_wait(bar, 0); waited = true; }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = j0 + lane + 32 * u < np;
        if (GATHER) {
          a0 = fma(in ? v[u].x : 0.0, lt[in ? c[u].x : 0], a0);
          a1 = fma(in ? v[u].y : 0.0, lt[in ? c[u].y : 0], a1);
        } else {
          a0 += in ? v[u].x + double(c[u].x) : 0.0;
          a1 += in ? v[u].y + double(c[u].y) : 0.0;
        }
      }
    }
    double t = a0 + a1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) out[r] = t;
    r = r2; lo = lo2; hi = hi2;
  }
}

int main() {
  const int64_t rows = 102104;
  std::vector<int64_t> ptr(rows + 1), pptr(rows + 1);
  uint64_t s = 12345;
  ptr[0] = 0; pptr[0] = 0;
  for (int64_t r = 0; r < rows; ++r) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    int64_t n = 470 + (s >> 33) % 34;
    n += n & 1;
    ptr[r + 1] = ptr[r] + n;
    pptr[r + 1] = pptr[r] + (n + 7) / 8;
  }
  const int64_t nnz = ptr[rows], nblk = pptr[rows];
  double *data; uint16_t *idx; uint8_t *packed; int64_t *dptr, *dpptr; double *out;
  CK(cudaMalloc(&data, nnz * 8)); CK(cudaMalloc(&idx, nnz * 2)); CK(cudaMalloc(&packed, nblk * 80));
  CK(cudaMalloc(&dptr, (rows + 1) * 8)); CK(cudaMalloc(&dpptr, (rows + 1) * 8)); CK(cudaMalloc(&out, rows * 8));
  CK(cudaMemset(data, 0, nnz * 8)); CK(cudaMemset(idx, 0, nnz * 2)); CK(cudaMemset(packed, 0, nblk * 80));
  {   // sorted distinct columns per row, like the C3 CSR (k = 4250, ~11% dense)
    std::vector<uint16_t> h(nnz);
    uint64_t z = 777;
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t n = ptr[r + 1] - ptr[r];
      int64_t c = 0;
      for (int64_t e = 0; e < n; ++e) {
        z = z * 6364136223846793005ull + 1442695040888963407ull;
        const int64_t left = 4250 - c - (n - e);
        c += 1 + (left > 0 ? (int64_t)((z >> 33) % (2 * left / (n - e) + 1)) : 0);
        h[ptr[r] + e] = static_cast<uint16_t>(c - 1 < 4249 ? c - 1 : 4249);
      }
    }
    if (getenv("ZERO_COLS") == nullptr) CK(cudaMemcpy(idx, h.data(), nnz * 2, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(dptr, ptr.data(), (rows + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpptr, pptr.data(), (rows + 1) * 8, cudaMemcpyHostToDevice));
  char *flush; const size_t fl = 512ull << 20;
  CK(cudaMalloc(&flush, fl));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    double *vec; CK(cudaMalloc(&vec, 4250 * 8)); CK(cudaMemset(vec, 0, 4250 * 8));
  const int sm_bytes = 16 + 4250 * 8;
  CK(cudaFuncSetAttribute(prod_kernel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
  CK(cudaFuncSetAttribute(prod_kernel<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
  CK(cudaFuncSetAttribute(prod_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
  for (int mode = 0; mode < 12; ++mode) {
    const double bytes = (mode == 0 || mode >= 3) ? nnz * 10.0 : mode == 1 ? nnz * 8.0 : nblk * 80.0;
    float best = 1e9, sum = 0; int cnt = 0;
    for (int it = 0; it < 12; ++it) {
      (void)fl;   // no flush: each launch streams ~500 MB > L2, and a write flush
                  // would leave 126 MB of dirty lines to write back inside the timing
      cudaEventRecord(e0);
      if (mode == 0) stream_kernel<0><<<sms * 4, 256>>>(dptr, data, idx, packed, dpptr, rows, out);
      if (mode == 1) stream_kernel<1><<<sms * 4, 256>>>(dptr, data, idx, packed, dpptr, rows, out);
      if (mode == 2) stream_kernel<2><<<sms * 4, 256>>>(dptr, data, idx, packed, dpptr, rows, out);
      if (mode == 3) stream2_kernel<3><<<sms * 4, 256>>>(dptr, data, idx, rows, out);
      if (mode == 4) stream2_kernel<4><<<sms * 4, 256>>>(dptr, data, idx, rows, out);
      if (mode == 5) stream2_kernel<5><<<sms * 3, 256>>>(dptr, data, idx, rows, out);
      if (mode == 6) stream2_kernel<3, 4><<<sms * 4, 256>>>(dptr, data, idx, rows, out);
      if (mode == 7) stream2_kernel<3, 16><<<sms * 4, 256>>>(dptr, data, idx, rows, out);
      if (mode == 8) prod_kernel<false, false, false><<<sms * 4, 256, 0>>>(dptr, data, idx, vec, 4250, rows, out);
      if (mode == 9) prod_kernel<true, false, false><<<sms * 4, 256, sm_bytes>>>(dptr, data, idx, vec, 4250, rows, out);
      if (mode == 10) prod_kernel<true, true, false><<<sms * 4, 256, sm_bytes>>>(dptr, data, idx, vec, 4250, rows, out);
      if (mode == 11) prod_kernel<true, true, true><<<sms * 4, 256, sm_bytes>>>(dptr, data, idx, vec, 4250, rows, out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { best = ms < best ? ms : best; sum += ms; ++cnt; }
    }
    printf("{\"mode\": %d, \"MB\": %.1f, \"ms_best\": %.4f, \"ms_avg\": %.4f, \"TBps_avg\": %.3f}\n", mode,
           bytes / 1e6, best, sum / cnt, bytes / (sum / cnt * 1e-3) / 1e12);
  }
  return 0;
}
