// Standalone probe (not part of the product): can a CTA's 1-D bulk copy
// (cp.async.bulk, into its own shared memory) complete on an mbarrier in the
// other CTA of its cluster?  (K7 pairs want both CTAs' copies on the leader's
// barrier; the tensor form has .cta_group::2 for that.)
// Measured on B200: no -- the leader waits forever (the run hits its timeout),
// so a pair needs the tensor form with .cta_group::2 (or a relay arrive).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I include tools/probe_bulk_remote_bar.cu -o tools/probe_bulk_remote_bar.bin
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1708_02845_b200/csrc/pf_tc.cuh"

__global__ void __cluster_dims__(2, 1, 1) k(const double *src, double *out) {
  __shared__ __align__(128) double buf[512];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = pf::tc::cluster_rank();
  if (threadIdx.x == 0) {
    pf::mbar_init(&bar, 1);
  }
  pf::tc::cluster_sync();
  if (threadIdx.x == 0 && rank == 0) pf::mbar_expect_tx(&bar, 2 * 4096);   // both CTAs' bytes
  pf::tc::cluster_sync();
  if (threadIdx.x == 0) {
    const uint32_t lb = pf::tc::mapa(&bar, 0);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(pf::smem_u32(buf)), "l"(src + rank * 512), "r"(4096), "r"(lb) : "memory");
  }
  if (rank == 0) pf::mbar_wait(&bar, 0);
  pf::tc::cluster_sync();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[rank * 512 + i] = buf[i];
}

int main() {
  double *src, *out;
  cudaMalloc(&src, 8192); cudaMalloc(&out, 8192);
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = i;
  cudaMemcpy(src, h, 8192, cudaMemcpyHostToDevice);
  cudaMemset(out, 0, 8192);
  k<<<2, 128>>>(src, out);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, out, 8192, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 1024; ++i) bad += h[i] != i;
  printf("{\"err\": \"%s\", \"mismatches\": %d}\n", cudaGetErrorString(e), bad);
  return 0;
}
