// Debug aid: pf_format_lines (wire.cu) on device vs format_double on the host.
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1708_02845_b200/csrc/pf_runtime.cu"
#include "../paper_1708_02845_b200/csrc/wire.cu"
int main(int argc, char **argv) {
  std::vector<double> v;
  for (int e = -1074; e < 1024; ++e) v.push_back(std::ldexp(1.0, e));
  v.push_back(8.41e21); v.push_back(4.35e-7); v.push_back(6.6e-75);
  const int n = v.size();
  for (int kind : {5, 4}) {
    for (int threads_mode = 0; threads_mode < 2; ++threads_mode) {
      double *dv; char *slots; int32_t *lens;
      cudaMalloc(&dv, n * 8); cudaMalloc(&slots, n * 64); cudaMalloc(&lens, n * 4);
      cudaMemcpy(dv, v.data(), n * 8, cudaMemcpyHostToDevice);
      cudaMemset(slots, 0, n * 64);
      if (threads_mode == 0) {
        pf_format_lines(dv, n, kind, 0, slots, lens, nullptr, nullptr);
      } else {  // one value per launch, one thread
        for (int i = 0; i < n; ++i) pf_format_lines(dv + i, 1, kind, 0, slots + 64 * i, lens + i, nullptr, nullptr);
      }
      cudaDeviceSynchronize();
      std::vector<char> hs(n * 64); std::vector<int32_t> hl(n);
      cudaMemcpy(hs.data(), slots, n * 64, cudaMemcpyDeviceToHost);
      cudaMemcpy(hl.data(), lens, n * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < n; ++i) {
        char ref[64];
        int k = pf::wire::format_double(v[i], kind == 5 ? 0 : 1, ref);
        if (k != hl[i] || memcmp(ref, &hs[64 * i], k)) {
          if (bad++ < 3) printf("  kind %d mode %d i %d v=%.17g ref=%.*s got=%.*s\n", kind, threads_mode, i, v[i], k, ref, hl[i], &hs[64 * i]);
        }
      }
      printf("kind %d mode %d bad %d of %d err=%s\n", kind, threads_mode, bad, n, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
