// pf_jit.cu — user-defined divergence generators on the device (NVRTC).
//
// The reference accepts any convex generator: FDivergence(name, f, ...) with
// an arbitrary numpy callable f (divergence.py:42-56), evaluated per element
// as q * f(p / q) inside dv_field / dv_at / dv_pair (:137-187).  The
// built-in generators have hand-written kernels (dense.cu); for any other f
// the Python side traces f symbolically into a scalar CUDA expression
// (paper_1708_02845_b200/_userf.py: only arithmetic, comparisons, where/clip
// and numpy math ufuncs, checked against f itself on sample points) and this
// file compiles it into the field / dv_at kernels below with NVRTC for
// sm_100a, loads the cubin with the runtime's library API, and launches it —
// the same warp-per-row streaming structure, settle rule, target zero and
// one-sided clamp flag as dense_generic_kernel.  NVRTC is bound at run time
// (dlopen), so the library has no link-time dependency on it.
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pf_common.cuh"

namespace {

const char *kUserSource = R"PFSRC(
typedef long long i64;
__device__ __forceinline__ double pf_user_f(double x) { return (PF_USER_EXPR); }
__device__ __forceinline__ double pf_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double pf_settle(double v) {
  return (v > -1e-10 && v < 0.0) ? 0.0 : v;   // divergence.py:39, 149, 181
}
// q * f(p / q) (default order) or p * f(q / p) (swap_order), divergence.py:146-148, 177-180
__device__ __forceinline__ double pf_term(double q, double p, int swap) {
  return swap ? __dmul_rn(p, pf_user_f(__ddiv_rn(q, p))) : __dmul_rn(q, pf_user_f(__ddiv_rn(p, q)));
}
extern "C" __global__ void __launch_bounds__(256) pf_user_field(
    const double *__restrict__ P, i64 ld, i64 rows, i64 k, const double *__restrict__ tgt,
    const unsigned char *__restrict__ tmask, double clamp, int swap, i64 row0, i64 target,
    const unsigned char *__restrict__ is_interior, double *__restrict__ out,
    unsigned int *__restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  bool clamped_any = false;
  for (i64 r = warp; r < rows; r += nwarps) {
    const double *row = P + r * ld;
    double a0 = 0.0, a1 = 0.0;
    bool fl = false;
    i64 b = lane;
    for (; b + 32 < k; b += 64) {
      const double x0 = row[b], x1 = row[b + 32];
      a0 += pf_term(fmax(x0, clamp), __ldg(tgt + b), swap);
      a1 += pf_term(fmax(x1, clamp), __ldg(tgt + b + 32), swap);
      fl |= ((x0 < clamp) != (tmask[b] != 0)) | ((x1 < clamp) != (tmask[b + 32] != 0));
    }
    if (b < k) {
      const double x0 = row[b];
      a0 += pf_term(fmax(x0, clamp), __ldg(tgt + b), swap);
      fl |= (x0 < clamp) != (tmask[b] != 0);
    }
    double val = pf_settle(pf_warp_sum(a0 + a1));
    if (row0 + r == target) val = 0.0;
    const bool interior = is_interior ? (is_interior[r] != 0) : true;
    clamped_any |= interior && __any_sync(0xffffffffu, fl);
    if (lane == 0) out[r] = val;
  }
  if (lane == 0 && clamped_any) atomicOr(&flags[0], 1u);
}
extern "C" __global__ void __launch_bounds__(256) pf_user_at(
    const double *__restrict__ P, i64 ld, i64 rows, i64 k, const double *__restrict__ tgt,
    double clamp, int swap, i64 row0, i64 target, const i64 *__restrict__ queries, i64 nq,
    double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < nq; i += nwarps) {
    const i64 q = queries[i], r = q - row0;
    double acc = 0.0;
    if (r >= 0 && r < rows)
      for (i64 b = lane; b < k; b += 32) acc += pf_term(fmax(P[r * ld + b], clamp), __ldg(tgt + b), swap);
    double val = pf_settle(pf_warp_sum(acc));
    if (q == target) val = 0.0;   // divergence.py:150
    if (lane == 0) out[i] = val;
  }
}
// divergence.py:296-299: other generators over supp(p) U supp(q), absent
// weights clamped at the row cut (row-aligned CSR of csr.cu: bit 0 of a row's
// end offset flags one trailing pad entry).
extern "C" __global__ void __launch_bounds__(256) pf_user_csr(
    const i64 *__restrict__ indptr, const int *__restrict__ indices,
    const double *__restrict__ data, i64 rows, const double *__restrict__ prow, i64 p_local,
    double cut, i64 row0, const i64 *__restrict__ queries, i64 nq, double *__restrict__ out,
    i64 *__restrict__ ops) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  const i64 count = queries ? nq : rows;
  const i64 pa = indptr[p_local], pb = indptr[p_local + 1];
  const i64 plo = pa & ~1LL, phi = (pb & ~1LL) - (pb & 1);
  for (i64 i = warp; i < count; i += nwarps) {
    const i64 r = queries ? queries[i] - row0 : i;
    const i64 a0 = indptr[r], b0 = indptr[r + 1];
    const i64 lo = a0 & ~1LL, hi = (b0 & ~1LL) - (b0 & 1);
    double a = 0.0;
    for (i64 e = lo + lane; e < hi; e += 32) {
      const double v = data[e];
      const double vp = fmax(__ldg(prow + indices[e]), cut);
      a += __dmul_rn(v, pf_user_f(__ddiv_rn(vp, v)));
    }
    int inter = 0;
    for (i64 e = plo + lane; e < phi; e += 32) {
      const int j = indices[e];
      i64 L = lo, R = hi;
      while (L < R) {
        const i64 M = (L + R) >> 1;
        if (indices[M] < j) L = M + 1; else R = M;
      }
      if (L < hi && indices[L] == j) {
        ++inter;
      } else {
        const double vp = fmax(__ldg(prow + j), cut);
        a += __dmul_rn(cut, pf_user_f(__ddiv_rn(vp, cut)));
      }
    }
    const double val = pf_settle(pf_warp_sum(a));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(0xffffffffu, inter, o);
    if (lane == 0) {
      out[i] = val;
      if (ops) ops[i] = (hi - lo) + (phi - plo) - inter;
    }
  }
}
)PFSRC";

struct Nvrtc {
  void *h = nullptr;
  nvrtcResult (*create)(nvrtcProgram *, const char *, const char *, int, const char *const *,
                        const char *const *) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char *const *) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t *) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char *) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t *) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char *) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram *) = nullptr;
};

Nvrtc g_nvrtc;
std::mutex g_nvrtc_mu;

template <typename F>
bool sym(void *h, const char *name, F *&fn) {
  fn = reinterpret_cast<F *>(dlsym(h, name));
  return fn != nullptr;
}

int load_nvrtc(const char *path) {
  std::lock_guard<std::mutex> lk(g_nvrtc_mu);
  if (g_nvrtc.h) return 0;
  void *h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);  // the toolkit's (12.9)
  if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
  if (!h && path && path[0]) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return pf::fail(PF_E_ARG, "dlopen libnvrtc.so.12: %s", dlerror());
  Nvrtc a;
  a.h = h;
  if (!(sym(h, "nvrtcCreateProgram", a.create) && sym(h, "nvrtcCompileProgram", a.compile) &&
        sym(h, "nvrtcGetProgramLogSize", a.log_size) && sym(h, "nvrtcGetProgramLog", a.log) &&
        sym(h, "nvrtcGetCUBINSize", a.cubin_size) && sym(h, "nvrtcGetCUBIN", a.cubin) &&
        sym(h, "nvrtcDestroyProgram", a.destroy)))
    return pf::fail(PF_E_ARG, "libnvrtc lacks a required symbol");
  g_nvrtc = a;
  return 0;
}

struct UserGen {
  std::vector<char> cubin;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t field = nullptr, at = nullptr, csr = nullptr;
};

int grid_for_rows(int64_t rows) {
  int64_t g = static_cast<int64_t>(pf::sm_count()) * 4, want = (rows + 7) / 8;
  if (g > want) g = want;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int pf_user_compile(const char *expr_host, const char *nvrtc_path_host, int load,
                    void **handle_host) {
  if (!expr_host || !handle_host) return pf::fail(PF_E_ARG, "user_compile: null");
  *handle_host = nullptr;
  if (int e = load_nvrtc(nvrtc_path_host)) return e;
  const std::string expr(expr_host);
  if (expr.find_first_of(";{}#\"'\\") != std::string::npos)
    return pf::fail(PF_E_ARG, "user_compile: not a scalar expression");
  const std::string src = "#define PF_USER_EXPR " + expr + "\n" + kUserSource;
  nvrtcProgram prog = nullptr;
  if (g_nvrtc.create(&prog, src.c_str(), "pf_user.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return pf::fail(PF_E_LAUNCH, "nvrtcCreateProgram failed");
  const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device"};
  const nvrtcResult rc = g_nvrtc.compile(prog, 3, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    g_nvrtc.log_size(prog, &n);
    std::string lg(n, '\0');
    if (n) g_nvrtc.log(prog, &lg[0]);
    g_nvrtc.destroy(&prog);
    return pf::fail(PF_E_DOMAIN, "nvrtc: %.400s", lg.c_str());
  }
  auto *ug = new UserGen;
  size_t n = 0;
  g_nvrtc.cubin_size(prog, &n);
  ug->cubin.resize(n);
  g_nvrtc.cubin(prog, ug->cubin.data());
  g_nvrtc.destroy(&prog);
  if (load) {
    cudaError_t e = cudaLibraryLoadData(&ug->lib, ug->cubin.data(), nullptr, nullptr, 0, nullptr,
                                        nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&ug->field, ug->lib, "pf_user_field");
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&ug->at, ug->lib, "pf_user_at");
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&ug->csr, ug->lib, "pf_user_csr");
    if (e != cudaSuccess) {
      if (ug->lib) cudaLibraryUnload(ug->lib);
      delete ug;
      return pf::fail(static_cast<int>(e), "user kernel load: %s", cudaGetErrorString(e));
    }
  }
  *handle_host = ug;
  return 0;
}

int pf_user_cubin_size(void *handle, int64_t *bytes_host) {
  if (!handle || !bytes_host) return pf::fail(PF_E_ARG, "user_cubin_size: null");
  *bytes_host = static_cast<int64_t>(static_cast<UserGen *>(handle)->cubin.size());
  return 0;
}

int pf_user_free(void *handle) {
  if (!handle) return 0;
  auto *ug = static_cast<UserGen *>(handle);
  if (ug->lib) cudaLibraryUnload(ug->lib);
  delete ug;
  return 0;
}

int pf_dense_user_f64(void *handle, const double *P, int64_t ld, int64_t rows, int64_t k,
                      const double *tgt, const uint8_t *tmask, double clamp, int swap_order,
                      int64_t row0, int64_t target, const uint8_t *is_interior, double *out,
                      uint32_t *flags, pf_stream_t stream) {
  auto *ug = static_cast<UserGen *>(handle);
  if (!ug || !ug->field) return pf::fail(PF_E_ARG, "dense_user: generator not loaded");
  if (!P || !tgt || !tmask || !out || !flags || ld < k || k <= 0 || rows < 0)
    return pf::fail(PF_E_ARG, "dense_user: bad args");
  if (rows == 0) return 0;
  int swap = swap_order != 0;
  void *args[] = {&P, &ld, &rows, &k, &tgt, &tmask, &clamp, &swap, &row0, &target,
                  &is_interior, &out, &flags};
  const cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void *>(ug->field),
                                         dim3(grid_for_rows(rows)), dim3(256), args, 0,
                                         pf::as_stream(stream));
  if (e != cudaSuccess) return pf::fail(static_cast<int>(e), "dense_user: %s", cudaGetErrorString(e));
  return 0;
}

int pf_dense_user_at_f64(void *handle, const double *P, int64_t ld, int64_t rows, int64_t k,
                         const double *tgt, double clamp, int swap_order, int64_t row0,
                         int64_t target, const int64_t *queries, int64_t nq, double *out,
                         pf_stream_t stream) {
  auto *ug = static_cast<UserGen *>(handle);
  if (!ug || !ug->at) return pf::fail(PF_E_ARG, "dense_user_at: generator not loaded");
  if (!P || !tgt || ld < k || k <= 0 || rows < 0 || (nq > 0 && (!queries || !out)))
    return pf::fail(PF_E_ARG, "dense_user_at: bad args");
  if (nq <= 0) return 0;
  int swap = swap_order != 0;
  void *args[] = {&P, &ld, &rows, &k, &tgt, &clamp, &swap, &row0, &target, &queries, &nq, &out};
  const cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void *>(ug->at),
                                         dim3(grid_for_rows(nq)), dim3(256), args, 0,
                                         pf::as_stream(stream));
  if (e != cudaSuccess)
    return pf::fail(static_cast<int>(e), "dense_user_at: %s", cudaGetErrorString(e));
  return 0;
}

int pf_csr_user_f64(void *handle, const int64_t *indptr, const int32_t *indices,
                    const double *data, int64_t rows, const double *prow, int64_t p_local,
                    double cut, int64_t row0, const int64_t *queries, int64_t nq, double *out,
                    int64_t *ops, pf_stream_t stream) {
  auto *ug = static_cast<UserGen *>(handle);
  if (!ug || !ug->csr) return pf::fail(PF_E_ARG, "csr_user: generator not loaded");
  if (!indptr || !indices || !data || !prow || !out || rows < 0 || p_local < 0 ||
      p_local >= rows)
    return pf::fail(PF_E_ARG, "csr_user: bad args");
  const int64_t count = queries ? nq : rows;
  if (count <= 0) return 0;
  void *args[] = {&indptr, &indices, &data, &rows, &prow, &p_local, &cut, &row0, &queries, &nq,
                  &out, &ops};
  const cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void *>(ug->csr),
                                         dim3(grid_for_rows(count)), dim3(256), args, 0,
                                         pf::as_stream(stream));
  if (e != cudaSuccess) return pf::fail(static_cast<int>(e), "csr_user: %s", cudaGetErrorString(e));
  return 0;
}

}  // extern "C"
