// dense32.cu — dense KL / TV with P stored in FP32 (half the HBM bytes).
//
// Same fields as dense.cu (divergence.py:154-187), with the query rows read
// from an FP32 copy of P; the target row, its logs, H and every accumulation
// stay FP64.  The north-star tolerance for this mode is 1e-5 relative.  H is
// the FP64 negentropy of the FP64 rows, so the FP32 rounding only touches the
// cross term, each c(Q) by at most eps32 = 2^-24 relative, and with every
// log c(Pt) <= 0
//     |KL32 - KL64| <= eps32 * sum c(Q) |log c(Pt)| = eps32 * |cross|,
//     |TV32 - TV64| <= eps32 * (sum c(Q) + sum c(Pt)) ~ 2 eps32,
// so a row whose value is below tau32 * |cross| (KL) or tau32 (TV), tau32 =
// 1e-2, cannot be certified to 1e-5 and is re-evaluated from the FP64 rows in
// place by the
// warp that found it: TV exactly (sum |c(Q) - c(Pt)|, one streaming pass); KL
// in the FP64 split form H64 - sum c(Q) log c(Pt) (one streaming FMA pass,
// ~1e-13 relative), and only if THAT cancels too (the FP64 guard, tau64) in
// the reference's per-element form, evaluated by the whole CTA after its
// loop exactly as the FP64 kernel does (pf_common.cuh GuardQueue).  Unflagged
// rows carry <= 6e-6 relative error by the bound above.
#include <cfloat>
#include <cmath>

#include "pf_common.cuh"

namespace pf {

constexpr int kT32 = 256;

__device__ __forceinline__ float4 ldg_stream4f(const float4 *p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__global__ void __launch_bounds__(kT32) row_negentropy32_kernel(const float *__restrict__ P,
                                                                int64_t ld, int64_t rows,
                                                                int64_t k, double clamp,
                                                                double *__restrict__ H) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const float *row = P + r * ld;
    double a = 0.0;
    for (int64_t b = lane; b < k; b += 32) {
      const double q = fmax(static_cast<double>(row[b]), clamp);
      a += __dmul_rn(q, log(q));
    }
    a = warp_sum(a);
    if (lane == 0) H[r] = a;
  }
}

// One element: q = max(stored FP32 entry, clamp) in FP32 (clamp rounded to FP32
// -- below FLT_MIN it is 0 and the max is skipped: P >= 0), widened to FP64.
// The FP32 clamp moves a clamped term by at most eps32 relative (the same
// order as the FP32 storage of P, inside the guard bound below), or by the
// clamp itself (< FLT_MIN, i.e. < 1.2e-38 absolute per entry).  fmax in FP64
// compiled to ~6 ALU instructions of NaN handling per element and left the
// kernel ALU-bound (ncu: ALU pipe ~80% at speed, DRAM 84%).
template <bool KL, bool CLAMP>
__device__ __forceinline__ void acc32(float q_raw, double t, float clamp32, double &a) {
  const double q = static_cast<double>(CLAMP ? fmaxf(q_raw, clamp32) : q_raw);
  if (KL)
    a = fma(q, t, a);  // t = log c(Pt)
  else
    a += fabs(q - t);  // t = c(Pt)
}

// KL (KL = true) or TV field over FP32 rows; vec = logt (KL) or tgt (TV), both
// FP64.  Each lane streams 4 x float4 per iteration (64 B in flight); the
// FP64 target vector is staged in shared memory split into two double2
// planes, lo[j] = (v[4j], v[4j+1]) and hi[j] = (v[4j+2], v[4j+3]), so the
// two 16-byte shared loads per float4 are bank-conflict free.  The clamp
// flag is not computed here: FP32 rounding flushes entries below the float
// range to zero, so the flag comes from the FP64 rows (pf_mask_compare_f64
// against the interior rows' shared mask, as for K7).
// FP64 re-evaluation of one guarded row from the FP64 copy of P, one warp: KL in
// the reference per-element form, TV as sum |c(Q) - c(Pt)|; then settle.
template <bool KL>
__device__ __forceinline__ double guard64_row(const double *__restrict__ prow, int64_t k,
                                              const double *__restrict__ tgt, double clamp,
                                              int lane) {
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t e = lane;
  for (; e + 96 < k; e += 128) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double q = fmax(prow[e + 32 * u], clamp), t = tgt[e + 32 * u];
      b[u] += KL ? __dmul_rn(q, -log(__ddiv_rn(t, q))) : fabs(q - t);
    }
  }
  for (; e < k; e += 32) {
    const double q = fmax(prow[e], clamp), t = tgt[e];
    b[0] += KL ? __dmul_rn(q, -log(__ddiv_rn(t, q))) : fabs(q - t);
  }
  return settle(warp_sum((b[0] + b[1]) + (b[2] + b[3])));
}

// FP64 split-form KL cross term sum_b c(Q_b) log c(Pt_b) of one FP64 row, one
// warp, logs from the staged lo / hi planes (and the ragged tail).
static __device__ __noinline__ double cross64_row(const double *__restrict__ prow, int64_t k,
                                              const double2 *lo, const double2 *hi,
                                              const double *tail, double clamp, int lane) {
  const int64_t nq4 = k >> 2;
  const double2 *row2 = reinterpret_cast<const double2 *>(prow);
  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = lane; i < 2 * nq4; i += 32) {
    const double2 v = ldg_stream2(row2 + i);
    const double2 t = (i & 1) ? hi[i >> 1] : lo[i >> 1];
    a0 = fma(fmax(v.x, clamp), t.x, a0);
    a1 = fma(fmax(v.y, clamp), t.y, a1);
  }
  for (int64_t b = 4 * nq4 + lane; b < k; b += 32) a0 = fma(fmax(prow[b], clamp), tail[b - 4 * nq4], a0);
  return warp_sum(a0 + a1);
}

template <bool KL, bool CLAMP, int U = 4, int MINB = 4>
__global__ void __launch_bounds__(kT32, MINB) dense32_kernel(
    const float *__restrict__ P, int64_t ld, int64_t rows, int64_t k,
    const double *__restrict__ H, const double *__restrict__ vec, double clamp, float clamp32,
    double tau, int64_t row0, int64_t target, const double *__restrict__ P64, int64_t ld64,
    const double *__restrict__ H64, double tau64, const double *__restrict__ tgt,
    double *__restrict__ out, uint32_t *__restrict__ flags, int64_t warp_mul) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ GuardRows gq;
  guard_init(gq);
  const int64_t nq4 = k >> 2;  // full float4 groups
  double2 *lo = reinterpret_cast<double2 *>(smem);
  double2 *hi = lo + nq4;
  double *tail = reinterpret_cast<double *>(hi + nq4);
  for (int64_t j = threadIdx.x; j < nq4; j += blockDim.x) {
    lo[j] = make_double2(vec[4 * j], vec[4 * j + 1]);
    hi[j] = make_double2(vec[4 * j + 2], vec[4 * j + 3]);
  }
  for (int64_t b = 4 * nq4 + threadIdx.x; b < k; b += blockDim.x) tail[b - 4 * nq4] = vec[b];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nq = static_cast<int>(nq4);                    // < 2^31 (k <= 25,600)
  const int nfull = nq / (32 * U) * (32 * U);               // chunks with every lane in range
  const int64_t first = (warp * warp_mul) % nwarps;  // scattered rows (pf_common.cuh)
  for (int64_t r = first; r < rows; r += nwarps) {
    const float4 *row = reinterpret_cast<const float4 *>(P + r * ld);
    const double h = KL ? H[r] : 0.0;
    double a0 = 0.0, a1 = 0.0;
    for (int j0 = lane; j0 < nfull; j0 += 32 * U) {   // no bounds checks in the hot loop
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldg_stream4f(row + j0 + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double2 t01 = lo[j0 + 32 * u], t23 = hi[j0 + 32 * u];
        acc32<KL, CLAMP>(v[u].x, t01.x, clamp32, a0);
        acc32<KL, CLAMP>(v[u].y, t01.y, clamp32, a1);
        acc32<KL, CLAMP>(v[u].z, t23.x, clamp32, a0);
        acc32<KL, CLAMP>(v[u].w, t23.y, clamp32, a1);
      }
    }
    if (nq - nfull > 32) {
      // a ragged chunk of several float4 per lane (short rows: C2' has k =
      // 1,310, 71 of its 327 float4 past the full chunk): all its loads in
      // flight at once (in-row clamped addresses), then the in-range ones
      // accumulated in the same per-lane order as the loop below
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = nfull + lane + 32 * u;
        v[u] = ldg_stream4f(row + (j < nq ? j : nq - 1));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = nfull + lane + 32 * u;
        if (j < nq) {
          const double2 t01 = lo[j], t23 = hi[j];
          acc32<KL, CLAMP>(v[u].x, t01.x, clamp32, a0);
          acc32<KL, CLAMP>(v[u].y, t01.y, clamp32, a1);
          acc32<KL, CLAMP>(v[u].z, t23.x, clamp32, a0);
          acc32<KL, CLAMP>(v[u].w, t23.y, clamp32, a1);
        }
      }
    } else {
      for (int j = nfull + lane; j < nq; j += 32) {   // the ragged chunk
        const float4 v = ldg_stream4f(row + j);
        const double2 t01 = lo[j], t23 = hi[j];
        acc32<KL, CLAMP>(v.x, t01.x, clamp32, a0);
        acc32<KL, CLAMP>(v.y, t01.y, clamp32, a1);
        acc32<KL, CLAMP>(v.z, t23.x, clamp32, a0);
        acc32<KL, CLAMP>(v.w, t23.y, clamp32, a1);
      }
    }
    for (int64_t b = 4 * nq4 + lane; b < k; b += 32)  // ragged tail (< 4 columns)
      acc32<KL, CLAMP>(P[r * ld + b], tail[b - 4 * nq4], clamp32, a0);
    const double s = warp_sum(a0 + a1);
    const bool is_t = (row0 + r == target);
    double val;
    bool guard;
    if (KL) {
      val = h - s;
      guard = fabs(val) < tau * fabs(s);
    } else {
      val = s;
      guard = fabs(val) < tau;
    }
    if (is_t) {
      val = 0.0;
    } else if (guard) {  // warp-uniform: re-evaluated in FP64 in place
      if (lane == 0) atomicAdd(&flags[PF_FLAG_GUARDED], 1u);
      if (KL && H64) {
        const double h64 = H64[r];
        const double c64 = cross64_row(P64 + r * ld64, k, lo, hi, tail, clamp, lane);
        val = h64 - c64;
        if (fabs(val) < tau64 * (fabs(h64) + fabs(c64))) {  // the FP64 guard
          guard_note(gq, r, out, lane);  // the reference form, by the CTA after the loop
          continue;
        } else {
          val = settle(val);
        }
      } else {
        val = guard64_row<KL>(P64 + r * ld64, k, tgt, clamp, lane);
      }
    } else {
      val = settle(val);
    }
    if (lane == 0) out[r] = val;
  }
  if (KL)  // partials reuse the staged lo / hi planes (dead after the loop)
    guard_drain(gq, reinterpret_cast<double *>(smem), P64, ld64, rows, k, tgt, clamp, out, flags,
                false, first, nwarps);
}

// flag[0] |= 1 if the below-clamp masks of rows a and b differ (k entries).
__global__ void mask_compare_kernel(const double *__restrict__ a, const double *__restrict__ b,
                                    int64_t k, double clamp, uint32_t *__restrict__ flag) {
  bool d = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    d |= (a[i] < clamp) != (b[i] < clamp);
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(flag, 1u);
}

__global__ void convert_f32_kernel(const double *__restrict__ P, int64_t ld, int64_t rows,
                                   int64_t k, float *__restrict__ out, int64_t ld32) {
  const int64_t n = rows * ld32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld32, c = i - r * ld32;
    out[i] = c < k ? __double2float_rn(P[r * ld + c]) : 0.0f;
  }
}

template <bool KL>
static int launch32(const float *P, int64_t ld, int64_t rows, int64_t k, const double *H,
                    const double *vec, double clamp, double tau, int64_t row0, int64_t target,
                    const double *P64, int64_t ld64, const double *H64, double tau64,
                    const double *tgt, double *out, uint32_t *flags, cudaStream_t stream) {
  size_t smem = static_cast<size_t>(k) * 8 + 32;
  if (smem < kGuardPartBytes) smem = kGuardPartBytes;
  if (smem > 200 * 1024) return fail(PF_E_DOMAIN, "dense32: k=%lld too large", (long long)k);
  // the clamp in FP32, rounded to nearest; flushed to 0 (no max) below FLT_MIN
  const float clamp32 = clamp >= static_cast<double>(FLT_MIN) ? static_cast<float>(clamp) : 0.0f;
  // 8 float4 per lane in flight, 3 CTAs x 8 warps per SM: re-tuned once the loop
  // stopped being ALU-bound (synthetic C4: (U, CTAs) = (8, 3) 6.96 / 6.96 TB/s
  // KL / TV, (4, 4) 6.86 / 6.87, (6, 4) 6.89 / 6.98, (6, 5) 6.81 / 6.93)
  auto kern = clamp32 > 0.0f ? dense32_kernel<KL, true, 8, 3> : dense32_kernel<KL, false, 8, 3>;
  if (int e = ensure_smem((const void *)kern, smem)) return e;
  const int occ = occupancy((const void *)kern, kT32, smem);
  int64_t g = static_cast<int64_t>(sm_count()) * occ, want = (rows + 7) / 8;
  if (g > want) g = want;
  if (g < 1) g = 1;
  if (!P64 || !tgt || !flags) return fail(PF_E_ARG, "dense32: the FP64 guard needs P64, tgt, flags");
  if ((ld64 & 1) || (reinterpret_cast<uintptr_t>(P64) & 15))
    return fail(PF_E_ALIGN, "dense32: FP64 rows must be 16-byte aligned");
  kern<<<static_cast<int>(g), kT32, smem, stream>>>(P, ld, rows, k, H, vec, clamp, clamp32, tau,
                                                    row0, target, P64, ld64, H64, tau64, tgt, out,
                                                    flags, guard_warp_mul(g * (kT32 / 32)));
  return check_launch("dense32");  // guarded rows were re-evaluated in place
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_convert_f32(const double *P, int64_t ld, int64_t rows, int64_t k, float *out,
                   int64_t ld32, pf_stream_t stream) {
  if (rows <= 0) return 0;
  if (!P || !out || ld32 < k || (ld32 & 3)) return fail(PF_E_ARG, "convert_f32: bad args");
  convert_f32_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(P, ld, rows, k, out, ld32);
  return check_launch("convert_f32");
}

int pf_row_negentropy_f32(const float *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                          double *H, pf_stream_t stream) {
  if (rows <= 0) return 0;
  if (!P || !H) return fail(PF_E_ARG, "row_negentropy_f32: null");
  row_negentropy32_kernel<<<sm_count() * 8, kT32, 0, as_stream(stream)>>>(P, ld, rows, k, clamp,
                                                                          H);
  return check_launch("row_negentropy_f32");
}

int pf_dense_kl_f32(const float *P, int64_t ld, int64_t rows, int64_t k, const double *H,
                    const double *tgt, const double *logt, const uint8_t *tmask, double clamp,
                    double tau, int64_t row0, int64_t target, const uint8_t *is_interior,
                    const double *P64, int64_t ld64, const double *H64, double tau64,
                    double *out, uint32_t *flags, pf_stream_t stream) {
  if (rows <= 0) return 0;
  if (!P || !H || !tgt || !logt || !tmask || !P64 || !out || !flags)
    return fail(PF_E_ARG, "dense_kl_f32: null");
  if ((ld & 3) || (reinterpret_cast<uintptr_t>(P) & 15))
    return fail(PF_E_ALIGN, "dense_kl_f32: FP32 rows must be 16-byte aligned");
  (void)tmask;
  (void)is_interior;
  return launch32<true>(P, ld, rows, k, H, logt, clamp, tau, row0, target, P64, ld64, H64, tau64,
                        tgt, out, flags, as_stream(stream));
}

int pf_dense_tv_f32(const float *P, int64_t ld, int64_t rows, int64_t k, const double *tgt,
                    const uint8_t *tmask, double clamp, double tau, int64_t row0, int64_t target,
                    const uint8_t *is_interior, const double *P64, int64_t ld64, double *out,
                    uint32_t *flags, pf_stream_t stream) {
  if (rows <= 0) return 0;
  if (!P || !tgt || !tmask || !P64 || !out || !flags) return fail(PF_E_ARG, "dense_tv_f32: null");
  if ((ld & 3) || (reinterpret_cast<uintptr_t>(P) & 15))
    return fail(PF_E_ALIGN, "dense_tv_f32: FP32 rows must be 16-byte aligned");
  (void)tmask;
  (void)is_interior;
  return launch32<false>(P, ld, rows, k, nullptr, tgt, clamp, tau, row0, target, P64, ld64,
                         nullptr, 0.0, tgt, out, flags, as_stream(stream));
}

int pf_mask_compare_f64(const double *a, const double *b, int64_t k, double clamp,
                        uint32_t *flag, pf_stream_t stream) {
  if (k <= 0) return 0;
  if (!a || !b || !flag) return fail(PF_E_ARG, "mask_compare: null");
  int blocks = static_cast<int>((k + 255) / 256);
  if (blocks > 64) blocks = 64;
  mask_compare_kernel<<<blocks, 256, 0, as_stream(stream)>>>(a, b, k, clamp, flag);
  return check_launch("mask_compare");
}

}  // extern "C"
