// csr.cu — thresholded sparse Poisson kernel (K4) and CSR KL/TV fields (K5/K6).
//
// Reference semantics: pathfield/divergence.py
//   sparsify              :194-240  (cut = threshold/k, keep P >= cut, or P > 0 at
//                                    threshold 0; CSR with ascending columns;
//                                    log views; dropped = clip(1 - rowsum, 0))
//   dv_pair_sparse_stats  :255-299  (kl: sum over supp(q) of v (log v - log_dense[p]);
//                                    tv: union sum |vp - vq| + dropped[p] + dropped[q])
//
// K4 is count -> scan -> fill over the dense rows (the pattern is bit-exact: the
// same FP64 compare against the same `cut` double).  `dropped` reproduces
// scipy's csr.sum(axis=1) = np.add.reduceat (first element + numpy pairwise sum
// of the rest) so it is bitwise the reference's.
//
// K5/K6 are warp-per-row segmented reductions over the CSR arrays with the
// per-target dense vector (log P[t,:] for KL, the sparsified target row for
// TV) staged once per CTA in shared memory by a TMA bulk copy.  KL uses the
// split form hs[q] - sum v*logPt with hs[q] = sum v log v precomputed at
// sparsify time, and the same cancellation guard + fixup pass as the dense KL
// (the fixup re-evaluates the reference form sum v*(log v - logPt) from the
// stored log view).  TV is restated as a single pass over supp(q):
//   sum_{supp q}(|vq - vp| - vp) + S_p + (dropped_p + dropped_q)
// which equals the union form (1.1e-13) and is exactly
// 2*dropped_p at q = p because S_p is reduced in the same lane order.
#include <cmath>

#include <algorithm>

#include "pf_common.cuh"

namespace pf {

constexpr int kCsrThreads = 256;
constexpr int kCsrMinBlocks = 4;
constexpr int kCsrU = 4;   // entry pairs per lane in flight
constexpr unsigned long long kCsrGuard = 0x7ff8dead0000c5a1ull;  // NaN payload

__device__ __forceinline__ bool keep_entry(double x, double cut, int strict_pos) {
  return strict_pos ? (x > 0.0) : (x >= cut);
}

// ------------------------------------------------------------ K4 count --
__global__ void __launch_bounds__(kCsrThreads) csr_count_kernel(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k, double cut,
    int strict_pos, int64_t *__restrict__ rownnz) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t npair = k >> 1;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const double2 *row = reinterpret_cast<const double2 *>(P + r * ld);
    int cnt = 0;
    for (int64_t j = lane; j < npair; j += 32) {
      const double2 v = ldg_stream2(row + j);
      cnt += keep_entry(v.x, cut, strict_pos) + keep_entry(v.y, cut, strict_pos);
    }
    if ((k & 1) && lane == 0) cnt += keep_entry(P[r * ld + k - 1], cut, strict_pos);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) rownnz[r] = cnt;
  }
}

// ------------------------------------------------------------ K4 fill --
// Columns are visited in ascending order 32 at a time; positions come from a
// ballot prefix, so the output order is scipy's (row-major, ascending).
__global__ void __launch_bounds__(kCsrThreads) csr_fill_kernel(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k, double cut,
    int strict_pos, const int64_t *__restrict__ indptr, int32_t *__restrict__ indices,
    double *__restrict__ data, double *__restrict__ log_data, double *__restrict__ hs) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lower = (1u << lane) - 1u;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const double *row = P + r * ld;
    const int64_t row_lo = indptr[r] & ~1LL;
    int64_t pos = row_lo;
    double acc = 0.0;
    for (int64_t c0 = 0; c0 < k; c0 += 32) {
      const int64_t c = c0 + lane;
      const double x = c < k ? ldg_stream(row + c) : 0.0;
      const bool kp = c < k && keep_entry(x, cut, strict_pos);
      const unsigned ball = __ballot_sync(0xffffffffu, kp);
      if (kp) {
        const int64_t at = pos + __popc(ball & lower);
        const double lg = log(x);
        indices[at] = static_cast<int32_t>(c);
        data[at] = x;
        log_data[at] = lg;
        acc += __dmul_rn(x, lg);
      }
      pos += __popc(ball);
    }
    const double h = warp_sum(acc);
    if (lane == 0) {
      hs[r] = h;
      if ((pos - row_lo) & 1) {  // odd row: one zero pad entry keeps the next row even
        indices[pos] = pos > row_lo ? indices[pos - 1] : 0;
        data[pos] = 0.0;
        log_data[pos] = 0.0;
      }
    }
  }
}

// Row extent of the row-aligned device CSR: every row starts at an even offset
// and a row with an odd number of entries ends with one zero pad entry (kept
// entries are never 0), which is excluded here.  Element order inside a row is
// therefore independent of where the row sits in the arrays, so a row slab of
// the CSR (multi-GPU) reduces every row exactly as the whole CSR does.
// The pad is flagged in bit 0 of the row's END offset (offsets are even), so
// the extent needs no dependent load: lo = ip[r] & ~1, hi = (ip[r+1] & ~1) -
// (ip[r+1] & 1).
__device__ __forceinline__ void row_extent(const int64_t *__restrict__ indptr,
                                           const double *__restrict__ data, int64_t r,
                                           int64_t &lo, int64_t &hi) {
  (void)data;
  const int64_t a = indptr[r], b = indptr[r + 1];
  lo = a & ~1LL;
  hi = (b & ~1LL) - (b & 1);
}

// np_pairwise_sum: pf_common.cuh

// dropped[r] = max(0, 1 - rowsum) with rowsum = np.add.reduceat semantics:
// data[lo] + pairwise(data[lo+1:hi]); empty rows sum to 0 (divergence.py:227-228).
__global__ void csr_dropped_kernel(const int64_t *__restrict__ indptr,
                                   const double *__restrict__ data, int64_t rows,
                                   double *__restrict__ dropped) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo, hi;
    row_extent(indptr, data, r, lo, hi);
    double s = 0.0;
    if (hi - lo == 1) s = data[lo];
    else if (hi - lo > 1) s = data[lo] + np_pairwise_sum(data + lo + 1, hi - lo - 1);
    const double d = 1.0 - s;
    dropped[r] = d < 0.0 ? 0.0 : d;  // np.clip(., 0, None)
  }
}

// Visit the CSR segment [lo, hi) of one row across a warp with 16-byte data
// loads (double2) and 8-byte index loads (int2): an odd head element is
// peeled so the vector body is aligned, the body is unrolled 2x for loads in
// flight, and an odd tail goes to lane 0.  The per-lane visiting order is a
// fixed function of (lo, hi), which K6 relies on (csr_target_prep sums S_p
// with this same traversal, so TV(p, p) cancels exactly).
// Index pairs: int32 columns load as int2 (8 B), 16-bit columns (k < 65,536,
// the B200 layout of pf_csr_narrow_u16) as ushort2 (4 B): 10 instead of 12
// streamed bytes per entry.
__device__ __forceinline__ int2 idx_pair(const int32_t *__restrict__ idx, int64_t s, int64_t j) {
  return __ldg(reinterpret_cast<const int2 *>(idx + s) + j);
}
__device__ __forceinline__ int2 idx_pair(const uint16_t *__restrict__ idx, int64_t s, int64_t j) {
  const ushort2 u = __ldg(reinterpret_cast<const ushort2 *>(idx + s) + j);
  return make_int2(u.x, u.y);
}

template <class Idx, class F>
__device__ __forceinline__ void csr_row_visit(const double *__restrict__ data,
                                              const Idx *__restrict__ idx, int64_t lo,
                                              int64_t hi, int lane, F &&f) {
  int64_t s = lo;
  if ((s & 1) && s < hi) {
    if (lane == 0) f(__ldg(data + s), (int32_t)__ldg(idx + s));
    ++s;
  }
  const int64_t npairs = (hi - s) >> 1;
  const double2 *d2 = reinterpret_cast<const double2 *>(data + s);
  // Up to 8 pairs per lane per block (a ~490-entry row is one block: one
  // memory round trip per row instead of ~3).  Pairs past the row's end load a
  // clamped in-row address and visit (0, column 0): +0 to a KL accumulator, and
  // an even number of visits leaves the lane's alternation unchanged; TV masks
  // them itself (a zero value).  The per-lane order of the real pairs is
  // lane, lane + 32, ... as before.
  if (npairs > 0) {
    for (int64_t j0 = 0; j0 < npairs; j0 += 32 * kCsrU) {
      double2 v[kCsrU];
      int2 cidx[kCsrU];
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        const int64_t j = j0 + lane + 32 * u;
        const int64_t jc = j < npairs ? j : npairs - 1;
        v[u] = __ldg(d2 + jc);
        cidx[u] = idx_pair(idx, s, jc);
      }
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        const bool in = j0 + lane + 32 * u < npairs;
        f(in ? v[u].x : 0.0, in ? cidx[u].x : 0);
        f(in ? v[u].y : 0.0, in ? cidx[u].y : 0);
      }
    }
  }
  if (((hi - s) & 1) && lane == 0) f(__ldg(data + hi - 1), (int32_t)__ldg(idx + hi - 1));
}

// ---------------------------------------------------- K5/K6 target prep --
// vp[k_pad]: the sparsified target row scattered dense (0 off-support);
// tscal[0] = S_p (reduced in the K6 lane order), tscal[1] = dropped[p],
// tscal[2] = nnz_p.  One CTA.
__global__ void csr_target_prep_kernel(const int64_t *__restrict__ indptr,
                                       const int32_t *__restrict__ indices,
                                       const double *__restrict__ data,
                                       const double *__restrict__ dropped, int64_t p, int64_t k,
                                       int64_t k_pad, double *__restrict__ vp,
                                       double *__restrict__ tscal) {
  for (int64_t i = threadIdx.x; i < k_pad; i += blockDim.x) vp[i] = 0.0;
  __syncthreads();
  int64_t lo, hi;
  row_extent(indptr, data, p, lo, hi);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) vp[indices[i]] = data[i];
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double a = 0.0;
    csr_row_visit(data, indices, lo, hi, lane, [&](double v, int32_t) { a += v; });
    a = warp_sum(a);
    if (lane == 0) {
      tscal[0] = a;
      tscal[1] = dropped[p];
      tscal[2] = static_cast<double>(hi - lo);
      tscal[3] = 0.0;
    }
  }
}

__device__ __forceinline__ const double *stage_vec(unsigned char *smem, const double *vec,
                                                   int64_t k_pad) {
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  double *s_vec = reinterpret_cast<double *>(smem + 16);
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t b = static_cast<uint32_t>(k_pad * 8);
    mbar_expect_tx(bar, b);
    bulk_g2s(s_vec, vec, b, bar);
  }
  mbar_wait(bar, 0);
  return s_vec;
}

// Reference form of one guarded CSR KL row, sum v * (log v - logPt)
// (divergence.py:279), one warp: every load of 4 elements per lane issued
// before the dependent logPt gathers, four accumulators, then settle.  Used in
// place by the field kernel and by the scan fixup (same order, same bits).
template <class Idx>
__device__ __forceinline__ double csr_kl_reference_row(const double *__restrict__ data,
                                                       const double *__restrict__ log_data,
                                                       const Idx *__restrict__ indices,
                                                       const double *__restrict__ lt,
                                                       int64_t lo, int64_t hi, int lane) {
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t e = lo + lane;
  for (; e + 96 < hi; e += 128) {
    double d[4], l[4];
    int c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      d[u] = __ldg(data + e + 32 * u);
      l[u] = __ldg(log_data + e + 32 * u);
      c[u] = static_cast<int>(__ldg(indices + e + 32 * u));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) b[u] += __dmul_rn(d[u], l[u] - lt[c[u]]);
  }
  for (; e < hi; e += 32) b[0] += __dmul_rn(__ldg(data + e), __ldg(log_data + e) - lt[__ldg(indices + e)]);
  return settle(warp_sum((b[0] + b[1]) + (b[2] + b[3])));
}

// Guarded rows of the field kernel: the loop only notes them (a shared-memory
// append, past kCsrGuardQ per CTA a sentinel in `out`); after the loop the
// CTA's warps evaluate them in the reference form — out of line, so the
// streaming loop keeps its registers (pf_common.cuh, "guarded KL rows").
constexpr int kCsrGuardQ = 64;
struct CsrGuard {
  int n;
  int64_t out_index[kCsrGuardQ];
};

template <class Idx>
static __device__ __noinline__ void csr_guard_drain(
    CsrGuard &g, const int64_t *__restrict__ indptr, const Idx *__restrict__ indices,
    const double *__restrict__ data, const double *__restrict__ log_data,
    const double *__restrict__ lt, int64_t row0, const int64_t *__restrict__ queries,
    int64_t count, double *__restrict__ out, uint32_t *__restrict__ flags, int64_t first,
    int64_t step) {
  __syncthreads();
  const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int total = g.n, n = total < kCsrGuardQ ? total : kCsrGuardQ;
  for (int j = wc; j < n; j += nw) {
    const int64_t i = g.out_index[j];
    const int64_t r = queries ? queries[i] - row0 : i;
    int64_t lo, hi;
    row_extent(indptr, data, r, lo, hi);
    const double v = csr_kl_reference_row(data, log_data, indices, lt, lo, hi, lane);
    if (lane == 0) out[i] = v;
  }
  if (threadIdx.x == 0 && total) atomicAdd(&flags[PF_FLAG_GUARDED], static_cast<uint32_t>(total));
  if (total > kCsrGuardQ) {  // the rest: sentinels among this warp's own rows
    for (int64_t i = first; i < count; i += step) {
      if (__double_as_longlong(out[i]) != static_cast<long long>(kCsrGuard)) continue;
      const int64_t r = queries ? queries[i] - row0 : i;
      int64_t lo, hi;
      row_extent(indptr, data, r, lo, hi);
      const double v = csr_kl_reference_row(data, log_data, indices, lt, lo, hi, lane);
      if (lane == 0) out[i] = v;
    }
  }
}

// ------------------------------------------------------------ K5 CSR KL --
template <bool STAGE, class Idx, int MINB = kCsrMinBlocks>
__global__ void __launch_bounds__(kCsrThreads, MINB) csr_kl_kernel(
    const int64_t *__restrict__ indptr, const Idx *__restrict__ indices,
    const double *__restrict__ data, const double *__restrict__ log_data,
    const double *__restrict__ hs, int64_t rows, int64_t k_pad,
    const double *__restrict__ logt, double tau, int64_t row0, const int64_t *__restrict__ queries,
    int64_t nq, double *__restrict__ out, int64_t *__restrict__ ops, bool fix_inline,
    uint32_t *__restrict__ flags) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ CsrGuard gq;
  if (threadIdx.x == 0) gq.n = 0;
  if (!STAGE) __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t count = queries ? nq : rows;
  const double *lt = STAGE ? stage_vec(smem, logt, k_pad) : logt;
  int64_t i = warp;
  int64_t r = i < count ? (queries ? queries[i] - row0 : i) : 0;
  int64_t lo = 0, hi = 0;
  if (i < count) row_extent(indptr, data, r, lo, hi);
  while (i < count) {
    // prefetch the next row's extent while this row streams
    const int64_t i2 = i + nwarps;
    const int64_t r2 = i2 < count ? (queries ? queries[i2] - row0 : i2) : 0;
    int64_t lo2 = 0, hi2 = 0;
    if (i2 < count) row_extent(indptr, data, r2, lo2, hi2);
    const double h = hs[r];
    double a0 = 0.0, a1 = 0.0;
    bool odd = false;
    csr_row_visit(data, indices, lo, hi, lane, [&](double v, int32_t c) {
      if (odd) a1 = fma(v, lt[c], a1); else a0 = fma(v, lt[c], a0);
      odd = !odd;
    });
    const double cross = warp_sum(a0 + a1);
    double val = h - cross;
    const bool guarded = fabs(val) < tau * (fabs(h) + fabs(cross));  // warp-uniform
    if (lane == 0) {
      if (guarded) {
        // the reference form after the loop (fix_inline) or by the fixup scan
        int slot = kCsrGuardQ;
        if (fix_inline) slot = atomicAdd(&gq.n, 1);
        if (slot < kCsrGuardQ)
          gq.out_index[slot] = i;
        else
          out[i] = __longlong_as_double(static_cast<long long>(kCsrGuard));
      } else {
        out[i] = settle(val);  // divergence.py:286
      }
      if (ops) ops[i] = hi - lo;  // divergence.py:276
    }
    i = i2;
    r = r2;
    lo = lo2;
    hi = hi2;
  }
  if (fix_inline)
    csr_guard_drain(gq, indptr, indices, data, log_data, lt, row0, queries, count, out, flags,
                    warp, nwarps);
}

// Guarded rows: reference form sum_{supp q} v * (log v - logPt) (divergence.py:279).
template <class Idx>
__global__ void __launch_bounds__(kCsrThreads) csr_kl_fixup_kernel(
    const int64_t *__restrict__ indptr, const Idx *__restrict__ indices,
    const double *__restrict__ data, const double *__restrict__ log_data, int64_t rows,
    const double *__restrict__ logt, int64_t row0, const int64_t *__restrict__ queries,
    int64_t nq, double *__restrict__ out, uint32_t *__restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t count = queries ? nq : rows;
  uint32_t done = 0;
  // interleaved rows: guarded rows cluster around the target, spread them out
  for (int64_t i0 = 0; warp + i0 * nwarps < count; i0 += 32) {
    const int64_t mine = warp + (i0 + lane) * nwarps;
    const bool flag = mine < count && static_cast<unsigned long long>(
                                          __double_as_longlong(out[mine])) == kCsrGuard;
    unsigned ball = __ballot_sync(0xffffffffu, flag);
    while (ball) {
      const int src = __ffs(ball) - 1;
      ball &= ball - 1;
      const int64_t i = warp + (i0 + src) * nwarps;
      const int64_t r = queries ? queries[i] - row0 : i;
      int64_t lo, hi;
      row_extent(indptr, data, r, lo, hi);
      const double val = csr_kl_reference_row(data, log_data, indices, logt, lo, hi, lane);
      if (lane == 0) out[i] = val;
      ++done;
    }
  }
  if (lane == 0 && done && flags) atomicAdd(&flags[PF_FLAG_GUARDED], done);
}

// ------------------------------------------------------------ K6 CSR TV --
template <bool STAGE, class Idx, int MINB = kCsrMinBlocks>
__global__ void __launch_bounds__(kCsrThreads, MINB) csr_tv_kernel(
    const int64_t *__restrict__ indptr, const Idx *__restrict__ indices,
    const double *__restrict__ data, const double *__restrict__ dropped, int64_t rows,
    int64_t k_pad, const double *__restrict__ vp, const double *__restrict__ tscal, int64_t row0,
    const int64_t *__restrict__ queries, int64_t nq, double *__restrict__ out,
    int64_t *__restrict__ ops) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t count = queries ? nq : rows;
  const double *v_p = STAGE ? stage_vec(smem, vp, k_pad) : vp;
  const double S_p = tscal[0], d_p = tscal[1];
  const int64_t nnz_p = static_cast<int64_t>(tscal[2]);
  int64_t i = warp;
  int64_t r = i < count ? (queries ? queries[i] - row0 : i) : 0;
  int64_t lo = 0, hi = 0;
  if (i < count) row_extent(indptr, data, r, lo, hi);
  while (i < count) {
    const int64_t i2 = i + nwarps;
    const int64_t r2 = i2 < count ? (queries ? queries[i2] - row0 : i2) : 0;
    int64_t lo2 = 0, hi2 = 0;
    if (i2 < count) row_extent(indptr, data, r2, lo2, hi2);
    const double d_q = dropped[r];
    // one accumulator per lane in csr_row_visit order (S_p uses the same order,
    // so q == p cancels exactly)
    double a = 0.0;
    int inter = 0;
    csr_row_visit(data, indices, lo, hi, lane, [&](double v, int32_t c) {
      const double w = v_p[c];
      a += fabs(v - w) - w;
      inter += (w != 0.0) && (v != 0.0);   // v == 0: a masked visit (stored entries are > 0)
    });
    const double base = warp_sum(a) + S_p;
    const double val = base + (d_p + d_q);  // divergence.py:293-295 (no settle)
    if (ops) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(0xffffffffu, inter, o);
    }
    if (lane == 0) {
      out[i] = val;
      if (ops) ops[i] = (hi - lo) + nnz_p - inter;  // |union|, divergence.py:289
    }
    i = i2;
    r = r2;
    lo = lo2;
    hi = hi2;
  }
}

// ---------------------------------------------------- other generators --
// divergence.py:275-299 for the remaining builtins.
//  alpha:   sum_{supp q} v (1 - exp(expo (logPt - log v))), times scale; settle.
//  chi2 / hellinger / power-p: the union form over supp(p) U supp(q) with
//  weights clamped at the row cut, vp = max(P[p, j], cut), vq = v (cut
//  off-support):  sum_{supp q} vq f(vp/vq) + sum_{supp p \ supp q} cut f(vp/cut),
//  the second sum by binary search of each supp(p) index in the sorted supp(q)
//  (no restated cancellation: these generators reach 1e18-scale terms).
template <int KIND>
__device__ __forceinline__ double gen_f(double x, double param) {
  if (KIND == PF_DIV_CHI2) return __dsub_rn(__dmul_rn(x, x), 1.0);
  if (KIND == PF_DIV_HELLINGER) {
    const double s = sqrt(x) - 1.0;
    return __dmul_rn(s, s);
  }
  const double d = fabs(1.0 - x);  // PF_DIV_POWER
  return (param == 2.0) ? d * d : pow(d, param);
}

template <int KIND>
__global__ void __launch_bounds__(kCsrThreads) csr_generic_kernel(
    const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
    const double *__restrict__ data, int64_t rows, const double *__restrict__ prow,
    int64_t p_local, double cut, double param, int64_t row0,
    const int64_t *__restrict__ queries, int64_t nq, double *__restrict__ out,
    int64_t *__restrict__ ops) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t count = queries ? nq : rows;
  int64_t plo, phi;
  row_extent(indptr, data, p_local, plo, phi);
  for (int64_t i = warp; i < count; i += nwarps) {
    const int64_t r = queries ? queries[i] - row0 : i;
    int64_t lo, hi;
    row_extent(indptr, data, r, lo, hi);
    double a = 0.0;
    for (int64_t e = lo + lane; e < hi; e += 32) {  // supp(q)
      const double v = data[e];
      const double vp = fmax(__ldg(prow + indices[e]), cut);
      a += __dmul_rn(v, gen_f<KIND>(__ddiv_rn(vp, v), param));
    }
    int inter = 0;
    for (int64_t e = plo + lane; e < phi; e += 32) {  // supp(p) \ supp(q)
      const int32_t j = indices[e];
      int64_t L = lo, R = hi;  // first index >= j in the sorted supp(q)
      while (L < R) {
        const int64_t M = (L + R) >> 1;
        if (indices[M] < j) L = M + 1; else R = M;
      }
      if (L < hi && indices[L] == j) {
        ++inter;
      } else {
        const double vp = fmax(__ldg(prow + j), cut);
        a += __dmul_rn(cut, gen_f<KIND>(__ddiv_rn(vp, cut), param));
      }
    }
    const double val = settle(warp_sum(a));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(0xffffffffu, inter, o);
    if (lane == 0) {
      out[i] = val;
      if (ops) ops[i] = (hi - lo) + (phi - plo) - inter;  // |union|, divergence.py:289
    }
  }
}

__global__ void __launch_bounds__(kCsrThreads) csr_alpha_kernel(
    const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
    const double *__restrict__ data, const double *__restrict__ log_data, int64_t rows,
    const double *__restrict__ logt, double alpha, int64_t row0,
    const int64_t *__restrict__ queries, int64_t nq, double *__restrict__ out,
    int64_t *__restrict__ ops) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t count = queries ? nq : rows;
  const double scale = 4.0 / (1.0 - alpha * alpha), expo = (1.0 + alpha) / 2.0;
  for (int64_t i = warp; i < count; i += nwarps) {
    const int64_t r = queries ? queries[i] - row0 : i;
    int64_t lo, hi;
    row_extent(indptr, data, r, lo, hi);
    double a = 0.0;
    for (int64_t e = lo + lane; e < hi; e += 32) {
      const double rp = exp(__dmul_rn(expo, __ldg(logt + indices[e]) - log_data[e]));
      a += __dmul_rn(data[e], 1.0 - rp);
    }
    const double val = settle(__dmul_rn(scale, warp_sum(a)));
    if (lane == 0) {
      out[i] = val;
      if (ops) ops[i] = hi - lo;
    }
  }
}

__global__ void log_clamped_kernel(const double *__restrict__ P, int64_t ld, int64_t rows,
                                   int64_t k, double clamp, double *__restrict__ out) {
  const int64_t n = rows * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k, c = i - r * k;
    out[i] = log(fmax(P[r * ld + c], clamp));
  }
}

static int grid_for(const void *kern, int threads, size_t smem, int64_t work_warps) {
  int occ = occupancy(kern, threads, smem);
  int64_t want = (work_warps + threads / 32 - 1) / (threads / 32);
  int64_t g = static_cast<int64_t>(sm_count()) * occ;
  if (g > want) g = want;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

template <typename K>
static int smem_attr(K kern, size_t smem) {
  return ensure_smem((const void *)kern, smem);
}

template <class Idx>
int csr_kl_launch(const int64_t *indptr, const Idx *indices, const double *data,
                  const double *log_data, const double *hs, int64_t rows, int64_t k,
                  const double *logt, double tau, int64_t row0, const int64_t *queries,
                  int64_t nq, double *out, int64_t *ops, uint32_t *flags, int inline_guard,
                  pf_stream_t stream) {
  if (inline_guard && (!flags || !log_data))
    return fail(PF_E_ARG, "csr_kl: in-place guard re-evaluation needs flags and log_data");
  if (!indptr || !indices || !hs || !logt || !out || rows < 0 || k <= 0)
    return fail(PF_E_ARG, "csr_kl: bad args");
  const int64_t count = queries ? nq : rows;
  if (count <= 0) return 0;
  const int64_t k_pad = round_up(k, 2);
  const size_t smem = 16 + static_cast<size_t>(k_pad) * 8;
  const bool staged = smem <= 200 * 1024;
  if (staged) {
    auto go = [&](auto kern) -> int {
      if (int e = smem_attr(kern, smem)) return e;
      const int g = grid_for((const void *)kern, kCsrThreads, smem, count);
      kern<<<g, kCsrThreads, smem, as_stream(stream)>>>(
          indptr, indices, data, log_data, hs, rows, k_pad, logt, tau, row0, queries, nq, out,
          ops, inline_guard != 0, flags);
      return 0;
    };
    // 4 CTAs x 8 warps per SM, <= 64 registers (5 or 6 CTAs spill: measured 2x slower)
    if (int e = go(csr_kl_kernel<true, Idx, kCsrMinBlocks>)) return e;
  } else {
    const int g = grid_for((const void *)csr_kl_kernel<false, Idx>, kCsrThreads, 0, count);
    csr_kl_kernel<false, Idx><<<g, kCsrThreads, 0, as_stream(stream)>>>(
        indptr, indices, data, log_data, hs, rows, k_pad, logt, tau, row0, queries, nq, out,
        ops, inline_guard != 0, flags);
  }
  if (int e = check_launch("csr_kl")) return e;
  if (inline_guard) return 0;  // guarded rows were fixed inline
  int64_t want = (count + 7) / 8;
  int64_t g2 = static_cast<int64_t>(sm_count()) * 4;
  if (g2 > want) g2 = want;
  if (g2 < 1) g2 = 1;
  csr_kl_fixup_kernel<Idx><<<static_cast<int>(g2), kCsrThreads, 0, as_stream(stream)>>>(
      indptr, indices, data, log_data, rows, logt, row0, queries, nq, out, flags);
  return check_launch("csr_kl_fixup");
}

template <class Idx>
int csr_tv_launch(const int64_t *indptr, const Idx *indices, const double *data,
                  const double *dropped, int64_t rows, int64_t k, const double *vp,
                  const double *tscal, int64_t row0, const int64_t *queries, int64_t nq,
                  double *out, int64_t *ops, pf_stream_t stream) {
  if (!indptr || !indices || !dropped || !vp || !tscal || !out || rows < 0 || k <= 0)
    return fail(PF_E_ARG, "csr_tv: bad args");
  const int64_t count = queries ? nq : rows;
  if (count <= 0) return 0;
  const int64_t k_pad = round_up(k, 2);
  const size_t smem = 16 + static_cast<size_t>(k_pad) * 8;
  if (smem <= 200 * 1024) {
    auto go = [&](auto kern) -> int {
      if (int e = smem_attr(kern, smem)) return e;
      const int g = grid_for((const void *)kern, kCsrThreads, smem, count);
      kern<<<g, kCsrThreads, smem, as_stream(stream)>>>(
          indptr, indices, data, dropped, rows, k_pad, vp, tscal, row0, queries, nq, out, ops);
      return 0;
    };
    // 4 CTAs x 8 warps per SM, <= 64 registers (5 or 6 CTAs spill: measured 2x slower)
    if (int e = go(csr_tv_kernel<true, Idx, kCsrMinBlocks>)) return e;
  } else {
    const int g = grid_for((const void *)csr_tv_kernel<false, Idx>, kCsrThreads, 0, count);
    csr_tv_kernel<false, Idx><<<g, kCsrThreads, 0, as_stream(stream)>>>(
        indptr, indices, data, dropped, rows, k_pad, vp, tscal, row0, queries, nq, out, ops);
  }
  return check_launch("csr_tv");
}

// Row-aligned device CSR -> scipy's layout (no pads): warp per row copies its
// entries to the row's scipy offset (the exclusive prefix of the real counts).
__global__ void __launch_bounds__(kCsrThreads) csr_unpad_kernel(
    const int64_t *__restrict__ indptr, const int64_t *__restrict__ sp_indptr, int64_t rows,
    const int32_t *__restrict__ indices, const double *__restrict__ data,
    const double *__restrict__ log_data, int32_t *__restrict__ o_indices,
    double *__restrict__ o_data, double *__restrict__ o_log) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    int64_t lo, hi;
    row_extent(indptr, data, r, lo, hi);
    const int64_t d = sp_indptr[r] - lo;
    for (int64_t e = lo + lane; e < hi; e += 32) {
      o_indices[e + d] = indices[e];
      if (o_data) o_data[e + d] = data[e];
      if (o_log) o_log[e + d] = log_data[e];
    }
  }
}

__global__ void narrow_u16_kernel(const int32_t *__restrict__ in, int64_t n,
                                  uint16_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<uint16_t>(in[i]);
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_csr_count_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double cut,
                     int strict_positive, int64_t *rownnz, pf_stream_t stream) {
  if ((!P && rows) || !rownnz || k <= 0 || ld < k || rows < 0)
    return fail(PF_E_ARG, "csr_count: bad args");
  if ((ld & 1) || (reinterpret_cast<uintptr_t>(P) & 15))
    return fail(PF_E_ALIGN, "csr_count: P rows must be 16-byte aligned");
  if (rows == 0) return 0;
  const int g = grid_for((const void *)csr_count_kernel, kCsrThreads, 0, rows);
  csr_count_kernel<<<g, kCsrThreads, 0, as_stream(stream)>>>(P, ld, rows, k, cut,
                                                             strict_positive, rownnz);
  return check_launch("csr_count");
}

int pf_csr_fill_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double cut,
                    int strict_positive, const int64_t *indptr, int32_t *indices, double *data,
                    double *log_data, double *hs, double *dropped, pf_stream_t stream) {
  if ((!P && rows) || !indptr || !hs || !dropped || k <= 0 || ld < k || rows < 0)
    return fail(PF_E_ARG, "csr_fill: bad args");
  if (k > 2147483647LL) return fail(PF_E_DOMAIN, "csr_fill: k exceeds int32 columns");
  if (rows == 0) return 0;
  const int g = grid_for((const void *)csr_fill_kernel, kCsrThreads, 0, rows);
  csr_fill_kernel<<<g, kCsrThreads, 0, as_stream(stream)>>>(P, ld, rows, k, cut, strict_positive,
                                                            indptr, indices, data, log_data, hs);
  if (int e = check_launch("csr_fill")) return e;
  int64_t blocks = (rows + 127) / 128;
  if (blocks > 65535) blocks = 65535;
  csr_dropped_kernel<<<static_cast<int>(blocks), 128, 0, as_stream(stream)>>>(indptr, data, rows,
                                                                             dropped);
  return check_launch("csr_dropped");
}

int pf_csr_target_prep_f64(const int64_t *indptr, const int32_t *indices, const double *data,
                           const double *dropped, int64_t p_local, int64_t k, double *vp,
                           double *tscal, pf_stream_t stream) {
  if (!indptr || !dropped || !vp || !tscal || k <= 0 || p_local < 0)
    return fail(PF_E_ARG, "csr_target_prep: bad args");
  csr_target_prep_kernel<<<1, 512, 0, as_stream(stream)>>>(indptr, indices, data, dropped,
                                                           p_local, k, round_up(k, 2), vp,
                                                           tscal);
  return check_launch("csr_target_prep");
}


int pf_csr_kl_f64(const int64_t *indptr, const int32_t *indices, const double *data,
                  const double *log_data, const double *hs, int64_t rows, int64_t k,
                  const double *logt, double tau, int64_t row0, const int64_t *queries,
                  int64_t nq, double *out, int64_t *ops, uint32_t *flags, int inline_guard,
                  pf_stream_t stream) {
  return csr_kl_launch(indptr, indices, data, log_data, hs, rows, k, logt, tau, row0, queries,
                       nq, out, ops, flags, inline_guard, stream);
}

int pf_csr_kl_u16_f64(const int64_t *indptr, const uint16_t *indices16, const double *data,
                      const double *log_data, const double *hs, int64_t rows, int64_t k,
                      const double *logt, double tau, int64_t row0, const int64_t *queries,
                      int64_t nq, double *out, int64_t *ops, uint32_t *flags, int inline_guard,
                      pf_stream_t stream) {
  if (k > 65536) return fail(PF_E_DOMAIN, "csr_kl_u16: k must be <= 65536");
  return csr_kl_launch(indptr, indices16, data, log_data, hs, rows, k, logt, tau, row0,
                       queries, nq, out, ops, flags, inline_guard, stream);
}

int pf_csr_tv_f64(const int64_t *indptr, const int32_t *indices, const double *data,
                  const double *dropped, int64_t rows, int64_t k, const double *vp,
                  const double *tscal, int64_t row0, const int64_t *queries, int64_t nq,
                  double *out, int64_t *ops, pf_stream_t stream) {
  return csr_tv_launch(indptr, indices, data, dropped, rows, k, vp, tscal, row0, queries, nq,
                       out, ops, stream);
}

int pf_csr_tv_u16_f64(const int64_t *indptr, const uint16_t *indices16, const double *data,
                      const double *dropped, int64_t rows, int64_t k, const double *vp,
                      const double *tscal, int64_t row0, const int64_t *queries, int64_t nq,
                      double *out, int64_t *ops, pf_stream_t stream) {
  if (k > 65536) return fail(PF_E_DOMAIN, "csr_tv_u16: k must be <= 65536");
  return csr_tv_launch(indptr, indices16, data, dropped, rows, k, vp, tscal, row0, queries, nq,
                       out, ops, stream);
}

int pf_csr_unpad(const int64_t *indptr, const int64_t *sp_indptr, int64_t rows,
                 const int32_t *indices, const double *data, const double *log_data,
                 int32_t *o_indices, double *o_data, double *o_log, pf_stream_t stream) {
  if (rows < 0 || (rows && (!indptr || !sp_indptr || !indices || !data || !o_indices)))
    return fail(PF_E_ARG, "csr_unpad: bad args");
  if (o_log && !log_data) return fail(PF_E_ARG, "csr_unpad: o_log needs log_data");
  if (rows == 0) return 0;
  const int g = grid_for((const void *)csr_unpad_kernel, kCsrThreads, 0, rows);
  csr_unpad_kernel<<<g, kCsrThreads, 0, as_stream(stream)>>>(indptr, sp_indptr, rows, indices,
                                                             data, log_data, o_indices, o_data,
                                                             o_log);
  return check_launch("csr_unpad");
}

int pf_csr_narrow_u16(const int32_t *indices, int64_t n, uint16_t *indices16,
                      pf_stream_t stream) {
  if (n < 0 || (n && (!indices || !indices16))) return fail(PF_E_ARG, "csr_narrow_u16: bad args");
  if (n == 0) return 0;
  narrow_u16_kernel<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, sm_count() * 32)), 256, 0, as_stream(stream)>>>(indices, n, indices16);
  return check_launch("csr_narrow_u16");
}

int pf_csr_generic_f64(const int64_t *indptr, const int32_t *indices, const double *data,
                       const double *log_data, int64_t rows, int64_t k, int kind, double param,
                       double cut, const double *prow, int64_t p_local, const double *logt,
                       int64_t row0, const int64_t *queries, int64_t nq, double *out,
                       int64_t *ops, pf_stream_t stream) {
  if (!indptr || !out || rows < 0 || k <= 0) return fail(PF_E_ARG, "csr_generic: bad args");
  const int64_t count = queries ? nq : rows;
  if (count <= 0) return 0;
  const int g = grid_for((const void *)csr_alpha_kernel, kCsrThreads, 0, count);
  if (kind == PF_DIV_ALPHA) {
    if (!logt) return fail(PF_E_ARG, "csr_generic: alpha needs logt");
    csr_alpha_kernel<<<g, kCsrThreads, 0, as_stream(stream)>>>(
        indptr, indices, data, log_data, rows, logt, param, row0, queries, nq, out, ops);
    return check_launch("csr_alpha");
  }
  if (!prow || p_local < 0 || p_local >= rows) return fail(PF_E_ARG, "csr_generic: target row");
#define PF_CSR_GEN(KIND)                                                                  \
  case KIND:                                                                              \
    csr_generic_kernel<KIND><<<g, kCsrThreads, 0, as_stream(stream)>>>(                   \
        indptr, indices, data, rows, prow, p_local, cut, param, row0, queries, nq, out, ops); \
    break;
  switch (kind) {
    PF_CSR_GEN(PF_DIV_CHI2)
    PF_CSR_GEN(PF_DIV_HELLINGER)
    PF_CSR_GEN(PF_DIV_POWER)
    default:
      return fail(PF_E_ARG, "csr_generic: kind %d not supported here", kind);
  }
#undef PF_CSR_GEN
  return check_launch("csr_generic");
}

int pf_log_clamped_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                       double *out, pf_stream_t stream) {
  if ((!P || !out) && rows > 0) return fail(PF_E_ARG, "log_clamped: null");
  if (rows <= 0) return 0;
  const int blocks = sm_count() * 8;
  log_clamped_kernel<<<blocks, 256, 0, as_stream(stream)>>>(P, ld, rows, k, clamp, out);
  return check_launch("log_clamped");
}

}  // extern "C"
