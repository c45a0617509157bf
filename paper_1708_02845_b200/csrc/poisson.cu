// poisson.cu — K11: the discrete Poisson kernel P on the GPU.
//
// Reference: pathfield/laplacian.py:29-134 (cotan assembly, SuperLU of
// -Lc_II) and pathfield/solvers.py:278-303 (P_IB = -Lc_II^{-1} Lc_IB, one
// back-substitution per boundary column, clip of tiny negatives, residual
// and row-sum diagnostics).
//
// Pipeline (host plan: nd_plan.cpp; orchestration: laplacian.py):
//   cotan_kernel / laplacian_diag_kernel   Lc, bitwise the reference's
//   mf_factor_kernel   per tree level      multifrontal Cholesky of A = -Lc_II
//   mf_forward_kernel  per tree level      L Y = B over active 32-column tiles
//   mf_backward_kernel per tree level      L^T X = Y, in place in P's rows
//   residual / finalize                    diagnostics, indicators, clip
//
// Fronts are dense row-major f x f FP64 blocks (lower triangle used); the
// pivot block is factored by one warp in shared memory, panel rows below it
// by a per-thread triangular solve, and the trailing (Schur) update runs in
// 64 x 64 shared-memory tiles.  Both solves stage 32 x 32 blocks of the
// factor and of the right-hand sides in shared memory; a CTA owns a front
// (and a range of column tiles), so no two CTAs ever write the same P entry
// and every sum has a fixed order: results are deterministic run to run.
#include <cfloat>

#include "pf_common.cuh"

namespace pf {
namespace {

constexpr int kT = 32;        // column tile of the solves (plan.tile)
constexpr int kThreads = 256;

// ---------------------------------------------------------------- cotan --
__device__ __forceinline__ int64_t find_col(const int64_t *nb_ptr, const int32_t *nb_idx,
                                            int32_t row, int32_t col) {
  int64_t lo = nb_ptr[row], hi = nb_ptr[row + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (nb_idx[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return lo;  // the edge exists by construction (neighbour CSR of the same mesh)
}

// laplacian.py:103-121, one thread per triangle: corner c contributes
// 0.5 * (u.w)/|u x w| to edge (c1, c2).  Explicit _rn intrinsics keep numpy's
// unfused products; the <= 2 contributions per directed entry are added to
// an initial -0.0 (x + y in either order is the same double).
__global__ void cotan_kernel(const double *__restrict__ V, const int32_t *__restrict__ T,
                             int64_t nt, const int64_t *__restrict__ nb_ptr,
                             const int32_t *__restrict__ nb_idx, double *off,
                             unsigned long long *bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v[3] = {T[3 * t], T[3 * t + 1], T[3 * t + 2]};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int32_t k0 = v[c], i1 = v[(c + 1) % 3], j2 = v[(c + 2) % 3];
      const double u0 = __dsub_rn(V[2 * i1], V[2 * k0]), u1 = __dsub_rn(V[2 * i1 + 1], V[2 * k0 + 1]);
      const double w0 = __dsub_rn(V[2 * j2], V[2 * k0]), w1 = __dsub_rn(V[2 * j2 + 1], V[2 * k0 + 1]);
      const double cross = __dsub_rn(__dmul_rn(u0, w1), __dmul_rn(u1, w0));
      if (cross == 0.0) atomicMin(bad, (unsigned long long)t);
      const double dot = __dadd_rn(__dmul_rn(u0, w0), __dmul_rn(u1, w1));
      const double half = __dmul_rn(0.5, __ddiv_rn(dot, fabs(cross)));
      atomicAdd(off + find_col(nb_ptr, nb_idx, i1, j2), half);
      atomicAdd(off + find_col(nb_ptr, nb_idx, j2, i1), half);
    }
  }
}

__global__ void init_bad_kernel(unsigned long long *bad) { *bad = 0x7fffffffffffffffull; }

__global__ void fill_kernel(double *p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// laplacian.py:127: diag = -off.sum(axis=1) — scipy reduces a CSR row with
// np.add.reduceat: first entry + numpy pairwise sum of the rest (sorted
// columns); an empty row sums to 0.
__global__ void laplacian_diag_kernel(const int64_t *__restrict__ nb_ptr,
                                      const double *__restrict__ off, int64_t n,
                                      double *__restrict__ diag) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = nb_ptr[v], hi = nb_ptr[v + 1];
    double s = 0.0;
    if (hi - lo == 1) s = off[lo];
    else if (hi - lo > 1) s = off[lo] + np_pairwise_sum(off + lo + 1, hi - lo - 1);
    diag[v] = -s;
  }
}

// ------------------------------------------------------- factorisation --
// One CTA per front of the level.
__global__ void __launch_bounds__(kThreads)
    mf_factor_kernel(pf_mf_plan_t p, const double *__restrict__ off,
                     const double *__restrict__ diag, const int32_t *__restrict__ nodes,
                     double *F, int32_t *err) {
  __shared__ double D[kT][kT + 1];
  __shared__ double Ai[64][kT + 1];
  __shared__ double Al[64][kT + 1];
  const int s = nodes[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s];
  double *Fs = F + p.foff[s];
  const int tid = threadIdx.x;
  const int64_t ff = (int64_t)f * f;
  for (int64_t i = tid; i < ff; i += kThreads) Fs[i] = 0.0;
  __syncthreads();
  for (int64_t e = p.a_ptr[s] + tid; e < p.a_ptr[s + 1]; e += kThreads) {
    const int64_t src = p.a_src[e];
    F[p.a_dst[e]] = src >= 0 ? -off[src] : -diag[-1 - src];
  }
  __syncthreads();
  // extend-add of the children's update matrices, one child at a time
  for (int q = p.ch_ptr[s]; q < p.ch_ptr[s + 1]; ++q) {
    const int ch = p.ch_idx[q];
    const int fc = p.fn[ch], cc = p.cn[ch], rc = p.rn[ch];
    const double *U = F + p.foff[ch] + (int64_t)cc * fc + cc;
    const int32_t *mp = p.relmap + p.relmap_off[ch];
    for (int a = tid / 32; a < rc; a += kThreads / 32) {
      const int64_t dst = (int64_t)mp[a] * f;
      for (int b = tid % 32; b <= a; b += 32) Fs[dst + mp[b]] += U[(int64_t)a * fc + b];
    }
    __syncthreads();
  }
  // partial Cholesky of the first c columns, 32-wide panels
  for (int p0 = 0; p0 < c; p0 += kT) {
    const int pb = min(kT, c - p0);
    for (int idx = tid; idx < kT * kT; idx += kThreads) {
      const int i = idx / kT, j = idx % kT;
      double v;
      if (i < pb && j <= i) v = Fs[(int64_t)(p0 + i) * f + p0 + j];
      else v = (i == j) ? 1.0 : 0.0;  // identity padding: the unrolled TRSM divides by it
      D[i][j] = v;
    }
    __syncthreads();
    if (tid < 32) {
      const int lane = tid;
      for (int j = 0; j < pb; ++j) {
        const double djj = D[j][j];
        if (!(djj > 0.0)) atomicOr(err, 1);
        const double d = sqrt(djj);
        __syncwarp();
        if (lane == j) D[j][j] = d;
        if (lane > j && lane < pb) D[lane][j] /= d;
        __syncwarp();
        if (lane > j && lane < pb) {
          const double lij = D[lane][j];
          for (int l = j + 1; l <= lane; ++l) D[lane][l] -= lij * D[l][j];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    for (int idx = tid; idx < pb * pb; idx += kThreads) {
      const int i = idx / pb, j = idx % pb;
      if (j <= i) Fs[(int64_t)(p0 + i) * f + p0 + j] = D[i][j];
    }
    // panel rows below the pivot block: x D^T = row
    for (int i = p0 + pb + tid; i < f; i += kThreads) {
      double *row = Fs + (int64_t)i * f + p0;
      double x[kT];
#pragma unroll
      for (int j = 0; j < kT; ++j) {
        double v = j < pb ? row[j] : 0.0;
#pragma unroll
        for (int l = 0; l < j; ++l) v -= x[l] * D[j][l];
        x[j] = v / D[j][j];
      }
#pragma unroll
      for (int j = 0; j < kT; ++j)
        if (j < pb) row[j] = x[j];
    }
    __syncthreads();
    // trailing update F[q0:, q0:] -= L[q0:, p0:p0+pb] L[q0:, p0:p0+pb]^T (lower)
    const int q0 = p0 + pb, nr = f - q0;
    const int nb = (nr + 63) / 64;
    const int ri = tid / 16, ci = tid % 16;
    for (int pr = 0; pr < nb * (nb + 1) / 2; ++pr) {
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= pr) ++ti;
      const int tl = pr - ti * (ti + 1) / 2;
      const int gi0 = q0 + ti * 64, gl0 = q0 + tl * 64;
      for (int idx = tid; idx < 64 * kT; idx += kThreads) {
        const int r = idx / kT, j = idx % kT;
        Ai[r][j] = (gi0 + r < f && j < pb) ? Fs[(int64_t)(gi0 + r) * f + p0 + j] : 0.0;
        Al[r][j] = (gl0 + r < f && j < pb) ? Fs[(int64_t)(gl0 + r) * f + p0 + j] : 0.0;
      }
      __syncthreads();
      double acc[4][4] = {};
      for (int j = 0; j < pb; ++j) {
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = Ai[ri + 16 * u][j];
          b[u] = Al[ci + 16 * u][j];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w = 0; w < 4; ++w) acc[u][w] += a[u] * b[w];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int gi = gi0 + ri + 16 * u;
        if (gi >= f) continue;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int gl = gl0 + ci + 16 * w;
          if (gl <= gi) Fs[(int64_t)gi * f + gl] -= acc[u][w];
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------- forward solve --
// One CTA per active (node, tile) item: W = [B_C; 0] + sum of children's V,
// Y_C = L_CC^{-1} W_C (into P's rows), V = W_R - L_RC Y_C.
__global__ void __launch_bounds__(kThreads)
    mf_forward_kernel(pf_mf_plan_t p, const double *__restrict__ F,
                      const double *__restrict__ off, const int32_t *__restrict__ item_node,
                      const int64_t *__restrict__ item_id, double *V, double *P, int64_t ldp) {
  __shared__ double D[kT][kT + 1];
  __shared__ double Y[kT][kT + 1];
  const int s = item_node[blockIdx.x];
  const int64_t it = item_id[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s], r = p.rn[s];
  const double *Fs = F + p.foff[s];
  const int tile = p.act_tile[it];
  const int64_t j0 = (int64_t)tile * kT;
  const int w = (int)min((int64_t)kT, p.k - j0);
  const int32_t *Cv = p.perm_orig + p.c0[s];
  double *Vs = V + p.act_voff[it];
  const int tid = threadIdx.x, t = tid % kT, g = tid / kT;
  auto Wrow = [&](int i) -> double * {
    return i < c ? P + (int64_t)Cv[i] * ldp + j0 : Vs + (int64_t)(i - c) * kT;
  };
  for (int i = g; i < f; i += kThreads / kT)
    if (t < w || i >= c) Wrow(i)[t] = 0.0;
  __syncthreads();
  for (int64_t e = p.b_ptr[s] + tid; e < p.b_ptr[s + 1]; e += kThreads) {
    const int64_t col = p.b_col[e] - j0;
    if (col >= 0 && col < w) Wrow(p.b_row[e])[col] = off[p.b_src[e]];
  }
  __syncthreads();
  for (int q = p.ch_ptr[s]; q < p.ch_ptr[s + 1]; ++q) {
    const int ch = p.ch_idx[q];
    const int64_t ic = p.tile_item[(int64_t)ch * p.ntiles + tile];
    if (ic < 0) continue;
    const int rc = p.rn[ch];
    const double *Vc = V + p.act_voff[ic];
    const int32_t *mp = p.relmap + p.relmap_off[ch];
    for (int a = g; a < rc; a += kThreads / kT)
      if (t < w) Wrow(mp[a])[t] += Vc[(int64_t)a * kT + t];
    __syncthreads();
  }
  for (int jb = 0; jb < c; jb += kT) {
    const int nb = min(kT, c - jb);
    for (int idx = tid; idx < kT * kT; idx += kThreads) {
      const int i = idx / kT, j = idx % kT;
      D[i][j] = (i < nb && j <= i) ? Fs[(int64_t)(jb + i) * f + jb + j] : 0.0;
      Y[i][j] = (i < nb && j < w) ? Wrow(jb + i)[j] : 0.0;
    }
    __syncthreads();
    if (tid < kT) {
      for (int j = 0; j < nb; ++j) {
        double y = Y[j][t];
        for (int l = 0; l < j; ++l) y -= D[j][l] * Y[l][t];
        Y[j][t] = y / D[j][j];
      }
    }
    __syncthreads();
    for (int i = g; i < nb; i += kThreads / kT)
      if (t < w) Wrow(jb + i)[t] = Y[i][t];
    for (int i = jb + nb + g; i < f; i += kThreads / kT) {
      const double *Lr = Fs + (int64_t)i * f + jb;
      double acc = 0.0;
      for (int l = 0; l < nb; ++l) acc += Lr[l] * Y[l][t];
      if (t < w || i >= c) Wrow(i)[t] -= acc;
    }
    __syncthreads();
  }
  (void)r;
}

// ------------------------------------------------------ backward solve --
// One CTA per (node, tiles [t0, t1)) item, levels top-down:
//   Z = Y_C - L_RC^T X_R ;  X_C = L_CC^{-T} Z   (in place in P's C rows).
__global__ void __launch_bounds__(kThreads)
    mf_backward_kernel(pf_mf_plan_t p, const double *__restrict__ F,
                       const int32_t *__restrict__ item_node, const int32_t *__restrict__ item_t0,
                       const int32_t *__restrict__ item_t1, double *P, int64_t ldp) {
  __shared__ double D[kT][kT + 1];
  __shared__ double Y[kT][kT + 1];
  constexpr int kRows = kThreads / kT;  // 8 row groups
  constexpr int kRB = 8;                // rows per thread in the R sweep
  const int s = item_node[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s], r = p.rn[s];
  if (c == 0) return;
  const double *Fs = F + p.foff[s];
  const int32_t *Cv = p.perm_orig + p.c0[s];
  const int32_t *Rv = p.r_orig + p.r_ptr[s];
  const int tid = threadIdx.x, t = tid % kT, g = tid / kT;
  for (int tile = item_t0[blockIdx.x]; tile < item_t1[blockIdx.x]; ++tile) {
    const int64_t j0 = (int64_t)tile * kT;
    const int w = (int)min((int64_t)kT, p.k - j0);
    const bool active = p.tile_item[(int64_t)s * p.ntiles + tile] >= 0;
    if (!active)
      for (int i = g; i < c; i += kRows)
        if (t < w) P[(int64_t)Cv[i] * ldp + j0 + t] = 0.0;
    __syncthreads();
    // Z -= L_RC^T X_R, C rows in blocks of kRows * kRB
    for (int ib = 0; ib < c; ib += kRows * kRB) {
      double acc[kRB] = {};
      for (int rb = 0; rb < r; rb += kT) {
        const int nr = min(kT, r - rb);
        for (int idx = tid; idx < kT * kT; idx += kThreads) {
          const int l = idx / kT, j = idx % kT;
          Y[l][j] = (l < nr && j < w) ? P[(int64_t)Rv[rb + l] * ldp + j0 + j] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kRB; ++u) {
          const int i = ib + g + kRows * u;
          if (i < c) {
            const double *Lc = Fs + (int64_t)(c + rb) * f + i;
            double a = 0.0;
            for (int l = 0; l < nr; ++l) a += Lc[(int64_t)l * f] * Y[l][t];
            acc[u] += a;
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < kRB; ++u) {
        const int i = ib + g + kRows * u;
        if (i < c && t < w) P[(int64_t)Cv[i] * ldp + j0 + t] -= acc[u];
      }
    }
    __syncthreads();
    // X_C = L_CC^{-T} Z, 32-row blocks from the bottom
    for (int jb = ((c - 1) / kT) * kT; jb >= 0; jb -= kT) {
      const int nb = min(kT, c - jb);
      for (int idx = tid; idx < kT * kT; idx += kThreads) {
        const int i = idx / kT, j = idx % kT;
        D[i][j] = (i < nb && j <= i) ? Fs[(int64_t)(jb + i) * f + jb + j] : 0.0;
        Y[i][j] = (i < nb && j < w) ? P[(int64_t)Cv[jb + i] * ldp + j0 + j] : 0.0;
      }
      __syncthreads();
      if (tid < kT) {
        for (int j = nb - 1; j >= 0; --j) {
          double x = Y[j][t];
          for (int l = j + 1; l < nb; ++l) x -= D[l][j] * Y[l][t];
          Y[j][t] = x / D[j][j];
        }
      }
      __syncthreads();
      for (int i = g; i < nb; i += kRows)
        if (t < w) P[(int64_t)Cv[jb + i] * ldp + j0 + t] = Y[i][t];
      for (int i = g; i < jb; i += kRows) {
        const double *Lc = Fs + (int64_t)jb * f + i;
        double a = 0.0;
        for (int l = 0; l < nb; ++l) a += Lc[(int64_t)l * f] * Y[l][t];
        if (t < w) P[(int64_t)Cv[i] * ldp + j0 + t] -= a;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------- diagnostics ------
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long *p, double v) {
  // non-negative doubles order like their bit patterns; NaN propagates as max
  atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

// Warp per interior row: max_j |diag[v] P[v,j] + sum_e off[e] P[u_e, j]|,
// boundary neighbours contributing off[e] to column bcol[u].
__global__ void residual_kernel(const double *__restrict__ P, int64_t ldp, int64_t n, int64_t k,
                                const uint8_t *__restrict__ isb, const int32_t *__restrict__ bcol,
                                const int64_t *__restrict__ nb_ptr,
                                const int32_t *__restrict__ nb_idx,
                                const double *__restrict__ off, const double *__restrict__ diag,
                                unsigned long long *out) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  double mx = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; v < n;
       v += warps) {
    if (isb[v]) continue;
    const int64_t e0 = nb_ptr[v], e1 = nb_ptr[v + 1];
    const double dv = diag[v];
    for (int64_t j = lane; j < k; j += 32) {
      double acc = dv * P[v * ldp + j];
      for (int64_t e = e0; e < e1; ++e) {
        const int32_t u = nb_idx[e];
        const double x = isb[u] ? (bcol[u] == j ? 1.0 : 0.0) : P[(int64_t)u * ldp + j];
        acc += off[e] * x;
      }
      mx = fmax(mx, fabs(acc));
    }
  }
  mx = warp_max(mx);
  if (lane == 0) atomic_max_nonneg(out, mx);
}

__global__ void finalize_kernel(double *P, int64_t ldp, int64_t n, int64_t k,
                                const uint8_t *__restrict__ isb, const int32_t *__restrict__ bcol,
                                unsigned long long *out) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  double mx = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; v < n;
       v += warps) {
    double *row = P + v * ldp;
    if (isb[v]) {
      const int32_t b = bcol[v];
      for (int64_t j = lane; j < ldp; j += 32) row[j] = (j == b) ? 1.0 : 0.0;
      continue;  // rows sum to exactly 1
    }
    double s = 0.0;
    for (int64_t j = lane; j < k; j += 32) {
      double x = row[j];
      if (x > -1e-12 && x < 0.0) {  // solvers.py:293-295
        x = 0.0;
        row[j] = 0.0;
      }
      s += x;
    }
    for (int64_t j = k + lane; j < ldp; j += 32) row[j] = 0.0;
    s = warp_sum(s);
    mx = fmax(mx, fabs(s - 1.0));
  }
  if (lane == 0) atomic_max_nonneg(out, mx);
}

int grid_for(int64_t work, int per_block) {
  const int64_t b = (work + per_block - 1) / per_block;
  const int64_t cap = (int64_t)sm_count() * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" {

int pf_cotan_laplacian_f64(const double *V, const int32_t *T, int64_t nt, const int64_t *nb_ptr,
                           const int32_t *nb_idx, int64_t n, int64_t nnz, double *off,
                           double *diag, int64_t *bad, pf_stream_t stream) {
  if (!V || !T || !nb_ptr || !nb_idx || !off || !diag || !bad || nt < 0 || n < 0 || nnz < 0)
    return fail(PF_E_ARG, "pf_cotan_laplacian_f64: bad argument");
  cudaStream_t st = as_stream(stream);
  init_bad_kernel<<<1, 1, 0, st>>>(reinterpret_cast<unsigned long long *>(bad));
  if (nnz > 0) fill_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(off, nnz, -0.0);
  if (nt > 0)
    cotan_kernel<<<grid_for(nt, 256), 256, 0, st>>>(V, T, nt, nb_ptr, nb_idx, off,
                                                    reinterpret_cast<unsigned long long *>(bad));
  if (n > 0) laplacian_diag_kernel<<<grid_for(n, 256), 256, 0, st>>>(nb_ptr, off, n, diag);
  return check_launch("pf_cotan_laplacian_f64");
}

int pf_mf_factor_level(const pf_mf_plan_t *plan, const double *off, const double *diag,
                       const int32_t *nodes, int64_t count, double *F, int32_t *err,
                       pf_stream_t stream) {
  if (!plan || !off || !diag || !nodes || !F || !err || count < 0 || plan->tile != kT)
    return fail(PF_E_ARG, "pf_mf_factor_level: bad argument");
  if (count == 0) return 0;
  mf_factor_kernel<<<(unsigned)count, kThreads, 0, as_stream(stream)>>>(*plan, off, diag, nodes,
                                                                        F, err);
  return check_launch("pf_mf_factor_level");
}

int pf_mf_forward_level(const pf_mf_plan_t *plan, const double *F, const double *off,
                        const int32_t *item_node, const int64_t *item_id, int64_t count,
                        double *V, double *P, int64_t ldp, pf_stream_t stream) {
  if (!plan || !F || !off || !item_node || !item_id || !V || !P || count < 0 ||
      plan->tile != kT || ldp < plan->k)
    return fail(PF_E_ARG, "pf_mf_forward_level: bad argument");
  if (count == 0) return 0;
  mf_forward_kernel<<<(unsigned)count, kThreads, 0, as_stream(stream)>>>(*plan, F, off, item_node,
                                                                         item_id, V, P, ldp);
  return check_launch("pf_mf_forward_level");
}

int pf_mf_backward_level(const pf_mf_plan_t *plan, const double *F, const int32_t *item_node,
                         const int32_t *item_t0, const int32_t *item_t1, int64_t count,
                         double *P, int64_t ldp, pf_stream_t stream) {
  if (!plan || !F || !item_node || !item_t0 || !item_t1 || !P || count < 0 ||
      plan->tile != kT || ldp < plan->k)
    return fail(PF_E_ARG, "pf_mf_backward_level: bad argument");
  if (count == 0) return 0;
  mf_backward_kernel<<<(unsigned)count, kThreads, 0, as_stream(stream)>>>(
      *plan, F, item_node, item_t0, item_t1, P, ldp);
  return check_launch("pf_mf_backward_level");
}

int pf_poisson_residual(const double *P, int64_t ldp, int64_t n, int64_t k,
                        const uint8_t *is_boundary, const int32_t *bcol, const int64_t *nb_ptr,
                        const int32_t *nb_idx, const double *off, const double *diag,
                        unsigned long long *out_max, pf_stream_t stream) {
  if (!P || !is_boundary || !bcol || !nb_ptr || !nb_idx || !off || !diag || !out_max ||
      n < 0 || k < 0 || ldp < k)
    return fail(PF_E_ARG, "pf_poisson_residual: bad argument");
  if (n == 0) return 0;
  residual_kernel<<<grid_for(n, 8), 256, 0, as_stream(stream)>>>(
      P, ldp, n, k, is_boundary, bcol, nb_ptr, nb_idx, off, diag, out_max);
  return check_launch("pf_poisson_residual");
}

int pf_poisson_finalize(double *P, int64_t ldp, int64_t n, int64_t k,
                        const uint8_t *is_boundary, const int32_t *bcol,
                        unsigned long long *out_max, pf_stream_t stream) {
  if (!P || !is_boundary || !bcol || !out_max || n < 0 || k < 0 || ldp < k)
    return fail(PF_E_ARG, "pf_poisson_finalize: bad argument");
  if (n == 0) return 0;
  finalize_kernel<<<grid_for(n, 8), 256, 0, as_stream(stream)>>>(P, ldp, n, k, is_boundary, bcol,
                                                                  out_max);
  return check_launch("pf_poisson_finalize");
}

}  // extern "C"
