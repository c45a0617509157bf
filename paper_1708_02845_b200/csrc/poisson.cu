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
#include <algorithm>
#include <cfloat>

#include "pf_common.cuh"

namespace pf {
namespace {

constexpr int kT = 32;        // panel / identity tile of the factorisation

// Offset of vertex v's row in the output: v * ldp for the whole P, or the
// row-slab build's table (slab rows first, then the scratch rows of the other
// fronts the slab depends on).
__device__ __forceinline__ int64_t row_off(const pf_mf_plan_t &p, int64_t v, int64_t ldp) {
  return p.rowoff ? p.rowoff[v] : v * ldp;
}
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

// FP64 tensor-core MMA (SASS DMMA): D(8x8) += A(8x4, row) B(4x8, col).
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------- factorisation --
// Building blocks shared by the one-CTA-per-front kernel (many small fronts)
// and the split kernels (few large fronts: every step spread over CTAs).

// Zero rows [r0, r1) of the front, scatter the A entries of those rows, then
// add each child's update matrix (child order) into those rows.  The row
// range makes the assembly of one front splittable across CTAs while every
// entry still receives its contributions in a fixed order.
__device__ __forceinline__ void front_assemble_rows(const pf_mf_plan_t &p, int s,
                                                    const double *__restrict__ off,
                                                    const double *__restrict__ diag, double *F,
                                                    int r0, int r1) {
  const int f = p.fn[s];
  double *Fs = F + p.foff[s];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t i = (int64_t)r0 * f + tid; i < (int64_t)r1 * f; i += nt) Fs[i] = 0.0;
  __syncthreads();
  for (int64_t e = p.a_ptr[s] + tid; e < p.a_ptr[s + 1]; e += nt) {
    const int64_t d = p.a_dst[e] - p.foff[s];
    const int row = (int)(d / f);
    if (row < r0 || row >= r1) continue;
    const int64_t src = p.a_src[e];
    Fs[d] = src >= 0 ? -off[src] : -diag[-1 - src];
  }
  __syncthreads();
  for (int q = p.ch_ptr[s]; q < p.ch_ptr[s + 1]; ++q) {
    const int ch = p.ch_idx[q];
    const int fc = p.fn[ch], cc = p.cn[ch], rc = p.rn[ch];
    const double *U = F + p.foff[ch] + (int64_t)cc * fc + cc;
    const int32_t *mp = p.relmap + p.relmap_off[ch];
    for (int a = tid / 32; a < rc; a += nt / 32) {
      const int ra = mp[a];
      if (ra < r0 || ra >= r1) continue;
      const int64_t dst = (int64_t)ra * f;
      for (int b = tid % 32; b <= a; b += 32) Fs[dst + mp[b]] += U[(int64_t)a * fc + b];
    }
    __syncthreads();
  }
}

// Load the pb x pb pivot block at p0 into D (identity-padded to kT) and, if
// `factor`, Cholesky-factor it with one warp and write it back.
__device__ __forceinline__ void panel_diag(double *Fs, int f, int p0, int pb,
                                           double (*D)[kT + 1], int32_t *err, bool factor,
                                           bool write = true) {
  const int tid = threadIdx.x;
  for (int idx = tid; idx < kT * kT; idx += blockDim.x) {
    const int i = idx / kT, j = idx % kT;
    double v;
    if (i < pb && j <= i) v = Fs[(int64_t)(p0 + i) * f + p0 + j];
    else v = (i == j) ? 1.0 : 0.0;  // identity padding: the unrolled TRSM divides by it
    D[i][j] = v;
  }
  __syncthreads();
  if (!factor) return;
  if (tid < 32) {
    // right-looking, lane i owns row i; the trailing update of step j goes
    // in batches of 8 whose loads all issue before their stores (a plain
    // loop serialises each load behind the previous possibly-aliasing store)
    const int lane = tid;
    for (int j = 0; j < pb; ++j) {
      const double djj = D[j][j];
      if (lane == 0 && !(djj > 0.0)) atomicOr(err, 1);
      const double rd = rsqrt(djj);  // one MUFU-seeded chain; d and the column
      const double d = djj * rd;      // scale both follow from it in parallel
      __syncwarp();
      if (lane == j) D[j][j] = d;
      if (lane > j && lane < pb) D[lane][j] *= rd;
      __syncwarp();
      const double lij = D[lane][j];
      const bool mine = lane > j && lane < pb;
      for (int l0 = j + 1; l0 <= lane; l0 += 8) {
        double cj[8], rv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = min(l0 + u, kT - 1);
          cj[u] = D[l][j];
          rv[u] = D[lane][l];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (mine && l0 + u <= lane) D[lane][l0 + u] = rv[u] - lij * cj[u];
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (!write) return;
  for (int idx = tid; idx < pb * pb; idx += blockDim.x) {
    const int i = idx / pb, j = idx % pb;
    if (j <= i) Fs[(int64_t)(p0 + i) * f + p0 + j] = D[i][j];
  }
}

// Panel rows below the pivot block on the FP64 tensor pipe: with the pivot
// block D factored in shared memory, Dinv = D^{-1} (lower, >= 0 on
// M-matrices: no cancellation) is formed by warp 0 (lane j = column j), then
// X = F[rows, p0:p0+pb] Dinv^T for 64-row chunks chunk0, chunk0 + cstep, ...
// (8 warps as 4 (rows) x 2 (columns), 16 x 16 warp tiles of m8n8k4 DMMAs).
constexpr int kSY = kT + 4;  // row stride 4 mod 16: conflict-free half-warp fragments
__device__ __forceinline__ void panel_trsm_dmma(double *Fs, int f, int p0, int pb,
                                                const double (*D)[kT + 1],
                                                double (*Dinv)[kSY], double (*Xs)[kSY],
                                                int chunk0, int cstep) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    // lane j solves L x = e_j right-looking in its Dinv column: once x_i is
    // final, x_k -= L[k][i] x_i (k > i) are independent FMAs, issued in
    // batches of 8 loads before 8 stores; x_i = x_i * (1 / L[i][i]) keeps
    // the divisions off the dependent chain (entries stay non-negative).
    const int j = tid;
    const double rdj = 1.0 / D[j][j];  // all 32 reciprocals at once, off the chain
    for (int i = 0; i < kT; ++i) Dinv[i][j] = (i == j) ? 1.0 : 0.0;
    for (int i = 0; i < kT; ++i) {
      const double xi = Dinv[i][j] * __shfl_sync(0xffffffffu, rdj, i);
      Dinv[i][j] = xi;
      for (int k0 = i + 1; k0 < kT; k0 += 8) {
        double dv[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = min(k0 + u, kT - 1);
          dv[u] = D[k][i];
          xv[u] = Dinv[k][j];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k0 + u < kT) Dinv[k0 + u][j] = xv[u] - dv[u] * xi;
      }
    }
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, fr = lane >> 2, fc = lane & 3;
  const int r0 = p0 + pb;
  for (int ch = chunk0; r0 + ch * 64 < f; ch += cstep) {
    const int i0 = r0 + ch * 64;
    for (int idx = tid; idx < 64 * kT; idx += blockDim.x) {
      const int r = idx / kT, j = idx % kT;
      Xs[r][j] = (i0 + r < f && j < pb) ? Fs[(int64_t)(i0 + r) * f + p0 + j] : 0.0;
    }
    __syncthreads();
    double acc[2][2][2] = {};
#pragma unroll
    for (int ks = 0; ks < kT; ks += 4) {
      double a[2], b[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) a[u] = Xs[wm * 16 + 8 * u + fr][ks + fc];
#pragma unroll
      for (int v = 0; v < 2; ++v) b[v] = Dinv[wn * 16 + 8 * v + fr][ks + fc];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) dmma884(acc[u][v][0], acc[u][v][1], a[u], b[v]);
    }
    __syncthreads();  // every warp has read Xs before the next chunk overwrites it
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + wm * 16 + 8 * u + fr;
      if (i >= f) continue;
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int col = wn * 16 + 8 * v + 2 * fc + q;
          if (col < pb) Fs[(int64_t)i * f + p0 + col] = acc[u][v][q];
        }
    }
  }
}

// Trailing-update tile (ti, tl), tl <= ti, of 64 x 64 at q0 = p0 + pb:
// F[i][l] -= sum_j L[i][p0+j] L[l][p0+j] (lower triangle only), on the FP64
// tensor pipe: 8 warps as 4 (i) x 2 (l), 16 x 32 warp tiles of m8n8k4 DMMAs
// over the (<= 32)-deep panel; A = the tile's panel rows, B = the other
// tile's panel rows transposed.  Row stride kSY = 36 (4 mod 16): conflict-free
// half-warp fragment loads.
__device__ __forceinline__ void panel_syrk_tile(double *Fs, int f, int p0, int pb, int ti,
                                                int tl, double (*Ai)[kSY], double (*Al)[kSY]) {
  const int tid = threadIdx.x;
  const int q0 = p0 + pb;
  const int gi0 = q0 + ti * 64, gl0 = q0 + tl * 64;
  for (int idx = tid; idx < 64 * kT; idx += blockDim.x) {
    const int r = idx / kT, j = idx % kT;
    Ai[r][j] = (gi0 + r < f && j < pb) ? Fs[(int64_t)(gi0 + r) * f + p0 + j] : 0.0;
    Al[r][j] = (gl0 + r < f && j < pb) ? Fs[(int64_t)(gl0 + r) * f + p0 + j] : 0.0;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, fr = lane >> 2, fc = lane & 3;
  double acc[2][4][2] = {};
  for (int ks = 0; ks < pb; ks += 4) {
    double a[2], b[4];
#pragma unroll
    for (int u = 0; u < 2; ++u) a[u] = Ai[wm * 16 + 8 * u + fr][ks + fc];
#pragma unroll
    for (int w = 0; w < 4; ++w) b[w] = Al[wn * 32 + 8 * w + fr][ks + fc];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int w = 0; w < 4; ++w) dmma884(acc[u][w][0], acc[u][w][1], a[u], b[w]);
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int gi = gi0 + wm * 16 + 8 * u + fr;
    if (gi >= f) continue;
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int gl = gl0 + wn * 32 + 8 * w + 2 * fc + q;
        if (gl <= gi) Fs[(int64_t)gi * f + gl] -= acc[u][w][q];
      }
  }
  __syncthreads();
}

__device__ __forceinline__ void tri_pair(int pr, int &ti, int &tl) {
  int t = (int)((sqrt(8.0 * pr + 1.0) - 1.0) * 0.5);
  while ((t + 1) * (t + 2) / 2 <= pr) ++t;
  while (t * (t + 1) / 2 > pr) --t;
  ti = t;
  tl = pr - t * (t + 1) / 2;
}

// One CTA per front of the level (many small fronts).
__global__ void __launch_bounds__(kThreads, 4)
    mf_factor_kernel(pf_mf_plan_t p, const double *__restrict__ off,
                     const double *__restrict__ diag, const int32_t *__restrict__ nodes,
                     double *F, int32_t *err) {
  __shared__ double D[kT][kT + 1];
  __shared__ double Ai[64][kSY];
  __shared__ double Al[64][kSY];
  const int s = nodes[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s];
  double *Fs = F + p.foff[s];
  front_assemble_rows(p, s, off, diag, F, 0, f);
  for (int p0 = 0; p0 < c; p0 += kT) {
    const int pb = min(kT, c - p0);
    panel_diag(Fs, f, p0, pb, D, err, true);
    panel_trsm_dmma(Fs, f, p0, pb, D, Ai, Al, 0, 1);
    __syncthreads();
    const int nb = (f - p0 - pb + 63) / 64;
    for (int pr = 0; pr < nb * (nb + 1) / 2; ++pr) {
      int ti, tl;
      tri_pair(pr, ti, tl);
      panel_syrk_tile(Fs, f, p0, pb, ti, tl, Ai, Al);
    }
  }
}

// Split path (few large fronts): grid (fronts, parts) per step.
__global__ void __launch_bounds__(kThreads)
    mf_assemble_split_kernel(pf_mf_plan_t p, const double *__restrict__ off,
                             const double *__restrict__ diag, const int32_t *__restrict__ nodes,
                             double *F) {
  const int s = nodes[blockIdx.x];
  const int f = p.fn[s];
  const int per = (f + gridDim.y - 1) / gridDim.y;
  const int r0 = min(f, (int)blockIdx.y * per), r1 = min(f, r0 + per);
  if (r0 >= r1) return;
  front_assemble_rows(p, s, off, diag, F, r0, r1);
}

__global__ void __launch_bounds__(kThreads, 4)
    mf_panel_trsm_kernel(pf_mf_plan_t p, const int32_t *__restrict__ nodes, int p0, double *F,
                         int32_t *err) {
  __shared__ double D[kT][kT + 1];
  __shared__ double Dinv[kT][kSY];
  __shared__ double Xs[64][kSY];
  const int s = nodes[blockIdx.x];
  const int c = p.cn[s], f = p.fn[s];
  if (p0 >= c) return;
  const int pb = min(kT, c - p0);
  double *Fs = F + p.foff[s];
  // the pivot block was factored by the previous launch (mf_panel_diag_kernel
  // for the first panel, the SYRK CTA owning tile (0, 0) after that): a CTA
  // of this grid factoring and writing it back would race the others' reads
  panel_diag(Fs, f, p0, pb, D, err, false);
  panel_trsm_dmma(Fs, f, p0, pb, D, Dinv, Xs, blockIdx.y, gridDim.y);
}

// First pivot block of each front on the split path (one warp per front).
__global__ void __launch_bounds__(32)
    mf_panel_diag_kernel(pf_mf_plan_t p, const int32_t *__restrict__ nodes, double *F,
                         int32_t *err) {
  __shared__ double D[kT][kT + 1];
  const int s = nodes[blockIdx.x];
  const int c = p.cn[s], f = p.fn[s];
  if (c <= 0) return;
  panel_diag(F + p.foff[s], f, 0, min(kT, c), D, err, true);
}

__global__ void __launch_bounds__(kThreads)
    mf_panel_syrk_kernel(pf_mf_plan_t p, const int32_t *__restrict__ nodes, int p0, double *F,
                         int32_t *err) {
  __shared__ double Ai[64][kSY];
  __shared__ double Al[64][kSY];
  __shared__ double D[kT][kT + 1];
  const int s = nodes[blockIdx.x];
  const int c = p.cn[s], f = p.fn[s];
  if (p0 >= c) return;
  const int pb = min(kT, c - p0);
  const int nb = (f - p0 - pb + 63) / 64;
  double *Fs = F + p.foff[s];
  for (int pr = blockIdx.y; pr < nb * (nb + 1) / 2; pr += gridDim.y) {
    int ti, tl;
    tri_pair(pr, ti, tl);
    panel_syrk_tile(Fs, f, p0, pb, ti, tl, Ai, Al);
  }
  // tile (0, 0), updated by this CTA alone, holds the next pivot block
  const int q0 = p0 + pb;
  if (blockIdx.y == 0 && q0 < c) panel_diag(Fs, f, q0, min(kT, c - q0), D, err, true);
}

// ------------------------------------------------- explicit inverses --
// Per front, Mt = [L_CC^{-1}; -L_RC L_CC^{-1}] (f x c, row stride ldc =
// round_up(c, 2)): the forward solve of the front against the identity.  A
// = -Lc_II is an M-matrix, so L_CC^{-1} >= 0 and -L_RC L_CC^{-1} >= 0: both
// solves below become sums of non-negative products (no cancellation, P keeps
// componentwise accuracy) and need no sequential triangular sweeps.
// One CTA per (node, 32 identity columns); rows above the tile stay zero.
__global__ void __launch_bounds__(kThreads)
    mf_inverse_kernel(pf_mf_plan_t p, const double *__restrict__ F,
                      const int32_t *__restrict__ item_node, const int32_t *__restrict__ item_ct,
                      double *Mt) {
  __shared__ double D[kT][kT + 1];
  __shared__ double Y[kT][kT + 1];
  __shared__ double Ls[64][kSY];   // stride 4 mod 16: conflict-free DMMA fragments
  __shared__ double Yb[kT][kSY];
  const int s = item_node[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s];
  const int ldc = (c + 15) & ~15;
  const int c0 = item_ct[blockIdx.x] * kT;
  const int w = min(kT, c - c0);
  const double *Fs = F + p.foff[s];
  double *W = Mt + p.mt_off[s] + c0;
  const int tid = threadIdx.x, t = tid % kT, g = tid / kT;
  for (int i = g; i < f; i += kThreads / kT)
    if (t < w) W[(int64_t)i * ldc + t] = (i == c0 + t) ? 1.0 : 0.0;
  __syncthreads();
  for (int jb = c0; jb < c; jb += kT) {
    const int nb = min(kT, c - jb);
    for (int idx = tid; idx < kT * kT; idx += kThreads) {
      const int i = idx / kT, j = idx % kT;
      D[i][j] = (i < nb && j <= i) ? Fs[(int64_t)(jb + i) * f + jb + j] : 0.0;
      Y[i][j] = (i < nb && j < w) ? W[(int64_t)(jb + i) * ldc + j] : 0.0;
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
      if (t < w) W[(int64_t)(jb + i) * ldc + t] = Y[i][t];
    // rows below the block: W[i] -= L[i, jb:jb+nb] Y, 64 rows at a time on the
    // FP64 tensor pipe (8 warps as 4 (rows) x 2 (columns), 16 x 16 warp tiles)
    for (int i0 = jb + nb; i0 < f; i0 += 64) {
      for (int idx = tid; idx < 64 * kT; idx += kThreads) {
        const int r = idx / kT, j = idx % kT;
        Ls[r][j] = (i0 + r < f && j < nb) ? Fs[(int64_t)(i0 + r) * f + jb + j] : 0.0;
      }
      for (int idx = tid; idx < kT * kT; idx += kThreads) {
        const int l = idx / kT, j = idx % kT;
        Yb[l][j] = Y[l][j];
      }
      __syncthreads();
      const int lane = tid & 31, warp = tid >> 5;
      const int wm = warp >> 1, wn = warp & 1, fr = lane >> 2, fc = lane & 3;
      double acc[2][2][2] = {};
      for (int ks = 0; ks < nb; ks += 4) {
        double a[2], b[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) a[u] = Ls[wm * 16 + 8 * u + fr][ks + fc];
#pragma unroll
        for (int v = 0; v < 2; ++v) b[v] = Yb[ks + fc][wn * 16 + 8 * v + fr];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) dmma884(acc[u][v][0], acc[u][v][1], a[u], b[v]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = i0 + wm * 16 + 8 * u + fr;
        if (i >= f) continue;
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int col = wn * 16 + 8 * v + 2 * fc + q;
            if (col < w) W[(int64_t)i * ldc + col] -= acc[u][v][q];
          }
      }
      __syncthreads();
    }
  }
}

// M = Mt^T (c x f, row stride ldf = round_up(f, 2)), one CTA per node.
__global__ void __launch_bounds__(kThreads)
    mf_transpose_kernel(pf_mf_plan_t p, const int32_t *__restrict__ nodes,
                        const double *__restrict__ Mt, double *M) {
  __shared__ double tile[32][33];
  const int s = nodes[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s];
  const int ldc = (c + 15) & ~15, ldf = (f + 15) & ~15;
  const double *A = Mt + p.mt_off[s];
  double *B = M + p.m_off[s];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  for (int l0 = 0; l0 < f; l0 += 32)
    for (int i0 = 0; i0 < c; i0 += 32) {
      for (int r = ty; r < 32; r += kThreads / 32)
        tile[r][tx] = (l0 + r < f && i0 + tx < c) ? A[(int64_t)(l0 + r) * ldc + i0 + tx] : 0.0;
      __syncthreads();
      for (int r = ty; r < 32; r += kThreads / 32)
        if (i0 + r < c && l0 + tx < f) B[(int64_t)(i0 + r) * ldf + l0 + tx] = tile[tx][r];
      __syncthreads();
    }
}

// ---------------------------------------------- gathered GEMM (DMMA) --
// acc(32 x 64) = A (32 rows, K contiguous per row) x B (K rows of 64 columns),
// A rows / B rows fetched through accessors (nullptr = zero row): 4 warps as
// 2 (m) x 2 (n), warp tile 16 x 32 of m8n8k4 FP64 MMAs (SASS DMMA), 16-deep
// K chunks through a 3-stage cp.async ring.  Column blocks are flattened into
// the K loop, so the ring never drains between them.
constexpr int kGT = 128, kGBM = 32, kGBN = 64, kGBK = 16, kGStages = 3;
// row strides: every half-warp fragment load hits 16 distinct bank pairs
constexpr int kSA = kGBK + 4, kSB = kGBN + 4;
constexpr int kStageA = kGBM * kSA, kStageB = kGBK * kSB;
constexpr int kGemmSmem = kGStages * (kStageA + kStageB) * 8;  // bytes of the ring

// zero-initialised source of "zero rows": one 16-byte chunk per lane (a
// single shared source address serialises cp.async across the warp)
__device__ __align__(128) double g_zero[kGBN];

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ncb column blocks x K; arow(i) / brow(cb, l) return row pointers (or
// nullptr); epi(cb, i, t, v) consumes each finished column block.
// As / Bs: kGStages x kStageA / kStageB doubles of shared memory.
template <class ARow, class BRow, class Epi>
__device__ __forceinline__ void gathered_gemm(double *As_, double *Bs_, int ma, int K, int ncb,
                                              ARow arow, BRow brow, Epi epi) {
  double(*As)[kStageA] = reinterpret_cast<double(*)[kStageA]>(As_);
  double(*Bs)[kStageB] = reinterpret_cast<double(*)[kStageB]>(Bs_);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, fr = lane >> 2, fc = lane & 3;
  const int nkt = (K + kGBK - 1) / kGBK;
  const int total = nkt * ncb;
  auto issue = [&](int it) {
    if (it < total) {
      const int st = it % kGStages, cb = it / nkt, k0 = (it % nkt) * kGBK;
      double *as = As[st], *bs = Bs[st];
#pragma unroll
      for (int u = 0; u < 2; ++u) {  // A: 32 rows x 8 chunks of 16 B
        const int e = tid + kGT * u, r = e >> 3, ch = e & 7;
        const double *src = r < ma ? arow(r) : nullptr;
        const bool ok = src != nullptr && k0 + 2 * ch < K;  // row pads are zero
        cp_async16(as + r * kSA + 2 * ch, ok ? src + k0 + 2 * ch : g_zero + 2 * ch);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // B: 16 rows x 32 chunks
        const int e = tid + kGT * u, r = e >> 5, ch = e & 31;
        const double *src = (k0 + r < K) ? brow(cb, k0 + r) : nullptr;
        cp_async16(bs + r * kSB + 2 * ch, (src ? src : g_zero) + 2 * ch);
      }
    }
    cp_commit();
  };
  double acc[2][4][2];
#pragma unroll
  for (int s = 0; s < kGStages - 1; ++s) issue(s);
  for (int it = 0; it < total; ++it) {
    if (it % nkt == 0) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    cp_wait<kGStages - 2>();
    __syncthreads();
    issue(it + kGStages - 1);
    const int st = it % kGStages;
    const double *as = As[st] + (wm * 16 + fr) * kSA + fc;
    const double *bs = Bs[st] + fc * kSB + wn * 32 + fr;
#pragma unroll
    for (int ks = 0; ks < kGBK; ks += 4) {
      double a[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = as[8 * i * kSA + ks];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[ks * kSB + 8 * j];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (it % nkt == nkt - 1) {
      const int cb = it / nkt;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q)
            epi(cb, wm * 16 + 8 * i + fr, wn * 32 + 8 * j + 2 * fc + q, acc[i][j][q]);
    }
  }
  cp_wait<0>();
}

// ------------------------------------------------------- forward solve --
// Level items (node, active 64-column tile).  Assemble W = [B_C; 0] + the
// children's V blocks (child order, one child at a time) into Wb ...
__global__ void __launch_bounds__(kThreads)
    mf_fwd_assemble_kernel(pf_mf_plan_t p, const double *__restrict__ off,
                           const int32_t *__restrict__ item_node,
                           const int64_t *__restrict__ item_id,
                           const int64_t *__restrict__ item_woff, const double *__restrict__ O,
                           double *Wb) {
  const int s = item_node[blockIdx.x];
  const int64_t it = item_id[blockIdx.x];
  const int f = p.fn[s];
  const int tile = p.act_tile[it];
  const int64_t j0 = (int64_t)tile * kGBN;
  double *W = Wb + item_woff[blockIdx.x];
  const int tid = threadIdx.x;
  for (int64_t e = tid; e < (int64_t)f * kGBN; e += kThreads) W[e] = 0.0;
  __syncthreads();
  for (int64_t e = p.b_ptr[s] + tid; e < p.b_ptr[s + 1]; e += kThreads) {
    const int64_t col = p.b_col[e] - j0;
    if (col >= 0 && col < kGBN) W[(int64_t)p.b_row[e] * kGBN + col] = off[p.b_src[e]];
  }
  __syncthreads();
  const int t = tid % kGBN, g = tid / kGBN;
  for (int q = p.ch_ptr[s]; q < p.ch_ptr[s + 1]; ++q) {
    const int ch = p.ch_idx[q];
    const int64_t ic = p.tile_item[(int64_t)ch * p.ntiles + tile];
    if (ic < 0) continue;
    const int rc = p.rn[ch], cc = p.cn[ch];
    const double *Vc = O + p.act_voff[ic] + (int64_t)cc * kGBN;
    const int32_t *mp = p.relmap + p.relmap_off[ch];
    for (int a = g; a < rc; a += kThreads / kGBN)
      W[(int64_t)mp[a] * kGBN + t] += Vc[(int64_t)a * kGBN + t];
    __syncthreads();
  }
}

// ... then O = Mt W_C + [0; W_R] (rows < c: Y_C = L_CC^{-1} W_C; rows >= c:
// V = W_R - L_RC Y_C), items (node, tile, 32-row block of the front).
__global__ void __launch_bounds__(kGT)
    mf_fwd_gemm_kernel(pf_mf_plan_t p, const double *__restrict__ Mt,
                       const int32_t *__restrict__ item_node, const int64_t *__restrict__ item_id,
                       const int64_t *__restrict__ item_woff, const int32_t *__restrict__ item_rb,
                       const double *__restrict__ Wb, double *O) {
  const int s = item_node[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s];
  const int ldc = (c + 15) & ~15;
  const int i0 = item_rb[blockIdx.x] * kGBM;
  const double *W = Wb + item_woff[blockIdx.x];
  double *Ob = O + p.act_voff[item_id[blockIdx.x]];
  const double *A = Mt + p.mt_off[s];
  __shared__ __align__(128) double ring[kGemmSmem / 8];
  gathered_gemm(
      ring, ring + kGStages * kStageA, min(kGBM, f - i0), c, 1, [&](int r) { return A + (int64_t)(i0 + r) * ldc; },
      [&](int, int l) { return W + (int64_t)l * kGBN; },
      [&](int, int r, int t, double v) {
        const int i = i0 + r;
        if (i < f) Ob[(int64_t)i * kGBN + t] = v + (i >= c ? W[(int64_t)i * kGBN + t] : 0.0);
      });
}

// ------------------------------------------------------ backward solve --
// Levels top-down; items (node, 32-row block of C, column blocks [cb0, cb1)):
//   X_C = M [Y_C; X_R],  M = Mt^T = [L_CC^{-T} | -L_CC^{-T} L_RC^T]
// Y_C from the forward blocks (zero where the tile was never reached), X_R
// gathered from P's rows (final: ancestors ran earlier), X_C into P.
// Output tile per CTA: 128 P columns (M dimension of the MMA) x NB rows of C
// (N dimension, NB in {8, 16, 32, 64} chosen per level from its separator
// sizes, so a 12-vertex separator pads to 16, not 64):
//   X_C^T (cols x NB) = Z^T (cols x f) . M^T (f x NB),  Z = [Y_C; X_R].
// Warp-specialised: one producer warp streams 16-deep K stages with TMA bulk
// copies (cp.async.bulk, one per gathered Z row of 128 doubles and per M row
// of 16) into a 3-stage ring guarded by full/empty mbarriers; 8 consumer
// warps each own 16 columns x NB (2 x NB/8 m8n8k4 DMMAs per 4-deep k step).
// Gather offsets are resolved in shared memory before the loop; column blocks
// whose tiles the forward never reached skip the zero Y rows of K.
constexpr int kBN = 128, kBT = 256, kBW = kBT / 32;  // consumer threads / warps
constexpr int kSB2 = kBN + 4;  // 4 mod 16: conflict-free half-warp fragment loads
constexpr int kZStage = kGBK * kSB2;
template <int NB>
constexpr int m_stage() { return kGBK * (NB + 4); }  // 16 k-rows of Mt, NB + 4 stride
template <int NB>
constexpr int bwd_ring_bytes() {
  return kGStages * (kZStage + m_stage<NB>()) * 8 + 2 * kGStages * 8;  // + mbarriers
}
__device__ __align__(128) double g_zero_row[kBN];  // zero source of 1 KB bulk copies

template <int NB>
__global__ void __launch_bounds__(kBT + 32, 2)
    mf_bwd_gemm_kernel(pf_mf_plan_t p, const double *__restrict__ M,
                       const double *__restrict__ O, const int32_t *__restrict__ item_node,
                       const int32_t *__restrict__ item_rb, const int32_t *__restrict__ item_cb0,
                       const int32_t *__restrict__ item_cb1, double *P, int64_t ldp) {
  constexpr int kMS = m_stage<NB>();
  constexpr uint32_t kStageBytes = (kGBK * kBN + NB * kGBK) * 8;
  // dynamic smem: [Z ring | M ring | full[S] | empty[S] | coff[NB] | ysrc[2 ncb] |
  //                kt0[ncb] | roff[f]]
  extern __shared__ __align__(128) double dyn[];
  double *Zs = dyn, *Ms = dyn + kGStages * kZStage;
  uint64_t *full = reinterpret_cast<uint64_t *>(Ms + kGStages * kMS);
  uint64_t *empty = full + kGStages;
  int64_t *coff = reinterpret_cast<int64_t *>(empty + kGStages);
  const double **ysrc = reinterpret_cast<const double **>(coff + NB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = kBT + 32;
  const int s = item_node[blockIdx.x];
  const int f = p.fn[s], c = p.cn[s];
  const int i0 = item_rb[blockIdx.x] * NB;
  const int cb0 = item_cb0[blockIdx.x], ncb = item_cb1[blockIdx.x] - cb0;
  int64_t *kt0 = reinterpret_cast<int64_t *>(ysrc + 2 * ncb);
  int64_t *roff = kt0 + ncb;
  {
    const int32_t *Cv = p.perm_orig + p.c0[s];
    const int32_t *Rv = p.r_orig + p.r_ptr[s];
    const int64_t *ti = p.tile_item + (int64_t)s * p.ntiles;
    // roff[l]: l < c -> Y row l of a 64-wide block; else the P row of X_R[l - c]
    for (int l = tid; l < f; l += nthr)
      roff[l] = l < c ? (int64_t)l * kGBN : row_off(p, Rv[l - c], ldp);
    for (int h = tid; h < 2 * ncb; h += nthr) {
      const int64_t tile = 2 * (int64_t)cb0 + h;
      const int64_t it = tile < p.ntiles ? ti[tile] : -1;
      ysrc[h] = it < 0 ? nullptr : O + p.act_voff[it];
    }
    for (int r = tid; r < NB; r += nthr) coff[r] = i0 + r < c ? row_off(p, Cv[i0 + r], ldp) : -1;
    if (tid == 0)
      for (int q = 0; q < kGStages; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], kBW);
      }
  }
  __syncthreads();
  // Mt's top block L_CC^{-1} is lower triangular: rows l < i0 are zero in
  // this CTA's columns, so K starts at i0's tile (or past Y_C when the
  // forward never reached these columns)
  for (int cb = tid; cb < ncb; cb += nthr)
    kt0[cb] = (ysrc[2 * cb] || ysrc[2 * cb + 1]) ? i0 / kGBK : c / kGBK;
  __syncthreads();
  const int nkt = (f + kGBK - 1) / kGBK;
  if (warp == kBW) {  // ------------------------------------------- producer
    // B operand straight from Mt (f x ldc): a K stage is 16 rows of Mt, each
    // the NB contiguous entries of this C-row block — the k-major layout the
    // DMMA B fragment wants (no transpose, one bulk copy per k-row)
    const int ldc = (c + 15) & ~15;
    const double *A = M + p.mt_off[s] + i0;
    const int mb = min(NB, ldc - i0);  // real columns in this row (pads are zero)
    int it = 0;
    for (int cb = 0; cb < ncb; ++cb) {
      const int64_t col = (int64_t)(cb0 + cb) * kBN;
      const bool whole = col + kBN <= ldp;  // else the upper half lies past the row end
      const double *yb0 = ysrc[2 * cb], *yb1 = ysrc[2 * cb + 1];
      for (int kt = (int)kt0[cb]; kt < nkt; ++kt, ++it) {
        const int st = it % kGStages;
        mbar_wait(&empty[st], ((it / kGStages) & 1) ^ 1);
        if (lane == 0) mbar_expect_tx(&full[st], kStageBytes);
        __syncwarp();
        const int k0 = kt * kGBK;
        if (lane < kGBK) {
          const int l = k0 + lane;
          double *dst = Zs + st * kZStage + lane * kSB2;
          if (l >= f) {
            bulk_g2s(dst, g_zero_row, kBN * 8, &full[st]);
          } else if (l < c) {
            bulk_g2s(dst, yb0 ? yb0 + roff[l] : g_zero_row, kGBN * 8, &full[st]);
            bulk_g2s(dst + kGBN, yb1 ? yb1 + roff[l] : g_zero_row, kGBN * 8, &full[st]);
          } else if (whole) {
            bulk_g2s(dst, P + roff[l] + col, kBN * 8, &full[st]);
          } else {
            bulk_g2s(dst, P + roff[l] + col, kGBN * 8, &full[st]);
            bulk_g2s(dst + kGBN, g_zero_row, kGBN * 8, &full[st]);
          }
        }
        if (lane < kGBK) {
          const int l = k0 + lane;
          double *dst = Ms + st * kMS + lane * (NB + 4);
          if (l < f) {
            bulk_g2s(dst, A + (int64_t)l * ldc, mb * 8, &full[st]);
            if (mb < NB) bulk_g2s(dst + mb, g_zero_row, (NB - mb) * 8, &full[st]);
          } else {
            bulk_g2s(dst, g_zero_row, NB * 8, &full[st]);
          }
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers
  const int fr = lane >> 2, fc = lane & 3;
  constexpr int NJ = NB / 8;
  const int njv = (min(NB, c - i0) + 7) >> 3;  // n-tiles holding real C rows (uniform)
  const int64_t k = p.k;
  int it = 0;
  for (int cb = 0; cb < ncb; ++cb) {
    double acc[2][NJ][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = (int)kt0[cb]; kt < nkt; ++kt, ++it) {
      const int st = it % kGStages;
      mbar_wait(&full[st], (it / kGStages) & 1);
      const double *zs = Zs + st * kZStage + fc * kSB2 + warp * 16 + fr;
      const double *ms = Ms + st * kMS + fc * (NB + 4) + fr;
      const int k0 = kt * kGBK;
#pragma unroll
      for (int ks = 0; ks < kGBK; ks += 4) {
        double av[2], bv[NJ];
#pragma unroll
        for (int i = 0; i < 2; ++i) av[i] = zs[ks * kSB2 + 8 * i];
#pragma unroll
        for (int j = 0; j < NJ; ++j) bv[j] = ms[ks * (NB + 4) + 8 * j];
        // n-tile j is all zero in L_CC^{-1} while its first column i0 + 8j
        // exceeds the step's last row (exact zeros: skipping is bitwise free)
        const int lmax = k0 + ks + 3 < c ? k0 + ks + 3 - i0 : NB;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          if (j < njv && 8 * j <= lmax) {
#pragma unroll
            for (int i = 0; i < 2; ++i) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    const int64_t colb = (int64_t)(cb0 + cb) * kBN + warp * 16 + fr;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t ro = coff[8 * j + 2 * fc + q];
        if (ro < 0) continue;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int64_t col = colb + 8 * i;
          if (col < k) P[ro + col] = acc[i][j][q];
        }
      }
  }
}

// ------------------------------------------------------- diagnostics ------
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long *p, double v) {
  // non-negative doubles order like their bit patterns; NaN propagates as max
  atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

// max_j |diag[v] P[v,j] + sum_e off[e] P[u_e, j]| over the interior rows v =
// order[i] (the nested-dissection order: consecutive rows are spatially
// compact leaf patches, so the rows their neighbours read are shared by the
// warps of the same CTA and stay in L1/L2), with nrow[e] the precomputed P
// offset of neighbour entry e (or -1 - its boundary column, contributing
// off[e] to that column).  Grid: x = row groups (a warp per row), y =
// 512-column chunks; columns go in 16-byte pairs.
constexpr int kResCols = 512;

// Per (row, column chunk): the warp's partial row sum (lane partials, then
// the butterfly sum: deterministic) into row_part[row * chunks + chunk], and
// the negative-entry flag into out[2].
__device__ __forceinline__ void residual_row_done(double *row_part, int64_t row,
                                                  unsigned chunks, double rs, bool neg,
                                                  unsigned long long *out) {
  if (!row_part) return;
  rs = warp_sum(rs);
  const bool any = __any_sync(0xffffffffu, neg);
  if ((threadIdx.x & 31) == 0) {
    row_part[row * chunks + blockIdx.y] = rs;
    if (any) atomicOr(out + 2, 1ull);
  }
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1024 / (WARPS * 32))
    residual_kernel(const double *__restrict__ P, int64_t ldp, int64_t k,
                    const int32_t *__restrict__ order, int64_t count,
                    const int64_t *__restrict__ rowoff,
                    const int64_t *__restrict__ nb_ptr, const int64_t *__restrict__ nrow,
                    const double *__restrict__ off, const double *__restrict__ diag,
                    double *__restrict__ row_part, unsigned long long *out) {
  // Neighbour rows are gathered in unrolled groups of 8 (all loads in flight
  // before the FMAs; missing slots point at row v with weight 0); boundary
  // neighbours add their weight to one column each, in a separate short list.
  constexpr int kG = 8, kMaxDeg = 32;
  __shared__ int64_t srow[WARPS][kMaxDeg];
  __shared__ double sw[WARPS][kMaxDeg];
  __shared__ int64_t bcl[WARPS][kMaxDeg];
  __shared__ double bw[WARPS][kMaxDeg];
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const int64_t j0 = (int64_t)blockIdx.y * kResCols, j1 = min(k, j0 + kResCols);
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  double mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + w; i < count; i += warps) {
    const int64_t v = order[i];
    const int64_t vo = rowoff ? rowoff[v] : v * ldp;  // this row's offset in P
    const int64_t e0 = nb_ptr[v];
    const int deg = (int)(nb_ptr[v + 1] - e0);
    const double dv = diag[v];
    // optional finalize work on the row's own entries (already loaded): the
    // chunk's partial row sum and whether any entry is negative (the clip)
    double rs = 0.0;
    bool neg = false;
    if (deg > kMaxDeg) {  // exact per-column evaluation for a (rare) high-valence row
      for (int64_t j = j0 + lane; j < j1; j += 32) {
        const double pj = P[vo + j];
        rs += pj;
        neg |= pj < 0.0;
        double acc = dv * pj;
        for (int64_t e = e0; e < e0 + deg; ++e) {
          const int64_t ro = nrow[e];
          acc += off[e] * (ro >= 0 ? P[ro + j] : (-1 - ro == j ? 1.0 : 0.0));
        }
        mx = fmax(mx, fabs(acc));
      }
      residual_row_done(row_part, vo / ldp, gridDim.y, rs, neg, out);
      continue;
    }
    __syncwarp();
    const int64_t me = lane < deg ? nrow[e0 + lane] : 0;
    const double mw = lane < deg ? off[e0 + lane] : 0.0;
    const bool inner = lane < deg && me >= 0;
    const unsigned bmask = __ballot_sync(0xffffffffu, lane < deg && me < 0);
    const int nbnd = __popc(bmask);
    srow[w][lane] = inner ? me : vo;  // all 32 slots: padding reads row v, weight 0
    sw[w][lane] = inner ? mw : 0.0;
    if (lane < deg && me < 0) {
      const int slot = __popc(bmask & ((1u << lane) - 1));
      bcl[w][slot] = -1 - me;
      bw[w][slot] = mw;
    }
    __syncwarp();
    if (deg <= kG) {
      // the common valence: the 8 slots live in registers for the whole
      // column chunk (re-reading them from shared memory per step cost a
      // third of the L1 data-pipe wavefronts), fetched once by shuffle
      int32_t ro[kG];  // row indices (every P row offset is a multiple of ldp)
      double wr[kG];
      const int32_t mr = (int32_t)((inner ? me : vo) / ldp);
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        ro[u] = __shfl_sync(0xffffffffu, mr, u);
        wr[u] = __shfl_sync(0xffffffffu, inner ? mw : 0.0, u);
      }
      for (int64_t j = j0 + 2 * lane; j < j1; j += 64) {
        const double2 pv = *reinterpret_cast<const double2 *>(P + vo + j);
        double2 x[kG];
#pragma unroll
        for (int u = 0; u < kG; ++u)
          x[u] = *reinterpret_cast<const double2 *>(P + (int64_t)ro[u] * ldp + j);
        double a0 = dv * pv.x, a1 = dv * pv.y;
#pragma unroll
        for (int u = 0; u < kG; ++u) {
          a0 += wr[u] * x[u].x;
          a1 += wr[u] * x[u].y;
        }
        for (int q = 0; q < nbnd; ++q) {
          const int64_t b = bcl[w][q];
          if (b == j) a0 += bw[w][q];
          if (b == j + 1) a1 += bw[w][q];
        }
        // row-sum work after the loads are in flight (the odd tail's partner
        // is a pad column)
        const bool two = j + 1 < k;
        rs += two ? pv.x + pv.y : pv.x;
        neg |= pv.x < 0.0 || (two && pv.y < 0.0);
        mx = fmax(mx, fabs(a0));
        if (two) mx = fmax(mx, fabs(a1));
      }
      residual_row_done(row_part, vo / ldp, gridDim.y, rs, neg, out);
      continue;
    }
    const int ngroups = (deg + kG - 1) / kG;
    for (int64_t j = j0 + 2 * lane; j < j1; j += 64) {
      const double2 pv = *reinterpret_cast<const double2 *>(P + vo + j);
      double a0 = dv * pv.x, a1 = dv * pv.y;
      for (int g = 0; g < ngroups; ++g) {
        double2 x[kG];
#pragma unroll
        for (int u = 0; u < kG; ++u)
          x[u] = *reinterpret_cast<const double2 *>(P + srow[w][g * kG + u] + j);
#pragma unroll
        for (int u = 0; u < kG; ++u) {
          const double we = sw[w][g * kG + u];
          a0 += we * x[u].x;
          a1 += we * x[u].y;
        }
      }
      for (int q = 0; q < nbnd; ++q) {
        const int64_t b = bcl[w][q];
        if (b == j) a0 += bw[w][q];
        if (b == j + 1) a1 += bw[w][q];
      }
      const bool two = j + 1 < k;
      rs += two ? pv.x + pv.y : pv.x;
      neg |= pv.x < 0.0 || (two && pv.y < 0.0);
      mx = fmax(mx, fabs(a0));
      if (two) mx = fmax(mx, fabs(a1));
    }
    residual_row_done(row_part, vo / ldp, gridDim.y, rs, neg, out);
  }
  mx = warp_max(mx);
  if (lane == 0) atomic_max_nonneg(out, mx);
}

// nrow[e] = nb_idx[e] * ldp for an interior neighbour, -1 - bcol for a
// boundary one (the residual's gather table, built once per mesh).
__global__ void residual_table_kernel(const int32_t *__restrict__ nb_idx, int64_t nnz,
                                      const uint8_t *__restrict__ isb,
                                      const int32_t *__restrict__ bcol, int64_t ldp,
                                      const int64_t *__restrict__ rowoff,
                                      int64_t *__restrict__ nrow) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = nb_idx[e];
    nrow[e] = isb[u] ? -1 - (int64_t)bcol[u] : (rowoff ? rowoff[u] : (int64_t)u * ldp);
  }
}

// Boundary rows -> indicators, pad columns -> 0, the reference's clip of
// (-1e-12, 0) on interior entries, max |row sum - 1|, and (fused K1) the
// per-row negentropy H[r] = sum_b c(P) log c(P), c = max(., clamp) with
// pf_row_negentropy_f64's exact lane order (pairs per lane, x / y
// accumulators, odd tail on lane 0), plus min(P) over columns < k — so the
// first KL field on a freshly built P does not stream it once more for K1.
__global__ void finalize_kernel(double *P, int64_t ldp, int64_t row0, int64_t n, int64_t k,
                                const uint8_t *__restrict__ isb, const int32_t *__restrict__ bcol,
                                double clamp, double *__restrict__ H, double *min_out,
                                unsigned long long *out) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t npair = k >> 1;
  double mx = 0.0, mn = INFINITY;
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; v < n;
       v += warps) {
    double *row = P + v * ldp;  // slab-local row v = global row row0 + v
    const bool bnd = isb[row0 + v];
    if (bnd) {
      const int32_t b = bcol[row0 + v];
      for (int64_t j = lane; j < ldp; j += 32) row[j] = (j == b) ? 1.0 : 0.0;
      __syncwarp();
    }
    double s0 = 0.0, s1 = 0.0, a0 = 0.0, a1 = 0.0;
    for (int64_t j = lane; j < npair; j += 32) {
      double2 x = reinterpret_cast<double2 *>(row)[j];
      if (!bnd) {
        const bool cx = x.x > -1e-12 && x.x < 0.0, cy = x.y > -1e-12 && x.y < 0.0;
        if (cx) x.x = 0.0;  // solvers.py:293-295
        if (cy) x.y = 0.0;
        if (cx || cy) reinterpret_cast<double2 *>(row)[j] = x;
      }
      s0 += x.x;
      s1 += x.y;
      if (H) {  // fused K1 (FP64 log per entry: only when the caller wants H)
        mn = fmin(mn, fmin(x.x, x.y));
        const double q0 = fmax(x.x, clamp), q1 = fmax(x.y, clamp);
        a0 += __dmul_rn(q0, log(q0));
        a1 += __dmul_rn(q1, log(q1));
      }
    }
    if ((k & 1) && lane == 0) {
      double x = row[k - 1];
      if (!bnd && x > -1e-12 && x < 0.0) {
        x = 0.0;
        row[k - 1] = 0.0;
      }
      s0 += x;
      if (H) {
        mn = fmin(mn, x);
        const double q = fmax(x, clamp);
        a0 += __dmul_rn(q, log(q));
      }
    }
    if (!bnd)
      for (int64_t j = k + lane; j < ldp; j += 32) row[j] = 0.0;
    if (H) {
      const double h = warp_sum(a0 + a1);
      if (lane == 0) H[v] = h;
    }
    const double sum = warp_sum(s0 + s1);
    if (!bnd) mx = fmax(mx, fabs(sum - 1.0));  // boundary rows sum to exactly 1
  }
  if (lane == 0) atomic_max_nonneg(out, mx);
  if (H && min_out) {
    mn = warp_min(mn);
    if (lane == 0 && mn < INFINITY) {  // ordered-integer atomic min (values may be < 0)
      unsigned long long *addr = reinterpret_cast<unsigned long long *>(min_out);
      unsigned long long old = *addr, assumed;
      do {
        assumed = old;
        if (__longlong_as_double(assumed) <= mn) break;
        old = atomicCAS(addr, assumed, __double_as_longlong(mn));
      } while (old != assumed);
    }
  }
}

// Finalize without a second pass over P (after residual_kernel filled
// row_part): boundary rows -> indicators, pad columns -> 0, max |row sum - 1|
// with each interior row's sum taken over its chunk partials in chunk order.
// (The clip of (-1e-12, 0) cannot apply: the caller runs finalize_kernel when
// the residual pass flagged a negative entry.)
__global__ void finalize_rows_kernel(double *P, int64_t ldp, int64_t row0, int64_t n, int64_t k,
                                     const uint8_t *__restrict__ isb,
                                     const int32_t *__restrict__ bcol,
                                     const double *__restrict__ row_part, int chunks,
                                     unsigned long long *out) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  double mx = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; v < n;
       v += warps) {
    double *row = P + v * ldp;
    if (isb[row0 + v]) {
      const int32_t b = bcol[row0 + v];
      for (int64_t j = lane; j < ldp; j += 32) row[j] = (j == b) ? 1.0 : 0.0;
      continue;  // sums to exactly 1
    }
    for (int64_t j = k + lane; j < ldp; j += 32) row[j] = 0.0;
    if (lane == 0) {
      double sum = 0.0;
      for (int c = 0; c < chunks; ++c) sum += row_part[v * chunks + c];
      mx = fmax(mx, fabs(sum - 1.0));
    }
  }
  mx = warp_max(mx);
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
                       const int32_t *nodes, int64_t count, int32_t max_f, int32_t max_c,
                       int split, double *F, int32_t *err, pf_stream_t stream) {
  if (!plan || !off || !diag || !nodes || !F || !err || count < 0 || max_f < 0 || max_c < 0)
    return fail(PF_E_ARG, "pf_mf_factor_level: bad argument");
  if (count == 0) return 0;
  cudaStream_t st = as_stream(stream);
  if (!split) {
    mf_factor_kernel<<<(unsigned)count, kThreads, 0, st>>>(*plan, off, diag, nodes, F, err);
    return check_launch("pf_mf_factor_level");
  }
  // few large fronts: spread every step of each front over ~2 waves of CTAs
  const int target = 8 * sm_count();
  const int per = (int)std::max<int64_t>(1, (target + count - 1) / count);
  mf_assemble_split_kernel<<<dim3((unsigned)count, (unsigned)std::min(per, std::max(1, max_f / 16))),
                             kThreads, 0, st>>>(*plan, off, diag, nodes, F);
  mf_panel_diag_kernel<<<(unsigned)count, 32, 0, st>>>(*plan, nodes, F, err);
  for (int p0 = 0; p0 < max_c; p0 += kT) {
    const int rows = max_f - p0;
    const int ty = std::max(1, std::min(per, (rows + 63) / 64));  // 64-row DMMA chunks
    mf_panel_trsm_kernel<<<dim3((unsigned)count, (unsigned)ty), kThreads, 0, st>>>(*plan, nodes,
                                                                                  p0, F, err);
    const int nb = (rows - 1 + 63) / 64;
    const int pairs = std::max(1, nb * (nb + 1) / 2);
    mf_panel_syrk_kernel<<<dim3((unsigned)count, (unsigned)std::min(pairs, std::max(per, 1))),
                           kThreads, 0, st>>>(*plan, nodes, p0, F, err);
  }
  return check_launch("pf_mf_factor_level");
}

int pf_mf_inverse(const pf_mf_plan_t *plan, const double *F, const int32_t *item_node,
                  const int32_t *item_ct, int64_t count, const int32_t *nodes, int64_t nnodes,
                  double *Mt, double *M, pf_stream_t stream) {
  if (count == 0 && nnodes == 0) return 0;  // no interior vertices: nothing to invert
  if (!plan || !F || (count && (!item_node || !item_ct)) || (nnodes && M && !nodes) || !Mt ||
      count < 0 || nnodes < 0 || plan->tile != kGBN)
    return fail(PF_E_ARG, "pf_mf_inverse: bad argument");
  cudaStream_t st = as_stream(stream);
  if (count > 0)
    mf_inverse_kernel<<<(unsigned)count, kThreads, 0, st>>>(*plan, F, item_node, item_ct, Mt);
  if (nnodes > 0 && M)  // M = Mt^T only on request (the solves read Mt)
    mf_transpose_kernel<<<(unsigned)nnodes, kThreads, 0, st>>>(*plan, nodes, Mt, M);
  return check_launch("pf_mf_inverse");
}

int pf_mf_forward_level(const pf_mf_plan_t *plan, const double *Mt, const double *off,
                        const int32_t *asm_node, const int64_t *asm_item, const int64_t *asm_woff,
                        int64_t n_asm, const int32_t *g_node, const int64_t *g_item,
                        const int64_t *g_woff, const int32_t *g_rb, int64_t n_gemm, double *Wb,
                        double *O, pf_stream_t stream) {
  if (!plan || !Mt || !off || !Wb || !O || n_asm < 0 || n_gemm < 0 || plan->tile != kGBN ||
      (n_asm && (!asm_node || !asm_item || !asm_woff)) ||
      (n_gemm && (!g_node || !g_item || !g_woff || !g_rb)))
    return fail(PF_E_ARG, "pf_mf_forward_level: bad argument");
  cudaStream_t st = as_stream(stream);
  if (n_asm > 0)
    mf_fwd_assemble_kernel<<<(unsigned)n_asm, kThreads, 0, st>>>(*plan, off, asm_node, asm_item,
                                                                 asm_woff, O, Wb);
  if (n_gemm > 0)
    mf_fwd_gemm_kernel<<<(unsigned)n_gemm, kGT, 0, st>>>(*plan, Mt, g_node, g_item, g_woff, g_rb,
                                                         Wb, O);
  return check_launch("pf_mf_forward_level");
}

int pf_mf_backward_level(const pf_mf_plan_t *plan, const double *M, const double *O,
                         const int32_t *item_node, const int32_t *item_rb,
                         const int32_t *item_cb0, const int32_t *item_cb1, int64_t count,
                         int32_t max_f, int32_t max_ncb, int32_t nb_rows, double *P,
                         int64_t ldp, pf_stream_t stream) {
  if (!plan || !M || !O || !item_node || !item_rb || !item_cb0 || !item_cb1 || !P || count < 0 ||
      plan->tile != kGBN || ldp < plan->k || (ldp % kGBN) != 0)
    return fail(PF_E_ARG, "pf_mf_backward_level: bad argument (ldp must be a multiple of 64)");
  if (count == 0) return 0;
  if (max_f < 1 || max_ncb < 1) return fail(PF_E_ARG, "pf_mf_backward_level: bad limits");
  cudaStream_t st = as_stream(stream);
  auto launch = [&](auto kern, int nb, size_t ring) -> int {
    const size_t smem = ring + 8 * ((size_t)nb + 3 * max_ncb + max_f);
    if (int rc = ensure_smem((const void *)kern, smem)) return rc;
    kern<<<(unsigned)count, kBT + 32, smem, st>>>(*plan, M, O, item_node, item_rb, item_cb0,
                                                  item_cb1, P, ldp);
    return 0;
  };
  int rc;
  switch (nb_rows) {
    case 8: rc = launch(mf_bwd_gemm_kernel<8>, 8, bwd_ring_bytes<8>()); break;
    case 16: rc = launch(mf_bwd_gemm_kernel<16>, 16, bwd_ring_bytes<16>()); break;
    case 32: rc = launch(mf_bwd_gemm_kernel<32>, 32, bwd_ring_bytes<32>()); break;
    case 64: rc = launch(mf_bwd_gemm_kernel<64>, 64, bwd_ring_bytes<64>()); break;
    default: return fail(PF_E_ARG, "pf_mf_backward_level: nb_rows must be 8, 16, 32 or 64");
  }
  if (rc) return rc;
  return check_launch("pf_mf_backward_level");
}

int pf_poisson_residual_table(const int32_t *nb_idx, int64_t nnz, const uint8_t *is_boundary,
                              const int32_t *bcol, int64_t ldp, const int64_t *rowoff,
                              int64_t *nrow, pf_stream_t stream) {
  if ((nnz && (!nb_idx || !nrow)) || !is_boundary || !bcol || nnz < 0 || ldp < 1)
    return fail(PF_E_ARG, "pf_poisson_residual_table: bad argument");
  if (nnz == 0) return 0;
  residual_table_kernel<<<grid_for(nnz, 256), 256, 0, as_stream(stream)>>>(
      nb_idx, nnz, is_boundary, bcol, ldp, rowoff, nrow);
  return check_launch("pf_poisson_residual_table");
}

static int residual_launch(const char *what, const double *P, int64_t ldp, int64_t k,
                           const int32_t *order, int64_t count, const int64_t *rowoff,
                           const int64_t *nb_ptr, const int64_t *nrow, const double *off,
                           const double *diag, double *row_part, unsigned long long *out_max,
                           pf_stream_t stream) {
  if (count == 0) return 0;  // a row slab with no interior rows
  if (!P || !order || !nb_ptr || !nrow || !off || !diag || !out_max || k < 0 || count < 0 ||
      ldp < k || (ldp & 1) || (reinterpret_cast<uintptr_t>(P) & 15))
    return fail(PF_E_ARG, "%s: bad argument (ldp even, P 16-byte aligned)", what);
  // (32-warp CTAs over consecutive nested-dissection rows measured slower: 19.1
  // vs 17.7 ms at C4 — the kernel is bound by L2 traffic, ~9 reads per entry)
  constexpr int kW = 8;
  const unsigned chunks = (unsigned)((k + kResCols - 1) / kResCols);
  const unsigned rows = (unsigned)std::min<int64_t>((count + kW - 1) / kW, (int64_t)sm_count() * 8);
  residual_kernel<kW><<<dim3(rows, std::max(1u, chunks)), kW * 32, 0, as_stream(stream)>>>(
      P, ldp, k, order, count, rowoff, nb_ptr, nrow, off, diag, row_part, out_max);
  return check_launch(what);
}

int pf_poisson_residual(const double *P, int64_t ldp, int64_t k, const int32_t *order,
                        int64_t count, const int64_t *rowoff, const int64_t *nb_ptr,
                        const int64_t *nrow, const double *off, const double *diag,
                        unsigned long long *out_max, pf_stream_t stream) {
  return residual_launch("pf_poisson_residual", P, ldp, k, order, count, rowoff, nb_ptr, nrow,
                         off, diag, nullptr, out_max, stream);
}

int pf_poisson_residual_rows(const double *P, int64_t ldp, int64_t k, const int32_t *order,
                             int64_t count, const int64_t *rowoff, const int64_t *nb_ptr,
                             const int64_t *nrow, const double *off, const double *diag,
                             double *row_part, unsigned long long *out_max, pf_stream_t stream) {
  if (!row_part && count > 0) return fail(PF_E_ARG, "pf_poisson_residual_rows: row_part is NULL");
  return residual_launch("pf_poisson_residual_rows", P, ldp, k, order, count, rowoff, nb_ptr,
                         nrow, off, diag, row_part, out_max, stream);
}

int pf_poisson_finalize_rows(double *P, int64_t ldp, int64_t row0, int64_t n, int64_t k,
                             const uint8_t *is_boundary, const int32_t *bcol,
                             const double *row_part, unsigned long long *out_max,
                             pf_stream_t stream) {
  if (!P || !is_boundary || !bcol || !out_max || (n > 0 && !row_part) || n < 0 || k < 0 ||
      row0 < 0 || ldp < k)
    return fail(PF_E_ARG, "pf_poisson_finalize_rows: bad argument");
  if (n == 0) return 0;
  const int chunks = (int)((k + kResCols - 1) / kResCols);
  finalize_rows_kernel<<<grid_for(n * 32, 256), 256, 0, as_stream(stream)>>>(
      P, ldp, row0, n, k, is_boundary, bcol, row_part, std::max(1, chunks), out_max);
  return check_launch("pf_poisson_finalize_rows");
}

int pf_poisson_finalize(double *P, int64_t ldp, int64_t row0, int64_t n, int64_t k,
                        const uint8_t *is_boundary, const int32_t *bcol, double clamp, double *H,
                        double *min_out, unsigned long long *out_max, pf_stream_t stream) {
  if (!P || !is_boundary || !bcol || !out_max || n < 0 || k < 0 || ldp < k || (ldp & 1) ||
      (reinterpret_cast<uintptr_t>(P) & 15))
    return fail(PF_E_ARG, "pf_poisson_finalize: bad argument");
  if (n == 0) return 0;
  finalize_kernel<<<grid_for(n, 8), 256, 0, as_stream(stream)>>>(
      P, ldp, row0, n, k, is_boundary, bcol, clamp, H, min_out, out_max);
  return check_launch("pf_poisson_finalize");
}

}  // extern "C"
