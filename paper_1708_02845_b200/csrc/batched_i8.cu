// batched_i8.cu — K7 on the int8 tensor pipe: the batched-target KL
// contraction as an exact-integer emulation of the FP64 GEMM (Ozaki scheme
// with fixed-point byte slices) on tcgen05.mma kind::i8, TMEM accumulators,
// TMA-fed shared memory.
//
// Reference semantics: T calls of pathfield/divergence.py dv_field(pk, kl, t)
// (:154-187).  The contraction is
//
//   S[q, t] = sum_b a_qb * b_tb,   a_qb = max(P_qb, clamp) >= 0,
//                                  b_tb = -log max(P_tb, clamp) >= 0,
//   KL[q, t] = H[q] + S[q, t]      (H = sum c(Q) log c(Q), K1),
//
// and both operands are non-negative, so each is written as a 56-bit
// unsigned fixed-point number against a per-row (a) / per-target (b)
// power-of-two scale and cut into seven unsigned bytes (most significant
// first):
//
//   a_qb = 2^ea_q * sum_{i=1..7} A_i[q,b] 2^-8i,  b_tb = 2^eb_t * sum_j B_j[t,b] 2^-8j
//   S    = 2^(ea+eb) * sum_{l=2..} acc_l 2^-8l,   acc_l = sum_{i+j=l} A_i . B_j^T
//
// Every acc_l is an exact integer GEMM (u8 x u8 -> s32 in TMEM; at most 7
// pairs x k x 255^2 < 2^31 for k <= 4717).  Levels 2..9 are kept (34 byte-
// pair GEMMs); the first dropped level is 2^-80 relative, and rounding each
// operand to 56 bits perturbs it by 2^-57 relative to its row / target
// maximum: with sum_b a_qb = 1 (rows of P are stochastic) the absolute error
// of S is ~1e-14, the same order as FP64 accumulation over k = 4102 terms.
// The split-form cancellation guard of K2/K7 (|KL| < tau (|H| + |S|),
// tau = 1e-3) sends the few pairs where that error could exceed 1e-10
// relative to the reference-form per-element fixup (batched.cu), exactly as
// the FP64 DMMA path does.
//
// Kernel shape: one CTA per 128 rows x 128 targets output tile, 320 threads.
// TMEM holds four N=128 s32 accumulators (all 512 columns), so each tile runs
// two passes over K: levels 2..5 (10 pairs, slices 1..4), then levels 6..9
// (24 pairs, slices 1..7), the first drained to FP64 registers in between.
//   warp 0 lane 0   TMA producer: per 32-byte K block one 3-D box of the A
//                   slices (128 rows) and one of the B slices (128 targets),
//                   SWIZZLE_32B, 4-stage ring (<= 56 KB / stage)
//   warp 1 lane 0   MMA issuer: M128 N128 K32 u8 x u8 -> s32
//   warps 2-9       epilogue: each the 32 TMEM lanes of its quarter x 64
//                   columns; tcgen05.ld, combine the levels in FP64, scale,
//                   fuse the guard / settle / target-zero, store.
// The int8 pipe draws the board to its 1000 W cap at this shape, so the
// kernel is power-bound (tools/probe_power.py); a 128 x 64 single-pass
// variant with eight N=64 level accumulators was 7% slower (tuning record in
// profiles/).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>

#include "pf_common.cuh"
#include "pf_tc.cuh"

namespace pf {

constexpr int kOzSlices = 7;                 // bytes per operand (56-bit fixed point)
constexpr int kOzPad = 64;                   // ldk % 64 == 0 (slice plane row pitch)
constexpr int kOzMaxK = 4717;                // 7 x k x 255^2 < 2^31
constexpr unsigned long long kOzGuard = 0x7ff8dead0000ba7cull;    // == batched.cu kBatchGuard

// ---------------------------------------------------------------- slicing --
// 8 consecutive values -> 7 byte planes (most significant byte in plane 0).
__device__ __forceinline__ void slice8(const double (&x)[8], int e, uint64_t (&w)[kOzSlices]) {
#pragma unroll
  for (int s = 0; s < kOzSlices; ++s) w[s] = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const unsigned long long N = __double2ull_rn(ldexp(x[u], 56 - e));  // < 2^56
#pragma unroll
    for (int s = 0; s < kOzSlices; ++s)
      w[s] |= static_cast<uint64_t>((N >> (8 * (kOzSlices - 1 - s))) & 0xffu) << (8 * u);
  }
}

__device__ __forceinline__ int scale_exp(double m) { return m > 0.0 ? ilogb(m) + 1 : 0; }

// Rows of the slab: a = max(P, clamp), warp per row.  slices: [7][rows][ldk].
__global__ void __launch_bounds__(256) slice_rows_kernel(const double *__restrict__ P, int64_t ld,
                                                         int64_t rows, int64_t k, double clamp,
                                                         int64_t ldk, uint8_t *__restrict__ out,
                                                         int32_t *__restrict__ exps) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t plane = rows * ldk;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const double *row = P + r * ld;
    double m = 0.0;
    for (int64_t b = lane; b < k; b += 32) m = fmax(m, fmax(row[b], clamp));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const int e = scale_exp(m);
    if (lane == 0) exps[r] = e;
    for (int64_t b0 = 8 * lane; b0 < ldk; b0 += 256) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = (b0 + u < k) ? fmax(row[b0 + u], clamp) : 0.0;
      uint64_t w[kOzSlices];
      slice8(x, e, w);
#pragma unroll
      for (int s = 0; s < kOzSlices; ++s)
        *reinterpret_cast<uint64_t *>(out + s * plane + r * ldk + b0) = w[s];
    }
  }
}

// Targets: b = -L (L = log max(Pt, clamp), batch_prep_kernel), block per
// target.  bad[0] |= 1 if some b < 0 (a target entry above 1: the caller then
// uses the FP64 path).  slices: [7][T][ldk].
__global__ void __launch_bounds__(256) slice_targets_kernel(const double *__restrict__ L,
                                                            int64_t ldl, int64_t T, int64_t k,
                                                            int64_t ldk, uint8_t *__restrict__ out,
                                                            int32_t *__restrict__ exps,
                                                            uint32_t *__restrict__ bad) {
  const int64_t t = blockIdx.x;
  if (t >= T) return;
  const double *row = L + t * ldl;
  __shared__ double red[8];
  double m = 0.0;
  bool neg = false;
  for (int64_t b = threadIdx.x; b < k; b += blockDim.x) {
    const double v = -row[b];
    neg |= v < 0.0;
    m = fmax(m, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  neg = __syncthreads_or(neg);
  m = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
  const int e = scale_exp(m);
  if (threadIdx.x == 0) {
    exps[t] = e;
    if (neg && bad) atomicOr(bad, 1u);
  }
  const int64_t plane = T * ldk;
  for (int64_t b0 = 8 * threadIdx.x; b0 < ldk; b0 += 8 * blockDim.x) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = (b0 + u < k) ? fmax(-row[b0 + u], 0.0) : 0.0;
    uint64_t w[kOzSlices];
    slice8(x, e, w);
#pragma unroll
    for (int s = 0; s < kOzSlices; ++s)
      *reinterpret_cast<uint64_t *>(out + s * plane + t * ldk + b0) = w[s];
  }
}

// v * 2^e with one rounding == ldexp(v, e) whenever 2^e is a normal double
__device__ __forceinline__ double pow2_scale(double v, int e) {
  return (e >= -1022 && e <= 1023)
             ? v * __longlong_as_double(static_cast<long long>(e + 1023) << 52)
             : ldexp(v, e);
}

// ------------------------------------------------------------------ GEMM --
// Two passes per 128 x 128 output tile, because TMEM holds four N=128
// accumulators (4 x 128 columns = all 512): pass 1 = levels 2..5 (10 byte
// pairs, slices 1..4), pass 2 = levels 6..9 (24 pairs, slices 1..7).  Between
// them the 8 epilogue warps drain pass 1 into FP64 registers (each warp: its
// 32 TMEM lanes x 64 columns) and release TMEM.  K blocks are 32 bytes
// (SWIZZLE_32B rows = one MMA K step), 4-stage TMA ring of up to 56 KB.
constexpr int kO2BN = 128, kO2BK = 32, kO2Stages = 4;
constexpr int kO2Tile = 128 * kO2BK;                     // one slice, 4 KB (A or B)
constexpr int kO2StageBytes = 2 * kOzSlices * kO2Tile;   // 57,344
constexpr int kO2Smem = kO2Stages * kO2StageBytes + 1024;
constexpr int kO2Threads = 320;                          // warp 0 TMA, 1 MMA, 2-9 epilogue
constexpr int kO2Pass1Slices = 4;

// Pass 2 covers levels 6..kMaxL with byte planes 1..kS: (7, 9) is the FP64
// grade (34 pairs in all), (5, 6) the FP32 grade of the north-star 1e-5
// tolerance (15 pairs, the top 40 bits of the same planes).
template <int kS, int kMaxL>
__global__ void __launch_bounds__(kO2Threads, 1) batched_kl_i8_n128_kernel(
    const __grid_constant__ CUtensorMap mapA7, const __grid_constant__ CUtensorMap mapA4,
    const __grid_constant__ CUtensorMap mapB7, const __grid_constant__ CUtensorMap mapB4,
    const int32_t *__restrict__ ea, const int32_t *__restrict__ eb, int64_t rows, int64_t T,
    int nkb, const double *__restrict__ H, const int64_t *__restrict__ targets, double tau,
    int64_t row0, double *__restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full_bar[kO2Stages], empty_bar[kO2Stages];
  __shared__ __align__(8) uint64_t pass_bar[2], drained_bar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t0 = blockIdx.x * kO2BN;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * 128;

  if (tid == 0) {
    tc::prefetch_map(&mapA7);
    tc::prefetch_map(&mapA4);
    tc::prefetch_map(&mapB7);
    tc::prefetch_map(&mapB4);
    for (int s = 0; s < kO2Stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&pass_bar[0], 1);
    mbar_init(&pass_bar[1], 1);
    mbar_init(&drained_bar, 8);  // one arrival per epilogue warp
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: pass-1 K blocks (4 slices each), then pass-2 (7)
      for (int it = 0; it < 2 * nkb; ++it) {
        const int s = it % kO2Stages;
        const uint32_t round = it / kO2Stages;
        const bool p1 = it < nkb;
        const int kb = p1 ? it : it - nkb;
        mbar_wait(&empty_bar[s], (round & 1) ^ 1);
        uint8_t *sa = smem + s * kO2StageBytes;
        uint8_t *sb = sa + kOzSlices * kO2Tile;
        mbar_expect_tx(&full_bar[s], (p1 ? kO2Pass1Slices : kS) * 2 * kO2Tile);
        tc::tma_load_3d(sa, p1 ? &mapA4 : &mapA7, kb * kO2BK, static_cast<int32_t>(q0), 0,
                        &full_bar[s]);
        tc::tma_load_3d(sb, p1 ? &mapB4 : &mapB7, kb * kO2BK, t0, 0, &full_bar[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer; each pass its own loop (a conditional commit inside
      // a shared loop compiles to a predicated UTCBAR that stalls every stage)
      constexpr uint32_t idesc = tc::idesc_i8(128, kO2BN, false, false);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kO2Stages;
        mbar_wait(&full_bar[s], (kb / kO2Stages) & 1);
        tc::fence_after();
        const uint32_t sa = smem_u32(smem + s * kO2StageBytes);
        const uint32_t sb = sa + kOzSlices * kO2Tile;
#pragma unroll
        for (int i = 1; i <= kO2Pass1Slices; ++i)
#pragma unroll
          for (int j = 1; j <= kO2Pass1Slices; ++j) {
            const int l = i + j;
            if (l > 5) continue;
            tc::mma_i8(tmem + (l - 2) * kO2BN, tc::sdesc<32>(sa + (i - 1) * kO2Tile),
                       tc::sdesc<32>(sb + (j - 1) * kO2Tile), idesc, !(kb == 0 && i == 1));
          }
        tc::commit(&empty_bar[s]);
      }
      tc::commit(&pass_bar[0]);
      mbar_wait(&drained_bar, 0);   // pass 2 reuses the accumulators
      tc::fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        const int it = nkb + kb, s = it % kO2Stages;
        mbar_wait(&full_bar[s], (it / kO2Stages) & 1);
        tc::fence_after();
        const uint32_t sa = smem_u32(smem + s * kO2StageBytes);
        const uint32_t sb = sa + kOzSlices * kO2Tile;
#pragma unroll
        for (int i = 1; i <= kS; ++i)
#pragma unroll
          for (int j = 1; j <= kS; ++j) {
            const int l = i + j;
            if (l < 6 || l > kMaxL) continue;
            const int first_i = l - kS > 1 ? l - kS : 1;
            tc::mma_i8(tmem + (l - 6) * kO2BN, tc::sdesc<32>(sa + (i - 1) * kO2Tile),
                       tc::sdesc<32>(sb + (j - 1) * kO2Tile), idesc, !(kb == 0 && i == first_i));
          }
        tc::commit(&empty_bar[s]);
      }
      tc::commit(&pass_bar[1]);
    }
  } else {
    // ---- epilogue warps 2..9: TMEM lanes 32 (warp % 4) .. +31, columns half * 64 .. +63
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const int64_t q = q0 + r;
    const bool row_ok = q < rows;
    const uint32_t base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + half * 64;
    double v1[64];
    mbar_wait(&pass_bar[0], 0);
    tc::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 8) {
      uint32_t acc[4][8];
#pragma unroll
      for (int l = 0; l < 4; ++l) tc::tmem_ld8(base + l * kO2BN + c0, acc[l]);
      tc::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        double v = static_cast<double>(acc[3][u]);
#pragma unroll
        for (int l = 2; l >= 0; --l) v = fma(v, 0x1p-8, static_cast<double>(acc[l][u]));
        v1[c0 + u] = v;
      }
    }
    tc::fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&drained_bar);
    mbar_wait(&pass_bar[1], 0);
    tc::fence_after();
    const double h = row_ok ? H[q] : 0.0;
    const int e_q = row_ok ? ea[q] : 0;
    const int64_t tq = row_ok ? row0 + q : -1;
    constexpr int kL2 = kMaxL - 5;  // pass-2 accumulators
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 8) {
      uint32_t acc[kL2][8];
#pragma unroll
      for (int l = 0; l < kL2; ++l) tc::tmem_ld8(base + l * kO2BN + c0, acc[l]);
      tc::tmem_ld_wait();
      if (!row_ok) continue;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t t = t0 + half * 64 + c0 + u;
        if (t >= T) continue;
        double v = static_cast<double>(acc[kL2 - 1][u]);
#pragma unroll
        for (int l = kL2 - 2; l >= 0; --l) v = fma(v, 0x1p-8, static_cast<double>(acc[l][u]));
        v = fma(v, 0x1p-32, v1[c0 + u]);
        const double S = pow2_scale(v, e_q + eb[t] - 16);
        double val = h + S;
        const bool is_t = (tq == targets[t]);
        if (!is_t && fabs(val) < tau * (fabs(h) + fabs(S)))
          val = __longlong_as_double(static_cast<long long>(kOzGuard));
        else
          val = is_t ? 0.0 : settle(val);
        out[q * ldo + t] = val;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem);
}

// PF_K7_DIAG bit 2: per-CTA %globaltimer stamps into out[cta * 8 + i]
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// ---------------------------------------------------------- GEMM, CTA pair --
// The same two-pass level schedule on a CTA pair (cta_group::2, cluster of 2
// CTAs on two row tiles): the leader issues M256 N128 K32 MMAs whose A rows
// 0-127 come from its own shared memory and 128-255 from the peer's, and whose
// B (the 128 targets) is split 64 / 64 between the two; each CTA's TMEM gets
// its own 128 rows.  Per SM and MMA the tensor pipe reads 4 KB of A + 2 KB of
// B from shared memory instead of 4 + 4 KB, and TMA writes 6 instead of 8 KB
// per slice: the 1-CTA kernel is shared-memory bound (UMMA operand reads +
// TMA writes ~151 B/clk against ~128).  5-stage ring of 42 KB per CTA.  The
// arithmetic is the same exact integers, so the outputs are bitwise the
// 1-CTA kernel's.
constexpr int kP2BN = 128, kP2HalfN = 64, kP2Stages = 5;
constexpr int kP2TileA = 128 * kO2BK;                         // 4 KB per slice
constexpr int kP2TileB = kP2HalfN * kO2BK;                    // 2 KB per slice
constexpr int kP2StageBytes = kOzSlices * (kP2TileA + kP2TileB);  // 43,008
constexpr int kP2Smem = kP2Stages * kP2StageBytes + 1024;

//
// kQuad: two such pairs in one cluster of 4 on the same row-tile pair and
// adjacent target tiles share every A tile by TMA multicast: each CTA loads
// one 64-row half of its row tile (one box per slice, the UMMA layout needs
// the halves interleaved within each slice plane) and multicasts it to the
// CTA of the other pair holding the same rows, so A crosses L2 -> SM once
// per two pairs.  Each slot's empty barrier then waits for both pairs' MMAs.
//
// kDiag (timing diagnostics only, PF_K7_DIAG, wrong outputs): bit 0 = no TMA
// loads (the MMAs run on stale shared memory), bit 1 = no epilogue arithmetic
// or stores (accumulators drained and dropped).
template <int kS, int kMaxL, bool kQuad, int kDiag = 0>
__global__ void __launch_bounds__(kO2Threads, 1)
    batched_kl_i8_pair_kernel(const __grid_constant__ CUtensorMap mapA7,
                              const __grid_constant__ CUtensorMap mapA4,
                              const __grid_constant__ CUtensorMap mapB7,
                              const __grid_constant__ CUtensorMap mapB4,
                              const int32_t *__restrict__ ea, const int32_t *__restrict__ eb,
                              int64_t rows, int64_t T, int nkb, const double *__restrict__ H,
                              const int64_t *__restrict__ targets, double tau, int64_t row0,
                              double *__restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full_bar[kP2Stages], empty_bar[kP2Stages];
  __shared__ __align__(8) uint64_t pass_bar[2], drained_bar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double *stamp = (kDiag & 4) ? out + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 8
                              : nullptr;
  if ((kDiag & 4) && tid == 0) stamp[0] = static_cast<double>(gtimer());
  // cluster (2, 1, 1): x = 2 x target tile + pair rank (the 2-CTA MMA pairs
  // adjacent x ranks), y = row-tile pair; the target tiles of one row pair are
  // consecutive CTAs, so its A tiles stream from HBM once and hit L2 after
  const uint32_t crank = tc::cluster_rank();
  const uint32_t rank = crank & 1;           // 0 = pair leader (issues the MMAs)
  const uint32_t pairi = crank >> 1;         // kQuad: which pair of the cluster
  const uint32_t leader = crank & 2;         // cluster rank of this pair's leader
  const int t0 = kQuad ? ((blockIdx.x >> 2) * 2 + pairi) * kP2BN : (blockIdx.x >> 1) * kP2BN;
  const int64_t q0 = (static_cast<int64_t>(blockIdx.y) * 2 + rank) * 128;   // this CTA's rows

  if (tid == 0) {
    tc::prefetch_map(&mapA7);
    tc::prefetch_map(&mapA4);
    tc::prefetch_map(&mapB7);
    tc::prefetch_map(&mapB4);
    for (int s = 0; s < kP2Stages; ++s) {
      mbar_init(&full_bar[s], 1);    // the leader's producer arrives (both CTAs' bytes)
      mbar_init(&empty_bar[s], kQuad ? 2 : 1);   // one multicast commit per pair
    }
    mbar_init(&pass_bar[0], 1);
    mbar_init(&pass_bar[1], 1);
    mbar_init(&drained_bar, 16);     // every epilogue warp of both CTAs
  }
  if (warp == 0) tc::tmem_alloc_pair<512>(&tmem_base);
  tc::fence_before();
  tc::cluster_sync();               // barriers of both CTAs initialised, TMEM allocated
  if ((kDiag & 4) && tid == 0) stamp[1] = static_cast<double>(gtimer());
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): own 128 A rows, own half of the targets
      const int32_t tb = t0 + static_cast<int32_t>(rank) * kP2HalfN;
      for (int it = 0; it < 2 * nkb; ++it) {
        const int s = it % kP2Stages;
        const uint32_t round = it / kP2Stages;
        const bool p1 = it < nkb;
        const int kb = p1 ? it : it - nkb;
        const int ns = p1 ? kO2Pass1Slices : kS;
        mbar_wait(&empty_bar[s], (round & 1) ^ 1);
        uint8_t *sa = smem + s * kP2StageBytes;
        uint8_t *sb = sa + kOzSlices * kP2TileA;
        if constexpr ((kDiag & 1) != 0) {
          if (rank == 0) mbar_arrive(&full_bar[s]);
          continue;
        }
        if (rank == 0) mbar_expect_tx(&full_bar[s], 2 * ns * (kP2TileA + kP2TileB));
        const uint32_t lb = tc::mapa(&full_bar[s], leader);
        if constexpr (kQuad) {   // mapA7 = 64-row, 1-slice boxes
          const uint16_t mc = static_cast<uint16_t>(5u << rank);   // {rank, rank + 2}
          for (int sl = 0; sl < ns; ++sl)
            tc::tma_load_3d_pair_mc(sa + sl * kP2TileA + pairi * (64 * kO2BK), &mapA7, kb * kO2BK,
                                    static_cast<int32_t>(q0 + pairi * 64), sl, &full_bar[s], mc);
        } else {
          tc::tma_load_3d_pair(sa, p1 ? &mapA4 : &mapA7, kb * kO2BK, static_cast<int32_t>(q0), 0,
                               lb);
        }
        tc::tma_load_3d_pair(sb, p1 ? &mapB4 : &mapB7, kb * kO2BK, tb, 0, lb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---- MMA issuer (leader only): M256 N128 K32.  The two passes are
      // separate loops: a conditional tcgen05.commit inside one loop compiles
      // to a predicated UTCBAR that stalls the issue every stage even when
      // its predicate is off (pass 1 ran at 94 instead of 64 clk per MMA).
      constexpr uint32_t idesc = tc::idesc_i8(256, kP2BN, false, false);
      const uint16_t own = static_cast<uint16_t>(3u << leader);
      constexpr uint16_t ring = kQuad ? 0xF : 3;
      auto wait_stage = [&](int it) -> uint32_t {
        const int s = it % kP2Stages;
        uint64_t tw0 = 0;
        if constexpr ((kDiag & 8) != 0) tw0 = clock64();
        if constexpr ((kDiag & 16) == 0) mbar_wait(&full_bar[s], (it / kP2Stages) & 1);
        if constexpr ((kDiag & 8) != 0) {
          if (blockIdx.x == 0 && blockIdx.y == 0) {
            double *tl = out + static_cast<int64_t>(gridDim.x) * gridDim.y * 8;
            tl[2 * it] = static_cast<double>(tw0);
            tl[2 * it + 1] = static_cast<double>(clock64());
          }
        }
        tc::fence_after();
        return smem_u32(smem + s * kP2StageBytes);
      };
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t sa = wait_stage(kb);
        const uint32_t sb = sa + kOzSlices * kP2TileA;
#pragma unroll
        for (int i = 1; i <= kO2Pass1Slices; ++i)
#pragma unroll
          for (int j = 1; j <= kO2Pass1Slices; ++j) {
            const int l = i + j;
            if (l > 5) continue;
            tc::mma_i8_pair(tmem + (l - 2) * kP2BN, tc::sdesc<32>(sa + (i - 1) * kP2TileA),
                            tc::sdesc<32>(sb + (j - 1) * kP2TileB), idesc, !(kb == 0 && i == 1));
          }
        tc::commit_pair_mask(&empty_bar[kb % kP2Stages], ring);
      }
      tc::commit_pair_mask(&pass_bar[0], own);
      // pass 2 reuses the accumulators: wait for both CTAs' drains
      if (kDiag & 4) stamp[2] = static_cast<double>(gtimer());
      mbar_wait(&drained_bar, 0);
      if (kDiag & 4) stamp[3] = static_cast<double>(gtimer());
      tc::fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t sa = wait_stage(nkb + kb);
        const uint32_t sb = sa + kOzSlices * kP2TileA;
#pragma unroll
        for (int i = 1; i <= kS; ++i)
#pragma unroll
          for (int j = 1; j <= kS; ++j) {
            const int l = i + j;
            if (l < 6 || l > kMaxL) continue;
            const int first_i = l - kS > 1 ? l - kS : 1;
            tc::mma_i8_pair(tmem + (l - 6) * kP2BN, tc::sdesc<32>(sa + (i - 1) * kP2TileA),
                            tc::sdesc<32>(sb + (j - 1) * kP2TileB), idesc,
                            !(kb == 0 && i == first_i));
          }
        tc::commit_pair_mask(&empty_bar[(nkb + kb) % kP2Stages], ring);
      }
      tc::commit_pair_mask(&pass_bar[1], own);
    }
  } else {
    // ---- epilogue warps 2..9 (both CTAs, own TMEM = own 128 rows x 128 targets)
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const int64_t q = q0 + r;
    const bool row_ok = q < rows;
    const uint32_t base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + half * 64;
    double v1[64];
    mbar_wait(&pass_bar[0], 0);
    tc::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 8) {
      uint32_t acc[4][8];
#pragma unroll
      for (int l = 0; l < 4; ++l) tc::tmem_ld8(base + l * kP2BN + c0, acc[l]);
      tc::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        double v = static_cast<double>(acc[3][u]);
#pragma unroll
        for (int l = 2; l >= 0; --l) v = fma(v, 0x1p-8, static_cast<double>(acc[l][u]));
        v1[c0 + u] = v;
      }
    }
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive_cluster(tc::mapa(&drained_bar, leader));
    mbar_wait(&pass_bar[1], 0);
    if ((kDiag & 4) && tid == 64) stamp[4] = static_cast<double>(gtimer());
    tc::fence_after();
    const double h = row_ok ? H[q] : 0.0;
    const int e_q = row_ok ? ea[q] : 0;
    const int64_t tq = row_ok ? row0 + q : -1;
    constexpr int kL2 = kMaxL - 5;
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 8) {
      uint32_t acc[kL2][8];
#pragma unroll
      for (int l = 0; l < kL2; ++l) tc::tmem_ld8(base + l * kP2BN + c0, acc[l]);
      tc::tmem_ld_wait();
      if (!row_ok || (kDiag & 2) != 0) continue;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t t = t0 + half * 64 + c0 + u;
        if (t >= T) continue;
        double v = static_cast<double>(acc[kL2 - 1][u]);
#pragma unroll
        for (int l = kL2 - 2; l >= 0; --l) v = fma(v, 0x1p-8, static_cast<double>(acc[l][u]));
        v = fma(v, 0x1p-32, v1[c0 + u]);
        const double S = pow2_scale(v, e_q + eb[t] - 16);
        double val = h + S;
        const bool is_t = (tq == targets[t]);
        if (!is_t && fabs(val) < tau * (fabs(h) + fabs(S)))
          val = __longlong_as_double(static_cast<long long>(kOzGuard));
        else
          val = is_t ? 0.0 : settle(val);
        out[q * ldo + t] = val;
      }
    }
  }
  if ((kDiag & 4) && tid == 64) stamp[5] = static_cast<double>(gtimer());
  tc::fence_before();
  tc::cluster_sync();   // both CTAs done with TMEM and with each other's barriers
  if ((kDiag & 4) && tid == 0) {
    stamp[6] = static_cast<double>(gtimer());
    stamp[7] = static_cast<double>(smid());
  }
  if (warp == 0) tc::tmem_free_pair<512>(tmem);
}

// ------------------------------------------------ GEMM, persistent CTA pair --
// The CTA-pair kernel made persistent (one cluster per SM pair, tiles
// strided over the clusters; consecutive clusters share a row pair so its A
// planes are read from HBM once and from L2 after) with the epilogue taken
// off the tensor pipe's critical path: the epilogue warps fold the pass-2
// accumulators into the FP64 pass-1 partials in registers, release TMEM to
// the MMA thread (free_bar), and only then apply the scale / guard / settle
// and store -- while the next tile's pass-1 MMAs run.  Same integers, same
// FP64 operation order: bitwise the 1-CTA kernel's outputs.
template <int kS, int kMaxL, int kDiag = 0>
__global__ void __launch_bounds__(kO2Threads, 1)
    batched_kl_i8_pp_kernel(const __grid_constant__ CUtensorMap mapA7,
                            const __grid_constant__ CUtensorMap mapA4,
                            const __grid_constant__ CUtensorMap mapB7,
                            const __grid_constant__ CUtensorMap mapB4,
                            const int32_t *__restrict__ ea, const int32_t *__restrict__ eb,
                            int64_t rows, int64_t T, int nkb, const double *__restrict__ H,
                            const int64_t *__restrict__ targets, double tau, int64_t row0,
                            double *__restrict__ out, int64_t ldo, int t_tiles, int ntiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full_bar[kP2Stages], empty_bar[kP2Stages];
  __shared__ __align__(8) uint64_t pass_bar[2], drained_bar, free_bar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();   // 0 = leader (issues the MMAs)
  const int cid = static_cast<int>(blockIdx.x >> 1), ncl = static_cast<int>(gridDim.x >> 1);

  if (tid == 0) {
    tc::prefetch_map(&mapA7);
    tc::prefetch_map(&mapA4);
    tc::prefetch_map(&mapB7);
    tc::prefetch_map(&mapB4);
    for (int s = 0; s < kP2Stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&pass_bar[0], 1);
    mbar_init(&pass_bar[1], 1);
    mbar_init(&drained_bar, 16);     // every epilogue warp of both CTAs, per tile
    mbar_init(&free_bar, 16);
  }
  if (warp == 0) tc::tmem_alloc_pair<512>(&tmem_base);
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): own 128 A rows, own half of the targets
      int it = 0;
      for (int w = cid; w < ntiles; w += ncl) {
        const int64_t q0 = (static_cast<int64_t>(w / t_tiles) * 2 + rank) * 128;
        const int32_t tb = (w % t_tiles) * kP2BN + static_cast<int32_t>(rank) * kP2HalfN;
        for (int pass = 0; pass < 2; ++pass) {
          const int ns = pass == 0 ? kO2Pass1Slices : kS;
          const CUtensorMap *ma = pass == 0 ? &mapA4 : &mapA7;
          const CUtensorMap *mb = pass == 0 ? &mapB4 : &mapB7;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % kP2Stages;
            mbar_wait(&empty_bar[s], ((it / kP2Stages) & 1) ^ 1);
            if constexpr ((kDiag & 1) != 0) {
              if (rank == 0) mbar_arrive(&full_bar[s]);
              continue;
            }
            uint8_t *sa = smem + s * kP2StageBytes;
            uint8_t *sb = sa + kOzSlices * kP2TileA;
            if (rank == 0) mbar_expect_tx(&full_bar[s], 2 * ns * (kP2TileA + kP2TileB));
            const uint32_t lb = tc::mapa(&full_bar[s], 0);
            tc::tma_load_3d_pair(sa, ma, kb * kO2BK, static_cast<int32_t>(q0), 0, lb);
            tc::tma_load_3d_pair(sb, mb, kb * kO2BK, tb, 0, lb);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---- MMA issuer (leader only): M256 N128 K32; each pass its own loop
      // (a conditional commit inside a shared loop costs a stall per stage)
      constexpr uint32_t idesc = tc::idesc_i8(256, kP2BN, false, false);
      int it = 0, k = 0;
      for (int w = cid; w < ntiles; w += ncl, ++k) {
        if (k > 0) {   // the previous tile's pass-2 accumulators drained
          mbar_wait(&free_bar, (k - 1) & 1);
          tc::fence_after();
        }
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kP2Stages;
          mbar_wait(&full_bar[s], (it / kP2Stages) & 1);
          tc::fence_after();
          const uint32_t sa = smem_u32(smem + s * kP2StageBytes);
          const uint32_t sb = sa + kOzSlices * kP2TileA;
#pragma unroll
          for (int i = 1; i <= kO2Pass1Slices; ++i)
#pragma unroll
            for (int j = 1; j <= kO2Pass1Slices; ++j) {
              const int l = i + j;
              if (l > 5) continue;
              tc::mma_i8_pair(tmem + (l - 2) * kP2BN, tc::sdesc<32>(sa + (i - 1) * kP2TileA),
                              tc::sdesc<32>(sb + (j - 1) * kP2TileB), idesc,
                              !(kb == 0 && i == 1));
            }
          tc::commit_pair(&empty_bar[s]);
        }
        tc::commit_pair(&pass_bar[0]);
        mbar_wait(&drained_bar, k & 1);   // pass 2 reuses the accumulators
        tc::fence_after();
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kP2Stages;
          mbar_wait(&full_bar[s], (it / kP2Stages) & 1);
          tc::fence_after();
          const uint32_t sa = smem_u32(smem + s * kP2StageBytes);
          const uint32_t sb = sa + kOzSlices * kP2TileA;
#pragma unroll
          for (int i = 1; i <= kS; ++i)
#pragma unroll
            for (int j = 1; j <= kS; ++j) {
              const int l = i + j;
              if (l < 6 || l > kMaxL) continue;
              const int first_i = l - kS > 1 ? l - kS : 1;
              tc::mma_i8_pair(tmem + (l - 6) * kP2BN, tc::sdesc<32>(sa + (i - 1) * kP2TileA),
                              tc::sdesc<32>(sb + (j - 1) * kP2TileB), idesc,
                              !(kb == 0 && i == first_i));
            }
          tc::commit_pair(&empty_bar[s]);
        }
        tc::commit_pair(&pass_bar[1]);
      }
    }
  } else {
    // ---- epilogue warps 2..9 (both CTAs, own TMEM = own 128 rows x 128 targets)
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + half * 64;
    const uint32_t drained_leader = tc::mapa(&drained_bar, 0);
    const uint32_t free_leader = tc::mapa(&free_bar, 0);
    constexpr int kL2 = kMaxL - 5;
    const bool pairs_ok = (ldo % 2 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    int k = 0;
    for (int w = cid; w < ntiles; w += ncl, ++k) {
      const int64_t q = (static_cast<int64_t>(w / t_tiles) * 2 + rank) * 128 + r;
      const int64_t tc0 = static_cast<int64_t>(w % t_tiles) * kP2BN + half * 64;
      double v[64];
      mbar_wait(&pass_bar[0], k & 1);
      tc::fence_after();
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 8) {
        uint32_t acc[4][8];
#pragma unroll
        for (int l = 0; l < 4; ++l) tc::tmem_ld8(base + l * kP2BN + c0, acc[l]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          double x = static_cast<double>(acc[3][u]);
#pragma unroll
          for (int l = 2; l >= 0; --l) x = fma(x, 0x1p-8, static_cast<double>(acc[l][u]));
          v[c0 + u] = x;
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(drained_leader);
      mbar_wait(&pass_bar[1], k & 1);
      tc::fence_after();
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 8) {
        uint32_t acc[kL2][8];
#pragma unroll
        for (int l = 0; l < kL2; ++l) tc::tmem_ld8(base + l * kP2BN + c0, acc[l]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          double x = static_cast<double>(acc[kL2 - 1][u]);
#pragma unroll
          for (int l = kL2 - 2; l >= 0; --l) x = fma(x, 0x1p-8, static_cast<double>(acc[l][u]));
          v[c0 + u] = fma(x, 0x1p-32, v[c0 + u]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(free_leader);   // TMEM free for the next tile
      if ((kDiag & 2) != 0 || q >= rows) continue;
      const double h = H[q];
      const int e_q = ea[q] - 16;
      const int64_t tq = row0 + q;
      double *orow = out + q * ldo + tc0;
      const bool full = pairs_ok && tc0 + 64 <= T;
#pragma unroll
      for (int c = 0; c < 64; c += 2) {
        double o[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t t = tc0 + c + u;
          const bool in = t < T;
          const double S = pow2_scale(v[c + u], e_q + (in ? eb[t] : 0));
          double val = h + S;
          const bool is_t = in && (tq == targets[t]);
          if (!is_t && fabs(val) < tau * (fabs(h) + fabs(S)))
            val = __longlong_as_double(static_cast<long long>(kOzGuard));
          else
            val = is_t ? 0.0 : settle(val);
          o[u] = val;
        }
        if (full) {
          *reinterpret_cast<double2 *>(orow + c) = make_double2(o[0], o[1]);
        } else {
          if (tc0 + c < T) orow[c] = o[0];
          if (tc0 + c + 1 < T) orow[c + 1] = o[1];
        }
      }
    }
  }
  tc::fence_before();
  tc::cluster_sync();   // both CTAs done with TMEM and with each other's barriers
  if (warp == 0) tc::tmem_free_pair<512>(tmem);
}

// Diagnostic: the int8 tensor pipe's issue-rate ceiling, back-to-back
// M128 N256 K32 u8 MMAs on shared-memory-resident operands, one CTA per SM;
// bench.py reports K7's int8 rate against it.
__global__ void __launch_bounds__(128, 1) umma_i8_probe_kernel(int iters, int random,
                                                              uint32_t *sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 + 256) * 64 / 4; i += 128) {
    uint32_t h = static_cast<uint32_t>(i + 4099 * blockIdx.x) * 2654435761u;   // random bytes
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t *>(smem)[i] = random ? h : 0x01010101u * (i & 3);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) mbar_init(&bar, 1);
  if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    constexpr uint32_t id = tc::idesc_i8(128, 256, false, false);
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * 64;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
        tc::mma_i8(tm, tc::sdesc<64>(sa + 32 * ks), tc::sdesc<64>(sb + 32 * ks), id,
                   (it | ks) != 0);
    tc::commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc::fence_after();
  uint32_t v[8];
  tc::tmem_ld8(tm + (static_cast<uint32_t>(warp * 32) << 16), v);
  tc::tmem_ld_wait();
  if (v[0] == 0x12345u) sink[0] = v[1];
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<256>(tm);
}

// ------------------------------------------------------------ tensor maps --
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D u8 map over slices [7][outer][ldk]: box {box_k, box_rows, box_slices},
// swizzle = box_k bytes, out-of-range rows read as zero.
static int slice_map(CUtensorMap *map, const uint8_t *base, int64_t outer, int64_t ldk,
                     uint32_t box_rows, uint32_t box_k, uint32_t box_slices) {
  auto fn = encode_fn();
  if (!fn) return fail(PF_E_LAUNCH, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(ldk), static_cast<cuuint64_t>(outer),
                        static_cast<cuuint64_t>(kOzSlices)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldk), static_cast<cuuint64_t>(outer * ldk)};
  cuuint32_t box[3] = {box_k, box_rows, box_slices};
  const CUtensorMapSwizzle sw = box_k == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : box_k == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_32B;
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PF_E_ARG, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

template <int kS, int kMaxL>
static int launch_i8(const CUtensorMap (&m)[4], const int32_t *ea, const int32_t *eb,
                     int64_t rows, int64_t T, int64_t k, const double *H, const int64_t *targets,
                     double tau, int64_t row0, double *out, int64_t ldo, int pair,
                     cudaStream_t stream) {
  const int nkb = static_cast<int>((k + kO2BK - 1) / kO2BK);
  const unsigned tiles = static_cast<unsigned>((rows + 127) / 128);
  if (pair) {  // a pair's second CTA may hold only out-of-range rows
    // 1: persistent pair (the product path), 2: two pairs sharing A by TMA
    // multicast, 3: one tile per pair (kept for A/B measurements)
    const bool quad = pair == 2, persistent = pair == 1;
    static const int diag = [] {
      const char *e = getenv("PF_K7_DIAG");
      return e ? atoi(e) : 0;
    }();
    using Kern = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, const int32_t *,
                          const int32_t *, int64_t, int64_t, int, const double *, const int64_t *,
                          double, int64_t, double *, int64_t);
    using KernP = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, const int32_t *,
                           const int32_t *, int64_t, int64_t, int, const double *,
                           const int64_t *, double, int64_t, double *, int64_t, int, int);
    Kern kern = quad ? batched_kl_i8_pair_kernel<kS, kMaxL, true>
                     : batched_kl_i8_pair_kernel<kS, kMaxL, false>;
    KernP kernp = diag == 1   ? batched_kl_i8_pp_kernel<kS, kMaxL, 1>
                  : diag == 2 ? batched_kl_i8_pp_kernel<kS, kMaxL, 2>
                  : diag == 3 ? batched_kl_i8_pp_kernel<kS, kMaxL, 3>
                              : batched_kl_i8_pp_kernel<kS, kMaxL, 0>;
    const void *kfn = persistent ? (const void *)kernp : (const void *)kern;
    if (int e = ensure_smem(kfn, kP2Smem)) return e;
    const unsigned ttiles = static_cast<unsigned>((T + kP2BN - 1) / kP2BN);
    const unsigned row_pairs = (tiles + 1) / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(quad ? 4 * ((ttiles + 1) / 2) : 2 * ttiles, row_pairs, 1);
    cfg.blockDim = dim3(kO2Threads, 1, 1);
    cfg.dynamicSmemBytes = kP2Smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = quad ? 4 : 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    const cudaError_t oe = cudaOccupancyMaxActiveClusters(&clusters, kfn, &cfg);
    if (oe != cudaSuccess || clusters == 0) {
      cudaGetLastError();
      return fail(PF_E_LAUNCH, "batched_kl_i8_pair: no CTA pair fits an SM pair (%s, %d)",
                  cudaGetErrorString(oe), clusters);
    }
    cudaError_t le;
    if (persistent) {
      const long long ntiles = static_cast<long long>(row_pairs) * ttiles;
      if (ntiles > INT32_MAX) return fail(PF_E_DOMAIN, "batched_kl_i8_pair: too many tiles");
      const unsigned ncl = static_cast<unsigned>(ntiles < clusters ? ntiles : clusters);
      cfg.gridDim = dim3(2 * ncl, 1, 1);
      le = cudaLaunchKernelEx(&cfg, kernp, m[0], m[1], m[2], m[3], ea, eb, rows, T, nkb, H,
                              targets, tau, row0, out, ldo, static_cast<int>(ttiles),
                              static_cast<int>(ntiles));
    } else {
      le = cudaLaunchKernelEx(&cfg, kern, m[0], m[1], m[2], m[3], ea, eb, rows, T, nkb, H, targets,
                              tau, row0, out, ldo);
    }
    if (le != cudaSuccess)
      return fail(static_cast<int>(le), "batched_kl_i8_pair: %s", cudaGetErrorString(le));
    return check_launch("batched_kl_i8_pair");
  }
  if (int e = ensure_smem((const void *)batched_kl_i8_n128_kernel<kS, kMaxL>, kO2Smem)) return e;
  dim3 grid(static_cast<unsigned>((T + kO2BN - 1) / kO2BN), tiles);
  batched_kl_i8_n128_kernel<kS, kMaxL><<<grid, kO2Threads, kO2Smem, stream>>>(
      m[0], m[1], m[2], m[3], ea, eb, rows, T, nkb, H, targets, tau, row0, out, ldo);
  return check_launch("batched_kl_i8");
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_slice_rows_u8(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                     int64_t ldk, uint8_t *slices, int32_t *exps, pf_stream_t stream) {
  if (rows <= 0) return 0;
  if (!P || !slices || !exps || k <= 0 || ldk < k || ldk % kOzPad)
    return fail(PF_E_ARG, "slice_rows: bad args (ldk %% 64 == 0, ldk >= k)");
  slice_rows_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(P, ld, rows, k, clamp, ldk,
                                                                    slices, exps);
  return check_launch("slice_rows");
}

int pf_slice_targets_u8(const double *L, int64_t ldl, int64_t T, int64_t k, int64_t ldk,
                        uint8_t *slices, int32_t *exps, uint32_t *bad, pf_stream_t stream) {
  if (T <= 0) return 0;
  if (!L || !slices || !exps || k <= 0 || ldk < k || ldk % kOzPad)
    return fail(PF_E_ARG, "slice_targets: bad args (ldk %% 64 == 0, ldk >= k)");
  slice_targets_kernel<<<static_cast<unsigned>(T), 256, 0, as_stream(stream)>>>(
      L, ldl, T, k, ldk, slices, exps, bad);
  return check_launch("slice_targets");
}

int pf_batched_kl_i8(const uint8_t *A, const int32_t *ea, int64_t rows, const uint8_t *B,
                     const int32_t *eb, int64_t T, int64_t k, int64_t ldk, const double *H,
                     const int64_t *targets, double tau, int64_t row0, double *out, int64_t ldo,
                     int grade, int cta_pair, pf_stream_t stream) {
  if (grade != 64 && grade != 32) return fail(PF_E_ARG, "batched_kl_i8: grade must be 64 or 32");
  const int kS = grade == 64 ? kOzSlices : 5;
  if (rows <= 0 || T <= 0) return 0;
  if (!A || !ea || !B || !eb || !H || !targets || !out) return fail(PF_E_ARG, "batched_kl_i8: null");
  if (k > kOzMaxK) return fail(PF_E_DOMAIN, "batched_kl_i8: k = %lld > %d", (long long)k, kOzMaxK);
  if (ldk % kOzPad || ldk < k || ldo < T)
    return fail(PF_E_ALIGN, "batched_kl_i8: ldk %% 64 == 0, ldo >= T");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    return fail(PF_E_ALIGN, "batched_kl_i8: slice planes must be 16-byte aligned");
  const int64_t row_tiles = (rows + 127) / 128;
  if (row_tiles > 65535) return fail(PF_E_DOMAIN, "batched_kl_i8: too many rows per launch");
  if (cta_pair < 0 || cta_pair > 3)
    return fail(PF_E_ARG, "batched_kl_i8: cta_pair must be 0 .. 3");
  const int pair = cta_pair;
  const uint32_t bn = pair ? kP2HalfN : kO2BN;   // each CTA of a pair loads half the targets
  CUtensorMap m[4];
  if (pair == 2) {   // multicast halves: 64-row boxes, one slice each
    if (int e = slice_map(&m[0], A, rows, ldk, 64, kO2BK, 1)) return e;
  } else if (int e = slice_map(&m[0], A, rows, ldk, 128, kO2BK, kS)) {
    return e;
  }
  if (int e = slice_map(&m[1], A, rows, ldk, 128, kO2BK, kO2Pass1Slices)) return e;
  if (int e = slice_map(&m[2], B, T, ldk, bn, kO2BK, kS)) return e;
  if (int e = slice_map(&m[3], B, T, ldk, bn, kO2BK, kO2Pass1Slices)) return e;
  return grade == 64 ? launch_i8<7, 9>(m, ea, eb, rows, T, k, H, targets, tau, row0, out, ldo,
                                       pair, as_stream(stream))
                     : launch_i8<5, 6>(m, ea, eb, rows, T, k, H, targets, tau, row0, out, ldo,
                                       pair, as_stream(stream));
}

int pf_probe_umma_i8(int64_t iters, int random_operands, int64_t *ops_host, uint32_t *sink,
                     pf_stream_t stream) {
  const int smem = (128 + 256) * 64 + 1024;
  if (int e = ensure_smem((const void *)umma_i8_probe_kernel, smem)) return e;
  const int blocks = sm_count();
  umma_i8_probe_kernel<<<blocks, 128, smem, as_stream(stream)>>>(static_cast<int>(iters),
                                                                  random_operands, sink);
  if (ops_host) *ops_host = 2LL * 128 * 256 * 64 * iters * blocks;
  return check_launch("probe_umma_i8");
}

}  // extern "C"
