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
#include <type_traits>

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

// Two layouts of the byte planes.  Row-major: [7][rows][ldk].  Tiled (the
// CTA-pair kernel's): [7][rows / R][nkb][R x 32 B], each R-row x 32-byte K
// block stored as the exact SWIZZLE_32B shared-memory image the MMA reads
// (16-byte chunk c of row r at r * 32 + (c ^ (r >> 2 & 1)) * 16), so one
// stage of one slice is one contiguous 4 KB (R = 128) or 2 KB (R = 64) run
// and the TMA box is {256 B, R / 8, slices} with 256-byte rows instead of R
// 32-byte rows: 53 B/clk/SM from L2 and the full HBM rate, against 32 and 6
// for the row-major box (tools/probe_umma_shapes.cu tma_rate).
struct SliceLayout {
  int64_t ldk;    // row-major pitch (0: tiled)
  int tile_rows;  // tiled: R
  int nkb;        // tiled: 32-byte K blocks per row
  __device__ __forceinline__ int64_t at(int64_t r, int64_t b0) const {   // b0 % 8 == 0
    if (ldk) return r * ldk + b0;
    return ((r / tile_rows) * nkb + (b0 >> 5)) * (tile_rows * 32) + (r % tile_rows) * 32 +
           ((((b0 >> 4) & 1) ^ ((r >> 2) & 1)) << 4) + (b0 & 15);
  }
  __device__ __forceinline__ int64_t kspan() const { return ldk ? ldk : int64_t(nkb) * 32; }
};

// Rows of the slab: a = max(P, clamp), warp per row; rows in [rows, rows_pad)
// are written as zeros (tiled padding).
__global__ void __launch_bounds__(256) slice_rows_kernel(const double *__restrict__ P, int64_t ld,
                                                         int64_t rows, int64_t rows_pad, int64_t k,
                                                         double clamp, SliceLayout lay,
                                                         int64_t plane, uint8_t *__restrict__ out,
                                                         int32_t *__restrict__ exps) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t span = lay.kspan();
  for (int64_t r = warp; r < rows_pad; r += nwarps) {
    const bool live = r < rows;
    const double *row = P + (live ? r : 0) * ld;
    double m = 0.0;
    if (live) {
      for (int64_t b = lane; b < k; b += 32) m = fmax(m, fmax(row[b], clamp));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    const int e = scale_exp(m);
    if (live && lane == 0) exps[r] = e;
    for (int64_t b0 = 8 * lane; b0 < span; b0 += 256) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = (live && b0 + u < k) ? fmax(row[b0 + u], clamp) : 0.0;
      uint64_t w[kOzSlices];
      slice8(x, e, w);
      const int64_t o = lay.at(r, b0);
#pragma unroll
      for (int s = 0; s < kOzSlices; ++s) *reinterpret_cast<uint64_t *>(out + s * plane + o) = w[s];
    }
  }
}

// Targets: b = -L (L = log max(Pt, clamp), batch_prep_kernel), block per
// target.  bad[0] |= 1 if some b < 0 (a target entry above 1: the caller then
// uses the FP64 path).  slices: [7][T][ldk].
// Blocks t in [T, gridDim.x) write the zero padding of the tiled layout.
__global__ void __launch_bounds__(256) slice_targets_kernel(const double *__restrict__ L,
                                                            int64_t ldl, int64_t T, int64_t k,
                                                            SliceLayout lay, int64_t plane,
                                                            uint8_t *__restrict__ out,
                                                            int32_t *__restrict__ exps,
                                                            uint32_t *__restrict__ bad) {
  const int64_t t = blockIdx.x;
  const bool live = t < T;
  const double *row = L + (live ? t : 0) * ldl;
  __shared__ double red[8];
  double m = 0.0;
  bool neg = false;
  for (int64_t b = threadIdx.x; live && b < k; b += blockDim.x) {
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
  if (live && threadIdx.x == 0) {
    exps[t] = e;
    // the pair kernel's epilogue packs eb + 64 into a byte (-L is 0 or
    // >= 2^-53, so eb >= -52 for any P <= 1; a target above that range is
    // a target row with an entry above 1 anyway)
    if ((neg || e < -64 || e > 191) && bad) atomicOr(bad, 1u);
  }
  const int64_t span = lay.kspan();
  for (int64_t b0 = 8 * threadIdx.x; b0 < span; b0 += 8 * blockDim.x) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = (live && b0 + u < k) ? fmax(-row[b0 + u], 0.0) : 0.0;
    uint64_t w[kOzSlices];
    slice8(x, e, w);
    const int64_t o = lay.at(t, b0);
#pragma unroll
    for (int s = 0; s < kOzSlices; ++s) *reinterpret_cast<uint64_t *>(out + s * plane + o) = w[s];
  }
}

// ldexp(v, e) for the Ozaki sums v (0 or within [2^-64, 2^64]), branch-free:
// v * 2^e1 is exact (normal, |e1| <= 900), the second power-of-two multiply
// rounds once -- the single rounding ldexp does; |e| beyond 1922 gives 0 or
// inf either way.
__device__ __forceinline__ double pow2_exact(int e) {   // 2^e, -1022 <= e <= 1023
  return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}
__device__ __forceinline__ double pow2_scale(double v, int e) {
  e = max(-1922, min(1922, e));
  const int e1 = max(-900, min(900, e));
  return (v * pow2_exact(e1)) * pow2_exact(e - e1);
}

// The epilogue value of one (row, target) from S = v 2^e >= 0: the split
// form h + S, or the guard sentinel when |h + S| < tau (|h| + S) (evaluated
// as fma(tau, S, tau |h|) -- two FP64 instructions per element in all: FP64
// issue is starved while the int8 MMAs run, ~5x slower than with the tensor
// pipe idle, measured by the stage stamps), settled, or 0 at the target.
// settle and the guard compare are integer compares of the bit patterns
// (same results as the FP64 forms for every input: the operands are finite
// and the magnitude bits of doubles order like the values).
__device__ __forceinline__ double k7_value(double S, double h, double tau, double tau_h, bool is_t,
                                           bool &guard) {
  const double val = h + S;
  const double thr = fma(tau, S, tau_h);
  // magnitude bits from the 32-bit halves (a 64-bit mask of the sign bit
  // would be folded back into an FP64 |x|)
  const int hi = __double2hiint(val);
  const unsigned lo = static_cast<unsigned>(__double2loint(val));
  const long long mag = (static_cast<long long>(hi & 0x7fffffff) << 32) | lo;
  guard = !is_t && mag < __double_as_longlong(thr);
  const bool noise = hi < 0 && mag != 0 && mag < __double_as_longlong(kNegNoise);   // settle()
  return guard ? __longlong_as_double(static_cast<long long>(kOzGuard))
               : ((is_t || noise) ? 0.0 : val);
}

// RNE((a0 2^24 + a1 2^16 + a2 2^8 + a3) 2^-24) for the s32 (non-negative)
// level accumulators of one pass: the same value as the FP64 chain
// x = a3; x = fma(x, 2^-8, a_l) for l = 2, 1, 0 (whose first two steps are
// exact, so it rounds once), from one 64-bit integer sum split into two
// exactly representable halves: 3 FP64 adds instead of 4 s32->f64
// conversions (4x slower than an add) and 3 FMAs.
__device__ __forceinline__ double levels4_f64(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
  const unsigned long long X = static_cast<unsigned long long>(a3) +
                               (static_cast<unsigned long long>(a2) << 8) +
                               (static_cast<unsigned long long>(a1) << 16) +
                               (static_cast<unsigned long long>(a0) << 24);   // < 2^56
  const double dh = __hiloint2double(0x43B00000, static_cast<int>(X >> 32)) - 0x1p60;   // Xh 2^8
  const double dl = __hiloint2double(0x41B00000, static_cast<int>(static_cast<uint32_t>(X))) -
                    0x1p28;   // Xl 2^-24
  return dh + dl;
}
__device__ __forceinline__ double u32_f64(uint32_t a) {   // exact
  return __hiloint2double(0x43300000, static_cast<int>(a)) - 0x1p52;
}

// v 2^e for v = 0 or within [2^-64, 2^64] and e within [-958, 959]: the
// exponent field moves, exactly (the result is normal).
__device__ __forceinline__ double pow2_scale_normal(double v, int e) {
  const long long b = __double_as_longlong(v);
  const int hi = static_cast<int>(b >> 32);
  return hi == 0 ? 0.0 : __hiloint2double(hi + (e << 20), static_cast<int>(b));
}
__device__ __forceinline__ double k7_scale(double v, int e) {   // == pow2_scale
  return (e >= -958 && e <= 959) ? pow2_scale_normal(v, e) : pow2_scale(v, e);
}

// Append the guarded (q, t) pairs of one thread's columns to the fixup list
// (list[0] = count, then q * T + t; entries past cap are dropped and the
// fixup falls back to scanning the output for sentinels).
__device__ __forceinline__ void push_guards(int64_t *list, int64_t cap, uint64_t mask, int64_t q,
                                            int64_t t0, int64_t T) {
  if (list == nullptr || mask == 0) return;
  const int n = __popcll(mask);
  const int64_t base = static_cast<int64_t>(
      atomicAdd(reinterpret_cast<unsigned long long *>(list), static_cast<unsigned long long>(n)));
  int j = 0;
  while (mask) {
    const int c = __ffsll(static_cast<long long>(mask)) - 1;
    mask &= mask - 1;
    if (base + j < cap) list[1 + base + j] = q * T + t0 + c;
    ++j;
  }
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
    int64_t row0, double *__restrict__ out, int64_t ldo, int64_t *guard_list, int64_t guard_cap) {
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
    uint64_t gmask = 0;
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
        const double S = k7_scale(v, e_q + eb[t] - 16);
        bool guard;
        const double val = k7_value(S, h, tau, tau * fabs(h), tq == targets[t], guard);
        if (guard) gmask |= 1ull << (c0 + u);
        out[q * ldo + t] = val;
      }
    }
    push_guards(guard_list, guard_cap, gmask, q, t0 + half * 64, T);
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

// ------------------------------------------------ GEMM, persistent CTA pair --
// The same two-pass level schedule on persistent CTA pairs (tcgen05
// cta_group::2, one cluster of 2 per SM pair, tiles strided over the
// clusters; consecutive clusters share a row pair so its A planes stream
// from HBM once and hit L2 after).  The leader issues M256 N128 K32 MMAs
// whose A rows 0-127 come from its own shared memory and 128-255 from the
// peer's, and whose B (the 128 targets) is split 64 / 64 between the two;
// each CTA's TMEM gets its own 128 rows.  Per SM and MMA the tensor pipe
// reads 4 KB of A + 2 KB of B instead of 4 + 4 KB.  The epilogue is off the
// tensor pipe's critical path: the epilogue warps fold the pass-2
// accumulators into the FP64 pass-1 partials in registers, release TMEM
// (free_bar), and only then scale / guard / settle / store while the next
// tile's pass-1 MMAs run.  Same integers, same FP64 operation order: bitwise
// the 1-CTA kernel's outputs.  5-stage ring of 42 KB per CTA.
//
// kDiag (timing diagnostics only, PF_K7_DIAG, wrong outputs): bit 0 = no TMA
// loads (the MMAs run on stale shared memory), bit 1 = no epilogue arithmetic
// or stores, bit 2 = SM-clock phase stamps of cluster 0 per tile k at
// out[k * 16 + i] (tools/probe_k7pp_stamps.py), bit 3 = per-stage timeline of
// cluster 0's leader in SM clocks (%globaltimer ticks too coarsely for
// stage-sized gaps): load issue at out[65536 + 2 s], full-barrier pass at
// out[65536 + 2 s + 1] (tools/probe_k7stages.py), bit 4 = the element loop
// without its stores, bit 5 = no MMAs (commits only; with bit 2: how fast the
// epilogue runs when the tensor pipe is idle).  kTiled: operands in the tiled
// layout (SliceLayout), the default; the row-major form stays for the
// pf_batched_kl_i8 ABI.
constexpr int kP2BN = 128, kP2HalfN = 64, kP2Stages = 5;
constexpr int kP2TileA = 128 * kO2BK;                         // 4 KB per slice
constexpr int kP2TileB = kP2HalfN * kO2BK;                    // 2 KB per slice
constexpr int kP2StageBytes = kOzSlices * (kP2TileA + kP2TileB);  // 43,008
constexpr int kP2Smem = kP2Stages * kP2StageBytes + 1024;

template <int kS, int kMaxL, int kDiag = 0, bool kTiled = false>
__global__ void __launch_bounds__(kO2Threads, 1)
    batched_kl_i8_pp_kernel(const __grid_constant__ CUtensorMap mapA7,
                            const __grid_constant__ CUtensorMap mapA4,
                            const __grid_constant__ CUtensorMap mapB7,
                            const __grid_constant__ CUtensorMap mapB4,
                            const int32_t *__restrict__ ea, const int32_t *__restrict__ eb,
                            int64_t rows, int64_t T, int nkb, const double *__restrict__ H,
                            const int64_t *__restrict__ targets, double tau, int64_t row0,
                            double *__restrict__ out, int64_t ldo, int t_tiles, int ntiles,
                            int64_t *guard_list, int64_t guard_cap) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full_bar[kP2Stages], empty_bar[kP2Stages];
  __shared__ __align__(8) uint64_t pass_bar[2], drained_bar, free_bar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();   // 0 = leader (issues the MMAs)
  const int cid = static_cast<int>(blockIdx.x >> 1), ncl = static_cast<int>(gridDim.x >> 1);
  // tile w: row pair w / t_tiles, target tile w % t_tiles
  // kDiag & 4: SM-clock stamps of cluster 0's leader, per tile k, at out[k * 16 + i]
  const bool stamping = (kDiag & 4) != 0 && blockIdx.x == 0;
#define PP_STAMP(k, i) \
  do {                 \
    if (stamping) out[(k) * 16 + (i)] = static_cast<double>(clock64()); \
  } while (0)

  if (tid == 0) {
    tc::prefetch_map(&mapA7);
    tc::prefetch_map(&mapA4);
    tc::prefetch_map(&mapB7);
    tc::prefetch_map(&mapB4);
    for (int s = 0; s < kP2Stages; ++s) {
      mbar_init(&full_bar[s], 1);    // the leader's producer arrives (both CTAs' bytes)
      mbar_init(&empty_bar[s], 1);   // one multicast MMA commit
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
      // ---- TMA producer (both CTAs): own 128 A rows, own half of the targets.
      // Every pass starts at ring slot 0 (slots left over at a pass end are
      // skipped), so the MMA loop below can be unrolled over the ring with
      // compile-time slot addresses; per-slot phases live in `ph`.
      uint32_t ph = 0;
      int gstage = 0;
      for (int w = cid; w < ntiles; w += ncl) {
        const int64_t q0 = (static_cast<int64_t>(w / t_tiles) * 2 + rank) * 128;
        const int32_t tb = (w % t_tiles) * kP2BN + static_cast<int32_t>(rank) * kP2HalfN;
        for (int pass = 0; pass < 2; ++pass) {
          const int ns = pass == 0 ? kO2Pass1Slices : kS;
          const CUtensorMap *ma = pass == 0 ? &mapA4 : &mapA7;
          const CUtensorMap *mb = pass == 0 ? &mapB4 : &mapB7;
          for (int kb0 = 0; kb0 < nkb; kb0 += kP2Stages) {
#pragma unroll
            for (int st = 0; st < kP2Stages; ++st) {
              const int kb = kb0 + st;
              if (kb >= nkb) break;
              mbar_wait(&empty_bar[st], ((ph >> st) & 1) ^ 1);
              ph ^= 1u << st;
              if constexpr ((kDiag & 8) != 0) {   // stage timeline of cluster 0's leader
                if (blockIdx.x == 0 && gstage < 4096)
                  out[65536 + 2 * gstage] = static_cast<double>(clock64());
                ++gstage;
              }
              if constexpr ((kDiag & 1) != 0) {
                if (rank == 0) mbar_arrive(&full_bar[st]);
                continue;
              }
              uint8_t *sa = smem + st * kP2StageBytes;
              uint8_t *sb = sa + kOzSlices * kP2TileA;
              if (rank == 0) mbar_expect_tx(&full_bar[st], 2 * ns * (kP2TileA + kP2TileB));
              const uint32_t lb = tc::mapa(&full_bar[st], 0);
              if constexpr (kTiled) {   // 256-byte box rows: 16 per A tile, 8 per B tile
                tc::tma_load_3d_pair(sa, ma, 0, static_cast<int32_t>((q0 / 128 * nkb + kb) * 16),
                                     0, lb);
                tc::tma_load_3d_pair(sb, mb, 0, (tb / kP2HalfN * nkb + kb) * 8, 0, lb);
              } else {
                tc::tma_load_3d_pair(sa, ma, kb * kO2BK, static_cast<int32_t>(q0), 0, lb);
                tc::tma_load_3d_pair(sb, mb, kb * kO2BK, tb, 0, lb);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---- MMA issuer (leader only): M256 N128 K32.  The tensor pipe keeps
      // almost no queue of its own, so whatever this thread does between two
      // MMAs beyond the executing MMA's 64 clocks is a pipe bubble: each pass
      // is its own loop (a conditional commit inside a shared loop costs a
      // stall per stage), and the ring is unrolled so that the descriptors
      // after each full-barrier wait are compile-time offsets of uniform
      // registers (a runtime slot address put an R2UR chain behind every wait:
      // ~145 clocks per stage, measured by tools/probe_umma_shapes.cu).
      constexpr uint32_t idesc = tc::idesc_i8(256, kP2BN, false, false);
      const uint32_t ring = smem_u32(smem);
      uint32_t ph = 0;
      int k = 0, mstage = 0;
      for (int w = cid; w < ntiles; w += ncl, ++k) {
        PP_STAMP(k, 0);
        if (k > 0) {   // the previous tile's pass-2 accumulators drained
          mbar_wait(&free_bar, (k - 1) & 1);
          tc::fence_after();
        }
        PP_STAMP(k, 1);
        for (int kb0 = 0; kb0 < nkb; kb0 += kP2Stages) {
#pragma unroll
          for (int st = 0; st < kP2Stages; ++st) {
            const int kb = kb0 + st;
            if (kb >= nkb) break;
            mbar_wait(&full_bar[st], (ph >> st) & 1);
            ph ^= 1u << st;
            if constexpr ((kDiag & 8) != 0) {
              if (blockIdx.x == 0 && mstage < 4096)
                out[65536 + 2 * mstage + 1] = static_cast<double>(clock64());
              ++mstage;
            }
            tc::fence_after();
            const uint32_t sa = ring + st * kP2StageBytes;
            const uint32_t sb = sa + kOzSlices * kP2TileA;
#pragma unroll
            for (int i = 1; i <= kO2Pass1Slices; ++i)
#pragma unroll
              for (int j = 1; j <= kO2Pass1Slices; ++j) {
                const int l = i + j;
                if (l > 5) continue;
                if constexpr ((kDiag & 32) != 0) continue;   // no MMAs (commits only)
                // A_i serves j = 1 .. 5 - i back to back: read it once (collector)
                const int jl = 5 - i;
                const int coll = jl == 1 ? 0 : (j == 1 ? 1 : (j == jl ? 3 : 2));
                const uint64_t ad = tc::sdesc<32>(sa + (i - 1) * kP2TileA);
                const uint64_t bd = tc::sdesc<32>(sb + (j - 1) * kP2TileB);
                const bool acc = !(kb == 0 && i == 1);
                if (coll == 1) tc::mma_i8_pair_c<1>(tmem + (l - 2) * kP2BN, ad, bd, idesc, acc);
                else if (coll == 2) tc::mma_i8_pair_c<2>(tmem + (l - 2) * kP2BN, ad, bd, idesc, acc);
                else if (coll == 3) tc::mma_i8_pair_c<3>(tmem + (l - 2) * kP2BN, ad, bd, idesc, acc);
                else tc::mma_i8_pair(tmem + (l - 2) * kP2BN, ad, bd, idesc, acc);
              }
            tc::commit_pair(&empty_bar[st]);
          }
        }
        tc::commit_pair(&pass_bar[0]);
        PP_STAMP(k, 2);
        mbar_wait(&drained_bar, k & 1);   // pass 2 reuses the accumulators
        tc::fence_after();
        PP_STAMP(k, 3);
        for (int kb0 = 0; kb0 < nkb; kb0 += kP2Stages) {
#pragma unroll
          for (int st = 0; st < kP2Stages; ++st) {
            const int kb = kb0 + st;
            if (kb >= nkb) break;
            mbar_wait(&full_bar[st], (ph >> st) & 1);
            ph ^= 1u << st;
            if constexpr ((kDiag & 8) != 0) {
              if (blockIdx.x == 0 && mstage < 4096)
                out[65536 + 2 * mstage + 1] = static_cast<double>(clock64());
              ++mstage;
            }
            tc::fence_after();
            const uint32_t sa = ring + st * kP2StageBytes;
            const uint32_t sb = sa + kOzSlices * kP2TileA;
#pragma unroll
            for (int i = 1; i <= kS; ++i)
#pragma unroll
              for (int j = 1; j <= kS; ++j) {
                const int l = i + j;
                if (l < 6 || l > kMaxL) continue;
                if constexpr ((kDiag & 32) != 0) continue;
                const int first_i = l - kS > 1 ? l - kS : 1;
                const int jf = 6 - i > 1 ? 6 - i : 1, jl = kMaxL - i < kS ? kMaxL - i : kS;
                const int coll = jl == jf ? 0 : (j == jf ? 1 : (j == jl ? 3 : 2));
                const uint64_t ad = tc::sdesc<32>(sa + (i - 1) * kP2TileA);
                const uint64_t bd = tc::sdesc<32>(sb + (j - 1) * kP2TileB);
                const bool acc = !(kb == 0 && i == first_i);
                if (coll == 1) tc::mma_i8_pair_c<1>(tmem + (l - 6) * kP2BN, ad, bd, idesc, acc);
                else if (coll == 2) tc::mma_i8_pair_c<2>(tmem + (l - 6) * kP2BN, ad, bd, idesc, acc);
                else if (coll == 3) tc::mma_i8_pair_c<3>(tmem + (l - 6) * kP2BN, ad, bd, idesc, acc);
                else tc::mma_i8_pair(tmem + (l - 6) * kP2BN, ad, bd, idesc, acc);
              }
            tc::commit_pair(&empty_bar[st]);
          }
        }
        tc::commit_pair(&pass_bar[1]);
        PP_STAMP(k, 4);
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
      if (tid == 64) PP_STAMP(k, 5);
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 4) {   // x4 chunks: v[64] + acc stay in 168 registers
        uint32_t acc[4][4];
#pragma unroll
        for (int l = 0; l < 4; ++l) tc::tmem_ld4(base + l * kP2BN + c0, acc[l]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u) v[c0 + u] = levels4_f64(acc[0][u], acc[1][u], acc[2][u], acc[3][u]);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(drained_leader);
      if (tid == 64) PP_STAMP(k, 6);
      mbar_wait(&pass_bar[1], k & 1);
      tc::fence_after();
      if (tid == 64) PP_STAMP(k, 7);
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 4) {
        uint32_t acc[kL2][4];
#pragma unroll
        for (int l = 0; l < kL2; ++l) tc::tmem_ld4(base + l * kP2BN + c0, acc[l]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          static_assert(kL2 == 4 || kL2 == 1, "pass-2 level count");
          const double x = kL2 == 4 ? levels4_f64(acc[0][u], acc[1][u], acc[2][u], acc[kL2 - 1][u])
                                    : u32_f64(acc[0][u]);
          v[c0 + u] = fma(x, 0x1p-32, v[c0 + u]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(free_leader);   // TMEM free for the next tile
      if (tid == 64) PP_STAMP(k, 8);
      if constexpr ((kDiag & 2) != 0) continue;
      // The element loop runs while the next tile's pass-1 MMAs do, and FP64
      // instructions issue ~5x slower then (PF_K7_DIAG=36 runs the loop without
      // MMAs: 21K against 103K clocks per tile), so it keeps two FP64
      // instructions per element (h + S and fma(tau, S, tau |h|), k7_value) and
      // no per-element shared-memory or shuffle traffic.  Per tile:
      //  * the 64 column exponents eb are loaded with 16-byte loads and packed
      //    as bytes eb + 64, 32 columns (8 registers) per half of the loop;
      //  * the columns whose target is this lane's row form a mask built from
      //    ballots over the owner-lane bits (at most one row per column);
      //  * S = v 2^(ea + eb - 16) moves the exponent field (exact: v is 0 or
      //    within [2^-64, 2^64], eb within [-52, 12] -- -L is 0 or >= 2^-53,
      //    and the slicing flags anything outside [-64, 191] as bad), rows
      //    whose exponents could leave the normal range take pow2_scale.
      auto pack4 = [](int a, int b, int c, int d) -> uint32_t {
        return (static_cast<uint32_t>(a + 64) & 255u) | ((static_cast<uint32_t>(b + 64) & 255u) << 8) |
               ((static_cast<uint32_t>(c + 64) & 255u) << 16) | (static_cast<uint32_t>(d + 64) << 24);
      };
      const bool eb_vec = tc0 + 64 <= T && (reinterpret_cast<uintptr_t>(eb) & 15) == 0;
      // 8 packed registers of 32 column exponents (the loop runs in two
      // halves so that v[64] + these fit the 168-register budget of 10 warps)
      auto load_eb = [&](int c0, uint32_t (&ebp)[8]) {
        if (eb_vec) {
          const int4 *ev = reinterpret_cast<const int4 *>(eb + tc0 + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int4 e4 = __ldg(ev + j);
            ebp[j] = pack4(e4.x, e4.y, e4.z, e4.w);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            int e4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int64_t tt = tc0 + c0 + 4 * j + u;
              e4[u] = tt < T ? eb[tt] : 0;
            }
            ebp[j] = pack4(e4[0], e4[1], e4[2], e4[3]);
          }
        }
      };
      const long long qw = row0 + q - lane;   // global row of this warp's lane 0
      const int64_t tA = tc0 + lane, tB = tc0 + 32 + lane;
      const long long oA = tA < T ? targets[tA] - qw : -1, oB = tB < T ? targets[tB] - qw : -1;
      uint32_t tmA = __ballot_sync(0xffffffffu, oA >= 0 && oA < 32);
      uint32_t tmB = __ballot_sync(0xffffffffu, oB >= 0 && oB < 32);
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        const uint32_t bA = __ballot_sync(0xffffffffu, (oA >> b) & 1);
        const uint32_t bB = __ballot_sync(0xffffffffu, (oB >> b) & 1);
        tmA &= ((lane >> b) & 1) ? bA : ~bA;
        tmB &= ((lane >> b) & 1) ? bB : ~bB;
      }
      const bool row_ok = q < rows;
      const double h = row_ok ? H[q] : 0.0;
      const double tau_h = tau * fabs(h);
      const int e_q = (row_ok ? ea[q] : 0) - 16;   // S = v 2^(e_q + eb), eb + 64 in a byte
      // every element of the row scales by moving the exponent field
      const bool fast = __all_sync(0xffffffffu, e_q - 64 >= -958 && e_q + 191 <= 959);
      double *orow = out + q * ldo + tc0;
      const bool full = row_ok && pairs_ok && tc0 + 64 <= T;
      uint32_t gm[2] = {0u, 0u};
      // two copies of the loop: the exponent-field scale (every row of the
      // warp in range, the rule) and pow2_scale
      auto columns = [&](auto fast_c) {
        constexpr bool kFast = decltype(fast_c)::value;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t ebp[8];
          load_eb(32 * hh, ebp);
          const uint32_t tm = hh ? tmB : tmA;
          auto element = [&](int cl) -> double {   // column 32 hh + cl
            const int cc = 32 * hh + cl;
            const int e = e_q - 64 + static_cast<int>((ebp[cl >> 2] >> (8 * (cl & 3))) & 255u);
            const double S = kFast ? pow2_scale_normal(v[cc], e) : pow2_scale(v[cc], e);
            bool guard;
            const double o = k7_value(S, h, tau, tau_h, (tm >> cl) & 1, guard);
            gm[hh] |= static_cast<uint32_t>(guard) << cl;
            return o;
          };
          if constexpr ((kDiag & 16) != 0) {   // the element math without the stores
            double x = 0.0;
#pragma unroll
            for (int c = 0; c < 32; ++c) x += element(c);
            if (x == 1.2345) orow[0] = x;
            continue;
          }
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const double o0 = element(c), o1 = element(c + 1);
            const int cc = 32 * hh + c;
            if (full) {
              *reinterpret_cast<double2 *>(orow + cc) = make_double2(o0, o1);
            } else if (row_ok) {
              if (tc0 + cc < T) orow[cc] = o0;
              if (tc0 + cc + 1 < T) orow[cc + 1] = o1;
            }
          }
        }
      };
      if (fast)
        columns(std::true_type{});
      else
        columns(std::false_type{});
      const uint64_t gmask = gm[0] | (static_cast<uint64_t>(gm[1]) << 32);
      if (row_ok) push_guards(guard_list, guard_cap, gmask, q, tc0, T);
      if (tid == 64) PP_STAMP(k, 9);
    }
  }
#undef PP_STAMP
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

// 3-D u8 map over a tiled layout [7][units][256 B]: box {256, box_units,
// box_slices}, no swizzle (the bytes already are the swizzled image).
static int tiled_map(CUtensorMap *map, const uint8_t *base, int64_t units, uint32_t box_units,
                     uint32_t box_slices) {
  auto fn = encode_fn();
  if (!fn) return fail(PF_E_LAUNCH, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {256, static_cast<cuuint64_t>(units), static_cast<cuuint64_t>(kOzSlices)};
  cuuint64_t strides[2] = {256, static_cast<cuuint64_t>(units * 256)};
  cuuint32_t box[3] = {256, box_units, box_slices};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PF_E_ARG, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

template <int kS, int kMaxL, bool kTiled>
static auto pp_kernel(int diag) {
  return diag == 1    ? batched_kl_i8_pp_kernel<kS, kMaxL, 1, kTiled>
         : diag == 2  ? batched_kl_i8_pp_kernel<kS, kMaxL, 2, kTiled>
         : diag == 3  ? batched_kl_i8_pp_kernel<kS, kMaxL, 3, kTiled>
         : diag == 4  ? batched_kl_i8_pp_kernel<kS, kMaxL, 4, kTiled>
         : diag == 10 ? batched_kl_i8_pp_kernel<kS, kMaxL, 10, kTiled>
         : diag == 20 ? batched_kl_i8_pp_kernel<kS, kMaxL, 20, kTiled>
         : diag == 36 ? batched_kl_i8_pp_kernel<kS, kMaxL, 36, kTiled>
                      : batched_kl_i8_pp_kernel<kS, kMaxL, 0, kTiled>;
}

template <int kS, int kMaxL, bool kTiled = false>
static int launch_i8(const CUtensorMap (&m)[4], const int32_t *ea, const int32_t *eb,
                     int64_t rows, int64_t T, int64_t k, const double *H, const int64_t *targets,
                     double tau, int64_t row0, double *out, int64_t ldo, bool pair,
                     int64_t *glist, int64_t gcap, cudaStream_t stream) {
  const int nkb = static_cast<int>((k + kO2BK - 1) / kO2BK);
  const unsigned tiles = static_cast<unsigned>((rows + 127) / 128);
  if (pair) {  // a pair's second CTA may hold only out-of-range rows
    static const int diag = [] {
      const char *e = getenv("PF_K7_DIAG");
      return e ? atoi(e) : 0;
    }();
    auto kern = pp_kernel<kS, kMaxL, kTiled>(diag);
    if (int e = ensure_smem((const void *)kern, kP2Smem)) return e;
    const unsigned ttiles = static_cast<unsigned>((T + kP2BN - 1) / kP2BN);
    const unsigned row_pairs = (tiles + 1) / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2, 1, 1);   // for the occupancy query
    cfg.blockDim = dim3(kO2Threads, 1, 1);
    cfg.dynamicSmemBytes = kP2Smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    const cudaError_t oe = cudaOccupancyMaxActiveClusters(&clusters, (const void *)kern, &cfg);
    if (oe != cudaSuccess || clusters == 0) {
      cudaGetLastError();
      return fail(PF_E_LAUNCH, "batched_kl_i8_pair: no CTA pair fits an SM pair (%s, %d)",
                  cudaGetErrorString(oe), clusters);
    }
    const long long ntiles = static_cast<long long>(row_pairs) * ttiles;
    if (ntiles > INT32_MAX) return fail(PF_E_DOMAIN, "batched_kl_i8_pair: too many tiles");
    const unsigned ncl = static_cast<unsigned>(ntiles < clusters ? ntiles : clusters);
    cfg.gridDim = dim3(2 * ncl, 1, 1);
    const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, m[0], m[1], m[2], m[3], ea, eb, rows, T,
                                              nkb, H, targets, tau, row0, out, ldo,
                                              static_cast<int>(ttiles), static_cast<int>(ntiles),
                                              glist, gcap);
    if (le != cudaSuccess)
      return fail(static_cast<int>(le), "batched_kl_i8_pair: %s", cudaGetErrorString(le));
    return check_launch("batched_kl_i8_pair");
  }
  if (int e = ensure_smem((const void *)batched_kl_i8_n128_kernel<kS, kMaxL>, kO2Smem)) return e;
  dim3 grid(static_cast<unsigned>((T + kO2BN - 1) / kO2BN), tiles);
  batched_kl_i8_n128_kernel<kS, kMaxL><<<grid, kO2Threads, kO2Smem, stream>>>(
      m[0], m[1], m[2], m[3], ea, eb, rows, T, nkb, H, targets, tau, row0, out, ldo, glist, gcap);
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
  slice_rows_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(
      P, ld, rows, rows, k, clamp, SliceLayout{ldk, 0, 0}, rows * ldk, slices, exps);
  return check_launch("slice_rows");
}

int64_t pf_i8_tiled_bytes(int64_t n, int64_t k) {
  if (n <= 0 || k <= 0) return 0;
  return int64_t(kOzSlices) * ((n + 127) / 128 * 128) * ((k + kO2BK - 1) / kO2BK * kO2BK);
}

int pf_slice_rows_u8_tiled(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                           uint8_t *tiles, int32_t *exps, pf_stream_t stream) {
  if (rows <= 0) return 0;
  if (!P || !tiles || !exps || k <= 0 || ld < k)
    return fail(PF_E_ARG, "slice_rows_tiled: bad args");
  if (reinterpret_cast<uintptr_t>(tiles) & 15)
    return fail(PF_E_ALIGN, "slice_rows_tiled: tiles must be 16-byte aligned");
  const int nkb = static_cast<int>((k + kO2BK - 1) / kO2BK);
  const int64_t rows_pad = (rows + 127) / 128 * 128;
  slice_rows_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(
      P, ld, rows, rows_pad, k, clamp, SliceLayout{0, 128, nkb}, pf_i8_tiled_bytes(rows, k) / 7,
      tiles, exps);
  return check_launch("slice_rows_tiled");
}

int pf_slice_targets_u8(const double *L, int64_t ldl, int64_t T, int64_t k, int64_t ldk,
                        uint8_t *slices, int32_t *exps, uint32_t *bad, pf_stream_t stream) {
  if (T <= 0) return 0;
  if (!L || !slices || !exps || k <= 0 || ldk < k || ldk % kOzPad)
    return fail(PF_E_ARG, "slice_targets: bad args (ldk %% 64 == 0, ldk >= k)");
  slice_targets_kernel<<<static_cast<unsigned>(T), 256, 0, as_stream(stream)>>>(
      L, ldl, T, k, SliceLayout{ldk, 0, 0}, T * ldk, slices, exps, bad);
  return check_launch("slice_targets");
}

int pf_slice_targets_u8_tiled(const double *L, int64_t ldl, int64_t T, int64_t k, uint8_t *tiles,
                              int32_t *exps, uint32_t *bad, pf_stream_t stream) {
  if (T <= 0) return 0;
  if (!L || !tiles || !exps || k <= 0 || ldl < k)
    return fail(PF_E_ARG, "slice_targets_tiled: bad args");
  if (reinterpret_cast<uintptr_t>(tiles) & 15)
    return fail(PF_E_ALIGN, "slice_targets_tiled: tiles must be 16-byte aligned");
  const int nkb = static_cast<int>((k + kO2BK - 1) / kO2BK);
  const int64_t T_pad = (T + 127) / 128 * 128;
  slice_targets_kernel<<<static_cast<unsigned>(T_pad), 256, 0, as_stream(stream)>>>(
      L, ldl, T, k, SliceLayout{0, kP2HalfN, nkb}, pf_i8_tiled_bytes(T, k) / 7, tiles, exps, bad);
  return check_launch("slice_targets_tiled");
}

int pf_batched_kl_i8(const uint8_t *A, const int32_t *ea, int64_t rows, const uint8_t *B,
                     const int32_t *eb, int64_t T, int64_t k, int64_t ldk, const double *H,
                     const int64_t *targets, double tau, int64_t row0, double *out, int64_t ldo,
                     int grade, int cta_pair, pf_stream_t stream) {
  return pf_batched_kl_i8_listed(A, ea, rows, B, eb, T, k, ldk, H, targets, tau, row0, out, ldo,
                                 grade, cta_pair, nullptr, 0, stream);
}

int pf_batched_kl_i8_listed(const uint8_t *A, const int32_t *ea, int64_t rows, const uint8_t *B,
                            const int32_t *eb, int64_t T, int64_t k, int64_t ldk, const double *H,
                            const int64_t *targets, double tau, int64_t row0, double *out,
                            int64_t ldo, int grade, int cta_pair, int64_t *guard_list,
                            int64_t guard_cap, pf_stream_t stream) {
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
  const bool pair = cta_pair != 0;
  const uint32_t bn = pair ? kP2HalfN : kO2BN;   // each CTA of a pair loads half the targets
  CUtensorMap m[4];
  if (int e = slice_map(&m[0], A, rows, ldk, 128, kO2BK, kS)) return e;
  if (int e = slice_map(&m[1], A, rows, ldk, 128, kO2BK, kO2Pass1Slices)) return e;
  if (int e = slice_map(&m[2], B, T, ldk, bn, kO2BK, kS)) return e;
  if (int e = slice_map(&m[3], B, T, ldk, bn, kO2BK, kO2Pass1Slices)) return e;
  return grade == 64 ? launch_i8<7, 9>(m, ea, eb, rows, T, k, H, targets, tau, row0, out, ldo,
                                       pair, guard_list, guard_cap, as_stream(stream))
                     : launch_i8<5, 6>(m, ea, eb, rows, T, k, H, targets, tau, row0, out, ldo,
                                       pair, guard_list, guard_cap, as_stream(stream));
}

int pf_batched_kl_i8_tiled(const uint8_t *A, const int32_t *ea, int64_t rows, const uint8_t *B,
                           const int32_t *eb, int64_t T, int64_t k, const double *H,
                           const int64_t *targets, double tau, int64_t row0, double *out,
                           int64_t ldo, int grade, int64_t *guard_list, int64_t guard_cap,
                           pf_stream_t stream) {
  if (grade != 64 && grade != 32) return fail(PF_E_ARG, "batched_kl_i8: grade must be 64 or 32");
  const int kS = grade == 64 ? kOzSlices : 5;
  if (rows <= 0 || T <= 0) return 0;
  if (!A || !ea || !B || !eb || !H || !targets || !out) return fail(PF_E_ARG, "batched_kl_i8: null");
  if (k > kOzMaxK) return fail(PF_E_DOMAIN, "batched_kl_i8: k = %lld > %d", (long long)k, kOzMaxK);
  if (ldo < T) return fail(PF_E_ALIGN, "batched_kl_i8: ldo >= T");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    return fail(PF_E_ALIGN, "batched_kl_i8: tiles must be 16-byte aligned");
  const int64_t row_tiles = (rows + 127) / 128;
  if (row_tiles > 65535) return fail(PF_E_DOMAIN, "batched_kl_i8: too many rows per launch");
  const int64_t ua = pf_i8_tiled_bytes(rows, k) / 7 / 256, ub = pf_i8_tiled_bytes(T, k) / 7 / 256;
  if (ua > INT32_MAX || ub > INT32_MAX) return fail(PF_E_DOMAIN, "batched_kl_i8: operand too large");
  CUtensorMap m[4];
  if (int e = tiled_map(&m[0], A, ua, kP2TileA / 256, kS)) return e;
  if (int e = tiled_map(&m[1], A, ua, kP2TileA / 256, kO2Pass1Slices)) return e;
  if (int e = tiled_map(&m[2], B, ub, kP2TileB / 256, kS)) return e;
  if (int e = tiled_map(&m[3], B, ub, kP2TileB / 256, kO2Pass1Slices)) return e;
  return grade == 64
             ? launch_i8<7, 9, true>(m, ea, eb, rows, T, k, H, targets, tau, row0, out, ldo, true,
                                     guard_list, guard_cap, as_stream(stream))
             : launch_i8<5, 6, true>(m, ea, eb, rows, T, k, H, targets, tau, row0, out, ldo, true,
                                     guard_list, guard_cap, as_stream(stream));
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
