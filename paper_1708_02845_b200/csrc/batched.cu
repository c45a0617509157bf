// batched.cu — KL to a batch of T targets as one dense contraction (K7).
//
// Reference semantics: T calls of pathfield/divergence.py dv_field(pk, kl, t)
// (:154-187); the reference has no batched API.
//
//   KL[q, t] = H[q] - sum_b c(Q_qb) * log c(Pt_b)      (c(x) = max(x, clamp))
//
// i.e. C = H 1^T - Qc * L^T with Qc the clamped P (n x k) and L (T x k) the
// clamped logs of the target rows: an FP64 GEMM n x T x k (C5: 1M x 1024 x
// 4102 = 8.4 TFLOP) with a fused epilogue (split-form cancellation guard ->
// sentinel, settle, KL[t, t] = 0).  tcgen05 has no FP64 kind, so the
// contraction runs on the FP64 tensor-core path, mma.sync m8n8k4 (SASS
// DMMA), fed by a 3-stage cp.async pipeline (tools/tune_gemm.cu records
// the DFMA and register-prefetch variants it replaced: 20-22 TFLOP/s vs
// 29.3).  Guarded pairs are re-evaluated per element in the reference form
// by batched_kl_fixup.
//
// The per-target `clamped` precision flag (divergence.py:172-175) is exact
// without an n x T x k compare: all interior rows share one below-clamp mask
// M* (pf_mask_uniform_f64 checks it once per P), so flag_t = !uniform ||
// mask(P[t]) != M*.
#include <cmath>

#include "pf_common.cuh"

namespace pf {

constexpr int kBK = 16, kGemmThreads = 256;
constexpr unsigned long long kBatchGuard = 0x7ff8dead0000ba7cull;

// L[t, b] = log(max(Pt[t, b], clamp)), Tc[t, b] = max(Pt[t, b], clamp), zero
// beyond k (L) / 1 (Tc) up to ldl; tflag[t] = mask(Pt[t]) != mask(ref).
__global__ void batch_prep_kernel(const double *__restrict__ Pt, int64_t ldp, int64_t T,
                                  int64_t k, int64_t ldl, double clamp,
                                  const double *__restrict__ ref, double *__restrict__ L,
                                  double *__restrict__ Tc, uint32_t *__restrict__ tflag) {
  const int64_t t = blockIdx.x;
  if (t >= T) return;
  bool diff = false;
  for (int64_t b = threadIdx.x; b < ldl; b += blockDim.x) {
    if (b < k) {
      const double p = Pt[t * ldp + b];
      const double c = clamp_lo(p, clamp);
      L[t * ldl + b] = log(c);
      Tc[t * ldl + b] = c;
      if (ref) diff |= (p < clamp) != (ref[b] < clamp);
    } else {
      L[t * ldl + b] = 0.0;
      Tc[t * ldl + b] = 1.0;
    }
  }
  diff = __syncthreads_or(diff);
  if (threadIdx.x == 0 && tflag) tflag[t] = diff ? 1u : 0u;
}

// nonuniform[0] |= some interior row's below-clamp mask differs from ref's.
__global__ void mask_uniform_kernel(const double *__restrict__ P, int64_t ld, int64_t rows,
                                    int64_t k, double clamp, const uint8_t *__restrict__ interior,
                                    const double *__restrict__ ref, uint32_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool diff = false;
  for (int64_t r = warp; r < rows; r += nwarps) {
    if (interior && !interior[r]) continue;
    const double *row = P + r * ld;
    for (int64_t b = lane; b < k; b += 32) diff |= (ldg_stream(row + b) < clamp) != (ref[b] < clamp);
  }
  if (__any_sync(0xffffffffu, diff) && lane == 0) atomicOr(out, 1u);
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// DMMA v2 (production): 3-stage cp.async pipeline (no register prefetch),
// block tile 128 (q) x 64 (t), 8 warps as 4 (m) x 2 (n) with 32 x 32 warp
// tiles (16 FP64 accumulators pairs per thread, ~100 registers: 2 CTAs/SM),
// tiles stored [row][k] with a 20-double stride so every fragment load is
// bank-conflict free.  Requires P and L pad columns (up to round_up(k,16))
// to be finite: the clamp is applied to A fragments after the shared load and
// pad columns of L are zero.
constexpr int kV2BM = 128, kV2BN = 64, kV2S = kBK + 4, kV2Stages = 3;
constexpr int kV2StageA = kV2BM * kV2S, kV2StageB = kV2BN * kV2S;

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kGemmThreads, 2) batched_kl_dmma2_kernel(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k,
    const double *__restrict__ H, const double *__restrict__ L, int64_t ldl, int64_t T,
    const int64_t *__restrict__ targets, double clamp, double tau, int64_t row0,
    double *__restrict__ out, int64_t ldo) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *As = reinterpret_cast<double *>(smem);           // [stages][128][20]
  double *Bs = As + kV2Stages * kV2StageA;                   // [stages][64][20]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kV2BN;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * kV2BM;
  const int64_t nkt = (k + kBK - 1) / kBK;
  const int fr = lane >> 2, fc = lane & 3;

  auto issue = [&](int64_t kt) {
    if (kt < nkt) {
      const int st = static_cast<int>(kt % kV2Stages);
      double *as = As + st * kV2StageA, *bs = Bs + st * kV2StageB;
      const int64_t k0 = kt * kBK;
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // A: 128 rows x 8 chunks of 16 B
        const int e = tid + kGemmThreads * u, row = e >> 3, ch = e & 7;
        const int64_t q = q0 + row;
        const bool ok = q < rows;
        cp_async16(as + row * kV2S + 2 * ch, P + (ok ? q : 0) * ld + k0 + 2 * ch, ok);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {  // B: 64 targets x 8 chunks
        const int e = tid + kGemmThreads * u, row = e >> 3, ch = e & 7;
        const int64_t t = t0 + row;
        const bool ok = t < T;
        cp_async16(bs + row * kV2S + 2 * ch, L + (ok ? t : 0) * ldl + k0 + 2 * ch, ok);
      }
    }
    cp_async_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kV2Stages - 1; ++s) issue(s);
  for (int64_t kt = 0; kt < nkt; ++kt) {
    cp_async_wait<kV2Stages - 2>();
    __syncthreads();
    issue(kt + kV2Stages - 1);
    const int st = static_cast<int>(kt % kV2Stages);
    const double *as = As + st * kV2StageA + (wm * 32 + fr) * kV2S + fc;
    const double *bs = Bs + st * kV2StageB + (wn * 32 + fr) * kV2S + fc;
#pragma unroll
    for (int ks = 0; ks < kBK; ks += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = clamp_lo(as[8 * i * kV2S + ks], clamp);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[8 * j * kV2S + ks];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t q = q0 + wm * 32 + 8 * i + fr;
    if (q >= rows) continue;
    const double h = H[q];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t t = t0 + wn * 32 + 8 * j + 2 * fc + c;
        if (t >= T) continue;
        const double cross = acc[i][j][c];
        double val = h - cross;
        const bool is_t = (row0 + q == targets[t]);
        if (!is_t && fabs(val) < tau * (fabs(h) + fabs(cross)))
          val = __longlong_as_double(static_cast<long long>(kBatchGuard));
        else
          val = is_t ? 0.0 : settle(val);
        out[q * ldo + t] = val;
      }
    }
  }
}

template <bool FAST>
__device__ __forceinline__ double fixup_pair_t(const double *__restrict__ prow,
                                             const double *__restrict__ trow, int64_t k,
                                             double clamp, int lane) {
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t c = lane;
  for (; c + 224 < k; c += 256) {   // two 128-element steps, 8 loads in flight
    double pv[8], tv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      pv[u] = ldg_stream(prow + c + 32 * u);
      tv[u] = __ldg(trow + c + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double qv = clamp_lo(pv[u], clamp);
      b[u & 3] += kl_term<FAST>(qv, tv[u]);
    }
  }
  for (; c + 96 < k; c += 128) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double qv = clamp_lo(prow[c + 32 * u], clamp);
      b[u] += kl_term<FAST>(qv, trow[c + 32 * u]);
    }
  }
  for (; c < k; c += 32) {
    const double qv = clamp_lo(prow[c], clamp);
    b[0] += kl_term<FAST>(qv, trow[c]);
  }
  return settle(warp_sum((b[0] + b[1]) + (b[2] + b[3])));
}

// clamp >= kFastTermMin: the branch-free terms (pf_common.cuh kl_term)
__device__ __forceinline__ double fixup_pair(const double *__restrict__ prow,
                                             const double *__restrict__ trow, int64_t k,
                                             double clamp, int lane) {
  return clamp >= kFastTermMin ? fixup_pair_t<true>(prow, trow, k, clamp, lane)
                               : fixup_pair_t<false>(prow, trow, k, clamp, lane);
}

// Per-element reference form for guarded (q, t) pairs (divergence.py:180).
__global__ void __launch_bounds__(256) batched_kl_fixup_kernel(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k,
    const double *__restrict__ Tc, int64_t ldl, int64_t T, double clamp,
    double *__restrict__ out, int64_t ldo, uint32_t *__restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = rows * T;
  uint32_t done = 0;
  // (q, t) entries interleaved across warps: guarded pairs cluster near each
  // target's row, so neighbouring entries must land on different warps.
  for (int64_t i0 = 0; warp + i0 * nwarps < total; i0 += 32) {
    const int64_t mine = warp + (i0 + lane) * nwarps;
    const int64_t mq = mine / T, mt = mine - mq * T;
    const bool flag = mine < total && static_cast<unsigned long long>(__double_as_longlong(
                                          out[mq * ldo + mt])) == kBatchGuard;
    unsigned ball = __ballot_sync(0xffffffffu, flag);
    while (ball) {
      const int src = __ffs(ball) - 1;
      ball &= ball - 1;
      const int64_t e = warp + (i0 + src) * nwarps, q = e / T, t = e - q * T;
      const double val = fixup_pair(P + q * ld, Tc + t * ldl, k, clamp, lane);
      if (lane == 0) out[q * ldo + t] = val;
      ++done;
    }
  }
  if (lane == 0 && done && count) atomicAdd(count, done);
}

// The same per-element reference form over a list of guarded pairs recorded
// by the K7 epilogue (guard_list[0] = count, then q * T + t entries): no scan
// of the rows x T output for sentinels (an 8 GB strided read at C5), and two
// iterations of loads in flight per lane (the fixup was latency-bound: ncu
// long-scoreboard on the row loads).  The per-lane order of the terms is the
// scan kernel's, so both give the same values.  A list that overflowed
// (count > cap) falls back to the scan.
__global__ void __launch_bounds__(256) batched_kl_fixup_list_kernel(
    const double *__restrict__ P, int64_t ld, int64_t rows, int64_t k,
    const double *__restrict__ Tc, int64_t ldl, int64_t T, double clamp,
    double *__restrict__ out, int64_t ldo, uint32_t *__restrict__ count,
    const int64_t *__restrict__ guard_list, int64_t cap, int scan_only) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = guard_list[0];
  if (n <= cap && scan_only) return;   // the staged kernel walks the list
  if (n > cap) {   // overflowed: the scan kernel's loop
    uint32_t done = 0;
    const int64_t total = rows * T;
    for (int64_t i0 = 0; warp + i0 * nwarps < total; i0 += 32) {
      const int64_t mine = warp + (i0 + lane) * nwarps;
      const int64_t mq = mine / T, mt = mine - mq * T;
      const bool flag = mine < total && static_cast<unsigned long long>(__double_as_longlong(
                                            out[mq * ldo + mt])) == kBatchGuard;
      unsigned ball = __ballot_sync(0xffffffffu, flag);
      while (ball) {
        const int src = __ffs(ball) - 1;
        ball &= ball - 1;
        const int64_t e = warp + (i0 + src) * nwarps, q = e / T, t = e - q * T;
        const double val = fixup_pair(P + q * ld, Tc + t * ldl, k, clamp, lane);
        if (lane == 0) out[q * ldo + t] = val;
        ++done;
      }
    }
    if (lane == 0 && done && count) atomicAdd(count, done);
    return;
  }
  uint32_t done = 0;
  const uint32_t row_bytes = static_cast<uint32_t>((k * 8 + 15) & ~15ll);
  auto prefetch_row = [&](int64_t j) {   // the P row of list entry j into L2
    if (lane == 0 && j < n) {
      const int64_t qj = guard_list[1 + j] / T;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P + qj * ld),
                   "r"(row_bytes)
                   : "memory");
    }
  };
  prefetch_row(warp);
  for (int64_t i = warp; i < n; i += nwarps) {
    const int64_t e = guard_list[1 + i], q = e / T, t = e - q * T;
    prefetch_row(i + nwarps);   // the next pair's row streams in while this one reduces
    const double val = fixup_pair(P + q * ld, Tc + t * ldl, k, clamp, lane);
    if (lane == 0) out[q * ldo + t] = val;
    ++done;
  }
  if (lane == 0 && done && count) atomicAdd(count, done);
}

// The list fixup with the rows staged through shared memory: each warp
// streams its pairs' P and target rows in 256-element chunks (both 2 KB)
// through a two-slot ring with cp.async.bulk, one chunk ahead of the chunk it
// reduces -- the register-loaded version left the FP64 pipe at ~50% on
// long-scoreboard stalls with 8 loads per lane in flight.  The terms are the
// branch-free ones (clamp >= kFastTermMin) and each lane adds them to the same
// four accumulators in the same order as fixup_pair_t: bitwise its values.
constexpr int kFxChunk = 256;                    // elements per chunk
constexpr int kFxWarps = 16;                     // 512 threads, one CTA per SM
constexpr int kFxSlots = 2;                      // chunks per warp in the ring (3: no faster)
constexpr int kFxSlotBytes = 2 * kFxChunk * 8;   // P + target chunk
constexpr int kFxSmem = kFxWarps * kFxSlots * kFxSlotBytes;   // 128 KB

__global__ void __launch_bounds__(kFxWarps * 32, 1) batched_kl_fixup_staged_kernel(
    const double *__restrict__ P, int64_t ld, int64_t k, const double *__restrict__ Tc,
    int64_t ldl, int64_t T, double clamp, double *__restrict__ out, int64_t ldo,
    uint32_t *__restrict__ count, const int64_t *__restrict__ guard_list, int64_t cap) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kFxWarps][kFxSlots];
  const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = guard_list[0];
  if (n > cap) return;   // overflowed: the scan (batched_kl_fixup_list_kernel) did it
  double *ring = reinterpret_cast<double *>(smem + wc * kFxSlots * kFxSlotBytes);
  if (lane == 0)
    for (int st = 0; st < kFxSlots; ++st) mbar_init(&bar[wc][st], 1);
  __syncwarp();
  const int64_t nch = (k + kFxChunk - 1) / kFxChunk;
  // the chunk stream: (pair i, chunk c) for i = warp, warp + nwarps, ...
  int64_t ii = warp, ic = 0;            // issue side
  auto issue = [&](int st) {
    if (lane == 0 && ii < n) {
      const int64_t e = guard_list[1 + ii], q = e / T, t = e - q * T;
      const int64_t base = ic * kFxChunk;
      const int64_t len = k - base < kFxChunk ? k - base : kFxChunk;
      const uint32_t bytes = static_cast<uint32_t>((len * 8 + 15) & ~15ll);
      double *dst = ring + st * 2 * kFxChunk;
      mbar_expect_tx(&bar[wc][st], 2 * bytes);
      bulk_g2s(dst, P + q * ld + base, bytes, &bar[wc][st]);
      bulk_g2s(dst + kFxChunk, Tc + t * ldl + base, bytes, &bar[wc][st]);
    }
    if (ii < n && ++ic == nch) {
      ic = 0;
      ii += nwarps;
    }
  };
#pragma unroll
  for (int st = 0; st < kFxSlots - 1; ++st) issue(st);
  uint32_t done = 0;
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t ci = warp, cc = 0;            // reduce side
  for (int64_t s = 0; ci < n; ++s) {
    issue(static_cast<int>((s + kFxSlots - 1) % kFxSlots));   // the slot freed by chunk s - 1
    const int st = static_cast<int>(s % kFxSlots);
    mbar_wait(&bar[wc][st], static_cast<uint32_t>((s / kFxSlots) & 1));
    const double *pc = ring + st * 2 * kFxChunk, *tcn = pc + kFxChunk;
    const int64_t base = cc * kFxChunk;
    if (base + kFxChunk <= k) {   // every 128-element block full for every lane: straight-line
      double tm[kFxChunk / 32];
#pragma unroll
      for (int u = 0; u < kFxChunk / 32; ++u)
        tm[u] = kl_term<true>(clamp_lo(pc[lane + 32 * u], clamp), tcn[lane + 32 * u]);
#pragma unroll
      for (int u = 0; u < kFxChunk / 32; ++u) b[u & 3] += tm[u];
    } else
#pragma unroll
    for (int u = 0; u < kFxChunk / 32; ++u) {
      const int64_t e = base + lane + 32 * u;   // this lane's elements, in order
      if (e < k) {
        // fixup_pair_t's accumulator: u & 3 inside a full 128-element block, else 0
        const int64_t blk = base + 128 * (u >> 2);
        const int acc = (blk + lane + 96 < k) ? (u & 3) : 0;
        const double term = kl_term<true>(clamp_lo(pc[lane + 32 * u], clamp), tcn[lane + 32 * u]);
        if (acc == 0) b[0] += term;
        else if (acc == 1) b[1] += term;
        else if (acc == 2) b[2] += term;
        else b[3] += term;
      }
    }
    __syncwarp();   // every lane is done with this slot before it is refilled
    if (++cc == nch) {
      const double val = settle(warp_sum((b[0] + b[1]) + (b[2] + b[3])));
      const int64_t e = guard_list[1 + ci];
      const int64_t q = e / T, t = e - q * T;
      if (lane == 0) out[q * ldo + t] = val;
      ++done;
      b[0] = b[1] = b[2] = b[3] = 0.0;
      cc = 0;
      ci += nwarps;
    }
  }
  if (lane == 0 && done && count) atomicAdd(count, done);
}

// Diagnostic: sustained DFMA throughput (8 independent chains per thread);
// bench.py reports K7's FLOP rate against it.
__global__ void __launch_bounds__(256) dfma_probe_kernel(int64_t iters, double *out) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-3 * (threadIdx.x + i);
  const double m = 0.999999, c = 1e-7;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 42.0) out[0] = s;  // keep the chains alive
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_batch_prep_f64(const double *Pt, int64_t ldp, int64_t T, int64_t k, int64_t ldl,
                      double clamp, const double *ref, double *L, double *Tc, uint32_t *tflag,
                      pf_stream_t stream) {
  if (T <= 0) return 0;
  if (!Pt || !L || !Tc || ldl < k || ldl % 16) return fail(PF_E_ARG, "batch_prep: bad args");
  batch_prep_kernel<<<static_cast<unsigned>(T), 256, 0, as_stream(stream)>>>(
      Pt, ldp, T, k, ldl, clamp, ref, L, Tc, tflag);
  return check_launch("batch_prep");
}

int pf_mask_uniform_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                        const uint8_t *is_interior, const double *ref, uint32_t *nonuniform,
                        pf_stream_t stream) {
  if (rows <= 0) return 0;
  if (!P || !ref || !nonuniform) return fail(PF_E_ARG, "mask_uniform: null");
  mask_uniform_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(P, ld, rows, k, clamp,
                                                                      is_interior, ref,
                                                                      nonuniform);
  return check_launch("mask_uniform");
}

int pf_batched_kl_f64(const double *P, int64_t ld, int64_t rows, int64_t k, const double *H,
                      const double *L, const double *Tc, int64_t ldl, int64_t T,
                      const int64_t *targets, double clamp, double tau, int64_t row0,
                      double *out, int64_t ldo, uint32_t *guarded, pf_stream_t stream) {
  if (rows <= 0 || T <= 0) return 0;
  if (!P || !H || !L || !Tc || !targets || !out) return fail(PF_E_ARG, "batched_kl: null");
  if ((ld & 1) || (reinterpret_cast<uintptr_t>(P) & 15) || ldl % 16 || ldl < k || ldo < T)
    return fail(PF_E_ALIGN, "batched_kl: alignment (ld even, ldl %% 16 == 0)");
  const size_t smem = static_cast<size_t>(kV2Stages) * (kV2StageA + kV2StageB) * sizeof(double);
  if (int e = ensure_smem((const void *)batched_kl_dmma2_kernel, smem)) return e;
  dim3 grid(static_cast<unsigned>((T + kV2BN - 1) / kV2BN),
            static_cast<unsigned>((rows + kV2BM - 1) / kV2BM));
  if (grid.y > 65535) return fail(PF_E_DOMAIN, "batched_kl: too many rows per launch (%lld)",
                                  (long long)rows);
  if (ld % 16) return fail(PF_E_ALIGN, "batched_kl: ld must be a multiple of 16 (pad columns zero)");
  batched_kl_dmma2_kernel<<<grid, kGemmThreads, smem, as_stream(stream)>>>(
      P, ld, rows, k, H, L, ldl, T, targets, clamp, tau, row0, out, ldo);
  if (int e = check_launch("batched_kl_gemm")) return e;
  batched_kl_fixup_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(
      P, ld, rows, k, Tc, ldl, T, clamp, out, ldo, guarded);
  return check_launch("batched_kl_fixup");
}

int pf_batched_kl_fixup_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                            const double *Tc, int64_t ldl, int64_t T, double clamp, double *out,
                            int64_t ldo, uint32_t *guarded, pf_stream_t stream) {
  if (rows <= 0 || T <= 0) return 0;
  if (!P || !Tc || !out) return fail(PF_E_ARG, "batched_kl_fixup: null");
  batched_kl_fixup_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(
      P, ld, rows, k, Tc, ldl, T, clamp, out, ldo, guarded);
  return check_launch("batched_kl_fixup");
}

int pf_batched_kl_fixup_list_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                                 const double *Tc, int64_t ldl, int64_t T, double clamp,
                                 double *out, int64_t ldo, uint32_t *guarded,
                                 const int64_t *guard_list, int64_t guard_cap, pf_stream_t stream) {
  if (rows <= 0 || T <= 0) return 0;
  if (!P || !Tc || !out || !guard_list) return fail(PF_E_ARG, "batched_kl_fixup_list: null");
  if (clamp >= kFastTermMin && (ld & 1) == 0 && (ldl & 1) == 0 &&
      (reinterpret_cast<uintptr_t>(P) & 15) == 0 && (reinterpret_cast<uintptr_t>(Tc) & 15) == 0) {
    // the staged version; a list that overflowed is the scan kernel's job
    if (int e = ensure_smem((const void *)batched_kl_fixup_staged_kernel, kFxSmem)) return e;
    batched_kl_fixup_list_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(
        P, ld, rows, k, Tc, ldl, T, clamp, out, ldo, guarded, guard_list, guard_cap, 1);
    if (int e = check_launch("batched_kl_fixup_list")) return e;
    batched_kl_fixup_staged_kernel<<<sm_count(), kFxWarps * 32, kFxSmem, as_stream(stream)>>>(
        P, ld, k, Tc, ldl, T, clamp, out, ldo, guarded, guard_list, guard_cap);
    return check_launch("batched_kl_fixup_staged");
  }
  batched_kl_fixup_list_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(
      P, ld, rows, k, Tc, ldl, T, clamp, out, ldo, guarded, guard_list, guard_cap, 0);
  return check_launch("batched_kl_fixup_list");
}

int pf_probe_dfma_f64(int64_t iters, int64_t *flops, double *out, pf_stream_t stream) {
  const int blocks = sm_count() * 8;
  dfma_probe_kernel<<<blocks, 256, 0, as_stream(stream)>>>(iters, out);
  if (flops) *flops = 2LL * 8 * iters * blocks * 256;
  return check_launch("dfma_probe");
}

}  // extern "C"
