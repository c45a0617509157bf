// Standalone probe (not part of the product): where does K7's int8 MMA rate
// go?  Back-to-back tcgen05.mma kind::i8 over shared-memory-resident slice
// planes laid out exactly as K7 stages them (SWIZZLE_32B K-major, 7 A and 7 B
// planes, levels 2..9 rotating over the TMEM accumulators), 1-CTA or CTA
// pair, N = 128 or 256, optionally with a concurrent bulk-copy stream into a
// scratch ring at K7's bytes-per-MMA ratio (the TMA writes that share the
// SM's shared-memory bandwidth with the UMMA operand reads).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//      tools/probe_umma_shapes.cu -o tools/probe_umma_shapes.bin -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1708_02845_b200/csrc/pf_tc.cuh"

using namespace pf;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

constexpr int kSlices = 7, kRing = 4, kChunk = 16384;

__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

template <bool kPair, int kMode>
__device__ __forceinline__ void pass1_bursts(int bursts, uint32_t a0, uint32_t tm, uint32_t id,
                                             uint64_t *full_bar, uint64_t *empty_bar,
                                             uint64_t *junk_bar, uint64_t *ready_bar,
                                             volatile uint32_t *flag) {
  constexpr int kTileA = 128 * 32, kTileB = (kPair ? 64 : 128) * 32;
  bool ready = false;
  uint32_t seen = 0;
  for (int it = 0; it < bursts; ++it) {
    if constexpr (kMode == 31 || kMode == 32) {
      if (seen < static_cast<uint32_t>(it + 1)) {   // rare: spin until the watcher saw it
        do { seen = *flag; } while (seen < static_cast<uint32_t>(it + 1));
      }
      tc::fence_after();
      seen = *flag;   // read early; consumed at the next stage boundary
    }
    if constexpr (kMode == 16) {
      if (!ready) mbar_wait(&full_bar[it % 5], (it / 5) & 1);
    }
    if constexpr (kMode >= 20 && kMode < 30) {   // busy-wait (kMode - 20) * 100 clk per burst
      const long long t0 = clock64();
      while (clock64() - t0 < (kMode - 20) * 100) {}
    }
    if constexpr (kMode == 11) mbar_wait(ready_bar, 0);
    if constexpr (kMode == 12) {
      asm volatile("{\n\t.reg .pred p;\nS_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%0], 0;"
                   "\n\t@!p bra S_%=;\n}" ::"r"(smem_u32(ready_bar)) : "memory");
    }
    if constexpr (kMode == 13) {
      while (*flag == 0) {}
    }
    if constexpr (kMode == 14) mbar_wait(&full_bar[it % 5], (it / 5) & 1);
    if constexpr (kMode == 33) mbar_wait(ready_bar, 0);
    if constexpr (kMode == 34) seen += *flag;
    if constexpr (kMode != 33) tc::fence_after();
    const uint32_t sa = a0 + (it % 5) * 43008, sbb = sa + 7 * kTileA;
#pragma unroll
    for (int i = 1; i <= 4; ++i)
#pragma unroll
      for (int j = 1; j <= 4; ++j) {
        if (i + j > 5) continue;
        const uint32_t d = tm + (i + j - 2) * 128;
        const uint64_t da = tc::sdesc<32>(sa + (i - 1) * kTileA);
        const uint64_t db = tc::sdesc<32>(sbb + (j - 1) * kTileB);
        if constexpr (kPair) tc::mma_i8_pair(d, da, db, id, true);
        else tc::mma_i8(d, da, db, id, true);
        if constexpr (kMode == 16) {
          if (i == 1 && j == 2) {   // look ahead: the next stage's barrier, non-blocking
            uint32_t ok;
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(smem_u32(&full_bar[(it + 1) % 5])), "r"(((it + 1) / 5) & 1)
                : "memory");
            ready = ok != 0;
          }
        }
      }
    if constexpr (kMode >= 14 && kMode != 31) {
      if constexpr (kPair) tc::commit_pair(&empty_bar[it % 5]);
      else tc::commit(&empty_bar[it % 5]);
    } else {
      if constexpr (kPair) tc::commit_pair(junk_bar);
      else tc::commit(junk_bar);
    }
  }
}

// kMode 35: mode 11 with the ring unrolled by 5 (stage offsets compile-time)
template <bool kPair, int kWaitKind>
__device__ __forceinline__ void pass1_bursts_unrolled(int bursts, uint32_t a0, uint32_t tm,
                                                      uint32_t id, uint64_t *ready_bar,
                                                      uint64_t *junk_bar) {
  constexpr int kTileA = 128 * 32, kTileB = (kPair ? 64 : 128) * 32;
  for (int it0 = 0; it0 < bursts; it0 += 5) {
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      if constexpr (kWaitKind == 1) mbar_wait(ready_bar, 0);
      tc::fence_after();
      const uint32_t sa = a0 + st * 43008, sbb = sa + 7 * kTileA;
#pragma unroll
      for (int i = 1; i <= 4; ++i)
#pragma unroll
        for (int j = 1; j <= 4; ++j) {
          if (i + j > 5) continue;
          const uint32_t d = tm + (i + j - 2) * 128;
          const uint64_t da = tc::sdesc<32>(sa + (i - 1) * kTileA);
          const uint64_t db = tc::sdesc<32>(sbb + (j - 1) * kTileB);
          if constexpr (kPair) tc::mma_i8_pair(d, da, db, id, true);
          else tc::mma_i8(d, da, db, id, true);
        }
      if constexpr (kPair) tc::commit_pair(junk_bar);
      else tc::commit(junk_bar);
    }
  }
}

// kPair: cta_group::2 (M256, B split 50/50); kN: MMA N; kSW: swizzle bytes =
// K bytes per slice row (32: K7's layout; 128: 4 K-steps per slice pair)
template <bool kPair, int kN, int kSW>
__global__ void __launch_bounds__(384, 1)
    shape_kernel(int iters, int tma_bytes_per_iter, const uint8_t *gsrc, int64_t gsrc_bytes,
                 uint32_t *sink, unsigned long long *cycles, int mode, int fill, int spin, int stride, int off) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int kNloc = kPair ? kN / 2 : kN;
  constexpr int kS = kSW == 32 ? kSlices : 3;          // SW128 planes are 4x larger
  constexpr int kTileA = 128 * kSW, kTileB = kNloc * kSW;
  constexpr int kAcc = 512 / kN;                        // accumulators that fit TMEM
  uint8_t *sa = smem, *sb = smem + kS * kTileA, *scratch = sb + kS * kTileB;
  __shared__ __align__(8) uint64_t done_bar, ring_bar[kRing], junk_bar, spin_bar;
  __shared__ __align__(8) uint64_t full_bar[5], empty_bar[5], ready_bar;
  __shared__ uint32_t flag;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = kPair ? tc::cluster_rank() : 0;
  const int init_bytes = mode >= 5 ? 5 * 43008 + 4096 : kS * (kTileA + kTileB);
  for (int i = tid; i < init_bytes / 4; i += 128) {
    uint32_t h = static_cast<uint32_t>(i) * 2654435761u + rank * 97u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t *>(smem)[i] = fill ? h : 0x01010101u * ((i * 7 + rank) & 3);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    mbar_init(&done_bar, 1);
    mbar_init(&junk_bar, 1 << 20);
    mbar_init(&spin_bar, 1);
    mbar_init(&ready_bar, 1);
    mbar_arrive(&ready_bar);   // phase 0 complete from the start
    flag = mode == 32 ? 0u : 1u << 30;
    for (int q = 0; q < 5; ++q) {
      mbar_init(&full_bar[q], 1);
      mbar_init(&empty_bar[q], 1);
    }
    for (int s = 0; s < kRing; ++s) mbar_init(&ring_bar[s], 1);
  }
  if (warp == 0) {
    if constexpr (kPair) tc::tmem_alloc_pair<512>(&tmem_base);
    else tc::tmem_alloc<512>(&tmem_base);
  }
  tc::fence_before();
  if constexpr (kPair) tc::cluster_sync();
  else __syncthreads();
  tc::fence_after();
  const uint32_t tm = tmem_base;
  const unsigned long long c0 = clock64();
  if (warp == 0 && tid == 0 && rank == 0) {
    constexpr uint32_t id = tc::idesc_i8(kPair ? 256 : 128, kN, false, false);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    if (mode >= 10 && kSW == 32 && kN == 128) {
      const int b = iters * 34 / 10;
      if (mode == 10) pass1_bursts<kPair, 10>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 11) pass1_bursts<kPair, 11>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 12) pass1_bursts<kPair, 12>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 13) pass1_bursts<kPair, 13>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 14) pass1_bursts<kPair, 14>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 15) pass1_bursts<kPair, 15>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 16) pass1_bursts<kPair, 16>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 21) pass1_bursts<kPair, 21>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 22) pass1_bursts<kPair, 22>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 23) pass1_bursts<kPair, 23>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 24) pass1_bursts<kPair, 24>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 26) pass1_bursts<kPair, 26>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 31) pass1_bursts<kPair, 31>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 32) pass1_bursts<kPair, 32>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 33) pass1_bursts<kPair, 33>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      if (mode == 34) {
        pass1_bursts<kPair, 34>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
      }
      if (mode == 35) pass1_bursts_unrolled<kPair, 1>(b, a0, tm, id, &ready_bar, &junk_bar);
      if (mode == 36) pass1_bursts_unrolled<kPair, 0>(b, a0, tm, id, &ready_bar, &junk_bar);
      if (mode == 29) pass1_bursts<kPair, 29>(b, a0, tm, id, full_bar, empty_bar, &junk_bar, &ready_bar, &flag);
    } else if (mode >= 5 && mode != 6 && kSW == 32 && kN == 128) {   // pass 1 over a rotating 5-stage ring
      for (int it = 0; it < iters * 34 / 10; ++it) {
        if (mode == 7) mbar_wait(&full_bar[it % 5], (it / 5) & 1);
        const uint32_t sa = a0 + off + (it % 5) * stride, sbb = sa + 7 * kTileA;
#pragma unroll
        for (int i = 1; i <= 4; ++i)
#pragma unroll
          for (int j = 1; j <= 4; ++j) {
            if (i + j > 5) continue;
            const uint32_t d = tm + (i + j - 2) * kN;
            const uint64_t da = tc::sdesc<kSW>(sa + (i - 1) * kTileA);
            const uint64_t db = tc::sdesc<kSW>(sbb + (j - 1) * kTileB);
            if constexpr (kPair) tc::mma_i8_pair(d, da, db, id, true);
            else tc::mma_i8(d, da, db, id, true);
          }
        if (mode >= 7) {
          if constexpr (kPair) tc::commit_pair(&empty_bar[it % 5]);
          else tc::commit(&empty_bar[it % 5]);
        } else {
          if constexpr (kPair) tc::commit_pair(&junk_bar);
          else tc::commit(&junk_bar);
        }
      }
    } else if (mode == 6 && kSW == 32 && kN == 128) {   // pass 2 over the ring
      for (int it = 0; it < iters * 34 / 24; ++it) {
        const uint32_t sa = a0 + (it % 5) * 43008, sbb = sa + 7 * kTileA;
#pragma unroll
        for (int i = 1; i <= 7; ++i)
#pragma unroll
          for (int j = 1; j <= 7; ++j) {
            if (i + j < 6 || i + j > 9) continue;
            const uint32_t d = tm + (i + j - 6) * kN;
            const uint64_t da = tc::sdesc<kSW>(sa + (i - 1) * kTileA);
            const uint64_t db = tc::sdesc<kSW>(sbb + (j - 1) * kTileB);
            if constexpr (kPair) tc::mma_i8_pair(d, da, db, id, true);
            else tc::mma_i8(d, da, db, id, true);
          }
        if constexpr (kPair) tc::commit_pair(&junk_bar);
        else tc::commit(&junk_bar);
      }
    } else if (mode >= 1 && kSW == 32) {
      // mode 1: every MMA into one accumulator (a dependent chain);
      // mode 2: K7 pass 1 (levels 2..5 of slices 1..4, acc l - 2), i-major,
      //         in bursts of 10 (34 per "iteration" for the op count);
      // mode 3: mode 2 + a tcgen05.commit after every 10 MMAs;
      // mode 4: K7 pass 1 reordered: L5 L4 L5 L3 L5 L4 L2 L5 L3 L4, + commits
      constexpr int ord[10][2] = {{1, 4}, {1, 3}, {2, 3}, {1, 2}, {3, 2},
                                  {2, 2}, {1, 1}, {4, 1}, {2, 1}, {3, 1}};
      constexpr int nat[10][2] = {{1, 1}, {1, 2}, {1, 3}, {1, 4}, {2, 1},
                                  {2, 2}, {2, 3}, {3, 1}, {3, 2}, {4, 1}};
      int cnt = 0;
      for (int it = 0; it < iters * 34 / 10; ++it) {
#pragma unroll
        for (int q = 0; q < 10; ++q) {
          const int i = mode == 4 ? ord[q][0] : nat[q][0];
          const int j = mode == 4 ? ord[q][1] : nat[q][1];
          const uint32_t d = mode == 1 ? tm : tm + (i + j - 2) * kN;
          const uint64_t da = tc::sdesc<kSW>(a0 + (i - 1) * kTileA);
          const uint64_t db = tc::sdesc<kSW>(b0 + (j - 1) * kTileB);
          if constexpr (kPair) tc::mma_i8_pair(d, da, db, id, true);
          else tc::mma_i8(d, da, db, id, true);
          ++cnt;
        }
        if (mode >= 3) {
          if constexpr (kPair) tc::commit_pair(&junk_bar);
          else tc::commit(&junk_bar);
        }
      }
      if (cnt == -1) sink[1] = 0;
    } else
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 1; i <= kS; ++i)
#pragma unroll
        for (int j = 1; j <= kS; ++j) {
          const int l = i + j;
          if (kSW == 32 && l > 9) continue;
#pragma unroll
          for (int ks = 0; ks < kSW / 32; ++ks) {
            const uint32_t d = tm + (l % kAcc) * kN;
            const uint64_t da = tc::sdesc<kSW>(a0 + (i - 1) * kTileA + ks * 32);
            const uint64_t db = tc::sdesc<kSW>(b0 + (j - 1) * kTileB + ks * 32);
            if constexpr (kPair) tc::mma_i8_pair(d, da, db, id, true);
            else tc::mma_i8(d, da, db, id, true);
          }
        }
    }
    if constexpr (kPair) tc::commit_pair(&done_bar);
    else tc::commit(&done_bar);
  } else if (warp == 2 && tid == 64 && mode == 32 && rank == 0) {
    for (int it = 0; it < iters * 34 / 10; ++it) {   // watcher: publish full stages
      mbar_wait(&full_bar[it % 5], (it / 5) & 1);
      asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(&flag)), "r"(it + 1) : "memory");
    }
  } else if (warp == 1 && tid == 32 && (mode == 7 || mode == 8 || (mode >= 14 && mode <= 30))) {
    // K7's ring handshake without loads: wait the slot's MMA commit, arrive
    for (int it = 0; it < iters * 34 / 10; ++it) {
      const int q = it % 5;
      mbar_wait(&empty_bar[q], ((it / 5) & 1) ^ 1);
      if (rank == 0) mbar_arrive(&full_bar[q]);
    }
  } else if (warp == 1 && tid == 32 && tma_bytes_per_iter > 0) {
    // bulk-copy stream into the scratch ring, kRing chunks in flight
    const int64_t total = static_cast<int64_t>(iters) * tma_bytes_per_iter;
    const int64_t nchunks = total / kChunk;
    const int64_t span = gsrc_bytes / kChunk;
    const int64_t base = (blockIdx.x * 977) % span;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int s = static_cast<int>(c % kRing);
      if (c >= kRing) mbar_wait(&ring_bar[s], ((c / kRing) - 1) & 1);
      mbar_expect_tx(&ring_bar[s], kChunk);
      bulk_g2s(scratch + s * kChunk, gsrc + ((base + c) % span) * kChunk, kChunk, &ring_bar[s]);
    }
    for (int64_t c = nchunks > kRing ? nchunks - kRing : 0; c < nchunks; ++c)
      mbar_wait(&ring_bar[c % kRing], (c / kRing) & 1);
    cycles[2 * blockIdx.x + 1] = clock64() - c0;
  }
  if (warp >= 4) {   // idle warps polling an mbarrier (spin 1) or backing off (spin 2)
    if (spin == 1) {
      mbar_wait(&spin_bar, 0);
    } else {
      while (!mbar_try(&spin_bar, 0)) __nanosleep(256);
    }
  }
  if (warp == 0) {
    __syncwarp();
    mbar_wait(&done_bar, 0);
    tc::fence_after();
    if (tid == 0) cycles[2 * blockIdx.x] = clock64() - c0;
    if (tid == 0) mbar_arrive(&spin_bar);
    uint32_t v[8];
    tc::tmem_ld8(tm, v);
    tc::tmem_ld_wait();
    if (v[0] == 0x12345u) sink[0] = v[1];
  }
  tc::fence_before();
  if constexpr (kPair) tc::cluster_sync();
  else __syncthreads();
  if (warp == 0) {
    if constexpr (kPair) tc::tmem_free_pair<512>(tm);
    else tc::tmem_free<512>(tm);
  }
}


// TMA ingest throughput per SM: a producer streaming 3-D boxes {box_k bytes,
// 128 rows, 7 slices} of a [7][rows][ldk] u8 slice array (K7's A operand
// shape) vs 1-D bulk copies of the same bytes, 4-deep ring, all SMs.
__global__ void __launch_bounds__(128, 1)
    tma_rate_kernel(const __grid_constant__ CUtensorMap map, const uint8_t *flat, int64_t flat_bytes,
                    int iters, int box_k, int bulk, unsigned long long *cycles, int rtiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t bar[4];
  const int tid = threadIdx.x;
  const uint32_t bytes = 7u * 128u * static_cast<uint32_t>(box_k);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
  }
  __syncthreads();
  if (tid == 0) {
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it & 3;
      if (it >= 4) mbar_wait(&bar[s], ((it >> 2) - 1) & 1);
      mbar_expect_tx(&bar[s], bytes);
      const int kb = (it * 7 + blockIdx.x * 13) % 120;
      const int rt = (blockIdx.x * 37 + it / 120) % rtiles;
      if (bulk >= 2) {   // pre-tiled operand: 3-D box {256 or 128 B, rows of it, 7}
        const int br = bulk == 2 ? 16 : 32;
        const int64_t units = flat_bytes / 7 / (bulk == 2 ? 256 : 128);
        const int64_t u = ((static_cast<int64_t>(rt) * 120 + kb) * br) % (units - br);
        tc::tma_load_3d(smem + s * 65536, &map, 0, static_cast<int32_t>(u), 0, &bar[s]);
      } else if (bulk) {
        const int64_t off = ((static_cast<int64_t>(rt) * 120 + kb) * bytes) % (flat_bytes - bytes);
        bulk_g2s(smem + s * 65536, flat + (off & ~15ll), bytes, &bar[s]);
      } else {
        tc::tma_load_3d(smem + s * 65536, &map, kb * box_k, rt * 128, 0, &bar[s]);
      }
    }
    for (int it = iters - 4; it < iters; ++it) mbar_wait(&bar[it & 3], (it >> 2) & 1);
    cycles[blockIdx.x] = clock64() - c0;
  }
}

template <bool kPair, int kN, int kSW>
void run(const char *name, int tma_per_iter, const uint8_t *gsrc, int64_t gbytes, uint32_t *sink,
         unsigned long long *cyc, int mode = 0, int fill = 0, int spin = 0, int stride = 43008,
         int off = 0) {
  constexpr int kNloc = kPair ? kN / 2 : kN;
  constexpr int kS = kSW == 32 ? kSlices : 3;
  int smem = kS * (128 * kSW + kNloc * kSW) + kRing * kChunk + 1024;
  if (mode >= 5) smem = 5 * 43008 + 1024 + 4096;
  auto kern = shape_kernel<kPair, kN, kSW>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int mmas = 0;
  for (int i = 1; i <= kS; ++i)
    for (int j = 1; j <= kS; ++j)
      if (!(kSW == 32 && i + j > 9)) mmas += kSW / 32;
  if (mode) mmas = 34;
  const int iters = kSW == 32 ? 3000 : 3000 * 34 / mmas;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148, 1, 1);
  cfg.blockDim = dim3(spin ? 384 : 128, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, kern, iters, tma_per_iter, gsrc, gbytes, sink, cyc, mode, fill, spin, stride, off));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep && ms < best) best = ms;
  }
  std::vector<unsigned long long> h(2 * 148);
  CK(cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost));
  double mma_c = 0, tma_c = 0;
  for (int b = 0; b < 148; ++b) {
    if (!kPair || b % 2 == 0) mma_c = mma_c > h[2 * b] ? mma_c : h[2 * b];
    tma_c = tma_c > h[2 * b + 1] ? tma_c : h[2 * b + 1];
  }
  const double ctas_mma = kPair ? 74.0 : 148.0;
  const double ops = 2.0 * (kPair ? 256 : 128) * kN * 32 * double(mmas) * iters * ctas_mma;
  const double per_sm_mma_clk = mma_c / (double(mmas) * iters);
  printf("{\"variant\": \"%s\", \"tma_bytes_per_34mma\": %d, \"ms\": %.4f, \"int8_tops\": %.1f, "
         "\"clk_per_mma\": %.2f, \"ideal_clk_per_mma\": %d, \"tma_B_per_clk_per_sm\": %.2f}\n",
         name, tma_per_iter * 34 / mmas, best, ops / (best * 1e-3) / 1e12, per_sm_mma_clk,
         (kPair ? 256 : 128) * kN * 32 / (kPair ? 2 : 1) / 8192,
         tma_c > 0 ? double(tma_per_iter) * iters / tma_c : 0.0);
  fflush(stdout);
}

#include <cudaTypedefs.h>
static void tma_rate(int box_k, int bulk, int64_t rows = 256 * 128) {
  const int64_t ldk = 4160;   // 7 x rows x 4160 (rows 32768: 954 MB > L2; 2048: 60 MB, L2-resident)
  uint8_t *A;
  CK(cudaMalloc(&A, 7 * rows * ldk));
  CK(cudaMemset(A, 3, 7 * rows * ldk));
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)ldk, (cuuint64_t)rows, 7};
  cuuint64_t strides[2] = {(cuuint64_t)ldk, (cuuint64_t)(rows * ldk)};
  cuuint32_t box[3] = {(cuuint32_t)box_k, 128, 7};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = box_k == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : box_k == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                        : CU_TENSOR_MAP_SWIZZLE_32B;
  if (bulk >= 2) {   // the same bytes viewed as [7][rows * ldk / W][W], W = 256 or 128
    const int64_t W = bulk == 2 ? 256 : 128;
    dims[0] = W;
    dims[1] = rows * ldk / W;
    strides[0] = W;
    box[0] = (cuuint32_t)W;
    box[1] = bulk == 2 ? 16 : 32;
    sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  }
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, A, dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    exit(1);
  }
  unsigned long long *cyc;
  CK(cudaMalloc(&cyc, 148 * 8));
  const int smem = 4 * 65536 > 227 * 1024 ? 3 * 65536 : 4 * 65536;
  CK(cudaFuncSetAttribute(tma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 57344 + 1024));
  const int iters = 2000;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0));
    tma_rate_kernel<<<148, 128, 4 * 57344 + 1024>>>(map, A, 7 * rows * ldk, iters, box_k, bulk, cyc,
                                                   static_cast<int>(rows / 128));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  std::vector<unsigned long long> h(148);
  CK(cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost));
  double mx = 0;
  for (auto v : h) mx = mx > v ? mx : v;
  const double bytes = 7.0 * 128 * box_k * iters;
  printf("{\"tma_rate\": \"%s box_k %d rows %lld\", \"ms\": %.3f, \"chip_TBps\": %.2f, \"B_per_clk_per_sm\": %.1f}\n",
         bulk == 3 ? "tiled128" : bulk == 2 ? "tiled256" : bulk ? "bulk" : "tensor3d", box_k, (long long)rows, best, bytes * 148 / (best * 1e-3) / 1e12, bytes / mx);
  fflush(stdout);
  CK(cudaFree(A));
  CK(cudaFree(cyc));
  (void)smem;
}

int main() {
  uint8_t *gsrc;
  const int64_t gbytes = 64ll << 20;
  CK(cudaMalloc(&gsrc, gbytes));
  CK(cudaMemset(gsrc, 1, gbytes));
  uint32_t *sink;
  unsigned long long *cyc;
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&cyc, 2 * 148 * 8));
  CK(cudaMemset(cyc, 0, 2 * 148 * 8));
  // K7 per CTA per 34 MMAs: 1-CTA 11 slices x 8 KB = 88 KB, pair 11 x 6 KB = 66 KB
  for (int64_t rows : {2048, 256 * 128})
    for (int mode : {0, 1, 2, 3}) tma_rate(32, mode, rows);
  return 0;
  for (int m : {10, 11, 35, 36}) {
    char nm[96];
    snprintf(nm, sizeof nm, "pair pass-1 bursts mode %d", m);
    run<true, 128, 32>(nm, 0, gsrc, gbytes, sink, cyc, m, 0, 0);
  }
  return 0;
  for (int m = 2; m <= 8; ++m) {
    if (m == 3 || m == 4 || m == 6) continue;
    char nm[64];
    snprintf(nm, sizeof nm, "pair M256 N128 SW32 mode %d", m);
    run<true, 128, 32>(nm, 0, gsrc, gbytes, sink, cyc, m, 0, 0);
    run<true, 128, 32>(nm, 0, gsrc, gbytes, sink, cyc, m, 0, 0);
  }
  return 0;
  for (int f = 0; f < 2; ++f)
    for (int m = 2; m <= 6; m += (m == 2 ? 3 : 1)) {
      char nm[64];
      snprintf(nm, sizeof nm, "pair M256 N128 SW32 mode %d fill %d", m, f);
      run<true, 128, 32>(nm, 0, gsrc, gbytes, sink, cyc, m, f);
      snprintf(nm, sizeof nm, "1cta M128 N128 SW32 mode %d fill %d", m, f);
      if (m != 5 && m != 6) run<false, 128, 32>(nm, 0, gsrc, gbytes, sink, cyc, m, f);
    }
  for (int m = 1; m <= 0; ++m) {
    char nm[64];
    snprintf(nm, sizeof nm, "pair M256 N128 SW32 mode %d", m);
    run<true, 128, 32>(nm, 0, gsrc, gbytes, sink, cyc, m);
    snprintf(nm, sizeof nm, "1cta M128 N128 SW32 mode %d", m);
    run<false, 128, 32>(nm, 0, gsrc, gbytes, sink, cyc, m);
  }
  for (int t = 0; t < 2; ++t) {
    run<false, 256, 128>("1cta M128 N256 SW128 (probe shape)", 0, gsrc, gbytes, sink, cyc);
    run<false, 128, 32>("1cta M128 N128 SW32 (K7)", t ? 88 * 1024 : 0, gsrc, gbytes, sink, cyc);
    run<true, 128, 32>("pair M256 N128 SW32 (K7 pair)", t ? 66 * 1024 : 0, gsrc, gbytes, sink, cyc);
    run<false, 256, 32>("1cta M128 N256 SW32", t ? 88 * 1024 : 0, gsrc, gbytes, sink, cyc);
    run<true, 256, 32>("pair M256 N256 SW32", t ? 88 * 1024 : 0, gsrc, gbytes, sink, cyc);
    run<true, 128, 128>("pair M256 N128 SW128", t ? 66 * 1024 : 0, gsrc, gbytes, sink, cyc);
    run<false, 128, 128>("1cta M128 N128 SW128", t ? 88 * 1024 : 0, gsrc, gbytes, sink, cyc);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
