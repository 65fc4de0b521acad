// K1/K2 on the tensor cores -- Gram matrix G = Phi^T Phi (SURVEY Sec. 8(a)
// row a4; B^T A of PAPER.md:337, 355 without D).  Plan-time.
//
// G is a dense contraction over points (N x r by N x r), so it runs on
// tcgen05.  Features are grouped in blocks of 64 frequencies; inside a block
// the 128 rows are [cos of the 64 frequencies; sin of the same 64] (the
// reduce kernel maps them back to the interleaved internal order).  A *unit*
// is one A block (the accumulator rows) against one or two B blocks (two
// 128 x 128 tiles, one 128 x 256 accumulator); the units cover the upper
// triangle of the block grid (the leftover tiles of the last block column
// are taken transposed, e.g. (3, [1, 3]) for T = 4).  Per K-step of 32 points:
//
//   * the MMA warp bulk-copies chunks of 8 steps' points into a shared-memory
//     ring (cp.async.bulk, mbarrier complete_tx), independent of the MMAs;
//   * 16 producer warps regenerate the step's feature values (a3: omega.x in
//     radians, one projection and one MUFU sin/cos pair per frequency and
//     point), split each as x = hi + lo in fp16 (|x - hi - lo| <= 2^-22 |x| +
//     2^-25) and store them in shared memory (canonical K-major, no swizzle);
//   * one elected lane of the MMA warp issues per 16-point K-slice
//         D += A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T
//     (tcgen05.mma kind::f16, A and B from shared memory, M = 128, N = 256
//     over both tiles, fp32 accumulate in TMEM).  On a diagonal tile the B
//     copy of the block holds 2 lo and the third product is skipped:
//     A_hi B_hi^T + A_hi (2 B_lo)^T = P + 2X, and G = (D + D^T) / 2.
//
// Measured on B200 (tools/microbench): the tensor core's shared-memory
// operand reads do not slow down under ~100 B/cycle of concurrent STS, so
// both operands come from shared memory and all of TMEM holds accumulators.
//
// Precision: the tensor core's fp32 accumulator is not round-to-nearest
// (measured: the error grows with the number of accumulating MMAs; G and C^
// leave the 1e-4 gate at 2048 points per accumulation on cfg 3), so D
// accumulates for an *epoch* of 16 K-steps (512 points); the producer warps
// then add it into a second TMEM accumulator L (tcgen05.ld, round-to-nearest
// fp32 adds, tcgen05.st: ~530 cycles per 128 x 256 drain, measured) while the
// MMA warp waits.  At the end of a unit segment L + D goes to a per-segment
// partial; K2 (gram_tc_reduce) sums the partials in a fixed order in fp64 --
// deterministic.
//
// Scheduling: one persistent CTA per SM.  The work items (cloud, unit, K-step)
// are laid out linearly and cut into contiguous CTA ranges of equal *cost*,
// so a CTA's range spans one or a few unit segments and no wave is left
// partly empty.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "rfd_internal.h"
#include "tc_ptx.cuh"

namespace rfd {
namespace {

// Debug bounds checks (compile with -DRFD_GRAM_CHECK): trap on the first
// out-of-range shared/global access, naming it.
#ifdef RFD_GRAM_CHECK
__device__ int g_check_count;
#define RFD_CHECK(cond, what, a, b)                                                      \
  do {                                                                                   \
    if (!(cond) && atomicAdd(&g_check_count, 1) < 8)                                     \
      printf("gram check failed: %s (%lld, %lld) cta %d warp %d lane %d\n", what,       \
             (long long)(a), (long long)(b), blockIdx.x, threadIdx.x / 32, threadIdx.x % 32); \
  } while (0)
// bounded wait: report (barrier tag, step) after ~2^26 probes, then give up
__device__ __forceinline__ void dbg_wait(uint64_t* bar, uint32_t par, int tag, int it) {
  for (long long i = 0; !tc::mbar_try_wait(bar, par); ++i)
    if (i == (1LL << 22)) {
      if (threadIdx.x % 32 == 0)
        printf("gram wait stuck: tag %d step %d cta %d warp %d state %llx\n", tag, it, blockIdx.x,
               threadIdx.x / 32, (unsigned long long)*reinterpret_cast<volatile uint64_t*>(bar));
      return;
    }
}
#define RFD_WAIT(bar, par, tag, it) dbg_wait((bar), (par), (tag), (it))
#else
#define RFD_WAIT(bar, par, tag, it) tc::mbar_wait((bar), (par))
#define RFD_CHECK(cond, what, a, b) \
  do {                              \
  } while (0)
#endif

constexpr int kBlk = 128;           // feature rows per block
constexpr int kFreqs = 64;          // frequencies per block
constexpr int kStep = 64;           // points per K-step (4 MMA K-slices of 16)
constexpr int kStages = 2;
constexpr int kProducerWarps = 16;
constexpr int kMmaWarp = kProducerWarps;        // MMA issue
constexpr int kLoadWarp = kProducerWarps + 1;   // point loads
constexpr int kThreads = (kProducerWarps + 2) * 32;
constexpr int kEpoch = 8;           // K-steps per TMEM accumulation epoch (power of 2)
constexpr int kMaxCtas = 160;
// Shared memory per stage (canonical K-major fp16 operands, 16 KB each):
//   [B hi: slot 0 rows | slot 1 rows][B lo: slot 0 | slot 1][A hi][A lo]
// (the N = 256 B operand is one 256-row matrix).  A hi is unused when the A
// block is a B block (its descriptor points at that slot's B hi).
constexpr uint32_t kOpBytes = kBlk * kStep * 2;   // 16 KB
constexpr uint32_t kBHi = 0, kBLo = 2 * kOpBytes, kAHi = 4 * kOpBytes, kALo = 5 * kOpBytes;
constexpr uint32_t kStageBytes = 6 * kOpBytes;    // 96 KB
// Canonical K-major layout (no swizzle): offset(row, k) = (row/8)*kSBO +
// (k/8)*kLBO + (row%8)*16 + (k%8)*2.
constexpr uint32_t kLBO = 128;
constexpr uint32_t kSBO = (kStep / 8) * 128;      // 1024
// Point ring: kChunks chunks of kChunkSteps K-steps, refilled as soon as the
// producers are done with a chunk (no dependence on MMA completion).
constexpr int kChunkSteps = 4;
constexpr int kChunks = 4;
// Points in the Gram layout: groups of 8 points, 128 B each: x[8] | y[8] |
// z[8] | pad[8] (packed FP32 pairs load straight into register pairs);
// each cloud padded with zero groups to whole K-steps.
constexpr uint32_t kGroupBytes = 128;
constexpr uint32_t kStepBytes = (kStep / 8) * kGroupBytes;    // 1 KB
constexpr uint32_t kChunkBytes = kChunkSteps * kStepBytes;    // 4 KB
constexpr int kMaxFreqs = 512;                               // RFD_MAX_M
constexpr int kRingOff = kStages * int(kStageBytes);
constexpr int kOmegaOff = kRingOff + kChunks * int(kChunkBytes);
constexpr int kSmemBytes = kOmegaOff + kMaxFreqs * 16;  // 216 KB
// TMEM columns: epoch accumulator D [0, 256), long-term sum L [256, 512).
constexpr uint32_t kColL = 256;

struct GramUnit {
  int a;     // A block (accumulator rows)
  int nb;    // tiles (1 or 2)
  int b[2];  // B block of tile tau
};

// Units covering the upper triangle of the T x T block grid: (i, [j, j+1])
// for j = i, i+2, ... while j+1 < T; the leftover tiles (i, T-1), (T-i) odd,
// paired as transposed tiles (T-1, [i1, i2]).
__host__ __device__ inline int gram_units(int T, int want, GramUnit* out) {
  int u = 0;
  for (int i = 0; i < T; ++i)
    for (int j = i; j + 1 < T; j += 2) {
      if (u == want) *out = GramUnit{i, 2, {j, j + 1}};
      ++u;
    }
  int first = -1;
  for (int i = 0; i < T; ++i) {
    if ((T - i) % 2 == 0) continue;
    if (first < 0) {
      first = i;
      continue;
    }
    if (u == want) *out = GramUnit{T - 1, 2, {first, i}};
    ++u;
    first = -1;
  }
  if (first >= 0) {
    if (u == want) *out = GramUnit{T - 1, 1, {first, first}};
    ++u;
  }
  return u;
}

// Work partition, passed by value (<= 1.4 KB of kernel parameters).
struct Sched {
  int G;          // CTAs
  int T;          // feature blocks
  int U;          // units per cloud
  int batch;
  int64_t S;      // K-steps per unit per cloud
  int64_t start[kMaxCtas + 1];  // first linear item (cloud*U + unit)*S + step of each CTA
};


// Producer-warp drain of a finished epoch: columns [64 q, 64 q + 64) of the
// warp's 32 TMEM lanes.  L = D (first epoch of a segment) or L += D
// (round-to-nearest fp32); on the segment's last epoch L + D goes to the
// segment partial (row-major [128][256] fp32) instead.  Arrives on acce once
// D has been read.
__device__ __forceinline__ void drain_epoch(uint32_t tm_lane, int q, int lane, int nb, bool first,
                                            bool last, float* row_out, uint64_t* acce_bar,
                                            bool skip = false) {
  tc::tc_fence_after();
  if (q * 64 < nb * 128 && !skip) {
    float4* o = reinterpret_cast<float4*>(row_out + q * 64);
    RFD_CHECK(nb == 1 || nb == 2, "nb", nb, q);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint32_t col = uint32_t(q * 64 + h * 16);
      float v[16];
      tc::tmem_ld16(tm_lane + col, v);
      if (!first) {
        float w[16];
        tc::tmem_ld16(tm_lane + kColL + col, w);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += w[j];
      }
      if (last) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          o[4 * h + j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      } else {
        uint32_t u[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) u[j] = __float_as_uint(v[j]);
        tc::tmem_st16(tm_lane + kColL + col, u);
      }
    }
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncwarp();
  if (lane == 0 && acce_bar) tc::mbar_arrive(acce_bar);  // D is free again
}

// Instrumentation (RFD_GRAM_TRACE=1, pair kernel): per-step timestamps of one
// CTA (RFD_GRAM_TRACE_CTA); results are unchanged.
__device__ long long g_trace[4096][8];
__device__ int g_trace_cta;

__global__ void __launch_bounds__(kThreads, 1)
gram_tc_kernel(const unsigned char* __restrict__ gpts, const float4* __restrict__ omega4, int m,
               int64_t n, const __grid_constant__ Sched sc, float* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], pts_bar[kChunks], pts_empty[kChunks];
  __shared__ uint64_t accf_bar, acce_bar;
  __shared__ uint32_t tmem_sh;

  const int cta = blockIdx.x;
  const int64_t L0 = sc.start[cta], L1 = sc.start[cta + 1];
  if (L0 >= L1) return;
  const int nsteps = int(L1 - L0);
  const int Si = int(sc.S);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = tc::smem_addr(smem);

  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], kProducerWarps);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int c = 0; c < kChunks; ++c) {
      tc::mbar_init(&pts_bar[c], 1);
      tc::mbar_init(&pts_empty[c], kProducerWarps);
    }
    tc::mbar_init(&accf_bar, 1);
    tc::mbar_init(&acce_bar, kProducerWarps);
    tc::mbar_fence_init();
  }
  {  // omega table (rows of padding frequencies >= m are zero)
    float4* om_s = reinterpret_cast<float4*>(smem + kOmegaOff);
    for (int k = tid; k < sc.T * kFreqs; k += kThreads)
      om_s[k] = (k < m) ? __ldg(omega4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;

  // Step walk (all 32-bit): unit segment bu = cloud * U + unit; the CTA's
  // steps of a segment are it in [seg_lo, seg_hi).
  const int bu0 = int(L0 / sc.S), t0 = int(L0 - int64_t(bu0) * sc.S);
  const int hi0 = int(min(L1, int64_t(bu0 + 1) * sc.S) - L0);

  if (warp == kLoadWarp) {
    // ============================================ point loads
    // Chunk ch = CTA steps [4 ch, 4 ch + 4) into ring slot ch % kChunks: one
    // bulk copy (cp.async.bulk, mbarrier complete_tx) per run of steps inside
    // one unit segment (contiguous groups), independent of the MMAs.
    const int nchunks = (nsteps + kChunkSteps - 1) / kChunkSteps;
    const int64_t cloud_bytes = int64_t(Si) * kStepBytes;
    int l_bu = bu0, l_t = t0;
    for (int ch = 0; ch < nchunks; ++ch) {
      // a ring slot is refilled once the producers are done with its previous
      // chunk (pts_empty: one phase per use of the slot -- waiting on a stage
      // barrier instead could alias phases two uses apart)
      if (ch >= kChunks) RFD_WAIT(&pts_empty[ch % kChunks], uint32_t(ch / kChunks - 1) & 1u, 1, ch);
      const int i0 = ch * kChunkSteps, i1 = min(nsteps, i0 + kChunkSteps);
      uint64_t* bar = &pts_bar[ch % kChunks];
      unsigned char* dst = smem + kRingOff + (ch % kChunks) * kChunkBytes;
      if (lane == 0) {
        // arm first (arrive + expect the chunk's bytes), then copy
        tc::mbar_arrive_expect_tx(bar, uint32_t(i1 - i0) * kStepBytes);
        for (int i = i0; i < i1;) {
          const int run = min(i1 - i, Si - l_t);
          RFD_CHECK(l_bu / sc.U < sc.batch && l_t + run <= Si && (i - i0 + run) <= kChunkSteps,
                    "bulk", l_bu, l_t);
          tc::bulk_g2s(dst + (i - i0) * kStepBytes,
                       gpts + int64_t(l_bu / sc.U) * cloud_bytes + int64_t(l_t) * kStepBytes,
                       uint32_t(run) * kStepBytes, bar);
          i += run;
          l_t += run;
          if (l_t == Si) {
            l_t = 0;
            ++l_bu;
          }
        }
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ============================================ MMA issue
    // The whole warp walks the steps (warp-uniform state: descriptors live in
    // uniform registers); one elected lane issues each tcgen05 op.
    int m_lo = 0, m_hi = hi0, m_bu = bu0, epoch = 0;
    // unit shape: nb - 1 | diag slot 0 << 1 | diag slot 1 << 2 | A is a B slot << 3
    auto unit_bits = [&](int u) {
      GramUnit X;
      gram_units(sc.T, u, &X);
      const int d0 = X.b[0] == X.a, d1 = X.nb > 1 && X.b[1] == X.a;
      return (X.nb - 1) | (d0 << 1) | (d1 << 2);
    };
    int ub = unit_bits(m_bu % sc.U);
    for (int it = 0; it < nsteps; ++it) {
      const int s = it % kStages;
      const int k = it - m_lo;
      const bool efirst = (k & (kEpoch - 1)) == 0;
      const bool elast = ((k + 1) & (kEpoch - 1)) == 0 || it + 1 == m_hi;
      if (efirst && epoch > 0) RFD_WAIT(&acce_bar, uint32_t(epoch - 1) & 1u, 2, it);
      RFD_WAIT(&full_bar[s], uint32_t(it / kStages) & 1u, 3, it);
      tc::tc_fence_after();
      __syncwarp();
      const uint32_t stage = sbase + uint32_t(s) * kStageBytes;
      const int nb = (ub & 1) + 1;
      const bool d0 = (ub >> 1) & 1, d1 = (ub >> 2) & 1;
      // A hi aliases the diagonal slot's B hi
      const uint32_t a_hi = stage + (d0 ? kBHi : (d1 ? kBHi + kOpBytes : kAHi));
      const uint32_t a_lo = stage + kALo;
      const uint32_t idesc_n = tc::make_idesc(0, 128, 128 * nb);
      const uint32_t idesc_1 = tc::make_idesc(0, 128, 128);
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < kStep / 16; ++kk) {
          const uint32_t ko = uint32_t(kk) * 2u * kLBO;
          const uint64_t ahi = tc::make_sdesc(a_hi + ko, kLBO, kSBO);
          const uint64_t alo = tc::make_sdesc(a_lo + ko, kLBO, kSBO);
          const uint64_t bhi = tc::make_sdesc(stage + kBHi + ko, kLBO, kSBO);
          const uint64_t blo = tc::make_sdesc(stage + kBLo + ko, kLBO, kSBO);
          const uint32_t acc0 = (efirst && kk == 0) ? 0u : 1u;
          {
            tc::mma_f16(tmem, ahi, bhi, idesc_n, acc0);
            tc::mma_f16(tmem, ahi, blo, idesc_n, 1u);
            if (!d0 && !d1) {
              tc::mma_f16(tmem, alo, bhi, idesc_n, 1u);
            } else if (nb == 2) {  // the off-diagonal tile only
              const uint32_t t = d0 ? 1u : 0u;
              tc::mma_f16(tmem + 128u * t, alo,
                          tc::make_sdesc(stage + kBHi + t * kOpBytes + ko, kLBO, kSBO), idesc_1,
                          1u);
            }
          }
        }
        tc::mma_commit(&empty_bar[s]);
        if (elast) tc::mma_commit(&accf_bar);
      }
      __syncwarp();
      if (elast) ++epoch;
      if (it + 1 == m_hi && it + 1 < nsteps) {
        ++m_bu;
        m_lo = it + 1;
        m_hi = min(nsteps, it + 1 + Si);
        ub = unit_bits(m_bu % sc.U);
      }
    }
  } else {
    // ============================================ producers (+ drains)
    const unsigned char* ring = smem + kRingOff;
    const float4* om_s = reinterpret_cast<const float4*>(smem + kOmegaOff);
    // Task = (frequency f of a block, 8-point group q): cos row f and sin row
    // 64 + f for 8 points.  Warp w: q = w % 8, frequencies 32 (w / 8) + lane:
    // the point loads are warp-wide broadcasts and an 8-lane store phase
    // covers the 8 rows of one core matrix (no bank conflicts).  Every warp
    // does one task of every local block per step.
    const int q = warp & 7, f = 32 * (warp >> 3) + lane;
    const uint32_t off_c = uint32_t(f >> 3) * kSBO + uint32_t(q) * kLBO + uint32_t(f & 7) * 16u;
    const uint32_t off_s = off_c + 8u * kSBO;  // row 64 + f
    const int lg = warp & 3, qd = warp >> 2;   // drain: TMEM lane group, column quarter
    const uint32_t lane_field = uint32_t(32 * lg) << 16;
    const int rho = 32 * lg + lane;

    // Local blocks of the current unit, in task order: the A block first, then
    // the B-only blocks.  Packed per local block i (8 bits): block (4 bits),
    // bit 4: stored as B slot, bit 5: which slot, bit 6: stored as A.
    int nloc = 1, locs = 0;
    auto setup_unit = [&](int u) {
      GramUnit U;
      gram_units(sc.T, u, &U);
      const bool dd0 = U.b[0] == U.a, dd1 = U.nb > 1 && U.b[1] == U.a;
      locs = U.a | 0x40 | (dd0 ? 0x10 : (dd1 ? 0x30 : 0));
      nloc = 1;
      for (int tau = 0; tau < U.nb; ++tau)
        if (U.b[tau] != U.a) locs |= (U.b[tau] | 0x10 | (tau << 5)) << (8 * nloc++);
      return U.nb;
    };
    // Epochs awaiting their drain, oldest first (-1: none); info = segment id
    // | (nb - 1) << 28 | first epoch of its segment << 29 | last << 30; last0/1
    // = the epoch's last step.
    int pend0 = -1, pend1 = -1, info0 = 0, info1 = 0, last0 = 0, last1 = 0;
    auto drain0 = [&]() {
      RFD_CHECK((info0 & 0x0FFFFFFF) < sc.G + sc.batch * sc.U, "seg", info0, pend0);
      drain_epoch(tmem + lane_field, qd, lane, ((info0 >> 28) & 1) + 1, (info0 >> 29) & 1,
                  (info0 >> 30) & 1,
                  partial + (int64_t(info0 & 0x0FFFFFFF) * 128 + rho) * 256, &acce_bar,
                  false);
      pend0 = pend1;
      info0 = info1;
      last0 = last1;
      pend1 = -1;
    };

    const int tail = int(n - int64_t(Si - 1) * kStep);  // points of a unit's last step
    int bu = bu0, seg_lo = 0, seg_hi = hi0, tail_it = Si - 1 - t0;
    int nb = setup_unit(bu % sc.U);
    int epoch = 0;
    // Every wait is on ONE barrier (a thread parked in try_wait wakes on that
    // barrier only).
    for (int it = 0; it < nsteps; ++it) {
      if (it == seg_hi) {
        ++bu;
        seg_lo = it;
        seg_hi = min(nsteps, it + Si);
        tail_it = it + Si - 1;
        nb = setup_unit(bu % sc.U);
      }
      const int k = it - seg_lo;
      const bool elast = ((k + 1) & (kEpoch - 1)) == 0 || it + 1 == seg_hi;
      const int s = it % kStages;
      const uint32_t ph = uint32_t(it / kStages) & 1u;
      const int ch = it / kChunkSteps;
      // drain the pending epoch right before a step whose stage needs an MMA
      // of a later epoch (the MMA warp waits for the drain before that epoch)
      while (pend0 >= 0 && it - kStages > last0) {
        RFD_WAIT(&accf_bar, uint32_t(pend0) & 1u, 4, it);
        __syncwarp();
        drain0();
      }
      if (it >= kStages) RFD_WAIT(&empty_bar[s], ph ^ 1u, 5, it);
      if (it % kChunkSteps == 0 || it == 0)  // a chunk's points arrive together
        RFD_WAIT(&pts_bar[ch % kChunks], uint32_t(ch / kChunks) & 1u, 6, it);
      __syncwarp();
      const int cnt = (it == tail_it) ? tail : kStep;
      const float* grp = reinterpret_cast<const float*>(
          ring + (ch % kChunks) * kChunkBytes + (it % kChunkSteps) * kStepBytes + q * kGroupBytes);
      float X[8], Y[8], Z[8];
#pragma unroll
      for (int j = 0; j < 8; j += 4) {
        *reinterpret_cast<float4*>(X + j) = *reinterpret_cast<const float4*>(grp + j);
        *reinterpret_cast<float4*>(Y + j) = *reinterpret_cast<const float4*>(grp + 8 + j);
        *reinterpret_cast<float4*>(Z + j) = *reinterpret_cast<const float4*>(grp + 16 + j);
      }
      const uint32_t stage = sbase + uint32_t(s) * kStageBytes;
      RFD_CHECK(stage + kStageBytes <= sbase + kRingOff, "stage", s, it);
      RFD_CHECK((const unsigned char*)grp >= ring && (const unsigned char*)grp + 128 <= ring + kChunks * kChunkBytes, "ring", ch, it);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        if (i >= nloc) break;
        RFD_CHECK((locs >> (8 * i) & 15) < sc.T, "block", locs, i);
        const int li = locs >> (8 * i);
        const float4 wi = om_s[(li & 15) * kFreqs + f];
        const float2 wx = make_float2(wi.x, wi.x), wy = make_float2(wi.y, wi.y),
                     wz = make_float2(wi.z, wi.z);
        // theta for two points per packed FP32 op (sm_100 FFMA2)
        float c[8], sn[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const float2 th = __ffma2_rn(wz, make_float2(Z[j], Z[j + 1]),
                                       __ffma2_rn(wy, make_float2(Y[j], Y[j + 1]),
                                                  __fmul2_rn(wx, make_float2(X[j], X[j + 1]))));
          __sincosf(th.x, &sn[j], &c[j]);
          __sincosf(th.y, &sn[j + 1], &c[j + 1]);
        }
        if (cnt < kStep) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (q * 8 + j >= cnt) c[j] = sn[j] = 0.0f;
        }
        uint32_t ch_[4], cl[4], sh[4], sl[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          tc::split_f16x2_v2(make_float2(c[2 * j], c[2 * j + 1]), ch_[j], cl[j]);
          tc::split_f16x2_v2(make_float2(sn[2 * j], sn[2 * j + 1]), sh[j], sl[j]);
        }
        if (li & 0x10) {  // B slot
          const uint32_t sb = stage + uint32_t((li >> 5) & 1) * kOpBytes;
          tc::st_shared_v4(sb + kBHi + off_c, ch_[0], ch_[1], ch_[2], ch_[3]);
          tc::st_shared_v4(sb + kBHi + off_s, sh[0], sh[1], sh[2], sh[3]);
          if (li & 0x40) {
            // diagonal tile: A lo = lo, B lo = 2 lo (exact in fp16)
            tc::st_shared_v4(stage + kALo + off_c, cl[0], cl[1], cl[2], cl[3]);
            tc::st_shared_v4(stage + kALo + off_s, sl[0], sl[1], sl[2], sl[3]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __half2 h = *reinterpret_cast<__half2*>(&cl[j]);
              h = __hadd2(h, h);
              cl[j] = *reinterpret_cast<uint32_t*>(&h);
              h = *reinterpret_cast<__half2*>(&sl[j]);
              h = __hadd2(h, h);
              sl[j] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          tc::st_shared_v4(sb + kBLo + off_c, cl[0], cl[1], cl[2], cl[3]);
          tc::st_shared_v4(sb + kBLo + off_s, sl[0], sl[1], sl[2], sl[3]);
        } else {  // A only
          tc::st_shared_v4(stage + kAHi + off_c, ch_[0], ch_[1], ch_[2], ch_[3]);
          tc::st_shared_v4(stage + kAHi + off_s, sh[0], sh[1], sh[2], sh[3]);
          tc::st_shared_v4(stage + kALo + off_c, cl[0], cl[1], cl[2], cl[3]);
          tc::st_shared_v4(stage + kALo + off_s, sl[0], sl[1], sl[2], sl[3]);
        }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(&full_bar[s]);
        if (it % kChunkSteps == kChunkSteps - 1 || it == nsteps - 1)
          tc::mbar_arrive(&pts_empty[ch % kChunks]);  // done with this chunk's points
      }
      if (elast) {
        if (pend1 >= 0) {  // queue full: the oldest epoch's MMAs are all issued
          RFD_WAIT(&accf_bar, uint32_t(pend0) & 1u, 7, it);
          __syncwarp();
          drain0();
        }
        const int info = (cta + bu) | ((nb - 1) << 28) | (k < kEpoch ? (1 << 29) : 0) |
                         (it + 1 == seg_hi ? (1 << 30) : 0);
        if (pend0 < 0) {
          pend0 = epoch;
          info0 = info;
          last0 = it;
        } else {
          pend1 = epoch;
          info1 = info;
          last1 = it;
        }
        ++epoch;
      }
    }
    while (pend0 >= 0) {
      RFD_WAIT(&accf_bar, uint32_t(pend0) & 1u, 8, nsteps);
      __syncwarp();
      drain0();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// K2: G[b] (interleaved r x r, fp64) from the segment partials, fixed order.
// grid: (16 chunks x upper tiles, batch); tile (bi <= bj) of the block grid.
__global__ void __launch_bounds__(256)
gram_tc_reduce_kernel(const float* __restrict__ partial, int m, const __grid_constant__ Sched sc,
                      double* __restrict__ G) {
  __shared__ int segs[kMaxCtas];
  __shared__ int nseg_sh;
  const int b = blockIdx.y;
  const int T = sc.T, r = 2 * m;
  int tile = blockIdx.x >> 4;
  const int chunk = blockIdx.x & 15;
  int bi = 0, row = T;
  while (tile >= row) {
    tile -= row;
    ++bi;
    --row;
  }
  const int bj = bi + tile;
  // the unit and accumulator tile holding (bi, bj), directly or transposed
  int unit = 0, tau = 0;
  bool transposed = false, found = false;
  for (int u = 0; u < sc.U && !found; ++u) {
    GramUnit X;
    gram_units(T, u, &X);
    for (int t = 0; t < X.nb && !found; ++t) {
      if (X.a == bi && X.b[t] == bj) {
        unit = u; tau = t; transposed = false; found = true;
      } else if (X.a == bj && X.b[t] == bi) {
        unit = u; tau = t; transposed = true; found = true;
      }
    }
  }
  const int64_t bu = int64_t(b) * sc.U + unit;
  if (threadIdx.x == 0) {
    int ns = 0;
    const int64_t lo = bu * sc.S, hi = (bu + 1) * sc.S;
    for (int c = 0; c < sc.G; ++c)
      if (sc.start[c] < sc.start[c + 1] && sc.start[c] < hi && sc.start[c + 1] > lo)
        segs[ns++] = int(c + bu);
    nseg_sh = ns;
  }
  __syncthreads();
  const int nseg = nseg_sh;
  const bool diag = (bi == bj);
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    const int e = chunk * 1024 + i * 256 + threadIdx.x;
    const int rr = e >> 7, cc = e & 127;  // cc fastest: coalesced partial reads
    const int fr = bi * kFreqs + (rr & 63), fc = bj * kFreqs + (cc & 63);
    if (fr >= m || fc >= m) continue;
    // partial[seg][row (128)][col (256)]; element (x, y) of tile tau at x*256 + tau*128 + y
    const int64_t o1 = transposed ? int64_t(cc) * 256 + tau * 128 + rr
                                  : int64_t(rr) * 256 + tau * 128 + cc;
    const int64_t o2 = int64_t(cc) * 256 + tau * 128 + rr;
    double s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < nseg; ++k) {
      const float* P = partial + int64_t(segs[k]) * (256 * 128);
      s1 += double(P[o1]);
      if (diag) s2 += double(P[o2]);
    }
    const double v = diag ? 0.5 * (s1 + s2) : s1;
    const int a = 2 * fr + (rr >> 6), c = 2 * fc + (cc >> 6);
    double* Gb = G + int64_t(b) * r * r;
    Gb[int64_t(a) * r + c] = v;
    Gb[int64_t(c) * r + a] = v;
  }
}

Sched make_sched(int m, int64_t n, int batch, int sms) {
  Sched sc{};
  sc.T = (m + kFreqs - 1) / kFreqs;
  sc.U = gram_units(sc.T, -1, nullptr);
  sc.batch = batch;
  sc.S = (n + kStep - 1) / kStep;
  const int64_t items = int64_t(batch) * sc.U * sc.S;
  int G = std::min(sms, kMaxCtas);
  if (int64_t(G) > items) G = int(items);
  sc.G = G;
  // cost of one K-step of each unit: max(MMA cycles, MUFU cycles)
  std::vector<int64_t> wgt(sc.U), pw(sc.U + 1, 0);
  for (int u = 0; u < sc.U; ++u) {
    GramUnit X;
    gram_units(sc.T, u, &X);
    int prod = 0, nloc = 1;
    for (int t = 0; t < X.nb; ++t) {
      prod += (X.b[t] == X.a) ? 2 : 3;
      if (X.b[t] != X.a) ++nloc;
    }
    wgt[u] = std::max<int64_t>(int64_t(prod) * 128, int64_t(nloc) * 256);
    pw[u + 1] = pw[u] + wgt[u];
  }
  const int64_t Wc = sc.S * pw[sc.U];
  const int64_t total = int64_t(batch) * Wc;
  for (int c = 0; c <= G; ++c) {
    const int64_t target = (c == G) ? total : int64_t((__int128)total * c / G);
    const int64_t b = target / Wc, rem = target - b * Wc;
    int u = 0;
    while (u + 1 < sc.U && pw[u + 1] * sc.S <= rem) ++u;
    const int64_t tt = (rem - pw[u] * sc.S + wgt[u] - 1) / wgt[u];
    int64_t L = (b * sc.U + u) * sc.S + tt;
    if (L > items) L = items;
    sc.start[c] = L;
  }
  sc.start[G] = items;
  return sc;
}


// ============================================================== CTA pairs
// Gram on CTA pairs (tcgen05 cta_group::2), used when there are >= 2 feature
// blocks.  Super-blocks of 256 features (2 blocks); a *pair-tile* (I <= J) is
// the 256 x 256 tile of super-blocks I and J, one MMA of M = N = 256 per
// K-slice on the SM pair.  CTA c of the pair holds A rows = block 2I + c and
// B rows = block 2J + c, so each SM generates half the features the tile
// needs (on a diagonal pair-tile A = B: one block per SM) and reads half the
// B operand -- twice the MMA work per generated feature of the 1-SM design.
// Diagonal pair-tiles use the symmetric two-product form (B lo = 2 lo, G =
// (D + D^T) / 2 over the 256 x 256 tile); off-diagonal ones three products.
// Each CTA accumulates its 128 rows in its own TMEM (epoch D + long-term L, as
// above) and writes them to the segment partial (256 x 256 per segment).
// Barriers: full / acce live in the leader (rank 0), arrived on by both CTAs
// (release at cluster scope); empty / accf are committed to both CTAs by the
// leader's MMA (multicast); the point ring is per CTA.

__host__ __device__ inline void pair_tile(int TS, int u, int& I, int& J) {
  int i = 0, row = TS;
  while (u >= row) {
    u -= row;
    ++i;
    --row;
  }
  I = i;
  J = i + u;
}

constexpr uint32_t kPAHi = 0, kPALo = kOpBytes, kPBHi = 2 * kOpBytes, kPBLo = 3 * kOpBytes;
constexpr uint32_t kPStageBytes = 4 * kOpBytes;                 // 64 KB
constexpr int kPStages = 3;
// Epoch of the pair kernel: 16 K-steps (1024 points).  Used for >= 2 feature
// blocks only (cfg 4: G, C^, Delta errors stay <= ~1.5e-5);
// the 1-SM kernel (small m, e.g. the 2048-point clouds of cfg 3) keeps 512.
constexpr int kPEpoch = 16;
constexpr int kPRingOff = kPStages * int(kPStageBytes);          // 192 KB
constexpr int kPOmegaOff = kPRingOff + kChunks * int(kChunkBytes);
constexpr int kPSmemBytes = kPOmegaOff + kMaxFreqs * 16;         // 216 KB

// kWeighted: G = sum_p w_p^2 phi(x_p) phi(x_p)^T with w_p in the pad slot of
// the point layout (the grid Gram of the spread path, k_nufft.cu).
template <bool kTrace, bool kWeighted = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gram_pair_kernel(const unsigned char* __restrict__ gpts, const float4* __restrict__ omega4, int m,
                 int64_t n, const __grid_constant__ Sched sc, float* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kPStages], empty_bar[kPStages], pts_bar[kChunks],
      pts_empty[kChunks];
  __shared__ uint64_t accf_bar, acce_bar;
  __shared__ uint32_t tmem_sh;

  const uint32_t rank = tc::cluster_rank();
  const int pair = blockIdx.x >> 1;
  const int64_t L0 = sc.start[pair], L1 = sc.start[pair + 1];
  if (L0 >= L1) return;  // both CTAs of the pair
  const int nsteps = int(L1 - L0);
  const int Si = int(sc.S);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = tc::smem_addr(smem);
  // diagnostics (RFD_GRAM_MODE=6): steps kTr0 .. kTr0 + 127 of CTA g_trace_cta,
  // timestamps in shared memory (cheap), copied out at the end
  __shared__ long long gtr[kTrace ? 128 : 1][8];
  constexpr int kTr0 = 400;
  const bool trc = kTrace && int(blockIdx.x) == g_trace_cta;

  if (tid == 0) {
    // full / acce: the CTA's 16 warps, plus (leader) the follower's relay
    for (int s = 0; s < kPStages; ++s) {
      tc::mbar_init(&full_bar[s], kProducerWarps + (rank == 0 ? 1 : 0));
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int c = 0; c < kChunks; ++c) {
      tc::mbar_init(&pts_bar[c], 1);
      tc::mbar_init(&pts_empty[c], kProducerWarps);
    }
    tc::mbar_init(&accf_bar, 1);
    tc::mbar_init(&acce_bar, kProducerWarps * (rank == 0 ? 2 : 1));
    tc::mbar_fence_init();
  }
  {  // omega table (rows of padding frequencies >= m are zero)
    float4* om_s = reinterpret_cast<float4*>(smem + kPOmegaOff);
    for (int k = tid; k < 2 * sc.T * kFreqs; k += kThreads)
      om_s[k] = (k < m) ? __ldg(omega4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (warp == 0) tc::tmem_alloc_pair<512>(&tmem_sh);
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;

  const int bu0 = int(L0 / sc.S), t0 = int(L0 - int64_t(bu0) * sc.S);
  const int hi0 = int(min(L1, int64_t(bu0 + 1) * sc.S) - L0);

  if (warp == kLoadWarp) {
    // ============================================ point loads (per CTA)
    const int nchunks = (nsteps + kChunkSteps - 1) / kChunkSteps;
    const int64_t cloud_bytes = int64_t(Si) * kStepBytes;
    int l_bu = bu0, l_t = t0;
    for (int ch = 0; ch < nchunks; ++ch) {
      if (ch >= kChunks) tc::mbar_wait(&pts_empty[ch % kChunks], uint32_t(ch / kChunks - 1) & 1u);
      const int i0 = ch * kChunkSteps, i1 = min(nsteps, i0 + kChunkSteps);
      uint64_t* bar = &pts_bar[ch % kChunks];
      unsigned char* dst = smem + kPRingOff + (ch % kChunks) * kChunkBytes;
      if (lane == 0) {
        tc::mbar_arrive_expect_tx(bar, uint32_t(i1 - i0) * kStepBytes);
        for (int i = i0; i < i1;) {
          const int run = min(i1 - i, Si - l_t);
          tc::bulk_g2s(dst + (i - i0) * kStepBytes,
                       gpts + int64_t(l_bu / sc.U) * cloud_bytes + int64_t(l_t) * kStepBytes,
                       uint32_t(run) * kStepBytes, bar);
          i += run;
          l_t += run;
          if (l_t == Si) {
            l_t = 0;
            ++l_bu;
          }
        }
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ============================================ MMA issue (leader) / relay (follower)
    if (rank == 1) {
      // Relay: the follower's producers arrive on its local full barriers
      // (release at CTA scope: cheap); one thread forwards each completed
      // phase to the leader with ONE release at cluster scope (that arrive
      // compiles to MEMBAR.GPU + L1 invalidate: too costly per warp and step).
      // The drains (once per epoch) arrive on the leader's acce directly.
      if (lane == 0) {
        const uint32_t full_lead0 = tc::mapa(&full_bar[0], 0);
        for (int fi = 0; fi < nsteps; ++fi) {
          tc::mbar_wait(&full_bar[fi % kPStages], uint32_t(fi / kPStages) & 1u);
          tc::mbar_arrive_cluster(full_lead0 + 8u * uint32_t(fi % kPStages));
        }
      }
      __syncwarp();
    } else {
      const uint32_t idesc = tc::make_idesc(0, 256, 256);
      int m_lo = 0, m_hi = hi0, m_bu = bu0, epoch = 0;
      auto is_diag = [&](int u) {
        int I, J;
        pair_tile(sc.T, u, I, J);
        return I == J;
      };
      bool diag = is_diag(m_bu % sc.U);
      for (int it = 0; it < nsteps; ++it) {
        const int s = it % kPStages;
        const int k = it - m_lo;
        const bool efirst = (k & (kPEpoch - 1)) == 0;
        const bool elast = ((k + 1) & (kPEpoch - 1)) == 0 || it + 1 == m_hi;
        if (efirst && epoch > 0) tc::mbar_wait_cluster(&acce_bar, uint32_t(epoch - 1) & 1u);
        if (kTrace && trc && (lane == 0) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][0] = clock64();
        tc::mbar_wait_cluster(&full_bar[s], uint32_t(it / kPStages) & 1u);
        if (kTrace && trc && (lane == 0) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][1] = clock64();
        tc::tc_fence_after();
        __syncwarp();
        const uint32_t stage = sbase + uint32_t(s) * kPStageBytes;
        if (tc::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kStep / 16; ++kk) {
            const uint32_t ko = uint32_t(kk) * 2u * kLBO;
            const uint64_t ahi = tc::make_sdesc(stage + kPAHi + ko, kLBO, kSBO);
            const uint64_t blo = tc::make_sdesc(stage + kPBLo + ko, kLBO, kSBO);
            const uint32_t acc0 = (efirst && kk == 0) ? 0u : 1u;
            if (diag) {  // A = B = H:  D += H H^T + H (2L)^T
              tc::mma_f16_pair(tmem, ahi, ahi, idesc, acc0);
              tc::mma_f16_pair(tmem, ahi, blo, idesc, 1u);
            } else {
              const uint64_t alo = tc::make_sdesc(stage + kPALo + ko, kLBO, kSBO);
              const uint64_t bhi = tc::make_sdesc(stage + kPBHi + ko, kLBO, kSBO);
              tc::mma_f16_pair(tmem, ahi, bhi, idesc, acc0);
              tc::mma_f16_pair(tmem, ahi, blo, idesc, 1u);
              tc::mma_f16_pair(tmem, alo, bhi, idesc, 1u);
            }
          }
          tc::mma_commit_pair(&empty_bar[s]);
          if (elast) tc::mma_commit_pair(&accf_bar);
        }
        __syncwarp();
        if (elast) ++epoch;
        if (it + 1 == m_hi && it + 1 < nsteps) {
          ++m_bu;
          m_lo = it + 1;
          m_hi = min(nsteps, it + 1 + Si);
          diag = is_diag(m_bu % sc.U);
        }
      }
    }
  } else {
    // ============================================ producers (+ drains)
    const unsigned char* ring = smem + kPRingOff;
    const float4* om_s = reinterpret_cast<const float4*>(smem + kPOmegaOff);
    const int q = warp & 7, f = 32 * (warp >> 3) + lane;
    const uint32_t off_c = uint32_t(f >> 3) * kSBO + uint32_t(q) * kLBO + uint32_t(f & 7) * 16u;
    const uint32_t off_s = off_c + 8u * kSBO;  // row 64 + f
    const int lg = warp & 3, qd = warp >> 2;
    const uint32_t lane_field = uint32_t(32 * lg) << 16;
    const int rho = 32 * lg + lane;
    // blocks of this CTA: A = 2I + rank, B = 2J + rank (diag: the same block)
    int blkA = 0, blkB = 0;
    bool diag = true;
    auto setup_unit = [&](int u) {
      int I, J;
      pair_tile(sc.T, u, I, J);
      blkA = 2 * I + int(rank);
      blkB = 2 * J + int(rank);
      diag = I == J;
    };
    int pend0 = -1, pend1 = -1, info0 = 0, info1 = 0, last0 = 0, last1 = 0;
    const uint32_t acce_lead = tc::mapa(&acce_bar, 0);
    auto drain0 = [&]() {
      drain_epoch(tmem + lane_field, qd, lane, 2, (info0 >> 29) & 1, (info0 >> 30) & 1,
                  partial + (int64_t(info0 & 0x0FFFFFFF) * 256 + 128 * rank + rho) * 256,
                  nullptr, false);
      if (lane == 0) {  // D is free again (the follower's drains: on the leader's barrier)
        if (rank == 0) tc::mbar_arrive(&acce_bar);
        else tc::mbar_arrive_cluster(acce_lead);
      }
      pend0 = pend1;
      info0 = info1;
      last0 = last1;
      pend1 = -1;
    };
    const int tail = int(n - int64_t(Si - 1) * kStep);
    int bu = bu0, seg_lo = 0, seg_hi = hi0, tail_it = Si - 1 - t0;
    setup_unit(bu % sc.U);
    int epoch = 0;
    for (int it = 0; it < nsteps; ++it) {
      if (it == seg_hi) {
        ++bu;
        seg_lo = it;
        seg_hi = min(nsteps, it + Si);
        tail_it = it + Si - 1;
        setup_unit(bu % sc.U);
      }
      const int k = it - seg_lo;
      const bool elast = ((k + 1) & (kPEpoch - 1)) == 0 || it + 1 == seg_hi;
      const int s = it % kPStages;
      const uint32_t ph = uint32_t(it / kPStages) & 1u;
      const int ch = it / kChunkSteps;
      // drain as soon as the epoch's MMAs are complete (non-parking probe), and
      // at the latest before a step whose stage needs a later epoch's MMA
      while (pend0 >= 0) {
        if (it - kPStages > last0)
          tc::mbar_wait(&accf_bar, uint32_t(pend0) & 1u);
        else if (!__any_sync(0xffffffffu, tc::mbar_test_wait(&accf_bar, uint32_t(pend0) & 1u)))
          break;
        __syncwarp();
        drain0();
      }
      if (kTrace && trc && (tid == 160) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][2] = clock64();
      if (it >= kPStages) tc::mbar_wait(&empty_bar[s], ph ^ 1u);
      if (it % kChunkSteps == 0 || it == 0)
        tc::mbar_wait(&pts_bar[ch % kChunks], uint32_t(ch / kChunks) & 1u);
      __syncwarp();
      if (kTrace && trc && (tid == 160) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][3] = clock64();
      const int cnt = (it == tail_it) ? tail : kStep;
      const float* grp = reinterpret_cast<const float*>(
          ring + (ch % kChunks) * kChunkBytes + (it % kChunkSteps) * kStepBytes + q * kGroupBytes);
      float X[8], Y[8], Z[8], Wt[8];
#pragma unroll
      for (int j = 0; j < 8; j += 4) {
        *reinterpret_cast<float4*>(X + j) = *reinterpret_cast<const float4*>(grp + j);
        *reinterpret_cast<float4*>(Y + j) = *reinterpret_cast<const float4*>(grp + 8 + j);
        *reinterpret_cast<float4*>(Z + j) = *reinterpret_cast<const float4*>(grp + 16 + j);
        if (kWeighted)
          *reinterpret_cast<float4*>(Wt + j) = *reinterpret_cast<const float4*>(grp + 24 + j);
      }
      const uint32_t stage = sbase + uint32_t(s) * kPStageBytes;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (i == 1 && diag) break;
        const int blk = (i == 0) ? blkA : blkB;
        const float4 wi = om_s[blk * kFreqs + f];
        const float2 wx = make_float2(wi.x, wi.x), wy = make_float2(wi.y, wi.y),
                     wz = make_float2(wi.z, wi.z);
        float c[8], sn[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const float2 th = __ffma2_rn(wz, make_float2(Z[j], Z[j + 1]),
                                       __ffma2_rn(wy, make_float2(Y[j], Y[j + 1]),
                                                  __fmul2_rn(wx, make_float2(X[j], X[j + 1]))));
          __sincosf(th.x, &sn[j], &c[j]);
          __sincosf(th.y, &sn[j + 1], &c[j + 1]);
        }
        if (kWeighted) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            c[j] *= Wt[j];
            sn[j] *= Wt[j];
          }
        }
        if (cnt < kStep) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (q * 8 + j >= cnt) c[j] = sn[j] = 0.0f;
        }
        uint32_t ch_[4], cl[4], sh[4], sl[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          tc::split_f16x2_v2(make_float2(c[2 * j], c[2 * j + 1]), ch_[j], cl[j]);
          tc::split_f16x2_v2(make_float2(sn[2 * j], sn[2 * j + 1]), sh[j], sl[j]);
        }
        const uint32_t hiR = stage + ((i == 0) ? kPAHi : kPBHi);
        tc::st_shared_v4(hiR + off_c, ch_[0], ch_[1], ch_[2], ch_[3]);
        tc::st_shared_v4(hiR + off_s, sh[0], sh[1], sh[2], sh[3]);
        if (diag) {  // B lo = 2 lo (exact in fp16); no A lo
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            __half2 h = *reinterpret_cast<__half2*>(&cl[j]);
            h = __hadd2(h, h);
            cl[j] = *reinterpret_cast<uint32_t*>(&h);
            h = *reinterpret_cast<__half2*>(&sl[j]);
            h = __hadd2(h, h);
            sl[j] = *reinterpret_cast<uint32_t*>(&h);
          }
        }
        const uint32_t loR = stage + ((i == 0 && !diag) ? kPALo : kPBLo);
        tc::st_shared_v4(loR + off_c, cl[0], cl[1], cl[2], cl[3]);
        tc::st_shared_v4(loR + off_s, sl[0], sl[1], sl[2], sl[3]);
      }
      if (kTrace && trc && (tid == 160) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][4] = clock64();
      // a second, mid-step probe: the MMA warp idles until the drain is done
      if (pend0 >= 0 && __any_sync(0xffffffffu, tc::mbar_test_wait(&accf_bar, uint32_t(pend0) & 1u))) {
        __syncwarp();
        drain0();
      }
      if (kTrace && trc && (tid == 160) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][5] = clock64();
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (kTrace && trc && (tid == 160) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][6] = clock64();
      if (lane == 0) {
        tc::mbar_arrive(&full_bar[s]);  // leader: counted; follower: relayed
        if (it % kChunkSteps == kChunkSteps - 1 || it == nsteps - 1)
          tc::mbar_arrive(&pts_empty[ch % kChunks]);
      }
      if (elast) {
        if (pend1 >= 0) {
          tc::mbar_wait(&accf_bar, uint32_t(pend0) & 1u);
          __syncwarp();
          drain0();
        }
        const int info = (pair + bu) | (k < kPEpoch ? (1 << 29) : 0) |
                         (it + 1 == seg_hi ? (1 << 30) : 0);
        if (pend0 < 0) {
          pend0 = epoch;
          info0 = info;
          last0 = it;
        } else {
          pend1 = epoch;
          info1 = info;
          last1 = it;
        }
        ++epoch;
      }
      if (kTrace && trc && (tid == 160) && unsigned(it - kTr0) < 128u) gtr[it - kTr0][7] = clock64();
    }
    while (pend0 >= 0) {
      tc::mbar_wait(&accf_bar, uint32_t(pend0) & 1u);
      __syncwarp();
      drain0();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (kTrace && trc)
    for (int i = tid; i < 128 * 8; i += kThreads) g_trace[i / 8][i % 8] = gtr[i / 8][i % 8];
  tc::cluster_sync();
  if (warp == 0) tc::tmem_dealloc_pair<512>(tmem);
}

// K2 (pairs), two steps: (1) Dsum[b][unit] = the fixed-order fp64 sum of the
// unit's segment partials, every element read coalesced once per segment;
// (2) G from Dsum, on diagonal pair tiles G = (D + D^T) / 2 (the transposed
// read touches the 256 x 256 sum once, not once per segment).
__global__ void __launch_bounds__(256)
gram_pair_sum_kernel(const float* __restrict__ partial, const __grid_constant__ Sched sc,
                     double* __restrict__ Dsum) {
  __shared__ int segs[kMaxCtas];
  __shared__ int nseg_sh;
  const int b = blockIdx.z, unit = blockIdx.y;
  const int64_t bu = int64_t(b) * sc.U + unit;
  if (threadIdx.x == 0) {
    int ns = 0;
    const int64_t lo = bu * sc.S, hi = (bu + 1) * sc.S;
    for (int c = 0; c < sc.G; ++c)
      if (sc.start[c] < sc.start[c + 1] && sc.start[c] < hi && sc.start[c + 1] > lo)
        segs[ns++] = int(c + bu);
    nseg_sh = ns;
  }
  __syncthreads();
  const int nseg = nseg_sh;
  const int e = blockIdx.x * 256 + threadIdx.x;  // 0 .. 65535
  double acc = 0.0;
  for (int k = 0; k < nseg; ++k) acc += double(partial[int64_t(segs[k]) * (256 * 256) + e]);
  Dsum[bu * (256 * 256) + e] = acc;
}

__global__ void __launch_bounds__(256)
gram_pair_write_kernel(const double* __restrict__ Dsum, int m, const __grid_constant__ Sched sc,
                       double* __restrict__ G) {
  const int b = blockIdx.z;
  const int r = 2 * m;
  const int e = blockIdx.x * 256 + threadIdx.x;  // (a, c) over the r x r upper triangle
  const int a = e / r, c = e - (e / r) * r;
  if (a >= r || c < a) return;
  // a = 2 f + (sin), block of the feature = f / 64, super-block = block / 2
  const int fa = a >> 1, fc = c >> 1;
  int bi = fa / kFreqs, bj = fc / kFreqs;
  int rr = (fa % kFreqs) + 64 * (a & 1), cc = (fc % kFreqs) + 64 * (c & 1);
  int x = 128 * (bi & 1) + rr, y = 128 * (bj & 1) + cc;
  int I = bi >> 1, J = bj >> 1;
  if (I > J) {  // (only when a's super-block exceeds c's: not in the upper triangle of blocks)
    const int t = I; I = J; J = t;
    const int u = x; x = y; y = u;
  }
  int unit = 0;
  for (int i = 0; i < I; ++i) unit += sc.T - i;
  unit += J - I;
  const double* D = Dsum + (int64_t(b) * sc.U + unit) * (256 * 256);
  const double v = (I == J) ? 0.5 * (D[x * 256 + y] + D[y * 256 + x]) : D[x * 256 + y];
  double* Gb = G + int64_t(b) * r * r;
  Gb[int64_t(a) * r + c] = v;
  Gb[int64_t(c) * r + a] = v;
}

Sched make_pair_sched(int m, int64_t n, int batch, int sms) {
  Sched sc{};
  const int T = (m + kFreqs - 1) / kFreqs;
  sc.T = (T + 1) / 2;  // super-blocks
  sc.U = sc.T * (sc.T + 1) / 2;
  sc.batch = batch;
  sc.S = (n + kStep - 1) / kStep;
  const int64_t items = int64_t(batch) * sc.U * sc.S;
  int G = std::min(sms, 2 * kMaxCtas) / 2;
  if (int64_t(G) > items) G = int(items);
  sc.G = G;
  // cost of one K-step: diagonal 8 pair-MMAs, off-diagonal 12 (x 128 cycles)
  std::vector<int64_t> wgt(sc.U), pw(sc.U + 1, 0);
  for (int u = 0; u < sc.U; ++u) {
    int I, J;
    pair_tile(sc.T, u, I, J);
    wgt[u] = (I == J) ? 2 : 3;
    pw[u + 1] = pw[u] + wgt[u];
  }
  const int64_t Wc = sc.S * pw[sc.U];
  const int64_t total = int64_t(batch) * Wc;
  for (int c = 0; c <= G; ++c) {
    const int64_t target = (c == G) ? total : int64_t((__int128)total * c / G);
    const int64_t b = target / Wc, rem = target - b * Wc;
    int u = 0;
    while (u + 1 < sc.U && pw[u + 1] * sc.S <= rem) ++u;
    const int64_t tt = (rem - pw[u] * sc.S + wgt[u] - 1) / wgt[u];
    int64_t L = (b * sc.U + u) * sc.S + tt;
    if (L > items) L = items;
    sc.start[c] = L;
  }
  sc.start[G] = items;
  return sc;
}

// CTA pairs from two 64-frequency blocks on (one pair-tile = 256 features).
bool use_pairs(int m) { return (m + kFreqs - 1) / kFreqs >= 2; }

}  // namespace

GramGeom gram_tc_geometry(int m, int64_t n, int batch, int sms) {
  const bool pairs = use_pairs(m);
  const Sched sc = pairs ? make_pair_sched(m, n, batch, sms) : make_sched(m, n, batch, sms);
  GramGeom g;
  g.r = 2 * m;
  g.tile = pairs ? 2 * kBlk : kBlk;  // 256: CTA-pair path
  g.tiles1d = sc.T;
  g.ntiles = sc.U;   // units
  g.chunks = sc.G;   // persistent CTAs
  g.chunk = sc.S;    // K-steps per unit
  return g;
}

// one partial per (CTA, unit segment) -- segment id = cta + cloud * U + unit --
// followed by the points in the Gram layout (S K-steps per cloud)
static size_t gram_tc_partial_only(const GramGeom& g, int batch) {
  return size_t(g.chunks + int64_t(batch) * g.ntiles) * 256 * g.tile;
}
// pair path: then the fp64 unit sums of the two-step reduce (16-byte aligned)
static size_t gram_tc_dsum_offset(const GramGeom& g, int batch) {
  return (gram_tc_partial_only(g, batch) + size_t(batch) * size_t(g.chunk) * (kStepBytes / 4) + 3) &
         ~size_t(3);
}
size_t gram_tc_partial_elems(const GramGeom& g, int batch) {
  const bool pairs = g.tile == 2 * kBlk;
  return gram_tc_dsum_offset(g, batch) +
         (pairs ? size_t(batch) * size_t(g.ntiles) * (256 * 256) * 2 : 0);
}
float* gram_points(const GramGeom& g, int batch, float* partial, int64_t* per_cloud) {
  *per_cloud = int64_t(g.chunk) * kStep;
  return partial + gram_tc_partial_only(g, batch);
}

bool gram_tc_pairs(int m) { return use_pairs(m); }

void launch_gram_tc(const float4* omega4, int m, int64_t n, int batch,
                    const GramGeom& g, float* partial, double* G, cudaStream_t s, bool weighted) {
  const bool pairs = g.tile == 2 * kBlk;
  // same partition as gram_tc_geometry (G = g.chunks CTAs or CTA pairs)
  const Sched sc = pairs ? make_pair_sched(m, n, batch, 2 * g.chunks)
                         : make_sched(m, n, batch, g.chunks);
  static bool configured = false;
  static bool trace = false;
  if (!configured) {
    cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    cudaFuncSetAttribute(gram_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kPSmemBytes);
    cudaFuncSetAttribute(gram_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kPSmemBytes);
    cudaFuncSetAttribute(gram_pair_kernel<false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmemBytes);
    const char* e = getenv("RFD_GRAM_TRACE");  // instrumentation only
    trace = e && e[0] == '1';
    configured = true;
  }
  // the points in the Gram layout were written by the pack kernel (gram_points)
  const float* gpts = partial + gram_tc_partial_only(g, batch);
  const unsigned char* gp = reinterpret_cast<const unsigned char*>(gpts);
  if (pairs) {
    {
      LaunchScope L("rfd_gram_tc", s);
      if (weighted) {
        gram_pair_kernel<false, true><<<2 * sc.G, kThreads, kPSmemBytes, s>>>(gp, omega4, m, n,
                                                                              sc, partial);
      } else if (trace) {
        const char* tc_env = getenv("RFD_GRAM_TRACE_CTA");
        const int tcta = tc_env ? atoi(tc_env) : 0;
        cudaMemcpyToSymbol(g_trace_cta, &tcta, sizeof(int));
        gram_pair_kernel<true><<<2 * sc.G, kThreads, kPSmemBytes, s>>>(gp, omega4, m, n, sc, partial);
        static long long h[4096][8];
        cudaMemcpyFromSymbol(h, g_trace, sizeof(h));
        // averages (cycles per step) over the 127 traced steps
        double mw = 0, pw = 0, pc = 0, pp = 0, pf = 0, pe = 0, pt = 0, st = 0;
        const int i0 = 0, i1 = 127;
        for (int i = i0; i < i1; ++i) {
          mw += double(h[i][1] - h[i][0]);
          pw += double(h[i][3] - h[i][2]);
          pc += double(h[i][4] - h[i][3]);
          pp += double(h[i][5] - h[i][4]);
          pf += double(h[i][6] - h[i][5]);
          pe += double(h[i][7] - h[i][6]);
          pt += double(h[i + 1][2] - h[i][7]);
          st += double(h[i + 1][2] - h[i][2]);
        }
        const double k = 1.0 / (i1 - i0);
        fprintf(stderr, "cta %d avg/step: step %.0f | mma full-wait %.0f | prod wait %.0f compute %.0f probe %.0f fence %.0f arrive %.0f top %.0f\n",
                tcta, st * k, mw * k, pw * k, pc * k, pp * k, pf * k, pe * k, pt * k);
      } else {
        gram_pair_kernel<false><<<2 * sc.G, kThreads, kPSmemBytes, s>>>(gp, omega4, m, n, sc, partial);
      }
    }
    {
      LaunchScope L("rfd_gram_reduce", s);
      // Dsum: U x batch 256 x 256 fp64 behind the segment partials and points
      double* Dsum = reinterpret_cast<double*>(partial + gram_tc_dsum_offset(g, batch));
      gram_pair_sum_kernel<<<dim3(256, sc.U, batch), 256, 0, s>>>(partial, sc, Dsum);
      const int r = 2 * m;
      gram_pair_write_kernel<<<dim3(unsigned((int64_t(r) * r + 255) / 256), 1, batch), 256, 0, s>>>(
          Dsum, m, sc, G);
    }
    return;
  }
  {
    LaunchScope L("rfd_gram_tc", s);
    gram_tc_kernel<<<sc.G, kThreads, kSmemBytes, s>>>(gp, omega4, m, n, sc, partial);
  }
  {
    LaunchScope L("rfd_gram_reduce", s);
    const int tiles = sc.T * (sc.T + 1) / 2;
    gram_tc_reduce_kernel<<<dim3(16 * tiles, batch), 256, 0, s>>>(partial, m, sc, G);
  }
}

}  // namespace rfd
