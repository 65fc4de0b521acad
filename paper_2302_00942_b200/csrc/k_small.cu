// Narrow fields (d <= 4): the whole inference of Eq. 13 (PAPER.md:351-358,
// SURVEY Sec. 8(a) rows a3, a6-a8) in ONE persistent cooperative launch:
//
//   phase 1  S partials = Phi^T F per (cloud, point segment)      [a6]
//   barrier
//   phase 2  S = fixed-order sum of the segment partials (fp64)    [a7]
//   barrier
//   phase 3  Y = C^ S (fp64 -> fp32)                               [a7]
//   barrier
//   phase 4  out = F + Phi Y                                       [a8]
//
// With d <= 4 the contraction is 2d FMA per (point, frequency) -- a handful
// of FP32 instructions next to the sin/cos pair -- so the tensor-core passes'
// per-feature overheads (fp16 hi/lo splits, TMEM stores, MMA pipeline) cost
// more than the contraction they move; here every (point, frequency) is
// ~5.5 + d SIMT instructions and the pass is MUFU-bound.  One launch instead
// of 2-4 also takes the launch and pipeline-fill latency of small clouds
// (cfgs 1-3) off the critical path.
//
// Phase 1 is frequency-stationary: thread = (frequency k, point group g);
// the segment's points and field rows are staged in shared memory (SoA) and
// read as broadcasts, 4 consecutive points per 16-byte load, 2 per packed
// FP32 instruction; the 2 x d accumulators (cos, sin per channel) stay in
// registers, then the point groups are added in a fixed order.  Phase 4 is
// point-stationary: 2 points per thread, omega and Y broadcast from shared
// memory.  Features (a3) are regenerated in registers in both phases, as in
// the tensor-core passes: fp32(2 pi omega) . x (centred), MUFU sin/cos.
// Deterministic: fixed partition and reduction order, no floating-point
// atomics.  Interleaved feature order (2k cos, 2k + 1 sin) as everywhere.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kLocalThreads = 256, kWideThreads = 768;  // CTA sizes (see the kernel)
constexpr int kBatchPts = 512;  // points staged per phase-1 batch
// points per phase-4 tile: 2 per thread

// Generation barrier over the whole (co-resident) grid, two levels: CTAs
// arrive on one of 32 group counters (same-address atomics serialise at L2:
// ~8 us for 592 CTAs on one counter), the last CTA of each group on the top
// counter, whose last arrival resets the counters and advances the
// generation; the others poll the generation with acquire loads.  Release /
// acquire at gpu scope order each CTA's writes before the barrier with the
// reads after it (thread 0 acts for the CTA after __syncthreads).
// Self-resetting: every launch starts from zero counts.  bar: [0] generation,
// [1] top counter, [2 .. 34) group counters.
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int atom_add_acqrel(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
constexpr int kBarGroups = 32;
constexpr int kBarWords = 2 + kBarGroups;
static_assert(kBarWords == kSmallBarWords, "barrier words");

__device__ __forceinline__ void grid_sync(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int my = ld_acquire(bar);
    const unsigned int grp = blockIdx.x % kBarGroups;
    const unsigned int in_grp = (gridDim.x - grp + kBarGroups - 1) / kBarGroups;
    const unsigned int ngrp = gridDim.x < kBarGroups ? gridDim.x : kBarGroups;
    bool last = atom_add_acqrel(bar + 2 + grp, 1u) == in_grp - 1;
    if (last) last = atom_add_acqrel(bar + 1, 1u) == ngrp - 1;
    if (last) {
      for (unsigned int g = 0; g < ngrp; ++g) bar[2 + g] = 0u;
      bar[1] = 0u;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    } else {
      // relaxed polling with a short back-off (hundreds of CTAs polling one
      // word with acquire loads slow the release down), then one acquire fence
      unsigned int v;
      do {
        __nanosleep(40);
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      } while (v == my);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  __syncthreads();
}

struct SmallArgs;
__device__ __forceinline__ void sync_all(const SmallArgs& a);

struct SmallArgs {
  const float4* pts;     // batch x n, centred (x, y, z, 0): one array, clouds back to back
  const float4* omega4;  // m: fp32(2 pi omega)
  int m, fb, nfb;        // frequencies; frequency block (32..256, power of two); blocks
  int64_t n;
  int batch, d;
  int R;                 // phase-1 point ranges (gridDim = R x nfb)
  int64_t L;             // points per phase-1 range (multiple of 4)
  int K;                 // partial slots per range (clouds a range can touch)
  int64_t L4;            // points per phase-4 range (one per CTA)
  const float* F;        // (batch x) n x d
  float* out;            // same shape (may alias F)
  const double* C;       // batch x r x r
  float* part;           // K x r x d x R: slot (range c, its k-th cloud) at [(k r d + e) R + c]
  double* S;             // batch x r x d
  float* Y;              // batch x r x d
  unsigned int* bar;     // kBarWords words, zero before the first launch
  int fuse_a7;           // 1: S and Y per cloud in phase 4's prologue (small r)
  int local;             // 1: one CTA per cloud (ranges = clouds): no grid barrier at all
  unsigned long long* trace;  // diagnostics (RFD_SMALL_TRACE=1): phase timestamps of CTA 0
};

// local mode: every CTA reads only what it wrote itself (its cloud's slot),
// so a CTA barrier orders phase 1's global writes before the reads
__device__ __forceinline__ void sync_all(const SmallArgs& a) {
  if (a.local) __syncthreads();
  else grid_sync(a.bar);
}

__device__ __forceinline__ void stamp(unsigned long long* tr, int i) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[i] = t;
  }
}
__device__ unsigned long long g_small_trace[8];
__device__ unsigned long long g_small_p1end[1024];  // trace: each CTA's end of phase 1
__device__ unsigned long long g_small_p1beg[1024];  // trace: each CTA's start
__device__ unsigned int g_small_smid[1024];
__device__ unsigned long long g_small_p4end[1024];  // trace: each CTA's end

// S[b][row][j] = sum over the ranges overlapping cloud b, in range order, of
// their slot for b (fp64).  Range c overlaps b iff [cL, cL+L) meets [bn, bn+n).
__device__ __forceinline__ double sum_slots(const SmallArgs& a, int b, int row, int j) {
  const int r = 2 * a.m;
  const int64_t lo = int64_t(b) * a.n, hi = lo + a.n;
  const int c0 = int(lo / a.L), c1 = int((hi - 1) / a.L);
  double acc = 0.0;
  for (int c = c0; c <= c1; ++c) {
    const int k = b - int((int64_t(c) * a.L) / a.n);
    acc += double(__ldg(a.part + ((int64_t(k) * r + row) * a.d + j) * a.R + c));
  }
  return acc;
}

// NT threads per CTA: 256 (3 CTAs per SM) in local mode; 768 (one CTA per
// SM) otherwise -- the same warps per SM for the MUFU work, a third of the
// phase-1 ranges for phase 2 to sum and of the CTAs in every grid barrier,
// and no uneven sharing of an SM by three CTAs (cfg 4: the SM's last CTA
// finished phase 1 at ~60 % of the MUFU rate; 58 -> see DESIGN.md).
template <int D, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : 1)
integrate_small_kernel(const SmallArgs a) {
  constexpr int kThreads = NT, kTilePts = 2 * NT;
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = 2 * a.m;
  const int d = a.d;
  const int64_t ntot = int64_t(a.batch) * a.n;
  stamp(a.trace, 0);
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    unsigned long long t;
    unsigned int sid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sid));
    g_small_p1beg[blockIdx.x] = t;
    g_small_smid[blockIdx.x] = sid;
  }

  // ------------------------------------------------ phase 1: S partials
  // CTA = (range c, frequency block f): the range's points in batches of <= 512
  // (never across a cloud boundary), one partial slot per (range, cloud) --
  // equal ranges: every CTA gets the same number of points whatever the
  // cloud sizes.  Batches are double-buffered: the next one is copied
  // (cp.async, global latency hidden) while this one is consumed.
  {
    // KF frequencies per thread (kk0, kk0 + fb / KF, ...): each broadcast
    // point / field load serves KF frequencies (2 in the wide CTAs: the
    // shared-memory loads share the MIO queue with MUFU)
    constexpr int KF = (NT == 768) ? 2 : 1;
    const int fbh = a.fb / KF;
    const int G = kThreads / fbh;  // point groups
    const int g = tid / fbh, kk0 = tid % fbh;
    const int c = blockIdx.x / a.nfb, fbk = blockIdx.x % a.nfb;
    // buffer b: points at sm + b * kBufF (float4 x 512), field rows after them
    constexpr int kBufF = (4 + D) * kBatchPts;  // floats per buffer
    auto pbuf = [&](int b) { return reinterpret_cast<float4*>(sm + b * kBufF); };
    auto fbuf = [&](int b) { return sm + b * kBufF + 4 * kBatchPts; };
    float* red = sm + 2 * kBufF;  // [G][fb][2D]
    float2 wx[KF], wy[KF], wz[KF];
#pragma unroll
    for (int u = 0; u < KF; ++u) {
      const int k = fbk * a.fb + kk0 + u * fbh;
      const float4 w = (k < a.m) ? a.omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
      wx[u] = make_float2(w.x, w.x);
      wy[u] = make_float2(w.y, w.y);
      wz[u] = make_float2(w.z, w.z);
    }
    const int64_t r0 = int64_t(c) * a.L, r1 = min(r0 + a.L, ntot);
    const int bfirst = int(r0 / a.n);
    // batch i: [start, end) -- at most 512 points, within one cloud
    auto batch_end = [&](int64_t start) {
      const int64_t cend = (start / a.n + 1) * a.n;
      return min(min(start + kBatchPts, r1), cend);
    };
    auto issue = [&](int64_t start, int64_t end, int buf) {
      const int np = int(end - start), np4 = (np + 3) & ~3;
      for (int i = tid; i < np4; i += kThreads) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(pbuf(buf) + i));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                     "l"(a.pts + (i < np ? start + i : start)), "r"(i < np ? 16 : 0) : "memory");
      }
      // F rows of the batch: np * D floats, contiguous, 16-byte chunks (zero-filled tail)
      const float* src = a.F + start * D;
      const int nf = np * D, nc = (np4 * D) / 4;
      for (int i = tid; i < nc; i += kThreads) {
        const int bytes = max(0, min(16, (nf - 4 * i) * 4));
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(fbuf(buf) + 4 * i));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                     "l"(bytes > 0 ? src + 4 * i : src), "r"(bytes) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float2 acc[KF][D];
#pragma unroll
    for (int u = 0; u < KF; ++u)
#pragma unroll
      for (int j = 0; j < D; ++j) acc[u][j] = make_float2(0.f, 0.f);
    int64_t bs = r0, be = batch_end(r0);
    if (bs < r1) issue(bs, be, 0);
    for (int it = 0; bs < r1; ++it) {
      const int buf = it & 1;
      const int64_t ns = be, ne = ns < r1 ? batch_end(ns) : ns;
      if (ns < r1) {
        issue(ns, ne, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const int np4 = (int(be - bs) + 3) & ~3;
      const float4* xs = pbuf(buf);
      const float* fs = fbuf(buf);
      // group g takes 4-point quads g, g + G, ... of the batch
      for (int q = 4 * g; q < np4; q += 4 * G) {
        const float4 p0 = xs[q], p1 = xs[q + 1], p2 = xs[q + 2], p3 = xs[q + 3];
        // the quad's field rows: 4 D floats = D 16-byte loads
        float f[4 * D];
#pragma unroll
        for (int v = 0; v < D; ++v)
          *reinterpret_cast<float4*>(f + 4 * v) = *reinterpret_cast<const float4*>(fs + q * D + 4 * v);
#pragma unroll
        for (int uf = 0; uf < KF; ++uf) {
          float2 t0 = __fmul2_rn(make_float2(p0.x, p1.x), wx[uf]);
          float2 t1 = __fmul2_rn(make_float2(p2.x, p3.x), wx[uf]);
          t0 = __ffma2_rn(make_float2(p0.y, p1.y), wy[uf], t0);
          t1 = __ffma2_rn(make_float2(p2.y, p3.y), wy[uf], t1);
          t0 = __ffma2_rn(make_float2(p0.z, p1.z), wz[uf], t0);
          t1 = __ffma2_rn(make_float2(p2.z, p3.z), wz[uf], t1);
          float2 cs[4];
          __sincosf(t0.x, &cs[0].y, &cs[0].x);
          __sincosf(t0.y, &cs[1].y, &cs[1].x);
          __sincosf(t1.x, &cs[2].y, &cs[2].x);
          __sincosf(t1.y, &cs[3].y, &cs[3].x);
#pragma unroll
          for (int j = 0; j < D; ++j) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              acc[uf][j] = __ffma2_rn(cs[u], make_float2(f[u * D + j], f[u * D + j]), acc[uf][j]);
          }
        }
      }
      // end of a cloud part: the G point groups, added in group order, into
      // slot (c, b - bfirst)
      const int b = int(bs / a.n);
      if (ns >= r1 || ns / a.n != b) {
#pragma unroll
        for (int uf = 0; uf < KF; ++uf)
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const int kk = kk0 + uf * fbh;
            red[(g * a.fb + kk) * 2 * D + 2 * j] = acc[uf][j].x;
            red[(g * a.fb + kk) * 2 * D + 2 * j + 1] = acc[uf][j].y;
            acc[uf][j] = make_float2(0.f, 0.f);
          }
        __syncthreads();
        float* slot = a.part + int64_t(b - bfirst) * r * d * a.R + c;  // element e at slot[e R]
        for (int e = tid; e < a.fb * 2 * d; e += kThreads) {
          const int kk = e / (2 * d), rem = e - kk * 2 * d, t = rem / d, j = rem - t * d;
          const int kg = fbk * a.fb + kk;
          if (kg >= a.m) continue;
          float sum = 0.0f;
          for (int gg = 0; gg < G; ++gg) sum += red[(gg * a.fb + kk) * 2 * D + 2 * j + t];
          slot[int64_t((2 * kg + t) * d + j) * a.R] = sum;
        }
      }
      __syncthreads();  // this buffer (and red) is rewritten next
      bs = ns;
      be = ne;
    }
  }
  stamp(a.trace, 1);
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_small_p1end[blockIdx.x] = t;
  }
  sync_all(a);
  stamp(a.trace, 2);

  if (!a.fuse_a7) {
    // ---------------------------------------------- phase 2: S (fp64, fixed order)
    // one warp per element (cloud b, row, j): lane l sums the slots of ranges
    // c0 + l, c0 + l + 32, ... in order (8 loads in flight), then the lane sums
    // in lane order
    const int64_t E = int64_t(a.batch) * r * d;
    const int64_t warps = int64_t(gridDim.x) * (kThreads / 32);
    for (int64_t e = int64_t(blockIdx.x) * (kThreads / 32) + warp; e < E; e += warps) {
      const int b = int(e / (int64_t(r) * d));
      const int rem = int(e - int64_t(b) * r * d);
      const int64_t lo = int64_t(b) * a.n, hi = lo + a.n;
      const int c0 = int(lo / a.L), c1 = int((hi - 1) / a.L);
      double acc = 0.0;
      auto slot = [&](int c) {  // consecutive lanes: consecutive ranges (coalesced)
        const int kk = b - int((int64_t(c) * a.L) / a.n);
        return __ldg(a.part + (int64_t(kk) * r * d + rem) * a.R + c);
      };
      int cc = c0 + lane;
      for (; cc + 7 * 32 <= c1; cc += 8 * 32) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = slot(cc + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += double(v[u]);
      }
      for (; cc <= c1; cc += 32) acc += double(slot(cc));
      double tot = 0.0;
#pragma unroll
      for (int l = 0; l < 32; ++l) tot += __shfl_sync(0xffffffffu, acc, l);
      if (lane == 0) a.S[e] = tot;
    }
    sync_all(a);
    stamp(a.trace, 3);
    // ---------------------------------------------- phase 3: Y = C^ S
    // one warp per (cloud, row a): lanes split the r columns, fixed-order butterfly
    const int64_t rows = int64_t(a.batch) * r;
    for (int64_t row = int64_t(blockIdx.x) * (kThreads / 32) + warp; row < rows;
         row += int64_t(gridDim.x) * (kThreads / 32)) {
      const int64_t b = row / r;
      const double* Crow = a.C + row * r;
      const double* Sb = a.S + b * r * d;
      double acc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) acc[j] = 0.0;
#pragma unroll 4
      for (int cc = lane; cc < r; cc += 32) {
        const double cv = __ldg(Crow + cc);
#pragma unroll
        for (int j = 0; j < D; ++j)
          if (j < d) acc[j] = fma(cv, __ldg(Sb + int64_t(cc) * d + j), acc[j]);
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
        if (lane == 0 && j < d) a.Y[row * d + j] = float(acc[j]);
      }
    }
    sync_all(a);
  }
  stamp(a.trace, 4);

  // ------------------------------------------------ phase 4: out = F + Phi Y
  // CTA c: points [c L4, (c+1) L4), sub-tiles of <= 512 points within one cloud
  {
    const int mp = (a.m + 3) & ~3;
    float* ox = sm;             // [mp] omega x, y, z (zero-padded)
    float* oy = ox + mp;
    float* oz = oy + mp;
    float* yc = oz + mp;        // [mp][2D]: Yc[k][0..D), Ys[k][0..D) (zero-padded)
    double* sb = reinterpret_cast<double*>(yc + mp * 2 * D + 2 * D);  // fused a7: S_b [r][D]
    double* yq = sb + r * D;                                          // fused a7: [4][r][D]
    for (int k = tid; k < mp; k += kThreads) {
      const float4 w = (k < a.m) ? a.omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
      ox[k] = w.x;
      oy[k] = w.y;
      oz[k] = w.z;
    }
    const int64_t q0 = int64_t(blockIdx.x) * a.L4, q1 = min(q0 + a.L4, ntot);
    int cur_b = -1;
    for (int64_t base = q0; base < q1;) {
      const int b = int(base / a.n);
      const int64_t tend = min(min(base + kTilePts, q1), int64_t(b + 1) * a.n);
      if (b != cur_b) {
        __syncthreads();
        if (a.fuse_a7) {
          // a7 for this cloud: S_b = its range slots in order (fp64), then
          // Y_b = C^_b S_b: thread (row, quarter) sums a quarter of the columns
          // with its loads in flight, the quarters added in order; the CTA
          // holding the cloud's first point writes S_b, Y_b (export)
          const bool owner = base == int64_t(b) * a.n;
          for (int e = tid; e < r * D; e += kThreads) {
            const int ar = e / D, j = e - ar * D;
            const double v = (j < d) ? sum_slots(a, b, ar, j) : 0.0;
            sb[e] = v;
            if (owner && j < d) a.S[(int64_t(b) * r + ar) * d + j] = v;
          }
          __syncthreads();
          const double* Cb = a.C + int64_t(b) * r * r;
          const int qw = (r + 3) / 4;
          for (int e = tid; e < 4 * r; e += kThreads) {
            const int ar = e % r, qq = e / r;
            const int cb = qq * qw, ce = min(r, cb + qw);
            double acc[D];
#pragma unroll
            for (int j = 0; j < D; ++j) acc[j] = 0.0;
#pragma unroll 8
            for (int cc = cb; cc < ce; ++cc) {
              const double cv = __ldg(Cb + int64_t(ar) * r + cc);
#pragma unroll
              for (int j = 0; j < D; ++j) acc[j] = fma(cv, sb[cc * D + j], acc[j]);
            }
#pragma unroll
            for (int j = 0; j < D; ++j) yq[(qq * r + ar) * D + j] = acc[j];
          }
          __syncthreads();
          for (int e = tid; e < mp * 2 * D; e += kThreads) {
            const int k = e / (2 * D), rem = e - k * 2 * D, tt = rem / D, j = rem - tt * D;
            float v = 0.0f;
            if (k < a.m && j < d) {
              const int ar = 2 * k + tt;
              const double y = ((yq[ar * D + j] + yq[(r + ar) * D + j]) + yq[(2 * r + ar) * D + j]) +
                               yq[(3 * r + ar) * D + j];
              v = float(y);
              if (owner) a.Y[(int64_t(b) * r + ar) * d + j] = v;
            }
            yc[e] = v;
          }
        } else {
          const float* Yb = a.Y + int64_t(b) * r * d;
          for (int e = tid; e < mp * 2 * D; e += kThreads) {
            const int k = e / (2 * D), rem = e - k * 2 * D, tt = rem / D, j = rem - tt * D;
            yc[e] = (k < a.m && j < d) ? Yb[(2 * k + tt) * d + j] : 0.0f;
          }
        }
        cur_b = b;
        __syncthreads();
      }
      const int64_t i0 = base + tid, i1 = base + tid + kThreads;
      const float4 p0 = (i0 < tend) ? __ldg(a.pts + i0) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 p1 = (i1 < tend) ? __ldg(a.pts + i1) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float2 X = make_float2(p0.x, p1.x), Yp = make_float2(p0.y, p1.y),
                   Z = make_float2(p0.z, p1.z);
      float2 acc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) acc[j] = make_float2(0.f, 0.f);
#pragma unroll 2
      for (int k = 0; k < mp; k += 4) {
        const float4 WX = *reinterpret_cast<const float4*>(ox + k);
        const float4 WY = *reinterpret_cast<const float4*>(oy + k);
        const float4 WZ = *reinterpret_cast<const float4*>(oz + k);
        const float wxs[4] = {WX.x, WX.y, WX.z, WX.w}, wys[4] = {WY.x, WY.y, WY.z, WY.w},
                    wzs[4] = {WZ.x, WZ.y, WZ.z, WZ.w};
        // Y of the 4 frequencies: 8D floats = 2D 16-byte loads
        float yv[8 * D];
#pragma unroll
        for (int v4 = 0; v4 < 2 * D; ++v4)
          *reinterpret_cast<float4*>(yv + 4 * v4) =
              *reinterpret_cast<const float4*>(yc + k * 2 * D + 4 * v4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float2 th = __fmul2_rn(X, make_float2(wxs[u], wxs[u]));
          th = __ffma2_rn(Yp, make_float2(wys[u], wys[u]), th);
          th = __ffma2_rn(Z, make_float2(wzs[u], wzs[u]), th);
          float2 cv, sv;
          __sincosf(th.x, &sv.x, &cv.x);
          __sincosf(th.y, &sv.y, &cv.y);
#pragma unroll
          for (int j = 0; j < D; ++j) {
            acc[j] = __ffma2_rn(cv, make_float2(yv[u * 2 * D + j], yv[u * 2 * D + j]), acc[j]);
            acc[j] = __ffma2_rn(sv, make_float2(yv[u * 2 * D + D + j], yv[u * 2 * D + D + j]), acc[j]);
          }
        }
      }
      // (F and out may alias: each row is read before it is written, by this thread)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j < d) {
          if (i0 < tend) a.out[i0 * d + j] = a.F[i0 * d + j] + acc[j].x;
          if (i1 < tend) a.out[i1 * d + j] = a.F[i1 * d + j] + acc[j].y;
        }
      }
      base = tend;
    }
  }
  stamp(a.trace, 5);
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_small_p4end[blockIdx.x] = t;
  }
}

template <int D, int NT>
int max_ctas(size_t smem, int sms) {
  static int occ = -1;
  static size_t occ_smem = 0;
  if (occ < 0 || occ_smem != smem) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(integrate_small_kernel<D, NT>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, integrate_small_kernel<D, NT>, NT, smem);
    if (occ < 1) occ = 1;
    if (occ > 4) occ = 4;
    occ_smem = smem;
  }
  return sms * occ;
}

template <int D, int NT>
cudaError_t launch_d(const SmallArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (a.local) {  // independent CTAs: a plain launch, any grid size
    static bool configured = false;
    if (!configured && smem > 48 * 1024) {
      cudaFuncSetAttribute(integrate_small_kernel<D, NT>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      configured = true;
    }
    integrate_small_kernel<D, NT><<<grid, NT, smem, s>>>(a);
    return cudaGetLastError();
  }
  // cooperative (all CTAs co-resident: the grid barriers), via cudaLaunchKernelEx
  // so that the launch can be captured in a CUDA graph
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, integrate_small_kernel<D, NT>, a);
}

int frequency_block(int m) { return m <= 32 ? 32 : (m <= 64 ? 64 : (m <= 128 ? 128 : 256)); }

// Phase-1 ranges: >= 256 points each, at most what is co-resident (small
// clouds get few CTAs: cheaper grid barriers; large ones the whole GPU);
// K = partial slots per range (the clouds one range can touch).
void small_geometry(int m, int64_t n, int batch, int cap, int* R, int64_t* L, int* K) {
  const int nfb = (m + frequency_block(m) - 1) / frequency_block(m);
  const int64_t ntot = n * batch;
  int64_t r = (ntot + 255) / 256;
  if (r * nfb > cap) r = cap / nfb;
  if (r < 1) r = 1;
  *L = ((ntot + r - 1) / r + 3) & ~int64_t(3);
  *R = int((ntot + *L - 1) / *L);
  int64_t k = (*L + n - 1) / n + 1;
  if (k > batch) k = batch;
  *K = int(k);
}

size_t smem_bytes(int m, int D, int nt) {
  const int mp = (m + 3) & ~3;
  const int kf = nt == 768 ? 2 : 1;  // frequencies per phase-1 thread (the kernel's KF)
  const size_t s1 = (size_t(2) * (4 + D) * kBatchPts + size_t(kf) * nt * 2 * D) * sizeof(float);
  const size_t s4 = (size_t(3) * mp + size_t(mp) * 2 * D + 2 * D) * sizeof(float) +
                    size_t(2 * m) * D * 5 * sizeof(double);
  return s1 > s4 ? s1 : s4;
}

bool local_mode(int m, int64_t n, int batch, int sms) {
  if (m > 256) return false;  // one frequency block per CTA
  return (n <= 1024 && batch == 1) || (n <= 8192 && batch >= 2 * sms / 3);
}

int dclass(int d) { return d <= 1 ? 1 : (d <= 2 ? 2 : (d <= 3 ? 3 : 4)); }

// (grid-barrier mode: the wide CTAs)
int cap_for(int m, int d, int sms) {
  const size_t smem = smem_bytes(m, dclass(d), kWideThreads);
  switch (dclass(d)) {
    case 1: return max_ctas<1, kWideThreads>(smem, sms);
    case 2: return max_ctas<2, kWideThreads>(smem, sms);
    case 3: return max_ctas<3, kWideThreads>(smem, sms);
    default: return max_ctas<4, kWideThreads>(smem, sms);
  }
}

}  // namespace

size_t small_partial_elems(int m, int64_t n, int batch, int d, int sms) {
  int R, K;
  int64_t L;
  small_geometry(m, n, batch, cap_for(m, d, sms), &R, &L, &K);
  if (local_mode(m, n, batch, sms)) {
    R = batch;
    K = 1;
  }
  return size_t(R) * size_t(K) * size_t(2 * m) * size_t(d);
}

cudaError_t launch_integrate_small(const float4* pts, const float4* omega4, int m, int64_t n,
                                   int batch, int sms, const float* F, int d, float* out,
                                   const double* C, float* part, double* S, float* Y,
                                   unsigned int* bar, cudaStream_t s) {
  LaunchScope Ls("rfd_integrate_small", s);
  SmallArgs a{};
  a.pts = pts;
  a.omega4 = omega4;
  a.m = m;
  a.fb = frequency_block(m);
  a.nfb = (m + a.fb - 1) / a.fb;
  a.n = n;
  a.batch = batch;
  a.d = d;
  a.F = F;
  a.out = out;
  a.C = C;
  a.part = part;
  a.S = S;
  a.Y = Y;
  a.bar = bar;
  static const bool trace = [] {
    const char* e = getenv("RFD_SMALL_TRACE");
    return e && e[0] == '1';
  }();
  if (trace) cudaGetSymbolAddress(reinterpret_cast<void**>(&a.trace), g_small_trace);

  const int D = dclass(d);
  // one CTA per cloud when the clouds are small and there are enough of them
  // to fill the GPU (cfg 3), or for one tiny cloud (cfg 1): no grid barriers
  a.local = local_mode(m, n, batch, sms) ? 1 : 0;
  if (a.local) {
    a.R = batch;
    a.L = n;
    a.K = 1;
  } else {
    small_geometry(m, n, batch, cap_for(m, d, sms), &a.R, &a.L, &a.K);
  }
  const int grid = a.R * a.nfb;
  const int64_t ntot = n * batch;
  a.L4 = a.local ? n : (ntot + grid - 1) / grid;
  // a7 in phase 4's prologue for small r (each CTA redoes it for the clouds it
  // touches): two grid barriers fewer
  a.fuse_a7 = (a.local || (2 * m <= 128 && (n + a.L - 1) / a.L + 1 <= 16)) ? 1 : 0;
  cudaError_t e = cudaSuccess;
  if (a.local) {
    const size_t smem = smem_bytes(m, D, kLocalThreads);
    switch (D) {
      case 1: e = launch_d<1, kLocalThreads>(a, grid, smem, s); break;
      case 2: e = launch_d<2, kLocalThreads>(a, grid, smem, s); break;
      case 3: e = launch_d<3, kLocalThreads>(a, grid, smem, s); break;
      default: e = launch_d<4, kLocalThreads>(a, grid, smem, s); break;
    }
  } else {
    const size_t smem = smem_bytes(m, D, kWideThreads);
    switch (D) {
      case 1: e = launch_d<1, kWideThreads>(a, grid, smem, s); break;
      case 2: e = launch_d<2, kWideThreads>(a, grid, smem, s); break;
      case 3: e = launch_d<3, kWideThreads>(a, grid, smem, s); break;
      default: e = launch_d<4, kWideThreads>(a, grid, smem, s); break;
    }
  }
  if (trace && e == cudaSuccess) {
    unsigned long long h[8], pe[1024];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(h, g_small_trace, sizeof(h));
    cudaMemcpyFromSymbol(pe, g_small_p1end, sizeof(pe));
    unsigned long long pb[1024], p4[1024];
    unsigned int sm[1024];
    cudaMemcpyFromSymbol(p4, g_small_p4end, sizeof(p4));
    unsigned long long e4 = 0;
    for (int i = 0; i < grid && i < 1024; ++i) e4 = p4[i] > e4 ? p4[i] : e4;
    fprintf(stderr, "  last CTA end: %.1f us after start\n", (e4 - h[0]) * 1e-3);
    cudaMemcpyFromSymbol(pb, g_small_p1beg, sizeof(pb));
    cudaMemcpyFromSymbol(sm, g_small_smid, sizeof(sm));
    unsigned long long mx = 0, mn = ~0ull, bmx = 0, bmn = ~0ull, dmx = 0, dmn = ~0ull;
    int per_sm[256] = {0};
    for (int i = 0; i < grid && i < 1024; ++i) {
      mx = pe[i] > mx ? pe[i] : mx;
      mn = pe[i] < mn ? pe[i] : mn;
      bmx = pb[i] > bmx ? pb[i] : bmx;
      bmn = pb[i] < bmn ? pb[i] : bmn;
      const unsigned long long du = pe[i] - pb[i];
      dmx = du > dmx ? du : dmx;
      dmn = du < dmn ? du : dmn;
      if (sm[i] < 256) per_sm[sm[i]]++;
    }
    int cmin = 1 << 30, cmax = 0;
    for (int i = 0; i < sms; ++i) {
      cmin = per_sm[i] < cmin ? per_sm[i] : cmin;
      cmax = per_sm[i] > cmax ? per_sm[i] : cmax;
    }
    double lo_sum = 0, hi_sum = 0, lo_max = 0, hi_max = 0;
    int lo_n = 0, hi_n = 0;
    for (int i = 0; i < grid && i < 1024; ++i) {
      const double du = (pe[i] - pb[i]) * 1e-3;
      if (sm[i] < unsigned(sms / 2)) { lo_sum += du; ++lo_n; lo_max = du > lo_max ? du : lo_max; }
      else { hi_sum += du; ++hi_n; hi_max = du > hi_max ? du : hi_max; }
    }
    fprintf(stderr, "  SMs < %d: mean %.1f max %.1f us (%d CTAs); SMs >= %d: mean %.1f max %.1f us (%d)\n",
            sms / 2, lo_sum / (lo_n ? lo_n : 1), lo_max, lo_n, sms / 2, hi_sum / (hi_n ? hi_n : 1),
            hi_max, hi_n);
    fprintf(stderr, "  phase-1 end over CTAs: first %.1f us, last %.1f us after start; CTA starts "
            "%.1f..%.1f us; own durations %.1f..%.1f us; CTAs per SM %d..%d\n",
            (mn - h[0]) * 1e-3, (mx - h[0]) * 1e-3, (bmn - h[0]) * 1e-3, (bmx - h[0]) * 1e-3,
            dmn * 1e-3, dmx * 1e-3, cmin, cmax);
    fprintf(stderr, "small n=%lld batch=%d m=%d d=%d grid=%d slots=%d fuse=%d: phase1 %.1f us, "
            "sync %.1f, S %.1f, Y %.1f, phase4 %.1f (total %.1f)\n", (long long)n, batch, m, d, grid,
            a.K, a.fuse_a7, (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3, (h[3] - h[2]) * 1e-3,
            (h[4] - h[3]) * 1e-3, (h[5] - h[4]) * 1e-3, (h[5] - h[0]) * 1e-3);
  }
  return e;
}

}  // namespace rfd
