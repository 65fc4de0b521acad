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

constexpr int kThreads = 256;
constexpr int kBatchPts = 512;  // points staged per phase-1 batch
constexpr int kTilePts = 512;   // points per phase-4 tile (2 per thread)

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
      while (ld_acquire(bar) == my) {
      }
    }
  }
  __syncthreads();
}

struct SmallArgs {
  const float4* pts;     // batch x n, centred (x, y, z, 0)
  const float4* omega4;  // m: fp32(2 pi omega)
  int m, fb, nfb;        // frequencies; frequency block (32..256, power of two); blocks
  int64_t n;
  int batch, d;
  int segs;              // point segments per cloud (phase 1)
  int64_t seg_len;       // points per segment (multiple of 4)
  const float* F;        // (batch x) n x d
  float* out;            // same shape (may alias F)
  const double* C;       // batch x r x r
  float* part;           // batch x segs x r x d
  double* S;             // batch x r x d
  float* Y;              // batch x r x d
  unsigned int* bar;     // kBarWords words, zero before the first launch
  int fuse_a7;           // 1: S and Y per cloud in phase 4's prologue (small r, few segments)
  unsigned long long* trace;  // diagnostics (RFD_SMALL_TRACE=1): phase timestamps of CTA 0
};

__device__ __forceinline__ void stamp(unsigned long long* tr, int i) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[i] = t;
  }
}
__device__ unsigned long long g_small_trace[8];

template <int D>
__global__ void __launch_bounds__(kThreads)
integrate_small_kernel(const SmallArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = 2 * a.m;
  const int d = a.d;
  stamp(a.trace, 0);

  // ------------------------------------------------ phase 1: S partials
  {
    const int G = kThreads / a.fb;  // point groups
    const int g = tid / a.fb;
    float* xs = sm;                         // [kBatchPts] x, y, z, then F[D][kBatchPts]
    float* ys = xs + kBatchPts;
    float* zs = ys + kBatchPts;
    float* fs = zs + kBatchPts;
    float* red = fs + D * kBatchPts;        // [G][fb][2D]
    const int64_t items = int64_t(a.batch) * a.segs * a.nfb;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int fbk = int(it % a.nfb);
      const int64_t bs = it / a.nfb;
      const int b = int(bs / a.segs), seg = int(bs % a.segs);
      const int k = fbk * a.fb + (tid % a.fb);
      const float4 w = (k < a.m) ? a.omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float2 wx = make_float2(w.x, w.x), wy = make_float2(w.y, w.y), wz = make_float2(w.z, w.z);
      float2 acc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) acc[j] = make_float2(0.f, 0.f);
      const int64_t p0 = int64_t(seg) * a.seg_len, p1 = min(p0 + a.seg_len, a.n);
      const float4* cloud = a.pts + int64_t(b) * a.n;
      const float* Fb = a.F + int64_t(b) * a.n * d;
      for (int64_t base = p0; base < p1; base += kBatchPts) {
        const int np = int(p1 - base < kBatchPts ? p1 - base : kBatchPts);
        const int np4 = (np + 3) & ~3;
        __syncthreads();  // the previous batch has been read
        for (int i = tid; i < np4; i += kThreads) {
          const float4 x = (i < np) ? __ldg(cloud + base + i) : make_float4(0.f, 0.f, 0.f, 0.f);
          xs[i] = x.x;
          ys[i] = x.y;
          zs[i] = x.z;
        }
        for (int i = tid; i < np4 * D; i += kThreads) {
          const int p = i / D, j = i - p * D;
          fs[j * kBatchPts + p] = (p < np && j < d) ? __ldg(Fb + (base + p) * d + j) : 0.0f;
        }
        __syncthreads();
        // group g takes 4-point quads g, g + G, ... of the batch
        for (int q = 4 * g; q < np4; q += 4 * G) {
          const float4 X = *reinterpret_cast<const float4*>(xs + q);
          const float4 Yv = *reinterpret_cast<const float4*>(ys + q);
          const float4 Z = *reinterpret_cast<const float4*>(zs + q);
          float2 t0 = __fmul2_rn(make_float2(X.x, X.y), wx);
          float2 t1 = __fmul2_rn(make_float2(X.z, X.w), wx);
          t0 = __ffma2_rn(make_float2(Yv.x, Yv.y), wy, t0);
          t1 = __ffma2_rn(make_float2(Yv.z, Yv.w), wy, t1);
          t0 = __ffma2_rn(make_float2(Z.x, Z.y), wz, t0);
          t1 = __ffma2_rn(make_float2(Z.z, Z.w), wz, t1);
          float2 cs[4];
          __sincosf(t0.x, &cs[0].y, &cs[0].x);
          __sincosf(t0.y, &cs[1].y, &cs[1].x);
          __sincosf(t1.x, &cs[2].y, &cs[2].x);
          __sincosf(t1.y, &cs[3].y, &cs[3].x);
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const float4 f = *reinterpret_cast<const float4*>(fs + j * kBatchPts + q);
            acc[j] = __ffma2_rn(cs[0], make_float2(f.x, f.x), acc[j]);
            acc[j] = __ffma2_rn(cs[1], make_float2(f.y, f.y), acc[j]);
            acc[j] = __ffma2_rn(cs[2], make_float2(f.z, f.z), acc[j]);
            acc[j] = __ffma2_rn(cs[3], make_float2(f.w, f.w), acc[j]);
          }
        }
      }
      // the G point groups, added in group order
#pragma unroll
      for (int j = 0; j < D; ++j) {
        red[(g * a.fb + tid % a.fb) * 2 * D + 2 * j] = acc[j].x;
        red[(g * a.fb + tid % a.fb) * 2 * D + 2 * j + 1] = acc[j].y;
      }
      __syncthreads();
      for (int e = tid; e < a.fb * 2 * d; e += kThreads) {
        const int kk = e / (2 * d), rem = e - kk * 2 * d, t = rem / d, j = rem - t * d;
        const int kg = fbk * a.fb + kk;
        if (kg >= a.m) continue;
        float s = 0.0f;
        for (int gg = 0; gg < G; ++gg) s += red[(gg * a.fb + kk) * 2 * D + 2 * j + t];
        a.part[((int64_t(b) * a.segs + seg) * r + 2 * kg + t) * d + j] = s;
      }
    }
  }
  stamp(a.trace, 1);
  grid_sync(a.bar);
  stamp(a.trace, 2);

  // ------------------------------------------------ phase 2: S (fp64, fixed order)
  if (!a.fuse_a7) {
    // element e of (batch x r x d): 8 lanes per element, lane l sums segments
    // l, l + 8, ... in order; then the 8 slice sums in order
    // one warp per element of (batch x r x d): lane l sums segments l, l + 32,
    // ... in order (8 loads in flight), then the 32 lane sums in lane order
    const int64_t E = int64_t(a.batch) * r * d;
    const int64_t warps = int64_t(gridDim.x) * (kThreads / 32);
    const int64_t st = int64_t(r) * d;
    for (int64_t e0 = int64_t(blockIdx.x) * (kThreads / 32) + warp; e0 < E; e0 += warps) {
      const int64_t b = e0 / st, rem = e0 - b * st;
      const float* src = a.part + b * a.segs * st + rem;
      double acc = 0.0;
      int sg = lane;
      for (; sg + 7 * 32 < a.segs; sg += 8 * 32) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (sg + 32 * u) * st);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += double(v[u]);
      }
      for (; sg < a.segs; sg += 32) acc += double(__ldg(src + sg * st));
      double tot = 0.0;
#pragma unroll
      for (int l = 0; l < 32; ++l) tot += __shfl_sync(0xffffffffu, acc, l);
      if (lane == 0) a.S[e0] = tot;
    }
  }
  if (!a.fuse_a7) grid_sync(a.bar);
  stamp(a.trace, 3);

  // ------------------------------------------------ phase 3: Y = C^ S
  if (!a.fuse_a7) {
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
      for (int c = lane; c < r; c += 32) {
        const double cv = __ldg(Crow + c);
#pragma unroll
        for (int j = 0; j < D; ++j)
          if (j < d) acc[j] = fma(cv, __ldg(Sb + int64_t(c) * d + j), acc[j]);
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
        if (lane == 0 && j < d) a.Y[row * d + j] = float(acc[j]);
      }
    }
  }
  if (!a.fuse_a7) grid_sync(a.bar);
  stamp(a.trace, 4);

  // ------------------------------------------------ phase 4: out = F + Phi Y
  {
    const int mp = (a.m + 3) & ~3;
    float* ox = sm;             // [mp] omega x, y, z (zero-padded)
    float* oy = ox + mp;
    float* oz = oy + mp;
    float* yc = oz + mp;        // [mp][2D]: Yc[k][0..D), Ys[k][0..D) (zero-padded)
    double* sb = reinterpret_cast<double*>(yc + mp * 2 * D + 2 * D);  // fused a7: S_b [r][D]
    for (int k = tid; k < mp; k += kThreads) {
      const float4 w = (k < a.m) ? a.omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
      ox[k] = w.x;
      oy[k] = w.y;
      oz[k] = w.z;
    }
    const int64_t tpc = (a.n + kTilePts - 1) / kTilePts;
    const int64_t tiles = tpc * a.batch;
    int cur_b = -1;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int b = int(t / tpc);
      const int64_t base = (t - int64_t(b) * tpc) * kTilePts;
      if (b != cur_b) {
        __syncthreads();
        if (a.fuse_a7) {
          // a7 for this cloud: S_b = sum of its segment partials (fixed order,
          // fp64), then Y_b = C^_b S_b by one warp per row (lanes over the
          // columns, fixed-order butterfly) straight into the Y staging;
          // the CTA holding the cloud's first tile also writes S_b, Y_b (export)
          const bool owner = base == 0;
          const float* pb = a.part + int64_t(b) * a.segs * r * d;
          for (int e = tid; e < r * D; e += kThreads) {
            const int ar = e / D, j = e - ar * D;
            double acc = 0.0;
            if (j < d)
              for (int sg = 0; sg < a.segs; ++sg) acc += double(__ldg(pb + (int64_t(sg) * r + ar) * d + j));
            sb[e] = acc;
            if (owner && j < d) a.S[(int64_t(b) * r + ar) * d + j] = acc;
          }
          for (int e = tid; e < mp * 2 * D; e += kThreads) yc[e] = 0.0f;
          __syncthreads();
          const double* Cb = a.C + int64_t(b) * r * r;
          for (int ar = warp; ar < r; ar += kThreads / 32) {
            double acc[D];
#pragma unroll
            for (int j = 0; j < D; ++j) acc[j] = 0.0;
            for (int c = lane; c < r; c += 32) {
              const double cv = __ldg(Cb + int64_t(ar) * r + c);
#pragma unroll
              for (int j = 0; j < D; ++j) acc[j] = fma(cv, sb[c * D + j], acc[j]);
            }
#pragma unroll
            for (int j = 0; j < D; ++j) {
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
            }
            if (lane == 0) {
              const int k = ar >> 1, tt = ar & 1;
#pragma unroll
              for (int j = 0; j < D; ++j) {
                if (j < d) {
                  yc[k * 2 * D + tt * D + j] = float(acc[j]);
                  if (owner) a.Y[(int64_t(b) * r + ar) * d + j] = float(acc[j]);
                }
              }
            }
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
      const float4* cloud = a.pts + int64_t(b) * a.n;
      const float4 p0 = (i0 < a.n) ? __ldg(cloud + i0) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 p1 = (i1 < a.n) ? __ldg(cloud + i1) : make_float4(0.f, 0.f, 0.f, 0.f);
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
          float2 c, s;
          __sincosf(th.x, &s.x, &c.x);
          __sincosf(th.y, &s.y, &c.y);
#pragma unroll
          for (int j = 0; j < D; ++j) {
            acc[j] = __ffma2_rn(c, make_float2(yv[u * 2 * D + j], yv[u * 2 * D + j]), acc[j]);
            acc[j] = __ffma2_rn(s, make_float2(yv[u * 2 * D + D + j], yv[u * 2 * D + D + j]), acc[j]);
          }
        }
      }
      const float* Fb = a.F + int64_t(b) * a.n * d;
      float* Ob = a.out + int64_t(b) * a.n * d;
      // (F and out may alias: each row is read before it is written, by this thread)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j < d) {
          if (i0 < a.n) Ob[i0 * d + j] = Fb[i0 * d + j] + acc[j].x;
          if (i1 < a.n) Ob[i1 * d + j] = Fb[i1 * d + j] + acc[j].y;
        }
      }
    }
  }
  stamp(a.trace, 5);
}

template <int D>
int max_ctas(size_t smem, int sms) {
  static int occ = -1;
  static size_t occ_smem = 0;
  if (occ < 0 || occ_smem != smem) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(integrate_small_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, integrate_small_kernel<D>, kThreads, smem);
    if (occ < 1) occ = 1;
    if (occ > 4) occ = 4;
    occ_smem = smem;
  }
  return sms * occ;
}

template <int D>
cudaError_t launch_d(const SmallArgs& a, int grid, size_t smem, cudaStream_t s) {
  // cooperative (all CTAs co-resident: the grid barriers), via cudaLaunchKernelEx
  // so that the launch can be captured in a CUDA graph
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, integrate_small_kernel<D>, a);
}

int frequency_block(int m) { return m <= 32 ? 32 : (m <= 64 ? 64 : (m <= 128 ? 128 : 256)); }

// Grid (CTAs) sized to the work, at most what is co-resident: small clouds
// get few CTAs (cheaper grid barriers), large ones the whole GPU.
int small_grid(int m, int64_t n, int batch, int cap) {
  const int nfb = (m + frequency_block(m) - 1) / frequency_block(m);
  const int64_t items = int64_t(batch) * nfb * ((n + 1023) / 1024);  // >= 1024-point segments
  const int64_t tiles = int64_t(batch) * ((n + kTilePts - 1) / kTilePts);
  int64_t g = items > tiles ? items : tiles;
  if (g > cap) g = cap;
  return g < 1 ? 1 : int(g);
}

}  // namespace

int small_segments(int m, int64_t n, int batch, int sms) {
  // one phase-1 item (cloud, segment, frequency block) per CTA of the largest
  // grid (4 CTAs per SM), whole 4-point quads
  const int nfb = (m + frequency_block(m) - 1) / frequency_block(m);
  const int grid = small_grid(m, n, batch, 4 * sms);
  int64_t segs = grid / (int64_t(batch) * nfb);
  const int64_t maxs = (n + 255) / 256;
  if (segs > maxs) segs = maxs;
  return segs < 1 ? 1 : int(segs);
}

cudaError_t launch_integrate_small(const float4* pts, const float4* omega4, int m, int64_t n,
                                   int batch, int sms, const float* F, int d, float* out,
                                   const double* C, float* part, double* S, float* Y,
                                   unsigned int* bar, cudaStream_t s) {
  LaunchScope L("rfd_integrate_small", s);
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
  const int D = d <= 1 ? 1 : (d <= 2 ? 2 : (d <= 3 ? 3 : 4));
  const int mp = (m + 3) & ~3;
  const size_t s1 = (size_t(3 + D) * kBatchPts + size_t(kThreads) * 2 * D) * sizeof(float);
  const size_t s4 = (size_t(3) * mp + size_t(mp) * 2 * D + 2 * D) * sizeof(float) +
                    size_t(2 * m) * D * sizeof(double);
  const size_t smem = s1 > s4 ? s1 : s4;
  int cap = 0;
  switch (D) {
    case 1: cap = max_ctas<1>(smem, sms); break;
    case 2: cap = max_ctas<2>(smem, sms); break;
    case 3: cap = max_ctas<3>(smem, sms); break;
    default: cap = max_ctas<4>(smem, sms); break;
  }
  const int grid = small_grid(m, n, batch, cap);
  a.segs = int(grid / (int64_t(batch) * a.nfb));
  if (a.segs > small_segments(m, n, batch, sms)) a.segs = small_segments(m, n, batch, sms);
  if (a.segs < 1) a.segs = 1;
  a.seg_len = ((n + a.segs - 1) / a.segs + 3) & ~int64_t(3);
  a.segs = int((n + a.seg_len - 1) / a.seg_len);
  // a7 in phase 4's prologue when every CTA's share of it is small (each CTA
  // redoes it for the clouds it touches): two grid barriers fewer
  a.fuse_a7 = (2 * m <= 128 && a.segs <= 64) ? 1 : 0;
  cudaError_t e = cudaSuccess;
  switch (D) {
    case 1: e = launch_d<1>(a, grid, smem, s); break;
    case 2: e = launch_d<2>(a, grid, smem, s); break;
    case 3: e = launch_d<3>(a, grid, smem, s); break;
    default: e = launch_d<4>(a, grid, smem, s); break;
  }
  if (trace && e == cudaSuccess) {
    unsigned long long h[8];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(h, g_small_trace, sizeof(h));
    fprintf(stderr, "small n=%lld batch=%d m=%d d=%d grid=%d segs=%d: phase1 %.1f us, sync %.1f, "
            "S %.1f, Y %.1f, phase4 %.1f (total %.1f)\n", (long long)n, batch, m, d, grid, a.segs,
            (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3, (h[3] - h[2]) * 1e-3, (h[4] - h[3]) * 1e-3,
            (h[5] - h[4]) * 1e-3, (h[5] - h[0]) * 1e-3);
  }
  return e;
}

}  // namespace rfd
