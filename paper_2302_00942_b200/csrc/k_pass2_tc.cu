// K6 on the tensor cores -- pass 2, out = F + Phi Y (SURVEY Sec. 8(a) row
// a8; the "x + A(...)" of Eq. 13).
//
// Per tile of 128 points the contraction Phi_tile (128 x r) . Y (r x 16) runs
// as tcgen05.mma kind::f16 with the A operand in TMEM: the 16 producer warps
// regenerate each point's feature row (a3: omega.x in radians, MUFU sin/cos)
// and write it, split x = hi + lo in fp16 (|x - hi - lo| <= 2^-22 |x| +
// 2^-25), straight into TMEM with tcgen05.st -- row = point = TMEM lane, so
// no shared-memory traffic for A.  Y^T, scaled per channel by a power of two
// into fp16 range (max |Y_j| 2^e_j <= 2^14; undone exactly in the epilogue)
// and split likewise, sits in shared memory as the B operand.  Per 128-feature
// chunk one thread issues
//     D += A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T   (M=128, N=16, K=16 x 8)
// (kind::f16 takes K = 16 per instruction, half the instructions of tf32:
// with N = 16 the instruction issue, not the tensor math, sets the pace)
// into a double-buffered TMEM accumulator; chunk stages are released by
// tcgen05.commit -> mbarrier, so feature generation of the next chunk
// overlaps the MMAs.  The epilogue (TMEM -> registers, + F, store) of tile t
// runs after the first chunk of tile t+1 has been produced.  Persistent CTAs
// over contiguous tile ranges; d is handled in column chunks of <= 16.
#include <cstdio>
#include <cstdlib>

#include "rfd_internal.h"
#include "tc_ptx.cuh"

namespace rfd {
namespace {

// Warp roles: PW producer warps (PW / 4 per TMEM lane group), one MMA warp,
// four epilogue warps (one per lane group).  PW = 16: 8 producers (32
// frequencies per warp and chunk: 9 % fewer instructions per feature) measured
// 10 % slower -- the producers need the warps to hide MUFU / FMA latency.
template <int PW>
struct Roles {
  static constexpr int kProducerWarps = PW;
  static constexpr int kMmaWarp = PW;
  static constexpr int kEpiWarp0 = PW + 1;
  static constexpr int kThreads = (PW + 5) * 32;
};
constexpr int kTile = 128;      // points per tile (= TMEM lanes)
#ifndef RFD_P2_STAGES
#define RFD_P2_STAGES 2
#endif
constexpr int kStages = RFD_P2_STAGES;
// TMEM columns: accumulators [0, nw) and [nw, 2 nw) (nw = the launch's column
// width, a multiple of 16, <= 64); stage s: hi at 2 nw + 128 s (64 cols = 128
// fp16), lo at +64.
constexpr uint32_t kLBO = 128;
constexpr size_t kPass2MaxSmem = 200 * 1024;
constexpr size_t kCStage = 32 * 1024;  // fused a7: C^ row-block staging

// KF = features per K-chunk: 128 (64 frequencies) or, for m <= 32, 64 (32
// frequencies: no chunk half filled with padding frequencies).
// Diagnostics (RFD_P2_TRACE=1): per-chunk / per-tile timestamps of CTA 0.
__device__ long long g_p2trace[1024][5];
__device__ long long g_p2tile[256][6];
__device__ long long g_p2load[4][8];

// kFuse (part != nullptr) is a separate instantiation: the fused a7 prologue
// is most of the kernel's code, and compiled into the plain kernel it cost
// 6 % (0.73 -> 0.78 ms at cfg 5).
template <int KF, bool kFuse, bool kTr = false, int PW = 16>
__global__ void __launch_bounds__(Roles<PW>::kThreads, 1)
pass2_tc_kernel(const float4* __restrict__ pts, const float4* __restrict__ omega4, int m, int64_t n,
                int batch, const float* __restrict__ Y, const float* F, float* out, int d, int c0,
                int dc, int nw, const float* __restrict__ part, int ranges,
                const double* __restrict__ C, double* __restrict__ S_out, float* __restrict__ Y_out) {
  // part != nullptr: fused a7 -- each CTA sums the cloud's pass-1 partials
  // (S, fp64, fixed order) and forms Y = C^ S itself (small r: no separate
  // reduce / apply launches); the CTA holding the cloud's first tile also
  // writes S and Y to the plan (export).
  // F and out may alias (in place): each epilogue thread reads F_i before
  // writing out_i.
  constexpr int kProducerWarps = Roles<PW>::kProducerWarps, kMmaWarp = Roles<PW>::kMmaWarp,
                kEpiWarp0 = Roles<PW>::kEpiWarp0, kThreads = Roles<PW>::kThreads;
  constexpr int QW = PW / 4;  // producer warps per lane group
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], dfull_bar[2], dempty_bar[2];
  __shared__ uint64_t yready_bar;
  __shared__ uint32_t tmem_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3;
  constexpr int kChunkF = KF, kFpc = KF / 2;  // features / frequencies per chunk
  const int nch = (m + kFpc - 1) / kFpc;       // chunks
  const int kpad = nch * kChunkF;              // padded feature count
  const uint32_t sbo = uint32_t(kpad / 8) * 128;
  unsigned char* yb = smem;                          // B hi: 16 x kpad fp16
  unsigned char* yl = smem + nw * kpad * 2;          // B lo
  // omega (radians) as SoA: x components of all frequencies, then y, then z
  float* ox = reinterpret_cast<float*>(smem + 2 * nw * kpad * 2);
  float* oy = ox + nch * kFpc;
  float* oz = oy + nch * kFpc;
  // fused a7: S_b (fp64 [2m][dc]) and Y_b (fp32 [2m][dc]) after the omegas
  double* Ss = reinterpret_cast<double*>(oz + nch * kFpc);
  float* Ys = reinterpret_cast<float*>(Ss + 2 * m * dc);
  // fused a7: row blocks of C^_b staged in shared memory (kCStage bytes)
  double* Cs = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(Ys + 2 * m * dc) + 15) & ~uintptr_t(15));
  __shared__ unsigned int ymax_bits[64];
  __shared__ float yscale_inv[64];
  const uint32_t kColA = 2 * nw;
  const uint32_t yb_s = tc::smem_addr(yb), yl_s = tc::smem_addr(yl);

  asm volatile("griddepcontrol.launch_dependents;");  // the next pass 1 may start its setup
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], kProducerWarps);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&dfull_bar[b], 1);
      tc::mbar_init(&dempty_bar[b], 4);
    }
    tc::mbar_init(&yready_bar, 1);
    tc::mbar_fence_init();
  }
  for (int k = tid; k < nch * kFpc; k += kThreads) {
    const float4 w = (k < m) ? omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    ox[k] = w.x;
    oy[k] = w.y;
    oz[k] = w.z;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // Programmatic dependent launch: the setup above (barriers, omegas: plan
  // data) may overlap the previous kernel's tail; everything below reads
  // its results (partials / Y) or the field.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // TMEM is allocated only after the wait: every CTA of the preceding
  // tcgen05 kernel has then exited and freed its columns, so a CTA of this
  // kernel never spins in tcgen05.alloc beside one it waits for, whatever the
  // occupancy.
  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t lane_field = uint32_t(lg * 32) << 16;
  const uint32_t idesc = tc::make_idesc(0, 128, nw);
  const bool trc = kTr && blockIdx.x == 0 && lane == 0;
  __shared__ long long trs[kTr ? 128 : 1][5], trt[kTr ? 32 : 1][6], trl[kTr ? 4 : 1][8];
  int ncc = 0;  // trace: cloud changes so far

  const int64_t tpc = (n + kTile - 1) / kTile;
  const int64_t ntiles = tpc * batch;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;

  // Y_b^T as the B operand; the CTA's tiles are contiguous, so the cloud
  // changes rarely.  (Re)loads run under a full-CTA barrier after every MMA
  // reading the old Y has completed.
  auto load_y = [&](int b, bool owner) {
    const int r = 2 * m;
    const float* Yb = Y + int64_t(b) * 2 * m * d;
    int ystride = d, ycol = c0;  // Y element (a, j) at Yb[a * ystride + ycol + j]
    if constexpr (kFuse) {
      // S = sum over the ranges' partials, in range order (fp64)
      const float* pb = part + int64_t(b) * ranges * r * dc;
#pragma unroll 1
      for (int e = tid; e < r * dc; e += kThreads) {
        double acc = 0.0;
#pragma unroll 4
        for (int rg = 0; rg < ranges; ++rg) acc += double(__ldg(pb + int64_t(rg) * r * dc + e));
        Ss[e] = acc;
      }
      __syncthreads();
      if (kTr && blockIdx.x == 0 && tid == 0 && ncc < 4) trl[ncc][5] = clock64();
      // Y = C^ S by blocks of rows: the block of C^_b is copied into shared
      // memory (row stride r + 1: conflict-free column walks), then one thread
      // per output (a, j) runs its dot product over k.  Compact on purpose:
      // this runs once per cloud from a cold instruction cache (the earlier
      // warp-per-row form, unrolled over 16 columns, took ~13k cycles at r = 64).
      const int cs = r + 1;
      const int rb = min(r, int(kCStage / (8 * cs)));
      for (int a0 = 0; a0 < r; a0 += rb) {
        const int nr = min(rb, r - a0);
        const double* src = C + (int64_t(b) * r + a0) * r;
        const double2* src2 = reinterpret_cast<const double2*>(src);  // r even: 16-byte rows
#pragma unroll 4
        for (int e = tid; e < nr * r / 2; e += kThreads) {  // loads in flight together
          const double2 v = __ldg(src2 + e);
          const int ar = (2 * e) / r, k = 2 * e - ar * r;
          Cs[ar * cs + k] = v.x;
          Cs[ar * cs + k + 1] = v.y;
        }
        __syncthreads();
        // 8 lanes per output (k = ks, ks + 8, ...; fixed-order butterfly)
        const int ks = lane & 7;
#pragma unroll 1
        for (int e0 = 0; e0 < nr * dc; e0 += kThreads / 8) {
          const int e = e0 + (tid >> 3);
          const bool ok = e < nr * dc;
          const int ar = ok ? e / dc : 0, j = ok ? e - ar * dc : 0;
          const double* Ca = Cs + ar * cs;
          double acc = 0.0;
#pragma unroll 4
          for (int k = ks; k < r; k += 8) acc = fma(Ca[k], Ss[k * dc + j], acc);
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          acc += __shfl_xor_sync(0xffffffffu, acc, 2);
          acc += __shfl_xor_sync(0xffffffffu, acc, 4);
          if (ok && ks == 0) Ys[(a0 + ar) * dc + j] = float(acc);
        }
        __syncthreads();  // the block buffer is rewritten next
      }
      __syncthreads();
      if (kTr && blockIdx.x == 0 && tid == 0 && ncc < 4) trl[ncc][6] = clock64();
      if (owner)
        for (int e = tid; e < r * dc; e += kThreads) {
          const int a = e / dc, j = e - (e / dc) * dc;
          S_out[(int64_t(b) * r + a) * d + c0 + j] = Ss[e];
          Y_out[(int64_t(b) * r + a) * d + c0 + j] = Ys[e];
        }
      Yb = Ys;
      ystride = dc;
      ycol = 0;
    }
    // per-channel power-of-two scale: max |Y_j| 2^e_j in [2^13, 2^14); one warp
    // per channel, lanes over the 2m rows (no atomics, no index division)
    if (tid < nw) ymax_bits[tid] = 0u;
    __syncthreads();
    for (int j = warp; j < dc; j += kThreads / 32) {
      float mx = 0.0f;
      for (int a = lane; a < 2 * m; a += 32)
        mx = fmaxf(mx, fabsf(Yb[int64_t(a) * ystride + ycol + j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) ymax_bits[j] = __float_as_uint(mx);
    }
    __syncthreads();
    float scale = 1.0f;
    if (tid < nw) {
      const float mx = __uint_as_float(ymax_bits[tid]);
      int ex = 0;
      if (mx > 0.0f && isfinite(mx)) {
        frexpf(mx, &ex);  // mx = f 2^ex, f in [0.5, 1)
        // clamped like pass 1's: 2^(14 - ex) overflows to inf for max |Y_j| <
        // 2^-113 (tiny lambda or field column); 2^126 still puts such a
        // column's max at >= 2^13 (ex <= -113), its inverse 2^-126 is normal
        scale = ldexpf(1.0f, min(126, max(-126, 14 - ex)));
      }
      yscale_inv[tid] = 1.0f / scale;  // exact (power of two)
      ymax_bits[tid] = __float_as_uint(scale);
    }
    __syncthreads();
    // Y^T (nw rows x kpad), scaled and split; one warp per feature row a,
    // lanes over channels
    for (int a = warp; a < kpad; a += kThreads / 32) {
      for (int j = lane; j < nw; j += 32) {
        const float val = (a < 2 * m && j < dc)
                              ? Yb[int64_t(a) * ystride + ycol + j] * __uint_as_float(ymax_bits[j])
                              : 0.0f;
        const __half h = __float2half_rn(val);
        const __half l = __float2half_rn(val - __half2float(h));
        const uint32_t off = uint32_t(j >> 3) * sbo + uint32_t(a >> 3) * kLBO +
                             uint32_t(j & 7) * 16 + uint32_t(a & 7) * 2;
        *reinterpret_cast<__half*>(yb + off) = h;
        *reinterpret_cast<__half*>(yl + off) = l;
      }
    }
    tc::fence_proxy_async_smem();
  };

  // Every role walks the same tile sequence; a cloud change is a CTA-wide
  // barrier, taken once all MMAs issued so far have completed.
  uint32_t g = 0, it = 0;
  int cur_b = -1;
  // Each producer lane's point, copied one tile ahead into a private 2-slot
  // shared-memory ring (cp.async: no register scoreboard on the global load).
  __shared__ __align__(16) float4 xring[2][kProducerWarps][32];
  auto copy_x = [&](int bt, int64_t tin, int slot) {
    const int64_t i = tin * kTile + lg * 32 + lane;
    // points past the cloud's end read its first point (finite; their rows
    // of the output are never stored)
    tc::cp_async16(tc::smem_addr(&xring[slot][warp][lane]), pts + int64_t(bt) * n + (i < n ? i : 0));
    tc::cp_async_commit();
  };
  // (cloud, tile within the cloud) advance incrementally: no 64-bit division
  // per tile (measured: ~1500 cycles of producer bubble at every tile change)
  int b = int(t_begin / tpc);
  int64_t tin = t_begin - int64_t(b) * tpc;
  for (int64_t tile = t_begin; tile < t_end; ++tile, ++it) {
    const int64_t base = tin * kTile;
    int nb = b;  // the next tile's cloud and index
    int64_t ntin = tin + 1;
    if (ntin == tpc) {
      ntin = 0;
      ++nb;
    }
    if (b != cur_b) {
      const bool trl_on = kTr && blockIdx.x == 0 && tid == 0 && ncc < 4;
      if (trl_on) trl[ncc][0] = clock64();
      if (g > 0) tc::mbar_wait(&empty_bar[(g - 1) % kStages], ((g - 1) / kStages) & 1);
      if (trl_on) trl[ncc][1] = clock64();
      __syncthreads();
      if (trl_on) trl[ncc][2] = clock64();
      load_y(b, tin == 0);  // this CTA holds the cloud's first tile
      if (trl_on) trl[ncc][3] = clock64();
      __syncthreads();
      if (trl_on) trl[ncc][4] = clock64();
      cur_b = b;
      ++ncc;
    }
    const uint32_t buf = it & 1;
    if (warp < kProducerWarps) {
      // ---------------- producers: 16 frequencies per thread per chunk -----
      const int q = warp >> 2;  // which 1/QW of the chunk's frequencies
      // This tile's point (prefetched during the previous tile) and the next's.
      if (trc && warp == 0 && it < 32) trt[it][5] = clock64();
      if (tile == t_begin) copy_x(b, tin, 0);
      if (tile + 1 < t_end) copy_x(nb, ntin, int(it + 1) & 1);
      else tc::cp_async_commit();
      tc::cp_async_wait<1>();  // this tile's copy
      const float4 x = xring[it & 1][warp][lane];
      const float2 xx = make_float2(x.x, x.x), xy = make_float2(x.y, x.y), xz = make_float2(x.z, x.z);
      for (int c = 0; c < nch; ++c) {
        const uint32_t gg = g + c, s = gg % kStages, u = gg / kStages;
        if (trc && warp == 0 && gg < 128) trs[gg][0] = clock64();
        if (u >= 1) tc::mbar_wait(&empty_bar[s], (u - 1) & 1);
        if (trc && warp == 0 && gg < 128) trs[gg][1] = clock64();
        const uint32_t acol = tmem + lane_field + kColA + 128 * s + (KF / (2 * QW)) * q;
#pragma unroll
        for (int h = 0; h < KF / (16 * QW); ++h) {  // groups of 8 frequencies (register pressure)
          float v[16];
          const int f0 = kFpc * c + (kFpc / QW) * q + 8 * h;
          // Frequencies beyond m (zero omega) meet zero rows of Y^T: no masking.
          // omega . x for 2 frequencies per packed FP32 instruction, in the
          // operation order of fmaf(wz, z, fmaf(wy, y, wx * x)).
#pragma unroll
          for (int j = 0; j < 8; j += 4) {
            const float4 WX = *reinterpret_cast<const float4*>(ox + f0 + j);
            const float4 WY = *reinterpret_cast<const float4*>(oy + f0 + j);
            const float4 WZ = *reinterpret_cast<const float4*>(oz + f0 + j);
            float2 t0 = __fmul2_rn(make_float2(WX.x, WX.y), xx);
            float2 t1 = __fmul2_rn(make_float2(WX.z, WX.w), xx);
            t0 = __ffma2_rn(make_float2(WY.x, WY.y), xy, t0);
            t1 = __ffma2_rn(make_float2(WY.z, WY.w), xy, t1);
            t0 = __ffma2_rn(make_float2(WZ.x, WZ.y), xz, t0);
            t1 = __ffma2_rn(make_float2(WZ.z, WZ.w), xz, t1);
            __sincosf(t0.x, &v[2 * j + 1], &v[2 * j]);
            __sincosf(t0.y, &v[2 * j + 3], &v[2 * j + 2]);
            __sincosf(t1.x, &v[2 * j + 5], &v[2 * j + 4]);
            __sincosf(t1.y, &v[2 * j + 7], &v[2 * j + 6]);
          }
          // interleaved features (2j = cos, 2j+1 = sin): one fp16 pair per column
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) tc::split_f16x2(v[2 * j], v[2 * j + 1], hi[j], lo[j]);
          tc::tmem_st8(acol + 8 * h, hi);
          tc::tmem_st8(acol + KF / 2 + 8 * h, lo);
        }
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (trc && warp == 0 && gg < 128) trs[gg][2] = clock64();
        if (lane == 0) tc::mbar_arrive(&full_bar[s]);
      }
    } else if (warp == kMmaWarp) {
      // ---------------- MMA issue: warp-uniform loop, one elected lane -----
      if (trc && it < 32) trt[it][0] = clock64();
      if (it >= 2) tc::mbar_wait(&dempty_bar[buf], ((it - 2) >> 1) & 1);
      if (trc && it < 32) trt[it][1] = clock64();
      const uint32_t dcol = tmem + nw * buf;
      const uint64_t bh0 = tc::make_sdesc(yb_s, kLBO, sbo);
      const uint64_t bl0 = tc::make_sdesc(yl_s, kLBO, sbo);
      for (int c = 0; c < nch; ++c) {
        const uint32_t gg = g + c, s = gg % kStages, u = gg / kStages;
        if (trc && gg < 128) trs[gg][3] = clock64();
        tc::mbar_wait(&full_bar[s], u & 1);
        if (trc && gg < 128) trs[gg][4] = clock64();
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t a0 = tmem + kColA + 128 * s;
#pragma unroll
          for (int kk = 0; kk < kChunkF / 16; ++kk) {
            // start-address field (bits 0-13, 16-byte units) advances by
            // (c * 8 + 2 kk) core matrices of 128 B
            const uint64_t adv = uint64_t(c * (kChunkF / 8) + 2 * kk) * (kLBO >> 4);
            const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
            tc::mma_f16_ts(dcol, a0 + 8 * kk, bh0 + adv, idesc, acc);
            tc::mma_f16_ts(dcol, a0 + 8 * kk, bl0 + adv, idesc, 1u);
            tc::mma_f16_ts(dcol, a0 + KF / 2 + 8 * kk, bh0 + adv, idesc, 1u);
          }
          tc::mma_commit(&empty_bar[s]);
          if (c == nch - 1) tc::mma_commit(&dfull_bar[buf]);
        }
        __syncwarp();
      }
    } else {
      // ---------------- epilogue warps: TMEM -> registers, + F, store -----
      // (16-column groups; D is released once every group has been read)
      const int64_t i = base + lg * 32 + lane;
      const int64_t idx = int64_t(b) * n + i;
      const bool tre = trc && warp == kEpiWarp0 && it < 32;
      if (tre) trt[it][2] = clock64();
      tc::mbar_wait(&dfull_bar[buf], (it >> 1) & 1);
      if (tre) trt[it][3] = clock64();
      tc::tc_fence_after();
      for (int g16 = 0; g16 < nw; g16 += 16) {
        const int dcg = min(16, dc - g16);
        const bool vec = (dcg == 16) && (d % 4 == 0) && ((c0 + g16) % 4 == 0);
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = 0.0f;
        if (i < n && dcg > 0) {
          const float* Fi = F + idx * d + c0 + g16;
          if (vec) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const float4 t4 = *reinterpret_cast<const float4*>(Fi + j);
              f[j] = t4.x; f[j + 1] = t4.y; f[j + 2] = t4.z; f[j + 3] = t4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < dcg) f[j] = Fi[j];
          }
        }
        float v[16];
        __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the F loads
        tc::tmem_ld16(tmem + lane_field + nw * buf + g16, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] *= yscale_inv[g16 + j];
        if (i < n && dcg > 0) {
          float* Oi = out + idx * d + c0 + g16;
          if (vec) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(Oi + j) =
                  make_float4(f[j] + v[j], f[j + 1] + v[j + 1], f[j + 2] + v[j + 2],
                              f[j + 3] + v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < dcg) Oi[j] = f[j] + v[j];
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (tre) trt[it][4] = clock64();
      if (lane == 0) tc::mbar_arrive(&dempty_bar[buf]);
    }
    g += nch;
    b = nb;
    tin = ntin;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (kTr && blockIdx.x == 0) {
    for (int i = tid; i < 128 * 5; i += kThreads) g_p2trace[i / 5][i % 5] = trs[i / 5][i % 5];
    for (int i = tid; i < 32 * 6; i += kThreads) g_p2tile[i / 6][i % 6] = trt[i / 6][i % 6];
    for (int i = tid; i < 4 * 8; i += kThreads) g_p2load[i / 8][i % 8] = trl[i / 8][i % 8];
  }
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

template <int KF, bool kFuse, bool kTr = false, int PW = 16>
void launch_p2(int64_t grid, size_t smem, cudaStream_t s, const float4* pts, const float4* omega4,
               int m, int64_t n, int batch, const float* Y, const float* F, float* out, int d,
               int c0, int dc, int nw, const float* part, int ranges, const double* C, double* S,
               float* Yw) {
  static bool configured = false;
  if (!configured) {  // (the trace variant's static trace buffers take 6 KB)
    cudaFuncSetAttribute(pass2_tc_kernel<KF, kFuse, kTr, PW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kPass2MaxSmem) - (kTr ? 8192 : 0));
    configured = true;
  }
  launch_pdl(pass2_tc_kernel<KF, kFuse, kTr, PW>, dim3(unsigned(grid)), dim3(Roles<PW>::kThreads),
             smem, s, pts,
             omega4, m, n, batch, Y, F, out, d, c0, dc, nw, part, ranges, C, S, Yw);
}

static void print_p2trace(cudaStream_t s, int nch) {
  static long long h[1024][5], t[256][6], L[4][8];
  cudaStreamSynchronize(s);
  cudaMemcpyFromSymbol(L, g_p2load, sizeof(L));
  for (int i = 0; i < 4; ++i)
    fprintf(stderr, "  cloud change %d: drain %lld, sync %lld, S-sum %lld, Y=CS %lld, max+convert %lld, sync %lld\n",
            i, L[i][1] - L[i][0], L[i][2] - L[i][1], L[i][5] - L[i][2], L[i][6] - L[i][5],
            L[i][3] - L[i][6], L[i][4] - L[i][3]);
  cudaMemcpyFromSymbol(h, g_p2trace, sizeof(h));
  cudaMemcpyFromSymbol(t, g_p2tile, sizeof(t));
  double pe = 0, pc = 0, pr = 0, mf = 0, per = 0;
  const int lo = 20, hi = 120;
  for (int c = lo; c < hi; ++c) {
    pe += h[c][1] - h[c][0];
    pc += h[c][2] - h[c][1];
    pr += h[c + 1][0] - h[c][2];
    mf += h[c][4] - h[c][3];
    per += h[c + 1][3] - h[c][3];
  }
  const double k = hi - lo;
  fprintf(stderr, "p2trace chunk: period %.0f | prod empty-wait %.0f compute %.0f rest %.0f | mma full-wait %.0f\n",
          per / k, pe / k, pc / k, pr / k, mf / k);
  double md = 0, ew = 0, ep = 0, tp = 0;
  const int tl = 5, th = 30;
  for (int i = tl; i < th; ++i) {
    md += t[i][1] - t[i][0];
    ew += t[i][3] - t[i][2];
    ep += t[i][4] - t[i][3];
    tp += t[i + 1][0] - t[i][0];
  }
  const double kt = th - tl;
  for (int i = 15; i < 19; ++i)
    fprintf(stderr, "  tile %d: prod tile-top at +%lld after the last arrive, first chunk wait at +%lld\n", i,
            t[i][5] - h[4 * i - 1][2], h[4 * i][0] - t[i][5]);
  for (int c = 60; c < 76; ++c)
    fprintf(stderr, "  chunk %d: mma period %lld full-wait %lld | prod empty-wait %lld compute %lld rest %lld\n",
            c, h[c + 1][3] - h[c][3], h[c][4] - h[c][3], h[c][1] - h[c][0], h[c][2] - h[c][1],
            h[c + 1][0] - h[c][2]);
  fprintf(stderr, "p2trace tile (%d chunks): period %.0f | mma dempty-wait %.0f | epi dfull-wait %.0f work %.0f\n",
          nch, tp / kt, md / kt, ew / kt, ep / kt);
}

size_t pass2_tc_smem(int m, int nw, int fuse_dc) {
  const int fpc = m <= 32 ? 32 : 64;  // frequencies per chunk (KF / 2)
  const int nch = (m + fpc - 1) / fpc;
  return size_t(2) * nw * nch * (2 * fpc) * 2 + size_t(nch * fpc) * 3 * sizeof(float) +
         size_t(2 * m) * fuse_dc * (sizeof(double) + sizeof(float)) +
         (fuse_dc > 0 ? kCStage + 16 : 0);
}

int pass2_tc_width(int m) {
  // widest column chunk (multiple of 16, <= 64) whose Y^T operand fits
  for (int nw = 64; nw > 16; nw -= 16)
    if (pass2_tc_smem(m, nw, 0) <= kPass2MaxSmem) return nw;
  return 16;
}

void launch_pass2_tc(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                     int sms, const float* Y, const float* F, float* out, int d, int c0, int dc,
                     const float* part, int ranges, const double* C, double* S, float* Yw,
                     cudaStream_t s) {
  LaunchScope L("rfd_pass2_tc", s);
  const int nw = (dc + 15) / 16 * 16;  // MMA N: the chunk's columns, padded to 16
  const size_t smem = pass2_tc_smem(m, nw, part ? dc : 0);
  const int64_t ntiles = ((n + kTile - 1) / kTile) * batch;
  int64_t grid = int64_t(sms);  // one CTA per SM (full TMEM)
  if (grid > ntiles) grid = ntiles;
  static const bool trace = [] {
    const char* e = getenv("RFD_P2_TRACE");
    return e && atoi(e) == 1;
  }();
  const bool fuse = part != nullptr;
  if (trace && m > 32 && !fuse) {
    launch_p2<128, false, true>(grid, smem, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc, nw,
                                part, ranges, C, S, Yw);
    print_p2trace(s, (m + 63) / 64);
  } else if (trace && m <= 32 && fuse) {
    launch_p2<64, true, true>(grid, smem, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc, nw,
                              part, ranges, C, S, Yw);
    print_p2trace(s, (m + 31) / 32);
  } else if (m <= 32) {
    if (fuse)
      launch_p2<64, true>(grid, smem, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc, nw, part,
                          ranges, C, S, Yw);
    else
      launch_p2<64, false>(grid, smem, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc, nw, part,
                           ranges, C, S, Yw);
  } else {
    if (fuse)
      launch_p2<128, true>(grid, smem, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc, nw, part,
                           ranges, C, S, Yw);
    else
      launch_p2<128, false>(grid, smem, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc, nw,
                            part, ranges, C, S, Yw);
  }
}

}  // namespace rfd
