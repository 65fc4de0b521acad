// K1/K2 on the tensor cores -- Gram matrix G = Phi^T Phi (SURVEY Sec. 8(a)
// row a4; B^T A of PAPER.md:337, 355 without D).  Plan-time.
//
// G is a dense contraction over points (N x r by N x r), so it runs on
// tcgen05: each CTA owns a "unit" of one or two 128 x 128 tiles of the upper
// triangle of G (a 128 x 256 accumulator in TMEM) and a chunk of points.  Per
// K-step of 32 points the CTA's 8 warps regenerate the feature rows of the
// unit's 128-feature blocks (a3: omega.x in turns, MUFU sin/cos) straight into
// shared memory as an fp16 hi/lo split, x = hi + lo (|x - hi - lo| <=
// 2^-22 |x| + 2^-25), and one thread issues
//     D += Hi_A Hi_B^T + Hi_A Lo_B^T + Lo_A Hi_B^T
// (tcgen05.mma kind::f16, M = 128, N = 128/256, K = 16, fp32 accumulate): the
// dropped Lo Lo^T term is below 2^-22, so the tile carries fp32-level
// products (DESIGN.md Sec. 6 "Gram precision").  Two shared-memory stages:
// feature generation of step t+1 overlaps the MMAs of step t; a
// tcgen05.commit -> mbarrier releases each stage.
//
// K2 (gram_tc_reduce): fixed-order fp64 sum of the chunk partials -> G,
// mirrored to the lower triangle.  Deterministic.
#include "rfd_internal.h"
#include "tc_ptx.cuh"

namespace rfd {
namespace {

constexpr int kBlk = 128;           // features per block (64 frequencies)
constexpr int kStepPts = 64;        // points per K-step (4 MMA K-slices of 16)
constexpr int kProducers = 512;     // 16 feature-producer warps
constexpr int kThreads = 544;       // + 1 MMA-issue warp (warp 16)
constexpr int kMaxLocal = 3;        // feature blocks per unit
// Per operand (Hi or Lo), per block: 128 rows x 64 points x 2 B = 16 KB.
constexpr int kBlkBytes = kBlk * kStepPts * 2;
constexpr int kStageBytes = 2 * kMaxLocal * kBlkBytes;  // Hi + Lo: 96 KB
constexpr int kStages = 2;
// K-steps per TMEM accumulation epoch: the tensor core accumulates at most
// kEpoch * 12 MMA updates in fp32 before the sum moves to registers, which
// bounds the accumulator's round-toward-zero bias.
constexpr int kEpoch = 8;
// Canonical K-major layout (no swizzle): offset(row, k) = (row/8)*kSBO +
// (k/8)*kLBO + (row%8)*16 + (k%8)*2.
constexpr uint32_t kLBO = 128;
constexpr uint32_t kSBO = (kStepPts / 8) * 128;  // 1024

struct GramUnit {
  int ngrp;
  int a_blk[2];   // global feature block of the A rows of group g
  int b_blk[2];   // first global block of the B rows of group g
  int nb[2];      // B blocks (1 or 2) -> N = 128 nb
  int nloc;       // distinct global blocks, local order
  int loc[kMaxLocal];
};

__host__ __device__ inline int local_of(const GramUnit& U, int blk) {
  for (int i = 0; i < U.nloc; ++i)
    if (U.loc[i] == blk) return i;
  return 0;
}

__host__ __device__ inline void add_loc(GramUnit& U, int blk) {
  for (int i = 0; i < U.nloc; ++i)
    if (U.loc[i] == blk) return;
  U.loc[U.nloc++] = blk;
}

// Enumerate units for T feature blocks: all pair units (i, [j, j+1]) row by
// row, then the row-end single tiles (i, T-1) two at a time.
__host__ __device__ inline int gram_units(int T, int u_want, GramUnit* out) {
  int u = 0;
  for (int i = 0; i < T; ++i)
    for (int j = i; j + 1 < T; j += 2) {
      if (u == u_want && out) {
        GramUnit U{};
        U.ngrp = 1;
        U.a_blk[0] = i; U.b_blk[0] = j; U.nb[0] = 2;
        add_loc(U, j); add_loc(U, j + 1); add_loc(U, i);
        *out = U;
      }
      ++u;
    }
  int singles[16];
  int ns = 0;
  for (int i = 0; i < T; ++i)
    if ((T - i) % 2 == 1) singles[ns++] = i;
  for (int s = 0; s < ns; s += 2) {
    if (u == u_want && out) {
      GramUnit U{};
      U.ngrp = (s + 1 < ns) ? 2 : 1;
      for (int g = 0; g < U.ngrp; ++g) {
        U.a_blk[g] = singles[s + g]; U.b_blk[g] = T - 1; U.nb[g] = 1;
      }
      add_loc(U, T - 1);
      for (int g = 0; g < U.ngrp; ++g) add_loc(U, U.a_blk[g]);
      *out = U;
    }
    ++u;
  }
  return u;
}

__device__ __forceinline__ void sincos_rad(float4 w, float4 x, float& c, float& s) {
  // w = fp32(2 pi omega): the argument in radians; MUFU reduces it in turns.
  const float t = fmaf(w.z, x.z, fmaf(w.y, x.y, w.x * x.x));
  __sincosf(t, &s, &c);
}

__global__ void __launch_bounds__(kThreads, 1)
gram_tc_kernel(const float4* __restrict__ pts, const float4* __restrict__ omega4, int m,
               int64_t n, int T, int nunits, int chunks, int64_t chunk,
               float* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t mma_bar[kStages];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float4 xs[2][kStepPts + kStepPts / 8];  // padded: point p at p + p/8

  const int unit = blockIdx.x, ch = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  GramUnit U;
  gram_units(T, unit, &U);
  const int nloc = U.nloc, ngrp = U.ngrp;

  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_sh);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) tc::mbar_init(&mma_bar[s], 1);
    tc::mbar_fence_init();
  }
  const int64_t p0 = int64_t(ch) * chunk;
  const int64_t p1 = min(p0 + chunk, n);
  const float4* cloud = pts + int64_t(b) * n;
  // xs holds a step's points with one float4 of padding per 8 (point p at
  // p + p/8): the point groups of an 8-lane phase hit distinct banks.
  if (tid < kStepPts)
    xs[0][tid + (tid >> 3)] =
        (p0 + tid < p1) ? __ldg(cloud + p0 + tid) : make_float4(0.f, 0.f, 0.f, 0.f);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sbase = tc::smem_addr(smem);

  // Tasks: each thread owns one frequency fl (0..63) of every local block and
  // one point group q (8 points).  Lane bits: [1:0] -> fl % 4, [2] -> q & 1,
  // [4:3] -> q >> 1; warps take consecutive groups of 4 frequencies.  Lanes
  // with odd q store their sin row first, so each 8-lane phase of a 16-byte
  // store covers all 8 rows of a core matrix: no bank conflicts.
  const int q = (((lane >> 3) & 3) << 1) | ((lane >> 2) & 1);
  const int fl = 4 * warp + (lane & 3), odd = q & 1;
  float4 w[kMaxLocal];
#pragma unroll
  for (int i = 0; i < kMaxLocal; ++i) {
    const int k = (i < nloc) ? U.loc[i] * 64 + fl : m;
    w[i] = (k < m) ? omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const uint32_t grp_off = uint32_t((2 * fl) / 8) * kSBO + uint32_t(q) * kLBO;
  const uint32_t off_first = grp_off + uint32_t((2 * fl + odd) % 8) * 16;
  const uint32_t off_second = grp_off + uint32_t((2 * fl + 1 - odd) % 8) * 16;

  // MMA operand offsets (thread 0): local block of A rows / first B rows.
  uint32_t a_off[2] = {0, 0}, b_off[2] = {0, 0}, idesc[2];
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    a_off[g] = uint32_t(local_of(U, U.a_blk[g])) * kBlkBytes;
    b_off[g] = uint32_t(local_of(U, U.b_blk[g])) * kBlkBytes;
    idesc[g] = tc::make_idesc(0, 128, 128 * U.nb[g]);
  }

  // fp32 register accumulators: TMEM lane group warp % 4, column quarter
  // warp / 4 (64 of the 256 accumulator columns).
  const int lg = warp & 3, quarter = warp >> 2;
  float acc[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) acc[j] = 0.0f;
  const int ncols = (ngrp == 2) ? 256 : 128 * U.nb[0];
  const bool drains = quarter * 64 < ncols;
  const uint32_t lane_base = tmem + (uint32_t(lg * 32) << 16) + uint32_t(quarter * 64);
  auto drain = [&](int dslot) {
    if (!drains || tid >= kProducers) return;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v[32];
      tc::tmem_ld32(lane_base + uint32_t(dslot * 256 + c * 32), v);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[c * 32 + j] += v[j];
    }
  };

  const int nsteps = int((p1 - p0 + kStepPts - 1) / kStepPts);
  for (int t = 0; t < nsteps; ++t) {
    const int s = t % kStages;
    const int slot = (t / kEpoch) & 1;
    if (t >= kStages) tc::mbar_wait(&mma_bar[s], ((t - kStages) / kStages) & 1);
    const uint32_t hi_base = sbase + s * kStageBytes;
    const uint32_t lo_base = hi_base + kMaxLocal * kBlkBytes;
    const int64_t base = p0 + int64_t(t) * kStepPts;
    const float4* xt = xs[t & 1];
    // Next step's points: load now (the global-memory latency hides behind
    // this step's feature generation), store to shared memory at the end.
    float4 xn = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid < kStepPts) {
      const int64_t pn = base + kStepPts + tid;
      if (pn < p1) xn = __ldg(cloud + pn);
    }
#pragma unroll
    for (int i = 0; i < kMaxLocal; ++i) {
      if (i >= nloc || tid >= kProducers) break;
      float c[8], sn[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) sincos_rad(w[i], xt[q * 9 + j], c[j], sn[j]);
      if (base + q * 8 + 8 > p1) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (base + q * 8 + j >= p1) { c[j] = 0.f; sn[j] = 0.f; }
      }
      uint32_t fh[4], fl_[4], sh[4], sl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t chh, cll, shh, sll;
        tc::split_f16x2(c[2 * j], c[2 * j + 1], chh, cll);
        tc::split_f16x2(sn[2 * j], sn[2 * j + 1], shh, sll);
        fh[j] = odd ? shh : chh;  fl_[j] = odd ? sll : cll;
        sh[j] = odd ? chh : shh;  sl[j] = odd ? cll : sll;
      }
      const uint32_t ob = uint32_t(i) * kBlkBytes;
      tc::st_shared_v4(hi_base + ob + off_first, fh[0], fh[1], fh[2], fh[3]);
      tc::st_shared_v4(lo_base + ob + off_first, fl_[0], fl_[1], fl_[2], fl_[3]);
      tc::st_shared_v4(hi_base + ob + off_second, sh[0], sh[1], sh[2], sh[3]);
      tc::st_shared_v4(lo_base + ob + off_second, sl[0], sl[1], sl[2], sl[3]);
    }
    // The next step's points become visible after this step's barrier.
    if (tid < kStepPts) xs[(t + 1) & 1][tid + (tid >> 3)] = xn;
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    if (warp == kProducers / 32) {
      // MMA warp: warp-uniform issue (descriptors in uniform registers), one
      // elected lane; the producer warps go straight on to the next step.
      tc::tc_fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < kStepPts / 16; ++kk) {
          const uint32_t koff = uint32_t(kk) * 2 * kLBO;
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            if (g >= ngrp) break;
            const uint64_t aH = tc::make_sdesc(hi_base + a_off[g] + koff, kLBO, kSBO);
            const uint64_t aL = tc::make_sdesc(lo_base + a_off[g] + koff, kLBO, kSBO);
            const uint64_t bH = tc::make_sdesc(hi_base + b_off[g] + koff, kLBO, kSBO);
            const uint64_t bL = tc::make_sdesc(lo_base + b_off[g] + koff, kLBO, kSBO);
            const uint32_t d = tmem + uint32_t(slot * 256 + g * 128);
            // The first MMA of an epoch starts its TMEM slot afresh.
            const uint32_t acc0 = ((t % kEpoch) > 0 || kk > 0) ? 1u : 0u;
            tc::mma_f16(d, aH, bH, idesc[g], acc0);
            tc::mma_f16(d, aH, bL, idesc[g], 1u);
            tc::mma_f16(d, aL, bH, idesc[g], 1u);
          }
        }
        tc::mma_commit(&mma_bar[s]);
      }
      __syncwarp();
    }
    // One step into epoch e+1, epoch e (the other TMEM slot) is complete --
    // the wait at the top of this step covered step t-2, its last MMA -- so
    // move it into the fp32 registers (round-to-nearest adds).
    if (t % kEpoch == 1 && t > kEpoch) {
      tc::tc_fence_after();
      drain(slot ^ 1);
      tc::tc_fence_before();
    }
  }
  if (nsteps > 0) {
    tc::mbar_wait(&mma_bar[(nsteps - 1) % kStages], ((nsteps - 1) / kStages) & 1);
    tc::tc_fence_after();
    const int last_e = (nsteps - 1) / kEpoch;
    if (last_e >= 1 && (nsteps - 1) % kEpoch == 0) drain((last_e - 1) & 1);
    drain(last_e & 1);
  }

  // partial[b][ch][unit][col (256)][row (128)] fp32 (rows contiguous).
  float* out = partial + ((int64_t(b) * chunks + ch) * nunits + unit) * (256 * 128);
  const int row = lg * 32 + lane;
  if (drains && tid < kProducers) {
#pragma unroll
    for (int j = 0; j < 64; ++j) out[int64_t(quarter * 64 + j) * 128 + row] = acc[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

__global__ void gram_tc_reduce_kernel(const float* __restrict__ partial, int r, int T, int nunits,
                                      int chunks, double* __restrict__ G) {
  // grid: (128*128/256, upper tiles, batch); tile t enumerates (ti <= tj).
  const int b = blockIdx.z;
  int t = blockIdx.y, ti = 0, row = T;
  while (t >= row) { t -= row; ++ti; --row; }
  const int tj = ti + t;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int lr = e & 127, lc = e >> 7;  // row-fastest: coalesced partial reads
  if (ti == tj && lr > lc) return;      // diagonal tile: upper half, mirrored
  const int a = ti * kBlk + lr, c = tj * kBlk + lc;
  if (a >= r || c >= r) return;
  // find the unit / accumulator column of tile (ti, tj)
  int unit = 0, col = 0;
  for (int u = 0; u < nunits; ++u) {
    GramUnit U;
    gram_units(T, u, &U);
    for (int g = 0; g < U.ngrp; ++g)
      if (U.a_blk[g] == ti && tj >= U.b_blk[g] && tj < U.b_blk[g] + U.nb[g]) {
        unit = u;
        col = g * 128 + (tj - U.b_blk[g]) * 128;
      }
  }
  const int64_t stride = int64_t(nunits) * 256 * 128;
  const float* src = partial + (int64_t(b) * chunks * nunits + unit) * (256 * 128) +
                     int64_t(col + lc) * 128 + lr;
  double sum = 0.0;
  for (int k = 0; k < chunks; ++k) sum += double(src[k * stride]);
  double* Gb = G + int64_t(b) * r * r;
  Gb[int64_t(a) * r + c] = sum;
  Gb[int64_t(c) * r + a] = sum;
}

}  // namespace

GramGeom gram_tc_geometry(int m, int64_t n, int batch, int sms) {
  GramGeom g;
  g.r = 2 * m;
  g.tile = kBlk;
  g.tiles1d = (g.r + kBlk - 1) / kBlk;
  g.ntiles = gram_units(g.tiles1d, -1, nullptr);  // units
  // One CTA per SM (full TMEM); about three waves of CTAs.
  int64_t chunks = 1;
  const int64_t want = (3LL * sms + int64_t(g.ntiles) * batch - 1) / (int64_t(g.ntiles) * batch);
  if (want > chunks) chunks = want;
  const int64_t maxc = (n + kStepPts - 1) / kStepPts;
  if (chunks > maxc) chunks = maxc;
  if (chunks < 1) chunks = 1;
  int64_t chunk = (n + chunks - 1) / chunks;
  chunk = (chunk + kStepPts - 1) / kStepPts * kStepPts;
  g.chunk = chunk;
  g.chunks = int((n + chunk - 1) / chunk);
  return g;
}

size_t gram_tc_partial_elems(const GramGeom& g, int batch) {
  return size_t(batch) * g.chunks * g.ntiles * 256 * 128;
}

void launch_gram_tc(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                    const GramGeom& g, float* partial, double* G, cudaStream_t s) {
  const int smem = kStages * kStageBytes;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  {
    LaunchScope L("rfd_gram_tc", s);
    gram_tc_kernel<<<dim3(g.ntiles, g.chunks, batch), kThreads, smem, s>>>(
        pts, omega4, m, n, g.tiles1d, g.ntiles, g.chunks, g.chunk, partial);
  }
  {
    LaunchScope L("rfd_gram_reduce", s);
    const int tiles = g.tiles1d * (g.tiles1d + 1) / 2;
    gram_tc_reduce_kernel<<<dim3(kBlk * kBlk / 256, tiles, batch), 256, 0, s>>>(
        partial, g.r, g.tiles1d, g.ntiles, g.chunks, G);
  }
}

}  // namespace rfd
