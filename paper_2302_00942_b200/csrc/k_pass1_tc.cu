// K4 on the tensor cores -- pass 1, S = Phi^T F (the
// first bracket "B^T x" of Eq. 13), for a chunk of up to 64
// columns of F per launch (NEXT-2: the features are generated once for all the
// chunk's columns).
//
// A CTA owns a tile of 128 frequencies (TMEM lanes) and a contiguous range of
// whole chunks of 64 points (the contraction dimension K).  Warp roles:
//
//   * 16 producer warps regenerate cos and sin of omega_k . x for their
//     lane's frequency (a3; 16 points per warp and chunk, read as one SoA
//     group copied ahead with cp.async, arguments in packed FP32) and write
//     them, split x = hi + lo in fp16 (|x - hi - lo| <= 2^-22 |x| + 2^-25),
//     straight into TMEM as the A operands (cos rows, sin rows);
//   * one elected lane of the MMA warp issues per chunk
//         D_cos += C_hi F_hi^T + C_hi F_lo^T + C_lo F_hi^T,  D_sin likewise
//     (tcgen05.mma kind::f16, M = 128, N = 16 NC, K = 16 x 4);
//   * 4 F/drain warps stage F: per epoch of E chunks they copy the epoch's
//     F block into shared memory (cp.async), scale each channel by a power of
//     two into fp16 range (max |F_j| 2^e_j in [2^13, 2^14) over the epoch) and
//     write it, split likewise, as the B operands of the epoch's chunks
//     (N channels x 64 points, K-major, double-buffered by epoch).  The tensor
//     core's fp32 accumulator is not round-to-nearest, so D accumulates one
//     epoch only; the same warps then add it, scaled back exactly (x 2^-e_j),
//     into a long-term fp32 sum L in TMEM (round-to-nearest FFMA), and at the
//     end write L as the CTA's 2 x N partial sums per frequency.  K5 reduces
//     the partials in a fixed order in fp64.
//
// TMEM: D [0, 2N) (cos N | sin N), L [2N, 4N), A stages at 4N + 128 s.
#include <cstdio>
#include <cstdlib>

#include "rfd_internal.h"
#include "tc_ptx.cuh"

namespace rfd {
namespace {

constexpr int kProducerWarps = 16;  // 4 per TMEM lane group
constexpr int kMmaWarp = 16;
constexpr int kFWarp0 = 17;         // warps 17..20: F staging + drains
constexpr int kThreads = 21 * 32;
constexpr int kChunk = 64;          // points per chunk (16 per producer warp)
constexpr int kArr = kChunk / 2;    // TMEM columns per A array (fp16 pairs)
constexpr uint32_t kLBO = 128;
constexpr uint32_t kSBO = (kChunk / 8) * 128;   // B: 8-channel groups

// Wide chunks (NC = 2..4 groups of 16 columns): one D buffer and the long-term
// sums L in TMEM (2N registers per lane would not fit); d <= 16 uses the
// one-chunk kernel below.
template <int NC>
struct P1 {
  static constexpr int N = 16 * NC;                          // MMA N: channels
  static constexpr int kStages = (512 - 4 * N) / 128 < 3 ? (512 - 4 * N) / 128 : 3;
  static constexpr int kEpoch = NC <= 2 ? 8 : 4;             // chunks per epoch
  static constexpr uint32_t kColL = 2 * N, kColA = 4 * N;
  static constexpr int kBBytes = N * kChunk * 2;             // one fp16 B operand
  static constexpr int kChunkB = 2 * kBBytes;                // hi + lo
  static constexpr int kEpochB = kEpoch * kChunkB;
  static constexpr int kRowF = N + 4;                        // staging row stride (floats)
  static constexpr int kStageF = kEpoch * kChunk * kRowF * 4;  // fp32 F block
  static constexpr int kSmem = 2 * kEpochB + kStageF;
};

template <int NC>
__global__ void __launch_bounds__(kThreads, 1)
pass1_tc_kernel(const float* __restrict__ pts16, const float4* __restrict__ omega4, int m,
                int64_t n, int ranges, const float* __restrict__ F, int d, int c0, int dc,
                float* __restrict__ partial) {
  using C = P1<NC>;
  constexpr int N = C::N, kStages = C::kStages, kEpoch = C::kEpoch;
  // [2 epochs][E chunks][hi | lo] B operands, then the fp32 F staging block
  extern __shared__ __align__(1024) unsigned char bsm[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], dfull_bar, dempty_bar, bready_bar[2],
      fst_bar;
  __shared__ uint32_t tmem_sh;
  // each producer warp's 16 points of a chunk as [x0..15 | y0..15 | z0..15],
  // 3 chunks deep (cp.async ring)
  __shared__ __align__(16) float xbuf[3][kProducerWarps][48];
  __shared__ float fmax_part[128];
  __shared__ float4 fmax4[128];
  __shared__ float fscale_inv[2][N];  // per epoch buffer

  const int ft = blockIdx.x, rg = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, lg = warp & 3;
  // ranges are whole chunks; only a cloud's last chunk is partial
  const int64_t cpc = (n + kChunk - 1) / kChunk, gpc = (n + 15) / 16;
  const int64_t ch0 = cpc * rg / ranges, ch1 = cpc * (rg + 1) / ranges;
  const int64_t p0 = ch0 * kChunk;
  const int nchunks = int(ch1 - ch0);
  const int nepochs = (nchunks + kEpoch - 1) / kEpoch;
  const float* cloud16 = pts16 + int64_t(b) * gpc * 48;

  asm volatile("griddepcontrol.launch_dependents;");  // pass 2 may start its setup
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], kProducerWarps);
      tc::mbar_init(&empty_bar[s], 1);
    }
    tc::mbar_init(&dfull_bar, 1);
    tc::mbar_init(&dempty_bar, 4);
    for (int i = 0; i < 2; ++i) tc::mbar_init(&bready_bar[i], 4);
    tc::mbar_init(&fst_bar, 1);
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // Programmatic dependent launch: the setup above may overlap the previous
  // kernel (pass 2 of an earlier integrate); F and the partials only after it.
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
  const int f = ft * 128 + lg * 32 + lane;  // this lane's frequency

  if (warp < kProducerWarps) {
    // ---------------- producers: 16 points per warp per chunk --------------
    const int q = warp >> 2;  // which 16 of the chunk's points
    const float4 w = (f < m) ? omega4[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float2 wx = make_float2(w.x, w.x), wy = make_float2(w.y, w.y), wz = make_float2(w.z, w.z);
    // The warp's 16 points (one SoA group, 192 B), copied two chunks ahead by
    // lanes 0-11 straight into shared memory (cp.async: global latency off the
    // critical path).  Groups past the cloud's end repeat its last group
    // (finite values that meet zero F).  Pointers and counters advance per
    // chunk (no 64-bit index arithmetic in the loop).
    const float* xsrc = cloud16 + ((ch0 * (kChunk / 16) + q) * 48 + 4 * lane);
    const float* xlast = cloud16 + ((gpc - 1) * 48 + 4 * lane);
    const int64_t xrem0 = gpc - (ch0 * (kChunk / 16) + q);
    int xrem = int(xrem0 > 0x7fffffff ? 0x7fffffff : xrem0);  // groups left
    constexpr uint32_t kRing = kProducerWarps * 48 * 4;           // bytes per ring slot
    const uint32_t x_s = tc::smem_addr(&xbuf[0][warp][0]);
    uint32_t xw = 0;
    auto load_x = [&](bool valid) {
      if (lane < 12 && valid) tc::cp_async16(x_s + xw * kRing + 16 * lane, xrem > 0 ? xsrc : xlast);
      tc::cp_async_commit();  // one group per chunk, empty past the end
      xsrc += 48 * (kChunk / 16);
      xrem -= kChunk / 16;
      xw = (xw == 2) ? 0 : xw + 1;
    };
    load_x(nchunks > 0);
    load_x(nchunks > 1);
    const uint32_t empty_s = tc::smem_addr(&empty_bar[0]), full_s = tc::smem_addr(&full_bar[0]);
    uint32_t s = 0, u = 0, xr = 0;  // stage, its round, ring slot read
    for (int c = 0; c < nchunks; ++c) {
      load_x(c + 2 < nchunks);  // the slot chunk c - 1 read (ordered by its __syncwarp)
      if (u >= 1) tc::mbar_wait(empty_s + 8 * s, (u - 1) & 1);
      // Points beyond the cloud meet zero columns of F^T, and lanes beyond m
      // are never written out: no masking of the features.
      tc::cp_async_wait<2>();  // chunk c's group (c + 1, c + 2 may be in flight)
      __syncwarp();
      const float* xs = &xbuf[0][warp][0] + xr * (kProducerWarps * 48);
      xr = (xr == 2) ? 0 : xr + 1;
      const uint32_t a = tmem + lane_field + C::kColA + 4 * kArr * s + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // two halves of 8 points (register pressure)
        float cs[8], sn[8];
#pragma unroll
        for (int j = 0; j < 8; j += 4) {
          // omega . x for 4 points in packed FP32 (2 points per instruction),
          // the same operation order as fmaf(wz, z, fmaf(wy, y, wx * x))
          const float4 X = *reinterpret_cast<const float4*>(xs + 8 * h + j);
          const float4 Y = *reinterpret_cast<const float4*>(xs + 16 + 8 * h + j);
          const float4 Z = *reinterpret_cast<const float4*>(xs + 32 + 8 * h + j);
          float2 t0 = __fmul2_rn(wx, make_float2(X.x, X.y));
          float2 t1 = __fmul2_rn(wx, make_float2(X.z, X.w));
          t0 = __ffma2_rn(wy, make_float2(Y.x, Y.y), t0);
          t1 = __ffma2_rn(wy, make_float2(Y.z, Y.w), t1);
          t0 = __ffma2_rn(wz, make_float2(Z.x, Z.y), t0);
          t1 = __ffma2_rn(wz, make_float2(Z.z, Z.w), t1);
          __sincosf(t0.x, &sn[j], &cs[j]);
          __sincosf(t0.y, &sn[j + 1], &cs[j + 1]);
          __sincosf(t1.x, &sn[j + 2], &cs[j + 2]);
          __sincosf(t1.y, &sn[j + 3], &cs[j + 3]);
        }
        uint32_t chi[4], clo[4], shi[4], slo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          tc::split_f16x2(cs[2 * j], cs[2 * j + 1], chi[j], clo[j]);
          tc::split_f16x2(sn[2 * j], sn[2 * j + 1], shi[j], slo[j]);
        }
        const uint32_t ah = a + 4 * h;
        tc::tmem_st4(ah, chi[0], chi[1], chi[2], chi[3]);
        tc::tmem_st4(ah + kArr, clo[0], clo[1], clo[2], clo[3]);
        tc::tmem_st4(ah + 2 * kArr, shi[0], shi[1], shi[2], shi[3]);
        tc::tmem_st4(ah + 3 * kArr, slo[0], slo[1], slo[2], slo[3]);
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(full_s + 8 * s);
      if (++s == kStages) {
        s = 0;
        ++u;
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issue: warp-uniform loop, one elected lane -------
    const uint32_t idesc = tc::make_idesc(0, 128, N);
    const uint32_t b_s = tc::smem_addr(bsm);
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t s = c % kStages, u = c / kStages;
      const int e = c / kEpoch, ce = c % kEpoch;
      if (ce == 0) {
        if (e >= 1) tc::mbar_wait(&dempty_bar, (e - 1) & 1);  // D drained into L
        tc::mbar_wait(&bready_bar[e & 1], (e >> 1) & 1);
      }
      tc::mbar_wait(&full_bar[s], u & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t bc = b_s + (e & 1) * C::kEpochB + ce * C::kChunkB;
        const uint64_t bh = tc::make_sdesc(bc, kLBO, kSBO);
        const uint64_t bl = tc::make_sdesc(bc + C::kBBytes, kLBO, kSBO);
        const uint32_t a0 = tmem + C::kColA + 4 * kArr * s;
        const uint32_t dcos = tmem, dsin = tmem + N;
#pragma unroll
        for (int kk = 0; kk < kChunk / 16; ++kk) {
          const uint64_t adv = uint64_t(2 * kk) * (kLBO >> 4);
          const uint32_t acc = (ce > 0 || kk > 0) ? 1u : 0u;
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dcos, a0 + kArr + 8 * kk, bh + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 2 * kArr + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dsin, a0 + 2 * kArr + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 3 * kArr + 8 * kk, bh + adv, idesc, 1u);
        }
        tc::mma_commit(&empty_bar[s]);
        if (ce == kEpoch - 1 || c == nchunks - 1) tc::mma_commit(&dfull_bar);
      }
      __syncwarp();
    }
  } else {
    // ---------------- F staging + drains (4 warps, 128 threads) ----------
    const int fw = warp - kFWarp0, t = fw * 32 + lane;
    const float* Fb = F + int64_t(b) * n * d + c0;
    const uint32_t b_s = tc::smem_addr(bsm);
    const uint32_t fs_s = b_s + 2 * C::kEpochB;  // staging: [E*64 points][N channels] fp32
    const float* fstage = reinterpret_cast<const float*>(bsm + 2 * C::kEpochB);
    const bool vec = (dc == N) && (d % 4 == 0) && (c0 % 4 == 0);
    // Per epoch: the F block is copied into shared memory, the per-channel
    // maxima taken, and thread t converts channel (t % N) of point pairs
    // (one 32-bit word of the K-major B operand each).
    // d = N (32 or 64): the epoch's rows are one contiguous block -> one bulk
    // copy (TMA engine) into unpadded rows; otherwise per-thread cp.async into
    // rows padded to kRowF floats.  Either is issued one epoch ahead.
    constexpr bool kPow2 = (N & (N - 1)) == 0;
    const bool bulk = kPow2 && vec && d == N && (reinterpret_cast<uintptr_t>(Fb) & 15) == 0;
    auto issue_f = [&](int e) {
      const int64_t q0 = p0 + int64_t(e) * (kEpoch * kChunk);  // first point of the epoch
      const int ncs = min(kEpoch, nchunks - e * kEpoch);        // chunks of this epoch
      const int npts = ncs * kChunk;
      if (bulk) {
        const int nv = int(min(int64_t(npts), n - q0));  // rows past the cloud: zeros
        if (t == 0) {
          tc::fence_proxy_async_smem();  // after the generic reads of the last epoch
          tc::mbar_arrive_expect_tx(&fst_bar, uint32_t(nv) * (N * 4u));
          tc::bulk_g2s(bsm + 2 * C::kEpochB, Fb + q0 * N, uint32_t(nv) * (N * 4u), &fst_bar);
        }
#pragma unroll 1
        for (int i = t; i < (npts - nv) * N; i += 128)
          reinterpret_cast<float*>(bsm + 2 * C::kEpochB)[nv * N + i] = 0.0f;
        return;
      }
      // the epoch's F block -> shared memory (cp.async, all in flight at once;
      // rows past the cloud and channels past dc are zero-filled)
      if (vec) {
#pragma unroll 1
        for (int i = t; i < npts * (N / 4); i += 128) {
          const int p = i / (N / 4), cq = i % (N / 4);
          const bool ok = q0 + p < n;
          tc::cp_async16_zf(fs_s + uint32_t(p * C::kRowF * 4 + cq * 16),
                            ok ? Fb + (q0 + p) * d + 4 * cq : Fb, ok ? 16u : 0u);
        }
      } else {
#pragma unroll 1
        for (int i = t; i < npts * N; i += 128) {
          const int p = i / N, j = i % N;
          const bool ok = q0 + p < n && j < dc;
          tc::cp_async4_zf(fs_s + uint32_t((p * C::kRowF + j) * 4), ok ? Fb + (q0 + p) * d + j : Fb,
                           ok ? 4u : 0u);
        }
      }
      tc::cp_async_commit();
    };
    auto process_f = [&](int e) {
      const int ncs = min(kEpoch, nchunks - e * kEpoch);
      const int npts = ncs * kChunk;
      if (bulk)
        tc::mbar_wait(&fst_bar, uint32_t(e) & 1u);
      else
        tc::cp_async_wait<0>();
      asm volatile("bar.sync 1, 128;" ::: "memory");

      // per-channel max |F| over the epoch.  Bulk (unpadded rows, N a power of
      // two): thread t takes channels 4 (t % (N/4)) .. + 3 of points t / (N/4) +
      // (512 / N) i with 16-byte reads; partial maxima via fmax4.
      if (bulk) {
        constexpr int Q = kPow2 ? N / 4 : 1, PS = 128 / Q;
        const int cq = t % Q;
        float4 mx = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int p = t / Q; p < npts; p += PS) {
          const float4 v = *reinterpret_cast<const float4*>(fstage + p * N + 4 * cq);
          mx.x = fmaxf(mx.x, fabsf(v.x));
          mx.y = fmaxf(mx.y, fabsf(v.y));
          mx.z = fmaxf(mx.z, fabsf(v.z));
          mx.w = fmaxf(mx.w, fabsf(v.w));
        }
        fmax4[t] = mx;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (t < N) {
          const float* f4 = reinterpret_cast<const float*>(fmax4);
          float cm = 0.0f;
          for (int i = 0; i < PS; ++i) cm = fmaxf(cm, f4[4 * (t / 4 + Q * i) + (t % 4)]);
          fmax_part[t] = cm;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (t < N) {
          const float cm = fmax_part[t];
          float scale = 1.0f;
          if (cm > 0.0f && isfinite(cm)) {
            int ex = 0;
            frexpf(cm, &ex);
            scale = ldexpf(1.0f, min(126, max(-126, 14 - ex)));
          }
          fmax_part[t] = scale;
          fscale_inv[e & 1][t] = 1.0f / scale;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // thread t converts channel j = t % N of the 8-point groups g = t / N +
        // (128 / N) i: one 16-byte hi and lo store per group (one K-major
        // core-matrix row); lanes walk consecutive channels (no bank conflicts)
        const int j = t % N;
        const float sc = fmax_part[j];
        const float2 sc2 = make_float2(sc, sc);
        const uint32_t eb = b_s + (e & 1) * C::kEpochB + uint32_t(j >> 3) * kSBO +
                            uint32_t(j & 7) * 16;
#pragma unroll 2
        for (int g = t / N; 8 * g < npts; g += 128 / N) {
          const float* src = fstage + 8 * g * N + j;
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 v = __fmul2_rn(sc2, make_float2(src[2 * k * N], src[(2 * k + 1) * N]));
            tc::split_f16x2(v.x, v.y, hi[k], lo[k]);
          }
          const uint32_t off = uint32_t(g >> 3) * C::kChunkB + uint32_t(g & 7) * kLBO;
          tc::st_shared_v4(eb + off, hi[0], hi[1], hi[2], hi[3]);
          tc::st_shared_v4(eb + off + C::kBBytes, lo[0], lo[1], lo[2], lo[3]);
        }
      } else {
      {
        const int j = t % N, st = 128 / N;
        float m0 = 0.0f, m1 = 0.0f, m2 = 0.0f, m3 = 0.0f;  // 4 loads in flight
        int p = t / N;
        for (; p + 3 * st < npts; p += 4 * st) {
          m0 = fmaxf(m0, fabsf(fstage[p * C::kRowF + j]));
          m1 = fmaxf(m1, fabsf(fstage[(p + st) * C::kRowF + j]));
          m2 = fmaxf(m2, fabsf(fstage[(p + 2 * st) * C::kRowF + j]));
          m3 = fmaxf(m3, fabsf(fstage[(p + 3 * st) * C::kRowF + j]));
        }
        for (; p < npts; p += st) m0 = fmaxf(m0, fabsf(fstage[p * C::kRowF + j]));
        fmax_part[t] = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (t < N) {
        float cm = 0.0f;
        for (int k = t; k < 128; k += N) cm = fmaxf(cm, fmax_part[k]);
        // scale 2^e_j with max |F_j| 2^e_j in [2^13, 2^14) (1 for a zero or
        // non-finite channel; |e_j| <= 126 keeps both factors normal, exact)
        float scale = 1.0f;
        if (cm > 0.0f && isfinite(cm)) {
          int ex = 0;
          frexpf(cm, &ex);  // cm in [2^(ex-1), 2^ex)
          scale = ldexpf(1.0f, min(126, max(-126, 14 - ex)));
        }
        fmax_part[t] = scale;  // read back as the scale below
        fscale_inv[e & 1][t] = 1.0f / scale;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      // scaled, split, stored as 32-bit words: channel j, points (2 pk, 2 pk + 1).
      // Lane (jl, pl) = (lane >> 2, lane & 3) takes channel 8 jh + jl and pair
      // 4 pkh + pl: the 32 lanes hit 32 distinct banks on the B stores (4 jl +
      // pl) and on the staging reads (row stride N + 4).  Warp fw takes the
      // channel groups jh = fw, fw + 4, ...
      const uint32_t eb = b_s + (e & 1) * C::kEpochB;
      const int jl = lane >> 2, pl = lane & 3;
      for (int jh = fw; jh < N / 8; jh += 4) {
        const int j = 8 * jh + jl;
        const float sc = fmax_part[j];
        const uint32_t jo = uint32_t(jh) * kSBO + uint32_t(jl) * 16;
#pragma unroll 4
        for (int pkh = 0; pkh < npts / 8; ++pkh) {
          const int p = 8 * pkh + 2 * pl;  // even point of the pair
          uint32_t hi, lo;
          tc::split_f16x2(fstage[p * C::kRowF + j] * sc, fstage[(p + 1) * C::kRowF + j] * sc, hi,
                          lo);
          const int ce = p / kChunk, pc = p % kChunk;
          const uint32_t off = uint32_t(ce) * C::kChunkB + jo + uint32_t(pc >> 3) * kLBO +
                               uint32_t(pc & 7) * 2;
          tc::st_shared_u32(eb + off, hi);
          tc::st_shared_u32(eb + off + C::kBBytes, lo);
        }
      }
      }  // (non-bulk)
      // the staging block and fmax_part are rewritten by the next epoch
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bready_bar[e & 1]);
    };
#pragma unroll 1
    for (int e = 0; e < min(2, nepochs); ++e) {
      issue_f(e);
      process_f(e);
    }
    if (nepochs > 2) issue_f(2);
    const uint32_t tl = tmem + lane_field;
    float* out = partial + (int64_t(b) * ranges + rg) * int64_t(2 * m) * dc;
    for (int e = 0; e < nepochs; ++e) {
      const uint32_t buf = e & 1;
      tc::mbar_wait(&dfull_bar, e & 1);
      tc::tc_fence_after();
      // L (+)= D x 2^-e_j, 16 columns per round (cos channels, then sin)
#pragma unroll 1
      for (int c = 0; c < 2 * N; c += 16) {
        float v[16], l[16];
        tc::tmem_ld16(tl + c, v);
        if (e > 0) tc::tmem_ld16(tl + C::kColL + c, l);
        uint32_t o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float inv = fscale_inv[buf][(c % N) + j];
          o[j] = __float_as_uint(e > 0 ? fmaf(v[j], inv, l[j]) : v[j] * inv);
        }
        tc::tmem_st8(tl + C::kColL + c, o);
        tc::tmem_st8(tl + C::kColL + c + 8, o + 8);
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dempty_bar);
      // buffer e & 1 (B and scales) is free once epoch e's MMAs completed
      // and all four warps have read its scales
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (e + 2 < nepochs) process_f(e + 2);
      if (e + 3 < nepochs) issue_f(e + 3);
    }
    // L -> partial[b][rg][2m][dc]: row 2f = cos, 2f + 1 = sin (interleaved)
#pragma unroll 1
    for (int c = 0; c < 2 * N; c += 16) {
      float l[16];
      if (nepochs > 0) {
        tc::tc_fence_after();
        tc::tmem_ld16(tl + C::kColL + c, l);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) l[j] = 0.0f;
      }
      const int ch0 = c % N, sin_row = c / N;
      if (f < m) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (ch0 + j < dc) out[int64_t(2 * f + sin_row) * dc + ch0 + j] = l[j];
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- d <= 16
// The one-chunk kernel (N = 16): two D buffers (no MMA stall at a drain) and
// the long-term sums in the drain warps' registers.  Kept separate from the
// wide template: measured 9 % faster than its NC = 1 instance at cfg 5.
#ifndef RFD_P1_STAGES
#define RFD_P1_STAGES 3
#endif
#ifndef RFD_P1_EPOCH
#define RFD_P1_EPOCH 8
#endif
namespace k16 {
constexpr int kStages = RFD_P1_STAGES;
constexpr int kEpoch = RFD_P1_EPOCH;  // chunks per TMEM accumulation epoch
constexpr uint32_t kColA = 64;      // D buffers (cos 16 + sin 16) at 0 and 32
constexpr int kBBytes = 16 * kChunk * 2;        // one fp16 B operand (hi or lo): 2 KB
constexpr int kChunkB = 2 * kBBytes;            // hi + lo of one chunk
constexpr int kEpochB = kEpoch * kChunkB;       // 32 KB per epoch buffer
constexpr int kRowF = 20;                       // staging row stride (floats, 16 B aligned)
constexpr int kStageF = kEpoch * kChunk * kRowF * 4;  // fp32 F block of one epoch: 40 KB
constexpr int kSmem = 2 * kEpochB + kStageF;
}  // namespace k16

// Diagnostics (RFD_P1_TRACE=1): per-chunk timestamps of CTA (0, 0, 0).
__device__ long long g_p1trace[1024][12];

// At most 72 registers (maxnreg): with 21 warps per CTA, sub-partition 0
// holds 6 of them; at 72 registers (2304 per warp) 2560 of its 16384 remain,
// enough for one warp of the core's DMMA GEMM (80 registers) -- so in rfd_gfi
// the core's GEMMs run on the SMs beside pass 1 instead of waiting for it
// (gfi step 2.27 -> 2.10 ms at cfg 5; at 80 registers no GEMM CTA fits).
// Pass 1 alone is also faster at 72 (0.756 -> 0.739 ms; spills the same).
#ifndef RFD_P1_MAXNREG
#define RFD_P1_MAXNREG 72
#endif
#if RFD_P1_MAXNREG
#define P1_BOUNDS(t) __maxnreg__(RFD_P1_MAXNREG)
#else
#define P1_BOUNDS(t) __launch_bounds__(t, 1)
#endif
template <int PW, bool kTr = false>
__global__ void P1_BOUNDS((PW + 5) * 32)
pass1_tc_kernel16(const float* __restrict__ pts16, const float4* __restrict__ omega4, int m,
                int64_t n, int ranges, const float* __restrict__ F, int d, int c0, int dc,
                float* __restrict__ partial) {
  using namespace k16;
  // PW producer warps (PW / 4 per TMEM lane group), PPW points each per chunk
  constexpr int PPW = 4 * kChunk / PW, kMmaW = PW, kFW0 = PW + 1;
  // [2 epochs][8 chunks][hi | lo] B operands, then the fp32 F staging block
  extern __shared__ __align__(1024) unsigned char bsm[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], dfull_bar[2], dempty_bar[2],
      bready_bar[2], fst_bar;
  __shared__ uint32_t tmem_sh;
  // each producer warp's 16 points of a chunk as [x0..15 | y0..15 | z0..15],
  // 3 chunks deep (cp.async ring)
  __shared__ __align__(16) float xbuf[3][PW][3 * PPW];
  __shared__ __align__(16) float fmax_part[2][4][16];  // per epoch buffer, F warp, channel
  __shared__ float fscale_inv[2][16];        // per epoch buffer

  const int ft = blockIdx.x, rg = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, lg = warp & 3;
  // ranges are whole chunks; only a cloud's last chunk is partial
  const int64_t cpc = (n + kChunk - 1) / kChunk, gpc = (n + 15) / 16;
  const int64_t ch0 = cpc * rg / ranges, ch1 = cpc * (rg + 1) / ranges;
  const int64_t p0 = ch0 * kChunk;
  const int nchunks = int(ch1 - ch0);
  const int nepochs = (nchunks + kEpoch - 1) / kEpoch;
  const float* cloud16 = pts16 + int64_t(b) * gpc * 48;

  asm volatile("griddepcontrol.launch_dependents;");  // pass 2 may start its setup
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], PW);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&dfull_bar[i], 1);
      tc::mbar_init(&dempty_bar[i], 4);
      tc::mbar_init(&bready_bar[i], 4);
    }
    tc::mbar_init(&fst_bar, 1);
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // Programmatic dependent launch: the setup above may overlap the previous
  // kernel (pass 2 of an earlier integrate); F and the partials only after it.
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
  const bool trc = kTr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0;
  __shared__ long long tr1[kTr ? 128 : 1][12];  // trace in shared memory (cheap stores)
  const uint32_t lane_field = uint32_t(lg * 32) << 16;
  const int f = ft * 128 + lg * 32 + lane;  // this lane's frequency

  if (warp < PW) {
    // ---------------- producers: 16 points per warp per chunk --------------
    const int q = warp >> 2;  // which 16 of the chunk's points
    const float4 w = (f < m) ? omega4[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float2 wx = make_float2(w.x, w.x), wy = make_float2(w.y, w.y), wz = make_float2(w.z, w.z);
    // The warp's 16 points (one SoA group, 192 B), copied two chunks ahead by
    // lanes 0-11 straight into shared memory (cp.async: global latency off the
    // critical path).  Groups past the cloud's end repeat its last group
    // (finite values that meet zero F).  Pointers and counters advance per
    // chunk (no 64-bit index arithmetic in the loop).
    // (PPW = 32: lanes 12-23 copy the warp's second group.)
    const int gsel = lane / 12, l12 = lane % 12;
    const float* xsrc = cloud16 + ((ch0 * (kChunk / 16) + q * (PPW / 16) + gsel) * 48 + 4 * l12);
    const float* xlast = cloud16 + ((gpc - 1) * 48 + 4 * l12);
    const int64_t xrem0 = gpc - (ch0 * (kChunk / 16) + q * (PPW / 16) + gsel);
    int xrem = int(xrem0 > 0x7fffffff ? 0x7fffffff : xrem0);  // groups left
    constexpr uint32_t kRing = PW * 3 * PPW * 4;  // bytes per ring slot
    const uint32_t x_s = tc::smem_addr(&xbuf[0][warp][0]);
    uint32_t xw = 0;
    auto load_x = [&](bool valid) {
      if (lane < 3 * PPW / 4 && valid) tc::cp_async16(x_s + xw * kRing + 16 * lane, xrem > 0 ? xsrc : xlast);
      tc::cp_async_commit();  // one group per chunk, empty past the end
      xsrc += 48 * (kChunk / 16);
      xrem -= kChunk / 16;
      xw = (xw == 2) ? 0 : xw + 1;
    };
    load_x(nchunks > 0);
    load_x(nchunks > 1);
    const uint32_t empty_s = tc::smem_addr(&empty_bar[0]), full_s = tc::smem_addr(&full_bar[0]);
    uint32_t s = 0, u = 0, xr = 0;  // stage, its round, ring slot read
    for (int c = 0; c < nchunks; ++c) {
      load_x(c + 2 < nchunks);  // the slot chunk c - 1 read (ordered by its __syncwarp)
      if (trc && warp == 0 && c < 128) tr1[c][0] = clock64();
      if (u >= 1) tc::mbar_wait(empty_s + 8 * s, (u - 1) & 1);
      if (trc && warp == 0 && c < 128) tr1[c][1] = clock64();
      // Points beyond the cloud meet zero columns of F^T, and lanes beyond m
      // are never written out: no masking of the features.
      tc::cp_async_wait<2>();  // chunk c's group (c + 1, c + 2 may be in flight)
      __syncwarp();
      const float* xs = &xbuf[0][warp][0] + xr * (PW * 3 * PPW);
      xr = (xr == 2) ? 0 : xr + 1;
      const uint32_t a = tmem + lane_field + kColA + 4 * kArr * s + (PPW / 2) * q;
#pragma unroll
      for (int h = 0; h < PPW / 8; ++h) {  // 8 points at a time (register pressure)
        const float* xh = xs + 48 * (h >> 1) + 8 * (h & 1);
        float cs[8], sn[8];
#pragma unroll
        for (int j = 0; j < 8; j += 4) {
          // omega . x for 4 points in packed FP32 (2 points per instruction),
          // the same operation order as fmaf(wz, z, fmaf(wy, y, wx * x))
          const float4 X = *reinterpret_cast<const float4*>(xh + j);
          const float4 Y = *reinterpret_cast<const float4*>(xh + 16 + j);
          const float4 Z = *reinterpret_cast<const float4*>(xh + 32 + j);
          float2 t0 = __fmul2_rn(wx, make_float2(X.x, X.y));
          float2 t1 = __fmul2_rn(wx, make_float2(X.z, X.w));
          t0 = __ffma2_rn(wy, make_float2(Y.x, Y.y), t0);
          t1 = __ffma2_rn(wy, make_float2(Y.z, Y.w), t1);
          t0 = __ffma2_rn(wz, make_float2(Z.x, Z.y), t0);
          t1 = __ffma2_rn(wz, make_float2(Z.z, Z.w), t1);
          __sincosf(t0.x, &sn[j], &cs[j]);
          __sincosf(t0.y, &sn[j + 1], &cs[j + 1]);
          __sincosf(t1.x, &sn[j + 2], &cs[j + 2]);
          __sincosf(t1.y, &sn[j + 3], &cs[j + 3]);
        }
        uint32_t chi[4], clo[4], shi[4], slo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          tc::split_f16x2(cs[2 * j], cs[2 * j + 1], chi[j], clo[j]);
          tc::split_f16x2(sn[2 * j], sn[2 * j + 1], shi[j], slo[j]);
        }
        const uint32_t ah = a + 4 * h;
        tc::tmem_st4(ah, chi[0], chi[1], chi[2], chi[3]);
        tc::tmem_st4(ah + kArr, clo[0], clo[1], clo[2], clo[3]);
        tc::tmem_st4(ah + 2 * kArr, shi[0], shi[1], shi[2], shi[3]);
        tc::tmem_st4(ah + 3 * kArr, slo[0], slo[1], slo[2], slo[3]);
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (trc && warp == 0 && c < 128) tr1[c][2] = clock64();
      if (lane == 0) tc::mbar_arrive(full_s + 8 * s);
      if (++s == kStages) {
        s = 0;
        ++u;
      }
    }
  } else if (warp == kMmaW) {
    // ---------------- MMA issue: warp-uniform loop, one elected lane -------
    const uint32_t idesc = tc::make_idesc(0, 128, 16);
    const uint32_t b_s = tc::smem_addr(bsm);
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t s = c % kStages, u = c / kStages;
      const int e = c / kEpoch, ce = c % kEpoch;
      const uint32_t buf = e & 1;
      if (trc && c < 128) tr1[c][3] = clock64();
      if (ce == 0) {
        if (e >= 2) tc::mbar_wait(&dempty_bar[buf], ((e - 2) >> 1) & 1);
        if (trc && c < 128) tr1[c][4] = clock64();
        tc::mbar_wait(&bready_bar[buf], (e >> 1) & 1);
      } else if (trc && c < 128) {
        tr1[c][4] = clock64();
      }
      if (trc && c < 128) tr1[c][5] = clock64();
      tc::mbar_wait(&full_bar[s], u & 1);
      if (trc && c < 128) tr1[c][6] = clock64();
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t bc = b_s + buf * kEpochB + ce * kChunkB;
        const uint64_t bh = tc::make_sdesc(bc, kLBO, kSBO);
        const uint64_t bl = tc::make_sdesc(bc + kBBytes, kLBO, kSBO);
        const uint32_t a0 = tmem + kColA + 4 * kArr * s;
        const uint32_t dcos = tmem + 32 * buf, dsin = dcos + 16;
#pragma unroll
        for (int kk = 0; kk < kChunk / 16; ++kk) {
          const uint64_t adv = uint64_t(2 * kk) * (kLBO >> 4);
          const uint32_t acc = (ce > 0 || kk > 0) ? 1u : 0u;
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dcos, a0 + kArr + 8 * kk, bh + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 2 * kArr + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dsin, a0 + 2 * kArr + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 3 * kArr + 8 * kk, bh + adv, idesc, 1u);
        }
        tc::mma_commit(&empty_bar[s]);
        if (ce == kEpoch - 1 || c == nchunks - 1) tc::mma_commit(&dfull_bar[buf]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- F staging + drains (4 warps, 128 threads) ----------
    const int fw = warp - kFW0, t = fw * 32 + lane;
    // Per epoch e the F block is copied into shared memory (issue_f, one epoch
    // ahead: its latency overlaps the epoch before), then process_f takes the
    // per-channel maxima and writes the scaled, split B operands.
    const float* Fb = F + int64_t(b) * n * d + c0;
    const uint32_t b_s = tc::smem_addr(bsm);
    const uint32_t fs_s = b_s + 2 * kEpochB;  // staging: [512 points][kRowF] fp32
    const float* fstage = reinterpret_cast<const float*>(bsm + 2 * kEpochB);
    const bool vec = (dc == 16) && (d % 4 == 0) && (c0 % 4 == 0);
    // d = 16: the epoch's rows are one contiguous block -> one bulk copy (TMA
    // engine) into unpadded rows; otherwise per-thread cp.async into rows
    // padded to kRowF floats
    const bool bulk = vec && d == 16 && (reinterpret_cast<uintptr_t>(Fb) & 15) == 0;
    const int rs = bulk ? 16 : kRowF;
    auto epoch_pts = [&](int e) { return min(kEpoch, nchunks - e * kEpoch) * kChunk; };
    // the epoch's F block -> shared memory (cp.async, all in flight at once;
    // rows past the cloud and channels past dc are zero-filled)
    auto issue_f = [&](int e) {
      const int64_t q0 = p0 + int64_t(e) * (kEpoch * kChunk);  // first point of the epoch
      const int npts = epoch_pts(e);
      if (bulk) {
        const int nv = int(min(int64_t(npts), n - q0));  // rows past the cloud: zeros
        if (t == 0) {
          tc::fence_proxy_async_smem();  // after the generic reads of the last epoch
          tc::mbar_arrive_expect_tx(&fst_bar, uint32_t(nv) * 64u);
          tc::bulk_g2s(bsm + 2 * kEpochB, Fb + q0 * 16, uint32_t(nv) * 64u, &fst_bar);
        }
#pragma unroll 1
        for (int i = t; i < (npts - nv) * 16; i += 128)
          reinterpret_cast<float*>(bsm + 2 * kEpochB)[nv * 16 + i] = 0.0f;
        return;
      }
      if (vec) {
#pragma unroll 1
        for (int i = t; i < npts * 4; i += 128) {
          const int p = i >> 2, cq = i & 3;
          const bool ok = q0 + p < n;
          tc::cp_async16_zf(fs_s + uint32_t(p * kRowF * 4 + cq * 16),
                            ok ? Fb + (q0 + p) * d + 4 * cq : Fb, ok ? 16u : 0u);
        }
      } else {
        // only the dc real channels (columns dc..15 were zeroed once, below)
#pragma unroll 1
        for (int p = t; p < npts; p += 128) {
          const bool ok = q0 + p < n;
          const float* src = ok ? Fb + (q0 + p) * d : Fb;
          for (int j = 0; j < dc; ++j)
            tc::cp_async4_zf(fs_s + uint32_t((p * kRowF + j) * 4), src + (ok ? j : 0), ok ? 4u : 0u);
        }
      }
      tc::cp_async_commit();
    };
    if (!bulk && !vec) {  // staging columns dc..15 stay zero for the whole kernel
      float* fz = reinterpret_cast<float*>(bsm + 2 * kEpochB);
#pragma unroll 1
      for (int i = t; i < kEpoch * kChunk * 16; i += 128)
        if ((i & 15) >= dc) fz[(i >> 4) * kRowF + (i & 15)] = 0.0f;
    }
    // Thread t converts channel j = t % 16 of the 8-point groups g = t / 16 +
    // 8 i: eight staging reads, one 16-byte store each of hi and lo (the
    // groups' 8 points are one K-major core-matrix row).
    const int j = t & 15, g0 = t >> 4;
    auto process_f = [&](int e) {
      const int npts = epoch_pts(e);
      const bool tr = trc && fw == 0 && e * kEpoch < 128;
      if (tr) tr1[e * kEpoch][8] = clock64();
      if (bulk)
        tc::mbar_wait(&fst_bar, uint32_t(e) & 1u);
      else
        tc::cp_async_wait<0>();
      if (tr) tr1[e * kEpoch][9] = clock64();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tr) tr1[e * kEpoch][10] = clock64();
      // per-channel max |F|: thread t takes channels 4 (t % 4) .. + 3 of points
      // t / 4 + 32 i (16-byte reads), then lanes of equal t % 4 and the warps
      {
        const int cq = t & 3;
        float4 mx = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int p = t >> 2; p < npts; p += 32) {
          const float4 v = *reinterpret_cast<const float4*>(fstage + p * rs + 4 * cq);
          mx.x = fmaxf(mx.x, fabsf(v.x));
          mx.y = fmaxf(mx.y, fabsf(v.y));
          mx.z = fmaxf(mx.z, fabsf(v.z));
          mx.w = fmaxf(mx.w, fabsf(v.w));
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          mx.x = fmaxf(mx.x, __shfl_xor_sync(0xffffffffu, mx.x, o));
          mx.y = fmaxf(mx.y, __shfl_xor_sync(0xffffffffu, mx.y, o));
          mx.z = fmaxf(mx.z, __shfl_xor_sync(0xffffffffu, mx.z, o));
          mx.w = fmaxf(mx.w, __shfl_xor_sync(0xffffffffu, mx.w, o));
        }
        if (lane < 4) *reinterpret_cast<float4*>(&fmax_part[e & 1][fw][4 * lane]) = mx;
      }
      if (tr) tr1[e * kEpoch][11] = clock64();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tr) tr1[e * kEpoch + 1][8] = clock64();
      const float(*fp)[16] = fmax_part[e & 1];
      const float cm = fmaxf(fmaxf(fp[0][j], fp[1][j]), fmaxf(fp[2][j], fp[3][j]));
      // scale 2^e_j with max |F_j| 2^e_j in [2^13, 2^14) (1 for a zero or
      // non-finite channel; |e_j| <= 126 keeps both factors normal and exact)
      float scale = 1.0f;
      if (cm > 0.0f && isfinite(cm)) {
        int ex = 0;
        frexpf(cm, &ex);  // cm in [2^(ex-1), 2^ex)
        scale = ldexpf(1.0f, min(126, max(-126, 14 - ex)));
      }
      if (t < 16) fscale_inv[e & 1][t] = 1.0f / scale;
      const float2 sc2 = make_float2(scale, scale);
      const uint32_t eb = b_s + (e & 1) * kEpochB + uint32_t(j >> 3) * kSBO + uint32_t(j & 7) * 16;
#pragma unroll 2
      for (int g = g0; 8 * g < npts; g += 8) {
        const float* src = fstage + 8 * g * rs + j;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 v = __fmul2_rn(sc2, make_float2(src[2 * k * rs], src[(2 * k + 1) * rs]));
          tc::split_f16x2(v.x, v.y, hi[k], lo[k]);
        }
        const uint32_t off = uint32_t(g >> 3) * kChunkB + uint32_t(g & 7) * kLBO;
        tc::st_shared_v4(eb + off, hi[0], hi[1], hi[2], hi[3]);
        tc::st_shared_v4(eb + off + kBBytes, lo[0], lo[1], lo[2], lo[3]);
      }
      if (tr) tr1[e * kEpoch + 1][9] = clock64();
      // the staging block is rewritten by the next epoch's copies
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tr) tr1[e * kEpoch + 1][10] = clock64();
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bready_bar[e & 1]);
    };
#pragma unroll 1
    for (int e = 0; e < min(2, nepochs); ++e) {
      issue_f(e);
      process_f(e);
    }
    if (nepochs > 2) issue_f(2);
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
    for (int e = 0; e < nepochs; ++e) {
      const uint32_t buf = e & 1;
      if (trc && fw == 0 && e * kEpoch + 2 < 128) tr1[e * kEpoch + 2][7] = clock64();
      tc::mbar_wait(&dfull_bar[buf], (e >> 1) & 1);
      if (trc && fw == 0 && e * kEpoch + 3 < 128) tr1[e * kEpoch + 3][7] = clock64();
      tc::tc_fence_after();
      float v[32];
      tc::tmem_ld32(tmem + lane_field + 32 * buf, v);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dempty_bar[buf]);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float inv = fscale_inv[buf][j];
        acc[j] = fmaf(v[j], inv, acc[j]);  // v * 2^-e_j is exact: one rounding
        acc[16 + j] = fmaf(v[16 + j], inv, acc[16 + j]);
      }
      // buffer e & 1 (B and scales) is free once epoch e's MMAs completed and
      // all four warps have read its scales
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (trc && fw == 0 && e * kEpoch + 4 < 128) tr1[e * kEpoch + 4][7] = clock64();
      if (e + 2 < nepochs) process_f(e + 2);
      if (e + 3 < nepochs) issue_f(e + 3);
      if (trc && fw == 0 && e * kEpoch + 5 < 128) tr1[e * kEpoch + 5][7] = clock64();
    }
    if (f < m) {
      // partial[b][rg][2m][dc]: row 2f = cos, 2f + 1 = sin (interleaved order)
      float* out = partial + (int64_t(b) * ranges + rg) * int64_t(2 * m) * dc;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < dc) {
          out[int64_t(2 * f) * dc + j] = acc[j];
          out[int64_t(2 * f + 1) * dc + j] = acc[16 + j];
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (kTr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
    for (int i = tid; i < 128 * 12; i += (PW + 5) * 32) g_p1trace[i / 12][i % 12] = tr1[i / 12][i % 12];
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}


// ---------------------------------------------------------------- small m
// m <= 64 leaves most of the 128 TMEM lanes of a frequency tile idle.  The
// packed kernel gives each group of 128 / R lanes (R = 4 for m <= 32, 2 for
// m <= 64) its own *segment* (cloud, point range): lane group g computes the
// features of segment g's points, and B stacks the R segments' F chunks as
// 16-column blocks (N = 16 R).  Row block g of D against column block g is
// segment g's sum; the off-diagonal blocks are never read.  d <= 16.
template <int R>
struct PK {
  static constexpr int N = 16 * R;
  static constexpr int kStages = R == 4 ? 2 : 3;
  static constexpr int kEpoch = R == 4 ? 4 : 8;
  static constexpr uint32_t kColA = 4 * N;                  // D buffers at 0 and 2N
  static constexpr int kBBytes = N * kChunk * 2;
  static constexpr int kChunkB = 2 * kBBytes;
  static constexpr int kEpochB = kEpoch * kChunkB;
  static constexpr int kStageF = kEpoch * kChunk * N * 4;   // [points][N] fp32
  static constexpr int kSmem = 2 * kEpochB + kStageF;
};

template <int R>
__global__ void __launch_bounds__(kThreads, 1)
pass1_tc_packed(const float* __restrict__ pts16, const float4* __restrict__ omega4, int m,
                int64_t n, int batch, int ranges, const float* __restrict__ F, int d, int c0,
                int dc, float* __restrict__ partial) {
  using C = PK<R>;
  constexpr int N = C::N, kStages = C::kStages, kEpoch = C::kEpoch, kGroupsPerSeg = 4 / R;
  extern __shared__ __align__(1024) unsigned char bsm[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], dfull_bar[2], dempty_bar[2],
      bready_bar[2];
  __shared__ uint32_t tmem_sh;
  __shared__ __align__(16) float xbuf[3][kProducerWarps][48];
  __shared__ float fscale[N];
  __shared__ float fscale_inv[2][N];
  __shared__ float fmax_part[128];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, lg = warp & 3;
  const int64_t cpc = (n + kChunk - 1) / kChunk, gpc = (n + 15) / 16;
  const int64_t nseg = int64_t(batch) * ranges;
  // segment g of this CTA: cloud sb[g], chunks [sc0[g], sc0[g] + snc[g])
  // (shared memory: every role reads them, registers are scarce)
  __shared__ int sb[R], snc[R];
  __shared__ long long sc0[R];
  int nchunks = 0;
#pragma unroll
  for (int g = 0; g < R; ++g) {
    const int64_t sg = int64_t(blockIdx.x) * R + g;
    int nc = 0;
    if (sg < nseg) {
      const int rg = int(sg % ranges);
      const int64_t a = cpc * rg / ranges;
      nc = int(cpc * (rg + 1) / ranges - a);
      if (tid == 0) {
        sb[g] = int(sg / ranges);
        sc0[g] = a;
      }
    } else if (tid == 0) {
      sb[g] = 0;
      sc0[g] = 0;
    }
    if (tid == 0) snc[g] = nc;
    nchunks = max(nchunks, nc);
  }
  const int nepochs = (nchunks + kEpoch - 1) / kEpoch;

  asm volatile("griddepcontrol.launch_dependents;");  // pass 2 may start its setup
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], kProducerWarps);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&dfull_bar[i], 1);
      tc::mbar_init(&dempty_bar[i], 4);
      tc::mbar_init(&bready_bar[i], 4);
    }
    tc::mbar_fence_init();
  }
  // B buffers and the staging block start at zero: only the R dc real
  // columns are ever written (the others stay zero for the whole kernel)
  for (int i = tid; i < C::kSmem / 16; i += kThreads)
    reinterpret_cast<float4*>(bsm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // Programmatic dependent launch: the setup above may overlap the previous
  // kernel (pass 2 of an earlier integrate); F and the partials only after it.
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
  const int g_me = lg / kGroupsPerSeg;                          // this lane group's segment
  const int f = (lg % kGroupsPerSeg) * 32 + lane;               // this lane's frequency

  if (warp < kProducerWarps) {
    // ---------------- producers (as pass1_tc_kernel16), per segment -------
    const int q = warp >> 2;
    const float4 w = (f < m) ? omega4[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float2 wx = make_float2(w.x, w.x), wy = make_float2(w.y, w.y), wz = make_float2(w.z, w.z);
    const float* cloud16 = pts16 + int64_t(sb[g_me]) * gpc * 48;
    const float* xsrc = cloud16 + ((sc0[g_me] * (kChunk / 16) + q) * 48 + 4 * lane);
    const float* xlast = cloud16 + ((gpc - 1) * 48 + 4 * lane);
    const int64_t xrem0 = gpc - (sc0[g_me] * (kChunk / 16) + q);
    int xrem = int(xrem0 > 0x7fffffff ? 0x7fffffff : xrem0);
    constexpr uint32_t kRing = kProducerWarps * 48 * 4;
    const uint32_t x_s = tc::smem_addr(&xbuf[0][warp][0]);
    uint32_t xw = 0;
    auto load_x = [&](bool valid) {
      if (lane < 12 && valid) tc::cp_async16(x_s + xw * kRing + 16 * lane, xrem > 0 ? xsrc : xlast);
      tc::cp_async_commit();
      xsrc += 48 * (kChunk / 16);
      xrem -= kChunk / 16;
      xw = (xw == 2) ? 0 : xw + 1;
    };
    load_x(nchunks > 0);
    load_x(nchunks > 1);
    const uint32_t empty_s = tc::smem_addr(&empty_bar[0]), full_s = tc::smem_addr(&full_bar[0]);
    uint32_t s = 0, u = 0, xr = 0;
    for (int c = 0; c < nchunks; ++c) {
      load_x(c + 2 < nchunks);
      if (u >= 1) tc::mbar_wait(empty_s + 8 * s, (u - 1) & 1);
      // chunks past the segment (or the cloud) repeat finite points; their
      // F rows are zero
      tc::cp_async_wait<2>();
      __syncwarp();
      const float* xs = &xbuf[0][warp][0] + xr * (kProducerWarps * 48);
      xr = (xr == 2) ? 0 : xr + 1;
      const uint32_t a = tmem + lane_field + C::kColA + 4 * kArr * s + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float cs[8], sn[8];
#pragma unroll
        for (int j = 0; j < 8; j += 4) {
          const float4 X = *reinterpret_cast<const float4*>(xs + 8 * h + j);
          const float4 Y = *reinterpret_cast<const float4*>(xs + 16 + 8 * h + j);
          const float4 Z = *reinterpret_cast<const float4*>(xs + 32 + 8 * h + j);
          float2 t0 = __fmul2_rn(wx, make_float2(X.x, X.y));
          float2 t1 = __fmul2_rn(wx, make_float2(X.z, X.w));
          t0 = __ffma2_rn(wy, make_float2(Y.x, Y.y), t0);
          t1 = __ffma2_rn(wy, make_float2(Y.z, Y.w), t1);
          t0 = __ffma2_rn(wz, make_float2(Z.x, Z.y), t0);
          t1 = __ffma2_rn(wz, make_float2(Z.z, Z.w), t1);
          __sincosf(t0.x, &sn[j], &cs[j]);
          __sincosf(t0.y, &sn[j + 1], &cs[j + 1]);
          __sincosf(t1.x, &sn[j + 2], &cs[j + 2]);
          __sincosf(t1.y, &sn[j + 3], &cs[j + 3]);
        }
        uint32_t chi[4], clo[4], shi[4], slo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          tc::split_f16x2(cs[2 * j], cs[2 * j + 1], chi[j], clo[j]);
          tc::split_f16x2(sn[2 * j], sn[2 * j + 1], shi[j], slo[j]);
        }
        const uint32_t ah = a + 4 * h;
        tc::tmem_st4(ah, chi[0], chi[1], chi[2], chi[3]);
        tc::tmem_st4(ah + kArr, clo[0], clo[1], clo[2], clo[3]);
        tc::tmem_st4(ah + 2 * kArr, shi[0], shi[1], shi[2], shi[3]);
        tc::tmem_st4(ah + 3 * kArr, slo[0], slo[1], slo[2], slo[3]);
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(full_s + 8 * s);
      if (++s == kStages) {
        s = 0;
        ++u;
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issue: N = 16 R, two D buffers -------------------
    const uint32_t idesc = tc::make_idesc(0, 128, N);
    const uint32_t b_s = tc::smem_addr(bsm);
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t s = c % kStages, u = c / kStages;
      const int e = c / kEpoch, ce = c % kEpoch;
      const uint32_t buf = e & 1;
      if (ce == 0) {
        if (e >= 2) tc::mbar_wait(&dempty_bar[buf], ((e - 2) >> 1) & 1);
        tc::mbar_wait(&bready_bar[buf], (e >> 1) & 1);
      }
      tc::mbar_wait(&full_bar[s], u & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t bc = b_s + buf * C::kEpochB + ce * C::kChunkB;
        const uint64_t bh = tc::make_sdesc(bc, kLBO, kSBO);
        const uint64_t bl = tc::make_sdesc(bc + C::kBBytes, kLBO, kSBO);
        const uint32_t a0 = tmem + C::kColA + 4 * kArr * s;
        const uint32_t dcos = tmem + 2 * N * buf, dsin = dcos + N;
#pragma unroll
        for (int kk = 0; kk < kChunk / 16; ++kk) {
          const uint64_t adv = uint64_t(2 * kk) * (kLBO >> 4);
          const uint32_t acc = (ce > 0 || kk > 0) ? 1u : 0u;
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dcos, a0 + kArr + 8 * kk, bh + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 2 * kArr + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dsin, a0 + 2 * kArr + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 3 * kArr + 8 * kk, bh + adv, idesc, 1u);
        }
        tc::mma_commit(&empty_bar[s]);
        if (ce == kEpoch - 1 || c == nchunks - 1) tc::mma_commit(&dfull_bar[buf]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- F staging + drains (4 warps, 128 threads) ----------
    const int fw = warp - kFWarp0, t = fw * 32 + lane;
    const uint32_t b_s = tc::smem_addr(bsm);
    const uint32_t fs_s = b_s + 2 * C::kEpochB;  // staging [E*64 points][N] fp32
    const float* fstage = reinterpret_cast<const float*>(bsm + 2 * C::kEpochB);
    const int ncol = R * dc;                     // real columns: 16 g + j, j < dc
    // the epoch's F block is copied one epoch ahead (issue_f), then maxima,
    // scales and B operands (process_f)
    auto issue_f = [&](int e) {
      const int npts = min(kEpoch, nchunks - e * kEpoch) * kChunk;
#pragma unroll 1
      for (int i = t; i < npts * ncol; i += 128) {
        const int p = i / ncol, cc = i % ncol, g = cc / dc, j = cc % dc;
        const int64_t cl = int64_t(e) * kEpoch * kChunk + p;  // point of segment g
        const int64_t pp = sc0[g] * kChunk + cl;
        const bool ok = cl < int64_t(snc[g]) * kChunk && pp < n;
        const float* src = F + (int64_t(sb[g]) * n + (ok ? pp : 0)) * d + c0 + j;
        tc::cp_async4_zf(fs_s + uint32_t((p * N + 16 * g + j) * 4), src, ok ? 4u : 0u);
      }
      tc::cp_async_commit();
    };
    auto process_f = [&](int e) {
      const int npts = min(kEpoch, nchunks - e * kEpoch) * kChunk;
      tc::cp_async_wait<0>();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      // per-column max |F| over the epoch (real columns; the rest keep scale 1)
      {
        const int cc = t % ncol, g = cc / dc, j = cc % dc, st = 128 / ncol;
        float mx = 0.0f;
        if (t < st * ncol)
          for (int p = t / ncol; p < npts; p += st) mx = fmaxf(mx, fabsf(fstage[p * N + 16 * g + j]));
        fmax_part[t] = mx;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (t < N) {
        const int g = t / 16, j = t % 16;
        float scale = 1.0f;
        if (j < dc) {
          const int cc = g * dc + j, st = 128 / ncol;
          float cm = 0.0f;
          for (int k = cc; k < st * ncol; k += ncol) cm = fmaxf(cm, fmax_part[k]);
          if (cm > 0.0f && isfinite(cm)) {
            int ex = 0;
            frexpf(cm, &ex);
            scale = ldexpf(1.0f, min(126, max(-126, 14 - ex)));
          }
        }
        fscale[t] = scale;
        fscale_inv[e & 1][t] = 1.0f / scale;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const uint32_t eb = b_s + (e & 1) * C::kEpochB;
      for (int i = t; i < ncol * (npts / 2); i += 128) {
        const int cc = i % ncol, pk = i / ncol, p = 2 * pk;
        const int col = 16 * (cc / dc) + cc % dc;
        const float sc = fscale[col];
        uint32_t hi, lo;
        tc::split_f16x2(fstage[p * N + col] * sc, fstage[(p + 1) * N + col] * sc, hi, lo);
        const int ce = p / kChunk, pc = p % kChunk;
        const uint32_t off = uint32_t(ce) * C::kChunkB + uint32_t(col >> 3) * kSBO +
                             uint32_t(pc >> 3) * kLBO + uint32_t(col & 7) * 16 + uint32_t(pc & 7) * 2;
        tc::st_shared_u32(eb + off, hi);
        tc::st_shared_u32(eb + off + C::kBBytes, lo);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bready_bar[e & 1]);
    };
#pragma unroll 1
    for (int e = 0; e < min(2, nepochs); ++e) {
      issue_f(e);
      process_f(e);
    }
    if (nepochs > 2) issue_f(2);
    // drains: lane group lg reads its segment's blocks (cos 16 g, sin N + 16 g)
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
    const uint32_t tl = tmem + lane_field + 16 * g_me;
    for (int e = 0; e < nepochs; ++e) {
      const uint32_t buf = e & 1;
      tc::mbar_wait(&dfull_bar[buf], (e >> 1) & 1);
      tc::tc_fence_after();
      float vc[16], vs[16];
      tc::tmem_ld16(tl + 2 * N * buf, vc);
      tc::tmem_ld16(tl + 2 * N * buf + N, vs);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dempty_bar[buf]);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float inv = fscale_inv[buf][16 * g_me + j];
        acc[j] = fmaf(vc[j], inv, acc[j]);
        acc[16 + j] = fmaf(vs[j], inv, acc[16 + j]);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (e + 2 < nepochs) process_f(e + 2);
      if (e + 3 < nepochs) issue_f(e + 3);
    }
    const int64_t sg = int64_t(blockIdx.x) * R + g_me;
    if (f < m && sg < nseg) {
      const int b = int(sg / ranges), rg = int(sg % ranges);
      float* out = partial + (int64_t(b) * ranges + rg) * int64_t(2 * m) * dc;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < dc) {
          out[int64_t(2 * f) * dc + j] = acc[j];
          out[int64_t(2 * f + 1) * dc + j] = acc[16 + j];
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int R>
void launch_packed(cudaStream_t s, const float* pts16, const float4* omega4, int m, int64_t n,
                   int batch, int ranges, const float* F, int d, int c0, int dc, float* partial) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(pass1_tc_packed<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PK<R>::kSmem);
    configured = true;
  }
  const int64_t ctas = (int64_t(batch) * ranges + R - 1) / R;
  launch_pdl(pass1_tc_packed<R>, dim3(unsigned(ctas)), dim3(kThreads), PK<R>::kSmem, s, pts16,
             omega4, m, n, batch, ranges, F, d, c0, dc, partial);
}

template <int NC>
void launch_nc(dim3 grid, cudaStream_t s, const float* pts16, const float4* omega4, int m,
               int64_t n, int ranges, const float* F, int d, int c0, int dc, float* partial) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(pass1_tc_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         P1<NC>::kSmem);
    configured = true;
  }
  launch_pdl(pass1_tc_kernel<NC>, grid, dim3(kThreads), P1<NC>::kSmem, s, pts16, omega4, m, n,
             ranges, F, d, c0, dc, partial);
}

}  // namespace

// RFD_P1_TRACE=1: the per-chunk timestamps of CTA (0, 0, 0), summarised.
static void print_p1trace(cudaStream_t s, int64_t n, int ranges) {
  static long long h[1024][12];
  cudaStreamSynchronize(s);
  cudaMemcpyFromSymbol(h, g_p1trace, sizeof(h));
  const int nc = int((((n + kChunk - 1) / kChunk) + ranges - 1) / ranges);
  const int lo = 16, hi = nc < 120 ? nc - 8 : 120;
  double pe = 0, pc = 0, mr = 0, mb = 0, mf = 0, per = 0;
  for (int c = lo; c < hi; ++c) {
    pe += h[c][1] - h[c][0];
    pc += h[c][2] - h[c][1];
    mr += h[c][4] - h[c][3];
    mb += h[c][5] - h[c][4];
    mf += h[c][6] - h[c][5];
    per += h[c + 1][3] - h[c][3];
  }
  const double k = hi - lo;
  fprintf(stderr,
          "p1trace chunks %d: period %.0f | prod empty-wait %.0f compute %.0f | mma "
          "dempty %.0f bready %.0f full %.0f\n",
          nc, per / k, pe / k, pc / k, mr / k, mb / k, mf / k);
  for (int c = 64; c < 84 && c < hi; ++c)
    fprintf(stderr, "  chunk %d: period %lld dempty %lld bready %lld full %lld | prod %lld %lld\n",
            c, h[c + 1][3] - h[c][3], h[c][4] - h[c][3], h[c][5] - h[c][4],
            h[c][6] - h[c][5], h[c][1] - h[c][0], h[c][2] - h[c][1]);
  for (int e = 8; e < 120 && e + 5 < hi; e += 8)
    fprintf(stderr,
            "  epoch %d: dfull wait %lld, stage_f %lld, mma at %lld..%lld | proc(e): cpwait "
            "%lld bar %lld max %lld bar %lld conv %lld bar %lld\n",
            e / 8, h[e + 3][7] - h[e + 2][7], h[e + 5][7] - h[e + 4][7],
            h[e][3] - h[e + 2][7], h[e + 8][3] - h[e + 2][7], h[e][9] - h[e][8],
            h[e][10] - h[e][9], h[e][11] - h[e][10], h[e + 1][8] - h[e][11],
            h[e + 1][9] - h[e + 1][8], h[e + 1][10] - h[e + 1][9]);
}

// Segments per CTA of the packed small-m kernel: R = 4 (m <= 32) or 2
// (m <= 64) when there are enough chunks to keep every SM busy with R of them
// (>= 2 per segment); otherwise 1 (one CTA per frequency tile and range).
int pass1_pack(int m, int64_t n, int batch, int sms) {
  const int R = m <= 32 ? 4 : (m <= 64 ? 2 : 1);
  const int64_t chunks = int64_t(batch) * ((n + kChunk - 1) / kChunk);
  return (R > 1 && chunks >= int64_t(sms) * R * 2) ? R : 1;
}

int pass1_tc_ranges(int m, int64_t n, int batch, int sms) {
  // ranges of whole chunks: about one CTA per SM (packed: R segments per CTA)
  const int ftiles = (m + 127) / 128;
  const int R = pass1_pack(m, n, batch, sms);
  int64_t ranges = (R > 1)
                       ? int64_t(sms) * R / batch
                       : (int64_t(sms) + int64_t(ftiles) * batch - 1) / (int64_t(ftiles) * batch);
  const int64_t maxr = (n + kChunk - 1) / kChunk;
  if (ranges > maxr) ranges = maxr;
  if (ranges < 1) ranges = 1;
  return int(ranges);
}

void launch_pass1_tc(const float* pts16, const float4* omega4, int m, int64_t n, int batch,
                     int sms, int ranges, const float* F, int d, int c0, int dc, float* partial,
                     cudaStream_t s) {
  LaunchScope L("rfd_pass1_tc", s);
  const dim3 grid((m + 127) / 128, ranges, batch);
  const int R = pass1_pack(m, n, batch, sms);
  if (dc <= 16 && R > 1) {  // packed segments (small m)
    if (R == 4)
      launch_packed<4>(s, pts16, omega4, m, n, batch, ranges, F, d, c0, dc, partial);
    else
      launch_packed<2>(s, pts16, omega4, m, n, batch, ranges, F, d, c0, dc, partial);
    return;
  }
  switch ((dc + 15) / 16) {
    case 1: {
      static bool configured = false;
      static bool trace = false;
      if (!configured) {
        const char* e = getenv("RFD_P1_TRACE");
        trace = e && atoi(e) == 1;
        cudaFuncSetAttribute(pass1_tc_kernel16<16, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, k16::kSmem);
        cudaFuncSetAttribute(pass1_tc_kernel16<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             k16::kSmem);
        // the whole shared-memory carveout: room for a core GEMM CTA beside
        cudaFuncSetAttribute(pass1_tc_kernel16<16>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             100);
        configured = true;
      }
      if (trace) {
        pass1_tc_kernel16<16, true><<<grid, kThreads, k16::kSmem, s>>>(pts16, omega4, m, n, ranges,
                                                                      F, d, c0, dc, partial);
        print_p1trace(s, n, ranges);
      } else {
        launch_pdl(pass1_tc_kernel16<16>, grid, dim3(kThreads), k16::kSmem, s, pts16, omega4, m, n,
                   ranges, F, d, c0, dc, partial);
      }
      break;
    }
    case 2: launch_nc<2>(grid, s, pts16, omega4, m, n, ranges, F, d, c0, dc, partial); break;
    case 3: launch_nc<3>(grid, s, pts16, omega4, m, n, ranges, F, d, c0, dc, partial); break;
    default: launch_nc<4>(grid, s, pts16, omega4, m, n, ranges, F, d, c0, dc, partial); break;
  }
}

}  // namespace rfd
