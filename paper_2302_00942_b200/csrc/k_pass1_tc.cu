// K4 on the tensor cores -- pass 1, S = Phi^T F (the
// first bracket "B^T x" of Eq. 13).
//
// A CTA owns a tile of 128 frequencies (TMEM lanes) and a contiguous range of
// points (the contraction dimension K).  Per chunk of 32 points the 16
// producer warps regenerate cos and sin of omega_k . x for their lane's
// frequency (a3) and write them, split x = hi + lo in tf32, straight into
// TMEM as two A operands (cos rows, sin rows); F's chunk, split likewise, is
// the B operand in shared memory (16 channels x 32 points, K-major).  One
// elected lane issues
//     D_cos += C_hi F_hi^T + C_hi F_lo^T + C_lo F_hi^T,  D_sin likewise
// (tcgen05.mma kind::tf32, M = 128, N = 16, K = 8 x 4).  The tensor core's
// fp32 accumulator is not round-to-nearest, so D accumulates for an epoch of
// 8 chunks (256 points) in one of two TMEM buffers and 4 drain warps move it
// into fp32 registers; at the end each lane writes its frequency's 2 x 16
// partial sums.  K5 then reduces the partials in a fixed order in fp64.
#include "rfd_internal.h"
#include "tc_ptx.cuh"

namespace rfd {
namespace {

constexpr int kProducerWarps = 16;  // 4 per TMEM lane group
constexpr int kMmaWarp = 16;
constexpr int kThreads = 21 * 32;   // + MMA warp + 4 drain warps (17..20)
constexpr int kChunk = 32;          // points per chunk
constexpr int kStages = 3;
constexpr int kEpoch = 8;           // chunks per TMEM accumulation epoch
// TMEM columns: D buffers (cos 16 + sin 16) at 0 and 32; stage s at
// 64 + 128 s: [cos_hi 32 | cos_lo 32 | sin_hi 32 | sin_lo 32].
constexpr uint32_t kColA = 64;
constexpr uint32_t kLBO = 128;
constexpr uint32_t kSBO = (kChunk / 4) * 128;   // B: 8-channel groups
constexpr int kBBytes = 16 * kChunk * 4;        // one B operand (hi or lo)

__device__ __forceinline__ void sincos_rad(float4 w, float4 x, float& c, float& s) {
  // w = fp32(2 pi omega): the argument in radians; MUFU reduces it in turns.
  const float t = fmaf(w.z, x.z, fmaf(w.y, x.y, w.x * x.x));
  __sincosf(t, &s, &c);
}

__global__ void __launch_bounds__(kThreads, 1)
pass1_tc_kernel(const float4* __restrict__ pts, const float4* __restrict__ omega4, int m,
                int64_t n, int ranges, const float* __restrict__ F, int d, int c0, int dc,
                float* __restrict__ partial) {
  __shared__ __align__(1024) unsigned char bsm[kStages][2 * kBBytes];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], dfull_bar[2], dempty_bar[2];
  __shared__ uint32_t tmem_sh;
  __shared__ float4 xbuf[kProducerWarps][8];  // each producer warp's 8 points of the chunk

  const int ft = blockIdx.x, rg = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, lg = warp & 3;
  const int64_t p0 = n * rg / ranges, p1 = n * (rg + 1) / ranges;
  const int nchunks = int((p1 - p0 + kChunk - 1) / kChunk);
  const float4* cloud = pts + int64_t(b) * n;
  const float* Fb = F + int64_t(b) * n * d;

  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], kProducerWarps);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&dfull_bar[i], 1);
      tc::mbar_init(&dempty_bar[i], 4);
    }
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t lane_field = uint32_t(lg * 32) << 16;
  const int f = ft * 128 + lg * 32 + lane;  // this lane's frequency

  if (warp < kProducerWarps) {
    // ---------------- producers: 8 points per warp per chunk ---------------
    const int q = warp >> 2;  // which 8 of the chunk's 32 points
    const float4 w = (f < m) ? omega4[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    // B operand element of this lane: (channel j, point p) of each chunk;
    // F is prefetched one chunk ahead (it streams from HBM).
    const int e = warp * 32 + lane, pe = e >> 4, je = e & 15;
    const uint32_t boff = uint32_t(je >> 3) * kSBO + uint32_t(pe >> 2) * kLBO +
                          uint32_t(je & 7) * 16 + uint32_t(pe & 3) * 4;
    auto load_f = [&](int c) {
      const int64_t pp = p0 + int64_t(c) * kChunk + pe;
      return (c < nchunks && pp < p1 && je < dc) ? __ldg(Fb + pp * d + c0 + je) : 0.0f;
    };
    float f_next = load_f(0);
    // The warp's 8 points, prefetched one chunk ahead by lanes 0-7 (global
    // latency off the critical path) and handed over through shared memory.
    auto load_x = [&](int c) {
      const int64_t pp = p0 + int64_t(c) * kChunk + q * 8 + (lane & 7);
      return __ldg(cloud + (pp < p1 ? pp : p1 - 1));
    };
    float4 x_next = load_x(0);
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t s = c % kStages, u = c / kStages;
      const float fv = f_next;
      f_next = load_f(c + 1);
      if (u >= 1) tc::mbar_wait(&empty_bar[s], (u - 1) & 1);
      {
        uint32_t hi, lo;
        tc::split_tf32(fv, hi, lo);
        *reinterpret_cast<uint32_t*>(&bsm[s][boff]) = hi;
        *reinterpret_cast<uint32_t*>(&bsm[s][kBBytes + boff]) = lo;
      }
      // Points beyond the range (clamped loads) meet zero columns of F^T, and
      // lanes beyond m are never written out: no masking of the features.
      uint32_t chi[8], clo[8], shi[8], slo[8];
      if (lane < 8) xbuf[warp][lane] = x_next;
      __syncwarp();
      if (c + 1 < nchunks) x_next = load_x(c + 1);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float cs, sn;
        sincos_rad(w, xbuf[warp][j], cs, sn);
        tc::split_tf32_fast(cs, chi[j], clo[j]);
        tc::split_tf32_fast(sn, shi[j], slo[j]);
      }
      const uint32_t a = tmem + lane_field + kColA + 128 * s + 8 * q;
      tc::tmem_st8(a, chi);
      tc::tmem_st8(a + 32, clo);
      tc::tmem_st8(a + 64, shi);
      tc::tmem_st8(a + 96, slo);
      tc::tmem_st_wait();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_bar[s]);
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issue: warp-uniform loop, one elected lane -------
    const uint32_t idesc = tc::make_idesc(2, 128, 16);
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t s = c % kStages, u = c / kStages;
      const int e = c / kEpoch;
      const uint32_t buf = e & 1;
      if (c % kEpoch == 0 && e >= 2) tc::mbar_wait(&dempty_bar[buf], ((e - 2) >> 1) & 1);
      tc::mbar_wait(&full_bar[s], u & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint64_t bh = tc::make_sdesc(tc::smem_addr(&bsm[s][0]), kLBO, kSBO);
        const uint64_t bl = tc::make_sdesc(tc::smem_addr(&bsm[s][kBBytes]), kLBO, kSBO);
        const uint32_t a0 = tmem + kColA + 128 * s;
        const uint32_t dcos = tmem + 32 * buf, dsin = dcos + 16;
#pragma unroll
        for (int kk = 0; kk < kChunk / 8; ++kk) {
          const uint64_t adv = uint64_t(2 * kk) * (kLBO >> 4);
          const uint32_t acc = (c % kEpoch > 0 || kk > 0) ? 1u : 0u;
          tc::mma_tf32_ts(dcos, a0 + 8 * kk, bh + adv, idesc, acc);
          tc::mma_tf32_ts(dcos, a0 + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_tf32_ts(dcos, a0 + 32 + 8 * kk, bh + adv, idesc, 1u);
          tc::mma_tf32_ts(dsin, a0 + 64 + 8 * kk, bh + adv, idesc, acc);
          tc::mma_tf32_ts(dsin, a0 + 64 + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_tf32_ts(dsin, a0 + 96 + 8 * kk, bh + adv, idesc, 1u);
        }
        tc::mma_commit(&empty_bar[s]);
        if (c % kEpoch == kEpoch - 1 || c == nchunks - 1) tc::mma_commit(&dfull_bar[buf]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- drain warps: epochs -> fp32 registers -> partial ---
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
    const int nepochs = (nchunks + kEpoch - 1) / kEpoch;
    for (int e = 0; e < nepochs; ++e) {
      const uint32_t buf = e & 1;
      tc::mbar_wait(&dfull_bar[buf], (e >> 1) & 1);
      tc::tc_fence_after();
      float v[32];
      tc::tmem_ld32(tmem + lane_field + 32 * buf, v);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dempty_bar[buf]);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] += v[j];
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
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

int pass1_tc_ranges(int m, int64_t n, int batch, int sms) {
  const int ftiles = (m + 127) / 128;
  int64_t ranges = (int64_t(sms) + int64_t(ftiles) * batch - 1) / (int64_t(ftiles) * batch);
  const int64_t maxr = (n + kChunk - 1) / kChunk;
  if (ranges > maxr) ranges = maxr;
  if (ranges < 1) ranges = 1;
  return int(ranges);
}

void launch_pass1_tc(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                     int ranges, const float* F, int d, int c0, int dc, float* partial,
                     cudaStream_t s) {
  LaunchScope L("rfd_pass1_tc", s);
  const dim3 grid((m + 127) / 128, ranges, batch);
  pass1_tc_kernel<<<grid, kThreads, 0, s>>>(pts, omega4, m, n, ranges, F, d, c0, dc, partial);
}

}  // namespace rfd
