// K6 on the tensor cores -- pass 2, out = F + Phi Y (SURVEY Sec. 8(a) row
// a8; the "x + A(...)" of Eq. 13).
//
// Per tile of 128 points the contraction Phi_tile (128 x r) . Y (r x 16) runs
// as tcgen05.mma kind::tf32 with the A operand in TMEM: the 8 producer warps
// regenerate each point's feature row (a3: omega.x in turns, MUFU sin/cos)
// and write it, split x = hi + lo in tf32 (|x - hi - lo| <= 2^-22 |x|),
// straight into TMEM with tcgen05.st -- row = point = TMEM lane, so no
// shared-memory traffic for A.  Y^T (split likewise) sits in shared memory as
// the B operand.  Per 32-feature chunk one thread issues
//     D += A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T   (M=128, N=16, K=8 x 4)
// into a double-buffered TMEM accumulator; chunk stages are released by
// tcgen05.commit -> mbarrier, so feature generation of the next chunk
// overlaps the MMAs.  The epilogue (TMEM -> registers, + F, store) of tile t
// runs after the first chunk of tile t+1 has been produced.  Persistent CTAs
// over contiguous tile ranges; d is handled in column chunks of <= 16.
#include "rfd_internal.h"
#include "tc_ptx.cuh"

namespace rfd {
namespace {

constexpr int kProducerWarps = 16;            // 4 per TMEM lane group
constexpr int kMmaWarp = 16;
constexpr int kEpiWarp0 = 17;                 // warps 17..20: epilogue
constexpr int kThreads = 21 * 32;
constexpr int kTile = 128;      // points per tile (= TMEM lanes)
constexpr int kChunkF = 64;     // features per chunk (32 frequencies)
constexpr int kStages = 3;
constexpr uint32_t kColD = 0;   // accumulators: cols [0,16) and [16,32)
constexpr uint32_t kColA = 32;  // stage s: hi at 32 + 128 s, lo at +64
constexpr uint32_t kLBO = 128;

__device__ __forceinline__ void sincos_rad(float4 w, float4 x, float& c, float& s) {
  // w = fp32(2 pi omega): the argument in radians; MUFU reduces it in turns.
  const float t = fmaf(w.z, x.z, fmaf(w.y, x.y, w.x * x.x));
  __sincosf(t, &s, &c);
}

__global__ void __launch_bounds__(kThreads, 1)
pass2_tc_kernel(const float4* __restrict__ pts, const float4* __restrict__ omega4, int m, int64_t n,
                int batch, const float* __restrict__ Y, const float* F, float* out, int d, int c0,
                int dc) {
  // F and out may alias (in place): each epilogue thread reads F_i before
  // writing out_i.
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], dfull_bar[2], dempty_bar[2];
  __shared__ uint64_t yready_bar;
  __shared__ uint32_t tmem_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3;
  const int nch = (m + 31) / 32;       // chunks of 32 frequencies
  const int kpad = nch * kChunkF;      // padded feature count
  const uint32_t sbo = uint32_t(kpad / 4) * 128;
  unsigned char* yb = smem;                          // B hi: 16 x kpad tf32
  unsigned char* yl = smem + 16 * kpad * 4;          // B lo
  float4* om = reinterpret_cast<float4*>(smem + 2 * 16 * kpad * 4);
  const uint32_t yb_s = tc::smem_addr(yb), yl_s = tc::smem_addr(yl);

  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
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
  for (int k = tid; k < nch * 32; k += kThreads)
    om[k] = (k < m) ? omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t lane_field = uint32_t(lg * 32) << 16;
  const uint32_t idesc = tc::make_idesc(2, 128, 16);

  const int64_t tpc = (n + kTile - 1) / kTile;
  const int64_t ntiles = tpc * batch;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  const bool vec = (dc == 16) && (d % 4 == 0) && (c0 % 4 == 0);

  // Y_b^T as the B operand; the CTA's tiles are contiguous, so the cloud
  // changes rarely.  (Re)loads run under a full-CTA barrier after every MMA
  // reading the old Y has completed.
  auto load_y = [&](int b) {
    const float* Yb = Y + int64_t(b) * 2 * m * d;
    for (int e = tid; e < 16 * kpad; e += kThreads) {
      const int a = e >> 4, j = e & 15;
      const float val = (a < 2 * m && j < dc) ? Yb[int64_t(a) * d + c0 + j] : 0.0f;
      uint32_t hi, lo;
      tc::split_tf32(val, hi, lo);
      const uint32_t off = uint32_t(j >> 3) * sbo + uint32_t(a >> 2) * kLBO +
                           uint32_t(j & 7) * 16 + uint32_t(a & 3) * 4;
      *reinterpret_cast<uint32_t*>(yb + off) = hi;
      *reinterpret_cast<uint32_t*>(yl + off) = lo;
    }
    tc::fence_proxy_async_smem();
  };

  // Every role walks the same tile sequence; a cloud change is a CTA-wide
  // barrier, taken once all MMAs issued so far have completed.
  uint32_t g = 0, it = 0;
  int cur_b = -1;
  float4 x_next = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t tile = t_begin; tile < t_end; ++tile, ++it) {
    const int b = int(tile / tpc);
    const int64_t base = (tile % tpc) * kTile;
    if (b != cur_b) {
      if (g > 0) tc::mbar_wait(&empty_bar[(g - 1) % kStages], ((g - 1) / kStages) & 1);
      __syncthreads();
      load_y(b);
      __syncthreads();
      cur_b = b;
    }
    const uint32_t buf = it & 1;
    if (warp < kProducerWarps) {
      // ---------------- producers: 8 frequencies per warp per chunk --------
      const int q = warp >> 2;  // which 8 of the chunk's 32 frequencies
      // This tile's point (prefetched during the previous tile) and the next's.
      if (tile == t_begin) {
        const int64_t i0 = base + lg * 32 + lane;
        x_next = (i0 < n) ? pts[int64_t(b) * n + i0] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const float4 x = x_next;
      if (tile + 1 < t_end) {
        const int bn = int((tile + 1) / tpc);
        const int64_t in = ((tile + 1) % tpc) * kTile + lg * 32 + lane;
        x_next = (in < n) ? pts[int64_t(bn) * n + in] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int c = 0; c < nch; ++c) {
        const uint32_t gg = g + c, s = gg % kStages, u = gg / kStages;
        if (u >= 1) tc::mbar_wait(&empty_bar[s], (u - 1) & 1);
        float v[16];
        const int f0 = 32 * c + 8 * q;
        // Frequencies beyond m (zero omega) meet zero rows of Y^T: no masking.
#pragma unroll
        for (int j = 0; j < 8; ++j) sincos_rad(om[f0 + j], x, v[2 * j], v[2 * j + 1]);
        // interleaved features: 2j = cos (first output of sincos_turns), 2j+1 = sin
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          // sincos_rad(w, x, c, s) writes c then s: v[2j] = cos, v[2j+1] = sin
          tc::split_tf32_fast(v[2 * j], hi[2 * j], lo[2 * j]);
          tc::split_tf32_fast(v[2 * j + 1], hi[2 * j + 1], lo[2 * j + 1]);
        }
        const uint32_t acol = tmem + lane_field + kColA + 128 * s + 16 * q;
        tc::tmem_st16(acol, hi);
        tc::tmem_st16(acol + 64, lo);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&full_bar[s]);
      }
    } else if (warp == kMmaWarp) {
      // ---------------- MMA issue: warp-uniform loop, one elected lane -----
      if (it >= 2) tc::mbar_wait(&dempty_bar[buf], ((it - 2) >> 1) & 1);
      const uint32_t dcol = tmem + kColD + 16 * buf;
      const uint64_t bh0 = tc::make_sdesc(yb_s, kLBO, sbo);
      const uint64_t bl0 = tc::make_sdesc(yl_s, kLBO, sbo);
      for (int c = 0; c < nch; ++c) {
        const uint32_t gg = g + c, s = gg % kStages, u = gg / kStages;
        tc::mbar_wait(&full_bar[s], u & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t a0 = tmem + kColA + 128 * s;
#pragma unroll
          for (int kk = 0; kk < kChunkF / 8; ++kk) {
            // start-address field (bits 0-13, 16-byte units) advances by
            // (c * 16 + 2 kk) core matrices of 128 B
            const uint64_t adv = uint64_t(c * (kChunkF / 4) + 2 * kk) * (kLBO >> 4);
            const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
            tc::mma_tf32_ts(dcol, a0 + 8 * kk, bh0 + adv, idesc, acc);
            tc::mma_tf32_ts(dcol, a0 + 8 * kk, bl0 + adv, idesc, 1u);
            tc::mma_tf32_ts(dcol, a0 + 64 + 8 * kk, bh0 + adv, idesc, 1u);
          }
          tc::mma_commit(&empty_bar[s]);
          if (c == nch - 1) tc::mma_commit(&dfull_bar[buf]);
        }
        __syncwarp();
      }
    } else {
      // ---------------- epilogue warps: TMEM -> registers, + F, store -----
      const int64_t i = base + lg * 32 + lane;
      const int64_t idx = int64_t(b) * n + i;
      float f[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) f[j] = 0.0f;
      if (i < n) {
        const float* Fi = F + idx * d + c0;
        if (vec) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 t4 = *reinterpret_cast<const float4*>(Fi + j);
            f[j] = t4.x; f[j + 1] = t4.y; f[j + 2] = t4.z; f[j + 3] = t4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < dc) f[j] = Fi[j];
        }
      }
      tc::mbar_wait(&dfull_bar[buf], (it >> 1) & 1);
      tc::tc_fence_after();
      float v[16];
      tc::tmem_ld16(tmem + lane_field + kColD + 16 * buf, v);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dempty_bar[buf]);
      if (i < n) {
        float* Oi = out + idx * d + c0;
        if (vec) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(Oi + j) =
                make_float4(f[j] + v[j], f[j + 1] + v[j + 1], f[j + 2] + v[j + 2],
                            f[j + 3] + v[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < dc) Oi[j] = f[j] + v[j];
        }
      }
    }
    g += nch;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

size_t pass2_tc_smem(int m) {
  const int nch = (m + 31) / 32;
  return size_t(2) * 16 * nch * kChunkF * 4 + size_t(nch * 32) * sizeof(float4);
}

void launch_pass2_tc(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                     int sms, const float* Y, const float* F, float* out, int d, int c0, int dc,
                     cudaStream_t s) {
  LaunchScope L("rfd_pass2_tc", s);
  const size_t smem = pass2_tc_smem(m);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(pass2_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  const int64_t ntiles = ((n + kTile - 1) / kTile) * batch;
  int64_t grid = int64_t(sms);  // one CTA per SM (full TMEM)
  if (grid > ntiles) grid = ntiles;
  pass2_tc_kernel<<<unsigned(grid), kThreads, smem, s>>>(pts, omega4, m, n, batch, Y, F, out, d,
                                                         c0, dc);
}

}  // namespace rfd
