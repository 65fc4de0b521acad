// K4 on the tensor cores -- pass 1, S = Phi^T F (the
// first bracket "B^T x" of Eq. 13).
//
// A CTA owns a tile of 128 frequencies (TMEM lanes) and a contiguous range of
// points (the contraction dimension K).  Per chunk of 64 points the 16
// producer warps regenerate cos and sin of omega_k . x for their lane's
// frequency (a3) and write them, split x = hi + lo in fp16 (|x - hi - lo| <=
// 2^-22 |x| + 2^-25), straight into TMEM as the A operands (cos rows, sin
// rows).  F's chunk is the B operand in shared memory (16 channels x 64
// points, K-major), scaled per channel by a power of two into fp16 range
// (max_i |F_ij| 2^e_j in [2^13, 2^14); undone exactly on the partial sums)
// and split likewise.  One elected lane issues
//     D_cos += C_hi F_hi^T + C_hi F_lo^T + C_lo F_hi^T,  D_sin likewise
// (tcgen05.mma kind::f16, M = 128, N = 16, K = 16 x 4).  With N = 16 the
// instruction count paces the tensor core, and kind::f16 needs half the
// instructions of kind::tf32 per point.  The fp32 accumulator of the tensor
// core is not round-to-nearest, so D accumulates for an epoch of 8 chunks (512
// points) in one of two TMEM buffers and 4 drain warps move it into fp32
// registers; at the end each lane writes its frequency's 2 x 16 partial sums.
// K5 then reduces the partials in a fixed order in fp64.
//
// The channel scales come from a column max-|F| pre-pass (one read of F).
#include "rfd_internal.h"
#include "tc_ptx.cuh"

namespace rfd {
namespace {

constexpr int kProducerWarps = 16;  // 4 per TMEM lane group
constexpr int kMmaWarp = 16;
constexpr int kThreads = 21 * 32;   // + MMA warp + 4 drain warps (17..20)
constexpr int kChunk = 64;          // points per chunk
constexpr int kStages = 3;
constexpr int kEpoch = 8;           // chunks per TMEM accumulation epoch
// TMEM columns: D buffers (cos 16 + sin 16) at 0 and 32; stage s at
// 64 + 128 s: [cos_hi 32 | cos_lo 32 | sin_hi 32 | sin_lo 32], two fp16
// points per column.
constexpr uint32_t kColA = 64;
constexpr uint32_t kLBO = 128;
constexpr uint32_t kSBO = (kChunk / 8) * 128;   // B: 8-channel groups
constexpr int kBBytes = 16 * kChunk * 2;        // one fp16 B operand (hi or lo)

// max_i |F[i, j]| for every column j over all rows of all clouds, as fp32
// bits (atomicMax on non-negative floats orders like their bit patterns: the
// result is order-independent).  F is read once as float4s: with a grid
// stride that is a multiple of d/4 (d % 4 == 0) each thread stays on the same
// 4 columns; otherwise element-wise.
constexpr int kColmaxThreads = 256;
__global__ void __launch_bounds__(kColmaxThreads)
colmax_kernel(const float* __restrict__ F, int64_t rows, int d, unsigned int* __restrict__ maxbits) {
  extern __shared__ unsigned int smax[];  // d
  for (int j = threadIdx.x; j < d; j += blockDim.x) smax[j] = 0u;
  __syncthreads();
  const int64_t total = rows * d;
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if ((d & 3) == 0) {
    const int q = d >> 2;                        // float4s per row
    const int64_t stride = (nthreads / q) * q;   // keeps (k mod q) fixed per thread
    const int64_t n4 = total >> 2;
    float4 mx = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < stride) {
      const float4* F4 = reinterpret_cast<const float4*>(F);
      int64_t k = t;
      for (; k + 3 * stride < n4; k += 4 * stride) {  // 4 loads in flight
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(F4 + k + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          mx.x = fmaxf(mx.x, fabsf(v[u].x));
          mx.y = fmaxf(mx.y, fabsf(v[u].y));
          mx.z = fmaxf(mx.z, fabsf(v[u].z));
          mx.w = fmaxf(mx.w, fabsf(v[u].w));
        }
      }
      for (; k < n4; k += stride) {
        const float4 v = __ldg(F4 + k);
        mx.x = fmaxf(mx.x, fabsf(v.x));
        mx.y = fmaxf(mx.y, fabsf(v.y));
        mx.z = fmaxf(mx.z, fabsf(v.z));
        mx.w = fmaxf(mx.w, fabsf(v.w));
      }
      const int j = int(t % q) * 4;
      if (mx.x > 0.f) atomicMax(smax + j, __float_as_uint(mx.x));
      if (mx.y > 0.f) atomicMax(smax + j + 1, __float_as_uint(mx.y));
      if (mx.z > 0.f) atomicMax(smax + j + 2, __float_as_uint(mx.z));
      if (mx.w > 0.f) atomicMax(smax + j + 3, __float_as_uint(mx.w));
    }
  } else {
    for (int64_t k = t; k < total; k += nthreads) {
      const float v = fabsf(__ldg(F + k));
      if (v > 0.f) atomicMax(smax + int(k % d), __float_as_uint(v));
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x)
    if (smax[j]) atomicMax(maxbits + j, smax[j]);
}

__global__ void __launch_bounds__(kThreads, 1)
pass1_tc_kernel(const float* __restrict__ pts16, const float4* __restrict__ omega4, int m,
                int64_t n, int ranges, const float* __restrict__ F, int d, int c0, int dc,
                const unsigned int* __restrict__ maxbits, float* __restrict__ partial) {
  __shared__ __align__(1024) unsigned char bsm[kStages][2 * kBBytes];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], dfull_bar[2], dempty_bar[2];
  __shared__ uint32_t tmem_sh;
  // each producer warp's 16 points of a chunk as [x0..15 | y0..15 | z0..15],
  // 3 chunks deep (cp.async ring)
  __shared__ __align__(16) float xbuf[3][kProducerWarps][48];
  __shared__ float fscale[16], fscale_inv[16];

  const int ft = blockIdx.x, rg = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, lg = warp & 3;
  // ranges are whole chunks; only a cloud's last chunk is partial
  const int64_t cpc = (n + kChunk - 1) / kChunk, gpc = (n + 15) / 16;
  const int64_t ch0 = cpc * rg / ranges, ch1 = cpc * (rg + 1) / ranges;
  const int64_t p0 = ch0 * kChunk;
  const int nchunks = int(ch1 - ch0);
  const float* cloud16 = pts16 + int64_t(b) * gpc * 48;
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
  if (tid >= 32 && tid < 48) {
    // channel scale 2^e_j with max |F_j| 2^e_j in [2^13, 2^14) (1 for a zero
    // or non-finite channel)
    const int j = tid - 32;
    const float mx = (j < dc) ? __uint_as_float(maxbits[c0 + j]) : 0.0f;
    float scale = 1.0f;
    if (mx > 0.0f && isfinite(mx)) {
      int ex = 0;
      frexpf(mx, &ex);  // mx in [2^(ex-1), 2^ex)
      scale = ldexpf(1.0f, min(126, max(-126, 14 - ex)));  // 2^+-126: normal, exact inverse
    }
    fscale[j] = scale;
    fscale_inv[j] = 1.0f / scale;  // exact: a power of two
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t lane_field = uint32_t(lg * 32) << 16;
  const int f = ft * 128 + lg * 32 + lane;  // this lane's frequency

  if (warp < kProducerWarps) {
    // ---------------- producers: 16 points per warp per chunk --------------
    const int q = warp >> 2;  // which 16 of the chunk's 64 points
    const float4 w = (f < m) ? omega4[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float2 wx = make_float2(w.x, w.x), wy = make_float2(w.y, w.y), wz = make_float2(w.z, w.z);
    // B operand elements of this lane: channel je of points 2 pe, 2 pe + 1 of
    // each chunk (one 32-bit word of the K-major core matrix); F is prefetched
    // one chunk ahead (it streams from HBM).  Pointers and counters advance
    // per chunk (no 64-bit index arithmetic in the loop).
    const int e = warp * 32 + lane, je = e & 15, pe = e >> 4;
    const uint32_t boff = uint32_t(je >> 3) * kSBO + uint32_t(pe >> 2) * kLBO +
                          uint32_t(je & 7) * 16 + uint32_t(pe & 3) * 4;
    const uint32_t b_s = tc::smem_addr(&bsm[0][0]) + boff;
    const float sc = fscale[je];
    const bool jok = je < dc;
    const float* fptr = Fb + (p0 + 2 * pe) * d + c0 + je;
    const int64_t fstep = int64_t(kChunk) * d;
    const int64_t frem0 = n - (p0 + 2 * pe);
    int frem = int(frem0 > 0x7fffffff ? 0x7fffffff : frem0);  // points left from the first
    auto load_f = [&]() {
      float2 v = make_float2(0.f, 0.f);
      if (jok && frem > 0) {
        v.x = __ldg(fptr);
        if (frem > 1) v.y = __ldg(fptr + d);
      }
      fptr += fstep;
      frem -= kChunk;
      return v;
    };
    float2 f_next = load_f();
    // The warp's 16 points (one SoA group, 192 B), copied two chunks ahead by
    // lanes 0-11 straight into shared memory (cp.async: global latency off the
    // critical path).  Groups past the cloud's end repeat its last group
    // (finite values that meet zero F).
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
      const float2 fv = f_next;
      f_next = load_f();
      load_x(c + 2 < nchunks);  // the slot chunk c - 1 read (ordered by its __syncwarp)
      if (u >= 1) tc::mbar_wait(empty_s + 8 * s, (u - 1) & 1);
      {
        uint32_t hi, lo;
        tc::split_f16x2(fv.x * sc, fv.y * sc, hi, lo);
        tc::st_shared_u32(b_s + s * (2 * kBBytes), hi);
        tc::st_shared_u32(b_s + s * (2 * kBBytes) + kBBytes, lo);
      }
      // Points beyond the cloud meet zero columns of F^T, and lanes beyond m
      // are never written out: no masking of the features.
      tc::cp_async_wait<2>();  // chunk c's group (c + 1, c + 2 may be in flight)
      __syncwarp();
      const float* xs = &xbuf[0][warp][0] + xr * (kProducerWarps * 48);
      xr = (xr == 2) ? 0 : xr + 1;
      const uint32_t a = tmem + lane_field + kColA + 128 * s + 8 * q;
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
        tc::tmem_st4(ah + 32, clo[0], clo[1], clo[2], clo[3]);
        tc::tmem_st4(ah + 64, shi[0], shi[1], shi[2], shi[3]);
        tc::tmem_st4(ah + 96, slo[0], slo[1], slo[2], slo[3]);
      }
      tc::tmem_st_wait();
      tc::fence_proxy_async_smem();
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
    const uint32_t idesc = tc::make_idesc(0, 128, 16);
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
        for (int kk = 0; kk < kChunk / 16; ++kk) {
          const uint64_t adv = uint64_t(2 * kk) * (kLBO >> 4);
          const uint32_t acc = (c % kEpoch > 0 || kk > 0) ? 1u : 0u;
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dcos, a0 + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dcos, a0 + 32 + 8 * kk, bh + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 64 + 8 * kk, bh + adv, idesc, acc);
          tc::mma_f16_ts(dsin, a0 + 64 + 8 * kk, bl + adv, idesc, 1u);
          tc::mma_f16_ts(dsin, a0 + 96 + 8 * kk, bh + adv, idesc, 1u);
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
          out[int64_t(2 * f) * dc + j] = acc[j] * fscale_inv[j];
          out[int64_t(2 * f + 1) * dc + j] = acc[16 + j] * fscale_inv[j];
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
  // ranges of whole chunks: about one CTA per SM
  const int ftiles = (m + 127) / 128;
  int64_t ranges = (int64_t(sms) + int64_t(ftiles) * batch - 1) / (int64_t(ftiles) * batch);
  const int64_t maxr = (n + kChunk - 1) / kChunk;
  if (ranges > maxr) ranges = maxr;
  if (ranges < 1) ranges = 1;
  return int(ranges);
}

void launch_colmax(const float* F, int64_t rows, int d, unsigned int* maxbits, cudaStream_t s) {
  LaunchScope L("rfd_colmax", s);
  cudaMemsetAsync(maxbits, 0, size_t(d) * sizeof(unsigned int), s);
  const size_t smem = size_t(d) * sizeof(unsigned int);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(colmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int64_t blocks = (rows * d / 4 + kColmaxThreads - 1) / kColmaxThreads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  colmax_kernel<<<int(blocks), kColmaxThreads, smem, s>>>(F, rows, d, maxbits);
}

void launch_pass1_tc(const float* pts16, const float4* omega4, int m, int64_t n, int batch,
                     int ranges, const float* F, int d, int c0, int dc,
                     const unsigned int* maxbits, float* partial, cudaStream_t s) {
  LaunchScope L("rfd_pass1_tc", s);
  const dim3 grid((m + 127) / 128, ranges, batch);
  pass1_tc_kernel<<<grid, kThreads, 0, s>>>(pts16, omega4, m, n, ranges, F, d, c0, dc, maxbits,
                                           partial);
}

}  // namespace rfd
