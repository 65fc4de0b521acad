// K0 -- frequency draw and importance weights.
//
// a1: omega_k ~ N(0, I_3) truncated to ||omega||_1 <= R (PAPER.md:316, 323,
//     374, 936), drawn from Philox4x32-10 with the stream layout of rfd.h.
// a2: nu_k = tau(omega_k) / (m p(omega_k)), tau(w) = prod_c sin(2 pi eps w_c)
//     / (pi w_c) (A1/A2), p = (2 pi)^{-3/2}
//     exp(-|w|^2/2) / C_R.
//
// m <= 512 frequencies: one CTA, one thread per frequency; negligible time.
#include "rfd_internal.h"

namespace rfd {
namespace {

// Philox4x32 round constants (Salmon et al., SC'11).
constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = kM0 * c.x, hi0 = __umulhi(kM0, c.x);
    const uint32_t lo1 = kM1 * c.z, hi1 = __umulhi(kM1, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += kW0;
    k.y += kW1;
  }
  return c;
}

// a2: nu_k = tau(omega_k) / (m p(omega_k)) with tau the product of the 1-D
// sinc factors sin(2 pi eps w) / (pi w) (2 eps at w = 0; reading A1) and p the
// truncated standard normal pdf (2 pi)^{-3/2} e^{-|w|^2/2} / C_R (A6, A7).
__device__ __forceinline__ double nu_of(float wx, float wy, float wz, double eps, int m,
                                        double c_r) {
  const double two_pi = 6.283185307179586;
  const double pi = 3.141592653589793;
  const double wc[3] = {double(wx), double(wy), double(wz)};
  double tau = 1.0, sq = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double w = wc[c];
    tau *= (w != 0.0) ? sin(two_pi * eps * w) / (pi * w) : 2.0 * eps;
    sq += w * w;
  }
  const double p = exp(-0.5 * sq) / (15.749609945722419 * c_r);  // (2 pi)^{3/2}
  return tau / (double(m) * p);
}

__global__ void freq_kernel(float4* __restrict__ omega4, float4* __restrict__ omega_rad4,
                            double* __restrict__ nu,
                            int* __restrict__ flags, int m, uint64_t seed,
                            double eps, double R, double c_r) {
  const uint2 key = make_uint2(uint32_t(seed & 0xffffffffu), uint32_t(seed >> 32));
  const double two_pi = 6.283185307179586;  // fl64(2 pi), as 2.0 * math.pi
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    double z0 = 0.0, z1 = 0.0, z2 = 0.0;
    bool ok = false;
    for (int a = 0; a < kMaxAttempts && !ok; ++a) {
      const uint4 w = philox10(make_uint4(uint32_t(k), uint32_t(a), kFreqTag, 0u), key);
      const double u0 = (double(w.x) + 0.5) * 0x1p-32;
      const double u1 = (double(w.y) + 0.5) * 0x1p-32;
      const double u2 = (double(w.z) + 0.5) * 0x1p-32;
      const double u3 = (double(w.w) + 0.5) * 0x1p-32;
      const double r01 = sqrt(-2.0 * log(u0));
      const double r23 = sqrt(-2.0 * log(u2));
      z0 = r01 * cos(two_pi * u1);
      z1 = r01 * sin(two_pi * u1);
      z2 = r23 * cos(two_pi * u3);
      ok = (fabs(z0) + fabs(z1) + fabs(z2)) <= R;
    }
    if (!ok) atomicOr(flags, 2);
    const float wx = float(z0), wy = float(z1), wz = float(z2);
    omega4[k] = make_float4(wx, wy, wz, 0.0f);
    // 2 pi omega rounded once from fp64: the tensor-core passes evaluate
    // sincos(2 pi omega . x) as MUFU sin/cos of (2 pi omega) . x in radians.
    omega_rad4[k] = make_float4(float(two_pi * double(wx)), float(two_pi * double(wy)),
                                float(two_pi * double(wz)), 0.0f);
    const double v = nu_of(wx, wy, wz, eps, m, c_r);
    nu[k] = v;
    if (!(v > 0.0)) atomicOr(flags, 1);
  }
}

// a2 alone, from the stored fp32 omega (re-parameterisation: nu depends on eps
// only; bit-identical to freq_kernel's nu for the same omega and eps).
__global__ void nu_kernel(const float4* __restrict__ omega4, double* __restrict__ nu,
                          int* __restrict__ flags, int m, double eps, double c_r) {
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const float4 w = omega4[k];
    const double v = nu_of(w.x, w.y, w.z, eps, m, c_r);
    nu[k] = v;
    if (!(v > 0.0)) atomicOr(flags, 1);
  }
}

// Centring (translation invariance of Eq. 9: W depends on n_i - n_j only,
// PAPER.md:288-295).  The passes evaluate the feature argument 2 pi omega.x in
// fp32, whose rounding error grows with |x|; every cloud is therefore moved to
// the midpoint c of its bounding box before anything else.  Exact for the
// operator: phi(c + y) = R(2 pi omega.c) phi(y) with R a 2x2 rotation per
// frequency, and D commutes with R, so out = F + Phi C^ Phi^T F is unchanged;
// G, C^, S and Y live in the rotated basis (rfd_plan_export rotates back).
// Min / max are order-independent, so the centre (and every result) is
// deterministic.  Ordered-integer encoding of floats: max over enc(x) is max x,
// max over ~enc(x) is min x (both start from 0 = the identity).
__device__ __forceinline__ unsigned int enc_f32(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float dec_f32(unsigned int e) {
  return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}

// One launch, two levels: every block writes its 6 encoded extrema (grid
// (chunks, batch)), and the last block of a cloud to finish (an atomic
// ticket) folds the cloud's chunks in chunk order: bbox[b][0..2] = max ~enc
// (the minima), bbox[b][3..5] = max enc (the maxima).  Loads: three float4s
// = four whole points per thread and step (no per-element component index);
// the unaligned head / ragged tail by scalar loads.  (Per-warp atomics on the
// same 6 words serialised at L2: 54 us at cfg 5; two launches with a 64-bit
// modulo per float4: 30 us.)  tickets: batch words, zero before the launch;
// the last block resets its cloud's word.
__global__ void __launch_bounds__(256)
bbox_kernel(const float* __restrict__ xyz, int64_t n, unsigned int* __restrict__ part,
            unsigned int* __restrict__ tickets, unsigned int* __restrict__ bbox) {
  __shared__ unsigned int red[8][6];
  __shared__ bool last;
  const int b = blockIdx.y;
  const float* src = xyz + int64_t(b) * n * 3;
  unsigned int v[6] = {0u, 0u, 0u, 0u, 0u, 0u};
  auto take = [&](int k, float x) {
    const unsigned int e = enc_f32(x);
    v[k] = max(v[k], ~e);
    v[3 + k] = max(v[3 + k], e);
  };
  // points [p0, p0 + 4 nq) as float4 triples when 16-byte aligned there
  const int64_t mis = (reinterpret_cast<uintptr_t>(src) >> 2) & 3;  // floats past 16 B
  const int64_t p0 = mis;  // 3 p0 + mis = 0 (mod 4): point p0 starts on 16 bytes
  const int64_t nq = n > p0 ? (n - p0) / 4 : 0;
  const float4* q4 = reinterpret_cast<const float4*>(src + 3 * p0);
  const int64_t per = (nq + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = int64_t(blockIdx.x) * per, t1 = min(t0 + per, nq);
#pragma unroll 4
  for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    const float4 a = __ldg(q4 + 3 * t), c = __ldg(q4 + 3 * t + 1), d = __ldg(q4 + 3 * t + 2);
    take(0, a.x); take(1, a.y); take(2, a.z);
    take(0, a.w); take(1, c.x); take(2, c.y);
    take(0, c.z); take(1, c.w); take(2, d.x);
    take(0, d.y); take(1, d.z); take(2, d.w);
  }
  if (blockIdx.x == 0) {  // the head points [0, p0) and the tail [p0 + 4 nq, n)
    auto take3 = [&](int64_t i) {
      take(0, __ldg(src + 3 * i));
      take(1, __ldg(src + 3 * i + 1));
      take(2, __ldg(src + 3 * i + 2));
    };
    for (int64_t i = threadIdx.x; i < min(p0, n); i += blockDim.x) take3(i);
    for (int64_t i = p0 + 4 * nq + threadIdx.x; i < n; i += blockDim.x) take3(i);
  }
#pragma unroll
  for (int c = 0; c < 6; ++c)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[c] = max(v[c], __shfl_xor_sync(0xffffffffu, v[c], o));
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int c = 0; c < 6; ++c) red[threadIdx.x >> 5][c] = v[c];
  __syncthreads();
  if (threadIdx.x < 6) {
    unsigned int mx = 0u;
    for (int w = 0; w < 8; ++w) mx = max(mx, red[w][threadIdx.x]);
    part[(int64_t(b) * gridDim.x + blockIdx.x) * 6 + threadIdx.x] = mx;
    __threadfence();  // (the threadFenceReduction pattern)
  }
  // the cloud's last block folds the chunks
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(tickets + b, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 6) {
    unsigned int mx = 0u;
    for (int k = 0; k < int(gridDim.x); ++k)
      mx = max(mx, __ldcg(part + (int64_t(b) * gridDim.x + k) * 6 + threadIdx.x));
    bbox[6 * b + threadIdx.x] = mx;
  }
  if (threadIdx.x == 0) tickets[b] = 0u;
}

__device__ __forceinline__ float4 bbox_centre(const unsigned int* bb) {
  float c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float lo = dec_f32(~bb[k]), hi = dec_f32(bb[3 + k]);
    c[k] = lo + 0.5f * (hi - lo);
  }
  return make_float4(c[0], c[1], c[2], 0.0f);
}

// Writes the centred points in all three layouts the kernels read:
//   pts    float4 (x - c, y - c, z - c, 0) per point (pass 2);
//   pts16  per cloud, groups of 16 points as [x0..x15 | y0..y15 | z0..z15]
//          (pass 1 reads a group with 12 16-byte copies and pairs neighbouring
//          points in packed FP32 math); the tail group is zero-padded (the
//          buffer is cleared first when n % 16 != 0);
//   gpts   the Gram's layout: per cloud, gper points (whole 64-point K-steps)
//          in groups of 8 as x[8] y[8] z[8] 0[8] (cleared first when padded);
//          not written when NULL (a4 through the spread grid);
// and with kCount the point's cell of a4's spread grid and its atomic rank
// inside the cell (CellCount, rfd_internal.h).
// centre[b] = c of cloud b.
// I: index type (32-bit when the batch's points fit: no 64-bit division per point)
template <typename I, bool kCount>
__global__ void pack_kernel(const float* __restrict__ xyz, const unsigned int* __restrict__ bbox,
                            float4* __restrict__ pts, float* __restrict__ pts16,
                            float* __restrict__ gpts, I gper, float4* __restrict__ centre, I n,
                            I total, const CellCount cc) {
  const I gpc = (n + 15) / 16;
  for (I i = blockIdx.x * I(blockDim.x) + threadIdx.x; i < total; i += I(gridDim.x) * blockDim.x) {
    const I b = i / n, k = i - b * n;
    const float4 c = bbox_centre(bbox + 6 * int64_t(b));
    const float x = xyz[int64_t(3) * i] - c.x, y = xyz[int64_t(3) * i + 1] - c.y,
                z = xyz[int64_t(3) * i + 2] - c.z;
    pts[i] = make_float4(x, y, z, 0.0f);
    if (k == 0) centre[b] = c;
    float* g = pts16 + (int64_t(b) * gpc + k / 16) * 48 + (k & 15);
    g[0] = x;
    g[16] = y;
    g[32] = z;
    if (gpts) {
      const int64_t gi = int64_t(b) * gper + k;
      float* h = gpts + (gi >> 3) * 32 + (gi & 7);
      h[0] = x;
      h[8] = y;
      h[16] = z;
      h[24] = 0.0f;
    }
    if (kCount) {
      const int c = grid_cell(x, y, z, cc);
      cc.cell[i] = c;
      cc.rank[i] = atomicAdd(cc.count + c, 1);
    }
  }
}

// Rotation back to the paper's (uncentred) basis for rfd_plan_export: per
// frequency k of cloud b, R_k = [[cos a, -sin a], [sin a, cos a]], a = 2 pi
// omega_k . c_b (fp64; omega and c are exact fp32 values).  Interleaved
// features (2k = cos, 2k + 1 = sin).  X is r x cols per cloud: out = R X, or
// R X R^T when `right` (cols = r).
__device__ __forceinline__ void rot_of(const float4* omega4, const float4* centre, int b, int k,
                                       double& cs, double& sn) {
  const float4 w = omega4[k], c = centre[b];
  const double t = double(w.x) * double(c.x) + double(w.y) * double(c.y) + double(w.z) * double(c.z);
  sincospi(2.0 * t, &sn, &cs);
}

__global__ void rotate_kernel(const double* __restrict__ X, const float* __restrict__ Xf, int r,
                              int cols, int batch, bool right, const float4* __restrict__ omega4,
                              const float4* __restrict__ centre, double* __restrict__ out) {
  const int64_t total = int64_t(batch) * r * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int b = int(e / (int64_t(r) * cols));
    const int rem = int(e - int64_t(b) * r * cols);
    const int a = rem / cols, c = rem - a * cols;
    const int64_t base = int64_t(b) * r * cols;
    auto at = [&](int i, int j) {
      const int64_t o = base + int64_t(i) * cols + j;
      return X ? X[o] : double(Xf[o]);
    };
    double ca, sa;
    rot_of(omega4, centre, b, a >> 1, ca, sa);
    const int a0 = a & ~1;
    // row a of R: (cos, -sin) for a cos row, (sin, cos) for a sin row
    const double ra0 = (a & 1) ? sa : ca, ra1 = (a & 1) ? ca : -sa;
    double v;
    if (!right) {
      v = ra0 * at(a0, c) + ra1 * at(a0 + 1, c);
    } else {
      double cc, sc;
      rot_of(omega4, centre, b, c >> 1, cc, sc);
      const int c0 = c & ~1;
      const double rc0 = (c & 1) ? sc : cc, rc1 = (c & 1) ? cc : -sc;
      v = ra0 * (rc0 * at(a0, c0) + rc1 * at(a0, c0 + 1)) +
          ra1 * (rc0 * at(a0 + 1, c0) + rc1 * at(a0 + 1, c0 + 1));
    }
    out[e] = v;
  }
}

}  // namespace

void launch_freq(float4* omega4, float4* omega_rad4, double* nu, int* flags, int m,
                 uint64_t seed, double eps, double R, double c_r, cudaStream_t s) {
  LaunchScope L("rfd_freq", s);
  freq_kernel<<<1, 256, 0, s>>>(omega4, omega_rad4, nu, flags, m, seed, eps, R, c_r);
}

void launch_nu(const float4* omega4, double* nu, int* flags, int m, double eps, double c_r,
               cudaStream_t s) {
  LaunchScope L("rfd_nu", s);
  nu_kernel<<<1, 256, 0, s>>>(omega4, nu, flags, m, eps, c_r);
}

int bbox_chunks(int64_t n, int batch, int sms) {
  // 2 blocks per SM (the blocks' tickets are same-address atomics: 8 per SM
  // serialised to ~12 us at cfg 5)
  int64_t chunks = (int64_t(sms) * 2 + batch - 1) / batch;
  const int64_t maxc = (n + 2047) / 2048;
  if (chunks > maxc) chunks = maxc;
  return chunks < 1 ? 1 : int(chunks);
}

void launch_bbox(const float* xyz, unsigned int* bbox, unsigned int* part, int64_t n, int batch,
                 int sms, cudaStream_t s) {
  LaunchScope L("rfd_bbox", s);
  const int chunks = bbox_chunks(n, batch, sms);
  // part: chunks * batch * 6 words, then batch ticket words (zeroed here)
  unsigned int* tickets = part + size_t(chunks) * batch * 6;
  cudaMemsetAsync(tickets, 0, size_t(batch) * sizeof(unsigned int), s);
  bbox_kernel<<<dim3(unsigned(chunks), unsigned(batch)), 256, 0, s>>>(xyz, n, part, tickets, bbox);
}

void launch_pack_points(const float* xyz, const unsigned int* bbox, float4* pts, float* pts16,
                        float* gpts, int64_t gper, float4* centre, int64_t n, int batch,
                        const CellCount* cc, cudaStream_t s) {
  LaunchScope L("rfd_pack_points", s);
  const int64_t total = n * batch;
  if (n % 16 != 0) cudaMemsetAsync(pts16, 0, size_t(batch) * ((n + 15) / 16) * 48 * sizeof(float), s);
  if (gpts && gper != n) cudaMemsetAsync(gpts, 0, size_t(batch) * gper * 4 * sizeof(float), s);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  const CellCount none{};
  if (total < (int64_t(1) << 30) && gper * batch < (int64_t(1) << 30)) {  // (i + grid stride < 2^31)
    if (cc)
      pack_kernel<int, true><<<int(blocks), 256, 0, s>>>(xyz, bbox, pts, pts16, gpts, int(gper),
                                                          centre, int(n), int(total), *cc);
    else
      pack_kernel<int, false><<<int(blocks), 256, 0, s>>>(xyz, bbox, pts, pts16, gpts, int(gper),
                                                           centre, int(n), int(total), none);
  } else {
    pack_kernel<int64_t, false><<<int(blocks), 256, 0, s>>>(xyz, bbox, pts, pts16, gpts, gper,
                                                            centre, n, total, none);
  }
}

void launch_rotate(const double* X, const float* Xf, int r, int cols, int batch, bool right,
                   const float4* omega4, const float4* centre, double* out, cudaStream_t s) {
  LaunchScope L("rfd_export_rotate", s);
  int64_t blocks = (int64_t(batch) * r * cols + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  rotate_kernel<<<unsigned(blocks), 256, 0, s>>>(X, Xf, r, cols, batch, right, omega4, centre, out);
}

}  // namespace rfd
