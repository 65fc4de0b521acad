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

// pts: float4 (x, y, z, 0) per point.  pts16: per cloud, groups of 16 points
// as [x0..x15 | y0..y15 | z0..z15] (pass 1 reads a group with 12 16-byte
// copies and pairs neighbouring points in packed FP32 math); the tail group is
// zero-padded (the buffer is cleared first when n % 16 != 0).
// I: index type (32-bit when the batch's points fit: no 64-bit division per point)
template <typename I>
__global__ void pack_kernel(const float* __restrict__ xyz, float4* __restrict__ pts,
                            float* __restrict__ pts16, I n, I total) {
  const I gpc = (n + 15) / 16;
  for (I i = blockIdx.x * I(blockDim.x) + threadIdx.x; i < total; i += I(gridDim.x) * blockDim.x) {
    const float x = xyz[int64_t(3) * i], y = xyz[int64_t(3) * i + 1], z = xyz[int64_t(3) * i + 2];
    pts[i] = make_float4(x, y, z, 0.0f);
    const I b = i / n, k = i - b * n;
    float* g = pts16 + (int64_t(b) * gpc + k / 16) * 48 + (k & 15);
    g[0] = x;
    g[16] = y;
    g[32] = z;
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

void launch_pack_points(const float* xyz, float4* pts, float* pts16, int64_t n, int batch,
                        cudaStream_t s) {
  LaunchScope L("rfd_pack_points", s);
  const int64_t total = n * batch;
  if (n % 16 != 0) cudaMemsetAsync(pts16, 0, size_t(batch) * ((n + 15) / 16) * 48 * sizeof(float), s);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  if (total < (int64_t(1) << 30))  // (i + grid stride stays below 2^31)
    pack_kernel<int><<<int(blocks), 256, 0, s>>>(xyz, pts, pts16, int(n), int(total));
  else
    pack_kernel<int64_t><<<int(blocks), 256, 0, s>>>(xyz, pts, pts16, n, total);
}

}  // namespace rfd
