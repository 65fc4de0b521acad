// NEXT-1 -- entropic Wasserstein barycenter, Appendix D Algorithm 1
// (lines 1036-1051) with FM_K = rfd_integrate, readings as SPEC.md:559 and
// 628-629 (A20): mu reset to all-ones per outer iteration,
// denominators clamped (1e-20), each v^i rescaled to max 1 per iteration (mu
// and d are invariant under it; it keeps fp32 in range), output normalised so
// <a, mu> = 1.
//
// The k distributions travel together as the k columns of an N x k field, so
// each FM_K application is ONE multi-column rfd_integrate (the features are
// generated once for all k columns).  Per outer iteration:
//
//   integrate(X = a * V)                      -> Y      (= K(a v) / s_i)
//   step1:  X = a * (M / max(s Y, clamp))      (w^i, already weighted by a)
//   integrate(X)                              -> Y
//   step2:  v' = s V; d = max(v' Y, clamp); mu = prod_i d_i^alpha_i (mu reset
//           to 1); V = v' mu / d;  X = a * V   (next iteration's input)
//           + per-block sums of |mu - mu_old|, column maxima of V, and a
//           non-finite flag;  s_i = 1 / max_n V_ni
// (v' = s V is v^i rescaled to max 1; by linearity K(a v') = s K(a V).)
//
// The elementwise steps are one pass each over N x k (vectorised rows of k).
// Deterministic: fixed-order block reductions, no floating-point atomics.
#include <math.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr float kClamp = 1e-20f;  // DESIGN.md A20 (SPEC.md:559 says 1e-30: out of fp32 range once inverted twice)
constexpr int kBaryThreads = 256;

__global__ void bary_init_kernel(const float* __restrict__ mu_in, const float* __restrict__ area,
                                 int64_t n, int k, float* __restrict__ Mt, float* __restrict__ V,
                                 float* __restrict__ X, float* __restrict__ mu) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    const float a = area[p];
    for (int i = 0; i < k; ++i) {
      Mt[p * k + i] = mu_in[int64_t(i) * n + p];  // k x N -> N x k
      V[p * k + i] = 1.0f;
      X[p * k + i] = a;
    }
    mu[p] = 1.0f;
  }
}

// X = a * (M / max(s Y, clamp))
__global__ void bary_step1_kernel(const float* __restrict__ area, const float* __restrict__ Mt,
                                  const float* __restrict__ Y, const float* __restrict__ sc,
                                  int64_t n, int k, float* __restrict__ X) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    const float a = area[p];
    for (int i = 0; i < k; ++i)
      X[p * k + i] = a * (Mt[p * k + i] / fmaxf(sc[i] * Y[p * k + i], kClamp));
  }
}

struct Alpha {
  float v[16];
};

// v' = s V; d = max(v' Y, clamp); mu = prod d^alpha; V = v' mu / d; X = a V
__global__ void __launch_bounds__(kBaryThreads)
bary_step2_kernel(const float* __restrict__ area, const float* __restrict__ Y, const Alpha al,
                  const float* __restrict__ sc, int64_t n, int k, float* __restrict__ V,
                  float* __restrict__ mu, float* __restrict__ X, double* __restrict__ part,
                  float* __restrict__ vmax_part, int* __restrict__ flag) {
  __shared__ double red[kBaryThreads / 32];
  __shared__ float redm[kBaryThreads / 32][16];
  double acc = 0.0;
  bool bad = false;
  float vmx[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) vmx[i] = 0.0f;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    float d[16], vs[16];
    float lg = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < k) {
        vs[i] = sc[i] * V[p * k + i];
        d[i] = fmaxf(vs[i] * Y[p * k + i], kClamp);
        lg += al.v[i] * logf(d[i]);
      }
    }
    const float m = expf(lg);
    const float a = area[p];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < k) {
        const float v = vs[i] * m / d[i];
        V[p * k + i] = v;
        X[p * k + i] = a * v;
        vmx[i] = fmaxf(vmx[i], v);
        bad |= !isfinite(v);
      }
    }
    bad |= !isfinite(m);
    acc += fabs(double(m) - double(mu[p]));
    mu[p] = m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmx[i] = fmaxf(vmx[i], __shfl_xor_sync(0xffffffffu, vmx[i], o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = acc;
#pragma unroll
    for (int i = 0; i < 16; ++i) redm[threadIdx.x >> 5][i] = vmx[i];
  }
  if (bad) atomicOr(flag, 1);  // integer flag: order-independent
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kBaryThreads / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
  if (threadIdx.x < 16) {
    float mx = 0.0f;
    for (int w = 0; w < kBaryThreads / 32; ++w) mx = fmaxf(mx, redm[w][threadIdx.x]);
    vmax_part[blockIdx.x * 16 + threadIdx.x] = mx;
  }
}

// s_i = 1 / max over the blocks' column maxima (max is order-independent)
__global__ void bary_scale_kernel(const float* __restrict__ vmax_part, int nb, int k,
                                  float* __restrict__ sc) {
  const int i = threadIdx.x;
  if (i >= k) return;
  float mx = 0.0f;
  for (int b = 0; b < nb; ++b) mx = fmaxf(mx, vmax_part[b * 16 + i]);
  sc[i] = mx > 0.0f ? 1.0f / mx : 1.0f;
}

// out[0] = sum of part[0..nb) (fixed order)
__global__ void bary_sum_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += 1024) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    out[0] = t;
  }
}

// part[block] = sum of a * mu over the block's points
__global__ void __launch_bounds__(kBaryThreads)
bary_mass_kernel(const float* __restrict__ area, const float* __restrict__ mu, int64_t n,
                 double* __restrict__ part) {
  __shared__ double red[kBaryThreads / 32];
  double acc = 0.0;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    acc += double(area[p]) * double(mu[p]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kBaryThreads / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void bary_normalize_kernel(const float* __restrict__ mu, const double* __restrict__ mass,
                                      int64_t n, float* __restrict__ out) {
  const double inv = 1.0 / mass[0];
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    out[p] = float(double(mu[p]) * inv);
}

int blocks_for(int64_t n) {
  int64_t b = (n + kBaryThreads - 1) / kBaryThreads;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : int(b);
}

}  // namespace

int bary_blocks(int64_t n) { return blocks_for(n); }

void launch_bary_init(const float* mu_in, const float* area, int64_t n, int k, float* Mt, float* V,
                      float* X, float* mu, float* sc, cudaStream_t s) {
  LaunchScope L("rfd_bary_init", s);
  bary_init_kernel<<<blocks_for(n), kBaryThreads, 0, s>>>(mu_in, area, n, k, Mt, V, X, mu);
  const float ones[16] = {1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};
  cudaMemcpyAsync(sc, ones, sizeof(ones), cudaMemcpyHostToDevice, s);
}

void launch_bary_step1(const float* area, const float* Mt, const float* Y, const float* sc,
                       int64_t n, int k, float* X, cudaStream_t s) {
  LaunchScope L("rfd_bary_step1", s);
  bary_step1_kernel<<<blocks_for(n), kBaryThreads, 0, s>>>(area, Mt, Y, sc, n, k, X);
}

void launch_bary_step2(const float* area, const float* Y, const float* alpha, int64_t n, int k,
                       float* V, float* mu, float* X, float* sc, double* part, float* vmax_part,
                       double* delta, int* flag, cudaStream_t s) {
  Alpha al{};
  for (int i = 0; i < k && i < 16; ++i) al.v[i] = alpha[i];
  const int nb = blocks_for(n);
  {
    LaunchScope L("rfd_bary_step2", s);
    bary_step2_kernel<<<nb, kBaryThreads, 0, s>>>(area, Y, al, sc, n, k, V, mu, X, part,
                                                  vmax_part, flag);
  }
  LaunchScope L("rfd_bary_sum", s);
  bary_sum_kernel<<<1, 1024, 0, s>>>(part, nb, delta);
  bary_scale_kernel<<<1, 32, 0, s>>>(vmax_part, nb, k, sc);
}

void launch_bary_finish(const float* area, const float* mu, int64_t n, double* part, double* mass,
                        float* out, cudaStream_t s) {
  const int nb = blocks_for(n);
  {
    LaunchScope L("rfd_bary_mass", s);
    bary_mass_kernel<<<nb, kBaryThreads, 0, s>>>(area, mu, n, part);
    bary_sum_kernel<<<1, 1024, 0, s>>>(part, nb, mass);
  }
  LaunchScope L("rfd_bary_normalize", s);
  bary_normalize_kernel<<<nb, kBaryThreads, 0, s>>>(mu, mass, n, out);
}

}  // namespace rfd
