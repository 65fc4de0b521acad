// NEXT-1 -- entropic Wasserstein barycenter, Appendix D Algorithm 1
// (lines 1036-1051) with FM_K = rfd_integrate, readings as SPEC.md:559 and
// 628-629 (A20): mu reset to all-ones per outer iteration, both
// denominators (FM_K(a v^i) and d^i) clamped at 1e-30, output normalised so
// <a, mu> = 1.
//
// The iterates (v, w, d, mu) are kept in fp64, as in the oracle; only the
// kernel applications run in fp32.  FM_K is linear, so each application is fed
// a power-of-two rescaled input and the scale is undone exactly afterwards:
//
//   X = fp32(a v^i s_i),  s_i = 2^-e with max_n a v^i_n s_i in [1/2, 1)
//   FM_K(a v^i) = integrate(X)_i / s_i
//
// (the rescale only keeps fp32 in range -- w^i can reach 1e30 where the clamp
// binds -- it does not change the algorithm).  Per outer iteration:
//
//   integrate(X = a v s)                            -> Y
//   step1:  w = mu_in / max(Y / s, 1e-30)            (+ block column maxima of a w)
//   scale:  s = 2^-e(max a w);  X = fp32(a w s)
//   integrate(X)                                    -> Y
//   step2:  d = max(v Y / s, 1e-30); mu = prod_i d_i^alpha_i (mu reset to 1);
//           v = v mu / d   (+ block sums of |mu - mu_old|, block column maxima
//           of a v, non-finite flag)
//   scale:  s = 2^-e(max a v);  X = fp32(a v s)      (next iteration's input)
//
// The k distributions travel together as the k columns of an N x k field, so
// each FM_K application is ONE multi-column rfd_integrate.  Deterministic:
// fixed-order block reductions, maxima (order-independent), no floating-point
// atomics.
#include <math.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr double kClamp = 1e-30;  // SPEC.md:559 (A20)
constexpr int kBaryThreads = 256;

struct Alpha {
  double v[16];
};

// per-block column maxima (k <= 16) -> part[block * 16 + i]
__device__ __forceinline__ void block_colmax(double (&mx)[16], double* part) {
  __shared__ double red[kBaryThreads / 32][16];
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[i] = fmax(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int i = 0; i < 16; ++i) red[threadIdx.x >> 5][i] = mx[i];
  __syncthreads();
  if (threadIdx.x < 16) {
    double m = 0.0;
    for (int w = 0; w < kBaryThreads / 32; ++w) m = fmax(m, red[w][threadIdx.x]);
    part[blockIdx.x * 16 + threadIdx.x] = m;
  }
}

// V = 1, mu = 1, Mt = mu_in^T (N x k), colmax(a v) = colmax(a)
__global__ void __launch_bounds__(kBaryThreads)
bary_init_kernel(const float* __restrict__ mu_in, const float* __restrict__ area, int64_t n, int k,
                 float* __restrict__ Mt, double* __restrict__ V, double* __restrict__ mu,
                 double* __restrict__ part) {
  double mx[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) mx[i] = 0.0;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    const double a = area[p];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < k) {
        Mt[p * k + i] = mu_in[int64_t(i) * n + p];  // k x N -> N x k
        V[p * k + i] = 1.0;
        mx[i] = fmax(mx[i], a);
      }
    mu[p] = 1.0;
  }
  block_colmax(mx, part);
}

// s_i = 2^-e with max_i 2^-e in [1/2, 1) (1 for an all-zero column); flag on a
// non-finite maximum
__global__ void bary_scale_kernel(const double* __restrict__ part, int nb, int k,
                                  double* __restrict__ sc, int* __restrict__ flag) {
  const int i = threadIdx.x;
  if (i >= k) return;
  double mx = 0.0;
  for (int b = 0; b < nb; ++b) mx = fmax(mx, part[b * 16 + i]);
  double s = 1.0;
  if (!isfinite(mx)) {
    atomicOr(flag, 1);
  } else if (mx > 0.0) {
    int e = 0;
    frexp(mx, &e);  // mx = f 2^e, f in [1/2, 1)
    s = ldexp(1.0, -e);
  }
  sc[i] = s;
}

// X = fp32(a Z s) (Z = v or w, N x k fp64)
__global__ void __launch_bounds__(kBaryThreads)
bary_input_kernel(const float* __restrict__ area, const double* __restrict__ Z,
                  const double* __restrict__ sc, int64_t n, int k, float* __restrict__ X) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    const double a = area[p];
    for (int i = 0; i < k; ++i) X[p * k + i] = float(a * Z[p * k + i] * sc[i]);
  }
}

// step 1: w = mu_in / max(Y / s, clamp); block column maxima of a w
__global__ void __launch_bounds__(kBaryThreads)
bary_step1_kernel(const float* __restrict__ area, const float* __restrict__ Mt,
                  const float* __restrict__ Y, const double* __restrict__ sc, int64_t n, int k,
                  double* __restrict__ W, double* __restrict__ part) {
  double mx[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) mx[i] = 0.0;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    const double a = area[p];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < k) {
        const double w = double(Mt[p * k + i]) / fmax(double(Y[p * k + i]) / sc[i], kClamp);
        W[p * k + i] = w;
        mx[i] = fmax(mx[i], a * w);
      }
  }
  block_colmax(mx, part);
}

// step 2: d = max(v Y / s, clamp); mu = prod d^alpha; v = v mu / d;
// block sums of |mu - mu_old|, block column maxima of a v, non-finite flag
__global__ void __launch_bounds__(kBaryThreads)
bary_step2_kernel(const float* __restrict__ area, const float* __restrict__ Y, const Alpha al,
                  const double* __restrict__ sc, int64_t n, int k, double* __restrict__ V,
                  double* __restrict__ mu, double* __restrict__ dpart, double* __restrict__ part,
                  int* __restrict__ flag) {
  __shared__ double red[kBaryThreads / 32];
  double acc = 0.0, mx[16];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 16; ++i) mx[i] = 0.0;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    double d[16], lg = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < k) {
        d[i] = fmax(V[p * k + i] * (double(Y[p * k + i]) / sc[i]), kClamp);
        lg += al.v[i] * log(d[i]);
      }
    const double m = exp(lg);
    const double a = area[p];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < k) {
        const double v = V[p * k + i] * m / d[i];
        V[p * k + i] = v;
        mx[i] = fmax(mx[i], a * v);
        bad |= !isfinite(v);
      }
    bad |= !isfinite(m);
    acc += fabs(m - mu[p]);
    mu[p] = m;
  }
  if (bad) atomicOr(flag, 1);  // integer flag: order-independent
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  block_colmax(mx, part);  // (its __syncthreads also publishes red)
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kBaryThreads / 32; ++w) s += red[w];
    dpart[blockIdx.x] = s;
  }
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
bary_mass_kernel(const float* __restrict__ area, const double* __restrict__ mu, int64_t n,
                 double* __restrict__ part) {
  __shared__ double red[kBaryThreads / 32];
  double acc = 0.0;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    acc += double(area[p]) * mu[p];
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

__global__ void bary_normalize_kernel(const double* __restrict__ mu, const double* __restrict__ mass,
                                      int64_t n, float* __restrict__ out) {
  const double inv = 1.0 / mass[0];
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    out[p] = float(mu[p] * inv);
}

int blocks_for(int64_t n) {
  int64_t b = (n + kBaryThreads - 1) / kBaryThreads;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : int(b);
}

}  // namespace

int bary_blocks(int64_t n) { return blocks_for(n); }

void launch_bary_init(const float* mu_in, const float* area, int64_t n, int k, float* Mt,
                      double* V, double* mu, double* part, double* sc, int* flag, float* X,
                      cudaStream_t s) {
  const int nb = blocks_for(n);
  {
    LaunchScope L("rfd_bary_init", s);
    bary_init_kernel<<<nb, kBaryThreads, 0, s>>>(mu_in, area, n, k, Mt, V, mu, part);
  }
  launch_bary_input(area, V, part, n, k, sc, flag, X, s);
}

void launch_bary_input(const float* area, const double* Z, const double* part, int64_t n, int k,
                       double* sc, int* flag, float* X, cudaStream_t s) {
  const int nb = blocks_for(n);
  {
    LaunchScope L("rfd_bary_scale", s);
    bary_scale_kernel<<<1, 32, 0, s>>>(part, nb, k, sc, flag);
  }
  LaunchScope L("rfd_bary_input", s);
  bary_input_kernel<<<nb, kBaryThreads, 0, s>>>(area, Z, sc, n, k, X);
}

void launch_bary_step1(const float* area, const float* Mt, const float* Y, const double* sc,
                       int64_t n, int k, double* W, double* part, cudaStream_t s) {
  LaunchScope L("rfd_bary_step1", s);
  bary_step1_kernel<<<blocks_for(n), kBaryThreads, 0, s>>>(area, Mt, Y, sc, n, k, W, part);
}

void launch_bary_step2(const float* area, const float* Y, const double* alpha, const double* sc,
                       int64_t n, int k, double* V, double* mu, double* dpart, double* part,
                       double* delta, int* flag, cudaStream_t s) {
  Alpha al{};
  for (int i = 0; i < k && i < 16; ++i) al.v[i] = alpha[i];
  const int nb = blocks_for(n);
  {
    LaunchScope L("rfd_bary_step2", s);
    bary_step2_kernel<<<nb, kBaryThreads, 0, s>>>(area, Y, al, sc, n, k, V, mu, dpart, part, flag);
  }
  LaunchScope L("rfd_bary_sum", s);
  bary_sum_kernel<<<1, 1024, 0, s>>>(dpart, nb, delta);
}

void launch_bary_finish(const float* area, const double* mu, int64_t n, double* part, double* mass,
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
