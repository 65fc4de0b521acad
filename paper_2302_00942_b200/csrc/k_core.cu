// K3 -- the core C^ = lambda D phi1(lambda G D),
// the inverse-free form of [exp(L B^T A) - I](B^T A)^{-1} in Eq. 13
// (A5).  Plan-time only, fp64.
//
// Route ("core"): when every nu > 0 the core is evaluated
// on the symmetric matrix Z = lambda D^1/2 G D^1/2 (similar to lambda G D),
// C^ = lambda D^1/2 phi1(Z) D^1/2; otherwise on Z = lambda G D directly,
// C^ = lambda D phi1(Z).  phi1 and exp are evaluated by scaling and
// doubling: Z0 = Z / 2^s with ||Z0||_1 <= 1/2, Taylor of degree 12 by Horner
// (P = sum_k Z0^k / (k+1)!, E = I + Z0 P), then s times
//     P <- (E + I) P / 2   (phi1(2Y) = (e^Y + I) phi1(Y) / 2),   E <- E E.
// No inverse, no Cholesky: G is numerically singular in practice (SURVEY
// Sec. 0.1 item 2).  The oracle instead takes the top-right block of
// scipy's expm of the augmented 2r x 2r matrix: a different algorithm.
//
// Dense fp64 GEMMs: 64 x 64 tiles, 256 threads x (4 x 4) outputs, batched
// over clouds via blockIdx.z.
#include <math.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kTaylor = 12;
constexpr double kTheta = 0.5;

__device__ __forceinline__ double dweight(const double* nu, int a) { return nu[a >> 1]; }

__global__ void core_prep_kernel(const double* __restrict__ G, const double* __restrict__ nu,
                                 const int* __restrict__ flags, double lambda, int r,
                                 double* __restrict__ Z) {
  const int b = blockIdx.y;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= int64_t(r) * r) return;
  const int a = int(e / r), c = int(e % r);
  const bool sym = (flags[0] & 1) == 0;
  const double g = G[int64_t(b) * r * r + e];
  const double da = dweight(nu, a), dc = dweight(nu, c);
  Z[int64_t(b) * r * r + e] = sym ? lambda * sqrt(da) * g * sqrt(dc) : lambda * g * dc;
}

__global__ void core_norm_kernel(const double* __restrict__ Z, int r, int* __restrict__ smax) {
  // s_b = smallest s >= 0 with ||Z_b||_1 / 2^s <= kTheta (max column abs sum).
  const int b = blockIdx.x;
  const double* Zb = Z + int64_t(b) * r * r;
  double best = 0.0;
  for (int c = threadIdx.x; c < r; c += blockDim.x) {
    double col = 0.0;
    for (int a = 0; a < r; ++a) col += fabs(Zb[int64_t(a) * r + c]);
    best = fmax(best, col);
  }
  __shared__ double red[256];
  red[threadIdx.x] = best;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double nrm = red[0];
    int s = 0;
    if (!isfinite(nrm)) s = 1 << 20;
    else
      while (ldexp(nrm, -s) > kTheta && s < 1000) ++s;
    atomicMax(smax, s);
  }
}

__global__ void scaled_identity_kernel(double* __restrict__ P, int r, double c) {
  const int b = blockIdx.y;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= int64_t(r) * r) return;
  P[int64_t(b) * r * r + e] = (e / r == e % r) ? c : 0.0;
}

struct GemmJob {
  const double* A;  // r x r, per-batch stride r*r
  const double* B;
  double* C;
  double alpha, sigma, gamma;  // C = alpha (A + sigma I) B + gamma I
};
struct GemmJobs {
  GemmJob job[2];
};

constexpr int kT = 64, kBK = 16;

__global__ void __launch_bounds__(256)
dgemm_kernel(GemmJobs jobs, int njobs, int r) {
  const int jb = blockIdx.z % njobs, b = blockIdx.z / njobs;
  const GemmJob J = (jb == 0) ? jobs.job[0] : jobs.job[1];
  const int64_t off = int64_t(b) * r * r;
  const double* __restrict__ A = J.A + off;
  const double* __restrict__ B = J.B + off;
  double* __restrict__ C = J.C + off;
  __shared__ double As[kBK][kT + 1];
  __shared__ double Bs[kBK][kT];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = blockIdx.y * kT, j0 = blockIdx.x * kT;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < r; k0 += kBK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int e = tid + 256 * l;
      const int row = e / kBK, kk = e % kBK;
      const int gi = i0 + row, gk = k0 + kk;
      double v = 0.0;
      if (gi < r && gk < r) v = A[int64_t(gi) * r + gk] + (gi == gk ? J.sigma : 0.0);
      As[kk][row] = v;
      const int kb = e / kT, col = e % kT;
      const int gkb = k0 + kb, gj = j0 + col;
      Bs[kb][col] = (gkb < r && gj < r) ? B[int64_t(gkb) * r + gj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gi = i0 + ty + 16 * i, gj = j0 + tx + 16 * j;
      if (gi < r && gj < r) C[int64_t(gi) * r + gj] = J.alpha * acc[i][j] + (gi == gj ? J.gamma : 0.0);
    }
}

__global__ void core_finalize_kernel(const double* __restrict__ P, const double* __restrict__ nu,
                                     const int* __restrict__ flags, double lambda, int r,
                                     double* __restrict__ C, int* __restrict__ oflag) {
  const int b = blockIdx.y;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= int64_t(r) * r) return;
  const int a = int(e / r), c = int(e % r);
  const bool sym = (flags[0] & 1) == 0;
  const double p = P[int64_t(b) * r * r + e];
  const double da = dweight(nu, a), dc = dweight(nu, c);
  const double v = sym ? lambda * sqrt(da) * p * sqrt(dc) : lambda * da * p;
  C[int64_t(b) * r * r + e] = v;
  if (!isfinite(v) || fabs(v) > 1e30) atomicOr(oflag, 1);
}

void gemm(const GemmJobs& jobs, int njobs, int r, int batch, cudaStream_t s) {
  LaunchScope L("rfd_core_dgemm", s);
  const int t = (r + kT - 1) / kT;
  dgemm_kernel<<<dim3(t, t, njobs * batch), 256, 0, s>>>(jobs, njobs, r);
}

}  // namespace

void launch_core_prep(const double* G, const double* nu, const int* flags, double lambda,
                      int m, int batch, double* Z, int* smax, cudaStream_t s) {
  const int r = 2 * m;
  const int64_t rr = int64_t(r) * r;
  {
    LaunchScope L("rfd_core_prep", s);
    core_prep_kernel<<<dim3(unsigned((rr + 255) / 256), batch), 256, 0, s>>>(G, nu, flags,
                                                                             lambda, r, Z);
  }
  {
    LaunchScope L("rfd_core_norm", s);
    core_norm_kernel<<<batch, 256, 0, s>>>(Z, r, smax);
  }
}

void launch_core_eval(const double* Z, const double* nu, const int* flags, double lambda,
                      int m, int batch, int s_scale, double* P0, double* P1, double* E0,
                      double* E1, double* C, int* oflag, cudaStream_t s) {
  const int r = 2 * m;
  const int64_t rr = int64_t(r) * r;
  const dim3 egrid(unsigned((rr + 255) / 256), batch);
  const double alpha = ldexp(1.0, -s_scale);
  // Taylor coefficients c_k = 1 / (k+1)!.
  double coef[kTaylor + 1];
  double f = 1.0;
  for (int k = 0; k <= kTaylor; ++k) {
    f *= double(k + 1);
    coef[k] = 1.0 / f;
  }
  {
    LaunchScope L("rfd_core_identity", s);
    scaled_identity_kernel<<<egrid, 256, 0, s>>>(P0, r, coef[kTaylor]);
  }
  double* P = P0;
  double* Pn = P1;
  for (int k = kTaylor - 1; k >= 0; --k) {  // P <- c_k I + Z0 P
    GemmJobs j{};
    j.job[0] = GemmJob{Z, P, Pn, alpha, 0.0, coef[k]};
    gemm(j, 1, r, batch, s);
    double* t = P; P = Pn; Pn = t;
  }
  {  // E = I + Z0 P
    GemmJobs j{};
    j.job[0] = GemmJob{Z, P, E0, alpha, 0.0, 1.0};
    gemm(j, 1, r, batch, s);
  }
  double* E = E0;
  double* En = E1;
  for (int i = 0; i < s_scale; ++i) {  // P <- (E + I) P / 2 ; E <- E E
    GemmJobs j{};
    j.job[0] = GemmJob{E, P, Pn, 0.5, 1.0, 0.0};
    j.job[1] = GemmJob{E, E, En, 1.0, 0.0, 0.0};
    gemm(j, 2, r, batch, s);
    double* t = P; P = Pn; Pn = t;
    t = E; E = En; En = t;
  }
  {
    LaunchScope L("rfd_core_finalize", s);
    core_finalize_kernel<<<egrid, 256, 0, s>>>(P, nu, flags, lambda, r, C, oflag);
  }
}

}  // namespace rfd
