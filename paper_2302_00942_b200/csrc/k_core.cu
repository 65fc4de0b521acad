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
// Dense fp64 GEMMs on the fp64 tensor cores (DMMA), batched over clouds via
// blockIdx.z.
#include <math.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kTaylor = 12;

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

__global__ void core_norm_kernel(const double* __restrict__ Z, int r,
                                 unsigned long long* __restrict__ norm_bits) {
  // ||Z_b||_1 = max column abs sum; block (32 columns x 8 row groups), the
  // max over blocks and clouds via atomicMax on the (non-negative) fp64 bits.
  const int b = blockIdx.y;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31), rg = threadIdx.x >> 5;
  const double* Zb = Z + int64_t(b) * r * r;
  double col = 0.0;
  if (c < r)
    for (int a = rg; a < r; a += 8) col += fabs(Zb[int64_t(a) * r + c]);
  __shared__ double red[8][33];
  red[rg][threadIdx.x & 31] = col;
  __syncthreads();
  if (threadIdx.x < 32) {
    double sum = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) sum += red[g][threadIdx.x];
    if (!isfinite(sum)) sum = __longlong_as_double(0x7FF0000000000000LL);  // +inf
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum = fmax(sum, __shfl_xor_sync(0xffffffffu, sum, o));
    if (threadIdx.x == 0) atomicMax(norm_bits, (unsigned long long)__double_as_longlong(sum));
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

// fp64 tensor-core GEMM (DMMA, mma.sync m8n8k4 f64): CTA tile 32 x 64,
// 4 warps side by side (each 32 x 16 = 4 x 2 fragments), K staged 16 at a
// time through shared memory (padded strides: conflict-free fragment loads).
constexpr int kBM = 32, kBN = 64, kBK = 16;
constexpr int kSA = kBK + 4;   // A tile row stride (doubles)
constexpr int kSB = kBN + 4;   // B tile row stride (doubles)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128)
dgemm_kernel(GemmJobs jobs, int njobs, int r) {
  const int jb = blockIdx.z % njobs, b = blockIdx.z / njobs;
  const GemmJob J = (jb == 0) ? jobs.job[0] : jobs.job[1];
  const int64_t off = int64_t(b) * r * r;
  const double* __restrict__ A = J.A + off;
  const double* __restrict__ B = J.B + off;
  double* __restrict__ C = J.C + off;
  __shared__ double As[kBM * kSA];
  __shared__ double Bs[kBK * kSB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = lane >> 2, tig = lane & 3;
  const int i0 = blockIdx.y * kBM, j0 = blockIdx.x * kBN;
  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  for (int k0 = 0; k0 < r; k0 += kBK) {
    // A tile 32 x 16 (4 per thread), B tile 16 x 64 (8 per thread)
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int e = tid + 128 * l, row = e >> 4, kk = e & 15;
      const int gi = i0 + row, gk = k0 + kk;
      double v = 0.0;
      if (gi < r && gk < r) v = A[int64_t(gi) * r + gk] + (gi == gk ? J.sigma : 0.0);
      As[row * kSA + kk] = v;
    }
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      const int e = tid + 128 * l, kk = e >> 6, col = e & 63;
      const int gk = k0 + kk, gj = j0 + col;
      Bs[kk * kSB + col] = (gk < r && gj < r) ? B[int64_t(gk) * r + gj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < kBK; k4 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[(mi * 8 + grp) * kSA + k4 + tig];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = Bs[(k4 + tig) * kSB + warp * 16 + ni * 8 + grp];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = i0 + mi * 8 + grp, gj = j0 + warp * 16 + ni * 8 + 2 * tig + h;
        if (gi < r && gj < r)
          C[int64_t(gi) * r + gj] = J.alpha * acc[mi][ni][h] + (gi == gj ? J.gamma : 0.0);
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
  const dim3 grid((r + kBN - 1) / kBN, (r + kBM - 1) / kBM, njobs * batch);
  dgemm_kernel<<<grid, 128, 0, s>>>(jobs, njobs, r);
}

}  // namespace

void launch_core_prep(const double* G, const double* nu, const int* flags, double lambda,
                      int m, int batch, double* Z, unsigned long long* norm_bits,
                      cudaStream_t s) {
  const int r = 2 * m;
  const int64_t rr = int64_t(r) * r;
  {
    LaunchScope L("rfd_core_prep", s);
    core_prep_kernel<<<dim3(unsigned((rr + 255) / 256), batch), 256, 0, s>>>(G, nu, flags,
                                                                             lambda, r, Z);
  }
  {
    LaunchScope L("rfd_core_norm", s);
    core_norm_kernel<<<dim3((r + 31) / 32, batch), 256, 0, s>>>(Z, r, norm_bits);
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
