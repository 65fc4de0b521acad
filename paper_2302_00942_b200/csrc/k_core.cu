// K3 -- the core C^ = lambda D phi1(lambda G D),
// the inverse-free form of [exp(L B^T A) - I](B^T A)^{-1} in Eq. 13
// (A5).  Plan-time only, fp64.
//
// Route ("core"): when every nu > 0 the core is evaluated
// on the symmetric matrix Z = lambda D^1/2 G D^1/2 (similar to lambda G D),
// C^ = lambda D^1/2 phi1(Z) D^1/2; otherwise on Z = lambda G D directly,
// C^ = lambda D phi1(Z).  phi1 and exp are evaluated by scaling and
// doubling: Z0 = Z / 2^s with ||Z0||_1 <= 2, Taylor of degree 20 of phi1
// evaluated by Paterson-Stockmeyer (P = sum_k Z0^k / (k+1)! from the powers
// Z0^2..Z0^5 and three Horner steps in Z0^5: 8 GEMMs instead of 20), E = I +
// Z0 P, then s times
//     P <- (E + I) P / 2   (phi1(2Y) = (e^Y + I) phi1(Y) / 2),   E <- E E.
// Truncation: ||Z0||^21 / 22! < 2e-15 for phi1, ||Z0||^22 / 22! < 4e-15 for exp.
// No inverse, no Cholesky: G is numerically singular in practice (SURVEY
// Sec. 0.1 item 2).  The oracle instead takes the top-right block of
// scipy's expm of the augmented 2r x 2r matrix: a different algorithm.
//
// Dense fp64 GEMMs on the fp64 tensor cores (DMMA, 64 FMA/clk/SM measured:
// tools/microbench/dmma_rate.cu), batched over clouds via blockIdx.z, with a
// 3-stage cp.async pipeline and a fused epilogue (scaled identity, sigma B and
// up to four extra matrices: the Paterson-Stockmeyer combinations).
#include <math.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kTaylor = 20;   // Taylor degree of phi1
constexpr int kPS = 5;        // Paterson-Stockmeyer block

__device__ __forceinline__ double dweight(const double* nu, int a) { return nu[a >> 1]; }

// Z_b = lambda D^1/2 G D^1/2 (symmetric route) or lambda G D, and ||Z_b||_1 =
// max column abs sum in the same pass: block (8 columns x 32 row groups, one
// cloud), the column sums reduced in shared memory in a fixed order, the max
// over blocks and clouds via atomicMax on the (non-negative) fp64 bits.
__global__ void __launch_bounds__(256)
core_prep_norm_kernel(const double* __restrict__ G, const double* __restrict__ nu,
                      const int* __restrict__ flags, double lambda, int r,
                      double* __restrict__ Z, unsigned long long* __restrict__ norm_bits) {
  const int b = blockIdx.y;
  const int cl = threadIdx.x & 7, rg = threadIdx.x >> 3;
  const int c = blockIdx.x * 8 + cl;
  const bool sym = (flags[0] & 1) == 0;
  const double* Gb = G + int64_t(b) * r * r;
  double* Zb = Z + int64_t(b) * r * r;
  double col = 0.0;
  if (c < r) {
    const double dc = dweight(nu, c), sdc = sqrt(dc);
    for (int a = rg; a < r; a += 32) {
      const int64_t e = int64_t(a) * r + c;
      const double da = dweight(nu, a);
      const double z = sym ? lambda * sqrt(da) * Gb[e] * sdc : lambda * Gb[e] * dc;
      Zb[e] = z;
      col += fabs(z);
    }
  }
  __shared__ double red[32][9];
  red[rg][cl] = col;
  __syncthreads();
  if (threadIdx.x < 8) {
    double sum = 0.0;
#pragma unroll 8
    for (int g = 0; g < 32; ++g) sum += red[g][threadIdx.x];
    if (!isfinite(sum)) sum = __longlong_as_double(0x7FF0000000000000LL);  // +inf
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) sum = fmax(sum, __shfl_xor_sync(0xffu, sum, o));
    if (threadIdx.x == 0) atomicMax(norm_bits, (unsigned long long)__double_as_longlong(sum));
  }
}

struct GemmJob {
  const double* A;  // r x r, per-batch stride r*r
  const double* B;
  double* C;
  // C = alpha (A + sigma I) B + gamma I + sum_i mc[i] M[i]
  double alpha, sigma, gamma;
  const double* M[4];
  double mc[4];
  int nm;
};
struct GemmJobs {
  GemmJob job[2];
};

// fp64 tensor-core GEMM (DMMA, mma.sync m8n8k4 f64): CTA tile 32 x 32, 4
// warps as 2 x 2 (each 16 x 16 = 2 x 2 fragments) per K group, two K groups
// splitting every K tile (partials added in group order), K in steps of 64 through a
// 3-stage cp.async pipeline (padded strides: conflict-free fragment loads);
// 105 KB of shared memory (r = 512: 256 tiles; measured per launch at r =
// 512: 21.0 us, vs 23.2 us with K steps of 32, 23.7 / 24.4 us with 128 / 64
// and 2 stages, 32 us with 32 x 64 tiles; splitting K over 8 warps, two
// accumulator sets per warp and a 4-CTA split-K cluster were slower).
// Every product of the core is a polynomial in Z, so on the symmetric route
// (Z = lambda D^1/2 G D^1/2) every result is symmetric: only the tiles on and
// above the diagonal are computed, and each writes C_ij and C_ji (i <= j).
#ifndef RFD_DGEMM_BK
#define RFD_DGEMM_BK 64
#endif
#ifndef RFD_DGEMM_STAGES
#define RFD_DGEMM_STAGES 3
#endif
#ifndef RFD_DGEMM_BM
#define RFD_DGEMM_BM 32
#endif
constexpr int kBM = RFD_DGEMM_BM, kBN = 32, kBK = RFD_DGEMM_BK, kGStages = RFD_DGEMM_STAGES;
static_assert(kBM == kBN, "the symmetric route enumerates square tiles");
#ifndef RFD_DGEMM_PDL
#define RFD_DGEMM_PDL 1  // (gfi step at cfg 5: 2.287 -> 2.279 ms)
#endif
#ifndef RFD_DGEMM_KSPLIT
#define RFD_DGEMM_KSPLIT 1  // (alone at r = 512: 18.4 / 17.6 / 19.1 us with 1 / 2 / 4; 2 groups
                            // do not fit beside pass 1: rfd_gfi 2.10 vs 2.24 ms)
#endif
constexpr int kKS = RFD_DGEMM_KSPLIT;  // warp groups splitting each K tile
constexpr int kGThreads = 64 * (kBM / 16) * kKS;  // warps of 16 x 16: (kBM / 16) x 2 per group
constexpr int kSA = kBK + 4;   // A tile row stride (doubles): 8g + 2t banks, distinct
constexpr int kSB = kBN + 4;   // B tile row stride (doubles)
constexpr int kGemmSmem = kGStages * (kBM * kSA + kBK * kSB) * 8;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 128 threads at <= 80 registers: one warp per sub-partition fits beside a
// pass-1 CTA (k_pass1_tc.cu, RFD_P1_MAXNREG), so rfd_gfi's core runs on the
// SMs beside pass 1 (uncapped, the 1-group kernel takes 96 registers)
#ifndef RFD_DGEMM_MINB
#define RFD_DGEMM_MINB (RFD_DGEMM_KSPLIT == 1 ? 6 : 1)
#endif
__global__ void __launch_bounds__(kGThreads, RFD_DGEMM_MINB)
dgemm_kernel(GemmJobs jobs, int njobs, int r, int sym) {
  extern __shared__ __align__(16) double gsm[];
  const int jb = blockIdx.z % njobs, b = blockIdx.z / njobs;
  int ti = blockIdx.y, tj = blockIdx.x;
  if (sym) {  // blockIdx.x enumerates the tiles on and above the diagonal, row by row
    const int T = (r + kBN - 1) / kBN;
    int t = blockIdx.x;
    ti = 0;
    while (t >= T - ti) t -= T - ti++;
    tj = ti + t;
  }
  const int i0 = ti * kBM, j0 = tj * kBN;
  const GemmJob& J = (jb == 0) ? jobs.job[0] : jobs.job[1];
  const int64_t off = int64_t(b) * r * r;
  const double* __restrict__ A = J.A + off;
  const double* __restrict__ B = J.B + off;
  double* __restrict__ C = J.C + off;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = lane >> 2, tig = lane & 3;
  constexpr int kWG = kBM / 16 * 2;  // warps per K group
  const int kh = warp / kWG, wq = warp % kWG;
  const int wm = (wq >> 1) * 16, wn = (wq & 1) * 16;  // the warp's 16 x 16
  double* As = gsm;                                  // [stage][kBM][kSA]
  double* Bs = gsm + kGStages * kBM * kSA;           // [stage][kBK][kSB]
#if RFD_DGEMM_PDL
  // programmatic dependent launch: the next product's CTAs may be scheduled
  // now; this one's operands are read only once the previous grid is done
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif

  auto load_tile = [&](int st, int k0) {
    // A: 32 rows x kBK doubles, B: kBK rows x 32 doubles, in 16-byte chunks
    constexpr int kAc = kBK / 2;  // chunks per A row
#pragma unroll
    for (int l = 0; l < kBM * kAc / kGThreads; ++l) {
      const int e = tid + kGThreads * l, row = e / kAc, kc = (e % kAc) * 2;
      const int gi = i0 + row, gk = k0 + kc;
      const bool ok = gi < r && gk < r;
      cp_async16(As + (st * kBM + row) * kSA + kc, ok ? A + int64_t(gi) * r + gk : A, ok);
    }
#pragma unroll
    for (int l = 0; l < kBK * 16 / kGThreads; ++l) {
      const int e = tid + kGThreads * l, kk = e >> 4, col = (e & 15) * 2;
      const int gk = k0 + kk, gj = j0 + col;
      const bool ok = gk < r && gj < r;
      cp_async16(Bs + (st * kBK + kk) * kSB + col, ok ? B + int64_t(gk) * r + gj : B, ok);
    }
  };

  double acc[2][2][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  const int nk = (r + kBK - 1) / kBK;
#pragma unroll
  for (int st = 0; st < kGStages - 1; ++st) {
    if (st < nk) load_tile(st, st * kBK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<kGStages - 2>();
    __syncthreads();
    // prefetch tile kt + 2 into the stage freed by tile kt - 1
    if (kt + kGStages - 1 < nk) load_tile((kt + kGStages - 1) % kGStages, (kt + kGStages - 1) * kBK);
    cp_async_commit();
    const double* as = As + (kt % kGStages) * kBM * kSA;
    const double* bs = Bs + (kt % kGStages) * kBK * kSB;
#pragma unroll
    for (int k4 = kh * (kBK / kKS); k4 < (kh + 1) * (kBK / kKS); k4 += 4) {
      double af[2], bf[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) af[mi] = as[(wm + mi * 8 + grp) * kSA + k4 + tig];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = bs[(k4 + tig) * kSB + wn + ni * 8 + grp];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  cp_async_wait<0>();
  if constexpr (kKS > 1) {  // the K groups' partial sums, added in group order
    __syncthreads();
    double* red = gsm + ((kh - 1) * kWG + wq) * 256 + lane;
    if (kh > 0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) red[32 * e] = acc[e >> 2][(e >> 1) & 1][e & 1];
    }
    __syncthreads();
    if (kh > 0) return;
#pragma unroll
    for (int g = 1; g < kKS; ++g)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        acc[e >> 2][(e >> 1) & 1][e & 1] += gsm[((g - 1) * kWG + wq) * 256 + lane + 32 * e];
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = i0 + wm + mi * 8 + grp, gj = j0 + wn + ni * 8 + 2 * tig + h;
        if (gi < r && gj < r && (!sym || gi <= gj)) {
          const int64_t e = int64_t(gi) * r + gj;
          double v = J.alpha * acc[mi][ni][h] + (gi == gj ? J.gamma : 0.0);
          if (J.sigma != 0.0) v += J.alpha * J.sigma * B[e];
          for (int t = 0; t < J.nm; ++t) v += J.mc[t] * J.M[t][off + e];
          C[e] = v;
          if (sym && gi != gj) C[int64_t(gj) * r + gi] = v;
        }
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

void gemm(const GemmJobs& jobs, int njobs, int r, int batch, bool sym, cudaStream_t s) {
  LaunchScope L("rfd_core_dgemm", s);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(dgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem);
    // (the whole carveout: the CTA fits beside a pass-1 CTA, rfd_gfi)
    cudaFuncSetAttribute(dgemm_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  // symmetric route: only the T (T + 1) / 2 tiles on and above the diagonal
  // are launched (launching all T^2 and returning early from the mirror ones
  // let two live CTAs share an SM while others idle: 21.1 -> 18.4 us at r = 512)
  const int T = (r + kBN - 1) / kBN;
  const dim3 grid = sym ? dim3(T * (T + 1) / 2, 1, njobs * batch)
                        : dim3((r + kBN - 1) / kBN, (r + kBM - 1) / kBM, njobs * batch);
#if RFD_DGEMM_PDL
  launch_pdl(dgemm_kernel, grid, dim3(kGThreads), kGemmSmem, s, jobs, njobs, r, sym ? 1 : 0);
#else
  dgemm_kernel<<<grid, kGThreads, kGemmSmem, s>>>(jobs, njobs, r, sym ? 1 : 0);
#endif
}

GemmJob job(const double* A, const double* B, double* C, double alpha, double sigma = 0.0,
            double gamma = 0.0) {
  GemmJob j{};
  j.A = A; j.B = B; j.C = C;
  j.alpha = alpha; j.sigma = sigma; j.gamma = gamma;
  j.nm = 0;
  return j;
}

// T = sum_i mc[i] M[i] + gamma I (elementwise; the first Horner operand)
__global__ void combo_kernel(double* __restrict__ T, const double* M0, const double* M1,
                             const double* M2, const double* M3, const double* M4, double c0,
                             double c1, double c2, double c3, double c4, double gamma, int r) {
  const int b = blockIdx.y;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= int64_t(r) * r) return;
  const int64_t o = int64_t(b) * r * r + e;
  const double t =
      c0 * M0[o] + c1 * M1[o] + c2 * M2[o] + c3 * M3[o] + ((e / r == e % r) ? gamma : 0.0);
  T[o] = t + c4 * M4[o];
}

}  // namespace

void launch_core_prep(const double* G, const double* nu, const int* flags, double lambda,
                      int m, int batch, double* Z, unsigned long long* norm_bits,
                      cudaStream_t s) {
  const int r = 2 * m;
  LaunchScope L("rfd_core_prep", s);
  core_prep_norm_kernel<<<dim3((r + 7) / 8, batch), 256, 0, s>>>(G, nu, flags, lambda, r, Z,
                                                                  norm_bits);
}

void launch_core_powers(const double* Z, int m, int batch, bool sym, double alpha, double* work,
                        cudaStream_t s) {
  const int r = 2 * m;
  const int64_t S = int64_t(r) * r * batch;
  double* Z2 = work;
  double* Z3 = work + S;
  double* Z4 = work + 2 * S;
  double* Z5 = work + 3 * S;
  // (alpha Z)^2 = a^2 Z Z; (alpha Z)^3 = a Z2 Z and (alpha Z)^4 = Z2 Z2
  // together; (alpha Z)^5 = a Z4 Z
  GemmJobs j{};
  j.job[0] = job(Z, Z, Z2, alpha * alpha);
  gemm(j, 1, r, batch, sym, s);
  j.job[0] = job(Z2, Z, Z3, alpha);
  j.job[1] = job(Z2, Z2, Z4, 1.0);
  gemm(j, 2, r, batch, sym, s);
  j.job[0] = job(Z4, Z, Z5, alpha);
  gemm(j, 1, r, batch, sym, s);
}

void launch_core_eval(const double* Z, const double* nu, const int* flags, double lambda,
                      int m, int batch, int s_scale, bool sym, double pw_alpha, double* work,
                      double* C, int* oflag, cudaStream_t s) {
  const int r = 2 * m;
  const int64_t rr = int64_t(r) * r;
  const dim3 egrid(unsigned((rr + 255) / 256), batch);
  const double alpha = ldexp(1.0, -s_scale);  // Z0 = alpha Z
  // work[0..4) holds (pw_alpha Z)^k, k = 2..5 (launch_core_powers); Z0^k =
  // q[k] (pw_alpha Z)^k with q[k] = (alpha / pw_alpha)^k, a power of two:
  // folded into the coefficients below (exact, so the result does not depend
  // on when the powers were formed)
  double q[6];
  q[0] = 1.0;
  for (int k = 1; k <= 5; ++k) q[k] = q[k - 1] * (alpha / pw_alpha);
  // Taylor coefficients of phi1: c_k = 1 / (k+1)!
  double c[kTaylor + 1];
  double f = 1.0;
  for (int k = 0; k <= kTaylor; ++k) {
    f *= double(k + 1);
    c[k] = 1.0 / f;
  }
  const int64_t S = rr * batch;  // one matrix (all clouds)
  double* Z2 = work;             // (pw_alpha Z)^2 .. (pw_alpha Z)^5
  double* Z3 = work + S;
  double* Z4 = work + 2 * S;
  double* Z5 = work + 3 * S;
  double* Ta = work + 4 * S;
  double* Tb = work + 5 * S;
  double* P = work + 6 * S;
  double* E = work + 7 * S;
  double* Pn = work + 8 * S;
  double* En = work + 9 * S;
  // B_q = sum_{i<5} c_{5q+i} Z0^i  (Z0^1 = alpha Z); Horner in Z0^5 from the top:
  // T = B_3 + c_20 Z0^5, then T <- Z0^5 T + B_q for q = 2, 1, 0.
  {  // T = B_3 + c_20 Z0^5
    LaunchScope L("rfd_core_combo", s);
    combo_kernel<<<egrid, 256, 0, s>>>(Ta, Z, Z2, Z3, Z4, Z5, c[16] * alpha, c[17] * q[2],
                                       c[18] * q[3], c[19] * q[4], c[20] * q[5], c[15], r);
  }
  double* T = Ta;
  double* Tn = Tb;
  for (int h = 2; h >= 0; --h) {
    GemmJobs j{};
    GemmJob g = job(Z5, T, h == 0 ? P : Tn, q[5], 0.0, c[kPS * h]);
    g.nm = 4;
    g.M[0] = Z; g.mc[0] = c[kPS * h + 1] * alpha;
    g.M[1] = Z2; g.mc[1] = c[kPS * h + 2] * q[2];
    g.M[2] = Z3; g.mc[2] = c[kPS * h + 3] * q[3];
    g.M[3] = Z4; g.mc[3] = c[kPS * h + 4] * q[4];
    j.job[0] = g;
    gemm(j, 1, r, batch, sym, s);
    double* t = T; T = Tn; Tn = t;
  }
  {  // E = I + Z0 P
    GemmJobs j{};
    j.job[0] = job(Z, P, E, alpha, 0.0, 1.0);
    gemm(j, 1, r, batch, sym, s);
  }
  for (int i = 0; i < s_scale; ++i) {  // P <- (E + I) P / 2 ; E <- E E (not after the last)
    GemmJobs j{};
    j.job[0] = job(E, P, Pn, 0.5, 1.0, 0.0);
    j.job[1] = job(E, E, En, 1.0, 0.0, 0.0);
    gemm(j, i + 1 < s_scale ? 2 : 1, r, batch, sym, s);
    double* t = P; P = Pn; Pn = t;
    t = E; E = En; En = t;
  }
  {
    LaunchScope L("rfd_core_finalize", s);
    core_finalize_kernel<<<egrid, 256, 0, s>>>(P, nu, flags, lambda, r, C, oflag);
  }
}

}  // namespace rfd
