// NEXT-3 -- spectrum of the diffusion kernel K = exp(lambda W~), W~ = Phi D
// Phi^T (N x N, never formed), by the low-rank route (SURVEY Sec. 8(f)
// NEXT-3; "the k smallest eigenvalues of the kernel matrix",
// computed through the low-rank decomposition).
//
// The nonzero eigenvalues of Phi D Phi^T are those of G D (2m x 2m), which for
// nu > 0 is similar to the symmetric M = D^1/2 G D^1/2 (PSD).  So:
//
//   K1 tridiag_kernel   M (formed on the fly from the plan's G and nu) is
//                       reduced to tridiagonal form by Householder
//                       reflections, H_j = I - beta v v^T per column j:
//                         p = beta A v,  w = p - (beta/2)(v^T p) v,
//                         A <- A - v w^T - w v^T   (trailing block)
//                       in fp64.  The trailing block lives in an L2-resident
//                       workspace; its rows are spread over a group of g CTAs
//                       (g = 1 for r <= 128: one CTA per cloud) that meet at
//                       a group barrier twice per column (matvec -> update).
//   K2 bisect_kernel    all r eigenvalues of the tridiagonal matrix by
//                       multisection on Sturm counts (a warp per index, 32
//                       points per step).
//   K3 merge_kernel     mu -> exp(lambda mu), merged with the eigenvalue 1 of
//                       multiplicity N - r, ascending; the first k returned.
//                       For N < r the r - N eigenvalues of smallest modulus
//                       (exact zeros of G D) are dropped (A19).
//
// Deterministic: fixed row ownership, fixed-order reductions, no atomics on
// floating point.  Rows written by other CTAs of the group are read through
// L2 (ld.global.cg / st.global.cg): L1 is not coherent across SMs.
#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double dweight_s(const double* nu, int a) {
  // interleaved internal order: index 2k and 2k + 1 carry nu_k
  return nu[a >> 1];
}

// Barrier of the g CTAs of a cloud group (g > 1: all co-resident, cooperative
// launch).  Generation counter: a CTA reads the generation before arriving;
// the last arrival resets the count and advances the generation.
__device__ __forceinline__ void group_sync(unsigned int* bar, int g) {
  __syncthreads();
  if (g > 1) {
    if (threadIdx.x == 0) {
      volatile unsigned int* gen = bar + 1;
      const unsigned int my = *gen;
      __threadfence();
      if (atomicAdd(bar, 1u) == unsigned(g - 1)) {
        atomicExch(bar, 0u);
        __threadfence();
        atomicAdd(bar + 1, 1u);
      } else {
        while (*gen == my) __nanosleep(64);
      }
      __threadfence();
    }
    __syncthreads();
  }
}

// Sum over the CTA in a fixed order (warp shuffles, then warp partials).
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(kThreads)
tridiag_kernel(const double* __restrict__ G, const double* __restrict__ nu, int r, int batch,
               int g, double* __restrict__ W, double* __restrict__ P,
               double* __restrict__ diag, double* __restrict__ off, unsigned int* bar) {
  extern __shared__ double sh[];  // v[r], w[r]
  __shared__ double red[kWarps];
  double* v = sh;
  double* w = sh + r;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = (g == 1) ? 0 : int(blockIdx.x);
  const int b0 = (g == 1) ? int(blockIdx.x) : 0, b1 = (g == 1) ? b0 + 1 : batch;
  for (int b = b0; b < b1; ++b) {
    double* A = W + int64_t(b) * r * r;
    double* Pb = P + int64_t(b) * r;
    const double* Gb = G + int64_t(b) * r * r;
    // M = D^1/2 G D^1/2, rows i = cta (mod g)
    for (int i = cta + g * warp; i < r; i += g * kWarps) {
      const double si = sqrt(dweight_s(nu, i));
      for (int k = lane; k < r; k += 32)
        __stcg(A + int64_t(i) * r + k, si * Gb[int64_t(i) * r + k] * sqrt(dweight_s(nu, k)));
    }
    group_sync(bar, g);
    for (int j = 0; j + 2 < r; ++j) {
      // (a) Householder vector of column j below the diagonal (every CTA)
      double ss = 0.0;
      for (int i = j + 1 + tid; i < r; i += kThreads) {
        const double x = __ldcg(A + int64_t(i) * r + j);
        v[i] = x;
        ss += x * x;
      }
      ss = block_sum(ss, red);  // ends with __syncthreads: v visible
      const double x0 = v[j + 1];
      const double nrm = sqrt(ss);
      const double alpha = (x0 >= 0.0) ? -nrm : nrm;
      const double vtv = 2.0 * nrm * (nrm + fabs(x0));  // |x - alpha e1|^2
      const double beta = (vtv > 0.0) ? 2.0 / vtv : 0.0;
      if (cta == 0 && tid == 0) {
        diag[int64_t(b) * r + j] = __ldcg(A + int64_t(j) * r + j);
        off[int64_t(b) * r + j] = (vtv > 0.0) ? alpha : x0;
      }
      __syncthreads();
      if (tid == 0) v[j + 1] = x0 - alpha;
      __syncthreads();
      // (b) p = beta A v on the owned trailing rows
      for (int i = j + 1 + cta + g * warp; i < r; i += g * kWarps) {
        const double* Ai = A + int64_t(i) * r;
        double s = 0.0;
        for (int k = j + 1 + lane; k < r; k += 32) s += __ldcg(Ai + k) * v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) __stcg(Pb + i, beta * s);
      }
      group_sync(bar, g);
      // (c) w = p - (beta/2)(v^T p) v (every CTA)
      double vp = 0.0;
      for (int i = j + 1 + tid; i < r; i += kThreads) {
        const double pi = __ldcg(Pb + i);
        w[i] = pi;
        vp += v[i] * pi;
      }
      vp = block_sum(vp, red);
      const double K = 0.5 * beta * vp;
      for (int i = j + 1 + tid; i < r; i += kThreads) w[i] -= K * v[i];
      __syncthreads();
      // (d) A <- A - v w^T - w v^T on the owned trailing rows
      for (int i = j + 1 + cta + g * warp; i < r; i += g * kWarps) {
        double* Ai = A + int64_t(i) * r;
        const double vi = v[i], wi = w[i];
        for (int k = j + 1 + lane; k < r; k += 32) __stcg(Ai + k, __ldcg(Ai + k) - (vi * w[k] + wi * v[k]));
      }
      group_sync(bar, g);
    }
    if (cta == 0 && tid == 0) {
      if (r >= 2) {
        diag[int64_t(b) * r + r - 2] = __ldcg(A + int64_t(r - 2) * r + r - 2);
        off[int64_t(b) * r + r - 2] = __ldcg(A + int64_t(r - 1) * r + r - 2);
      }
      diag[int64_t(b) * r + r - 1] = __ldcg(A + int64_t(r - 1) * r + r - 1);
    }
    group_sync(bar, g);
  }
}

// Number of eigenvalues of the tridiagonal (d, e) below x (Sturm sequence of
// the LDL^T pivots; a zero pivot is nudged to a tiny negative-safe value).
__device__ __forceinline__ int sturm_count(const double* d, const double* e, int r, double x) {
  int cnt = 0;
  double q = d[0] - x;
  if (q < 0.0) ++cnt;
  for (int k = 1; k < r; ++k) {
    if (q == 0.0) q = 1e-300;
    q = d[k] - x - e[k - 1] * e[k - 1] / q;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// The i-th smallest eigenvalue by multisection: a warp per eigenvalue; per
// step the 32 lanes evaluate Sturm counts at 32 interior points of the
// bracket, which shrinks 33-fold (fp64 resolution in ~11 steps).
__global__ void __launch_bounds__(256)
bisect_kernel(const double* __restrict__ diag, const double* __restrict__ off, int r,
              double* __restrict__ mu) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= r) return;
  const double* d = diag + int64_t(b) * r;
  const double* e = off + int64_t(b) * r;
  // Gershgorin interval (lanes split the rows, then a max/min reduction)
  double lo = 1e300, hi = -1e300;
  for (int k = lane; k < r; k += 32) {
    const double rad = (k > 0 ? fabs(e[k - 1]) : 0.0) + (k + 1 < r ? fabs(e[k]) : 0.0);
    lo = fmin(lo, d[k] - rad);
    hi = fmax(hi, d[k] + rad);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const double span = fmax(fabs(lo), fabs(hi));
  lo -= 1e-12 * span + 1e-300;
  hi += 1e-12 * span + 1e-300;
  // invariant: count(lo) <= i < count(hi)
  for (int it = 0; it < 64; ++it) {
    const double x = lo + (hi - lo) * double(lane + 1) / 33.0;
    const bool above = (x > lo && x < hi) ? (sturm_count(d, e, r, x) > i) : (x >= hi);
    const unsigned mask = __ballot_sync(0xffffffffu, above);
    const int first = mask ? __ffs(mask) - 1 : 32;  // first point with count > i
    const double xf = __shfl_sync(0xffffffffu, x, first < 32 ? first : 31);
    const double xp = __shfl_sync(0xffffffffu, x, first > 0 ? first - 1 : 0);
    const double nlo = (first == 0) ? lo : xp;
    const double nhi = (first == 32) ? hi : xf;
    if (nlo == lo && nhi == hi) break;  // fp64 resolution reached
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) mu[int64_t(b) * r + i] = 0.5 * (lo + hi);
}

__global__ void merge_kernel(const double* __restrict__ mu, int r, int64_t n, double lambda,
                             int k, double* __restrict__ out) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  const double* m = mu + int64_t(b) * r;
  // mu ascending; for n < r drop the r - n smallest (the exact zeros of the
  // PSD matrix, smallest modulus)
  const int lo = (n < r) ? int(r - n) : 0;
  const int cnt = r - lo;
  const int64_t ones = (n > r) ? n - r : 0;
  // exp(lambda mu) ascending: mu descending for lambda < 0
  int a = 0;
  int64_t o = 0;
  for (int t = 0; t < k; ++t) {
    double val;
    if (a < cnt) {
      const int idx = (lambda < 0.0) ? (r - 1 - a) : (lo + a);
      const double ev = exp(lambda * m[idx]);
      if (o < ones && 1.0 < ev) {
        val = 1.0;
        ++o;
      } else {
        val = ev;
        ++a;
      }
    } else {
      val = 1.0;
      ++o;
    }
    out[int64_t(b) * k + t] = val;
  }
}

}  // namespace

int spectrum_group(int r) {
  int g = r / 16;
  if (g < 1) g = 1;
  if (r <= 128) g = 1;
  if (g > 64) g = 64;
  return g;
}

cudaError_t launch_spectrum(const double* G, const double* nu, int m, int batch, int64_t n,
                            double lambda, int k, double* W, double* P, double* diag,
                            double* off, double* mu, unsigned int* bar, double* out,
                            cudaStream_t s) {
  const int r = 2 * m;
  const int g = spectrum_group(r);
  const size_t smem = size_t(2) * r * sizeof(double);
  {
    LaunchScope L("rfd_spec_tridiag", s);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (g == 1) {
      tridiag_kernel<<<batch, kThreads, smem, s>>>(G, nu, r, batch, g, W, P, diag, off, bar);
    } else {
      cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned int), s);
      void* args[] = {(void*)&G, (void*)&nu, (void*)&r, (void*)&batch, (void*)&g,
                      (void*)&W, (void*)&P, (void*)&diag, (void*)&off, (void*)&bar};
      const cudaError_t e = cudaLaunchCooperativeKernel((const void*)tridiag_kernel, dim3(g),
                                                        dim3(kThreads), args, smem, s);
      if (e != cudaSuccess) return e;
    }
  }
  {
    LaunchScope L("rfd_spec_bisect", s);
    bisect_kernel<<<dim3((r + 7) / 8, batch), 256, 0, s>>>(diag, off, r, mu);
  }
  {
    LaunchScope L("rfd_spec_merge", s);
    merge_kernel<<<batch, 32, 0, s>>>(mu, r, n, lambda, k, out);
  }
  return cudaGetLastError();
}

}  // namespace rfd
