// NEXT-1 fused -- the whole of Alg. 1 (Appendix D;
// readings A20: mu reset per iteration, both denominators clamped at 1e-30,
// tol stop on ||mu_new - mu_old||_1, <a, mu> = 1) in ONE persistent
// cooperative launch, for the paper's barycenter regime (m <= 32 random
// features -- the paper uses m = 30, PAPER.md:1061 -- k <= 4 distributions,
// N up to 148 x 512 points: the 5k-19k-node meshes of Table 2).
//
// Every FM_K application of Alg. 1 (two per iteration) is Eq. 13's
// out = X + Phi C^ Phi^T X.  The feature rows phi(x_p) do not change between
// applications, so each CTA computes the rows of its 512 points ONCE (the
// only sin/cos of the whole run) and keeps them in shared memory (fp32,
// 2 m x 512 = 128 KB at m = 32; never in HBM); each application is then two
// contractions against the cached rows:
//
//   sweep:  out_p = Z_p + sum_k [cos_kp Yc_k + sin_kp Ys_k]      (pass 2 of
//           the previous application) -> the elementwise update of Alg. 1 ->
//           the next input Z'_p -> S' partial += phi_p Z'_p      (pass 1 of
//           the next application), all on the same cached rows, per point
//   ONE grid barrier; every CTA adds the CTA partials in CTA order (fp64)
//   and forms Y' = C^ S' in its shared memory
//
// Point-stationary throughout (thread = 2 points); the S partials are
// reduced over the CTA by warp shuffles in a fixed pattern and the warps in
// order: deterministic.  Everything after the fp32 feature rows is fp64 --
// the iterates v, w, d, mu, the inputs Z = a v, a w and both contractions --
// so no input rescaling (and no barrier for it) is needed where the clamp
// lets w grow by 1e30 per iteration; a non-finite value is ERANGE.
#include <math.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kThreads = 256;
constexpr int kPts = 512;  // points per CTA (2 per thread)
constexpr double kClamp = 1e-30;  // SPEC.md:559 (A20)

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Generation barrier (grid <= 148 CTAs: one counter); self-resetting.
__device__ __forceinline__ void grid_sync(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int my = ld_acquire(bar);
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar + 1) : "memory");
    if (old == gridDim.x - 1) {
      bar[1] = 0u;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    } else {
      unsigned int v;
      do {
        __nanosleep(20);
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      } while (v == my);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  __syncthreads();
}

struct BaryArgs {
  const float4* pts;     // n centred points (plan layout)
  const float4* omega4;  // m: fp32(2 pi omega)
  const double* C;       // r x r (interleaved)
  const float* mu_in;    // k x n
  const float* area;     // n
  Alpha16 alpha;
  int m, k;
  int64_t n;
  int max_iter;
  double tol;
  double* part;          // 2 x gridDim x (r x k) CTA partials (fp64, alternating)
  double* S;             // r x k
  double* red;           // 3 x gridDim: two alternating delta buffers, mass partials
  unsigned int* bar;     // 2 words (generation, count)
  int* status;           // [0] non-finite flag, [1] iterations run
  float* out;            // n
};

template <int K>
__global__ void __launch_bounds__(kThreads, 1) bary_fused_kernel(const BaryArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = a.m, r = 2 * m;
  const int G = int(gridDim.x);
  float* feat = sm;                                                 // [m][2][kPts]
  double* ys = reinterpret_cast<double*>(feat + m * 2 * kPts + 2);  // [r][K] Y (fp64)
  double* ss = ys + r * K;                                          // [r][K] S (fp64)
  double* wpart = ss + r * K;                                       // [8][r][K] warp partials
  double* yq = wpart + 8 * r * K;                                   // [4][r][K] Y quarters
  __shared__ double redw[8][2];
  __shared__ double bcast[2];

  const int64_t pbase = int64_t(blockIdx.x) * kPts;
  const int64_t ip[2] = {pbase + tid, pbase + tid + kThreads};
  bool ok[2];
  double ar[2];
  // ---- the CTA's feature rows: the only sin/cos of the run (a3)
  {
    float4 x[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      ok[q] = ip[q] < a.n;
      x[q] = ok[q] ? __ldg(a.pts + ip[q]) : make_float4(0.f, 0.f, 0.f, 0.f);
      ar[q] = ok[q] ? double(__ldg(a.area + ip[q])) : 0.0;
    }
    for (int kk = 0; kk < m; ++kk) {
      const float4 w = __ldg(a.omega4 + kk);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float t = fmaf(w.z, x[q].z, fmaf(w.y, x[q].y, w.x * x[q].x));
        float sn, c;
        __sincosf(t, &sn, &c);
        feat[(kk * 2 + 0) * kPts + tid + q * kThreads] = ok[q] ? c : 0.0f;
        feat[(kk * 2 + 1) * kPts + tid + q * kThreads] = ok[q] ? sn : 0.0f;
      }
    }
  }
  // per-point state: fp64 iterates; Z = the current FM_K input (a v or a w)
  double v[2][K], mu[2], Z[2][K];
  float mui[2][K];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    mu[q] = 1.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      v[q][i] = 1.0;
      mui[q][i] = (ok[q] && i < a.k) ? __ldg(a.mu_in + int64_t(i) * a.n + ip[q]) : 0.0f;
      Z[q][i] = (ok[q] && i < a.k) ? ar[q] : 0.0;  // a v, v = 1
    }
  }
  __syncthreads();

  // S = Phi^T Z on the cached rows (the products in fp64: no rescaling is
  // needed to keep the iterates in range), then Y = C^ S, in every CTA:
  // CTA partial (warp butterflies in a fixed pattern, warps in order) ->
  // ONE grid barrier -> every CTA adds all CTA partials in CTA order itself.
  // The partial buffers alternate between calls (a CTA can be one call ahead
  // of a CTA still reading the previous partials, never two).
  int call = 0;
  auto apply_S = [&]() {
    double* part = a.part + int64_t(call & 1) * G * r * K;
    for (int k4 = 0; k4 < m; k4 += 4) {
      double acc[4][2][K];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k4 + u;
        double c0 = 0.0, s0 = 0.0, c1 = 0.0, s1 = 0.0;
        if (kk < m) {
          c0 = feat[(kk * 2) * kPts + tid];
          s0 = feat[(kk * 2 + 1) * kPts + tid];
          c1 = feat[(kk * 2) * kPts + tid + kThreads];
          s1 = feat[(kk * 2 + 1) * kPts + tid + kThreads];
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
          acc[u][0][i] = fma(c1, Z[1][i], c0 * Z[0][i]);
          acc[u][1][i] = fma(s1, Z[1][i], s0 * Z[0][i]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int i = 0; i < K; ++i) {
            double x = acc[u][t][i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0 && k4 + u < m) wpart[(warp * r + 2 * (k4 + u) + t) * K + i] = x;
          }
    }
    __syncthreads();
    for (int e = tid; e < r * K; e += kThreads) {
      double sum = 0.0;
#pragma unroll
      for (int w8 = 0; w8 < 8; ++w8) sum += wpart[w8 * r * K + e];
      part[int64_t(blockIdx.x) * r * K + e] = sum;
    }
    grid_sync(a.bar);
    for (int e = tid; e < r * K; e += kThreads) {
      double sum = 0.0;
      for (int c = 0; c < G; ++c) sum += part[int64_t(c) * r * K + e];
      ss[e] = sum;
    }
    __syncthreads();
    // Y = C^ S: thread (row, quarter) sums a quarter of the columns, the
    // quarters added in order
    const int qw = (r + 3) / 4;
    for (int e = tid; e < 4 * r; e += kThreads) {
      const int row = e % r, qq = e / r;
      const int cb = qq * qw, ce = min(r, cb + qw);
      double acc[K];
#pragma unroll
      for (int i = 0; i < K; ++i) acc[i] = 0.0;
#pragma unroll 8
      for (int cc = cb; cc < ce; ++cc) {
        const double cv = __ldg(a.C + int64_t(row) * r + cc);
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = fma(cv, ss[cc * K + i], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < K; ++i) yq[(qq * r + row) * K + i] = acc[i];
    }
    __syncthreads();
    for (int e = tid; e < r * K; e += kThreads)
      ys[e] = ((yq[e] + yq[r * K + e]) + yq[2 * r * K + e]) + yq[3 * r * K + e];
    __syncthreads();
    ++call;
  };
  // out = Z + Phi Y on the cached rows (fp64 accumulation)
  auto apply_out = [&](double (&o)[2][K]) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < K; ++i) o[q][i] = Z[q][i];
    for (int kk = 0; kk < m; ++kk) {
      const double c0 = feat[(kk * 2) * kPts + tid], s0 = feat[(kk * 2 + 1) * kPts + tid];
      const double c1 = feat[(kk * 2) * kPts + tid + kThreads];
      const double s1 = feat[(kk * 2 + 1) * kPts + tid + kThreads];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const double yc = ys[(2 * kk) * K + i], yn = ys[(2 * kk + 1) * K + i];
        o[0][i] = fma(c0, yc, fma(s0, yn, o[0][i]));
        o[1][i] = fma(c1, yc, fma(s1, yn, o[1][i]));
      }
    }
  };

  apply_S();  // S = Phi^T (a v), v = 1
  int it = 0;
  bool bad = false;
  for (it = 1; it <= a.max_iter; ++it) {
    double o[2][K];
    // 1. w^i = mu^i / FM_K(a v^i); the next input a w^i
    apply_out(o);
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const double w = double(mui[q][i]) / fmax(o[q][i], kClamp);
        Z[q][i] = (ok[q] && i < a.k) ? ar[q] * w : 0.0;
        bad |= !isfinite(Z[q][i]);
      }
    apply_S();
    // 2. d^i = v^i FM_K(a w^i); 3. mu = prod_i (d^i)^alpha_i; 4. v^i = v^i mu / d^i;
    // the next input a v^i
    apply_out(o);
    double dl = 0.0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!ok[q]) continue;
      double dd[K], lg = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i < a.k) {
          dd[i] = fmax(v[q][i] * o[q][i], kClamp);
          lg += a.alpha.v[i] * log(dd[i]);
        }
      const double mn = exp(lg);
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i < a.k) {
          v[q][i] = v[q][i] * mn / dd[i];
          Z[q][i] = ar[q] * v[q][i];
          bad |= !isfinite(v[q][i]);
        }
      bad |= !isfinite(mn);
      dl += fabs(mn - mu[q]);
      mu[q] = mn;
    }
    // ||mu_new - mu_old||_1 and the non-finite flag travel with the next S
    // (published by its grid barrier; buffers alternate by iteration)
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) dl += __shfl_xor_sync(0xffffffffu, dl, o2);
    if (lane == 0) redw[warp][0] = dl;
    if (bad) atomicOr(a.status, 1);
    __syncthreads();
    double* red = a.red + int64_t(it & 1) * G;
    if (tid == 0) {
      double sum = 0.0;
      for (int w8 = 0; w8 < 8; ++w8) sum += redw[w8][0];
      red[blockIdx.x] = sum;
    }
    apply_S();
    if (tid == 0) {
      double sum = 0.0;
      for (int c = 0; c < G; ++c) sum += red[c];
      bcast[0] = sum;
      bcast[1] = double(*reinterpret_cast<volatile int*>(a.status));
    }
    __syncthreads();
    if (bcast[1] != 0.0) break;                    // non-finite: stop (uniform)
    if (a.tol > 0.0 && bcast[0] < a.tol) break;    // converged (uniform)
  }
  if (it > a.max_iter) it = a.max_iter;
  // <a, mu> = 1
  double ms = 0.0;
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (ok[q]) ms += ar[q] * mu[q];
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o2);
  if (lane == 0) redw[warp][1] = ms;
  __syncthreads();
  double* mred = a.red + 2 * G;
  if (tid == 0) {
    double sum = 0.0;
    for (int w8 = 0; w8 < 8; ++w8) sum += redw[w8][1];
    mred[blockIdx.x] = sum;
  }
  grid_sync(a.bar);
  if (tid == 0) {
    double sum = 0.0;
    for (int c = 0; c < G; ++c) sum += mred[c];
    bcast[0] = sum;
  }
  __syncthreads();
  const double inv = 1.0 / bcast[0];
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (ok[q]) a.out[ip[q]] = float(mu[q] * inv);
  if (blockIdx.x == 0 && tid == 0) a.status[1] = it;
}

template <int K>
cudaError_t launch_k(const BaryArgs& a, int grid, size_t smem, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(bary_fused_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(bary_fused_smem(32, 4)));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, bary_fused_kernel<K>, a);
}

}  // namespace

size_t bary_fused_smem(int m, int k) {
  const int r = 2 * m;
  return size_t(m) * 2 * kPts * sizeof(float) + 2 * sizeof(float) +
         size_t(1 + 1 + 8 + 4) * r * k * sizeof(double) + 16;
}

int64_t bary_fused_max_points(int sms) { return int64_t(sms) * kPts; }

cudaError_t launch_bary_fused(const float4* pts, const float4* omega4, const double* C,
                              const float* mu_in, const float* area, const double* alpha, int m,
                              int k, int64_t n, int max_iter, double tol, double* part, double* S,
                              double* red, unsigned int* bar, int* status, float* out,
                              cudaStream_t s) {
  LaunchScope L("rfd_bary_fused", s);
  // (red: 2 alternating delta buffers and the mass partials, one per CTA each;
  // part: 2 alternating partial buffers)
  BaryArgs a{};
  a.pts = pts;
  a.omega4 = omega4;
  a.C = C;
  a.mu_in = mu_in;
  a.area = area;
  for (int i = 0; i < k && i < 16; ++i) a.alpha.v[i] = alpha[i];
  a.m = m;
  a.k = k;
  a.n = n;
  a.max_iter = max_iter;
  a.tol = tol;
  a.part = part;
  a.S = S;
  a.red = red;
  a.bar = bar;
  a.status = status;
  a.out = out;
  const int grid = int((n + kPts - 1) / kPts);
  const size_t smem = bary_fused_smem(m, k <= 1 ? 1 : (k <= 2 ? 2 : (k <= 3 ? 3 : 4)));
  switch (k <= 1 ? 1 : (k <= 2 ? 2 : (k <= 3 ? 3 : 4))) {
    case 1: return launch_k<1>(a, grid, smem, s);
    case 2: return launch_k<2>(a, grid, smem, s);
    case 3: return launch_k<3>(a, grid, smem, s);
    default: return launch_k<4>(a, grid, smem, s);
  }
}

}  // namespace rfd
