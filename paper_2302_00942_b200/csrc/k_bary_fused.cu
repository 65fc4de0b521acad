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
//   sweep:  out_p = X_p + sum_k [cos_kp Yc_k + sin_kp Ys_k]      (pass 2 of
//           the previous application) -> the elementwise update of Alg. 1 ->
//           the next input X'_p -> S' partial += phi_p X'_p      (pass 1 of
//           the next application), all on the same cached rows, per point
//   grid barrier; S' = fixed-order sum of the CTA partials (fp64)
//   grid barrier; every CTA forms Y' = C^ S' (fp64 -> fp32) in shared memory
//
// Point-stationary throughout (thread = 2 points); the S partials are
// reduced over the CTA by warp shuffles in a fixed pattern and the warps in
// order: deterministic.  The iterates v, mu (and w, d) are fp64 as in the
// unfused path; the FM_K inputs are fp32(a v), fp32(a w) without rescaling:
// fp32 is scale-invariant under powers of two, so the unfused path's
// power-of-two rescale only guards the range, which the clamp bounds here
// (|a w| <= max mu^i / 1e-30); a non-finite value is reported as ERANGE.
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
  double* part;          // gridDim x (r x k) CTA partials (fp64)
  double* S;             // r x k
  double* red;           // gridDim x 2: per-CTA delta / mass partials
  double* smax;          // gridDim x 4: per-CTA column maxima of the next input
  unsigned int* bar;     // 2 words (generation, count)
  int* status;           // [0] non-finite flag, [1] iterations run
  float* out;            // n
};

template <int K>
__global__ void __launch_bounds__(kThreads, 1) bary_fused_kernel(const BaryArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = a.m, r = 2 * m;
  float* feat = sm;                                   // [m][2][kPts]
  float* ys = feat + m * 2 * kPts;                    // [r][K] fp32 Y
  double* wpart = reinterpret_cast<double*>(ys + r * K + 4);  // [8][r][K] warp partials
  double* yq = wpart + 8 * r * K;                     // [4][r][K] Y quarters
  __shared__ double redw[8][2];
  __shared__ double bcast[2];
  __shared__ double redm[8][K];
  __shared__ double scs[K];

  const int64_t pbase = int64_t(blockIdx.x) * kPts;
  const int64_t ip[2] = {pbase + tid, pbase + tid + kThreads};
  bool ok[2];
  float ar[2];
  // ---- the CTA's feature rows: the only sin/cos of the run (a3)
  {
    float4 x[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      ok[q] = ip[q] < a.n;
      x[q] = ok[q] ? __ldg(a.pts + ip[q]) : make_float4(0.f, 0.f, 0.f, 0.f);
      ar[q] = ok[q] ? __ldg(a.area + ip[q]) : 0.0f;
    }
    for (int kk = 0; kk < m; ++kk) {
      const float4 w = __ldg(a.omega4 + kk);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float t = fmaf(w.z, x[q].z, fmaf(w.y, x[q].y, w.x * x[q].x));
        float s, c;
        __sincosf(t, &s, &c);
        feat[(kk * 2 + 0) * kPts + tid + q * kThreads] = ok[q] ? c : 0.0f;
        feat[(kk * 2 + 1) * kPts + tid + q * kThreads] = ok[q] ? s : 0.0f;
      }
    }
  }
  // per-point state (fp64 iterates), FM_K input X (fp32)
  double v[2][K], mu[2];
  float mui[2][K], X[2][K];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    mu[q] = 1.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      v[q][i] = 1.0;
      mui[q][i] = (ok[q] && i < a.k) ? __ldg(a.mu_in + int64_t(i) * a.n + ip[q]) : 0.0f;
    }
  }
  __syncthreads();

  // The next FM_K input X = fp32(az sc), az = a v or a w (fp64), sc a power of
  // two per column putting the column maximum in [1/2, 1) -- exact by
  // linearity (FM_K(az) = FM_K(X) / sc), it keeps fp32 in range (v and w can
  // grow by 1e30 per iteration where the clamp binds).  One grid barrier.
  double sc[K];
  auto set_inputs = [&](const double (&az)[2][K]) {
    double mx[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      mx[i] = fmax(ok[0] ? fabs(az[0][i]) : 0.0, ok[1] ? fabs(az[1][i]) : 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx[i] = fmax(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
      if (lane == 0) redm[warp][i] = mx[i];
    }
    __syncthreads();
    if (tid < K) {
      double m8 = 0.0;
      for (int w8 = 0; w8 < 8; ++w8) m8 = fmax(m8, redm[w8][tid]);
      a.smax[4 * blockIdx.x + tid] = m8;
    }
    grid_sync(a.bar);
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double m = 0.0;
        for (int c = lane; c < int(gridDim.x); c += 32) m = fmax(m, a.smax[4 * c + i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) {
          double sv = 1.0;
          if (isfinite(m) && m > 0.0) {
            int e = 0;
            frexp(m, &e);
            sv = ldexp(1.0, -e);
          }
          scs[i] = sv;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < K; ++i) {
      sc[i] = scs[i];
#pragma unroll
      for (int q = 0; q < 2; ++q) X[q][i] = (ok[q] && i < a.k) ? float(az[q][i] * sc[i]) : 0.0f;
    }
  };
  {
    double az[2][K];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < K; ++i) az[q][i] = double(ar[q]);  // a v, v = 1
    set_inputs(az);
  }

  // S partial of the CTA for the current X (pass 1 on the cached rows), then
  // grid-wide S, then Y = C^ S in every CTA's shared memory
  auto apply_S = [&]() {
    for (int k4 = 0; k4 < m; k4 += 4) {
      double acc[4][2][K];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k4 + u;
        float c0 = 0.f, s0 = 0.f, c1 = 0.f, s1 = 0.f;
        if (kk < m) {
          c0 = feat[(kk * 2) * kPts + tid];
          s0 = feat[(kk * 2 + 1) * kPts + tid];
          c1 = feat[(kk * 2) * kPts + tid + kThreads];
          s1 = feat[(kk * 2 + 1) * kPts + tid + kThreads];
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
          acc[u][0][i] = double(fmaf(c1, X[1][i], c0 * X[0][i]));
          acc[u][1][i] = double(fmaf(s1, X[1][i], s0 * X[0][i]));
        }
      }
      // warp sum (fixed butterfly), lane 0 keeps the warp's partial
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
      double s = 0.0;
#pragma unroll
      for (int w8 = 0; w8 < 8; ++w8) s += wpart[w8 * r * K + e];
      a.part[int64_t(blockIdx.x) * r * K + e] = s;
    }
    grid_sync(a.bar);
    // S = the CTA partials in CTA order: one warp per element, lane l takes
    // CTAs l, l + 32, ..., the lane sums added in lane order
    for (int e = blockIdx.x * (kThreads / 32) + warp; e < r * K; e += gridDim.x * (kThreads / 32)) {
      double s = 0.0;
      for (int c = lane; c < int(gridDim.x); c += 32) s += a.part[int64_t(c) * r * K + e];
      double tot = 0.0;
#pragma unroll
      for (int l = 0; l < 32; ++l) tot += __shfl_sync(0xffffffffu, s, l);
      if (lane == 0) a.S[e] = tot;
    }
    grid_sync(a.bar);
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
        for (int i = 0; i < K; ++i) acc[i] = fma(cv, a.S[cc * K + i], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < K; ++i) yq[(qq * r + row) * K + i] = acc[i];
    }
    __syncthreads();
    for (int e = tid; e < r * K; e += kThreads)
      ys[e] = float(((yq[e] + yq[r * K + e]) + yq[2 * r * K + e]) + yq[3 * r * K + e]);
    __syncthreads();
  };
  // out = X + Phi Y on the cached rows (pass 2)
  auto apply_out = [&](float (&o)[2][K]) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < K; ++i) o[q][i] = 0.0f;
    for (int kk = 0; kk < m; ++kk) {
      const float c0 = feat[(kk * 2) * kPts + tid], s0 = feat[(kk * 2 + 1) * kPts + tid];
      const float c1 = feat[(kk * 2) * kPts + tid + kThreads];
      const float s1 = feat[(kk * 2 + 1) * kPts + tid + kThreads];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const float yc = ys[(2 * kk) * K + i], yn = ys[(2 * kk + 1) * K + i];
        o[0][i] = fmaf(c0, yc, fmaf(s0, yn, o[0][i]));
        o[1][i] = fmaf(c1, yc, fmaf(s1, yn, o[1][i]));
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < K; ++i) o[q][i] += X[q][i];
  };

  apply_S();  // S = Phi^T (a v), v = 1
  int it = 0;
  bool bad = false;
  for (it = 1; it <= a.max_iter; ++it) {
    float o[2][K];
    // 1. w^i = mu^i / FM_K(a v^i); the next input a w^i
    apply_out(o);
    double aw[2][K];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const double w = double(mui[q][i]) / fmax(double(o[q][i]) / sc[i], kClamp);
        aw[q][i] = double(ar[q]) * w;
        bad |= !isfinite(w);
      }
    set_inputs(aw);
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
          dd[i] = fmax(v[q][i] * (double(o[q][i]) / sc[i]), kClamp);
          lg += a.alpha.v[i] * log(dd[i]);
        }
      const double mn = exp(lg);
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i < a.k) {
          v[q][i] = v[q][i] * mn / dd[i];
          bad |= !isfinite(v[q][i]);
        }
      bad |= !isfinite(mn);
      dl += fabs(mn - mu[q]);
      mu[q] = mn;
    }
    // ||mu_new - mu_old||_1 and the non-finite flag, then the next S
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) dl += __shfl_xor_sync(0xffffffffu, dl, o2);
    if (lane == 0) redw[warp][0] = dl;
    if (bad) atomicOr(a.status, 1);
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w8 = 0; w8 < 8; ++w8) s += redw[w8][0];
      a.red[2 * blockIdx.x] = s;
    }
    {
      double av[2][K];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < K; ++i) av[q][i] = double(ar[q]) * v[q][i];
      set_inputs(av);
    }
    apply_S();  // (its grid barriers publish the delta partials and the flag)
    if (tid == 0) {
      double s = 0.0;
      for (int c = 0; c < int(gridDim.x); ++c) s += a.red[2 * c];
      bcast[0] = s;
      bcast[1] = double(*reinterpret_cast<volatile int*>(a.status));
    }
    __syncthreads();
    if (bcast[1] != 0.0) break;                    // non-finite: stop (uniform)
    if (a.tol > 0.0 && bcast[0] < a.tol) break;    // converged (uniform)
    // (red is rewritten only after the next apply_S's barriers: every CTA has
    // read it by then)
  }
  if (it > a.max_iter) it = a.max_iter;
  // <a, mu> = 1
  double ms = 0.0;
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (ok[q]) ms += double(ar[q]) * mu[q];
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o2);
  if (lane == 0) redw[warp][1] = ms;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w8 = 0; w8 < 8; ++w8) s += redw[w8][1];
    a.red[2 * blockIdx.x + 1] = s;
  }
  grid_sync(a.bar);
  if (tid == 0) {
    double s = 0.0;
    for (int c = 0; c < int(gridDim.x); ++c) s += a.red[2 * c + 1];
    bcast[0] = s;
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
  return size_t(m) * 2 * kPts * sizeof(float) + (size_t(r) * k + 4) * sizeof(float) +
         size_t(8 + 4) * r * k * sizeof(double) + 16;
}

int64_t bary_fused_max_points(int sms) { return int64_t(sms) * kPts; }

cudaError_t launch_bary_fused(const float4* pts, const float4* omega4, const double* C,
                              const float* mu_in, const float* area, const double* alpha, int m,
                              int k, int64_t n, int max_iter, double tol, double* part, double* S,
                              double* red, unsigned int* bar, int* status, float* out,
                              cudaStream_t s) {
  LaunchScope L("rfd_bary_fused", s);
  // (red holds 2 per CTA for the delta / mass partials, then 4 per CTA for the
  // input column maxima)
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
  a.smax = red + 2 * ((n + kPts - 1) / kPts);
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
