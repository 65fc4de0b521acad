// K4/K5/K6 -- the inference passes of Eq. 13, in the
// paper's bracket order:
//   K4 pass1       S_partial = Phi^T F per (frequency block, point chunk)
//   K5 reduce_S    S = fixed-order fp64 sum of the chunk partials
//      core_apply  Y = C^ S (fp64 in, fp32 out)
//   K6 pass2       out = F + Phi Y
// Feature rows (a3) are regenerated in registers in both passes and never
// stored: t = omega.x in turns (fp32), reduced to [-1/2, 1/2], MUFU sin/cos.
//
// Pass 1 is frequency-stationary: lane l of every warp owns frequency
// 32 * blockIdx.x + l and keeps 2 x DC fp32 accumulators; the 8 warps of a
// CTA take interleaved points of a shared-memory batch (x and F broadcast).
// Pass 2 is point-stationary: each thread owns PPT points and DC outputs;
// omega and Y are broadcast from shared memory.  Persistent grid.
#include <algorithm>

#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kPB1 = 64;   // points per pass-1 shared-memory batch
constexpr int kWarps = 8;  // warps per CTA (256 threads)

__device__ __forceinline__ void feature_pair(float4 w, float4 x, float& c, float& s) {
  const float t = fmaf(w.z, x.z, fmaf(w.y, x.y, w.x * x.x));
  const float u = t - rintf(t);
  __sincosf(6.28318530717958647f * u, &s, &c);
}

template <int DC>
__global__ void __launch_bounds__(256)
pass1_kernel(const float4* __restrict__ pts, const float4* __restrict__ omega4, int m,
             int64_t n, int chunks, int64_t chunk, const float* __restrict__ F, int d, int c0,
             int dc, float* __restrict__ partial) {
  __shared__ float4 xs[kPB1];
  __shared__ __align__(16) float fs[kPB1][DC];
  __shared__ float red[kWarps][32][2 * DC + 1];

  const int fb = blockIdx.x, ch = blockIdx.y, b = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = fb * 32 + lane;
  const float4 w = (k < m) ? omega4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t p0 = int64_t(ch) * chunk;
  const int64_t p1 = min(p0 + chunk, n);
  const float4* cloud = pts + int64_t(b) * n;
  const float* Fb = F + int64_t(b) * n * d;

  float ac[DC], as[DC];
#pragma unroll
  for (int j = 0; j < DC; ++j) ac[j] = as[j] = 0.0f;

  for (int64_t base = p0; base < p1; base += kPB1) {
    const int np = (p1 - base < kPB1) ? int(p1 - base) : kPB1;
    if (threadIdx.x < kPB1 && threadIdx.x < np) xs[threadIdx.x] = cloud[base + threadIdx.x];
    for (int e = threadIdx.x; e < np * DC; e += 256) {
      const int p = e / DC, j = e % DC;
      fs[p][j] = (j < dc) ? Fb[(base + p) * d + c0 + j] : 0.0f;
    }
    __syncthreads();
    for (int p = warp; p < np; p += kWarps) {
      float c, s;
      feature_pair(w, xs[p], c, s);
      if constexpr (DC % 4 == 0) {
#pragma unroll
        for (int j = 0; j < DC; j += 4) {
          const float4 f = *reinterpret_cast<const float4*>(&fs[p][j]);
          ac[j] = fmaf(c, f.x, ac[j]); ac[j + 1] = fmaf(c, f.y, ac[j + 1]);
          ac[j + 2] = fmaf(c, f.z, ac[j + 2]); ac[j + 3] = fmaf(c, f.w, ac[j + 3]);
          as[j] = fmaf(s, f.x, as[j]); as[j + 1] = fmaf(s, f.y, as[j + 1]);
          as[j + 2] = fmaf(s, f.z, as[j + 2]); as[j + 3] = fmaf(s, f.w, as[j + 3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < DC; ++j) {
          const float f = fs[p][j];
          ac[j] = fmaf(c, f, ac[j]);
          as[j] = fmaf(s, f, as[j]);
        }
      }
    }
    __syncthreads();
  }
  // Cross-warp reduction in fixed warp order, then one partial per CTA.
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    red[warp][lane][j] = ac[j];
    red[warp][lane][DC + j] = as[j];
  }
  __syncthreads();
  const int r = 2 * m;
  float* out = partial + (int64_t(b) * chunks + ch) * int64_t(r) * dc;
  for (int e = threadIdx.x; e < 32 * 2 * DC; e += 256) {
    const int l = e / (2 * DC), q = e % (2 * DC);
    const int kk = fb * 32 + l;
    const int t = q / DC, j = q % DC;  // t = 0 cos, 1 sin
    if (kk >= m || j >= dc) continue;
    float sum = 0.0f;
#pragma unroll
    for (int wp = 0; wp < kWarps; ++wp) sum += red[wp][l][q];
    out[int64_t(2 * kk + t) * dc + j] = sum;
  }
}

// S[b] = sum over the `chunks` partials, fp64, in a fixed order: each CTA
// takes 32 consecutive elements x 8 chunk slices (slice l sums chunks l, l + 8,
// ... in order, 8 loads in flight), then the 8 slice sums are added in order.
__global__ void __launch_bounds__(256)
reduce_S_kernel(const float* __restrict__ partial, int r, int chunks, int d, int c0, int dc,
                double* __restrict__ S) {
  asm volatile("griddepcontrol.launch_dependents;");  // core_apply may launch
  __shared__ double red[8][33];
  const int b = blockIdx.y;
  const int el = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + el;
  const int64_t st = int64_t(r) * dc;
  double acc = 0.0;
  if (e < r * dc) {
    const float* src = partial + int64_t(b) * chunks * st + e;
    int ch = sl;
    for (; ch + 56 < chunks; ch += 64) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (ch + 8 * u) * st);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += double(v[u]);
    }
    for (; ch < chunks; ch += 8) acc += double(__ldg(src + ch * st));
  }
  red[sl][el] = acc;
  __syncthreads();
  if (sl == 0 && e < r * dc) {
    double sum = 0.0;
#pragma unroll
    for (int l = 0; l < 8; ++l) sum += red[l][el];
    const int a = e / dc, j = e % dc;
    S[(int64_t(b) * r + a) * d + c0 + j] = sum;
  }
}

// Y = C^ S: a CTA takes 8 x rpw rows of one cloud's C^ (rpw rows per warp;
// small r: the whole cloud in one CTA) and a chunk of <= 16 columns; the chunk
// of S is staged transposed in shared memory (St[j][k]: conflict-free reads),
// lanes split k (k = lane + 32 i), then a butterfly reduction per column
// (fixed order: deterministic).
__global__ void __launch_bounds__(256)
core_apply_kernel(const double* __restrict__ C, const double* __restrict__ S, int r, int d,
                  int rpw, float* __restrict__ Y) {
  asm volatile("griddepcontrol.launch_dependents;");  // pass 2 may start its setup
  asm volatile("griddepcontrol.wait;" ::: "memory");  // S from reduce_S
  extern __shared__ double St[];  // [dc][r]
  const int b = blockIdx.y, c0 = blockIdx.z * 16;
  const int dc = min(16, d - c0);
  const double* Sb = S + int64_t(b) * r * d + c0;
#pragma unroll 8
  for (int i = threadIdx.x; i < dc * r; i += 256) {  // loads in flight together
    const int k = i / dc, j = i - k * dc;
    St[j * r + k] = __ldg(Sb + int64_t(k) * d + j);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = 0; t < rpw; ++t) {
    const int a = (blockIdx.x * 8 + warp) * rpw + t;
    if (a >= r) break;
    const double* Ca = C + (int64_t(b) * r + a) * r;
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll 4
    for (int k = lane; k < r; k += 32) {
      const double c = __ldg(Ca + k);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < dc) acc[j] = fma(c, St[j * r + k], acc[j]);
    }
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < dc) {
        double x = acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (j == lane) v = x;
      }
    }
    if (lane < dc) Y[(int64_t(b) * r + a) * d + c0 + lane] = float(v);
  }
}

template <int DC, int PPT>
__global__ void __launch_bounds__(256)
pass2_kernel(const float4* __restrict__ pts, const float4* __restrict__ omega4, int m, int64_t n,
             int batch, const float* __restrict__ Y, const float* F, float* out, int d, int c0,
             int dc) {
  // F and out may alias (in-place integrate): each thread reads F_i before
  // writing out_i, so they carry no __restrict__.
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* om = reinterpret_cast<float4*>(smem_raw);
  float* ys = reinterpret_cast<float*>(om + m);  // [m][2][DC]
  constexpr int TP = 256 * PPT;
  const int64_t tiles_per_cloud = (n + TP - 1) / TP;
  const int64_t ntiles = tiles_per_cloud * batch;
  const bool vec = (DC % 4 == 0) && (dc == DC) && (d % 4 == 0) && (c0 % 4 == 0);

  for (int k = threadIdx.x; k < m; k += 256) om[k] = omega4[k];
  int cur_b = -1;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int b = int(tile / tiles_per_cloud);
    const int64_t base = (tile % tiles_per_cloud) * TP;
    if (b != cur_b) {
      __syncthreads();
      const float* Yb = Y + int64_t(b) * 2 * m * d;
      for (int e = threadIdx.x; e < 2 * m * DC; e += 256) {
        const int a = e / DC, j = e % DC;
        ys[e] = (j < dc) ? Yb[int64_t(a) * d + c0 + j] : 0.0f;
      }
      cur_b = b;
      __syncthreads();
    }
    float4 x[PPT];
    float acc[PPT][DC];
    int64_t idx[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      const int64_t i = base + threadIdx.x + 256 * p;
      idx[p] = (i < n) ? int64_t(b) * n + i : -1;
      x[p] = (i < n) ? pts[idx[p]] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < DC; ++j) acc[p][j] = 0.0f;
    }
#pragma unroll 2
    for (int k = 0; k < m; ++k) {
      const float4 w = om[k];
      const float* yk = ys + 2 * DC * k;
      float cs[PPT], sn[PPT];
#pragma unroll
      for (int p = 0; p < PPT; ++p) feature_pair(w, x[p], cs[p], sn[p]);
      if constexpr (DC % 4 == 0) {
#pragma unroll
        for (int j = 0; j < DC; j += 4) {
          const float4 yc = *reinterpret_cast<const float4*>(yk + j);
          const float4 yn = *reinterpret_cast<const float4*>(yk + DC + j);
#pragma unroll
          for (int p = 0; p < PPT; ++p) {
            acc[p][j] = fmaf(cs[p], yc.x, fmaf(sn[p], yn.x, acc[p][j]));
            acc[p][j + 1] = fmaf(cs[p], yc.y, fmaf(sn[p], yn.y, acc[p][j + 1]));
            acc[p][j + 2] = fmaf(cs[p], yc.z, fmaf(sn[p], yn.z, acc[p][j + 2]));
            acc[p][j + 3] = fmaf(cs[p], yc.w, fmaf(sn[p], yn.w, acc[p][j + 3]));
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < DC; ++j) {
          const float yc = yk[j], yn = yk[DC + j];
#pragma unroll
          for (int p = 0; p < PPT; ++p) acc[p][j] = fmaf(cs[p], yc, fmaf(sn[p], yn, acc[p][j]));
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      if (idx[p] < 0) continue;
      const float* Fi = F + idx[p] * d + c0;
      float* Oi = out + idx[p] * d + c0;
      if (vec) {
#pragma unroll
        for (int j = 0; j < DC; j += 4) {
          float4 f = *reinterpret_cast<const float4*>(Fi + j);
          f.x += acc[p][j]; f.y += acc[p][j + 1]; f.z += acc[p][j + 2]; f.w += acc[p][j + 3];
          *reinterpret_cast<float4*>(Oi + j) = f;
        }
      } else {
#pragma unroll
        for (int j = 0; j < DC; ++j)
          if (j < dc) Oi[j] = Fi[j] + acc[p][j];
      }
    }
  }
}

int pick_dc(int dc) {
  if (dc <= 1) return 1;
  if (dc <= 2) return 2;
  if (dc <= 3) return 3;
  if (dc <= 4) return 4;
  if (dc <= 8) return 8;
  return 16;
}

template <int DC>
void pass1_t(dim3 grid, cudaStream_t s, const float4* pts, const float4* omega4, int m,
             int64_t n, int chunks, int64_t chunk, const float* F, int d, int c0, int dc,
             float* partial) {
  pass1_kernel<DC><<<grid, 256, 0, s>>>(pts, omega4, m, n, chunks, chunk, F, d, c0, dc, partial);
}

template <int DC>
void pass2_t(int blocks, cudaStream_t s, const float4* pts, const float4* omega4, int m,
             int64_t n, int batch, const float* Y, const float* F, float* out, int d, int c0,
             int dc) {
  constexpr int PPT = (DC >= 8) ? 2 : 4;
  const size_t smem = size_t(m) * sizeof(float4) + size_t(2) * m * DC * sizeof(float);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(pass2_kernel<DC, PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         160 * 1024);
    configured = true;
  }
  static size_t occ_smem = ~size_t(0);
  static int occ = 1;
  if (occ_smem != smem) {  // occupancy depends only on the shared-memory size
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass2_kernel<DC, PPT>, 256, smem);
    if (occ < 1) occ = 1;
    occ_smem = smem;
  }
  constexpr int TP = 256 * PPT;
  const int64_t ntiles = ((n + TP - 1) / TP) * batch;
  int64_t grid = int64_t(blocks) * occ;
  if (grid > ntiles) grid = ntiles;
  pass2_kernel<DC, PPT><<<unsigned(grid), 256, smem, s>>>(pts, omega4, m, n, batch, Y, F, out, d,
                                                         c0, dc);
}

}  // namespace

PassGeom pass_geometry(int m, int64_t n, int batch, int sms) {
  PassGeom g;
  g.fblocks = (m + 31) / 32;
  const int64_t want = 8LL * sms;
  int64_t chunks = (want + int64_t(g.fblocks) * batch - 1) / (int64_t(g.fblocks) * batch);
  const int64_t maxc = std::max<int64_t>(1, (n + 255) / 256);
  if (chunks > maxc) chunks = maxc;
  if (chunks < 1) chunks = 1;
  int64_t chunk = (n + chunks - 1) / chunks;
  chunk = (chunk + kPB1 - 1) / kPB1 * kPB1;
  g.chunk = chunk;
  g.chunks = int((n + chunk - 1) / chunk);
  g.p2_blocks = sms;
  return g;
}

void launch_pass1(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                  const PassGeom& g, const float* F, int d, int c0, int dc, float* partial,
                  cudaStream_t s) {
  LaunchScope L("rfd_pass1", s);
  const dim3 grid(g.fblocks, g.chunks, batch);
  switch (pick_dc(dc)) {
    case 1: pass1_t<1>(grid, s, pts, omega4, m, n, g.chunks, g.chunk, F, d, c0, dc, partial); break;
    case 2: pass1_t<2>(grid, s, pts, omega4, m, n, g.chunks, g.chunk, F, d, c0, dc, partial); break;
    case 3: pass1_t<3>(grid, s, pts, omega4, m, n, g.chunks, g.chunk, F, d, c0, dc, partial); break;
    case 4: pass1_t<4>(grid, s, pts, omega4, m, n, g.chunks, g.chunk, F, d, c0, dc, partial); break;
    case 8: pass1_t<8>(grid, s, pts, omega4, m, n, g.chunks, g.chunk, F, d, c0, dc, partial); break;
    default: pass1_t<16>(grid, s, pts, omega4, m, n, g.chunks, g.chunk, F, d, c0, dc, partial); break;
  }
}

void launch_reduce_S(const float* partial, int m, int batch, int chunks, int d, int c0, int dc,
                     double* S, cudaStream_t s) {
  LaunchScope L("rfd_reduce_S", s);
  const int r = 2 * m;
  // (a normal launch: launched early, its waiting CTAs would sit beside pass 1's)
  reduce_S_kernel<<<dim3((r * dc + 31) / 32, batch), 256, 0, s>>>(partial, r, chunks, d, c0, dc,
                                                                   S);
}

void launch_core_apply(const double* C, const double* S, int m, int batch, int d, float* Y,
                       cudaStream_t s) {
  LaunchScope L("rfd_core_apply", s);
  const int r = 2 * m;
  const size_t smem = size_t(16) * r * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(core_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         16 * 1024 * int(sizeof(double)));  // r <= 2 RFD_MAX_M = 1024
    configured = true;
  }
  // rows per warp: 1 while that leaves < ~2 CTAs per SM, more for many small
  // clouds (at most the whole cloud in one CTA)
  int64_t rpw64 = (int64_t(r) * batch) / (8 * 148 * 2);
  if (rpw64 > (r + 7) / 8) rpw64 = (r + 7) / 8;
  const int rpw = rpw64 < 1 ? 1 : int(rpw64);
  launch_pdl(core_apply_kernel, dim3((r + 8 * rpw - 1) / (8 * rpw), batch, (d + 15) / 16),
             dim3(256), smem, s, C, S, r, d, rpw, Y);
}

void launch_pass2(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                  const PassGeom& g, const float* Y, const float* F, float* out, int d, int c0,
                  int dc, cudaStream_t s) {
  LaunchScope L("rfd_pass2", s);
  switch (pick_dc(dc)) {
    case 1: pass2_t<1>(g.p2_blocks, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc); break;
    case 2: pass2_t<2>(g.p2_blocks, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc); break;
    case 3: pass2_t<3>(g.p2_blocks, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc); break;
    case 4: pass2_t<4>(g.p2_blocks, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc); break;
    case 8: pass2_t<8>(g.p2_blocks, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc); break;
    default: pass2_t<16>(g.p2_blocks, s, pts, omega4, m, n, batch, Y, F, out, d, c0, dc); break;
  }
}

}  // namespace rfd
