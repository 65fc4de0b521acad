// K1/K2 -- Gram matrix G = Phi^T Phi (the B^T A of
// PAPER.md:337, 355 without D).  Plan-time only.
//
// K1 (gram_partial): grid (upper tile, point chunk, cloud).  Each CTA
// regenerates the feature rows of its tile pair for the points of its chunk
// in shared memory (a3, never stored in HBM) and accumulates the TILE x TILE
// outer products in fp32 registers (8 x 8 per thread for TILE = 128).  Chunks
// hold <= 8192 points so fp32 partial sums stay short.
// K2 (gram_reduce): fixed-order fp64 sum of the chunk partials -> G (full
// symmetric, interleaved feature order).  Deterministic: no atomics.
#include "rfd_internal.h"

namespace rfd {
namespace {

constexpr int kPB = 32;  // points per shared-memory batch

__device__ __forceinline__ void feature_pair(float4 w, float4 x, float& c, float& s) {
  // t = omega . x in turns (fp32), reduced to [-1/2, 1/2], then MUFU sin/cos.
  const float t = fmaf(w.z, x.z, fmaf(w.y, x.y, w.x * x.x));
  const float u = t - rintf(t);
  __sincosf(6.28318530717958647f * u, &s, &c);
}

__device__ __forceinline__ void decode_upper(int t, int T, int& ti, int& tj) {
  // t enumerates (ti <= tj) row by row.
  ti = 0;
  int row = T;
  while (t >= row) { t -= row; ++ti; --row; }
  tj = ti + t;
}

template <int TILE>
__global__ void __launch_bounds__(256)
gram_partial_kernel(const float4* __restrict__ pts, const float4* __restrict__ omega4,
                    int m, int64_t n, int tiles1d, int ntiles, int chunks, int64_t chunk,
                    float* __restrict__ partial) {
  constexpr int TM = TILE / 16;
  constexpr int HALF = TILE / 2;
  __shared__ float4 xs[kPB];
  __shared__ __align__(16) float fa[kPB][TILE];
  __shared__ __align__(16) float fb[kPB][TILE];

  const int tile = blockIdx.x, ch = blockIdx.y, b = blockIdx.z;
  int ti, tj;
  decode_upper(tile, tiles1d, ti, tj);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t p0 = int64_t(ch) * chunk;
  const int64_t p1 = min(p0 + chunk, n);
  const float4* cloud = pts + int64_t(b) * n;

  float acc[TM][TM];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TM; ++j) acc[i][j] = 0.0f;

  for (int64_t base = p0; base < p1; base += kPB) {
    const int np = (p1 - base < kPB) ? int(p1 - base) : kPB;
    if (tid < kPB) xs[tid] = (tid < np) ? cloud[base + tid] : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    for (int idx = tid; idx < kPB * TILE; idx += 256) {
      const int p = idx / TILE, j = idx % TILE;
      const bool isA = j < HALF;
      const int k = isA ? ti * HALF + j : tj * HALF + (j - HALF);
      float c = 0.0f, s = 0.0f;
      if (k < m && p < np) feature_pair(omega4[k], xs[p], c, s);
      float* dst = isA ? &fa[p][2 * j] : &fb[p][2 * (j - HALF)];
      dst[0] = c;
      dst[1] = s;
    }
    __syncthreads();
#pragma unroll 4
    for (int p = 0; p < kPB; ++p) {
      float av[TM], bv[TM];
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        const float4 va = *reinterpret_cast<const float4*>(&fa[p][ty * TM + i]);
        const float4 vb = *reinterpret_cast<const float4*>(&fb[p][tx * TM + i]);
        av[i] = va.x; av[i + 1] = va.y; av[i + 2] = va.z; av[i + 3] = va.w;
        bv[i] = vb.x; bv[i + 1] = vb.y; bv[i + 2] = vb.z; bv[i + 3] = vb.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TM; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }

  float* out = partial + ((int64_t(b) * chunks + ch) * ntiles + tile) * (TILE * TILE);
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TM; j += 4)
      *reinterpret_cast<float4*>(&out[(ty * TM + i) * TILE + tx * TM + j]) =
          make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
}

__global__ void gram_reduce_kernel(const float* __restrict__ partial, int r, int tile_sz,
                                   int tiles1d, int ntiles, int chunks,
                                   double* __restrict__ G) {
  const int tile = blockIdx.y, b = blockIdx.z;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tile_sz * tile_sz) return;
  int ti, tj;
  decode_upper(tile, tiles1d, ti, tj);
  const int a = ti * tile_sz + e / tile_sz, c = tj * tile_sz + e % tile_sz;
  if (a >= r || c >= r) return;
  const int64_t stride = int64_t(ntiles) * tile_sz * tile_sz;
  const float* src = partial + (int64_t(b) * chunks * ntiles + tile) * tile_sz * tile_sz + e;
  double sum = 0.0;
  for (int ch = 0; ch < chunks; ++ch) sum += double(src[ch * stride]);
  double* Gb = G + int64_t(b) * r * r;
  Gb[int64_t(a) * r + c] = sum;
  Gb[int64_t(c) * r + a] = sum;
}

}  // namespace

GramGeom gram_geometry(int m, int64_t n, int batch, int sms) {
  GramGeom g;
  g.r = 2 * m;
  g.tile = (g.r <= 64) ? 64 : 128;
  g.tiles1d = (g.r + g.tile - 1) / g.tile;
  g.ntiles = g.tiles1d * (g.tiles1d + 1) / 2;
  int64_t chunks = (n + 8191) / 8192;
  const int64_t want = (4LL * sms + int64_t(g.ntiles) * batch - 1) / (int64_t(g.ntiles) * batch);
  if (want > chunks) chunks = want;
  const int64_t maxc = (n + kPB - 1) / kPB;
  if (chunks > maxc) chunks = maxc;
  if (chunks < 1) chunks = 1;
  int64_t chunk = (n + chunks - 1) / chunks;
  chunk = (chunk + kPB - 1) / kPB * kPB;
  g.chunk = chunk;
  g.chunks = int((n + chunk - 1) / chunk);
  return g;
}

size_t gram_partial_elems(const GramGeom& g, int batch) {
  return size_t(batch) * g.chunks * g.ntiles * g.tile * g.tile;
}

void launch_gram(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                 const GramGeom& g, float* partial, double* G, cudaStream_t s) {
  {
    LaunchScope L("rfd_gram_partial", s);
    dim3 grid(g.ntiles, g.chunks, batch);
    if (g.tile == 128)
      gram_partial_kernel<128><<<grid, 256, 0, s>>>(pts, omega4, m, n, g.tiles1d, g.ntiles,
                                                    g.chunks, g.chunk, partial);
    else
      gram_partial_kernel<64><<<grid, 256, 0, s>>>(pts, omega4, m, n, g.tiles1d, g.ntiles,
                                                   g.chunks, g.chunk, partial);
  }
  {
    LaunchScope L("rfd_gram_reduce", s);
    dim3 grid((g.tile * g.tile + 255) / 256, g.ntiles, batch);
    gram_reduce_kernel<<<grid, 256, 0, s>>>(partial, g.r, g.tile, g.tiles1d, g.ntiles,
                                            g.chunks, G);
  }
}

}  // namespace rfd
