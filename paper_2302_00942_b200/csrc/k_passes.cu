// K5 -- the small middle step of Eq. 13 in the paper's
// bracket order, between the tensor-core passes
// (k_pass1_tc.cu: S partials = Phi^T F; k_pass2_tc.cu: out = F + Phi Y):
//   reduce_S    S = fixed-order fp64 sum of the pass-1 range partials
//   core_apply  Y = C^ S (fp64 in, fp32 out)
// For r <= 128 both run fused in pass 2's prologue instead.
#include <algorithm>

#include "rfd_internal.h"

namespace rfd {
namespace {

// S[b] = sum over the `chunks` (pass-1 range) partials, fp64, in a fixed order: each CTA
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

}  // namespace

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

}  // namespace rfd
