// one cloud's points partitioned across the ranks of a
// process group (one GPU per rank).  G = sum_i phi(x_i) phi(x_i)^T (the B^T A
// of PAPER.md:337, 355) and S = Phi^T F (Eq. 13's first bracket) are sums over
// points ("linear in N"), so each rank forms its shard's partial
// and the ranks exchange partials once per sum; the caller's collective
// library all-gathers them (rank-major) and these kernels add them in rank
// order -- the same fixed order on every rank, so every rank holds bitwise the
// same G (hence C^) and S (hence Y).  The bounding box that centres the cloud
// (k_freq.cu) is merged the same way, so all shards share one centre.
#include <math.h>

#include "rfd_internal.h"

namespace rfd {
namespace {

__device__ __forceinline__ float dec_f32(unsigned int e) {
  return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}
__device__ __forceinline__ unsigned int enc_f32(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// send[0..5] = (min x, min y, min z, max x, max y, max z) (exact fp32 values
// as fp64), send[6] = the shard's point count
__global__ void bbox_export_kernel(const unsigned int* __restrict__ bbox, int64_t n_local,
                                   double* __restrict__ send) {
  const int c = threadIdx.x;
  if (c < 3) send[c] = double(dec_f32(~bbox[c]));
  else if (c < 6) send[c] = double(dec_f32(bbox[c]));
  else if (c == 6) send[6] = double(n_local);
}

// bbox = the union of the gathered shard boxes (min / max: order-independent)
__global__ void bbox_merge_kernel(const double* __restrict__ recv, int world,
                                  unsigned int* __restrict__ bbox) {
  const int c = threadIdx.x;
  if (c >= 6) return;
  float v = float(recv[c]);
  for (int q = 1; q < world; ++q) {
    const float w = float(recv[q * 7 + c]);
    v = (c < 3) ? fminf(v, w) : fmaxf(v, w);
  }
  bbox[c] = (c < 3) ? ~enc_f32(v) : enc_f32(v);
}

// out[e] = sum over ranks q = 0 .. world-1 (in that order) of parts[q][e]
__global__ void __launch_bounds__(256)
sum_parts_kernel(const double* __restrict__ parts, int world, int64_t count,
                 double* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count;
       e += int64_t(gridDim.x) * blockDim.x) {
    double s = parts[e];
    for (int q = 1; q < world; ++q) s += parts[int64_t(q) * count + e];
    out[e] = s;
  }
}

}  // namespace

void launch_bbox_export(const unsigned int* bbox, int64_t n_local, double* send, cudaStream_t s) {
  LaunchScope L("rfd_shard_bbox", s);
  bbox_export_kernel<<<1, 32, 0, s>>>(bbox, n_local, send);
}

void launch_bbox_merge(const double* recv, int world, unsigned int* bbox, cudaStream_t s) {
  LaunchScope L("rfd_shard_bbox", s);
  bbox_merge_kernel<<<1, 32, 0, s>>>(recv, world, bbox);
}

void launch_sum_parts(const double* parts, int world, int64_t count, double* out, cudaStream_t s) {
  LaunchScope L("rfd_shard_sum", s);
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  sum_parts_kernel<<<unsigned(blocks), 256, 0, s>>>(parts, world, count, out);
}

}  // namespace rfd
