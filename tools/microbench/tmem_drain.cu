// Microbenchmark: cost of draining a 128 x 256 fp32 TMEM accumulator with 16
// warps (each 32 lanes x 64 columns): (a) tcgen05.ld only, (b) ld + ld + add +
// tcgen05.st into a second accumulator (TMEM -> TMEM long-term sum).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_00942_b200/csrc \
//        tools/microbench/tmem_drain.cu -o tools/microbench/tmem_drain
#include <cstdio>
#include "tc_ptx.cuh"

using namespace rfd;

template <int kKind>
__global__ void __launch_bounds__(512, 1) bench(int iters, long long* out, float* sink) {
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const int lg = warp & 3, q = warp >> 2;
  const uint32_t base = tmem + (uint32_t(32 * lg) << 16) + uint32_t(q * 64);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      float v[16];
      tc::tmem_ld16(base + h * 16, v);
      if (kKind == 0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
      } else {
        float w[16];
        tc::tmem_ld16(base + 256 + h * 16, w);
        uint32_t u[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) u[j] = __float_as_uint(v[j] + w[j]);
        tc::tmem_st16(base + 256 + h * 16, u);
      }
    }
    if (kKind == 1) tc::tmem_st_wait();
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * 512 + threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int kKind>
void run(const char* name) {
  long long* d; float* s;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&s, 148 * 512 * sizeof(float));
  const int iters = 200;
  bench<kKind><<<148, 512>>>(iters, d, s);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-34s cycles per 128x256 drain %8.1f  err=%s\n", name, double(h) / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("ld only (128 KB)");
  run<1>("ld + ld + add + st (TMEM->TMEM)");
  return 0;
}
