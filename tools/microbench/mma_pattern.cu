// Microbenchmark: the Gram kernel's per-step MMA pattern (2 K-slices x 2
// tiles x 3 products, N = 128, A from TMEM, B from 2 smem slots, 6 stages),
// one commit per step, the issuer waiting for step j - depth before issuing
// step j (the producers' stage reuse).  Prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_00942_b200/csrc \
//        tools/microbench/mma_pattern.cu -o tools/microbench/mma_pattern
#include <cstdio>
#include "tc_ptx.cuh"

using namespace rfd;

template <int kDepth, bool kSameD>
__global__ void __launch_bounds__(128, 1) bench(int steps, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar[6];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
  for (int i = threadIdx.x; i < 192 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { for (int s = 0; s < 6; ++s) tc::mbar_init(&bar[s], 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t sb = tc::smem_addr(smem);
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc(0, 128, 128);
    long long t0 = clock64();
    for (int it = 0; it < steps; ++it) {
      const int s = it % 6;
      if (it >= kDepth) tc::mbar_wait(&bar[(it - kDepth) % 6], uint32_t((it - kDepth) / 6) & 1u);
      const uint32_t stage = sb + uint32_t(s) * 32768u;
      for (int kk = 0; kk < 2; ++kk) {
        const uint32_t a_hi = tmem + 256 + 32u * s + 8u * kk, a_lo = a_hi + 16;
        for (int tau = 0; tau < 2; ++tau) {
          const uint32_t bo = stage + tau * 16384u + kk * 256u;
          const uint64_t bh = tc::make_sdesc(bo, 128, 512), bl = tc::make_sdesc(bo + 8192, 128, 512);
          const uint32_t d = kSameD ? tmem : tmem + 128u * tau;
          tc::mma_f16_ts(d, a_hi, bh, idesc, 1u);
          tc::mma_f16_ts(d, a_hi, bl, idesc, 1u);
          tc::mma_f16_ts(d, a_lo, bh, idesc, 1u);
        }
      }
      tc::mma_commit(&bar[s]);
    }
    for (int it = steps - 1; it >= 0 && it >= steps - 6; --it) tc::mbar_wait(&bar[it % 6], uint32_t(it / 6) & 1u);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int kDepth, bool kSameD>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * sizeof(long long));
  auto k = bench<kDepth, kSameD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
  const int steps = 3000;
  k<<<148, 128, 192 * 1024>>>(12, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, 192 * 1024>>>(steps, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-26s cycles/MMA %6.1f (ideal 64)  %.3f ms  err=%s\n", name, double(h[0]) / (steps * 12.0), ms,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<1, false>("depth 1");
  run<2, false>("depth 2");
  run<3, false>("depth 3");
  run<5, false>("depth 5");
  run<5, true>("depth 5, one accumulator");
  return 0;
}
