// Microbenchmark: do tensor-core shared-memory operand reads (tcgen05.mma SS,
// M=128 N=256 K=16 fp16) contend with STS traffic from other warps?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_00942_b200/csrc \
//        tools/microbench/smem_contention.cu -o tools/microbench/smem_contention
#include <cstdio>
#include "tc_ptx.cuh"

using namespace rfd;

template <bool TS>
__global__ void __launch_bounds__(544, 1) bench(int iters, int sts_warps, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_sh;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); done = 0; }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t sb = tc::smem_addr(smem);
  if (warp == 16) {
    if (lane == 0) {
      const uint32_t idesc = tc::make_idesc(0, 128, 256);
      const uint64_t a = tc::make_sdesc(sb, 128, 256);
      const uint64_t b = tc::make_sdesc(sb + 16384, 128, 256);
      long long t0 = clock64();
      uint32_t ph = 0;
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (TS) tc::mma_f16_ts(tmem, tmem + 256, b, idesc, 1u);
          else tc::mma_f16(tmem, a, b, idesc, 1u);
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, ph);
        ph ^= 1u;
      }
      out[blockIdx.x * 2] = clock64() - t0;
      done = 1;
    }
  } else if (warp < sts_warps) {
    // STS.128 stream into a separate 64 KB region (conflict-free, 512 B / warp-instr)
    long long n = 0;
    const uint32_t base = sb + 65536 + (warp & 7) * 8192 + lane * 16;
    while (!done) {
#pragma unroll
      for (int r = 0; r < 16; ++r) tc::st_shared_v4(base + (r & 15) * 512, r, r, r, r);
      n += 16;
    }
    if (lane == 0) atomicAdd((unsigned long long*)&out[blockIdx.x * 2 + 1], (unsigned long long)n);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <bool TS>
void run(int sts_warps) {
  long long* d; cudaMalloc(&d, 148 * 2 * sizeof(long long));
  cudaMemset(d, 0, 148 * 2 * sizeof(long long));
  auto k = bench<TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int iters = 400;
  k<<<148, 544, 128 * 1024>>>(iters, sts_warps, d);
  cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double cyc = double(h[0]) / (iters * 32.0);
  const double sts_bytes_per_cyc = double(h[1]) * 512.0 / double(h[0]);
  printf("%s sts_warps=%2d  cycles/MMA(N=256) %6.1f (ideal 128)  STS %6.1f B/cycle  err=%s\n",
         TS ? "TS" : "SS", sts_warps, cyc, sts_bytes_per_cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int w : {0, 2, 4, 8, 16}) run<false>(w);
  for (int w : {0, 4, 16}) run<true>(w);
  return 0;
}
