// Microbenchmark: tcgen05.mma kind::f16 issue rate on one SM per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_00942_b200/csrc \
//        tools/microbench/mma_rate.cu -o /tmp/mma_rate && /tmp/mma_rate
// Variants: A from TMEM (ts) or shared memory (ss); N = 64/128/256; the
// number of MMAs between commits.  Prints cycles per MMA (clock64 around a
// loop of MMAs + commit + wait) and the implied dense fp16 TFLOP/s per GPU.
#include <cstdio>
#include "tc_ptx.cuh"

using namespace rfd;

template <int N, bool TS, int kPerCommit>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tmem_sh);
  // zero the operands
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t sb = tc::smem_addr(smem);
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc(0, 128, N);
    const uint64_t a = tc::make_sdesc(sb, 128, 256);
    const uint64_t b = tc::make_sdesc(sb + 16384, 128, 256);
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < kPerCommit; ++j) {
        if (TS) tc::mma_f16_ts(tmem + ((j & 1) ? 0 : 0), tmem + 256, b, idesc, 1u);
        else tc::mma_f16(tmem, a, b, idesc, 1u);
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, ph);
      ph ^= 1u;
    }
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int N, bool TS, int kPerCommit>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * sizeof(long long));
  auto k = bench<N, TS, kPerCommit>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 2000;
  k<<<148, 128, 64 * 1024>>>(10, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, 64 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = double(h[0]) / (double(iters) * kPerCommit);
  double flop = 2.0 * 128 * N * 16 * double(iters) * kPerCommit * 148;
  printf("%-28s cycles/MMA %7.1f   (ideal %5.1f)  %7.1f TFLOP/s  err=%s\n", name, cyc,
         128.0 * N / 256.0, flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<128, true, 1>("ts N=128 x1/commit");
  run<128, true, 8>("ts N=128 x8/commit");
  run<128, true, 32>("ts N=128 x32/commit");
  run<256, true, 32>("ts N=256 x32/commit");
  run<64, true, 32>("ts N=64 x32/commit");
  run<128, false, 32>("ss N=128 x32/commit");
  run<256, false, 32>("ss N=256 x32/commit");
  return 0;
}
