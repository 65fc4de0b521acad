// Semantics test for tcgen05.mma.cta_group::2 (CTA pair, M = 256, N = 256,
// K = 16, fp16, A and B both in shared memory): each CTA of the pair holds
// 128 rows of A and 128 rows of B at the same shared-memory offsets; the
// leader issues the MMA; each CTA reads its 128 TMEM lanes.  Checks against a
// host GEMM with A = [A_0; A_1], B = [B_0; B_1], D = A B^T.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_00942_b200/csrc \
//        tools/microbench/pair_mma_test.cu -o tools/microbench/pair_mma_test
#include <cstdio>
#include <cmath>
#include <vector>
#include "tc_ptx.cuh"

using namespace rfd;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
pair_kernel(const __half* A, const __half* B, float* D) {
  __shared__ __align__(1024) unsigned char sm[2 * 128 * 16 * 2];  // A rows then B rows (K=16)
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_sh;
  const uint32_t rank = cta_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // canonical K-major, no swizzle: offset(row, k) = (row/8)*256 + (k/8)*128 + (row%8)*16 + (k%8)*2
  for (int e = tid; e < 2 * 128 * 16; e += 128) {
    const int which = e / (128 * 16), rem = e % (128 * 16), row = rem / 16, k = rem % 16;
    const __half v = which == 0 ? A[(rank * 128 + row) * 16 + k] : B[(rank * 128 + row) * 16 + k];
    const int off = which * 128 * 16 * 2 + (row / 8) * 256 + (k / 8) * 128 + (row % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<__half*>(sm + off) = v;
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tc::smem_addr(&tmem_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_sh;
  if (rank == 0 && tid == 0) {
    const uint32_t sa = tc::smem_addr(sm);
    const uint64_t a = tc::make_sdesc(sa, 128, 256);
    const uint64_t b = tc::make_sdesc(sa + 128 * 16 * 2, 128, 256);
    const uint32_t idesc = tc::make_idesc(0, 256, 256);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem), "l"(a), "l"(b), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(tc::smem_addr(&bar)), "h"((unsigned short)3) : "memory");
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  // each warp reads its 32 lanes x 256 columns
  for (int c = 0; c < 256; c += 32) {
    float v[32];
    tc::tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c, v);
    for (int j = 0; j < 32; ++j) D[(rank * 128 + warp * 32 + lane) * 256 + c + j] = v[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  std::vector<__half> hA(256 * 16), hB(256 * 16);
  std::vector<float> fA(256 * 16), fB(256 * 16);
  for (int i = 0; i < 256 * 16; ++i) {
    fA[i] = float((i * 7 + 3) % 17 - 8) / 8.0f;
    fB[i] = float((i * 5 + 1) % 13 - 6) / 4.0f;
    hA[i] = __float2half(fA[i]); hB[i] = __float2half(fB[i]);
  }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dD, 256 * 256 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, 256 * 256 * 4);
  pair_kernel<<<2, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> hD(256 * 256);
  cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int bad = 0;
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < 256; ++j) {
      double ref = 0;
      for (int k = 0; k < 16; ++k) ref += double(fA[i * 16 + k]) * fB[j * 16 + k];
      const double err = fabs(ref - hD[i * 256 + j]);
      if (err > 1e-3 && bad++ < 5) printf("mismatch D[%d][%d] = %f ref %f\n", i, j, hD[i * 256 + j], ref);
      maxerr = fmax(maxerr, err);
    }
  printf("err=%s maxerr=%g bad=%d\n", cudaGetErrorString(e), maxerr, bad);
  return 0;
}
