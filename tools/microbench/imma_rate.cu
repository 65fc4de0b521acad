// Microbenchmark: legacy mma.sync throughput per SM on sm_100a for the
// integer (m16n8k32 u8 x u8 -> s32) and f16 (m16n8k16 f16 -> f32) shapes,
// register operands only (the spread-grid candidates).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/imma_rate.cu -o /tmp/imma_rate
#include <cstdio>

__global__ void ki8(int iters, int* out, long long* cyc) {
  unsigned a0 = threadIdx.x * 0x01010101u, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = 0x02020202u + threadIdx.x, b1 = b0 + 5;
  int d[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) d[i][j] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[i][0]), "+r"(d[i][1]), "+r"(d[i][2]), "+r"(d[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  int s = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void kf16(int iters, int* out, long long* cyc) {
  unsigned a0 = 0x3c003c00u + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = 0x3c003c00u, b1 = b0 + 5;
  float d[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) d[i][j] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = int(s);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  for (int warps : {4, 8, 16}) {
    const int iters = 2000;
    long long h;
    ki8<<<148, 32 * warps>>>(10, o, c);
    ki8<<<148, 32 * warps>>>(iters, o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double mac = double(iters) * 8 * 4096 * warps;  // m16n8k32 = 4096 MAC
    printf("u8  m16n8k32 warps %2d: %7.1f MAC/clk/SM  %s\n", warps, mac / h, cudaGetErrorString(cudaGetLastError()));
    kf16<<<148, 32 * warps>>>(10, o, c);
    kf16<<<148, 32 * warps>>>(iters, o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    mac = double(iters) * 8 * 2048 * warps;  // m16n8k16 = 2048 MAC
    printf("f16 m16n8k16 warps %2d: %7.1f MAC/clk/SM  %s\n", warps, mac / h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
