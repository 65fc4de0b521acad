// Microbenchmark: fp64 tensor-core (DMMA) throughput per SM on sm_100a:
// mma.sync m8n8k4 and m16n8k16 f64, register operands only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/dmma_rate.cu -o /tmp/dmma_rate
#include <cstdio>

__global__ void k8(int iters, double* out, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[8][2];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k16(int iters, double* out, long long* cyc) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
  double d[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) d[i][j] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                     "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 148 * 8);
  for (int warps : {4, 8, 16}) {
    const int iters = 2000;
    k8<<<148, 32 * warps>>>(10, o, c);
    k8<<<148, 32 * warps>>>(iters, o, c);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double fma = double(iters) * 8 * 256 * warps;  // m8n8k4 = 256 FMA per warp-instr
    printf("m8n8k4   warps %2d: %6.1f FMA/clk/SM  (%.1f TFLOP/s at 1.9 GHz)  %s\n", warps, fma / h,
           fma / h * 2 * 148 * 1.9e9 / 1e12, cudaGetErrorString(cudaGetLastError()));
    k16<<<148, 32 * warps>>>(10, o, c);
    k16<<<148, 32 * warps>>>(iters, o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    fma = double(iters) * 4 * 2048 * warps;  // m16n8k16 = 2048 FMA
    printf("m16n8k16 warps %2d: %6.1f FMA/clk/SM  (%.1f TFLOP/s at 1.9 GHz)  %s\n", warps, fma / h,
           fma / h * 2 * 148 * 1.9e9 / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
