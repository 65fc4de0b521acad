// Microbenchmark: per-SM throughput of the instructions the feature pipeline
// uses (MUFU.SIN, F2FP fp32->fp16x2 pack, HADD2.F32 unpack, FFMA, FFMA2,
// LOP3): 16 warps per SM, 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/microbench/pipe_rates.cu -o /tmp/pipe_rates
#include <cstdio>
#include <cuda_fp16.h>

template <int K>
__global__ void __launch_bounds__(512) bench(int iters, float seed, float* out, long long* cyc) {
  float a[8];
  unsigned u[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = seed + threadIdx.x * 1e-3f + j; u[j] = __float_as_uint(a[j]); }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (K == 0) a[j] = __sinf(a[j]);
      if (K == 1) {  // F2FP pack and back (pack + unpack chain)
        __half2 h = __floats2half2_rn(a[j], a[(j + 1) & 7]);
        a[j] = __low2float(h) + 1e-3f;
      }
      if (K == 2) a[j] = fmaf(a[j], 1.0001f, 1e-7f);
      if (K == 3) {
        float2 v = __ffma2_rn(make_float2(a[j], a[(j + 4) & 7]), make_float2(1.0001f, 1.0001f),
                              make_float2(1e-7f, 1e-7f));
        a[j] = v.x; a[(j + 4) & 7] = v.y;
      }
      if (K == 4) u[j] = (u[j] & 0xFFFFE000u) ^ (u[j] >> 3);
      if (K == 5) {  // F2FP only (pack), consumed as integer
        __half2 h = __floats2half2_rn(a[j], a[j]);
        u[j] ^= *reinterpret_cast<unsigned*>(&h);
        a[j] += 1e-3f;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j] + __uint_as_float(u[j]);
  out[blockIdx.x * 512 + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(const char* name, int ops_per_inner) {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  const int iters = 4096;
  bench<K><<<148, 512>>>(16, 1.0f, o, c);
  bench<K><<<148, 512>>>(iters, 1.0f, o, c);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double thread_ops = double(iters) * 8 * ops_per_inner * 512;
  printf("%-28s %7.1f thread-ops/clk/SM  err=%s\n", name, thread_ops / double(h),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("MUFU.SIN (+FMUL.RZ)", 1);
  run<1>("F2FP pack + unpack + FADD", 1);
  run<5>("F2FP pack + LOP + FADD", 1);
  run<2>("FFMA", 1);
  run<3>("FFMA2 (2 FMA each)", 1);
  run<4>("LOP3+SHF", 1);
  return 0;
}
