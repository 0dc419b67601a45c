// Dependent-chain latency (cycles per instruction) of DFMA, FFMA, IMAD.WIDE+add64, LDS on one warp
// (sm_100a). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu
#include <cstdio>
#include <cuda_runtime.h>
#define N 4096
__global__ void k(double* od, float* of, long long* oi, int* os, long long* cyc, double a, float b, int c) {
  __shared__ int sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 3) & 1023;
  __syncthreads();
  double d = a; float f = b; long long acc = c; int p = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) d = fma(d, a, 0.5);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = fmaf(f, b, 0.5f);
  long long t2 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) { long long r; asm volatile("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"((int)acc), "r"(c), "l"(acc)); acc = r; }
  long long t3 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) p = sm[p];
  long long t4 = clock64();
  double dd = d;
#pragma unroll 16
  for (int i = 0; i < N; ++i) { dd = __longlong_as_double(__double_as_longlong(fma(dd, a, 6755399441055744.0)) ); }
  long long t5 = clock64();
  od[threadIdx.x] = d + dd; of[threadIdx.x] = f; oi[threadIdx.x] = acc; os[threadIdx.x] = p;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* od; float* of; long long* oi; int* os; long long* cyc;
  cudaMalloc(&od, 1024 * 8); cudaMalloc(&of, 1024 * 4); cudaMalloc(&oi, 1024 * 8); cudaMalloc(&os, 1024 * 4); cudaMalloc(&cyc, 64);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(od, of, oi, os, cyc, 0.999999, 0.9999f, 3);
  long long h[5]; cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op (1 warp): DFMA %.2f  FFMA %.2f  IMAD.WIDE-acc %.2f  LDS %.2f  DFMA-magic %.2f\n",
         h[0] / (double)N, h[1] / (double)N, h[2] / (double)N, h[3] / (double)N, h[4] / (double)N);
  return 0;
}
