// Second pipe microbenchmark: dependent-index LDS (not hoistable), LDS+SHFL concurrency,
// REDUX.SUM, IMAD.WIDE, IADD3+FFMA2 dual issue.
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
#define ITERS 256
template <int OP>
__global__ void __launch_bounds__(1024) kern(int* out, long long* cyc, int seed) {
  __shared__ int sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (i * 7 + seed) & 31;
  __syncthreads();
  int x[CH]; long long w[CH]; unsigned long long p[CH];
  int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < CH; c++) { x[c] = (lane + c) & 31; w[c] = c; float2 t = make_float2(1.f + c, 2.f); p[c] = *reinterpret_cast<unsigned long long*>(&t); }
  float2 a2f = make_float2(0.999f, 0.999f), b2f = make_float2(0.001f, 0.001f);
  unsigned long long a2 = *reinterpret_cast<unsigned long long*>(&a2f), b2 = *reinterpret_cast<unsigned long long*>(&b2f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
#pragma unroll
      for (int c = 0; c < CH; c++) {
        int base = ((wp * 8 + c) & 63) * 128;
        if (OP == 0) x[c] = sm[base + ((x[c] + lane) & 31)];                  // LDS.32 dependent
        if (OP == 1) { int4 v = reinterpret_cast<int4*>(sm)[(base >> 2) + ((x[c] + lane) & 31)]; x[c] = (v.x + v.y + v.z + v.w) & 31; } // LDS.128 dependent (+3 IADD)
        if (OP == 2) { if (c & 1) x[c] = sm[base + ((x[c] + lane) & 31)]; else x[c] = __shfl_sync(0xffffffffu, x[c], (lane + 1) & 31); } // LDS + SHFL mix
        if (OP == 3) x[c] = __reduce_add_sync(0xffffffffu, x[c] + c) & 31;    // REDUX.SUM
        if (OP == 4) w[c] = (long long)x[c] * (long long)(c + 12345) + w[c];   // IMAD.WIDE
        if (OP == 5) { x[c] = x[c] + lane - c; asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(a2), "l"(b2)); } // IADD3 + FFMA2
        if (OP == 6) { sm[base + ((x[c] + lane + it) & 127)] = x[c]; x[c] += lane; } // STS (+IADD)
      }
    }
  }
  long long t1 = clock64();
  int acc = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc += x[c] + (int)w[c] + (int)(p[c] >> 7); }
  if (acc == 123456789) out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
void run(const char* name, int* dout, long long* dcyc, int nsm, double per) {
  kern<OP><<<nsm, 1024>>>(dout, dcyc, 3);
  cudaDeviceSynchronize();
  kern<OP><<<nsm, 1024>>>(dout, dcyc, 3);
  cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < nsm; i++) mx = h[i] > mx ? h[i] : mx;
  printf("%-22s %8.2f per clk/SM  (%lld cyc)\n", name, 1024.0 * ITERS * 4 * CH * per / mx, mx);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* dout; long long* dcyc; cudaMalloc(&dout, 4096 * 4); cudaMalloc(&dcyc, 256 * 8);
  run<0>("LDS.32 dep (lanes)", dout, dcyc, nsm, 1);
  run<1>("LDS.128 dep (words)", dout, dcyc, nsm, 4);
  run<2>("LDS+SHFL mix (lanes)", dout, dcyc, nsm, 1);
  run<3>("REDUX.SUM (lanes)", dout, dcyc, nsm, 1);
  run<4>("IMAD.WIDE (lanes)", dout, dcyc, nsm, 1);
  run<5>("IADD3+FFMA2 (pairs)", dout, dcyc, nsm, 1);
  run<6>("STS.32 (+IADD)", dout, dcyc, nsm, 1);
  return 0;
}
