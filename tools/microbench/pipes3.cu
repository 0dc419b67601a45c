// IMAD.WIDE, F2I.S32, I2FP throughput with independent chains that cannot be folded.
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
#define ITERS 512
template <int OP>
__global__ void __launch_bounds__(1024) kern(long long* out, long long* cyc, int seed) {
  long long acc[CH]; int x[CH]; float f[CH];
  int lane = threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc[c] = c; x[c] = (lane * 7 + c * 13 + seed) | 1; f[c] = 1.5f + c + lane * 1e-3f; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      if (OP == 0) { acc[c] += (long long)x[c] * (long long)(x[(c + 1) % CH]); x[c] += (int)acc[c]; }     // IMAD.WIDE + IADD
      if (OP == 1) { x[c] = __float2int_rn(f[c] * 1000.f) ^ x[c]; f[c] = __int_as_float((x[c] & 0x3FFFFF) | 0x3F800000); } // F2I + LOP + FMUL
      if (OP == 2) { f[c] = (float)x[c] * 1.0001f; x[c] = __float_as_int(f[c]) ^ (c + it); }    // I2FP + FMUL + LOP
      if (OP == 3) { acc[c] += (long long)x[c] * 12345LL; x[c] += 3; }                           // IMAD.WIDE by const
    }
  }
  long long t1 = clock64();
  long long s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += acc[c] + x[c] + (long long)f[c];
  if (s == 42) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* nm, long long* o, long long* cy, int nsm) {
  kern<OP><<<nsm, 1024>>>(o, cy, 3); cudaDeviceSynchronize();
  kern<OP><<<nsm, 1024>>>(o, cy, 3); cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, cy, nsm * 8, cudaMemcpyDeviceToHost); long long mx = 0;
  for (int i = 0; i < nsm; i++) mx = h[i] > mx ? h[i] : mx;
  printf("%-28s %8.2f ops/clk/SM (per op = one chain step)\n", nm, 1024.0 * ITERS * CH / mx);
}
int main() { int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *o, *cy; cudaMalloc(&o, 8192); cudaMalloc(&cy, 4096);
  run<0>("IMAD.WIDE+IADD (x*y)", o, cy, nsm); run<3>("IMAD.WIDE by const+IADD", o, cy, nsm);
  run<1>("F2I+LOP+LOP+FMUL", o, cy, nsm); run<2>("I2FP+FMUL+LOP", o, cy, nsm); }
