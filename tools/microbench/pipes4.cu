// Shared-memory / conversion / wide-multiply throughput on the B200 (sm_100a), with addresses
// that change every iteration (nothing hoistable). One 1024-thread CTA per SM, 8 independent
// chains per thread; reports per-SM rates from clock64().
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
#define ITERS 256
template <int OP>
__global__ void __launch_bounds__(1024) kern(int* out, long long* cyc, int seed) {
  __shared__ __align__(16) int sm[12288];
  for (int i = threadIdx.x; i < 12288; i += blockDim.x) sm[i] = (i * 7 + seed) & 1023;
  __syncthreads();
  int x[CH]; long long w[CH]; float f[CH];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < CH; c++) { x[c] = lane + c; w[c] = c; f[c] = 1.f + c * 0.25f + lane * 1e-3f; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    const int rot = (it * 37 + wp * 64) & 4095;
#pragma unroll
    for (int c = 0; c < CH; c++) {
      if (OP == 0) x[c] += sm[(rot + c * 128 + lane) & 8191];                                  // LDS.32
      if (OP == 1) { int2 v = reinterpret_cast<int2*>(sm)[((rot >> 1) + c * 64 + lane) & 4095]; x[c] += v.x ^ v.y; }   // LDS.64
      if (OP == 2) { int4 v = reinterpret_cast<int4*>(sm)[((rot >> 2) + c * 32 + lane) & 2047]; x[c] += (v.x ^ v.y) + (v.z ^ v.w); } // LDS.128
      if (OP == 3) { sm[(rot + c * 128 + lane) & 8191] = x[c]; x[c] += 3; }                    // STS.32
      if (OP == 4) { reinterpret_cast<int4*>(sm)[((rot >> 2) + c * 32 + lane) & 2047] = make_int4(x[c], x[c] + 1, x[c] + 2, x[c] + 3); x[c] += 5; } // STS.128
      if (OP == 5) w[c] += (long long)x[c] * (long long)(x[(c + 3) % CH] | 1);                 // IMAD.WIDE (indep.)
      if (OP == 6) { x[c] = __float2int_rn(f[c] * 1000.f) + x[c]; f[c] += 1.0f; }              // F2I (+FMUL/IADD/FADD)
      if (OP == 7) { x[c] += sm[(rot + c * 128 + lane) & 8191]; f[c] = fmaf(f[c], 0.999f, 0.001f); f[c] = fmaf(f[c], 0.999f, 0.001f); f[c] = fmaf(f[c], 0.999f, 0.001f); f[c] = fmaf(f[c], 0.999f, 0.001f); } // LDS + 4 FFMA
      if (OP == 8) x[c] += sm[(rot * 33 + c * 129 + lane * 33) & 8191];                        // LDS.32 stride-33 (conflict-free)
      if (OP == 9) w[c] += (long long)__umulhi((unsigned)x[c], 0x9E3779B9u + c);              // IMAD.HI
    }
  }
  long long t1 = clock64();
  long long acc = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) acc += x[c] + w[c] + (long long)f[c];
  if (acc == 123456789) out[threadIdx.x] = (int)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
void run(const char* name, int* dout, long long* dcyc, int nsm, double per) {
  kern<OP><<<nsm, 1024>>>(dout, dcyc, 3);
  cudaDeviceSynchronize();
  kern<OP><<<nsm, 1024>>>(dout, dcyc, 3);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nsm; i++) mx = h[i] > mx ? h[i] : mx;
  printf("%-26s %8.2f per clk/SM\n", name, 1024.0 * ITERS * CH * per / mx);
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
}
int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* dout; long long* dcyc;
  cudaMalloc(&dout, 4096 * 4); cudaMalloc(&dcyc, 256 * 8);
  run<0>("LDS.32 (words)", dout, dcyc, nsm, 1);
  run<1>("LDS.64 (words)", dout, dcyc, nsm, 2);
  run<2>("LDS.128 (words)", dout, dcyc, nsm, 4);
  run<8>("LDS.32 stride33 (words)", dout, dcyc, nsm, 1);
  run<3>("STS.32 (words)", dout, dcyc, nsm, 1);
  run<4>("STS.128 (words)", dout, dcyc, nsm, 4);
  run<5>("IMAD.WIDE (ops)", dout, dcyc, nsm, 1);
  run<9>("IMAD.HI (ops)", dout, dcyc, nsm, 1);
  run<6>("F2I (ops)", dout, dcyc, nsm, 1);
  run<7>("LDS.32 + 4 FFMA (LDS)", dout, dcyc, nsm, 1);
  return 0;
}
