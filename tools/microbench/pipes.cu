// Pipe-throughput microbenchmark for the B200 (sm_100a): measures lane-ops per SM clock
// for the instruction mix the bilateral-filter kernel design depends on.
// Each thread runs CH independent dependency chains so latency is hidden; cycles are
// read with clock64() per block (one 1024-thread block per SM, grid = #SMs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 256

template <int OP>
__global__ void __launch_bounds__(1024) kern(float* out, long long* cyc, float seed) {
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = seed + i;
  __syncthreads();
  float f[CH]; double d[CH]; int x[CH]; unsigned long long p[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) { f[c] = seed * (c + 1) + threadIdx.x; d[c] = f[c]; x[c] = threadIdx.x * (c + 3);
    float2 t = make_float2(f[c], f[c] + 1.f); p[c] = *reinterpret_cast<unsigned long long*>(&t); }
  const float a = seed * 0.999f, b = seed * 0.001f;
  const double da = a, db = b;
  float2 a2f = make_float2(a, a), b2f = make_float2(b, b);
  unsigned long long a2 = *reinterpret_cast<unsigned long long*>(&a2f), b2 = *reinterpret_cast<unsigned long long*>(&b2f);
  int lane = threadIdx.x & 31;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
#pragma unroll
      for (int c = 0; c < CH; c++) {
        if (OP == 0) f[c] = fmaf(f[c], a, b);                       // FFMA
        if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(a2), "l"(b2));  // FFMA2
        if (OP == 2) f[c] = f[c] + b;                              // FADD
        if (OP == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(b2));   // FADD2
        if (OP == 4) d[c] = d[c] + db;                             // DADD
        if (OP == 5) d[c] = fma(d[c], da, db);                     // DFMA
        if (OP == 6) { double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[c])); f[c] = __int_as_float(__double2hiint(t) ^ c); } // F2F.F64.F32 (+LOP)
        if (OP == 7) { float t; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(t) : "d"(d[c])); d[c] = __hiloint2double(__float_as_int(t), c); } // F2F.F32.F64
        if (OP == 8) { float t; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(t) : "r"(x[c])); x[c] = __float_as_int(t) ^ c; } // I2F
        if (OP == 9) x[c] = x[c] + x[(c + 1) % CH] - c;           // IADD3
        if (OP == 10) f[c] += sm[(lane + (int)f[c] * 0 + c * 32 + u * 256) & 4095];   // LDS.32 (+FADD)
        if (OP == 11) { float4 v = reinterpret_cast<float4*>(sm)[((lane + c * 32 + u * 256) & 1023)]; f[c] += v.x + v.y + v.z + v.w; } // LDS.128
        if (OP == 12) f[c] = __shfl_xor_sync(0xffffffffu, f[c], 1 + c % 31);   // SHFL
        if (OP == 13) { double t; asm volatile("cvt.rn.f64.s32 %0, %1;" : "=d"(t) : "r"(x[c])); x[c] = __double2hiint(t) ^ c; } // I2F.F64
        if (OP == 14) x[c] = x[c] * 3 + c;                          // IMAD
        if (OP == 15) f[c] = __fmul_rn(f[c], a);                    // FMUL
        if (OP == 16) { float s_, c_; sincospif(f[c] * 1e-3f, &s_, &c_); f[c] = s_ + c_; } // sincospif
        if (OP == 17) { sm[(lane + c * 32 + u * 256 + (it & 7) * 128) & 4095] = f[c]; f[c] += b; } // STS.32 (+FADD)
        if (OP == 18) f[c] = __fadd_rn(f[c], __int_as_float(x[c]));   // placeholder
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc += f[c] + (float)d[c] + (float)x[c]; float2 t = *reinterpret_cast<float2*>(&p[c]); acc += t.x + t.y; }
  acc += sm[threadIdx.x];
  if (acc == 1234.5f) out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, float* dout, long long* dcyc, int nsm, double ops_per_iter_lane) {
  kern<OP><<<nsm, 1024>>>(dout, dcyc, 1.0001f);
  cudaEventRecord(0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<nsm, 1024>>>(dout, dcyc, 1.0001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024]; cudaMemcpy(h, dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < nsm; i++) mx = h[i] > mx ? h[i] : mx;
  double lane_ops = 1024.0 * ITERS * 4 * CH * ops_per_iter_lane;
  printf("%-14s %8.2f lane-ops/clk/SM   (%lld cyc, %.3f ms, implied SM clk %.0f MHz)\n", name, lane_ops / mx, mx, ms, mx / (ms * 1e3));
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* dout; long long* dcyc; cudaMalloc(&dout, 4096 * 4); cudaMalloc(&dcyc, 1024 * 8);
  printf("SMs %d\n", nsm);
  run<0>("FFMA", dout, dcyc, nsm, 1);
  run<1>("FFMA2(x2)", dout, dcyc, nsm, 2);
  run<2>("FADD", dout, dcyc, nsm, 1);
  run<3>("FADD2(x2)", dout, dcyc, nsm, 2);
  run<15>("FMUL", dout, dcyc, nsm, 1);
  run<4>("DADD", dout, dcyc, nsm, 1);
  run<5>("DFMA", dout, dcyc, nsm, 1);
  run<6>("F2F.F64.F32", dout, dcyc, nsm, 1);
  run<7>("F2F.F32.F64", dout, dcyc, nsm, 1);
  run<8>("I2F.F32", dout, dcyc, nsm, 1);
  run<13>("I2F.F64", dout, dcyc, nsm, 1);
  run<9>("IADD3", dout, dcyc, nsm, 1);
  run<14>("IMAD", dout, dcyc, nsm, 1);
  run<10>("LDS32(+FADD)", dout, dcyc, nsm, 1);
  run<11>("LDS128(vals)", dout, dcyc, nsm, 4);
  run<17>("STS32(+FADD)", dout, dcyc, nsm, 1);
  run<12>("SHFL", dout, dcyc, nsm, 1);
  run<16>("sincospif", dout, dcyc, nsm, 1);
  return 0;
}
