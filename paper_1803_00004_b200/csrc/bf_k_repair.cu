// fp64 repair of ill-conditioned pixels (reading Q27).
//
// The fused kernels flag a pixel when its denominator is small against the clipped spatial
// mass (cond = den / sum K~_s < tau, or den <= 0): there out = num / den amplifies the integer
// format's rounding (relative ~1e-8 of the full-window denominator) by 1 / cond, and the
// fallback decision (den <= 0, Q18) rides on it. This kernel re-evaluates each flagged pixel in
// fp64 from the approximated kernels themselves, the direct double loop of pin P1
//     num(x) = sum_y K~_s(x - y) K~_r(I(x) - I(y)) I(y),   den(x) = sum_y K~_s(x - y) K~_r(I(x) - I(y)),
// K~_r(t) = sum_k a_k cos(pi k t / T) (eq:trigonometric_N_terms), K~_s the lowered
// boxes (eq:Box_N_terms), which equals the box evaluation eq:numerator_2D_box_N_terms
// mathematically. The window is cut into chunks of rows, one CTA per (pixel, chunk):
// fp64 partial sums in a fixed order, rounded to a fixed-point int64 (|error| <= 2^-62 of the
// whole window's absolute mass) and added exactly, so the result is deterministic. f32 inputs
// evaluate K~_r(I(x) - I(y)) from a piecewise degree-13 Taylor table (host-computed, remainder
// < 1e-15 of sum |a_k|; where the table would be too large: fp64 polynomial base angles and the
// Chebyshev recurrence); u8 inputs tabulate K~_r exactly on the 511 integer differences.
#include <algorithm>
#include <atomic>

#include "bf_device.cuh"

namespace bf {

__device__ unsigned g_rep_count[REPAIR_SLOTS];
__device__ unsigned long long g_rep_list[REPAIR_SLOTS][REPAIR_CAP];
__device__ RepAcc g_rep_acc[REPAIR_SLOTS][REPAIR_CAP];

namespace {

constexpr int RT = 256;

// (cos, sin)(pi I / T) in fp64 for I in [0, T]: Taylor polynomials of sin(pi t') / t' and
// cos(pi t') in t' = I / T - 1/2 (truncation < 2e-18), as base_angle_f64 of the fused kernels
__device__ __forceinline__ void angle64(double I, double invT, double& c, double& s) {
  constexpr double kS[11] = {3.14159265358979312e+00, -5.16771278004996937e+00, 2.55016403987734508e+00,
                             -5.99264529320791883e-01, 8.21458866111281910e-02, -7.37043094571434784e-03,
                             4.66302805767612337e-04, -2.19153534478302037e-05, 7.95205400147550838e-07,
                             -2.29484289972698565e-08, 5.39266466260812482e-10};
  constexpr double kC[12] = {1.0, -4.93480220054467900e+00, 4.05871212641676760e+00, -1.33526276885458928e+00,
                             2.35330630358893123e-01, -2.58068913900140508e-02, 1.92957430940392206e-03,
                             -1.04638104924845650e-04, 4.30306958703294391e-06, -1.38789524622137608e-07,
                             3.60473079746249822e-09, -7.70070713060134610e-11};
  const double t = fma(I, invT, -0.5);
  const double z = t * t;
  double p = kS[10];
#pragma unroll
  for (int i = 9; i >= 0; --i) p = fma(p, z, kS[i]);
  double q = kC[11];
#pragma unroll
  for (int i = 10; i >= 0; --i) q = fma(q, z, kC[i]);
  c = -p * t;
  s = q;
}

// K~_r(theta) = sum_i a_i cos(k_i theta) of plan q from x = cos(theta): Chebyshev recurrence
// T_{k+1}(x) = 2 x T_k(x) - T_{k-1}(x) (cos(k theta) = T_k(cos theta)), exact to fp64 rounding
__device__ __forceinline__ double range_cheb(const RParams& R, int q, double x) {
  const double x2 = x + x;
  double tp = x, tc = 1.0, acc = 0.0;   // T_{-1} = T_1 = x (cos is even), T_0 = 1
  int kk = 0;
  const int n = R.nkp[q];
  for (int i = 0; i < n; ++i) {
    const int ki = R.k[q][i];
    for (; kk < ki; ++kk) {
      const double tn = fma(x2, tc, -tp);
      tp = tc;
      tc = tn;
    }
    acc = fma(R.a[q][i], tc, acc);
  }
  return acc;
}

// One CTA per (flagged pixel, chunk of window rows): the chunk's partial num / den of the direct
// double loop in fp64 (fixed tap order, fixed reduction tree), rounded to fixed point and added
// to the pixel's exact int64 accumulators; the chunk that arrives last finishes the pixel. The
// result does not depend on the order in which chunks run (integer additions).
__global__ void __launch_bounds__(RT) bf_repair_kernel(const RParams R, const void* __restrict__ in,
                                                       float* __restrict__ out) {
  extern __shared__ double sm[];
  const int n1 = 2 * R.rad + 1;
  double* fx = sm;                   // [ns][n1]: fx_s(u), u = -rad..rad
  double* fy = sm + R.ns * n1;       // [ns][n1]
  double* klut = sm + 2 * R.ns * n1; // [511] K~_r(t), t = -255..255 (u8), or the Taylor table (f32)
  __shared__ double red[2][RT / 32];
  __shared__ int last;
  const int tid = threadIdx.x;
  // nothing flagged (the common case), or more CTAs than (pixel, chunk) items: leave before the
  // table fills
  const unsigned n = min(*R.count, R.cap);
  if ((unsigned long long)blockIdx.x >= (unsigned long long)n * (unsigned)R.nch) return;
  for (int i = tid; i < R.ns * n1; i += RT) {
    const int s = i / n1, o = i % n1 - R.rad;
    double wx = 0.0, wy = 0.0;
    for (int b = 0; b < R.nbx[s]; ++b)
      if (o >= R.lox[s][b] && o <= R.hix[s][b]) wx += R.wx[s][b];
    for (int b = 0; b < R.nby[s]; ++b)
      if (o >= R.loy[s][b] && o <= R.hiy[s][b]) wy += R.wy[s][b];
    fx[i] = wx;
    fy[i] = wy;
  }
  if (R.repaired && blockIdx.x == 0 && tid == 0 && n) atomicAdd(R.repaired, (unsigned long long)n);
  const double invT = 1.0 / R.T;
  for (int i = tid; i < R.ntab * (REP_DEG + 1); i += RT) klut[i] = R.tab[i];
  const double inv2h = R.ntab ? 0.5 / R.tab_h : 0.0;
  int lut_q = -1;
  const unsigned long long items = (unsigned long long)n * (unsigned)R.nch;
  for (unsigned long long it = blockIdx.x; it < items; it += gridDim.x) {
    const unsigned pi = (unsigned)(it / (unsigned)R.nch);
    const int chunk = (int)(it - (unsigned long long)pi * (unsigned)R.nch);
    const unsigned long long e = R.list[pi];
    const int q = R.nplans > 1 ? (int)(e / (unsigned long long)R.plan_stride) : 0;
    const long long pix = (long long)(e - (unsigned long long)q * (unsigned long long)R.plan_stride);
    const long long f = pix / R.frame_elems;
    const long long rem = pix - f * R.frame_elems;
    const int y = (int)(rem / R.W), x = (int)(rem % R.W);
    const long long fbase = f * R.frame_elems;
    __syncthreads();   // (previous item's table / reduction done)
    if (R.u8 && lut_q != q) {
      for (int t = tid; t < 511; t += RT) {
        double c, s;
        sincospi((double)(t - 255) * invT, &s, &c);
        klut[t] = range_cheb(R, q, c);
      }
      lut_q = q;
    }
    __syncthreads();
    const double Ix = R.u8 ? (double)reinterpret_cast<const unsigned char*>(in)[pix]
                           : (double)reinterpret_cast<const float*>(in)[pix];
    double cx = 0.0, sx = 0.0;
    if (!R.u8) angle64(Ix, invT, cx, sx);
    const int v0 = -R.rad + chunk * R.rpc, v1 = min(R.rad, v0 + R.rpc - 1);
    const int ya = max(0, y + v0), yb = min(R.H - 1, y + v1);
    const int xa = max(0, x - R.rad), xb = min(R.W - 1, x + R.rad);
    double num = 0.0, den = 0.0;
    for (int row = ya; row <= yb; ++row) {
      const int v = row - y + R.rad;
      const double fy0 = fy[v], fy1 = R.ns > 1 ? fy[n1 + v] : 0.0;
      bool any = fy0 != 0.0 || fy1 != 0.0;
      for (int s = 2; s < R.ns && !any; ++s) any = fy[s * n1 + v] != 0.0;
      if (!any) continue;
      const long long rbase = fbase + (long long)row * R.W;
      for (int col = xa + tid; col <= xb; col += RT) {
        const int u = col - x + R.rad;
        double ks = R.ns > 1 ? fma(fx[n1 + u], fy1, fx[u] * fy0) : fx[u] * fy0;
        for (int s = 2; s < R.ns; ++s) ks = fma(fx[s * n1 + u], fy[s * n1 + v], ks);
        if (ks == 0.0) continue;
        double Iy, kr;
        if (R.u8) {
          const int iy = reinterpret_cast<const unsigned char*>(in)[rbase + col];
          Iy = (double)iy;
          kr = klut[(int)Ix - iy + 255];
        } else {
          Iy = (double)__ldg(reinterpret_cast<const float*>(in) + rbase + col);
          if (R.ntab) {   // Taylor polynomial of the interval holding |Ix - Iy|
            const double t = fabs(Ix - Iy);
            const int i = min((int)(t * inv2h), R.ntab - 1);
            const double s = t - (2 * i + 1) * R.tab_h;
            const double* c = klut + i * (REP_DEG + 1);
            kr = c[REP_DEG];
#pragma unroll
            for (int m = REP_DEG - 1; m >= 0; --m) kr = fma(kr, s, c[m]);
          } else {
            double cy, sy;
            angle64(Iy, invT, cy, sy);
            kr = range_cheb(R, q, fma(cx, cy, sx * sy));   // cos(pi (Ix - Iy) / T)
          }
        }
        const double w = ks * kr;
        den += w;
        num = fma(w, Iy, num);
      }
    }
    // fixed-order block reduction
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = num;
      red[1][tid >> 5] = den;
    }
    __syncthreads();
    if (tid == 0) {
      double sn = 0.0, sd = 0.0;
      for (int w = 0; w < RT / 32; ++w) {
        sn += red[0][w];
        sd += red[1][w];
      }
      RepAcc* A = R.acc + pi;
      atomicAdd(reinterpret_cast<unsigned long long*>(&A->num), (unsigned long long)__double2ll_rn(sn * R.qscale));
      atomicAdd(reinterpret_cast<unsigned long long*>(&A->den), (unsigned long long)__double2ll_rn(sd * R.qscale));
      __threadfence();
      last = atomicAdd(&A->arrived, 1u) == (unsigned)R.nch - 1;
    }
    __syncthreads();
    if (last && tid == 0) {
      __threadfence();
      const RepAcc* A = R.acc + pi;
      const long long qn = atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<long long*>(&A->num)), 0ull);
      const long long qd = atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<long long*>(&A->den)), 0ull);
      const bool fb = !(qd > 0);
      out[e] = fb ? (float)Ix : (float)((double)qn / (double)qd);
      if (R.fb_mask) R.fb_mask[e] = fb ? 1 : 0;
      if (fb && R.fb_count) atomicAdd(R.fb_count, 1ULL);
    }
  }
}

}  // namespace

cudaError_t repair_slot(unsigned s, unsigned** count, unsigned long long** list, RepAcc** acc) {
  // symbol addresses per device, looked up once (no runtime query inside a stream capture later)
  static std::atomic<void*> cache_c[64], cache_l[64], cache_a[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  void* c = dev < 64 ? cache_c[dev].load() : nullptr;
  void* l = dev < 64 ? cache_l[dev].load() : nullptr;
  void* a = dev < 64 ? cache_a[dev].load() : nullptr;
  if (!c || !l || !a) {
    e = cudaGetSymbolAddress(&c, g_rep_count);
    if (e == cudaSuccess) e = cudaGetSymbolAddress(&l, g_rep_list);
    if (e == cudaSuccess) e = cudaGetSymbolAddress(&a, g_rep_acc);
    if (e != cudaSuccess) return e;
    if (dev < 64) {
      cache_c[dev].store(c);
      cache_l[dev].store(l);
      cache_a[dev].store(a);
    }
  }
  *count = static_cast<unsigned*>(c) + s;
  *list = static_cast<unsigned long long*>(l) + (size_t)s * REPAIR_CAP;
  *acc = static_cast<RepAcc*>(a) + (size_t)s * REPAIR_CAP;
  return cudaSuccess;
}

cudaError_t launch_repair(const RParams& R, const void* in, float* out, cudaStream_t st) {
  const size_t smem =
      sizeof(double) * (2 * (size_t)R.ns * (2 * (size_t)R.rad + 1) + std::max(512, R.ntab * (REP_DEG + 1)));
  cudaError_t e = cudaFuncSetAttribute(bf_repair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  bf_repair_kernel<<<4 * std::max(1, nsm), RT, smem, st>>>(R, in, out);
  return cudaGetLastError();
}

}  // namespace bf
