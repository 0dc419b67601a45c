// Fused sm_100a kernel of the joint-acceleration bilateral filter (bf_apply).
//
// Evaluates eq:numerator_2D_box_N_terms with T = D (Q1): for every selected
// cosine term k the four channels g^c_k, g^s_k, G^c_k = I g^c_k, G^s_k = I g^s_k are
// generated in registers, box-filtered with the separable Haar-box kernel
// K~_s(u, v) = fx(u) fy(v) (eq:2D_box_N_terms_s, Appendix A), and recombined with
// a_k g^c_k(x), a_k g^s_k(x); out = num / den (eq:BF).
//
// Layout of one CTA: a vertical strip of TW output columns plus the horizontal halo
// (NTC = blockDim.x extended columns, one thread per column) and a band of TH output rows.
// Per output row:
//   V  each thread slides the vertical box sums of all channels of its column down one row:
//      channels at the entering / leaving rows of every box are regenerated from I (rotation
//      recurrence from an accurately reduced base angle) and quantised to 22-bit fixed point
//      with one FFMA (x*s + 1.5*2^23), so the sliding sums are EXACT int32 arithmetic with no
//      drift; U = sum_b wy_b S_b is re-quantised and written to shared memory.
//   H  walker threads (channel, segment) slide the horizontal box sums of U along the row in
//      exact int32 arithmetic and write F = sum_b wx_b H_b (fp32) to shared memory.
//   C  one thread per output pixel regenerates its weights a_k cos/sin(pi k I(x)/D) and
//      accumulates num / den (fp32 products, fp64 accumulation per group of k), then divides.
// Nothing but the input image and the output image touches HBM.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "bf_internal.h"

namespace {

constexpr int QMAX = (1 << 22) - 1;       // |quantised value| <= QMAX
constexpr float MAGIC = 12582912.0f;      // 1.5 * 2^23
constexpr int MAGIC_BITS = 0x4B400000;    // bit pattern of MAGIC
constexpr int MAXB = 2;                   // boxes per axis on the GPU path (N_s = 1 or 9)

struct KParams {
  int H, W;
  int nk;                   // cosine terms handled by this launch
  int kstep[BF_MAX_TERMS];  // rotation steps from the previous term (first: from k = 0)
  float a[BF_MAX_TERMS];    // a_k
  int k0;                   // k of the term before the first one of this launch (0 for pass 0)
  int nbx, nby;
  int lox[MAXB], hix[MAXB], loy[MAXB], hiy[MAXB];
  float wx[MAXB], wy[MAXB];
  int rlo_x;                // -min lox (left halo)
  int TW, TH;               // output strip width / band height
  float invD_hi, invD_lo;   // 1/D as a float-float pair
  float qD;                 // QMAX / D
  float uscale;             // QMAX / U_bound
  float D;
  int pass;                 // 0 = only pass; 1 = first; 2 = middle; 3 = last
  long long frame_elems;    // H * W (batched frames)
};

__device__ __forceinline__ float load_pixel(const void* in, bool u8, long long idx) {
  if (u8) return (float)__ldg(reinterpret_cast<const unsigned char*>(in) + idx);
  return __ldg(reinterpret_cast<const float*>(in) + idx);
}

// cos(pi I / D), sin(pi I / D) with I/D carried as a float-float pair and a first-order
// correction for its low part (the naive fp32 phase fails the tolerance).
__device__ __forceinline__ void base_angle(float I, const KParams& P, float& c1, float& s1) {
  float t = I * P.invD_hi;
  float e = fmaf(I, P.invD_hi, -t) + I * P.invD_lo;
  float s, c;
  sincospif(t, &s, &c);
  float pe = 3.14159265358979323846f * e;
  c1 = fmaf(-s, pe, c);
  s1 = fmaf(c, pe, s);
}

__device__ __forceinline__ void rotate(float& c, float& s, float c1, float s1) {
  float cn = fmaf(c, c1, -s * s1);
  float sn = fmaf(s, c1, c * s1);
  c = cn;
  s = sn;
}

__device__ __forceinline__ int qbits(float x, float scale) { return __float_as_int(fmaf(x, scale, MAGIC)); }

// Per-tap state: base angle, scales (0 for pixels outside the image, Q16) and the current
// (cos, sin) of the rotation recurrence.
struct Tap {
  float c1, s1, sc1, scD, c, s;
};

template <bool U8>
__device__ __forceinline__ Tap make_tap(const void* in, const KParams& P, const float2* lut, int row, int col,
                                        long long fbase) {
  Tap t;
  bool valid = (row >= 0) & (row < P.H) & (col >= 0) & (col < P.W);
  float I = 0.f;
  if (valid) I = load_pixel(in, U8, fbase + (long long)row * P.W + col);
  if (U8) {
    float2 v = lut[(int)I];
    t.c1 = v.x;
    t.s1 = v.y;
  } else {
    base_angle(I, P, t.c1, t.s1);
  }
  t.sc1 = valid ? (float)QMAX : 0.f;
  t.scD = valid ? I * P.qD : 0.f;
  t.c = 1.f;
  t.s = 0.f;
  for (int j = 0; j < P.k0; ++j) rotate(t.c, t.s, t.c1, t.s1);
  return t;
}

template <int MAXK, bool U8, int NT>
__global__ void __launch_bounds__(NT, 1) bf_strip_kernel(const KParams P, const void* __restrict__ in,
                                                         float* __restrict__ out, double2* __restrict__ ws) {
  constexpr int C = 4 * MAXK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int NTC = NT;
  const int UPITCH = NTC + 1;
  const int FPITCH = P.TW + 1;
  int* Ubuf = reinterpret_cast<int*>(smem_raw);                       // [C][UPITCH]
  float* Fbuf = reinterpret_cast<float*>(Ubuf + C * UPITCH);          // [C][FPITCH]
  float2* lut = reinterpret_cast<float2*>(Fbuf + C * FPITCH);         // [256] (u8 only)

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P.TW;
  const int y0 = blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int col = x0 - P.rlo_x + tid;
  const int nch = 4 * P.nk;
  const int TWv = min(P.TW, P.W - x0);
  const int yend = min(y0 + P.TH, P.H);

  if (U8) {
    for (int i = tid; i < 256; i += NT) {
      double s, c;
      sincospi((double)i / (double)P.D, &s, &c);
      lut[i] = make_float2((float)c, (float)s);
    }
    __syncthreads();
  }

  // ---- vertical state: exact int32 box sums of every channel, per box of fy
  int S[MAXB][C];
#pragma unroll
  for (int b = 0; b < MAXB; ++b)
#pragma unroll
    for (int ch = 0; ch < C; ++ch) S[b][ch] = 0;

  {
    int rmin = P.loy[0], rmax = P.hiy[0];
    for (int b = 1; b < P.nby; ++b) {
      rmin = min(rmin, P.loy[b]);
      rmax = max(rmax, P.hiy[b]);
    }
    for (int v = rmin; v <= rmax; ++v) {
      Tap t = make_tap<U8>(in, P, lut, y0 + v, col, fbase);
      bool inb0 = (v >= P.loy[0]) & (v <= P.hiy[0]);
      bool inb1 = (P.nby > 1) & (v >= P.loy[1]) & (v <= P.hiy[1]);
#pragma unroll
      for (int i = 0; i < MAXK; ++i) {
        if (i < P.nk) {
          for (int j = 0; j < P.kstep[i]; ++j) rotate(t.c, t.s, t.c1, t.s1);
          int q0 = qbits(t.c, t.sc1) - MAGIC_BITS, q1 = qbits(t.s, t.sc1) - MAGIC_BITS;
          int q2 = qbits(t.c, t.scD) - MAGIC_BITS, q3 = qbits(t.s, t.scD) - MAGIC_BITS;
          if (inb0) { S[0][4 * i] += q0; S[0][4 * i + 1] += q1; S[0][4 * i + 2] += q2; S[0][4 * i + 3] += q3; }
          if (MAXB > 1 && inb1) { S[1][4 * i] += q0; S[1][4 * i + 1] += q1; S[1][4 * i + 2] += q2; S[1][4 * i + 3] += q3; }
        }
      }
    }
  }

  // walker assignment for the H phase
  const int nseg = max(1, NT / max(nch, 1));
  const int seglen = (TWv + nseg - 1) / nseg;
  const int wch = tid / nseg, wseg = tid % nseg;

  for (int y = y0; y < yend; ++y) {
    // ---------------------------------------------------------------- V: slide one row
    if (y > y0) {
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        if (b < P.nby) {
          Tap te = make_tap<U8>(in, P, lut, y + P.hiy[b], col, fbase);
          Tap tl = make_tap<U8>(in, P, lut, y - 1 + P.loy[b], col, fbase);
#pragma unroll
          for (int i = 0; i < MAXK; ++i) {
            if (i < P.nk) {
              for (int j = 0; j < P.kstep[i]; ++j) {
                rotate(te.c, te.s, te.c1, te.s1);
                rotate(tl.c, tl.s, tl.c1, tl.s1);
              }
              S[b][4 * i] += qbits(te.c, te.sc1) - qbits(tl.c, tl.sc1);
              S[b][4 * i + 1] += qbits(te.s, te.sc1) - qbits(tl.s, tl.sc1);
              S[b][4 * i + 2] += qbits(te.c, te.scD) - qbits(tl.c, tl.scD);
              S[b][4 * i + 3] += qbits(te.s, te.scD) - qbits(tl.s, tl.scD);
            }
          }
        }
      }
    }
#pragma unroll
    for (int ch = 0; ch < C; ++ch) {
      if (ch < nch) {
        float U = P.wy[0] * (float)S[0][ch];
        if (MAXB > 1 && P.nby > 1) U = fmaf(P.wy[1], (float)S[1][ch], U);
        Ubuf[ch * UPITCH + tid] = qbits(U, P.uscale);
      }
    }
    __syncthreads();

    // ---------------------------------------------------------------- H: horizontal slide
    if (wch < nch) {
      const int xs = wseg * seglen;
      const int xe = min(xs + seglen, TWv);
      if (xs < xe) {
        const int* Ur = Ubuf + wch * UPITCH + P.rlo_x;
        int Hs0 = 0, Hs1 = 0;
        for (int j = xs + P.lox[0]; j <= xs + P.hix[0]; ++j) Hs0 += Ur[j] - MAGIC_BITS;
        if (MAXB > 1 && P.nbx > 1)
          for (int j = xs + P.lox[1]; j <= xs + P.hix[1]; ++j) Hs1 += Ur[j] - MAGIC_BITS;
        float* Fr = Fbuf + wch * FPITCH;
        for (int x = xs; x < xe; ++x) {
          if (x > xs) {
            Hs0 += Ur[x + P.hix[0]] - Ur[x - 1 + P.lox[0]];
            if (MAXB > 1 && P.nbx > 1) Hs1 += Ur[x + P.hix[1]] - Ur[x - 1 + P.lox[1]];
          }
          float F = P.wx[0] * (float)Hs0;
          if (MAXB > 1 && P.nbx > 1) F = fmaf(P.wx[1], (float)Hs1, F);
          Fr[x] = F;
        }
      }
    }
    __syncthreads();

    // ---------------------------------------------------------------- C: combine, divide
    if (tid < TWv) {
      const long long pix = fbase + (long long)y * P.W + (x0 + tid);
      float I = load_pixel(in, U8, pix);
      float c1, s1;
      if (U8) {
        float2 v = lut[(int)I];
        c1 = v.x;
        s1 = v.y;
      } else {
        base_angle(I, P, c1, s1);
      }
      float c = 1.f, s = 0.f;
      for (int j = 0; j < P.k0; ++j) rotate(c, s, c1, s1);
      double num = 0.0, den = 0.0;
      float tn = 0.f, td = 0.f;
#pragma unroll
      for (int i = 0; i < MAXK; ++i) {
        if (i < P.nk) {
          for (int j = 0; j < P.kstep[i]; ++j) rotate(c, s, c1, s1);
          const float a = P.a[i];
          tn = fmaf(a, fmaf(c, Fbuf[(4 * i + 2) * FPITCH + tid], s * Fbuf[(4 * i + 3) * FPITCH + tid]), tn);
          td = fmaf(a, fmaf(c, Fbuf[(4 * i) * FPITCH + tid], s * Fbuf[(4 * i + 1) * FPITCH + tid]), td);
          if ((i & 3) == 3) {
            num += (double)tn;
            den += (double)td;
            tn = td = 0.f;
          }
        }
      }
      num += (double)tn;
      den += (double)td;
      const long long opix = pix;
      if (P.pass == 1) {
        ws[opix] = make_double2(num, den);
      } else {
        if (P.pass >= 2) {
          double2 acc = ws[opix];
          num += acc.x;
          den += acc.y;
        }
        if (P.pass == 2) {
          ws[opix] = make_double2(num, den);
        } else {
          float o = (den > 0.0 && isfinite(den)) ? (float)((double)P.D * num / den) : I;
          out[opix] = o;
        }
      }
    }
    // the next row's V phase only writes Ubuf, which no thread reads after the H phase
  }
}

// ------------------------------------------------------------------ host side

struct LaunchShape {
  int NT, MAXK, TW, TH, passes;
};

template <int MAXK, bool U8, int NT>
cudaError_t launch_one(const KParams& P, const void* in, float* out, double2* ws, dim3 grid, cudaStream_t st) {
  constexpr int C = 4 * MAXK;
  size_t smem = (size_t)C * (NT + 1) * 4 + (size_t)C * (P.TW + 1) * 4 + 256 * sizeof(float2);
  auto kfn = bf_strip_kernel<MAXK, U8, NT>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kfn<<<grid, NT, smem, st>>>(P, in, out, ws);
  return cudaGetLastError();
}

template <bool U8>
cudaError_t dispatch(int NT, int MAXK, const KParams& P, const void* in, float* out, double2* ws, dim3 grid,
                     cudaStream_t st) {
  if (NT == 256 && MAXK == 8) return launch_one<8, U8, 256>(P, in, out, ws, grid, st);
  if (NT == 256 && MAXK == 16) return launch_one<16, U8, 256>(P, in, out, ws, grid, st);
  if (NT == 512 && MAXK == 8) return launch_one<8, U8, 512>(P, in, out, ws, grid, st);
  return cudaErrorInvalidConfiguration;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

bf_status run_filter(const bf_plan* p, const void* d_in, float* d_out, int n_frames, int H, int W,
                     cudaStream_t st) {
  if (!p || !d_in || !d_out || H <= 0 || W <= 0 || n_frames <= 0) return BF_ERR_INVALID_ARG;
  if ((long long)H * W > (1LL << 40) / n_frames) return BF_ERR_INVALID_ARG;
  if ((const void*)d_out == d_in) return BF_ERR_INVALID_ARG;
  if (!p->separable || p->nbx > MAXB || p->nby > MAXB) return BF_ERR_UNSUPPORTED;
  int rlo = 0, rhi = 0;
  for (int b = 0; b < p->nbx; ++b) {
    rlo = std::max(rlo, -p->lox[b]);
    rhi = std::max(rhi, p->hix[b]);
  }
  const int halo = rlo + rhi;
  int NT;
  if (halo + 32 <= 256) NT = 256;
  else if (halo + 64 <= 512) NT = 512;
  else return BF_ERR_UNSUPPORTED;
  const int MAXK = (NT == 512) ? 8 : (p->n_k <= 8 ? 8 : 16);
  const int passes = (p->n_k + MAXK - 1) / MAXK;
  const int TW = NT - halo;
  const int nstrips = (W + TW - 1) / TW;
  // band height: whole waves of 1-CTA-per-SM work, init (2r+1 rows) amortised over >= 4r rows
  const int nsm = sm_count();
  int ry = 0;
  for (int b = 0; b < p->nby; ++b) ry = std::max(ry, p->hiy[b] - p->loy[b] + 1);
  long long best_cost = -1;
  int best_nb = 1;
  for (int nb = 1; nb <= H; ++nb) {
    int TH = (H + nb - 1) / nb;
    if (nb > 1 && TH < 32) break;
    long long ctas = (long long)nstrips * nb * n_frames;
    long long waves = (ctas + nsm - 1) / nsm;
    long long cost = waves * (4LL * TH + ry);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_nb = nb;
    }
  }
  const int TH = (H + best_nb - 1) / best_nb;

  KParams P;
  std::memset(&P, 0, sizeof(P));
  P.H = H;
  P.W = W;
  P.nbx = p->nbx;
  P.nby = p->nby;
  for (int b = 0; b < p->nbx; ++b) {
    P.lox[b] = p->lox[b];
    P.hix[b] = p->hix[b];
    P.wx[b] = (float)p->wx[b];
  }
  double ubound = 0.0;
  for (int b = 0; b < p->nby; ++b) {
    P.loy[b] = p->loy[b];
    P.hiy[b] = p->hiy[b];
    P.wy[b] = (float)p->wy[b];
    ubound += std::fabs((double)P.wy[b]) * (p->hiy[b] - p->loy[b] + 1) * (double)QMAX;
  }
  P.rlo_x = rlo;
  P.TW = TW;
  P.TH = TH;
  const double invD = 1.0 / p->D;
  P.invD_hi = (float)invD;
  P.invD_lo = (float)(invD - (double)P.invD_hi);
  P.qD = (float)((double)QMAX / p->D);
  P.uscale = (float)((double)QMAX / (ubound * 1.000001));
  P.D = (float)p->D;
  P.frame_elems = (long long)H * W;

  double2* ws = nullptr;
  if (passes > 1) {
    if (cudaMallocAsync(&ws, sizeof(double2) * (size_t)H * W * n_frames, st) != cudaSuccess) return BF_ERR_CUDA;
  }
  dim3 grid(nstrips, best_nb, n_frames);
  const bool u8 = (p->input_dtype == BF_IN_U8);
  cudaError_t err = cudaSuccess;
  int prevk = 0;
  for (int pass = 0; pass < passes && err == cudaSuccess; ++pass) {
    const int first = pass * MAXK;
    const int nk = std::min(MAXK, p->n_k - first);
    P.nk = nk;
    P.k0 = prevk;
    for (int i = 0; i < nk; ++i) {
      int kk = p->k[first + i];
      P.kstep[i] = kk - (i == 0 ? prevk : p->k[first + i - 1]);
      P.a[i] = (float)p->a[first + i];
    }
    prevk = p->k[first + nk - 1];
    P.pass = (passes == 1) ? 0 : (pass == 0 ? 1 : (pass == passes - 1 ? 3 : 2));
    err = u8 ? dispatch<true>(NT, MAXK, P, d_in, d_out, ws, grid, st)
             : dispatch<false>(NT, MAXK, P, d_in, d_out, ws, grid, st);
  }
  if (ws) cudaFreeAsync(ws, st);
  return err == cudaSuccess ? BF_OK : BF_ERR_CUDA;
}

// Device buffers for bf_apply_host, grown on demand.
struct HostCache {
  std::mutex mu;
  void* din = nullptr;
  float* dout = nullptr;
  size_t in_bytes = 0, out_bytes = 0;
  ~HostCache() {
    // freed at process exit; the CUDA context may already be gone, so errors are ignored
    if (din) cudaFree(din);
    if (dout) cudaFree(dout);
  }
};
HostCache g_cache;

}  // namespace

extern "C" bf_status bf_apply(const bf_plan* plan, const void* d_in, float* d_out, int H, int W, bf_stream stream) {
  return run_filter(plan, d_in, d_out, 1, H, W, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" bf_status bf_apply_batched(const bf_plan* plan, const void* d_in, float* d_out, int n_frames, int H,
                                      int W, bf_stream stream) {
  return run_filter(plan, d_in, d_out, n_frames, H, W, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" bf_status bf_apply_host(const bf_plan* plan, const void* h_in, float* h_out, int H, int W,
                                   bf_stream stream) {
  if (!plan || !h_in || !h_out || H <= 0 || W <= 0) return BF_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t n = (size_t)H * W;
  const size_t ib = n * (plan->input_dtype == BF_IN_U8 ? 1 : 4), ob = n * 4;
  std::lock_guard<std::mutex> lk(g_cache.mu);
  if (g_cache.in_bytes < ib) {
    if (g_cache.din) cudaFree(g_cache.din);
    g_cache.din = nullptr;
    if (cudaMalloc(&g_cache.din, ib) != cudaSuccess) return BF_ERR_CUDA;
    g_cache.in_bytes = ib;
  }
  if (g_cache.out_bytes < ob) {
    if (g_cache.dout) cudaFree(g_cache.dout);
    g_cache.dout = nullptr;
    if (cudaMalloc(&g_cache.dout, ob) != cudaSuccess) return BF_ERR_CUDA;
    g_cache.out_bytes = ob;
  }
  if (cudaMemcpyAsync(g_cache.din, h_in, ib, cudaMemcpyHostToDevice, st) != cudaSuccess) return BF_ERR_CUDA;
  bf_status s = run_filter(plan, g_cache.din, g_cache.dout, 1, H, W, st);
  if (s != BF_OK) return s;
  if (cudaMemcpyAsync(h_out, g_cache.dout, ob, cudaMemcpyDeviceToHost, st) != cudaSuccess) return BF_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return BF_ERR_CUDA;
  return BF_OK;
}
