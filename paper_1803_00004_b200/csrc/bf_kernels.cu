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

constexpr int QMAX = (1 << 22) - 1;       // |quantised channel value| <= QMAX
constexpr float MAGIC = 12582912.0f;      // 1.5 * 2^23: fma(x, s, MAGIC) has bits 0x4B400000 + rint(x*s)
constexpr int MAXB = 4;                   // boxes per axis of the separable spatial factor
constexpr int ABITS = 27;                 // integer horizontal box weights
constexpr int WBITS = 29;                 // integer combine weights

struct KParams {
  int H, W;
  int nk;                   // cosine terms handled by this launch
  int kstep[BF_MAX_TERMS];  // rotation steps from the previous term (first: from k0)
  float a[BF_MAX_TERMS];    // a_k
  int k0;                   // k of the term before the first one of this launch (0 for pass 0)
  int nbx, nby;
  int lox[MAXB], hix[MAXB], loy[MAXB], hiy[MAXB];
  int ax[MAXB];             // horizontal box weights as integers: round(wx_b / max|wx| * 2^27)
  int fshift;               // F32 = (sum_b ax_b H_b) >> fshift fits in int32
  int ay[MAXB];             // vertical box weights as integers: round(wy_b / max|wy| * 2^27)
  float qD;                 // QMAX / D (scale of the I cos / I sin channels; cos / sin use QMAX)
  int vlo, vhi;             // union of the vertical boxes (rows v with some box containing v)
  int rlo_x;                // -min lox (left halo)
  int ushift;               // U' = (sum_b ay_b S_b) >> ushift keeps the horizontal sums in int32
  int TW, TH;               // output strip width / band height
  float invD_hi, invD_lo;   // 1/D as a float-float pair
  float D;
  float aw[BF_MAX_TERMS];   // a_k * 2^WBITS: combine weights quantised as rint(aw * cos/sin)
  int pass;                 // 0 = only pass; 1 = first; 2 = middle; 3 = last
  long long frame_elems;    // H * W (batched frames)
};

typedef unsigned long long u64;

// ---- packed fp32x2 helpers (sm_100a FFMA2 / FMUL2: two lanes of work per issue slot)
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// (lo - hi) of the integer bit patterns of a packed pair of quantised values
__device__ __forceinline__ int diff_bits(u64 v) {
  int a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
  return a - b;
}

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

template <bool U8>
__device__ __forceinline__ void tap_base(const void* in, const KParams& P, const float2* lut, int row, int col,
                                         long long fbase, float& c1, float& s1, float& I, bool& valid) {
  valid = (row >= 0) & (row < P.H) & (col >= 0) & (col < P.W);
  I = 0.f;
  if (valid) I = load_pixel(in, U8, fbase + (long long)row * P.W + col);
  if (U8) {
    float2 v = lut[(int)I];
    c1 = v.x;
    s1 = v.y;
  } else {
    base_angle(I, P, c1, s1);
  }
}

// Channels of one cosine term for a packed pair of taps (lo half = entering row, hi half =
// leaving row): cos, sin, I cos, I sin quantised with FFMA against MAGIC; the state gains
// q(enter) - q(leave) exactly (int32 arithmetic on the bit patterns, the bias cancels).
__device__ __forceinline__ void accumulate_pair(int* St, u64 C, u64 S, u64 SC1, u64 SCD) {
  const u64 MM = pk(MAGIC, MAGIC);
  St[0] += diff_bits(fma2(C, SC1, MM));
  St[1] += diff_bits(fma2(S, SC1, MM));
  St[2] += diff_bits(fma2(C, SCD, MM));
  St[3] += diff_bits(fma2(S, SCD, MM));
}

__device__ __forceinline__ void rotate2(u64& C, u64& S, u64 C1, u64 S1, u64 NS1) {
  u64 Cn = fma2(S, NS1, mul2(C, C1));
  u64 Sn = fma2(C, S1, mul2(S, C1));
  C = Cn;
  S = Sn;
}

// sum of U[a..b] (inclusive), 16-byte vector loads where aligned
__device__ __forceinline__ int range_sum(const int* U, int a, int b) {
  int s = 0, j = a;
  for (; j <= b && (reinterpret_cast<uintptr_t>(U + j) & 15) != 0; ++j) s += U[j];
  for (; j + 3 <= b; j += 4) {
    const int4 v = *reinterpret_cast<const int4*>(U + j);
    s += v.x + v.y + v.z + v.w;
  }
  for (; j <= b; ++j) s += U[j];
  return s;
}

// F = (sum_b ax_b H_b) >> fshift: exact int64 weighted box sum narrowed to int32.
template <int NB>
__device__ __forceinline__ int combine_boxes(const int* Hs, const KParams& P) {
  long long f = (long long)P.ax[0] * Hs[0];
#pragma unroll
  for (int b = 1; b < NB; ++b)
    if (b < P.nbx) f += (long long)P.ax[b] * Hs[b];
  return (int)(f >> P.fshift);
}

template <int MAXK, bool U8, int NT, bool CONSEC, int NB>
__global__ void __launch_bounds__(NT, 1) bf_strip_kernel(const KParams P, const void* __restrict__ in,
                                                         float* __restrict__ out, longlong2* __restrict__ ws) {
  constexpr int C = 4 * MAXK;
  constexpr int R = 2;                                                // output rows per iteration
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int UPITCH = NT + 1;
  const int FPITCH = P.TW + 1;
  const int nch = 4 * P.nk;                                           // channels of this launch
  float2* lut = reinterpret_cast<float2*>(smem_raw);                  // [256] (u8 only)
  int* Ubuf = reinterpret_cast<int*>(lut + 256);                      // [R][nch][UPITCH]
  int* Fbuf = Ubuf + R * nch * UPITCH;                                // [R][nch][FPITCH]

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P.TW;
  const int y0 = blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int col = x0 - P.rlo_x + tid;
  const bool colok = (col >= 0) & (col < P.W);
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

  // ---- vertical state at row y0 - 1: exact int32 box sums S_b of every channel, one per box
  //      of fy (each channel value quantised ONCE at full 22-bit scale; folding the box weights
  //      into the quantisation loses the tolerance).
  int S[NB][C];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int ch = 0; ch < C; ++ch) S[b][ch] = 0;

  for (int v = P.vlo; v <= P.vhi; ++v) {
    float c1, s1, I;
    bool valid;
    tap_base<U8>(in, P, lut, y0 - 1 + v, col, fbase, c1, s1, I, valid);
    const float sc1 = valid ? (float)QMAX : 0.f, scD = valid ? P.qD * I : 0.f;
    bool inb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) inb[b] = (b < P.nby) && v >= P.loy[b] && v <= P.hiy[b];
    float c = 1.f, s = 0.f;
    for (int j = 0; j < P.k0; ++j) rotate(c, s, c1, s1);
#pragma unroll
    for (int i = 0; i < MAXK; ++i) {
      if (i < P.nk) {
        if (CONSEC) {
          if (i > 0) rotate(c, s, c1, s1);
        } else {
          for (int j = 0; j < P.kstep[i]; ++j) rotate(c, s, c1, s1);
        }
        const int q0 = __float_as_int(fmaf(c, sc1, MAGIC)) - 0x4B400000;
        const int q1 = __float_as_int(fmaf(s, sc1, MAGIC)) - 0x4B400000;
        const int q2 = __float_as_int(fmaf(c, scD, MAGIC)) - 0x4B400000;
        const int q3 = __float_as_int(fmaf(s, scD, MAGIC)) - 0x4B400000;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (inb[b]) {
            S[b][4 * i] += q0;
            S[b][4 * i + 1] += q1;
            S[b][4 * i + 2] += q2;
            S[b][4 * i + 3] += q3;
          }
        }
      }
    }
  }

  // tap rows of the iteration whose first output row is ya, per box b:
  //   j=0 enter(ya) = ya + hi, j=1 leave(ya) = ya - 1 + lo, j=2 enter(ya+1), j=3 leave(ya+1)
  float Ipre[NB][4];
  auto load_taps = [&](int ya) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int row = ya + ((j & 2) ? 1 : 0) + ((j & 1) ? (P.loy[b] - 1) : P.hiy[b]);
        const bool ok = (b < P.nby) && colok && row >= 0 && row < P.H;
        Ipre[b][j] = ok ? load_pixel(in, U8, fbase + (long long)row * P.W + col) : 0.f;
      }
    }
  };
  load_taps(y0);

  // walker assignment for the H phase: (row r, channel, segment)
  const int nwalk = R * nch;
  const int nseg = max(1, NT / max(nwalk, 1));
  const int seglen = (TWv + nseg - 1) / nseg;
  const int wr = tid / (nch * nseg);
  const int wch = (tid / nseg) % max(nch, 1);
  const int wseg = tid % nseg;
  const long long uround = P.ushift > 0 ? (1LL << (P.ushift - 1)) : 0;

  for (int ya = y0; ya < yend; ya += R) {
    // ---------------------------------------------------------------- V: slide two rows
    {
      u64 C1A[NB], S1A[NB], NS1A[NB], SC1A[NB], SCDA[NB], CA[NB], SA[NB];
      u64 C1B[NB], S1B[NB], NS1B[NB], SC1B[NB], SCDB[NB], CB[NB], SB[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float c1[4], s1[4], sc1[4], scD[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int row = ya + ((j & 2) ? 1 : 0) + ((j & 1) ? (P.loy[b] - 1) : P.hiy[b]);
          const bool ok = (b < P.nby) && colok && row >= 0 && row < P.H;
          const float I = Ipre[b][j];
          if (U8) {
            const float2 t = lut[(int)I];
            c1[j] = t.x;
            s1[j] = t.y;
          } else {
            base_angle(I, P, c1[j], s1[j]);
          }
          sc1[j] = ok ? (float)QMAX : 0.f;
          scD[j] = ok ? P.qD * I : 0.f;
        }
        C1A[b] = pk(c1[0], c1[1]);
        S1A[b] = pk(s1[0], s1[1]);
        NS1A[b] = pk(-s1[0], -s1[1]);
        SC1A[b] = pk(sc1[0], sc1[1]);
        SCDA[b] = pk(scD[0], scD[1]);
        C1B[b] = pk(c1[2], c1[3]);
        S1B[b] = pk(s1[2], s1[3]);
        NS1B[b] = pk(-s1[2], -s1[3]);
        SC1B[b] = pk(sc1[2], sc1[3]);
        SCDB[b] = pk(scD[2], scD[3]);
        if (CONSEC) {
          CA[b] = CB[b] = pk(1.f, 1.f);
          SA[b] = SB[b] = pk(0.f, 0.f);
        } else {
          float cc[4] = {1.f, 1.f, 1.f, 1.f}, ss[4] = {0.f, 0.f, 0.f, 0.f};
          for (int j = 0; j < P.k0; ++j)
#pragma unroll
            for (int t = 0; t < 4; ++t) rotate(cc[t], ss[t], c1[t], s1[t]);
          CA[b] = pk(cc[0], cc[1]);
          SA[b] = pk(ss[0], ss[1]);
          CB[b] = pk(cc[2], cc[3]);
          SB[b] = pk(ss[2], ss[3]);
        }
      }
      if (ya + R < yend) load_taps(ya + R);   // prefetch: completes during the H and C phases
      const u64 MM = pk(MAGIC, MAGIC);
#pragma unroll
      for (int i = 0; i < MAXK; ++i) {
        if (i < P.nk) {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (CONSEC) {
              if (i > 0) {
                rotate2(CA[b], SA[b], C1A[b], S1A[b], NS1A[b]);
                rotate2(CB[b], SB[b], C1B[b], S1B[b], NS1B[b]);
              }
            } else {
              for (int j = 0; j < P.kstep[i]; ++j) {
                rotate2(CA[b], SA[b], C1A[b], S1A[b], NS1A[b]);
                rotate2(CB[b], SB[b], C1B[b], S1B[b], NS1B[b]);
              }
            }
          }
          int da[NB][4], db[NB][4];
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            da[b][0] = diff_bits(fma2(CA[b], SC1A[b], MM));
            da[b][1] = diff_bits(fma2(SA[b], SC1A[b], MM));
            da[b][2] = diff_bits(fma2(CA[b], SCDA[b], MM));
            da[b][3] = diff_bits(fma2(SA[b], SCDA[b], MM));
            db[b][0] = diff_bits(fma2(CB[b], SC1B[b], MM));
            db[b][1] = diff_bits(fma2(SB[b], SC1B[b], MM));
            db[b][2] = diff_bits(fma2(CB[b], SCDB[b], MM));
            db[b][3] = diff_bits(fma2(SB[b], SCDB[b], MM));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ch = 4 * i + j;
            long long ua = uround, ub = uround;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              if (b < P.nby) {
                S[b][ch] += da[b][j];
                ua += (long long)P.ay[b] * S[b][ch];
                S[b][ch] += db[b][j];
                ub += (long long)P.ay[b] * S[b][ch];
              }
            }
            Ubuf[ch * UPITCH + tid] = (int)(ua >> P.ushift);
            Ubuf[(nch + ch) * UPITCH + tid] = (int)(ub >> P.ushift);
          }
        }
      }
    }
    __syncthreads();

    // ---------------------------------------------------------------- H: horizontal slide
    // Each walker (row, channel, segment) slides the exact int32 box sums H_b of U' along the
    // row and writes F = (sum_b ax_b H_b) >> fshift (exact int64 product sum, narrowed).
    if (wr < R && wch < nch && ya + wr < yend) {
      const int xs = wseg * seglen;
      const int xe = min(xs + seglen, TWv);
      if (xs < xe) {
        const int* Ur = Ubuf + (wr * nch + wch) * UPITCH + P.rlo_x;
        int* Fr = Fbuf + (wr * nch + wch) * FPITCH;
        int Hs[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) Hs[b] = (b < P.nbx) ? range_sum(Ur, xs + P.lox[b], xs + P.hix[b]) : 0;
        Fr[xs] = combine_boxes<NB>(Hs, P);
        const int* pe[NB];
        const int* pl[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          pe[b] = Ur + xs + 1 + P.hix[b];
          pl[b] = Ur + xs + P.lox[b];
        }
        int x = xs + 1;
        for (; x + 7 < xe; x += 8) {
          int e[NB][8], l[NB][8];
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              e[b][j] = pe[b][j];
              l[b][j] = pl[b][j];
            }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int b = 0; b < NB; ++b) Hs[b] += e[b][j] - l[b][j];
            Fr[x + j] = combine_boxes<NB>(Hs, P);
          }
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            pe[b] += 8;
            pl[b] += 8;
          }
        }
        for (; x < xe; ++x) {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            Hs[b] += pe[b][0] - pl[b][0];
            pe[b] += 1;
            pl[b] += 1;
          }
          Fr[x] = combine_boxes<NB>(Hs, P);
        }
      }
    }
    __syncthreads();

    // ---------------------------------------------------------------- C: combine, divide
    // num = sum_k a_k (cos F_Ic + sin F_Is), den = sum_k a_k (cos F_c + sin F_s) with the weights
    // quantised to WBITS and the products accumulated exactly in int64 (an fp32 combine of the
    // box sums loses the tolerance at ill-conditioned pixels).
    for (int o = tid; o < R * TWv; o += NT) {
      const int r = o / TWv, xo = o - r * TWv;
      const int y = ya + r;
      if (y >= yend) continue;
      const long long pix = fbase + (long long)y * P.W + (x0 + xo);
      const int* Fr = Fbuf + r * nch * FPITCH + xo;
      float c1, s1, I;
      bool valid;
      tap_base<U8>(in, P, lut, y, x0 + xo, fbase, c1, s1, I, valid);
      float c = 1.f, s = 0.f;
      for (int j = 0; j < P.k0; ++j) rotate(c, s, c1, s1);
      long long num = 0, den = 0;
#pragma unroll
      for (int i = 0; i < MAXK; ++i) {
        if (i < P.nk) {
          if (CONSEC) {
            if (i > 0) rotate(c, s, c1, s1);
          } else {
            for (int j = 0; j < P.kstep[i]; ++j) rotate(c, s, c1, s1);
          }
          const long long wc = __float2int_rn(P.aw[i] * c), wsn = __float2int_rn(P.aw[i] * s);
          den += wc * Fr[(4 * i) * FPITCH] + wsn * Fr[(4 * i + 1) * FPITCH];
          num += wc * Fr[(4 * i + 2) * FPITCH] + wsn * Fr[(4 * i + 3) * FPITCH];
        }
      }
      if (P.pass == 1) {
        ws[pix] = make_longlong2(num, den);
      } else {
        if (P.pass >= 2) {
          const longlong2 acc = ws[pix];
          num += acc.x;
          den += acc.y;
        }
        if (P.pass == 2) {
          ws[pix] = make_longlong2(num, den);
        } else {
          out[pix] = (den > 0) ? (float)((double)P.D * (double)num / (double)den) : I;
        }
      }
    }
    // the next iteration's V phase only writes Ubuf, which no thread reads after the H phase
  }
}

// ------------------------------------------------------------------ host side

struct LaunchShape {
  int NT, MAXK, TW, TH, passes;
};

template <int MAXK, bool U8, int NT, bool CONSEC, int NB>
cudaError_t launch_one(const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid, cudaStream_t st) {
  constexpr int C = 4 * MAXK;
  const size_t nch = 4 * (size_t)P.nk;
  size_t smem = 2 * (nch * (NT + 1) * 4 + nch * (P.TW + 1) * 4) + 256 * sizeof(float2);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  auto kfn = bf_strip_kernel<MAXK, U8, NT, CONSEC, NB>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kfn<<<grid, NT, smem, st>>>(P, in, out, ws);
  return cudaGetLastError();
}

template <int MAXK, bool U8, int NT>
cudaError_t dispatch_shape(bool consec, int nb, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                           cudaStream_t st) {
  if (consec) {
    if (nb == 1) return launch_one<MAXK, U8, NT, true, 1>(P, in, out, ws, grid, st);
    if (nb == 2) return launch_one<MAXK, U8, NT, true, 2>(P, in, out, ws, grid, st);
  } else {
    if (nb == 1) return launch_one<MAXK, U8, NT, false, 1>(P, in, out, ws, grid, st);
    if (nb == 2) return launch_one<MAXK, U8, NT, false, 2>(P, in, out, ws, grid, st);
  }
  return launch_one<MAXK, U8, NT, false, 4>(P, in, out, ws, grid, st);
}

template <bool U8>
cudaError_t dispatch(int NT, int MAXK, bool consec, int nb, const KParams& P, const void* in, float* out, longlong2* ws,
                     dim3 grid, cudaStream_t st) {
  if (NT == 256 && MAXK == 8) return dispatch_shape<8, U8, 256>(consec, nb, P, in, out, ws, grid, st);
  if (NT == 256 && MAXK == 16) return dispatch_shape<16, U8, 256>(consec, nb, P, in, out, ws, grid, st);
  if (NT == 512 && MAXK == 8) return dispatch_shape<8, U8, 512>(consec, nb, P, in, out, ws, grid, st);
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
  const int TW = NT - halo;
  // channels per launch: as many as fit the registers (MAXK) and the two-row shared-memory
  // buffers (2 rows x nch x (NT + 1 + TW + 1) ints); otherwise several accumulating launches
  auto smem_for = [&](int nk) { return 2 * (4.0 * nk * (NT + 1) * 4 + 4.0 * nk * (TW + 1) * 4) + 2048; };
  int MAXK = (NT == 512) ? 8 : (p->n_k <= 8 ? 8 : 16);
  while (MAXK > 8 && smem_for(std::min(MAXK, p->n_k)) > 227.0 * 1024) MAXK = 8;
  if (smem_for(std::min(MAXK, p->n_k)) > 227.0 * 1024) return BF_ERR_UNSUPPORTED;
  const int passes = (p->n_k + MAXK - 1) / MAXK;
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
  best_nb = (H + TH - 1) / TH;

  KParams P;
  std::memset(&P, 0, sizeof(P));
  P.H = H;
  P.W = W;
  P.nbx = p->nbx;
  P.nby = p->nby;
  double wxmax = 0.0;
  for (int b = 0; b < p->nbx; ++b) wxmax = std::max(wxmax, std::fabs(p->wx[b]));
  for (int b = 0; b < p->nbx; ++b) {
    P.lox[b] = p->lox[b];
    P.hix[b] = p->hix[b];
    P.ax[b] = (int)std::lround(std::ldexp(p->wx[b] / wxmax, ABITS));
  }
  // vertical box weights as integers; S_b bounded by n_b * (QMAX + 1/2)
  double wymax = 0.0;
  for (int b = 0; b < p->nby; ++b) wymax = std::max(wymax, std::fabs(p->wy[b]));
  double sbound = 0.0;  // bound of |sum_b ay_b S_b|
  P.vlo = p->loy[0];
  P.vhi = p->hiy[0];
  for (int b = 0; b < p->nby; ++b) {
    P.loy[b] = p->loy[b];
    P.hiy[b] = p->hiy[b];
    P.ay[b] = (int)std::lround(std::ldexp(p->wy[b] / wymax, ABITS));
    sbound += std::fabs((double)P.ay[b]) * ((double)QMAX + 0.5) * (p->hiy[b] - p->loy[b] + 1);
    P.vlo = std::min(P.vlo, p->loy[b]);
    P.vhi = std::max(P.vhi, p->hiy[b]);
    if ((p->hiy[b] - p->loy[b] + 1) * ((double)QMAX + 0.5) >= 2147483647.0) return BF_ERR_UNSUPPORTED;
  }
  P.qD = (float)((double)QMAX / p->D);
  // U' = S >> ushift so that every horizontal box sum of U' stays inside int32
  int nxmax = 1;
  for (int b = 0; b < p->nbx; ++b) nxmax = std::max(nxmax, p->hix[b] - p->lox[b] + 1);
  P.ushift = 0;
  while ((sbound / std::ldexp(1.0, P.ushift) + 1.0) * nxmax >= 2147483647.0) ++P.ushift;
  {
    // bound of |sum_b ax_b H_b| -> shift that narrows F to int32
    const double ub = sbound / std::ldexp(1.0, P.ushift) + 1.0;
    double fb = 0.0;
    for (int b = 0; b < p->nbx; ++b) fb += std::fabs((double)P.ax[b]) * ub * (p->hix[b] - p->lox[b] + 1);
    P.fshift = 0;
    while (fb / std::ldexp(1.0, P.fshift) >= 2147483000.0) ++P.fshift;
  }
  P.rlo_x = rlo;
  P.TW = TW;
  P.TH = TH;
  const double invD = 1.0 / p->D;
  P.invD_hi = (float)invD;
  P.invD_lo = (float)(invD - (double)P.invD_hi);
  P.D = (float)p->D;
  P.frame_elems = (long long)H * W;
  const int nbmax = std::max(p->nbx, p->nby);
  longlong2* ws = nullptr;
  if (passes > 1) {
    if (cudaMallocAsync(&ws, sizeof(longlong2) * (size_t)H * W * n_frames, st) != cudaSuccess) return BF_ERR_CUDA;
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
      P.aw[i] = (float)std::ldexp(p->a[first + i], WBITS);
    }
    prevk = p->k[first + nk - 1];
    P.pass = (passes == 1) ? 0 : (pass == 0 ? 1 : (pass == passes - 1 ? 3 : 2));
    bool consec = (P.k0 == 0);
    for (int i = 0; i < nk; ++i) consec = consec && (p->k[first + i] == i);
    err = u8 ? dispatch<true>(NT, MAXK, consec, nbmax, P, d_in, d_out, ws, grid, st)
             : dispatch<false>(NT, MAXK, consec, nbmax, P, d_in, d_out, ws, grid, st);
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
