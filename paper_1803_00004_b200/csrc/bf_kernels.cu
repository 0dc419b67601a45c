// sm_100a kernels of the joint-acceleration bilateral filter (bf_apply) and their host dispatch.
//
// Evaluates eq:numerator_2D_box_N_terms with T = D (Q1): for every selected cosine
// term k the four channels g^c_k = cos(w_k I), g^s_k = sin(w_k I), G^c_k = I g^c_k,
// G^s_k = I g^s_k are generated in registers, box-filtered with the Haar-box kernel
// K~_s (eq:2D_box_N_terms_s, Appendix A; separable, or rank 2 for N_s = 5), and
// recombined with a_k g^c_k(x), a_k g^s_k(x) (Q17); out = num / den (eq:BF).
//
// A CTA owns a vertical strip (TW output columns plus the horizontal halo) and a band of TH
// output rows. Per row y, in every kernel:
//   V(y)  one thread per extended column slides the vertical box sums of all channels down one
//         row. The box weight wy_b is folded into the per-tap quantisation scale, so the state
//         is ONE exact int32 per channel (U = sum_b sum_v rint(wy_b X 2^q)); the taps' channels
//         come from a polynomial (f32) or LUT (u8) base angle and the rotation recurrence, and
//         are quantised with one FFMA2 per tap pair (x*s + 1.5*2^23 holds rint(x*s) in its low
//         mantissa bits). U' = U >> ush goes to shared memory.
//   H(y)  exact int32 horizontal box sums H_b of U', weighted into F = sum_b mulhi(H_b, ax_b):
//         by walkers (kernel 1) or as differences of in-place prefix rows (kernels 2, 2b).
//   C(y)  per output pixel: combine weights a_k cos/sin(k pi I(x)/D) in fp64, rounded to int32,
//         num / den accumulated exactly in int64; out = D num / den (or I(x) if den <= 0, Q18).
// Kernel 1 (bf_band_kernel) runs V / C and H in barrier-separated intervals; kernel 2
// (bf_ws_kernel) and kernel 2b (bf_ws2_kernel, the default) specialise warps by role and hand
// rows over through named barriers, kernel 2b fusing the box differences into the combine.
// Kernel 3 (bf_literal_kernel) is the paper-literal z-window on u8 levels (NEXT f1). All three
// T = D kernels perform the same integer arithmetic: their outputs are bitwise equal.
// Nothing but the input image and the output image touches HBM (plus an int64 num/den
// workspace when the terms do not fit one pass).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "bf_internal.h"

namespace {

constexpr float MAGIC = 12582912.0f;              // 1.5 * 2^23
constexpr int MAGIC_BITS = 0x4B400000;            // bit pattern of MAGIC
constexpr double MAGIC64 = 6755399441055744.0;    // 1.5 * 2^52: low word of fma(x, s, MAGIC64) = rint(x*s)
constexpr int QBITS_MAX = 22;                     // channel quantisation (the FFMA trick's range)
constexpr int ABITS = 30;                         // horizontal integer box weights (mulhi multipliers)
constexpr int MAXB = 4;                           // boxes per axis
constexpr int MAXP = BF_MAX_PLANS;                // range plans of one bf_apply_multi

struct KParams {
  int H, W;
  long long frame_elems;
  int TW, TH, rlo_x;
  int yb, ye;                 // output rows [yb, ye) of this launch (bf_apply_host pipelines row chunks)
  int ns;                     // box-pair terms: K~_s = sum_{s < ns} fx_s(u) fy_s(v) (1 = separable)
  int nby;                    // vertical boxes (shared by the ns terms: one set of taps)
  int vlo[MAXB], vhi[MAXB];   // vertical boxes: row offsets (inclusive)
  float qs[2][MAXB];          // per term s: quantisation scales wy_sb / max|wy| * 2^q (cos / sin channels)
  float qsD[2][MAXB];         // qs_sb / D (I cos / I sin channels)
  int vmin, vmax;             // union of the vertical boxes
  int urnd, ush;              // U' = (U + urnd) >> ush; urnd is folded into the initial state
  int nbx[2];                 // horizontal boxes of term s
  int hlo[2][MAXB], hhi[2][MAXB];   // their column offsets (inclusive)
  int ax[2][MAXB];            // their integer weights round(wx_sb / max|wx| * 2^abits):
                              // F = sum_tb mulhi(H_tb, ax_tb) (high words of the int64 products)
  int nk;                     // terms of this pass
  int kstep[BF_MAX_TERMS];    // Chebyshev steps before term i (term 0: from k = 0)
  double aw[BF_MAX_PLANS][16];   // a_k * 2^wbits of each range plan (bf_apply_multi; one plan otherwise)
  int nplans;                 // range plans sharing the box-filtered channels (Case 1)
  long long plan_stride;      // output elements between consecutive plans' images
  float invD_hi, invD_lo;     // 1/D as a float-float pair
  double invD, D;
  int pass;                   // 0 = only pass; 1 = first; 2 = middle; 3 = last
  int ngrp, nseg, seglen;     // walkers: 32-channel groups x row segments
  int wpar;                   // paired-load walker: parity of box 1's leave stream (0 / 1), -1 = scalar walker
  int wv;                     // kernel 2b: extended columns written and scanned (TW + halo rounded up to 8)
  int f_off, l_off;           // shared-memory carve-up: U' [4 nk][NT+1] int, F [TW][4 MAXK + 4] int,
                              // LUTs (u8) float2[256] + double2[256]
};

typedef unsigned long long u64;

// ---- packed fp32x2 helpers (sm_100a FFMA2: two lanes of work per issue slot)
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
// q(lo) - q(hi) of a packed pair of quantised values (the MAGIC bias cancels)
__device__ __forceinline__ int diff_bits(u64 v) {
  int a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
  return a - b;
}
// c + (int64) a * b as ONE IMAD.WIDE (the compiler otherwise widens a shifted-and-narrowed operand
// to a full 64 x 64 product)
__device__ __forceinline__ long long mad_wide(int a, int b, long long c) {
  long long r;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}
__device__ __forceinline__ int quant(float x, float s) { return __float_as_int(fmaf(x, s, MAGIC)) - MAGIC_BITS; }

__device__ __forceinline__ float load_pixel(const void* in, bool u8, long long idx) {
  if (u8) return (float)__ldg(reinterpret_cast<const unsigned char*>(in) + idx);
  return __ldg(reinterpret_cast<const float*>(in) + idx);
}

// cos(pi I / D), sin(pi I / D) in fp32 for I in [0, D]: t' = I/D - 1/2 (float-float 1/D),
// sin(pi t') = t' P(t'^2), cos(pi t') = Q(t'^2) (least-squares minimax fits, |err| <= 2e-7,
// tools/numerics_v6.py), cos(pi t) = -sin(pi t'), sin(pi t) = cos(pi t').
__device__ __forceinline__ void base_angle_f32(float I, const KParams& P, float& c1, float& s1) {
  float t = fmaf(I, P.invD_hi, -0.5f);
  t = fmaf(I, P.invD_lo, t);
  const float z = t * t;
  float p = -7.022163365e-03f;
  p = fmaf(p, z, 8.204647899e-02f);
  p = fmaf(p, z, -5.992513299e-01f);
  p = fmaf(p, z, 2.550163269e+00f);
  p = fmaf(p, z, -5.167712688e+00f);
  p = fmaf(p, z, 3.141592741e+00f);
  float q = -1.004332444e-04f;
  q = fmaf(q, z, 1.927883714e-03f);
  q = fmaf(q, z, -2.580653690e-02f);
  q = fmaf(q, z, 2.353305817e-01f);
  q = fmaf(q, z, -1.335262775e+00f);
  q = fmaf(q, z, 4.058712006e+00f);
  q = fmaf(q, z, -4.934802055e+00f);
  q = fmaf(q, z, 1.0f);
  c1 = -p * t;
  s1 = q;
}

// The same angle in fp64 for the combine weights: Taylor series of sin(pi t') / t' and
// cos(pi t') to degree 21 / 22 (truncation < 2e-18 on |t'| <= 1/2), Horner in DFMA.
__constant__ double kSinPi64[11] = {3.14159265358979312e+00, -5.16771278004996937e+00, 2.55016403987734508e+00,
                                     -5.99264529320791883e-01, 8.21458866111281910e-02, -7.37043094571434784e-03,
                                     4.66302805767612337e-04, -2.19153534478302037e-05, 7.95205400147550838e-07,
                                     -2.29484289972698565e-08, 5.39266466260812482e-10};
__constant__ double kCosPi64[12] = {1.0, -4.93480220054467900e+00, 4.05871212641676760e+00, -1.33526276885458928e+00,
                                    2.35330630358893123e-01, -2.58068913900140508e-02, 1.92957430940392206e-03,
                                    -1.04638104924845650e-04, 4.30306958703294391e-06, -1.38789524622137608e-07,
                                    3.60473079746249822e-09, -7.70070713060134610e-11};

// The same angle in fp64 for the combine weights: Taylor series of sin(pi t') / t' and
// cos(pi t') to degree 21 / 22 (truncation < 2e-18 on |t'| <= 1/2), Horner in DFMA with the
// coefficients as constant-bank operands.
__device__ __forceinline__ void base_angle_f64(float I, double invD, double& c1, double& s1) {
  const double t = fma((double)I, invD, -0.5);
  const double z = t * t;
  double p = kSinPi64[10];
#pragma unroll
  for (int i = 9; i >= 0; --i) p = fma(p, z, kSinPi64[i]);
  double q = kCosPi64[11];
#pragma unroll
  for (int i = 10; i >= 0; --i) q = fma(q, z, kCosPi64[i]);
  c1 = -p * t;
  s1 = q;
}

__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// base_angle_f32 on a packed pair of inputs (FFMA2 / FMUL2), bit-identical per lane: the sine
// polynomial runs with negated coefficients so that its product with t' is -p t' directly.
__device__ __forceinline__ void base_angle_f32x2(float Ia, float Ib, const KParams& P, u64& C1, u64& S1) {
  const u64 I2 = pk(Ia, Ib);
  u64 t = fma2(I2, pk(P.invD_hi, P.invD_hi), pk(-0.5f, -0.5f));
  t = fma2(I2, pk(P.invD_lo, P.invD_lo), t);
  const u64 z = mul2(t, t);
  u64 p = pk(7.022163365e-03f, 7.022163365e-03f);
  p = fma2(p, z, pk(-8.204647899e-02f, -8.204647899e-02f));
  p = fma2(p, z, pk(5.992513299e-01f, 5.992513299e-01f));
  p = fma2(p, z, pk(-2.550163269e+00f, -2.550163269e+00f));
  p = fma2(p, z, pk(5.167712688e+00f, 5.167712688e+00f));
  p = fma2(p, z, pk(-3.141592741e+00f, -3.141592741e+00f));
  u64 q = pk(-1.004332444e-04f, -1.004332444e-04f);
  q = fma2(q, z, pk(1.927883714e-03f, 1.927883714e-03f));
  q = fma2(q, z, pk(-2.580653690e-02f, -2.580653690e-02f));
  q = fma2(q, z, pk(2.353305817e-01f, 2.353305817e-01f));
  q = fma2(q, z, pk(-1.335262775e+00f, -1.335262775e+00f));
  q = fma2(q, z, pk(4.058712006e+00f, 4.058712006e+00f));
  q = fma2(q, z, pk(-4.934802055e+00f, -4.934802055e+00f));
  q = fma2(q, z, pk(1.0f, 1.0f));
  C1 = mul2(p, t);
  S1 = q;
}

// Rotation recurrence (c, s)_{k+1} = (c c1 - s s1, s c1 + c s1) on a packed pair of taps:
// 2 FMUL2 + 2 FFMA2 per step, no register shuffling. rot1() is the bit-identical scalar form.
struct Rot2 {
  u64 C, S, C1, S1, NS1;
  __device__ __forceinline__ void init(float ca, float sa, float cb, float sb) {
    C = pk(1.f, 1.f);
    S = pk(0.f, 0.f);
    C1 = pk(ca, cb);
    S1 = pk(sa, sb);
    NS1 = pk(-sa, -sb);
  }
  __device__ __forceinline__ void init2(u64 c1, u64 s1) {
    C = pk(1.f, 1.f);
    S = pk(0.f, 0.f);
    C1 = c1;
    S1 = s1;
    NS1 = s1 ^ 0x8000000080000000ull;
  }
  __device__ __forceinline__ void step() {
    const u64 Cn = fma2(S, NS1, mul2(C, C1));
    const u64 Sn = fma2(C, S1, mul2(S, C1));
    C = Cn;
    S = Sn;
  }
};
__device__ __forceinline__ void rot1(float& c, float& s, float c1, float s1) {
  const float cn = fmaf(s, -s1, c * c1);
  const float sn = fmaf(c, s1, s * c1);
  c = cn;
  s = sn;
}

struct Cheb64 {
  double c, s, cp, sp, c2;
  __device__ __forceinline__ void init(double c1, double s1) {
    c = 1.0;
    s = 0.0;
    cp = c1;
    sp = -s1;
    c2 = c1 + c1;
  }
  __device__ __forceinline__ void step() {
    const double cn = fma(c2, c, -cp);
    const double sn = fma(c2, s, -sp);
    cp = c;
    sp = s;
    c = cn;
    s = sn;
  }
};


// Spatial forms the kernels are instantiated for: NS box-pair terms, NBY vertical boxes (shared
// taps), NBX horizontal boxes per term.
template <int FORM>
struct Form;
template <> struct Form<1> { static constexpr int NS = 1, NBY = 1, NBX = 1; };   // one box (box K_s)
template <> struct Form<2> { static constexpr int NS = 1, NBY = 2, NBX = 2; };   // separable, 2 nested boxes (N_s = 9)
template <> struct Form<4> { static constexpr int NS = 1, NBY = 4, NBX = 4; };   // separable, up to 4 boxes
template <> struct Form<5> { static constexpr int NS = 2, NBY = 2, NBX = 1; };   // rank 2 (N_s = 5, three boxes)

// ------------------------------------------------------------------ the four steps of a row
// They are shared by the two kernels below (barrier-interval kernel, warp-specialised kernel).

// Vertical state at row y0 - 1: U = urnd + sum over the rows v of the vertical boxes of the
// quantised channels (every tap's scale carries the box weight, nested boxes add up).
template <int MAXK, int NB, int NS, bool U8, bool CONSEC, bool FULL>
__device__ __forceinline__ void v_init(const KParams& P, const void* __restrict__ in, const float2* lut,
                                       long long fbase, int col, bool colok, int y0, int (&U)[NS * 4 * MAXK]) {
  const int nk = P.nk;
#pragma unroll
  for (int ch = 0; ch < NS * 4 * MAXK; ++ch) U[ch] = P.urnd;
  for (int v = P.vmin; v <= P.vmax; ++v) {
    const int row = y0 - 1 + v;
    const bool ok = colok && row >= 0 && row < P.H;
    const float I = ok ? load_pixel(in, U8, fbase + (long long)row * P.W + col) : 0.f;
    float c1, s1;
    if (U8) {
      const float2 t = lut[(int)I];
      c1 = t.x;
      s1 = t.y;
    } else {
      base_angle_f32(I, P, c1, s1);
    }
    float scb[NS][NB], scIb[NS][NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const bool in_b = ok && (b < P.nby) && v >= P.vlo[b] && v <= P.vhi[b];
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        scb[t][b] = in_b ? P.qs[t][b] : 0.f;
        scIb[t][b] = in_b ? P.qsD[t][b] * I : 0.f;
      }
    }
    float gc = 1.f, gs = 0.f;
    for (int j = 0; j < P.kstep[0]; ++j) rot1(gc, gs, c1, s1);
#pragma unroll
    for (int i = 0; i < MAXK; ++i) {
      if (FULL || i < nk) {
        if (i > 0) {
          if (CONSEC) rot1(gc, gs, c1, s1);
          else
            for (int j = 0; j < P.kstep[i]; ++j) rot1(gc, gs, c1, s1);   // (init rows only)
        }
#pragma unroll
        for (int t = 0; t < NS; ++t)
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            int* Ut = U + t * 4 * MAXK;
            Ut[4 * i + 0] += quant(gc, scb[t][b]);
            Ut[4 * i + 1] += quant(gs, scb[t][b]);
            Ut[4 * i + 2] += quant(gc, scIb[t][b]);
            Ut[4 * i + 3] += quant(gs, scIb[t][b]);
          }
      }
    }
  }
}

// input pixels of the taps of output row y, box b: enter y + vhi_b, leave y + vlo_b - 1
template <int NB, bool U8>
__device__ __forceinline__ void load_taps(const KParams& P, const void* __restrict__ in, long long fbase, int col,
                                          bool colok, int y, float (&Ipre)[NB][2]) {
#pragma unroll
  for (int b = 0; b < NB; ++b) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int row = y + (j ? (P.vlo[b] - 1) : P.vhi[b]);
      const bool ok = (b < P.nby) && colok && row >= 0 && row < P.H;
      Ipre[b][j] = ok ? load_pixel(in, U8, fbase + (long long)row * P.W + col) : 0.f;
    }
  }
}

// V(y): slide the vertical state one row (enter / leave taps of every box, packed in pairs)
// and store U' = U >> ush of every channel slot at Ucol[slot * UP].
struct GroupSync;   // per-channel-group barriers of the warp-specialised kernel (defined with it)

template <int MAXK, int NB, int NS, bool U8, bool CONSEC, bool FULL, int UP, class Hook = GroupSync>
__device__ __forceinline__ void v_row(const KParams& P, const float2* lut, bool colok, int y, const float (&Ipre)[NB][2],
                                      int (&U)[NS * 4 * MAXK], int* Ucol, const Hook* hook = nullptr) {
  const int nk = P.nk;
  u64 QS[NS][NB], QI[NS][NB];
  Rot2 g2[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const float Ie = Ipre[b][0], Il = Ipre[b][1];
    if (U8) {
      const float2 te = lut[(int)Ie], tl = lut[(int)Il];
      g2[b].init(te.x, te.y, tl.x, tl.y);
    } else {
      u64 c1, s1;
      base_angle_f32x2(Ie, Il, P, c1, s1);
      g2[b].init2(c1, s1);
    }
    const int re = y + P.vhi[b], rl = y + P.vlo[b] - 1;
    const bool oke = (b < P.nby) && colok && re >= 0 && re < P.H;
    const bool okl = (b < P.nby) && colok && rl >= 0 && rl < P.H;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      QS[t][b] = pk(oke ? P.qs[t][b] : 0.f, okl ? P.qs[t][b] : 0.f);
      QI[t][b] = pk(oke ? P.qsD[t][b] * Ie : 0.f, okl ? P.qsD[t][b] * Il : 0.f);
    }
    for (int j = 0; j < P.kstep[0]; ++j) g2[b].step();
  }
  const u64 MM = pk(MAGIC, MAGIC);
#pragma unroll
  for (int i = 0; i < MAXK; ++i) {
    if (FULL || i < nk) {
      if (hook && (i & 7) == 0) hook->begin(i >> 3);   // channel group i / 8 starts: its buffer free
      if (i > 0) {   // k_i - k_{i-1} >= 1 recurrence steps, all boxes under one loop test
#pragma unroll
        for (int b = 0; b < NB; ++b) g2[b].step();
        if (!CONSEC)
          for (int j = 1; j < P.kstep[i]; ++j)
#pragma unroll
            for (int b = 0; b < NB; ++b) g2[b].step();
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const u64 C = g2[b].C, Sn = g2[b].S;
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          int* Ut = U + t * 4 * MAXK;
          Ut[4 * i + 0] += diff_bits(fma2(C, QS[t][b], MM));
          Ut[4 * i + 1] += diff_bits(fma2(Sn, QS[t][b], MM));
          Ut[4 * i + 2] += diff_bits(fma2(C, QI[t][b], MM));
          Ut[4 * i + 3] += diff_bits(fma2(Sn, QI[t][b], MM));
        }
      }
#pragma unroll
      for (int t = 0; t < NS; ++t)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          Ucol[(t * 4 * nk + 4 * i + c) * UP] = U[t * 4 * MAXK + 4 * i + c] >> P.ush;
      // channel group i / 8 written (FULL: the last term is known at compile time)
      if (hook && ((i & 7) == 7 || (FULL ? i + 1 == MAXK : i + 1 == nk))) hook->end(i >> 3);
    }
  }
}

// H(y) for one channel slot over output columns [xs, xe): slide the exact int32 horizontal box
// sums H_tb of U'_t (term t, box b) and write F = sum_tb mulhi(H_tb, ax_tb) (int64 products,
// narrowed) to Fcol[x * FPX]. Ur[o + u] is U'_0 at output column o, offset u; U'_t = Ur + t*srow.
template <int NB, int NS, int FPX>
__device__ __forceinline__ void walk_row(const KParams& P, const int* Ur, int srow, int* Fcol, int xs, int xe) {
  constexpr int M = NS * NB;   // (term, box) streams
  int hlo[M], hhi[M], ax[M];
  int Hs[M];
  const int* base[M];
#pragma unroll
  for (int t = 0; t < NS; ++t)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int m = t * NB + b;
      const bool on = b < P.nbx[t];
      hlo[m] = on ? P.hlo[t][b] : 0;
      hhi[m] = on ? P.hhi[t][b] : -1;   // empty box: no taps, H = 0
      ax[m] = on ? P.ax[t][b] : 0;
      base[m] = Ur + t * srow;
    }
  // initial window sums at xs; a box nested in the previous box of its term reuses the inner sum
#pragma unroll
  for (int t = 0; t < NS; ++t)
#pragma unroll
    for (int b = NB - 1; b >= 0; --b) {
      const int m = t * NB + b;
      const int* Urt = base[m];
      int lo = xs + hlo[m], hi = xs + hhi[m];
      int acc = 0, lo2 = hi + 1, hi2 = hi;
      if (b + 1 < NB && hhi[m + 1] >= hlo[m + 1] && hlo[m] <= hlo[m + 1] && hhi[m + 1] <= hhi[m]) {
        acc = Hs[m + 1];
        lo2 = xs + hhi[m + 1] + 1;
        hi = xs + hlo[m + 1] - 1;
      }
      int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        int j = pass ? lo2 : lo;
        const int je = pass ? hi2 : hi;
        for (; j + 3 <= je; j += 4) {
          a0 += Urt[j];
          a1 += Urt[j + 1];
          a2 += Urt[j + 2];
          a3 += Urt[j + 3];
        }
        for (; j <= je; ++j) a0 += Urt[j];
      }
      Hs[m] = acc + (a0 + a1) + (a2 + a3);
    }
  const int* pe[M];
  const int* pl[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    pe[m] = base[m] + xs + 1 + hhi[m];
    pl[m] = base[m] + xs + hlo[m];
  }
  int* pf = Fcol + xs * FPX;
  // software-pipelined: the taps of the next 4 outputs are loaded while these 4 are formed
  // (reads past the segment end stay inside the shared-memory carve-up and are discarded)
  int en[M][4], ln[M][4];
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      en[m][j] = pe[m][j];
      ln[m][j] = pl[m][j];
    }
  int x = xs;
  for (; x + 4 <= xe; x += 4) {
    int e[M][4], l[M][4];
#pragma unroll
    for (int m = 0; m < M; ++m) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        e[m][j] = en[m][j];
        l[m][j] = ln[m][j];
      }
      pe[m] += 4;
      pl[m] += 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        en[m][j] = pe[m][j];
        ln[m][j] = pl[m][j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int f = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) f += __mulhi(Hs[m], ax[m]);
      pf[j * FPX] = f;
#pragma unroll
      for (int m = 0; m < M; ++m) Hs[m] += e[m][j] - l[m][j];
    }
    pf += 4 * FPX;
  }
  for (int j = 0; x < xe; ++x, ++j) {   // tail (< 4 outputs)
    int f = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) f += __mulhi(Hs[m], ax[m]);
    *pf = f;
    pf += FPX;
#pragma unroll
    for (int m = 0; m < M; ++m) Hs[m] += pe[m][j] - pl[m][j];
  }
}

// walk_row for symmetric odd-width boxes (one box per stream pair, at most two pairs), with
// 64-bit shared-memory loads: the U' rows have an even pitch and the segments start at even x, so
// every leave stream has a fixed parity (box 0 even, box 1 even iff LPAR1 == 0) and its enter
// stream the opposite one (the box width 2r + 1 is odd). Even streams read aligned pairs; odd
// streams carry the high word of the previous pair. Half the load instructions of walk_row for
// the same shared-memory words. Same arithmetic as walk_row (bitwise equal results).
template <int M, int FPX, int LPAR1>
__device__ __forceinline__ void walk_row_pairs(const KParams& P, const int* Ur, int srow, int* Fcol, int xs, int xe) {
  int lo[M], hi[M], ax[M], Hs[M];
  const int* base[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int t = (M == 2 && P.ns == 2) ? m : 0;    // rank 2: one box per term
    const int b = (M == 2 && P.ns == 2) ? 0 : m;
    lo[m] = P.hlo[t][b];
    hi[m] = P.hhi[t][b];
    ax[m] = P.ax[t][b];
    base[m] = Ur + t * srow;
  }
  // initial window sums at xs (inner box first, the outer one reuses it when nested)
#pragma unroll
  for (int m = M - 1; m >= 0; --m) {
    const int* U = base[m];
    int a = xs + lo[m], b = xs + hi[m];
    int acc = 0, a2 = b + 1, b2 = b;
    if (M == 2 && m == 0 && P.ns == 1 && lo[0] <= lo[1] && hi[1] <= hi[0]) {
      acc = Hs[1];
      a2 = xs + hi[1] + 1;
      b = xs + lo[1] - 1;
    }
    int s0 = 0, s1 = 0;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      int j = pass ? a2 : a;
      const int je = pass ? b2 : b;
      if (j <= je && ((reinterpret_cast<uintptr_t>(U + j) >> 2) & 1)) s0 += U[j++];   // to an even word
      for (; j + 1 <= je; j += 2) {
        const int2 v = *reinterpret_cast<const int2*>(U + j);
        s0 += v.x;
        s1 += v.y;
      }
      if (j <= je) s0 += U[j];
    }
    Hs[m] = acc + s0 + s1;
  }
  // stream pointers: leave at xs + lo (parity lpar), enter at xs + hi + 1 (parity 1 - lpar)
  const int* pl[M];
  const int* pe[M];
  int cl[M], ce[M];   // carried high words of the odd streams
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int lpar = (m == 1) ? LPAR1 : 0;
    pl[m] = base[m] + xs + lo[m] - lpar;          // even word
    pe[m] = base[m] + xs + hi[m] + 1 - (1 - lpar);
    if (lpar) cl[m] = pl[m][1];
    else ce[m] = pe[m][1];
  }
  int* pf = Fcol + xs * FPX;
  int x = xs;
  for (; x + 4 <= xe; x += 4) {
    int e[M][4], l[M][4];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int lpar = (m == 1) ? LPAR1 : 0;
      if (lpar == 0) {   // leave even: aligned pairs at pl, pl + 2; enter odd: carry + pairs at pe + 2, pe + 4
        const int2 a0 = *reinterpret_cast<const int2*>(pl[m]);
        const int2 a1 = *reinterpret_cast<const int2*>(pl[m] + 2);
        const int2 b0 = *reinterpret_cast<const int2*>(pe[m] + 2);
        const int2 b1 = *reinterpret_cast<const int2*>(pe[m] + 4);
        l[m][0] = a0.x; l[m][1] = a0.y; l[m][2] = a1.x; l[m][3] = a1.y;
        e[m][0] = ce[m]; e[m][1] = b0.x; e[m][2] = b0.y; e[m][3] = b1.x;
        ce[m] = b1.y;
      } else {           // leave odd, enter even
        const int2 a0 = *reinterpret_cast<const int2*>(pl[m] + 2);
        const int2 a1 = *reinterpret_cast<const int2*>(pl[m] + 4);
        const int2 b0 = *reinterpret_cast<const int2*>(pe[m]);
        const int2 b1 = *reinterpret_cast<const int2*>(pe[m] + 2);
        l[m][0] = cl[m]; l[m][1] = a0.x; l[m][2] = a0.y; l[m][3] = a1.x;
        cl[m] = a1.y;
        e[m][0] = b0.x; e[m][1] = b0.y; e[m][2] = b1.x; e[m][3] = b1.y;
      }
      pl[m] += 4;
      pe[m] += 4;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int f = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) f += __mulhi(Hs[m], ax[m]);
      pf[j * FPX] = f;
#pragma unroll
      for (int m = 0; m < M; ++m) Hs[m] += e[m][j] - l[m][j];
    }
    pf += 4 * FPX;
  }
  for (; x < xe; ++x) {   // tail (< 4 outputs): scalar
    int f = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) f += __mulhi(Hs[m], ax[m]);
    *pf = f;
    pf += FPX;
#pragma unroll
    for (int m = 0; m < M; ++m) Hs[m] += base[m][x + 1 + hi[m]] - base[m][x + lo[m]];
  }
}

// F from exclusive prefix rows (no window init, no dependency between outputs): Q[e] holds
// sum_{e' < e} U'[e'] (mod 2^32: the box differences are exact because every box sum fits
// int32), so H_m(x) = Q[x + hi + 1] - Q[x + lo] is read with the same paired loads as the
// walker's enter / leave streams.
template <int M, int FPX, int LPAR1>
__device__ __forceinline__ void prefix_row_pairs(const KParams& P, const int* Ur, int srow, int* Fcol, int xs, int xe) {
  int lo[M], hi[M], ax[M];
  const int* base[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int t = (M == 2 && P.ns == 2) ? m : 0;    // rank 2: one box per term
    const int b = (M == 2 && P.ns == 2) ? 0 : m;
    lo[m] = P.hlo[t][b];
    hi[m] = P.hhi[t][b];
    ax[m] = P.ax[t][b];
    base[m] = Ur + t * srow;
  }
  // stream pointers: leave at xs + lo (parity lpar), enter at xs + hi + 1 (parity 1 - lpar)
  const int* pl[M];
  const int* pe[M];
  int cl[M], ce[M];   // carried high words of the odd streams
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int lpar = (m == 1) ? LPAR1 : 0;
    pl[m] = base[m] + xs + lo[m] - lpar;          // even word
    pe[m] = base[m] + xs + hi[m] + 1 - (1 - lpar);
    if (lpar) cl[m] = pl[m][1];
    else ce[m] = pe[m][1];
  }
  int* pf = Fcol + xs * FPX;
  int x = xs;
  for (; x + 4 <= xe; x += 4) {
    int e[M][4], l[M][4];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int lpar = (m == 1) ? LPAR1 : 0;
      if (lpar == 0) {   // leave even: aligned pairs at pl, pl + 2; enter odd: carry + pairs at pe + 2, pe + 4
        const int2 a0 = *reinterpret_cast<const int2*>(pl[m]);
        const int2 a1 = *reinterpret_cast<const int2*>(pl[m] + 2);
        const int2 b0 = *reinterpret_cast<const int2*>(pe[m] + 2);
        const int2 b1 = *reinterpret_cast<const int2*>(pe[m] + 4);
        l[m][0] = a0.x; l[m][1] = a0.y; l[m][2] = a1.x; l[m][3] = a1.y;
        e[m][0] = ce[m]; e[m][1] = b0.x; e[m][2] = b0.y; e[m][3] = b1.x;
        ce[m] = b1.y;
      } else {           // leave odd, enter even
        const int2 a0 = *reinterpret_cast<const int2*>(pl[m] + 2);
        const int2 a1 = *reinterpret_cast<const int2*>(pl[m] + 4);
        const int2 b0 = *reinterpret_cast<const int2*>(pe[m]);
        const int2 b1 = *reinterpret_cast<const int2*>(pe[m] + 2);
        l[m][0] = cl[m]; l[m][1] = a0.x; l[m][2] = a0.y; l[m][3] = a1.x;
        cl[m] = a1.y;
        e[m][0] = b0.x; e[m][1] = b0.y; e[m][2] = b1.x; e[m][3] = b1.y;
      }
      pl[m] += 4;
      pe[m] += 4;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int f = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) f += __mulhi(e[m][j] - l[m][j], ax[m]);   // box sum = Q[hi+1] - Q[lo]
      pf[j * FPX] = f;
    }
    pf += 4 * FPX;
  }
  for (; x < xe; ++x) {   // tail (< 4 outputs): scalar
    int f = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) f += __mulhi(base[m][x + 1 + hi[m]] - base[m][x + lo[m]], ax[m]);
    *pf = f;
    pf += FPX;
  }
}

// H(y) dispatch: the paired-load walker when the host found the box layout for it (wpar >= 0)
template <int NBX, int NS, int FPX>
__device__ __forceinline__ void walk(const KParams& P, const int* Ur, int srow, int* Fcol, int xs, int xe) {
  constexpr int M = NS * NBX;
  if constexpr (M <= 2) {
    if (P.wpar == 0) return walk_row_pairs<M, FPX, 0>(P, Ur, srow, Fcol, xs, xe);
    if (P.wpar == 1) return walk_row_pairs<M, FPX, 1>(P, Ur, srow, Fcol, xs, xe);
  }
  walk_row<NBX, NS, FPX>(P, Ur, srow, Fcol, xs, xe);
}

// C: num = sum_k W_c F_Ic + W_s F_Is, den = sum_k W_c F_c + W_s F_s for one output pixel with
// the weights a_k cos / sin(k pi I(x) / D) in fp64 rounded to int32 (exact int64 sums); then
// out = D num / den (den <= 0: out = I(x), Q18), or the int64 pair to the multi-pass workspace.
template <int MAXK, bool U8, bool CONSEC, bool FULL, bool MULTI>
__device__ __forceinline__ void combine_pixel(const KParams& P, const double2* lut64, const int4* Fr, float Ic,
                                              long long pix, float* __restrict__ out, longlong2* __restrict__ ws) {
  const int nk = P.nk;
  double c1, s1;
  if (U8) {
    const double2 t = lut64[(int)Ic];
    c1 = t.x;
    s1 = t.y;
  } else {
    base_angle_f64(Ic, P.invD, c1, s1);
  }
  Cheb64 g;
  g.init(c1, s1);
  for (int j = 0; j < P.kstep[0]; ++j) g.step();
  long long num = 0, den = 0;
#pragma unroll
  for (int i = 0; i < MAXK; ++i) {
    if (FULL || i < nk) {
      if (i > 0) {
        if (CONSEC) g.step();
        else
          for (int j = 0; j < P.kstep[i]; ++j) g.step();
      }
      const int wc = __double2loint(fma(g.c, P.aw[0][i], MAGIC64));
      const int wsn = __double2loint(fma(g.s, P.aw[0][i], MAGIC64));
      const int4 f = Fr[i];   // (F_c, F_s, F_Ic, F_Is) of term i
      den += (long long)wc * f.x;
      den += (long long)wsn * f.y;
      num += (long long)wc * f.z;
      num += (long long)wsn * f.w;
    }
  }
  if (MULTI) {   // bf_apply_multi: plans 1.. reuse the same F (single pass, no workspace)
    out[pix] = (den > 0) ? (float)(P.D * (double)num / (double)den) : Ic;
    g.init(c1, s1);
    for (int j = 0; j < P.kstep[0]; ++j) g.step();
    long long nu[MAXP - 1] = {}, de[MAXP - 1] = {};
#pragma unroll
    for (int i = 0; i < MAXK; ++i) {
      if (FULL || i < nk) {
        if (i > 0) {
          if (CONSEC) g.step();
          else
            for (int j = 0; j < P.kstep[i]; ++j) g.step();
        }
        const int4 f = Fr[i];
#pragma unroll
        for (int q = 1; q < MAXP; ++q) {
          if (q < P.nplans) {
            const int wc = __double2loint(fma(g.c, P.aw[q][i], MAGIC64));
            const int wsn = __double2loint(fma(g.s, P.aw[q][i], MAGIC64));
            de[q - 1] += (long long)wc * f.x + (long long)wsn * f.y;
            nu[q - 1] += (long long)wc * f.z + (long long)wsn * f.w;
          }
        }
      }
    }
#pragma unroll
    for (int q = 1; q < MAXP; ++q)
      if (q < P.nplans)
        out[pix + q * P.plan_stride] = (de[q - 1] > 0) ? (float)(P.D * (double)nu[q - 1] / (double)de[q - 1]) : Ic;
    return;
  }
  if (P.pass == 1) {
    ws[pix] = make_longlong2(num, den);
  } else {
    if (P.pass >= 2) {
      const longlong2 acc = ws[pix];
      num += acc.x;
      den += acc.y;
    }
    if (P.pass == 2) ws[pix] = make_longlong2(num, den);
    else out[pix] = (den > 0) ? (float)(P.D * (double)num / (double)den) : Ic;
  }
}

template <bool U8>
__device__ __forceinline__ void fill_luts(const KParams& P, float2* lut, double2* lut64, int tid, int nthreads) {
  if (U8) {
    for (int i = tid; i < 256; i += nthreads) {
      double s, c;
      sincospi((double)i * P.invD, &s, &c);
      lut[i] = make_float2((float)c, (float)s);
      lut64[i] = make_double2(c, s);
    }
  }
}

// ------------------------------------------------------------------ kernel 1: barrier intervals
// One thread per extended column; per row interval A = V(y) + C(y-1), interval B = H(y).
// Used for wide halos (NT = 512) and as the reference structure.
template <int MAXK, int NT>
struct Occ {
  static constexpr int value = NT > 256 ? 1 : 2;
};

// FULL: nk == MAXK (no per-term runtime checks). CONSEC: the selected k are consecutive.
template <int MAXK, int FORM, bool U8, int NT, bool CONSEC, bool FULL, bool MULTI>
__global__ void __launch_bounds__(NT, (Occ<MAXK, NT>::value))
    bf_band_kernel(const KParams P, const void* __restrict__ in, float* __restrict__ out,
                   longlong2* __restrict__ ws) {
  constexpr int NS = Form<FORM>::NS, NB = Form<FORM>::NBY, NBX = Form<FORM>::NBX;
  constexpr int UP = NT + 1;           // channel-row pitch (== 1 mod 32: lanes = channels are conflict-free)
  constexpr int FPX = 4 * MAXK + 4;    // F pitch per output column (4 * odd: conflict-free int4 reads)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* Ubuf = reinterpret_cast<int*>(smem_raw);                               // [NS][4 nk][UP]
  int* Fbuf = reinterpret_cast<int*>(smem_raw + P.f_off);                     // [TW][FPX]
  float2* lut = reinterpret_cast<float2*>(smem_raw + P.l_off);                // [256]
  double2* lut64 = reinterpret_cast<double2*>(lut + 256);                     // [256]

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P.TW;
  const int y0 = P.yb + blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int col = x0 - P.rlo_x + tid;
  const bool colok = (col >= 0) & (col < P.W);
  const int TWv = min(P.TW, P.W - x0);
  const int yend = min(y0 + P.TH, P.ye);

  fill_luts<U8>(P, lut, lut64, tid, NT);
  if (U8) __syncthreads();
  int U[NS * 4 * MAXK];
  v_init<MAXK, NB, NS, U8, CONSEC, FULL>(P, in, lut, fbase, col, colok, y0, U);
  float Ipre[NB][2];
  load_taps<NB, U8>(P, in, fbase, col, colok, y0, Ipre);

  // walker of this thread (interval B): lane = channel slot, warp = (slot group, segment)
  const int wgrp = (tid >> 5) % P.ngrp;
  const int wseg = (tid >> 5) / P.ngrp;
  const int wslot = wgrp * 32 + (tid & 31);
  const bool wact = (wslot < 4 * P.nk) && (wseg < P.nseg);
  float Ic = 0.f;   // I(y - 1, x0 + tid) for the combine of row y - 1 (threads < TWv)

  for (int y = y0; y <= yend; ++y) {
    // ============================================================ interval A
    if (y < yend) {
      float Icur[NB][2];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        Icur[b][0] = Ipre[b][0];
        Icur[b][1] = Ipre[b][1];
      }
      if (y + 1 < yend) load_taps<NB, U8>(P, in, fbase, col, colok, y + 1, Ipre);   // prefetch
      v_row<MAXK, NB, NS, U8, CONSEC, FULL, UP>(P, lut, colok, y, Icur, U, Ubuf + tid);
    }
    if (y > y0 && tid < TWv)
      combine_pixel<MAXK, U8, CONSEC, FULL, MULTI>(P, lut64, reinterpret_cast<const int4*>(Fbuf + tid * FPX), Ic,
                                            fbase + (long long)(y - 1) * P.W + x0 + tid, out, ws);
    if (y >= yend) break;
    if (tid < TWv) Ic = load_pixel(in, U8, fbase + (long long)y * P.W + x0 + tid);
    __syncthreads();
    // ============================================================ interval B: H(y)
    if (wact) {
      const int xs = wseg * P.seglen;
      const int xe = min(xs + P.seglen, TWv);
      if (xs < xe) walk_row<NBX, NS, FPX>(P, Ubuf + wslot * UP + P.rlo_x, 4 * P.nk * UP, Fbuf + wslot, xs, xe);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ kernel 2: warp-specialised
// Four warp roles connected by double-buffered shared-memory rows and named barriers, pipelined
// per 32-channel group (a group = 8 terms = one walker warp's lanes), so the vertical pass of
// row y+1, the horizontal pass of row y and the combine of row y-1 overlap:
//   warps 0-7    V: one thread per extended column (NT = 256), writes U'(y) group by group
//   warps 8-9    S: warp g turns group g's U' rows into exclusive prefix rows Q in place
//   warps 10-15  F: box sums Q[x + hi + 1] - Q[x + lo] -> F rows (warp = group x segment)
//   warps 16-19  C: combine / normalise / store, F -> output
// Registers are redistributed with setmaxnreg (V 152, S / F / C 56; 640 x 96 at launch). Named
// barriers (all 16, barrier 0 reused after the opening __syncthreads):
//   U_FULL(b,g) 0-3   V arrive, S_g sync        U_EMPTY(b,g) 4-7  F_g arrive, V sync
//   Q_FULL(b,g) 8-11  S_g arrive, F_g sync      F_FULL(b) 12-13   F arrive, C sync
//   F_EMPTY(b) 14-15  C arrive, F sync          (b = row parity, g = channel group)
constexpr int WS_V = 256, WS_S = 64, WS_F = 192, WS_C = 128, WS_THREADS = WS_V + WS_S + WS_F + WS_C;
constexpr int WS_H = WS_S + WS_F;
constexpr int KERN_BAND = 0, KERN_WS = 1, KERN_WS2 = 2;
constexpr int BAR_U_FULL = 0, BAR_U_EMPTY = 4, BAR_Q_FULL = 8, BAR_F_FULL = 12, BAR_F_EMPTY = 14;

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// V's per-group hooks: wait until group g's buffer of this row parity is free (F_g done with
// row y-2), and publish group g once written
struct GroupSync {
  int b, nfree, nfull;
  bool wait;
  __device__ __forceinline__ void begin(int g) const {
    if (wait) bar_sync(BAR_U_EMPTY + 2 * b + g, nfree);
  }
  __device__ __forceinline__ void end(int g) const { bar_arrive(BAR_U_FULL + 2 * b + g, nfull); }
};

template <int MAXK, int FORM, bool U8, bool CONSEC, bool FULL, bool MULTI>
__global__ void __launch_bounds__(WS_THREADS, 1)
    bf_ws_kernel(const KParams P, const void* __restrict__ in, float* __restrict__ out, longlong2* __restrict__ ws) {
  constexpr int NS = Form<FORM>::NS, NB = Form<FORM>::NBY, NBX = Form<FORM>::NBX;
  constexpr int M = NS * NBX;
  static_assert(M <= 2, "the prefix-form H role handles at most two horizontal boxes");
  constexpr int NT = WS_V;
  constexpr int UP = NT + 2;           // even pitch (== 2 mod 64): conflict-free LDS.64 with lanes = channels
  constexpr int FPX = 4 * MAXK + 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int srow = 4 * P.nk * UP;                                             // ints per term's U' rows
  const int ustride = NS * srow;                                              // ints per U' buffer
  int* Ubuf = reinterpret_cast<int*>(smem_raw);                               // [2][NS][4 nk][UP]
  int* Fbuf = reinterpret_cast<int*>(smem_raw + P.f_off);                     // [2][TW][FPX]
  const int fstride = P.TW * FPX;
  float2* lut = reinterpret_cast<float2*>(smem_raw + P.l_off);
  double2* lut64 = reinterpret_cast<double2*>(lut + 256);

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P.TW;
  const int y0 = P.yb + blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int TWv = min(P.TW, P.W - x0);
  const int yend = min(y0 + P.TH, P.ye);
  const int ngrp = P.ngrp;                       // channel groups (1 or 2)
  const int nfw = (WS_F / 32) / ngrp;            // F warps per group
  const int n_uempty = WS_V + 32 * nfw;          // U_EMPTY: F_g arrive, V sync
  const int n_ufull = WS_V + 32;                 // U_FULL: V arrive, S_g sync
  const int n_qfull = 32 + 32 * nfw;             // Q_FULL: S_g arrive, F_g sync
  constexpr int n_f = WS_F + WS_C;               // F_FULL / F_EMPTY

  fill_luts<U8>(P, lut, lut64, tid, WS_THREADS);
  __syncthreads();

  if (tid < WS_V) {
    // ------------------------------------------------------------ V role
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;");
    const int col = x0 - P.rlo_x + tid;
    const bool colok = (col >= 0) & (col < P.W);
    int U[NS * 4 * MAXK];
    v_init<MAXK, NB, NS, U8, CONSEC, FULL>(P, in, lut, fbase, col, colok, y0, U);
    float Ipre[NB][2];
    load_taps<NB, U8>(P, in, fbase, col, colok, y0, Ipre);
    for (int y = y0; y < yend; ++y) {
      const int b = (y - y0) & 1;
      float Icur[NB][2];
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
        Icur[bb][0] = Ipre[bb][0];
        Icur[bb][1] = Ipre[bb][1];
      }
      if (y + 1 < yend) load_taps<NB, U8>(P, in, fbase, col, colok, y + 1, Ipre);
      const GroupSync hook{b, n_uempty, n_ufull, y - y0 >= 2};
      v_row<MAXK, NB, NS, U8, CONSEC, FULL, UP>(P, lut, colok, y, Icur, U, Ubuf + b * ustride + tid, &hook);
    }
    // drain: the F warps' last releases
    for (int y = max(y0, yend - 2); y < yend; ++y)
      for (int g = 0; g < ngrp; ++g) bar_sync(BAR_U_EMPTY + 2 * ((y - y0) & 1) + g, n_uempty);
  } else if (tid < WS_V + WS_S) {
    // ------------------------------------------------------------ S role: prefix scans
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    const int g = (tid - WS_V) >> 5;
    if (g < ngrp) {
      const int slot = 32 * g + (tid & 31);
      const bool act = slot < 4 * P.nk;
      for (int y = y0; y < yend; ++y) {
        const int b = (y - y0) & 1;
        bar_sync(BAR_U_FULL + 2 * b + g, n_ufull);
        if (act) {
#pragma unroll
          for (int t = 0; t < NS; ++t) {
            int* Q = Ubuf + b * ustride + t * srow + slot * UP;
            // exclusive prefix in place, 8 columns per step: the carry chain is one add per 8
            // columns (rows are 8-byte aligned: pitch NT + 2); int32 wrap-around keeps every box
            // difference exact (each box sum fits int32)
            int carry = 0;
#pragma unroll 2
            for (int e = 0; e < NT; e += 8) {
              const int2 a0 = *reinterpret_cast<const int2*>(Q + e), a1 = *reinterpret_cast<const int2*>(Q + e + 2);
              const int2 b0 = *reinterpret_cast<const int2*>(Q + e + 4), b1 = *reinterpret_cast<const int2*>(Q + e + 6);
              const int p1 = a0.x, p2 = a0.x + a0.y, p3 = p2 + a1.x, p4 = p3 + a1.y;
              const int q1 = b0.x, q2 = b0.x + b0.y, q3 = q2 + b1.x, q4 = q3 + b1.y;
              const int c4 = carry + p4;
              *reinterpret_cast<int2*>(Q + e) = make_int2(carry, carry + p1);
              *reinterpret_cast<int2*>(Q + e + 2) = make_int2(carry + p2, carry + p3);
              *reinterpret_cast<int2*>(Q + e + 4) = make_int2(c4, c4 + q1);
              *reinterpret_cast<int2*>(Q + e + 6) = make_int2(c4 + q2, c4 + q3);
              carry = c4 + q4;
            }
            Q[NT] = carry;
          }
        }
        bar_arrive(BAR_Q_FULL + 2 * b + g, n_qfull);
      }
    }
  } else if (tid < WS_V + WS_H) {
    // ------------------------------------------------------------ F role: box differences
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    const int ft = tid - WS_V - WS_S;
    const int g = (ft >> 5) % ngrp;
    const int seg = (ft >> 5) / ngrp;
    const int slot = 32 * g + (ft & 31);
    const bool act = (slot < 4 * P.nk) && (seg < P.nseg);
    const int xs = seg * P.seglen;
    const int xe = min(xs + P.seglen, TWv);
    for (int y = y0; y < yend; ++y) {
      const int b = (y - y0) & 1;
      bar_sync(BAR_Q_FULL + 2 * b + g, n_qfull);
      if (y - y0 >= 2) bar_sync(BAR_F_EMPTY + b, n_f);
      if (act && xs < xe) {
        const int* Qr = Ubuf + b * ustride + slot * UP + P.rlo_x;
        int* Fr = Fbuf + b * fstride + slot;
        if (P.wpar == 0) prefix_row_pairs<M, FPX, 0>(P, Qr, srow, Fr, xs, xe);
        else prefix_row_pairs<M, FPX, 1>(P, Qr, srow, Fr, xs, xe);
      }
      bar_arrive(BAR_U_EMPTY + 2 * b + g, n_uempty);
      bar_arrive(BAR_F_FULL + b, n_f);
    }
    for (int y = max(y0, yend - 2); y < yend; ++y) bar_sync(BAR_F_EMPTY + ((y - y0) & 1), n_f);
  } else {
    // ------------------------------------------------------------ C role
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    const int ct = tid - WS_V - WS_H;
    for (int y = y0; y < yend; ++y) {
      const int b = (y - y0) & 1;
      float Iv[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int o = ct + j * WS_C;
        Iv[j] = (o < TWv) ? load_pixel(in, U8, fbase + (long long)y * P.W + x0 + o) : 0.f;
      }
      bar_sync(BAR_F_FULL + b, n_f);
#pragma unroll 1
      for (int j = 0; j < 2; ++j) {
        const int o = ct + j * WS_C;
        if (o < TWv)
          combine_pixel<MAXK, U8, CONSEC, FULL, MULTI>(P, lut64, reinterpret_cast<const int4*>(Fbuf + b * fstride + o * FPX),
                                                       Iv[j], fbase + (long long)y * P.W + x0 + o, out, ws);
      }
      bar_arrive(BAR_F_EMPTY + b, n_f);
    }
  }
}

// ------------------------------------------------------------------ kernel 2b: fused box-difference + combine
// Three roles; the F row buffer of kernel 2 is gone, which pays for 384 extended columns
// (TW = min(320, 384 - halo) outputs: halo overhead 1.33x instead of 1.6x at r = 48):
//   warps 12-23  V: one thread per extended column, writes U'(y) group by group (as kernel 2)
//   warps 10-11  S: warp g turns group g's U' rows into exclusive prefix rows Q in place
//   warps 0-9    FH: one thread per output pixel: for every channel slot of group g,
//                F = sum_b mulhi(Q[x + hi_b + 1] - Q[x + lo_b], ax_b) (lanes = consecutive
//                x: conflict-free), accumulated straight into the exact int64 num / den with the
//                pixel's fp64 combine weights (per range plan for bf_apply_multi); then out = D num / den
// setmaxnreg: V 112, S / FH 48 (768 x 80 at launch). Named barriers:
//   U_FULL(b,g) 0-3   V arrive, S_g sync        U_EMPTY(b,g) 4-7  FH arrive, V sync
//   Q_FULL(b,g) 8-11  S_g arrive, FH sync       (b = row parity, g = channel group)
constexpr int W2_V = 384, W2_S = 64, W2_H = 320, W2_THREADS = W2_V + W2_S + W2_H;
// thread ranges of the roles: FH first (warps 0-9), then S (10-11), then V (12-23) — the warp
// schedulers favour older (lower) warps, and FH is the role on the critical path
constexpr int W2_H0 = 0, W2_S0 = W2_H, W2_V0 = W2_H + W2_S;
constexpr int W2_UP = W2_V + 4;   // == 4 mod 32: conflict-free LDS.128 / STS.128 with lanes = channels

// Exclusive prefix of one U' row in place, 8 columns per step (two 16-byte loads / stores, one
// IADD3 per column); int32 wrap-around keeps every box difference exact. Q[n] = total.
__device__ __forceinline__ void prefix_row(int* Q, int n) {
  int carry = 0;
#pragma unroll 8
  for (int e = 0; e < n; e += 8) {
    const int4 a = *reinterpret_cast<const int4*>(Q + e), b = *reinterpret_cast<const int4*>(Q + e + 4);
    const int o1 = carry + a.x;
    const int o2 = carry + a.x + a.y;
    const int o3 = o1 + a.y + a.z;
    const int o4 = o2 + a.z + a.w;
    const int o5 = o3 + a.w + b.x;
    const int o6 = o4 + b.x + b.y;
    const int o7 = o5 + b.y + b.z;
    const int o8 = o6 + b.z + b.w;
    *reinterpret_cast<int4*>(Q + e) = make_int4(carry, o1, o2, o3);
    *reinterpret_cast<int4*>(Q + e + 4) = make_int4(o4, o5, o6, o7);
    carry = o8;
  }
  Q[n] = carry;
}

// out = D num / den (den <= 0: I(x), Q18), or the int64 pair to / from the multi-pass workspace
__device__ __forceinline__ void finish_pixel(const KParams& P, long long num, long long den, float Ic, long long pix,
                                             float* __restrict__ out, longlong2* __restrict__ ws) {
  if (P.pass == 1) {
    ws[pix] = make_longlong2(num, den);
    return;
  }
  if (P.pass >= 2) {
    const longlong2 acc = ws[pix];
    num += acc.x;
    den += acc.y;
  }
  if (P.pass == 2) ws[pix] = make_longlong2(num, den);
  else out[pix] = (den > 0) ? (float)(P.D * (double)num / (double)den) : Ic;
}

template <int MAXK, int FORM, bool U8, bool CONSEC, bool FULL, bool MULTI>
__global__ void __launch_bounds__(W2_THREADS, 1)
    bf_ws2_kernel(const KParams P, const void* __restrict__ in, float* __restrict__ out, longlong2* __restrict__ ws) {
  constexpr int NS = Form<FORM>::NS, NB = Form<FORM>::NBY, NBX = Form<FORM>::NBX;
  constexpr int M = NS * NBX;
  constexpr int NPL = MULTI ? MAXP : 1;   // range plans combined per pixel
  static_assert(NS == 1 && M <= 2, "the FH role handles separable forms with at most two x boxes");
  constexpr int UP = W2_UP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int srow = 4 * P.nk * UP;                                             // ints per term's U' rows
  const int ustride = NS * srow;                                              // ints per U' buffer
  int* Ubuf = reinterpret_cast<int*>(smem_raw);                               // [2][NS][4 nk][UP]
  float2* lut = reinterpret_cast<float2*>(smem_raw + P.l_off);
  double2* lut64 = reinterpret_cast<double2*>(lut + 256);

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P.TW;
  const int y0 = P.yb + blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int TWv = min(P.TW, P.W - x0);
  const int yend = min(y0 + P.TH, P.ye);
  const int wv = P.wv;                            // extended columns scanned (multiple of 8, <= W2_V)
  const int ngrp = P.ngrp;                        // channel groups (1 or 2)
  constexpr int n_ufull = W2_V + 32;              // U_FULL: V arrive, S_g sync
  constexpr int n_uempty = W2_V + W2_H;           // U_EMPTY: FH arrive, V sync
  constexpr int n_qfull = 32 + W2_H;              // Q_FULL: S_g arrive, FH sync

  fill_luts<U8>(P, lut, lut64, tid, W2_THREADS);
  __syncthreads();

  if (tid >= W2_V0) {
    // ------------------------------------------------------------ V role
    asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    const int vt = tid - W2_V0;                   // extended column
    const int col = x0 - P.rlo_x + vt;
    const bool colok = (col >= 0) & (col < P.W) & (vt < wv);
    const bool vwork = (vt & ~31) < wv;           // warps wholly past the scanned columns only sync
    int U[NS * 4 * MAXK];
    if (vwork) v_init<MAXK, NB, NS, U8, CONSEC, FULL>(P, in, lut, fbase, col, colok, y0, U);
    float Ipre[NB][2];
    if (vwork) load_taps<NB, U8>(P, in, fbase, col, colok, y0, Ipre);
    for (int y = y0; y < yend; ++y) {
      const int b = (y - y0) & 1;
      const GroupSync hook{b, n_uempty, n_ufull, y - y0 >= 2};
      if (vwork) {
        float Icur[NB][2];
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {
          Icur[bb][0] = Ipre[bb][0];
          Icur[bb][1] = Ipre[bb][1];
        }
        if (y + 1 < yend) load_taps<NB, U8>(P, in, fbase, col, colok, y + 1, Ipre);
        v_row<MAXK, NB, NS, U8, CONSEC, FULL, UP>(P, lut, colok, y, Icur, U, Ubuf + b * ustride + vt, &hook);
      } else {
        for (int g = 0; g < ngrp; ++g) {
          hook.begin(g);
          hook.end(g);
        }
      }
    }
    // drain: the FH warps' last releases
    for (int y = max(y0, yend - 2); y < yend; ++y)
      for (int g = 0; g < ngrp; ++g) bar_sync(BAR_U_EMPTY + 2 * ((y - y0) & 1) + g, n_uempty);
  } else if (tid >= W2_S0) {
    // ------------------------------------------------------------ S role: prefix scans
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;");
    const int g = (tid - W2_S0) >> 5;
    if (g < ngrp) {
      const int slot = 32 * g + (tid & 31);
      const bool act = slot < 4 * P.nk;
      for (int y = y0; y < yend; ++y) {
        const int b = (y - y0) & 1;
        bar_sync(BAR_U_FULL + 2 * b + g, n_ufull);
        if (act) {
#pragma unroll
          for (int t = 0; t < NS; ++t) prefix_row(Ubuf + b * ustride + t * srow + slot * UP, wv);
        }
        bar_arrive(BAR_Q_FULL + 2 * b + g, n_qfull);
      }
    }
  } else {
    // ------------------------------------------------------------ FH role
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;");
    const int o = tid - W2_H0;
    const bool act = o < TWv;
    if ((o & ~31) >= TWv) {   // warp wholly past the strip: only the barriers
      for (int y = y0; y < yend; ++y) {
        const int b = (y - y0) & 1;
        for (int g = 0; g < ngrp; ++g) {
          bar_sync(BAR_Q_FULL + 2 * b + g, n_qfull);
          bar_arrive(BAR_U_EMPTY + 2 * b + g, n_uempty);
        }
      }
      return;
    }
    const int oc = act ? o : 0;
    // Q offsets (extended index o + rlo) of the x boxes: F = sum_b mulhi(Q[e_b] - Q[l_b], ax_b)
    const bool two = (M == 2) && P.nbx[0] == 2;
    const int e0 = oc + P.rlo_x + P.hhi[0][0] + 1, l0 = oc + P.rlo_x + P.hlo[0][0];
    const int e1 = two ? oc + P.rlo_x + P.hhi[0][1] + 1 : e0, l1 = two ? oc + P.rlo_x + P.hlo[0][1] : l0;
    const int ax0 = P.ax[0][0], ax1 = two ? P.ax[0][1] : 0;
    const long long prow = fbase + x0 + oc;
    float Inext = act ? load_pixel(in, U8, prow + (long long)y0 * P.W) : 0.f;
    for (int y = y0; y < yend; ++y) {
      const int b = (y - y0) & 1;
      const float Ic = Inext;
      if (act && y + 1 < yend) Inext = load_pixel(in, U8, prow + (long long)(y + 1) * P.W);
      double c1, s1;
      if (U8) {
        const double2 t = lut64[(int)Ic];
        c1 = t.x;
        s1 = t.y;
      } else {
        base_angle_f64(Ic, P.invD, c1, s1);
      }
      Cheb64 gk;
      gk.init(c1, s1);
      for (int j = 0; j < P.kstep[0]; ++j) gk.step();
      const int* Qb = Ubuf + b * ustride;
      long long num[NPL] = {}, den[NPL] = {};
#pragma unroll
      for (int i = 0; i < MAXK; ++i) {
        if (FULL || i < P.nk) {
          if ((i & 7) == 0) bar_sync(BAR_Q_FULL + 2 * b + (i >> 3), n_qfull);
          if (i > 0) {   // k_i - k_{i-1} >= 1 steps
            gk.step();
            if (!CONSEC)
              for (int j = 1; j < P.kstep[i]; ++j) gk.step();
          }
          int F[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int* q = Qb + (4 * i + c) * UP;
            F[c] = __mulhi(q[e0] - q[l0], ax0);
            if (M == 2) F[c] += __mulhi(q[e1] - q[l1], ax1);
          }
#pragma unroll
          for (int q = 0; q < NPL; ++q) {   // Case 1 (bf_apply_multi): every plan over the same F
            if (q == 0 || q < P.nplans) {
              const int wc = __double2loint(fma(gk.c, P.aw[q][i], MAGIC64));
              const int wsn = __double2loint(fma(gk.s, P.aw[q][i], MAGIC64));
              den[q] = mad_wide(wc, F[0], den[q]);
              den[q] = mad_wide(wsn, F[1], den[q]);
              num[q] = mad_wide(wc, F[2], num[q]);
              num[q] = mad_wide(wsn, F[3], num[q]);
            }
          }
          if ((i & 7) == 7 || (FULL ? i + 1 == MAXK : i + 1 == P.nk)) bar_arrive(BAR_U_EMPTY + 2 * b + (i >> 3), n_uempty);
        }
      }
      if (act) {
#pragma unroll
        for (int q = 0; q < NPL; ++q)
          if (q == 0 || q < P.nplans) finish_pixel(P, num[q], den[q], Ic, prow + (long long)y * P.W + q * P.plan_stride, out, ws);
      }
    }
  }
}

// ------------------------------------------------------------------ kernel 3: the literal window
// NEXT f1: the paper's dimension-promoted 3-D box filter with the window [I(x) - T_r, I(x) + T_r]
// (eq:1D_box_N_terms, eq:numerator_2D_box_N_terms) on u8 images. The auxiliary
// images F_c(y, z) = G^c_k(y) delta_{I(y)}(z) depend on y only through the level z = I(y), so
// their 3-D box sums factor into the spatially weighted level counts
//     C_z(x) = sum_y K~_s(x - y) [I(y) = z]
// and the numerator / denominator become
//     num(x) = sum_{|z - I(x)| <= T_r} C_z(x) z K_lit(I(x) - z),  den likewise without z,
// with K_lit(t) = sum_k a_k cos(pi k t / T_r) (eq:trigonometric_N_terms): the shiftable split of
// P:460-468 recombined per level (an exact identity, pinned by the oracle's bf_promoted).
// One CTA = a strip of LIT_NT extended columns x a band of rows; each thread keeps its column's
// level counts for the two vertical boxes packed in one int32 (lo / hi 16 bits) in shared memory,
// sliding them down one row per step (4 taps); the output threads then sum, for every level of
// their window, the counts over the horizontal boxes and accumulate the integer products with
// K_lit quantised to 2^30 exactly in int64; the box weights are applied once per pixel in fp64.
constexpr int LIT_NT = 128;
constexpr int LIT_KB = 30;

struct LParams {
  int H, W, TW, TH, rlo_x;
  int nbx, nby;
  int vlo[2], vhi[2], vmin, vmax;
  int hlo[2], hhi[2];
  double wxy[2][2];   // wy_b * wx_b' (b vertical, b' horizontal)
  int Tw;             // window half-width in levels: |z - I(x)| <= Tw
  long long frame_elems;
};

__global__ void __launch_bounds__(LIT_NT, 1)
    bf_literal_kernel(const LParams P, const int* __restrict__ klut, const unsigned char* __restrict__ in,
                      float* __restrict__ out) {
  constexpr int NTP = LIT_NT + 1;                   // level-row pitch (odd: scattered updates spread)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* cnt = reinterpret_cast<int*>(smem_raw);      // [256][NTP] packed counts (box 0 lo16, box 1 hi16)
  int* K = cnt + 256 * NTP;                         // [511] K_lit(t) * 2^30, t = -255..255
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P.TW;
  const int y0 = blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int col = x0 - P.rlo_x + tid;
  const bool colok = (col >= 0) & (col < P.W);
  const int TWv = min(P.TW, P.W - x0);
  const int yend = min(y0 + P.TH, P.H);

  for (int i = tid; i < 256 * NTP; i += LIT_NT) cnt[i] = 0;
  for (int i = tid; i < 511; i += LIT_NT) K[i] = klut[i];
  __syncthreads();
  // counts of the vertical boxes at row y0 - 1
  if (colok) {
    for (int v = P.vmin; v <= P.vmax; ++v) {
      const int row = y0 - 1 + v;
      if (row < 0 || row >= P.H) continue;
      const int z = in[fbase + (long long)row * P.W + col];
      int inc = 0;
      for (int b = 0; b < P.nby; ++b)
        if (v >= P.vlo[b] && v <= P.vhi[b]) inc += 1 << (16 * b);
      cnt[z * NTP + tid] += inc;
    }
  }
  for (int y = y0; y < yend; ++y) {
    // ---- slide the column's counts down one row: enter y + vhi_b, leave y + vlo_b - 1
    if (colok) {
      for (int b = 0; b < P.nby; ++b) {
        const int re = y + P.vhi[b], rl = y + P.vlo[b] - 1;
        if (re >= 0 && re < P.H) cnt[in[fbase + (long long)re * P.W + col] * NTP + tid] += 1 << (16 * b);
        if (rl >= 0 && rl < P.H) cnt[in[fbase + (long long)rl * P.W + col] * NTP + tid] -= 1 << (16 * b);
      }
    }
    __syncthreads();
    // ---- windowed level sums for the output pixels of row y
    if (tid < TWv) {
      const long long pix = fbase + (long long)y * P.W + x0 + tid;
      const int I0 = in[pix];
      const int zlo = max(0, I0 - P.Tw), zhi = min(255, I0 + P.Tw);
      long long A[2][2] = {{0, 0}, {0, 0}}, B[2][2] = {{0, 0}, {0, 0}};
      const int* base = cnt + tid + P.rlo_x;
      for (int z = zlo; z <= zhi; ++z) {
        const int* rowz = base + z * NTP;
        const int kz = K[I0 - z + 255];
        // horizontal boxes, the inner (b' = 1, nested) first
        int s1 = 0;
        if (P.nbx > 1)
          for (int u = P.hlo[1]; u <= P.hhi[1]; ++u) s1 += rowz[u];
        int s0 = 0;
        if (P.nbx > 1 && P.hlo[0] <= P.hlo[1] && P.hhi[1] <= P.hhi[0]) {
          s0 = s1;
          for (int u = P.hlo[0]; u < P.hlo[1]; ++u) s0 += rowz[u];
          for (int u = P.hhi[1] + 1; u <= P.hhi[0]; ++u) s0 += rowz[u];
        } else {
          for (int u = P.hlo[0]; u <= P.hhi[0]; ++u) s0 += rowz[u];
        }
        const int sb[2] = {s0, s1};
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
#pragma unroll
          for (int by = 0; by < 2; ++by) {
            const int c = (sb[bx] >> (16 * by)) & 0xFFFF;
            A[by][bx] += (long long)c * kz;
            B[by][bx] += (long long)(c * z) * kz;
          }
        }
      }
      double num = 0.0, den = 0.0;
#pragma unroll
      for (int by = 0; by < 2; ++by)
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
          num += P.wxy[by][bx] * (double)B[by][bx];
          den += P.wxy[by][bx] * (double)A[by][bx];
        }
      out[pix] = (den > 0.0) ? (float)(num / den) : (float)I0;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

// Stream-ordered scratch (multi-pass num / den workspace, the literal kernel's table) from a
// library-owned memory pool per device that keeps its memory (release threshold = max): the
// default pool would return a 1 GB workspace to the OS at every synchronisation and map it
// again on the next call (measured 90-130 ms instead of ~90 ms on cfg4).
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, st);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props;
      std::memset(&props, 0, sizeof(props));
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t pool;
      e = cudaMemPoolCreate(&pool, &props);
      if (e != cudaSuccess) return e;
      unsigned long long keep = ~0ULL;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = pool;
    }
  }
  return cudaMallocFromPoolAsync(p, bytes, pools[dev], st);
}

size_t smem_layout(KParams& P, int NT, int MAXK, bool u8) {
  auto up16 = [](size_t v) { return (v + 15) / 16 * 16; };
  size_t off = up16(sizeof(int) * P.ns * 4 * (size_t)P.nk * (NT + 1));
  P.f_off = (int)off;
  off = up16(off + sizeof(int) * (size_t)P.TW * (4 * MAXK + 4));
  P.l_off = (int)off;
  if (u8) off += 256 * (sizeof(float2) + sizeof(double2));
  return off;
}

// warp-specialised kernel: two U' row buffers and two F row buffers
size_t smem_layout_ws2(KParams& P, bool u8) {
  size_t off = (sizeof(int) * 2 * P.ns * 4 * (size_t)P.nk * W2_UP + 15) / 16 * 16;
  P.f_off = (int)off;
  P.l_off = (int)off;
  if (u8) off += 256 * (sizeof(float2) + sizeof(double2));
  return off;
}

size_t smem_layout_ws(KParams& P, int MAXK, bool u8) {
  auto up16 = [](size_t v) { return (v + 15) / 16 * 16; };
  size_t off = up16(sizeof(int) * 2 * P.ns * 4 * (size_t)P.nk * (WS_V + 2));
  P.f_off = (int)off;
  off = up16(off + sizeof(int) * 2 * (size_t)P.TW * (4 * MAXK + 4));
  P.l_off = (int)off;
  if (u8) off += 256 * (sizeof(float2) + sizeof(double2));
  return off;
}

template <int MAXK, int FORM, bool U8, int NT, bool CONSEC, bool FULL = false, bool MULTI = false>
cudaError_t launch_one(KParams P, const void* in, float* out, longlong2* ws, dim3 grid, cudaStream_t st, int kern) {
  if constexpr (NT == WS_V && FORM != 4) {
    if (kern == KERN_WS2) {
      if constexpr (FORM != 5) {
        auto kfn = bf_ws2_kernel<MAXK, FORM, U8, CONSEC, FULL, MULTI>;
        const size_t smem = smem_layout_ws2(P, U8);
        if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kfn<<<grid, W2_THREADS, smem, st>>>(P, in, out, ws);
        return cudaGetLastError();
      }
      return cudaErrorInvalidConfiguration;
    }
    if (kern == KERN_WS && !MULTI) {   // (the Case 1 multi-plan combine runs on kernel 1)
      auto kfn = bf_ws_kernel<MAXK, FORM, U8, CONSEC, FULL, false>;
      const size_t smem = smem_layout_ws(P, MAXK, U8);
      if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
      cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kfn<<<grid, WS_THREADS, smem, st>>>(P, in, out, ws);
      return cudaGetLastError();
    }
  }
  auto kfn = bf_band_kernel<MAXK, FORM, U8, NT, CONSEC, FULL, MULTI>;
  const size_t smem = smem_layout(P, NT, MAXK, U8);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kfn<<<grid, NT, smem, st>>>(P, in, out, ws);
  return cudaGetLastError();
}

template <int MAXK, int FORM, bool U8, int NT>
cudaError_t dispatch_consec(bool consec, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                            cudaStream_t st, int kern) {
  if (P.nplans > 1) {   // Case 1 multi-plan combine: its own instantiation (register pressure)
    if constexpr (FORM == 1 || FORM == 2) {
      return consec ? launch_one<MAXK, FORM, U8, NT, true, false, true>(P, in, out, ws, grid, st, kern)
                    : launch_one<MAXK, FORM, U8, NT, false, false, true>(P, in, out, ws, grid, st, kern);
    }
    return cudaErrorInvalidConfiguration;
  }
  if (consec && P.nk == MAXK) return launch_one<MAXK, FORM, U8, NT, true, true>(P, in, out, ws, grid, st, kern);
  if (consec) return launch_one<MAXK, FORM, U8, NT, true>(P, in, out, ws, grid, st, kern);
  return launch_one<MAXK, FORM, U8, NT, false>(P, in, out, ws, grid, st, kern);
}

template <int MAXK, bool U8, int NT>
cudaError_t dispatch_form(int form, bool consec, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                          cudaStream_t st, int kern) {
  switch (form) {
    case 1: return dispatch_consec<MAXK, 1, U8, NT>(consec, P, in, out, ws, grid, st, kern);
    case 2: return dispatch_consec<MAXK, 2, U8, NT>(consec, P, in, out, ws, grid, st, kern);
    case 4: return launch_one<MAXK, 4, U8, NT, false>(P, in, out, ws, grid, st, KERN_BAND);
    default: break;
  }
  return cudaErrorInvalidConfiguration;
}

struct Shape {
  int NT, MAXK;
  int kern;   // KERN_BAND; KERN_WS / KERN_WS2 (warp-specialised, NT = 256 class, at most 2 box streams)
  int form;   // Form<FORM>: 1, 2, 4 separable with that many boxes; 5 rank 2
};

// Thread-block shape per plan: NT extended columns (TW = NT - halo outputs, TW >= NT/2 where
// possible), MAXK terms per pass (the vertical state is NS * 4 * MAXK registers per thread) and
// the spatial form. Returns NT = 0 if the plan has no GPU form.
Shape plan_shape(const bf_plan* p, int& rlo, int& rhi) {
  Shape sh{0, 0, KERN_BAND, 0};
  rlo = rhi = 0;
  if (p->ns < 1 || p->ns > 2) return sh;
  int nbx = 0, nby = p->snby[0];
  for (int t = 0; t < p->ns; ++t) {
    if (p->snbx[t] < 1 || p->snbx[t] > MAXB || p->snby[t] != nby) return sh;
    nbx = std::max(nbx, p->snbx[t]);
    for (int b = 0; b < p->snbx[t]; ++b) {
      rlo = std::max(rlo, -p->slox[t][b]);
      rhi = std::max(rhi, p->shix[t][b]);
    }
    for (int b = 0; b < nby; ++b)
      if (p->sloy[t][b] != p->sloy[0][b] || p->shiy[t][b] != p->shiy[0][b]) return sh;
  }
  if (nby < 1 || nby > MAXB) return sh;
  if (p->ns == 2) {
    if (nbx > 1 || nby > 2) return sh;
    sh.form = 5;
  } else {
    const int nb = std::max(nbx, nby);
    sh.form = nb <= 1 ? 1 : (nb == 2 ? 2 : 4);
  }
  const int halo = rlo + rhi;
  const int nk = p->n_k;
  // warp-specialised for NT = 256 (its prefix-form H role measured 2.32 vs 2.50 ms on cfg2)
  if (halo <= 128) {
    sh.NT = 256;
    sh.MAXK = (nk <= 8 || p->ns == 2) ? 8 : 16;
    // kernel 2b for the separable forms; the rank-2 form's vertical state (NS = 2 taps sets)
    // needs more than 2b's 112 V registers, it keeps kernel 2
    sh.kern = sh.form == 4 ? KERN_BAND : (sh.form == 5 ? KERN_WS : KERN_WS2);
  } else {
    sh.NT = 512;
    // 16 terms per pass for the two-box separable form (128 registers, no spills; cfg4
    // 62.2 -> 55.4 ms with two passes instead of three), else 8
    sh.MAXK = (sh.form == 2 && nk > 8) ? 16 : 8;
    sh.kern = KERN_BAND;
  }
  if (const char* e = std::getenv("BF_MAXK")) sh.MAXK = (std::atoi(e) <= 8 || p->ns == 2) ? 8 : 16;   // tuning hook
  if (const char* e = std::getenv("BF_KERNEL")) {   // tuning hook: force one kernel
    if (std::strcmp(e, "band") == 0) sh.kern = KERN_BAND;
    if (std::strcmp(e, "ws") == 0) sh.kern = (sh.NT == 256 && sh.form != 4) ? KERN_WS : KERN_BAND;
    if (std::strcmp(e, "ws2") == 0) sh.kern = (sh.NT == 256 && sh.form != 4) ? KERN_WS2 : KERN_BAND;
    if (std::strcmp(e, "ws2") == 0 && sh.form == 5) sh.kern = KERN_WS;
  }
  if (sh.NT == 512 && sh.form != 2) sh.MAXK = 8;   // (NT = 512 x 16 terms: form 2 only)
  if (halo + 32 > sh.NT) sh.NT = 0;
  return sh;
}

template <bool U8>
cudaError_t dispatch(const Shape& sh, bool consec, const KParams& P, const void* in, float* out, longlong2* ws,
                     dim3 grid, cudaStream_t st) {
  if (sh.form == 5) {   // rank 2: NS * 4 * 8 = 64 state registers, NT = 256 only
    if (sh.NT != 256 || sh.MAXK != 8) return cudaErrorInvalidConfiguration;
    return dispatch_consec<8, 5, U8, 256>(consec, P, in, out, ws, grid, st, sh.kern);
  }
  if (sh.NT == 256 && sh.MAXK == 8) return dispatch_form<8, U8, 256>(sh.form, consec, P, in, out, ws, grid, st, sh.kern);
  if (sh.NT == 256 && sh.MAXK == 16)
    return dispatch_form<16, U8, 256>(sh.form, consec, P, in, out, ws, grid, st, sh.kern);
  if (sh.NT == 512 && sh.MAXK == 8) return dispatch_form<8, U8, 512>(sh.form, consec, P, in, out, ws, grid, st, KERN_BAND);
  if (sh.NT == 512 && sh.MAXK == 16 && sh.form == 2)
    return dispatch_consec<16, 2, U8, 512>(consec, P, in, out, ws, grid, st, KERN_BAND);
  return cudaErrorInvalidConfiguration;
}

// The literal-window path (kernel 3): u8 input, levels 0..255 (D = 255), separable plans with
// at most two boxes per axis whose halo fits the 128-column strip.
bf_status run_literal(const bf_plan* p, const void* d_in, float* d_out, int n_frames, int H, int W, cudaStream_t st,
                      bf_launch_config* dry) {
  if (p->input_dtype != BF_IN_U8 || p->D != 255.0 || p->ns != 1 || p->snbx[0] > 2 || p->snby[0] > 2)
    return BF_ERR_UNSUPPORTED;
  LParams L;
  std::memset(&L, 0, sizeof(L));
  int rlo = 0, rhi = 0;
  L.nbx = p->snbx[0];
  L.nby = p->snby[0];
  for (int b = 0; b < L.nbx; ++b) {
    L.hlo[b] = p->slox[0][b];
    L.hhi[b] = p->shix[0][b];
    rlo = std::max(rlo, -L.hlo[b]);
    rhi = std::max(rhi, L.hhi[b]);
  }
  if (rlo + rhi + 32 > LIT_NT) return BF_ERR_UNSUPPORTED;
  // the packed 16-bit counts must not overflow: (box height) x (box width) < 2^15
  for (int b = 0; b < L.nby; ++b)
    if ((long long)(p->shiy[0][b] - p->sloy[0][b] + 1) * (rlo + rhi + 1) >= 32768) return BF_ERR_UNSUPPORTED;
  L.vmin = p->sloy[0][0];
  L.vmax = p->shiy[0][0];
  for (int b = 0; b < L.nby; ++b) {
    L.vlo[b] = p->sloy[0][b];
    L.vhi[b] = p->shiy[0][b];
    L.vmin = std::min(L.vmin, L.vlo[b]);
    L.vmax = std::max(L.vmax, L.vhi[b]);
  }
  for (int by = 0; by < 2; ++by)
    for (int bx = 0; bx < 2; ++bx)
      L.wxy[by][bx] = (by < L.nby && bx < L.nbx) ? p->swy[0][by] * p->swx[0][bx] : 0.0;
  L.H = H;
  L.W = W;
  L.rlo_x = rlo;
  L.TW = LIT_NT - (rlo + rhi);
  L.frame_elems = (long long)H * W;
  L.Tw = (int)std::floor(p->T + 1e-9);
  // K_lit(t) = sum_k a_k cos(pi k t / T_r) for |t| <= T_r (eq:trigonometric_N_terms), 0 outside
  // the window, quantised to 2^30: |num|, |den| < 2^63 for |K_lit| < 2
  int hk[511];
  for (int t = -255; t <= 255; ++t) {
    double k = 0.0;
    if (std::abs(t) <= L.Tw)
      for (int i = 0; i < p->n_k; ++i) k += p->a[i] * std::cos(M_PI * p->k[i] * t / p->T);
    if (!(std::fabs(k) < 2.0)) return BF_ERR_NUMERIC;
    hk[t + 255] = (int)std::lrint(std::ldexp(k, LIT_KB));
  }
  const int nstrips = (W + L.TW - 1) / L.TW;
  const int nsm = sm_count();
  const int ry = L.vmax - L.vmin + 1;
  long long best_cost = -1;
  int best_nb = 1;
  for (int nb = 1; nb <= H; ++nb) {
    const int TH = (H + nb - 1) / nb;
    if (nb > 1 && TH < 16) break;
    const long long ctas = (long long)nstrips * nb * n_frames;
    const long long waves = (ctas + nsm - 1) / nsm;
    const long long cost = waves * (4LL * TH + ry);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_nb = nb;
    }
  }
  L.TH = (H + best_nb - 1) / best_nb;
  if (const char* e = std::getenv("BF_TH")) L.TH = std::max(1, std::min(H, std::atoi(e)));   // test hook
  best_nb = (H + L.TH - 1) / L.TH;
  const size_t smem = sizeof(int) * (256 * (LIT_NT + 1) + 512);
  if (dry) {
    *dry = bf_launch_config{1, "bf_literal_kernel", LIT_NT, nstrips, best_nb, n_frames, L.TW, L.TH, smem};
    return BF_OK;
  }
  int* dk = nullptr;   // the 2 KB table travels through a stream-ordered allocation
  if (scratch_alloc(reinterpret_cast<void**>(&dk), sizeof(hk), st) != cudaSuccess) return BF_ERR_CUDA;
  cudaError_t err = cudaMemcpyAsync(dk, hk, sizeof(hk), cudaMemcpyHostToDevice, st);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(bf_literal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err == cudaSuccess) {
    bf_literal_kernel<<<dim3(nstrips, best_nb, n_frames), LIT_NT, smem, st>>>(
        L, dk, reinterpret_cast<const unsigned char*>(d_in), d_out);
    err = cudaGetLastError();
  }
  cudaFreeAsync(dk, st);
  return err == cudaSuccess ? BF_OK : BF_ERR_CUDA;
}

// Plans that can share one pass of box-filtered channels: same spatial form, D and input type.
bool same_channels(const bf_plan* a, const bf_plan* b) {
  if (a->ns != b->ns || a->D != b->D || a->input_dtype != b->input_dtype) return false;
  for (int t = 0; t < a->ns; ++t) {
    if (a->snbx[t] != b->snbx[t] || a->snby[t] != b->snby[t]) return false;
    for (int i = 0; i < a->snbx[t]; ++i)
      if (a->slox[t][i] != b->slox[t][i] || a->shix[t][i] != b->shix[t][i] || a->swx[t][i] != b->swx[t][i])
        return false;
    for (int i = 0; i < a->snby[t]; ++i)
      if (a->sloy[t][i] != b->sloy[t][i] || a->shiy[t][i] != b->shiy[t][i] || a->swy[t][i] != b->swy[t][i])
        return false;
  }
  return true;
}

// dry != nullptr: describe the launches (bf_apply_config) instead of enqueueing them
// ya, yb: output rows [ya, yb) (default: all); the input rows the halo needs must be resident.
bf_status run_filter(const bf_plan* const* plans, int nplans, const void* d_in, float* d_out, int n_frames, int H,
                     int W, cudaStream_t st, bf_launch_config* dry = nullptr, int ya = 0, int yb = -1) {
  if (yb < 0) yb = H;
  if (ya < 0 || ya >= yb || yb > H) return BF_ERR_INVALID_ARG;
  const int Hr = yb - ya;
  if (!plans || nplans < 1 || nplans > MAXP || (!dry && (!d_in || !d_out)) || H <= 0 || W <= 0 || n_frames <= 0)
    return BF_ERR_INVALID_ARG;
  for (int q = 0; q < nplans; ++q)
    if (!plans[q]) return BF_ERR_INVALID_ARG;
  // union of the plans' selected k (one set of channels); a single plan is its own union
  bf_plan merged = *plans[0];
  if (nplans > 1) {
    if (n_frames != 1) return BF_ERR_INVALID_ARG;
    int ks[BF_MAX_TERMS * MAXP], nks = 0;
    for (int q = 0; q < nplans; ++q) {
      if (!same_channels(plans[0], plans[q])) return BF_ERR_INVALID_ARG;
      for (int i = 0; i < plans[q]->n_k; ++i) ks[nks++] = plans[q]->k[i];
    }
    std::sort(ks, ks + nks);
    nks = (int)(std::unique(ks, ks + nks) - ks);
    if (nks > 16) return BF_ERR_UNSUPPORTED;
    merged.n_k = nks;
    for (int i = 0; i < nks; ++i) {
      merged.k[i] = ks[i];
      merged.a[i] = 0.0;
    }
  }
  const bf_plan* p = &merged;
  if (p->literal) {
    if (nplans != 1 || ya != 0 || yb != H) return BF_ERR_UNSUPPORTED;
    return run_literal(p, d_in, d_out, n_frames, H, W, st, dry);
  }
  if ((long long)H * W > (1LL << 40) / n_frames) return BF_ERR_INVALID_ARG;
  if (!dry && (const void*)d_out == d_in) return BF_ERR_INVALID_ARG;
  int rlo, rhi;
  Shape sh = plan_shape(p, rlo, rhi);
  if (sh.NT == 0) return BF_ERR_UNSUPPORTED;
  const int ns = p->ns;
  // paired-load layout of the horizontal boxes (warp-specialised kernel): every box symmetric
  // [-r_b, r_b] (odd width), at most two boxes in all, box 0 the widest (leave stream even)
  int wpar = -1;
  {
    int m = 0, r0 = -1, r1 = -1;
    bool ok = true;
    for (int t = 0; t < ns; ++t)
      for (int b = 0; b < p->snbx[t]; ++b) {
        if (p->slox[t][b] != -p->shix[t][b]) ok = false;
        if (m == 0) r0 = p->shix[t][b];
        else r1 = p->shix[t][b];
        ++m;
      }
    if (ok && m <= 2 && r0 == rlo && (m == 1 || r1 <= r0)) wpar = (m == 2) ? ((r0 - r1) & 1) : 0;
  }
  if (nplans > 1 && sh.kern != KERN_WS2) sh.kern = KERN_BAND;   // Case 1 multi-plan combine: kernel 2b or 1
  if (sh.kern == KERN_WS && wpar < 0) sh.kern = KERN_BAND;
  if ((4 * std::min(sh.MAXK, p->n_k) + 31) / 32 > 2) sh.kern = KERN_BAND;   // two scan warps
  const int halo = rlo + rhi;
  int TW = (sh.kern == KERN_WS2) ? std::min(W2_H, W2_V - halo) : sh.NT - halo;   // widest strip

  KParams P;
  std::memset(&P, 0, sizeof(P));
  P.H = H;
  P.W = W;
  P.yb = ya;
  P.ye = yb;
  P.frame_elems = (long long)H * W;
  P.TW = TW;
  P.rlo_x = rlo;
  P.ns = ns;
  P.nby = p->snby[0];
  // ---- vertical: scales wy_tb / max|wy| * 2^q, q as large as the int32 states allow
  double wymax = 0.0;
  for (int t = 0; t < ns; ++t)
    for (int b = 0; b < P.nby; ++b) wymax = std::max(wymax, std::fabs(p->swy[t][b]));
  double wsum = 0.0;
  for (int t = 0; t < ns; ++t) {
    double w = 0.0;
    for (int b = 0; b < P.nby; ++b) w += std::fabs(p->swy[t][b]) / wymax * (p->shiy[t][b] - p->sloy[t][b] + 1);
    wsum = std::max(wsum, w);
  }
  int qb = QBITS_MAX;
  while (qb > 8 && std::ldexp(wsum, qb) + 4.0 * (p->shiy[0][0] - p->sloy[0][0] + 8) >= 2147483647.0 - 65536.0) --qb;
  double ubound = 0.0;   // bound of |U_t| before the shift, over the terms
  P.vmin = p->sloy[0][0];
  P.vmax = p->shiy[0][0];
  for (int b = 0; b < P.nby; ++b) {
    P.vlo[b] = p->sloy[0][b];
    P.vhi[b] = p->shiy[0][b];
    P.vmin = std::min(P.vmin, P.vlo[b]);
    P.vmax = std::max(P.vmax, P.vhi[b]);
  }
  for (int t = 0; t < ns; ++t) {
    double ub = 0.0;
    for (int b = 0; b < P.nby; ++b) {
      P.qs[t][b] = (float)std::ldexp(p->swy[t][b] / wymax, qb);
      P.qsD[t][b] = (float)((double)P.qs[t][b] / p->D);
      ub += (std::fabs((double)P.qs[t][b]) + 0.5) * (P.vhi[b] - P.vlo[b] + 1);
    }
    ubound = std::max(ubound, ub);
  }
  // ---- U' = U >> ush: every horizontal box sum H of U' fits int32
  int nxmax = 1;
  for (int t = 0; t < ns; ++t)
    for (int b = 0; b < p->snbx[t]; ++b) nxmax = std::max(nxmax, p->shix[t][b] - p->slox[t][b] + 1);
  P.ush = 0;
  while ((ubound / std::ldexp(1.0, P.ush) + 1.0) * nxmax >= 2147483000.0) ++P.ush;
  P.urnd = P.ush > 0 ? (1 << (P.ush - 1)) : 0;
  const double uprime = ubound / std::ldexp(1.0, P.ush) + 1.0;
  // ---- horizontal: integer weights ax = round(wx / max|wx| * 2^abits), F = sum mulhi(H, ax)
  //      (one IMAD.HI per box; each high word truncates, so |F - exact| < ns * nbx) fits int32
  double wxmax = 0.0, rw = 0.0;
  for (int t = 0; t < ns; ++t)
    for (int b = 0; b < p->snbx[t]; ++b) wxmax = std::max(wxmax, std::fabs(p->swx[t][b]));
  for (int t = 0; t < ns; ++t)
    for (int b = 0; b < p->snbx[t]; ++b) rw += std::fabs(p->swx[t][b]) / wxmax * (p->shix[t][b] - p->slox[t][b] + 1);
  int abits = ABITS;
  while (abits > 16 && uprime * rw * std::ldexp(1.0, abits - 32) + 8.0 >= 2147483000.0) --abits;
  for (int t = 0; t < ns; ++t) {
    P.nbx[t] = p->snbx[t];
    for (int b = 0; b < p->snbx[t]; ++b) {
      P.hlo[t][b] = p->slox[t][b];
      P.hhi[t][b] = p->shix[t][b];
      P.ax[t][b] = (int)std::lround(std::ldexp(p->swx[t][b] / wxmax, abits));
    }
  }
  // ---- combine weights a_k * 2^wbits: |W| < 2^31 and |num|, |den| < 2^62
  double asum = 0.0, amax = 0.0;
  for (int q = 0; q < nplans; ++q) {
    double s1 = 0.0;
    for (int i = 0; i < plans[q]->n_k; ++i) {
      s1 += std::fabs(plans[q]->a[i]);
      amax = std::max(amax, std::fabs(plans[q]->a[i]));
    }
    asum = std::max(asum, s1);
  }
  int wbits = 29;
  while (wbits > 8 && (std::ldexp(asum, wbits) * 2.0 * 2147483648.0 >= 4.0e18 || std::ldexp(amax, wbits) >= 2.0e9))
    --wbits;
  const double invD = 1.0 / p->D;
  P.invD = invD;
  P.invD_hi = (float)invD;
  P.invD_lo = (float)(invD - (double)P.invD_hi);
  P.D = p->D;

  const int passes = (p->n_k + sh.MAXK - 1) / sh.MAXK;
  if (nplans > 1 && passes > 1) return BF_ERR_UNSUPPORTED;   // shared channels must fit one pass
  P.nplans = nplans;
  P.plan_stride = (long long)H * W;
  if (sh.kern == KERN_WS) {   // the double-buffered rows must fit the 227 KB of shared memory
    KParams Q = P;
    Q.nk = std::min(sh.MAXK, p->n_k);
    if (smem_layout_ws(Q, sh.MAXK, p->input_dtype == BF_IN_U8) > 227 * 1024) sh.kern = KERN_BAND;
  }
  // ---- tile: band height TH (kernel 2b: and strip width TW) minimising the modelled time: CTAs
  //      in whole waves of the resident slots, each TH rows at the row cost plus the initial
  //      vertical sum over vmax - vmin + 1 rows. Kernel 2b's row time: warp-instructions per
  //      role (ncu, cfg2: V 694 per 32 extended columns, FH 942 per 32 outputs, S ~4 per column;
  //      V init 373 per 32 columns) at the measured ~0.55 IPC per SM sub-partition, but never
  //      below the ~6000 cycles one warp's dependent chain takes (measured at 128-column strips):
  //      a narrower strip can fill the 148 SMs better.
  const int nsm = sm_count();
  const int slots = nsm * ((sh.NT > 256 || sh.kern != KERN_BAND) ? 1 : 2);
  const int ry = P.vmax - P.vmin + 1;
  double best_cost = -1.0;
  int best_nb = 1, best_tw = TW;
  for (int tw = TW; tw >= 1; tw = (tw % 32) ? tw - tw % 32 : tw - 32) {
    if (tw != TW && (sh.kern != KERN_WS2 || tw < 128)) break;
    double row = 4.0, init = 1.0;
    if (sh.kern == KERN_WS2) {
      const int wv = (tw + halo + 7) & ~7;
      row = std::max(6000.0, (694.0 * ((wv + 31) / 32) + 942.0 * ((tw + 31) / 32) + 4.0 * wv) / (4 * 0.55));
      init = std::max(1500.0, 373.0 * ((wv + 31) / 32) / (4 * 0.55));
    }
    const long long strips = (W + tw - 1) / tw;
    for (int nb = 1; nb <= Hr; ++nb) {
      const int TH = (Hr + nb - 1) / nb;
      if (nb > 1 && TH < 16) break;
      const long long ctas = strips * nb * n_frames;
      const long long waves = (ctas + slots - 1) / slots;
      const double cost = (double)waves * (TH * row + ry * init);
      if (best_cost < 0 || cost < best_cost * (1.0 - 1e-9)) {
        best_cost = cost;
        best_nb = nb;
        best_tw = tw;
      }
    }
  }
  TW = best_tw;
  P.TW = TW;
  const int nstrips = (W + TW - 1) / TW;
  P.TH = (Hr + best_nb - 1) / best_nb;
  if (const char* e = std::getenv("BF_TH")) P.TH = std::max(1, std::min(Hr, std::atoi(e)));   // test hook
  best_nb = (Hr + P.TH - 1) / P.TH;

  if (dry) {
    KParams Q = P;
    Q.nk = std::min(sh.MAXK, p->n_k);
    const bool u8 = (p->input_dtype == BF_IN_U8);
    size_t smem = 0;
    const char* name = "bf_band_kernel";
    int threads = sh.NT;
    if (sh.kern == KERN_WS2) {
      smem = smem_layout_ws2(Q, u8);
      name = "bf_ws2_kernel";
      threads = W2_THREADS;
    } else if (sh.kern == KERN_WS) {
      smem = smem_layout_ws(Q, sh.MAXK, u8);
      name = "bf_ws_kernel";
      threads = WS_THREADS;
    } else {
      smem = smem_layout(Q, sh.NT, sh.MAXK, u8);
    }
    *dry = bf_launch_config{passes, name, threads, nstrips, best_nb, n_frames, TW, P.TH, smem};
    return BF_OK;
  }
  longlong2* ws = nullptr;
  if (passes > 1) {
    if (scratch_alloc(reinterpret_cast<void**>(&ws), sizeof(longlong2) * (size_t)H * W * n_frames, st) != cudaSuccess)
      return BF_ERR_CUDA;
  }
  dim3 grid(nstrips, best_nb, n_frames);
  const bool u8 = (p->input_dtype == BF_IN_U8);
  cudaError_t err = cudaSuccess;
  for (int pass = 0; pass < passes && err == cudaSuccess; ++pass) {
    const int first = pass * sh.MAXK;
    const int nk = std::min(sh.MAXK, p->n_k - first);
    P.nk = nk;
    P.ngrp = (4 * nk + 31) / 32;
    bool consec = true;
    for (int i = 0; i < nk; ++i) {
      const int kk = p->k[first + i];
      P.kstep[i] = (i == 0) ? kk : kk - p->k[first + i - 1];
      if (i > 0 && P.kstep[i] != 1) consec = false;
      if (nplans == 1) {
        P.aw[0][i] = std::ldexp(p->a[first + i], wbits);
      } else {
        for (int q = 0; q < nplans; ++q) {   // a_k of plan q, 0 where q did not select k
          double a = 0.0;
          for (int j = 0; j < plans[q]->n_k; ++j)
            if (plans[q]->k[j] == kk) a = plans[q]->a[j];
          P.aw[q][i] = std::ldexp(a, wbits);
        }
      }
    }
    // walker segments: ngrp * nseg warps; long segments amortise the initial window sums
    const int max_tasks = sh.kern == KERN_WS ? WS_H / 32 : sh.NT / 32;   // (prefix form: WS_F / 32, set below)
    int nseg = std::max(1, max_tasks / P.ngrp);
    const int min_len = sh.kern == KERN_WS ? 24 : std::max(32, 2 * (rlo + rhi + 1) / 3);
    while (nseg > 1 && (TW + nseg - 1) / nseg < min_len) --nseg;
    // wide halos (NT = 512): the other warps idle through interval B behind one long walker;
    // four segments measured best on cfg4 (r = 192: 77.0 -> 62.2 ms; 1 / 2 / 8 / 16 segments:
    // 77.0 / 67.0 / 67.7 / 82.5 ms)
    if (sh.kern == KERN_BAND && sh.NT == 512) nseg = std::min(4, std::max(1, max_tasks / P.ngrp));
    if (const char* e = std::getenv("BF_NSEG")) nseg = std::max(1, std::min(max_tasks / P.ngrp, std::atoi(e)));  // tuning hook
    P.nseg = nseg;
    P.seglen = (TW + nseg - 1) / nseg;
    P.seglen += P.seglen & 1;   // even segment starts (paired loads)
    P.wpar = sh.kern == KERN_WS ? wpar : -1;
    P.wv = (TW + halo + 7) & ~7;
    if (sh.kern == KERN_WS) {   // F warps of the warp-specialised kernel: (WS_F / 32) / ngrp segments per group
      P.nseg = std::max(1, (WS_F / 32) / P.ngrp);
      P.seglen = (TW + P.nseg - 1) / P.nseg;
      P.seglen += P.seglen & 1;
    }
    P.pass = (passes == 1) ? 0 : (pass == 0 ? 1 : (pass == passes - 1 ? 3 : 2));
    err = u8 ? dispatch<true>(sh, consec, P, d_in, d_out, ws, grid, st)
             : dispatch<false>(sh, consec, P, d_in, d_out, ws, grid, st);
  }
  if (ws) cudaFreeAsync(ws, st);
  return err == cudaSuccess ? BF_OK : BF_ERR_CUDA;
}

// Device buffers, streams and events for bf_apply_host (grown / created on demand, per process
// and device).
constexpr int HOST_CHUNKS = 9, HOST_CHUNKS_DEFAULT = 5;
struct HostCache {
  std::mutex mu;
  int dev = -1;
  void* din = nullptr;
  float* dout = nullptr;
  size_t in_bytes = 0, out_bytes = 0;
  cudaStream_t s_in = nullptr, s_k = nullptr, s_k2 = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_in[HOST_CHUNKS] = {}, ev_k[HOST_CHUNKS] = {};
  ~HostCache() {
    // freed at process exit; the CUDA context may already be gone, so errors are ignored
    if (din) cudaFree(din);
    if (dout) cudaFree(dout);
  }
  cudaError_t setup(int device) {
    if (dev == device) return cudaSuccess;
    if (dev >= 0) return cudaErrorInvalidDevice;   // one device per process (torchrun ranks)
    cudaError_t e = cudaSuccess;
    for (cudaStream_t* q : {&s_in, &s_k, &s_k2, &s_out})
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(q, cudaStreamNonBlocking);
    for (cudaEvent_t* v : {&ev_start, &ev_end})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(v, cudaEventDisableTiming);
    for (int j = 0; j < HOST_CHUNKS && e == cudaSuccess; ++j) {
      e = cudaEventCreateWithFlags(&ev_in[j], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_k[j], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) dev = device;
    return e;
  }
};
HostCache g_cache;

}  // namespace

extern "C" bf_status bf_apply_launches(const bf_plan* p, int H, int W, int* n) {
  if (!p || !n || H <= 0 || W <= 0) return BF_ERR_INVALID_ARG;
  *n = 0;
  if (p->literal) {
    *n = 1;
    return BF_OK;
  }
  int rlo, rhi;
  const Shape sh = plan_shape(p, rlo, rhi);
  if (sh.NT == 0) return BF_ERR_UNSUPPORTED;
  *n = (p->n_k + sh.MAXK - 1) / sh.MAXK;
  return BF_OK;
}

extern "C" bf_status bf_apply_config(const bf_plan* plan, int n_frames, int H, int W, bf_launch_config* cfg) {
  if (!plan || !cfg || H <= 0 || W <= 0 || n_frames <= 0) return BF_ERR_INVALID_ARG;
  return run_filter(&plan, 1, nullptr, nullptr, n_frames, H, W, nullptr, cfg);
}

extern "C" bf_status bf_apply(const bf_plan* plan, const void* d_in, float* d_out, int H, int W, bf_stream stream) {
  return run_filter(&plan, 1, d_in, d_out, 1, H, W, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" bf_status bf_apply_multi(const bf_plan* const* plans, int n_plans, const void* d_in, float* d_out, int H,
                                    int W, bf_stream stream) {
  return run_filter(plans, n_plans, d_in, d_out, 1, H, W, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" bf_status bf_apply_batched(const bf_plan* plan, const void* d_in, float* d_out, int n_frames, int H,
                                      int W, bf_stream stream) {
  return run_filter(&plan, 1, d_in, d_out, n_frames, H, W, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" bf_status bf_apply_host(const bf_plan* plan, const void* h_in, float* h_out, int H, int W,
                                   bf_stream stream) {
  if (!plan || !h_in || !h_out || H <= 0 || W <= 0) return BF_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t n = (size_t)H * W;
  const size_t isz = plan->input_dtype == BF_IN_U8 ? 1 : 4;
  const size_t ib = n * isz, ob = n * 4;
  std::lock_guard<std::mutex> lk(g_cache.mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || g_cache.setup(dev) != cudaSuccess) return BF_ERR_CUDA;
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
  // Row chunks pipelined over three streams: the copy of input piece j+1, the filter of output
  // rows [b_j, b_j+1) and the copy back of chunk j-1 overlap. Input piece j holds rows
  // [b_j + rv, b_j+1 + rv) (piece 0 from row 0, the last to row H), so the filter of chunk j,
  // which reads rows b_j - rv .. b_j+1 - 1 + rv, needs pieces 0..j only. Small images, the
  // literal kernel and chunks shorter than 512 rows take one chunk.
  int rv = 0;
  for (int b = 0; b < plan->snby[0]; ++b) rv = std::max(rv, std::max(-plan->sloy[0][b], plan->shiy[0][b]));
  // K chunks, the first and the last half as tall as the others (the pipeline's fill and drain
  // are one input piece and one output chunk)
  int K = plan->literal || n < (1u << 20) ? 1 : std::min(HOST_CHUNKS_DEFAULT, 1 + H / std::max(512, 2 * rv + 2));
  if (const char* ev = std::getenv("BF_HOST_CHUNKS"))   // tuning hook
    K = std::min(HOST_CHUNKS, std::max(1, std::min(std::atoi(ev), H / std::max(1, 2 * rv + 2))));
  K = std::max(K, 1);
  cudaError_t e = cudaEventRecord(g_cache.ev_start, st);   // ordered after the caller's prior work
  for (cudaStream_t q : {g_cache.s_in, g_cache.s_k, g_cache.s_k2, g_cache.s_out})
    if (e == cudaSuccess) e = cudaStreamWaitEvent(q, g_cache.ev_start, 0);
  if (e != cudaSuccess) return BF_ERR_CUDA;
  const unsigned char* hin = static_cast<const unsigned char*>(h_in);
  unsigned char* din = static_cast<unsigned char*>(g_cache.din);
  // boundary j of K chunks with weights w, 1, ..., 1, w (w = 1/2; BF_HOST_EDGE = 1/w tuning hook)
  int edge = 2;
  if (const char* ev = std::getenv("BF_HOST_EDGE")) edge = std::max(1, std::atoi(ev));
  auto bnd = [&](int j) {
    if (K <= 2) return (int)((long long)H * j / K);
    if (j <= 0) return 0;
    if (j >= K) return H;
    return (int)((long long)H * (edge * (j - 1) + 1) / (edge * (K - 2) + 2));
  };
  for (int j = 0; j < K && e == cudaSuccess; ++j) {
    const int r0 = j == 0 ? 0 : std::min(H, bnd(j) + rv), r1 = j == K - 1 ? H : std::min(H, bnd(j + 1) + rv);
    if (r1 > r0)
      e = cudaMemcpyAsync(din + (size_t)r0 * W * isz, hin + (size_t)r0 * W * isz, (size_t)(r1 - r0) * W * isz,
                          cudaMemcpyHostToDevice, g_cache.s_in);
    if (e == cudaSuccess) e = cudaEventRecord(g_cache.ev_in[j], g_cache.s_in);
  }
  bf_status s = BF_OK;
  for (int j = 0; j < K && e == cudaSuccess && s == BF_OK; ++j) {
    // alternate two compute streams: chunk j+1 may start on the SMs chunk j's last CTAs leave
    cudaStream_t sk = (j & 1) ? g_cache.s_k2 : g_cache.s_k;
    e = cudaStreamWaitEvent(sk, g_cache.ev_in[j], 0);
    if (e != cudaSuccess) break;
    s = run_filter(&plan, 1, g_cache.din, g_cache.dout, 1, H, W, sk, nullptr, bnd(j), bnd(j + 1));
    if (s != BF_OK) break;
    e = cudaEventRecord(g_cache.ev_k[j], sk);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(g_cache.s_out, g_cache.ev_k[j], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h_out + (size_t)bnd(j) * W, g_cache.dout + (size_t)bnd(j) * W,
                          (size_t)(bnd(j + 1) - bnd(j)) * W * 4, cudaMemcpyDeviceToHost, g_cache.s_out);
  }
  // join: the caller's stream waits for all three, then the call returns with h_out complete
  for (cudaStream_t q : {g_cache.s_in, g_cache.s_k, g_cache.s_k2, g_cache.s_out}) {
    cudaEventRecord(g_cache.ev_end, q);
    cudaStreamWaitEvent(st, g_cache.ev_end, 0);
  }
  const cudaError_t es = cudaStreamSynchronize(st);
  if (s != BF_OK) return s;
  return (e == cudaSuccess && es == cudaSuccess) ? BF_OK : BF_ERR_CUDA;
}
