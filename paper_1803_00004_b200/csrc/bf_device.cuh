// Device building blocks of the T = D kernels (sm_100a). Included by the kernel translation units.
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
//   H(y)  exact int32 horizontal box sums H_b of U', weighted into F = round(sum_b H_b ax_b / 2^32):
//         by walkers (kernel 1) or as differences of in-place prefix rows (kernels 2, 2b).
//   C(y)  per output pixel: combine weights a_k cos/sin(k pi I(x)/D) in fp64, rounded to int32,
//         num / den accumulated exactly in int64; out = D num / den (or I(x) if den <= 0, Q18).
// All T = D kernels perform the same integer arithmetic: their outputs are bitwise equal.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bf_params.h"

namespace bf {

constexpr float MAGIC = 12582912.0f;              // 1.5 * 2^23
constexpr int MAGIC_BITS = 0x4B400000;            // bit pattern of MAGIC
constexpr double MAGIC64 = 6755399441055744.0;    // 1.5 * 2^52: low word of fma(x, s, MAGIC64) = rint(x*s)

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
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
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
// F = round(sum_b H_b ax_b / 2^32): the box sums' exact int64 products accumulated from FRND = 2^31
// (one unbiased rounding; truncating each box's high word biased F by -1/2 per box, which the
// ill-conditioned pixels of wide-radius plans amplify, tools/numerics_pixel.py), high word taken
constexpr long long FRND = 1LL << 31;
__device__ __forceinline__ int fhi(long long f) { return (int)(f >> 32); }
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
// cos(pi t') to degree 21 / 22 (truncation < 2e-18 on |t'| <= 1/2), Horner in DFMA with the
// coefficients as constant-bank operands.
__device__ __forceinline__ void base_angle_f64(float I, double invD, double& c1, double& s1) {
  constexpr double kS[11] = {3.14159265358979312e+00, -5.16771278004996937e+00, 2.55016403987734508e+00,
                             -5.99264529320791883e-01, 8.21458866111281910e-02, -7.37043094571434784e-03,
                             4.66302805767612337e-04, -2.19153534478302037e-05, 7.95205400147550838e-07,
                             -2.29484289972698565e-08, 5.39266466260812482e-10};
  constexpr double kC[12] = {1.0, -4.93480220054467900e+00, 4.05871212641676760e+00, -1.33526276885458928e+00,
                             2.35330630358893123e-01, -2.58068913900140508e-02, 1.92957430940392206e-03,
                             -1.04638104924845650e-04, 4.30306958703294391e-06, -1.38789524622137608e-07,
                             3.60473079746249822e-09, -7.70070713060134610e-11};
  const double t = fma((double)I, invD, -0.5);
  const double z = t * t;
  double p = kS[10];
#pragma unroll
  for (int i = 9; i >= 0; --i) p = fma(p, z, kS[i]);
  double q = kC[11];
#pragma unroll
  for (int i = 10; i >= 0; --i) q = fma(q, z, kC[i]);
  c1 = -p * t;
  s1 = q;
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
// The first term k0 of a CTA is reached by k0 single steps from k = 0 (POW = false: every
// single-CTA launch, whose k0 is 0, so all kernels compute the same channel values bitwise), or
// by binary powering of (c1, s1) (POW = true: the CTAs of a cluster split whose terms begin at
// k0 = 8, 16, 24 would otherwise step k0 times per tap and row).
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
  // (C, S) = (c1, s1)^k0 by binary powering (k0 < 64; k0 = 0 leaves (C, S) = (1, 0))
  __device__ __forceinline__ void start(int k0) {
    if (k0 == 0) return;
    if ((k0 & (k0 - 1)) == 0) {
      // k0 = 2^m (the cluster split's first terms, 8 and 16): the general loop below reduces to m
      // squarings of (c1, s1) with the same operations; without its per-bit bookkeeping
      // (k0 = 8 and 16 as straight-line code: the loop's counter, branches and register moves
      // were a tenth of the two-column V role's instructions)
      u64 bc = C1, bs = S1;
      auto square = [&] {
        const u64 nbs = bs ^ 0x8000000080000000ull;
        const u64 bcn = fma2(bs, nbs, mul2(bc, bc));
        const u64 bsn = fma2(bc, bs, mul2(bs, bc));
        bc = bcn;
        bs = bsn;
      };
      if (k0 == 8) {
        square();
        square();
        square();
      } else if (k0 == 16) {
        square();
        square();
        square();
        square();
      } else {
#pragma unroll 1
        for (int k = k0; k > 1; k >>= 1) square();
      }
      C = bc;
      S = bs;
      return;
    }
    u64 bc = C1, bs = S1, nbs = NS1;
    bool first = true;
#pragma unroll 1
    for (int k = k0; k; k >>= 1) {
      if (k & 1) {
        if (first) {
          C = bc;
          S = bs;
          first = false;
        } else {
          const u64 Cn = fma2(S, nbs, mul2(C, bc));
          const u64 Sn = fma2(C, bs, mul2(S, bc));
          C = Cn;
          S = Sn;
        }
      }
      if (k > 1) {
        const u64 bcn = fma2(bs, nbs, mul2(bc, bc));
        const u64 bsn = fma2(bc, bs, mul2(bs, bc));
        bc = bcn;
        bs = bsn;
        nbs = bsn ^ 0x8000000080000000ull;
      }
    }
  }
};
__device__ __forceinline__ void rot1(float& c, float& s, float c1, float s1) {
  const float cn = fmaf(s, -s1, c * c1);
  const float sn = fmaf(c, s1, s * c1);
  c = cn;
  s = sn;
}
// scalar Rot2::start (bit-identical per lane)
__device__ __forceinline__ void rot1_start(float& c, float& s, float c1, float s1, int k0) {
  if (k0 == 0) return;
  float bc = c1, bs = s1;
  bool first = true;
#pragma unroll 1
  for (int k = k0; k; k >>= 1) {
    if (k & 1) {
      if (first) {
        c = bc;
        s = bs;
        first = false;
      } else {
        rot1(c, s, bc, bs);
      }
    }
    if (k > 1) {
      const float bcn = fmaf(bs, -bs, bc * bc);
      const float bsn = fmaf(bc, bs, bs * bc);
      bc = bcn;
      bs = bsn;
    }
  }
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

// n - 1 further steps of a recurrence (n = k_i - k_{i-1} >= 1 for non-consecutive terms), the
// common small gaps unrolled (a counted loop costs register moves and branches per step)
template <class F>
__device__ __forceinline__ void extra_steps(int n, F&& step) {
  if (n > 1) {
    step();
    if (n > 2) {
      step();
      if (n > 3) {
        step();
#pragma unroll 1
        for (int j = 4; j < n; ++j) step();
      }
    }
  }
}

// Spatial forms the kernels are instantiated for: NS box-pair terms, NBY vertical boxes (shared
// taps), NBX horizontal boxes per term.
template <int FORM>
struct Form;
template <> struct Form<1> { static constexpr int NS = 1, NBY = 1, NBX = 1; };   // one box (box K_s)
template <> struct Form<2> { static constexpr int NS = 1, NBY = 2, NBX = 2; };   // separable, 2 nested boxes (N_s = 9)
template <> struct Form<4> { static constexpr int NS = 1, NBY = 4, NBX = 4; };   // separable, up to 4 boxes
template <> struct Form<5> { static constexpr int NS = 2, NBY = 2, NBX = 1; };   // rank 2 (N_s = 5, three boxes)

// ------------------------------------------------------------------ the steps of a row

// (cos, sin)(pi i / D) of a u8 level by direct evaluation: the values the Case 2 LUT holds
__device__ __forceinline__ float2 u8_direct(float I, double invD) {
  double s, c;
  sincospi((double)I * invD, &s, &c);
  return make_float2((float)c, (float)s);
}

// sum of a packed pair of quantised values, q(lo) + q(hi) (both MAGIC biases removed)
__device__ __forceinline__ int sum_bits(u64 v) {
  int a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
  return (int)((unsigned)a + (unsigned)b - 2u * (unsigned)MAGIC_BITS);
}

// Vertical state at row y0 - 1 of the terms [t0, t0 + nk): U = urnd + sum over the rows v of the
// vertical boxes of the quantised channels (every tap's scale carries the box weight, nested
// boxes add up). Two rows per step on packed lanes (FFMA2 / FMUL2), each lane bit-identical to the tap
// arithmetic of v_row (same base angle, recurrence and quantisation), so the state equals the one
// the sliding enter / leave taps would build exactly; a row outside the window of box b (or the
// image, or the odd last row) gets scale 0, which quantises to exactly 0.
template <int MAXK, int NB, int NS, bool U8, bool CONSEC, bool FULL, bool POW = false, bool DIRECT = false>
__device__ __forceinline__ void v_init(const KParams& P, const void* __restrict__ in, const float2* lut,
                                       long long fbase, int col, bool colok, int y0, int t0, int nk,
                                       int (&U)[NS * 4 * MAXK]) {
#pragma unroll
  for (int ch = 0; ch < NS * 4 * MAXK; ++ch) U[ch] = P.urnd;
  const u64 MM = pk(MAGIC, MAGIC);
  const int k0 = P.kval[t0];
  for (int v = P.vmin; v <= P.vmax; v += 2) {
    const int ra = y0 - 1 + v, rb = ra + 1;
    const bool oka = colok && ra >= 0 && ra < P.H;
    const bool okb = colok && v + 1 <= P.vmax && rb >= 0 && rb < P.H;
    const float Ia = oka ? load_pixel(in, U8, fbase + (long long)ra * P.W + col) : 0.f;
    const float Ib = okb ? load_pixel(in, U8, fbase + (long long)rb * P.W + col) : 0.f;
    Rot2 g2;
    if (U8) {
      const float2 ta = DIRECT ? u8_direct(Ia, P.invD) : lut[(int)Ia];
      const float2 tb = DIRECT ? u8_direct(Ib, P.invD) : lut[(int)Ib];
      g2.init(ta.x, ta.y, tb.x, tb.y);
    } else {
      u64 c1, s1;
      base_angle_f32x2(Ia, Ib, P, c1, s1);
      g2.init2(c1, s1);
    }
    u64 QS[NS][NB], QI[NS][NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const bool ina = oka && (b < P.nby) && v >= P.vlo[b] && v <= P.vhi[b];
      const bool inb = okb && (b < P.nby) && v + 1 >= P.vlo[b] && v + 1 <= P.vhi[b];
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        QS[t][b] = pk(ina ? P.qs[t][b] : 0.f, inb ? P.qs[t][b] : 0.f);
        QI[t][b] = pk(ina ? P.qsD[t][b] * Ia : 0.f, inb ? P.qsD[t][b] * Ib : 0.f);
      }
    }
    if (POW) g2.start(k0);
    else
      for (int j = 0; j < k0; ++j) g2.step();
#pragma unroll
    for (int i = 0; i < MAXK; ++i) {
      if (FULL || i < nk) {
        if (i > 0) {
          g2.step();
          if (!CONSEC) extra_steps(P.kstep[t0 + i], [&] { g2.step(); });
        }
#pragma unroll
        for (int t = 0; t < NS; ++t)
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            int* Ut = U + t * 4 * MAXK;
            Ut[4 * i + 0] += sum_bits(fma2(g2.C, QS[t][b], MM));
            Ut[4 * i + 1] += sum_bits(fma2(g2.S, QS[t][b], MM));
            Ut[4 * i + 2] += sum_bits(fma2(g2.C, QI[t][b], MM));
            Ut[4 * i + 3] += sum_bits(fma2(g2.S, QI[t][b], MM));
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

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Named barriers of the warp-specialised kernels (b = row parity, g = channel group)
constexpr int BAR_U_FULL = 0, BAR_U_EMPTY = 4, BAR_Q_FULL = 8, BAR_F_FULL = 12, BAR_F_EMPTY = 14;

// V's per-group hooks: wait until group g's buffer of this row parity is free (its consumers
// are done with row y-2), and publish group g once written
struct GroupSync {
  int b, nfree, nfull;
  bool wait;
  __device__ __forceinline__ void begin(int g) const {
    if (wait) bar_sync(BAR_U_EMPTY + 2 * b + g, nfree);
  }
  __device__ __forceinline__ void end(int g) const { bar_arrive(BAR_U_FULL + 2 * b + g, nfull); }
};

// V(y): slide the vertical state one row (enter / leave taps of every box, packed in pairs)
// and store U' = U >> ush of every channel slot at Ucol[slot * UP]. Terms [t0, t0 + nk).
template <int MAXK, int NB, int NS, bool U8, bool CONSEC, bool FULL, int UP, class Hook = GroupSync, bool POW = false,
          bool DIRECT = false>
__device__ __forceinline__ void v_row(const KParams& P, const float2* lut, bool colok, int y, int t0, int nk,
                                      const float (&Ipre)[NB][2], int (&U)[NS * 4 * MAXK], int* Ucol,
                                      const Hook* hook = nullptr) {
  u64 QS[NS][NB], QI[NS][NB];
  Rot2 g2[NB];
  const int k0 = P.kval[t0];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const float Ie = Ipre[b][0], Il = Ipre[b][1];
    if (U8) {
      const float2 te = DIRECT ? u8_direct(Ie, P.invD) : lut[(int)Ie];
      const float2 tl = DIRECT ? u8_direct(Il, P.invD) : lut[(int)Il];
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
    if (POW) g2[b].start(k0);
    else
      for (int j = 0; j < k0; ++j) g2[b].step();
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
          extra_steps(P.kstep[t0 + i], [&] {
#pragma unroll
            for (int b = 0; b < NB; ++b) g2[b].step();
          });
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

// Exclusive prefix of one U' row in place, 8 columns per step (two 16-byte loads / stores, one
// IADD3 per column); int32 wrap-around keeps every box difference exact. Q[n] = total.
// prefix_part scans columns [e0, e1) with the running total carried in and returned (a row scanned
// in pieces, as its columns become available, equals the row scanned at once).
#ifndef BF_SCAN_UNROLL
#define BF_SCAN_UNROLL 8
#endif
constexpr int SCAN_UNROLL = BF_SCAN_UNROLL;
__device__ __forceinline__ int prefix_part(int* Q, int e0, int e1, int carry) {
#pragma unroll SCAN_UNROLL
  for (int e = e0; e < e1; e += 8) {
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
  return carry;
}
__device__ __forceinline__ void prefix_row(int* Q, int n) { Q[n] = prefix_part(Q, 0, n, 0); }

// Fallback bookkeeping (Q18): optional per-pixel mask and a warp-aggregated counter.
__device__ __forceinline__ void note_fallback(unsigned long long* cnt, unsigned char* mask, long long pix, bool fb) {
  if (mask) mask[pix] = fb ? 1 : 0;   // (a flagged pixel's entry is rewritten by the repair pass)
  if (cnt) {
    const unsigned act = __activemask();
    const unsigned m = __ballot_sync(act, fb);
    if (m && (threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(cnt, (unsigned long long)__popc(m));
  }
}

// Appends the pixel to the repair list when den < tau mass (RepairSink): den and mass in the same
// units (mass = the k = 0 cosine channel's box sum; mass_full scaled by mass_unit when that channel
// is not at hand). Returns true if flagged (its fallback bookkeeping is then the repair pass's).
__device__ __forceinline__ bool flag_bool(const RepairSink& R, bool fl, long long pix) {
  const unsigned act = __activemask();
  const unsigned bal = __ballot_sync(act, fl);
  if (bal) {
    const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(R.count, (unsigned)__popc(bal));
    base = __shfl_sync(act, base, leader);
    if (fl) {
      const unsigned i = base + __popc(bal & ((1u << lane) - 1));
      if (i < R.cap) {
        R.list[i] = (unsigned long long)pix;
        R.acc[i] = RepAcc{0, 0, 0u, 0u};
      }
    }
  }
  return fl;
}
__device__ __forceinline__ bool flag_pixel(const RepairSink& R, double den, double mass, double mass_unit,
                                           long long pix) {
  if (!R.count) return false;
  const double m = mass > 0 ? mass : R.mass_full * mass_unit;
  return flag_bool(R, den < R.tau_w * m, pix);
}
__device__ __forceinline__ bool flag_pixel(const RepairSink& R, long long den, int mass, long long pix) {
  return flag_pixel(R, (double)den, (double)mass, 1.0, pix);
}

// General plans (several separable passes, P.dunit != 0): the launch's num / den, converted to
// absolute units (n with the factor D of the I channels), go to / from the fp64 workspace; the last
// launch divides. The repair flag then compares den with tau times the unclipped spatial mass in
// the same units (rep.tau_w = tau, rep.mass_full = sum K~_s).
__device__ __forceinline__ void finish_dws(const KParams& P, double n, double d, float Ic, long long pix,
                                           float* __restrict__ out, void* ws) {
  double2* w = static_cast<double2*>(ws);
  if (P.pass >= 2) {
    const double2 a = w[pix];
    n += a.x;
    d += a.y;
  }
  if (P.pass == 1 || P.pass == 2) {
    w[pix] = make_double2(n, d);
    return;
  }
  const bool fb = !(d > 0);
  out[pix] = fb ? Ic : (float)(n / d);
  const bool fl = flag_pixel(P.rep, d, 0.0, 1.0, pix);
  note_fallback(P.fb_count, P.fb_mask, pix, fb && !fl);
}

// out = D num / den (den <= 0: I(x), Q18), or the int64 pair to / from the multi-pass workspace;
// mass = the k = 0 cosine channel's F of this pixel (0 if not at hand) for the repair flag
__device__ __forceinline__ void finish_pixel(const KParams& P, long long num, long long den, float Ic, long long pix,
                                             float* __restrict__ out, longlong2* __restrict__ ws, bool count = true,
                                             int mass = 0) {
  if (P.dunit != 0.0) {
    finish_dws(P, (double)num * P.dunit * P.D, (double)den * P.dunit, Ic, pix, out, ws);
    return;
  }
  if (P.pass == 1) {
    ws[pix] = make_longlong2(num, den);
    return;
  }
  if (P.pass >= 2) {
    const longlong2 acc = ws[pix];
    num += acc.x;
    den += acc.y;
  }
  if (P.pass == 2) {
    ws[pix] = make_longlong2(num, den);
    return;
  }
  const bool fb = !(den > 0);
  out[pix] = fb ? Ic : (float)(P.D * (double)num / (double)den);
  const bool fl = flag_pixel(P.rep, den, mass, pix);
  if (count) note_fallback(P.fb_count, P.fb_mask, pix, fb && !fl);
}

// Kernel 2b's finish from the per-box accumulators num_b = sum W H_b, den_b (exact int64):
// num = sum_b ax_b num_b, den likewise, formed in fp64 (relative rounding 2^-53, far below the
// channel values' fp32 error); out = D num / den, or I(x) if den <= 0 (Q18). mass is in the same
// units (sum_b ax_b H_b of the k = 0 cosine channel's box sums hm_b, 2^32 times the F units of
// finish_pixel; hm_b = 0: not at hand), formed only when den is below tau times the bound of any
// clipped mass.
__device__ __forceinline__ void finish_pixel_pb(const KParams& P, const long long (&num)[2], const long long (&den)[2],
                                                int ax0, int ax1, float Ic, long long pix, float* __restrict__ out,
                                                int hm0, int hm1, void* ws) {
  const double n = fma((double)num[1], (double)ax1, (double)num[0] * (double)ax0);
  const double d = fma((double)den[1], (double)ax1, (double)den[0] * (double)ax0);
  if (P.dunit != 0.0) {
    const double u = P.dunit * 2.3283064365386963e-10;   // / 2^32: F units
    finish_dws(P, n * u * P.D, d * u, Ic, pix, out, ws);
    return;
  }
  const bool fb = !(d > 0);
  out[pix] = fb ? Ic : (float)(P.D * n / d);
  if (!P.rep.count) {
    note_fallback(P.fb_count, P.fb_mask, pix, fb);
    return;
  }
  const RepairSink& R = P.rep;
  bool cand = d < R.tau_w * (R.mass_bound * 4294967296.0);
  if (cand) {
    const double mass = (hm0 | hm1) ? fma((double)hm1, (double)ax1, (double)hm0 * (double)ax0) : 0.0;
    cand = d < R.tau_w * (mass > 0 ? mass : R.mass_full * 4294967296.0);
  }
  const bool fl = flag_bool(R, cand, pix);
  note_fallback(P.fb_count, P.fb_mask, pix, fb && !fl);
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

// fp64 (cos, sin)(pi I / D) of an output pixel: LUT (u8) or polynomial (f32)
template <bool U8, bool DIRECT = false>
__device__ __forceinline__ void pixel_angle(const KParams& P, const double2* lut64, float Ic, double& c1, double& s1) {
  if (U8) {
    if (DIRECT) {
      sincospi((double)Ic * P.invD, &s1, &c1);
      return;
    }
    const double2 t = lut64[(int)Ic];
    c1 = t.x;
    s1 = t.y;
  } else {
    base_angle_f64(Ic, P.invD, c1, s1);
  }
}

}  // namespace bf
