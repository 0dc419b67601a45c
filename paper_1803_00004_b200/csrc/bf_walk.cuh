// Horizontal box-sum helpers of kernels 1 and 2 (walkers and paired prefix differences).
#pragma once

#include "bf_device.cuh"

namespace bf {

// H(y) for one channel slot over output columns [xs, xe): slide the exact int32 horizontal box
// sums H_tb of U'_t (term t, box b) and write F = round(sum_tb H_tb ax_tb / 2^32) (exact int64 products,
// one rounding) to Fcol[x * FPX]. Ur[o + u] is U'_0 at output column o, offset u; U'_t = Ur + t*srow.
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
      long long f = FRND;
#pragma unroll
      for (int m = 0; m < M; ++m) f = mad_wide(Hs[m], ax[m], f);
      pf[j * FPX] = fhi(f);
#pragma unroll
      for (int m = 0; m < M; ++m) Hs[m] += e[m][j] - l[m][j];
    }
    pf += 4 * FPX;
  }
  for (int j = 0; x < xe; ++x, ++j) {   // tail (< 4 outputs)
    long long f = FRND;
#pragma unroll
    for (int m = 0; m < M; ++m) f = mad_wide(Hs[m], ax[m], f);
    *pf = fhi(f);
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
      long long f = FRND;
#pragma unroll
      for (int m = 0; m < M; ++m) f = mad_wide(Hs[m], ax[m], f);
      pf[j * FPX] = fhi(f);
#pragma unroll
      for (int m = 0; m < M; ++m) Hs[m] += e[m][j] - l[m][j];
    }
    pf += 4 * FPX;
  }
  for (; x < xe; ++x) {   // tail (< 4 outputs): scalar
    long long f = FRND;
#pragma unroll
    for (int m = 0; m < M; ++m) f = mad_wide(Hs[m], ax[m], f);
    *pf = fhi(f);
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
      long long f = FRND;
#pragma unroll
      for (int m = 0; m < M; ++m) f = mad_wide(e[m][j] - l[m][j], ax[m], f);   // box sum = Q[hi+1] - Q[lo]
      pf[j * FPX] = fhi(f);
    }
    pf += 4 * FPX;
  }
  for (; x < xe; ++x) {   // tail (< 4 outputs): scalar
    long long f = FRND;
#pragma unroll
    for (int m = 0; m < M; ++m) f = mad_wide(base[m][x + 1 + hi[m]] - base[m][x + lo[m]], ax[m], f);
    *pf = fhi(f);
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
template <int MAXK, bool U8, bool CONSEC, bool FULL, bool MULTI, bool DIRECT = false>
__device__ __forceinline__ void combine_pixel(const KParams& P, const double2* lut64, const int4* Fr, float Ic,
                                              long long pix, float* __restrict__ out, longlong2* __restrict__ ws) {
  const int nk = P.nk;
  double c1, s1;
  pixel_angle<U8, DIRECT>(P, lut64, Ic, c1, s1);
  Cheb64 g;
  g.init(c1, s1);
  for (int j = 0; j < P.kval[0]; ++j) g.step();
  long long num = 0, den = 0;
  int mass = 0;   // F of the k = 0 cosine channel (the clipped spatial mass) for the repair flag
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
      if (P.kval[i] == 0) mass = f.x;
      den += (long long)wc * f.x;
      den += (long long)wsn * f.y;
      num += (long long)wc * f.z;
      num += (long long)wsn * f.w;
    }
  }
  if (MULTI) {   // bf_apply_multi: plans 1.. reuse the same F (single pass, no workspace)
    finish_pixel(P, num, den, Ic, pix, out, ws, true, mass);
    g.init(c1, s1);
    for (int j = 0; j < P.kval[0]; ++j) g.step();
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
      if (q < P.nplans) finish_pixel(P, nu[q - 1], de[q - 1], Ic, pix + q * P.plan_stride, out, ws, false, mass);
    return;
  }
  finish_pixel(P, num, den, Ic, pix, out, ws, true, mass);
}

}  // namespace bf
