// Kernel 2b's vertical state in tensor memory (TMEM). The V role's exact int32 sliding sums U
// (4 channels per range term) live in TMEM instead of registers: a 128-lane x
// 512-column array of 32-bit cells per SM that a warp reaches only in its own 32-lane quarter
// (lane quarter = warp id % 4) through tcgen05.ld / tcgen05.st. Every V thread owns one TMEM lane
// and 4 * MAXK consecutive columns; it moves its state in batches of four terms (16 cells, one
// 32x32b.x16 load and store each), which frees the ~64 registers the state held for the roles
// that are latency-bound (the FH role). The arithmetic is that of v_init / v_row lane for lane:
// the results are bitwise unchanged.
#pragma once

#include "bf_device.cuh"

namespace bf {
namespace tm {

__device__ __forceinline__ void ld16(unsigned taddr, int (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void st16(unsigned taddr, const int (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One warp allocates `cols` columns (a power of two >= 32) and publishes the base address through
// shared memory; every thread reads it after the fence / barrier / fence sequence.
__device__ __forceinline__ void alloc(unsigned* slot, unsigned cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(slot)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(unsigned taddr, unsigned cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// v_init (bf_device.cuh) with the state in TMEM, one batch of four terms (16 cells in registers)
// of one column: row pairs inner; the batch re-derives its terms' channels from k0 with the same
// recurrence steps, so every cell equals v_init's bitwise. Batches are independent, so any warp
// of the column's lane quarter can compute any of them (the caller spreads them over every warp
// of the SM sub-partition, the FH and S warps included: they have nothing else to do before the
// first row). The caller waits for the stores (wait_st) and orders them before the first v_row.
template <int MAXK, int NB, bool U8, bool CONSEC, bool FULL, bool POW>
__device__ __forceinline__ void v_init_batch(const KParams& P, const void* __restrict__ in, const float2* lut,
                                             long long fbase, int col, bool colok, int y0, int t0, int nk, int bt,
                                             unsigned taddr_bt) {
  const u64 MM = pk(MAGIC, MAGIC);
  const int k0 = P.kval[t0];
  int ub[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) ub[c] = P.urnd;
  for (int v = P.vmin; v <= P.vmax; v += 2) {
    const int ra = y0 - 1 + v, rb = ra + 1;
    const bool oka = colok && ra >= 0 && ra < P.H;
    const bool okb = colok && v + 1 <= P.vmax && rb >= 0 && rb < P.H;
    const float Ia = oka ? load_pixel(in, U8, fbase + (long long)ra * P.W + col) : 0.f;
    const float Ib = okb ? load_pixel(in, U8, fbase + (long long)rb * P.W + col) : 0.f;
    Rot2 g2;
    if (U8) {
      const float2 ta = lut[(int)Ia], tb = lut[(int)Ib];
      g2.init(ta.x, ta.y, tb.x, tb.y);
    } else {
      u64 c1, s1;
      base_angle_f32x2(Ia, Ib, P, c1, s1);
      g2.init2(c1, s1);
    }
    u64 QS[NB], QI[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const bool ina = oka && (b < P.nby) && v >= P.vlo[b] && v <= P.vhi[b];
      const bool inb = okb && (b < P.nby) && v + 1 >= P.vlo[b] && v + 1 <= P.vhi[b];
      QS[b] = pk(ina ? P.qs[0][b] : 0.f, inb ? P.qs[0][b] : 0.f);
      QI[b] = pk(ina ? P.qsD[0][b] * Ia : 0.f, inb ? P.qsD[0][b] * Ib : 0.f);
    }
    if (POW) g2.start(k0);
    else
      for (int j = 0; j < k0; ++j) g2.step();
    // the terms before this batch: recurrence steps only
    for (int i = 1; i <= 4 * bt; ++i) {
      g2.step();
      if (!CONSEC) extra_steps(P.kstep[t0 + i], [&] { g2.step(); });
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = 4 * bt + j;
      if (FULL || i < nk) {
        if (j > 0) {
          g2.step();
          if (!CONSEC) extra_steps(P.kstep[t0 + i], [&] { g2.step(); });
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          ub[4 * j + 0] += sum_bits(fma2(g2.C, QS[b], MM));
          ub[4 * j + 1] += sum_bits(fma2(g2.S, QS[b], MM));
          ub[4 * j + 2] += sum_bits(fma2(g2.C, QI[b], MM));
          ub[4 * j + 3] += sum_bits(fma2(g2.S, QI[b], MM));
        }
      }
    }
  }
  st16(taddr_bt, ub);
}

// v_row (bf_device.cuh) with the state in TMEM, one batch of four terms in registers at a time.
// HOOK: the per-group hand-off barriers run inside (one column per thread); without, the caller
// brackets the columns of a thread (COLS = 2, one channel group).
template <int MAXK, int NB, bool U8, bool CONSEC, bool FULL, int UP, bool POW, bool HOOK = true>
__device__ __forceinline__ void v_row(const KParams& P, const float2* lut, bool colok, int y, int t0, int nk,
                                      const float (&Ipre)[NB][2], unsigned taddr, int* Ucol, const GroupSync& hook) {
  u64 QS[NB], QI[NB];
  Rot2 g2[NB];
  const int k0 = P.kval[t0];
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
    QS[b] = pk(oke ? P.qs[0][b] : 0.f, okl ? P.qs[0][b] : 0.f);
    QI[b] = pk(oke ? P.qsD[0][b] * Ie : 0.f, okl ? P.qsD[0][b] * Il : 0.f);
    if (POW) g2[b].start(k0);
    else
      for (int j = 0; j < k0; ++j) g2[b].step();
  }
  const u64 MM = pk(MAGIC, MAGIC);
  wait_st();   // the previous row's stores have landed
  int ub[16];
#pragma unroll
  for (int i = 0; i < MAXK; ++i) {
    if (FULL || i < nk) {
      if (HOOK && (i & 7) == 0) hook.begin(i >> 3);
      if ((i & 3) == 0) {
        ld16(taddr + 4 * i, ub);
        wait_ld();
      }
      if (i > 0) {
        if (CONSEC) {
#pragma unroll
          for (int b = 0; b < NB; ++b) g2[b].step();
        } else {   // k_i - k_{i-1} >= 1 steps as one loop (no separate paths for the gaps to merge)
          int n = P.kstep[t0 + i];
#pragma unroll 1
          do {
#pragma unroll
            for (int b = 0; b < NB; ++b) g2[b].step();
          } while (--n > 0);
        }
      }
      const int j = i & 3;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const u64 C = g2[b].C, Sn = g2[b].S;
        ub[4 * j + 0] += diff_bits(fma2(C, QS[b], MM));
        ub[4 * j + 1] += diff_bits(fma2(Sn, QS[b], MM));
        ub[4 * j + 2] += diff_bits(fma2(C, QI[b], MM));
        ub[4 * j + 3] += diff_bits(fma2(Sn, QI[b], MM));
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) Ucol[(4 * i + c) * UP] = ub[4 * j + c] >> P.ush;
      if (j == 3 || (FULL ? i + 1 == MAXK : i + 1 == nk)) st16(taddr + 4 * (i - j), ub);
      if (HOOK && ((i & 7) == 7 || (FULL ? i + 1 == MAXK : i + 1 == nk))) hook.end(i >> 3);
    }
  }
}

}  // namespace tm
}  // namespace bf
