// Kernel 2b: fused box differences + combine (bf_ws2_kernel), the default T = D kernel for
// separable plans with at most two boxes per axis. Three warp-specialised roles joined by a
// two-deep ring of U' rows and named barriers (bar.arrive / bar.sync per row parity and
// 32-channel group):
//   FH  warps 0..      one thread per output pixel: for every channel slot of group g,
//                      F = round(sum_b (Q[x + hi_b + 1] - Q[x + lo_b]) ax_b / 2^32) (lanes = consecutive
//                      x: conflict-free), accumulated straight into the exact int64 num / den with
//                      the pixel's fp64 combine weights (per range plan for bf_apply_multi)
//   S   next warps     warp g turns group g's U' rows into exclusive prefix rows Q in place
//   V   last 12 warps  COLS extended columns per thread: slides the vertical sums, writes U'(y)
// These are LOGICAL warp ids: the host maps them onto the physical warps (KParams::wmap, built by
// ws2_warp_map in bf_apply.cu from a measured placement rule) so that the S warps share one SM
// sub-partition and the working FH / V warps are spread evenly over the four; within a
// sub-partition the V warps take the lowest physical ids. Before the first row every warp, whatever
// its role, computes part of the band's initial vertical state (tm::v_init_batch).
//
// COLS = 2 (wide radii, e.g. cfg4's r = 192): each V thread keeps the vertical state of two
// columns 384 apart, so a strip covers 768 extended columns (output strip 352 wide instead of
// 0 at a 384-column halo) with 8 terms per CTA.
//
// CL: the range terms are split over a cluster of G CTAs on the same strip and band (CTA c owns
// terms [c tpc, c tpc + tpc)): every CTA computes its partial int64 (num_b, den_b) per output
// pixel; CTAs 1..G-1 add them into CTA 0's per-row-parity slot with red.async.add (distributed
// shared memory, exact integer adds in any order), completing CTA 0's mbarrier FULL[b] by
// transaction bytes; CTA 0 adds the slot to its own partials (the result is bitwise that of one
// CTA doing all terms), clears it and releases it through the senders' EMPTY[b] mbarriers. No HBM
// workspace and one launch for up to G * tpc terms (cfg4: 24 terms = 3 CTAs x 8).
//
// PB (one range plan): num / den are accumulated per horizontal box b, num_b = sum W H_b with the
// exact box sums H_b, and combined as sum_b ax_b num_b in fp64 at the end (no rounded F).
//
// DUMP (bf_precompute, Case 1 of P:1200-1219): FH writes the box-filtered channels F of its pixel
// to the cache planes instead of combining them.
#pragma once

#include "bf_device.cuh"
#include "bf_tm.cuh"

namespace bf {
namespace ws2 {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned map_rank(unsigned laddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(laddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned a, unsigned bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n}" ::"r"(a),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned raddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
__device__ __forceinline__ void st_async_pair(unsigned raddr, long long a, long long b, unsigned rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.s64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(a), "l"(b), "r"(rmbar)
               : "memory");
}
// exact int64 add into another CTA's shared memory, completing its mbarrier by 8 transaction bytes
__device__ __forceinline__ void red_async_add(unsigned raddr, long long v, unsigned rmbar) {
  asm volatile("red.async.relaxed.cluster.shared::cluster.mbarrier::complete_tx::bytes.add.u64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(v), "r"(rmbar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int MBAR_BYTES = 64;
#ifndef BF_TM
#define BF_TM 1
#endif
#ifndef BF_TM_VREG
#define BF_TM_VREG 64
#endif
#ifndef BF_TM_VREG2
#define BF_TM_VREG2 80
#endif
#ifndef BF_TM_FHREG
#define BF_TM_FHREG 80
#endif
constexpr int W2_LAUNCH_REG = 80;   // registers per thread at launch (768 threads, one CTA per SM)
constexpr int BAR_TM_DONE = 15;   // V warps: every TMEM access done (the allocating warp then frees)
constexpr int BAR_INIT = 12;      // every warp: the band's initial vertical state is in TMEM

// diagnostic builds only (tools/build_variant.py): drop one role's arithmetic, keep its barriers
#ifndef BF_S_REG
#define BF_S_REG 0   // S role registers (0 = default 48 / 56)
#endif
#ifndef BF_HALFSCAN
#define BF_HALFSCAN 1
#endif
#ifndef BF_X_NOV
#define BF_X_NOV 0
#endif
#ifndef BF_X_NOS
#define BF_X_NOS 0
#endif
#ifndef BF_X_NOFH
#define BF_X_NOFH 0
#endif
#ifndef BF_X_NOW
#define BF_X_NOW 0
#endif
#ifndef BF_X_NOLDS
#define BF_X_NOLDS 0
#endif   // mbarriers at the start of shared memory (FULL[XS], EMPTY[XS])

template <int MAXK, int FORM, bool U8, bool CONSEC, bool FULL, int NPL, int COLS, bool CL, bool DUMP>
__global__ void __launch_bounds__(W2_THREADS, 1)
    bf_ws2_kernel(const KParams P, const void* __restrict__ in, float* __restrict__ out, longlong2* __restrict__ ws) {
  constexpr int NS = Form<FORM>::NS, NB = Form<FORM>::NBY, NBX = Form<FORM>::NBX;
  constexpr int M = NS * NBX;
  static_assert(NS == 1 && M <= 2, "the FH role handles separable forms with at most two x boxes");
  static_assert(COLS == 1 || MAXK == 8, "two columns per V thread: 8 terms per CTA (one channel group)");
  constexpr int NTH = W2_THREADS;
  constexpr int NFH = w2_nfh(COLS), NSW = w2_ns(COLS);
  constexpr int H0 = 0, S0 = NFH, V0 = NFH + NSW;
  static_assert(V0 + W2_V == NTH, "role sizes");
  constexpr int LREG = W2_LAUNCH_REG;
  constexpr int XS = W2_XSLOTS;   // row slots of the cluster exchange
  constexpr int UP = w2_up(COLS);
  constexpr bool PB = NPL == 1 && !DUMP;   // per-box accumulators (see the FH role)
  // TM: the V role's sliding sums in tensor memory (bf_tm.cuh; one column per V thread), which
  // moves registers from V to the latency-bound FH role
  constexpr bool TM = BF_TM;
  // registers per role (setmaxnreg; the pool is the launch's LREG x NTH):
  //   TM     V 384 x 64 + FH 320 x 80 + S 64 x 48 = 53248 <= 768 x 80 (measured: V at 64 is
  //          1.83 ms on cfg2 against 1.89 at 72 and 80)
  //          two columns: V 384 x 80 + FH 352 x 80 + S 32 x 48 = 60416 (cfg4 32.2 ms; 37.3 at 64)
  //   else   V 384 x 112 + (FH + S) 384 x 48      = 61440
  constexpr int VREG = TM ? (COLS == 2 ? BF_TM_VREG2 : BF_TM_VREG) : (NPL > 1 ? 104 : 112);
  constexpr int OREG = BF_S_REG ? BF_S_REG : (NPL > 1 ? 56 : 48);
  constexpr int FHREG = TM ? BF_TM_FHREG : OREG;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(smem_raw);   // FULL[XS], EMPTY[XS]
  int* Ubuf = reinterpret_cast<int*>(smem_raw + MBAR_BYTES);                     // [2][4 nk][UP]
  float2* lut = reinterpret_cast<float2*>(smem_raw + P.l_off);
  double2* lut64 = reinterpret_cast<double2*>(lut + 256);
  longlong2* red = reinterpret_cast<longlong2*>(smem_raw + P.r_off);              // [2][TW][2]: sum of the senders' (num_b, den_b)

  // Warp roles by a host-built map (P.wmap: physical warp -> logical warp): the four SM
  // sub-partitions (physical warp id mod 4) get equal shares of the roles' issue load, whatever part
  // of the FH / V warps the strip width leaves idle. Everything below uses the logical thread id.
  const int pw = (int)threadIdx.x >> 5;
  const int tid = ((int)P.wmap[pw] << 5) | ((int)threadIdx.x & 31);
  const int G = CL ? P.G : 1;
  // the CTA's rank in its (G, 1, 1) cluster, from blockIdx so that the compiler sees a warp-uniform
  // value: the per-term branches on kval / kstep of this CTA's terms then run on the uniform datapath
  const int rank = CL ? (int)(blockIdx.x % (unsigned)P.G) : 0;
  const int t0 = CL ? rank * P.tpc : 0;                      // this CTA's terms [t0, t0 + nkc)
  const int nkc = CL ? min(P.tpc, P.nk - t0) : P.nk;
  const int ngrp = (4 * nkc + 31) >> 5;
  const int x0 = (CL ? (int)blockIdx.x / G : (int)blockIdx.x) * P.TW;
  const int y0 = P.yb + blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int TWv = min(P.TW, P.W - x0);
  const int yend = min(y0 + P.TH, P.ye);
  const int wv = P.wv;                            // extended columns scanned (multiple of 8, <= W2_V * COLS)
  const int srow = 4 * nkc * UP;                  // ints per U' buffer
  constexpr int n_ufull = W2_V + 32;              // U_FULL: V arrive, S_g sync
  constexpr int n_uempty = W2_V + NFH;            // U_EMPTY: FH arrive, V sync
  constexpr int n_qfull = 32 + NFH;               // Q_FULL: S_g arrive, FH sync

  fill_luts<U8>(P, lut, lut64, tid, NTH);
  __shared__ unsigned tmem_slot;
  if constexpr (TM) {
    if (tid >= V0 && tid < V0 + 32) tm::alloc(&tmem_slot, (unsigned)P.tmcols);   // the first V warp allocates
    tm::fence_before();
  }
  if constexpr (CL) {
    if (tid == 0) {
      for (int i = 0; i < XS; ++i) {
        mbar_init(smem_u32(&mbar[i]), 1);               // FULL[slot]: CTA 0's expect_tx arrival + the senders' bytes
        mbar_init(smem_u32(&mbar[XS + i]), NFH / 32);   // EMPTY[slot]: every FH warp of CTA 0 once per row
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < XS * 2 * P.TW; i += NTH) red[i] = make_longlong2(0, 0);   // every slot
    cluster_sync();
  } else {
    __syncthreads();
  }

  if constexpr (TM) {
    // ---------------------------------------------------------- vertical state of the band's first row
    // Every warp of the CTA takes part: the units (working V warp, column, batch of four terms) of
    // a lane quarter are dealt round-robin to the six warps of that SM sub-partition (a warp
    // reaches exactly its own quarter of TMEM), so the FH and S warps, idle until the first row
    // arrives, halve the time before it.
    tm::fence_after();
    if (!BF_X_NOV) {
      const int q = pw & 3;
      const int nbt = FULL ? MAXK / 4 : (nkc + 3) >> 2;
      const int upw = COLS * nbt, nun = (int)P.nvq[q] * upw;
      const unsigned tq = tmem_slot + ((unsigned)(32 * q) << 16);
      for (int u = pw >> 2; u < nun; u += NTH / 128) {
        const int k = u / upw, r = u - k * upw, j = r / nbt, bt = r - j * nbt;
        const int e = (((int)P.vq[q][k]) << 5 | ((int)threadIdx.x & 31)) + j * W2_V;   // extended column
        if ((e & ~31) < wv) {
          const int cj = x0 - P.rlo_x + e;
          tm::v_init_batch<MAXK, NB, U8, CONSEC, FULL, CL>(P, in, lut, fbase, cj, (cj >= 0) & (cj < P.W) & (e < wv), y0, t0,
                                                           nkc, bt, tq + (unsigned)((k * COLS + j) * 4 * MAXK + 16 * bt));
        }
      }
      tm::wait_st();
    }
    tm::fence_before();
    bar_sync(BAR_INIT, NTH);
    tm::fence_after();
  }
  if (tid >= V0) {
    // ------------------------------------------------------------ V role
    if constexpr (VREG > LREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(VREG));
    else if constexpr (VREG < LREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(VREG));
    const int vt = tid - V0;
    int col[COLS];
    bool colok[COLS], vwork[COLS];
#pragma unroll
    for (int j = 0; j < COLS; ++j) {
      const int e = vt + j * W2_V;                  // extended column
      col[j] = x0 - P.rlo_x + e;
      colok[j] = (col[j] >= 0) & (col[j] < P.W) & (e < wv);
      vwork[j] = ((vt & ~31) + j * W2_V) < wv;     // warp-uniform: this block of 32 columns is scanned
    }
    int U[TM ? 1 : COLS][TM ? 1 : NS * 4 * MAXK];
    // TM: this thread's TMEM lane (the lane quarter of its PHYSICAL warp) and COLS x 4 MAXK columns
    // (the V warps of a quarter take consecutive blocks, P.tmblk; column j of the thread at + 4 MAXK j)
    const unsigned taddr = TM ? tmem_slot + ((unsigned)(32 * (pw & 3)) << 16) +
                                    (unsigned)((int)P.tmblk[pw] * COLS * 4 * MAXK)
                              : 0u;
    // prefetched taps: COLS == 1 the next row's; COLS == 2 the next (row, column) in the order
    // (y, 0), (y, 1), (y + 1, 0), ... (one column's worth of registers)
    float Ipre[NB][2];
    if constexpr (!TM) {
#pragma unroll
      for (int j = 0; j < COLS; ++j)
        if (vwork[j] && !BF_X_NOV)
          v_init<MAXK, NB, NS, U8, CONSEC, FULL, CL>(P, in, lut, fbase, col[j], colok[j], y0, t0, nkc, U[j]);
    }
    load_taps<NB, U8>(P, in, fbase, col[0], colok[0], y0, Ipre);
    for (int y = y0; y < yend; ++y) {
      const int b = (y - y0) & 1;
      const GroupSync hook{b, n_uempty, n_ufull, y - y0 >= 2};
      int* Ub = Ubuf + b * srow + vt;
      if constexpr (COLS == 1) {
        if (vwork[0] && !BF_X_NOV) {
          float Icur[NB][2];
#pragma unroll
          for (int bb = 0; bb < NB; ++bb) {
            Icur[bb][0] = Ipre[bb][0];
            Icur[bb][1] = Ipre[bb][1];
          }
          if (y + 1 < yend) load_taps<NB, U8>(P, in, fbase, col[0], colok[0], y + 1, Ipre);
          if constexpr (TM) tm::v_row<MAXK, NB, U8, CONSEC, FULL, UP, CL>(P, lut, colok[0], y, t0, nkc, Icur, taddr, Ub, hook);
          else v_row<MAXK, NB, NS, U8, CONSEC, FULL, UP, GroupSync, CL>(P, lut, colok[0], y, t0, nkc, Icur, U[0], Ub, &hook);
        } else {
          for (int g = 0; g < ngrp; ++g) {
            hook.begin(g);
            hook.end(g);
          }
        }
      } else {
        hook.begin(0);
#pragma unroll
        for (int j = 0; j < COLS; ++j) {
          // the column's coordinates are recomputed per row (cheap) rather than held across the
          // loop: with two 32-channel states the V role has no registers to spare
          const int e = vt + j * W2_V;
          const int cj = x0 - P.rlo_x + e;
          const bool okj = (cj >= 0) & (cj < P.W) & (e < wv);
          float Icur[NB][2];
#pragma unroll
          for (int bb = 0; bb < NB; ++bb) {
            Icur[bb][0] = Ipre[bb][0];
            Icur[bb][1] = Ipre[bb][1];
          }
          {   // prefetch the taps of the next (row, column)
            const int jn = (j + 1) % COLS, yn = j + 1 < COLS ? y : y + 1;
            const int en = vt + jn * W2_V, cn = x0 - P.rlo_x + en;
            if (yn < yend) load_taps<NB, U8>(P, in, fbase, cn, (cn >= 0) & (cn < P.W) & (en < wv), yn, Ipre);
          }
          if (((vt & ~31) + j * W2_V) < wv) {
            if constexpr (TM)
              tm::v_row<MAXK, NB, U8, CONSEC, FULL, UP, CL, false>(P, lut, okj, y, t0, nkc, Icur, taddr + 4 * MAXK * j,
                                                                   Ub + j * W2_V, hook);
            else
              v_row<MAXK, NB, NS, U8, CONSEC, FULL, UP, GroupSync, CL>(P, lut, okj, y, t0, nkc, Icur, U[j],
                                                                      Ub + j * W2_V);
          }
          // the first W2_V columns are written: the S warp scans them while the second column of
          // every V thread is still being computed (barrier ids of group 1, unused with one group)
          if (BF_HALFSCAN && j == 0) bar_arrive(BAR_U_FULL + 2 * b + 1, n_ufull);
        }
        hook.end(0);
      }
    }
    // drain: the FH warps' last releases
    for (int y = max(y0, yend - 2); y < yend; ++y)
      for (int g = 0; g < ngrp; ++g) bar_sync(BAR_U_EMPTY + 2 * ((y - y0) & 1) + g, n_uempty);
    if constexpr (TM) {   // every V warp's TMEM accesses are done: the allocating (V) warp frees
      tm::fence_before();
      bar_sync(BAR_TM_DONE, W2_V);
      tm::fence_after();
      if (tid < V0 + 32) tm::dealloc(tmem_slot, (unsigned)P.tmcols);
    }
  } else if (tid >= S0) {
    // ------------------------------------------------------------ S role: prefix scans
    if constexpr (OREG < LREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(OREG));
    const int g = (tid - S0) >> 5;
    if (g < ngrp) {
      const int slot = 32 * g + (tid & 31);
      const bool act = slot < 4 * nkc;
      for (int y = y0; y < yend; ++y) {
        const int b = (y - y0) & 1;
        if (COLS == 2 && BF_HALFSCAN) {   // the row in two pieces, as the V threads' columns complete
          int* Q = Ubuf + b * srow + slot * UP;
          const int h = min(W2_V, wv);
          int carry = 0;
          bar_sync(BAR_U_FULL + 2 * b + 1, n_ufull);
          if (act && !BF_X_NOS) carry = prefix_part(Q, 0, h, 0);
          bar_sync(BAR_U_FULL + 2 * b, n_ufull);
          if (act && !BF_X_NOS) Q[wv] = prefix_part(Q, h, wv, carry);
        } else {
          bar_sync(BAR_U_FULL + 2 * b + g, n_ufull);
          if (act && !BF_X_NOS) prefix_row(Ubuf + b * srow + slot * UP, wv);
        }
        bar_arrive(BAR_Q_FULL + 2 * b + g, n_qfull);
      }
    }
  } else {
    // ------------------------------------------------------------ FH role
    if constexpr (FHREG > LREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(FHREG));
    else if constexpr (FHREG < LREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(FHREG));
    const int o = tid - H0;
    const bool act = o < TWv;
    const bool wact = (o & ~31) < TWv;             // warp has pixels of the strip
    const int oc = act ? o : 0;
    // Q offsets (extended index o + rlo) of the x boxes: F = round(sum_b (Q[e_b] - Q[l_b]) ax_b / 2^32)
    const bool two = (M == 2) && P.nbx[0] == 2;
    const int e0 = oc + P.rlo_x + P.hhi[0][0] + 1, l0 = oc + P.rlo_x + P.hlo[0][0];
    const int e1 = two ? oc + P.rlo_x + P.hhi[0][1] + 1 : e0, l1 = two ? oc + P.rlo_x + P.hlo[0][1] : l0;
    const int ax0 = P.ax[0][0], ax1 = two ? P.ax[0][1] : 0;
    const long long prow = fbase + x0 + oc;
    const int k0 = P.kval[t0];
    // cluster reduction addresses (CL)
    unsigned full_l = 0, red_l = 0;
    if constexpr (CL) {
      full_l = smem_u32(&mbar[0]);
      red_l = smem_u32(red);
    }
    float Inext = act ? load_pixel(in, U8, prow + (long long)y0 * P.W) : 0.f;
    for (int y = y0; y < yend; ++y) {
      const int b = (y - y0) & 1;
      const float Ic = Inext;
      if (act && y + 1 < yend) Inext = load_pixel(in, U8, prow + (long long)(y + 1) * P.W);
      // PB: per-box exact accumulators num_b = sum W H_b, den_b (no F rounding); num = sum_b ax_b num_b
      long long num[PB ? 2 : NPL] = {}, den[PB ? 2 : NPL] = {};
      int hm0 = 0, hm1 = 0;   // box sums H_b of the k = 0 cosine channel (the clipped spatial mass, on demand)
      if (wact && !BF_X_NOFH) {
        double c1, s1;
        pixel_angle<U8>(P, lut64, Ic, c1, s1);
        Cheb64 gk;
        gk.init(c1, s1);
#pragma unroll 4
        for (int j = 0; j < k0; ++j) gk.step();
        const int* Qb = Ubuf + b * srow;
#pragma unroll
        for (int i = 0; i < MAXK; ++i) {
          if (FULL || i < nkc) {
            if ((i & 7) == 0) bar_sync(BAR_Q_FULL + 2 * b + (i >> 3), n_qfull);
            if (!DUMP && i > 0 && !BF_X_NOW) {   // k_i - k_{i-1} >= 1 steps
              if (CONSEC) gk.step();
              else {
                int n = P.kstep[t0 + i];
#pragma unroll 1
                do gk.step();
                while (--n > 0);
              }
            }
            int h0[4], h1[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int* q = Qb + (4 * i + c) * UP;
              if (BF_X_NOLDS) {
                h0[c] = e0 * (c + 3) + i;
                h1[c] = l1 * (c + 1) - i;
              } else {
                h0[c] = q[e0] - q[l0];
                h1[c] = (M == 2) ? q[e1] - q[l1] : 0;
              }
            }
            if (i == 0 && k0 == 0) {
              hm0 = h0[0];
              hm1 = h1[0];
            }
            if constexpr (DUMP) {
              if (act) {
                // cache plane k: the pixel's four channels as one 16-byte entry
                int4* cp = reinterpret_cast<int4*>(P.cache) + (long long)P.kval[t0 + i] * P.cache_plane +
                           (long long)y * P.W + x0 + o;
                int F[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  long long f = mad_wide(h0[c], ax0, FRND);
                  if (M == 2) f = mad_wide(h1[c], ax1, f);
                  F[c] = fhi(f);
                }
                __stcs(cp, make_int4(F[0], F[1], F[2], F[3]));
              }
            } else if constexpr (PB) {
              const int wc = BF_X_NOW ? 1000 + i * e1 : __double2loint(fma(gk.c, P.aw[0][t0 + i], MAGIC64));
              const int wsn = BF_X_NOW ? 77 + i * l0 : __double2loint(fma(gk.s, P.aw[0][t0 + i], MAGIC64));
              den[0] = mad_wide(wc, h0[0], den[0]);
              den[0] = mad_wide(wsn, h0[1], den[0]);
              num[0] = mad_wide(wc, h0[2], num[0]);
              num[0] = mad_wide(wsn, h0[3], num[0]);
              if (M == 2) {
                den[1] = mad_wide(wc, h1[0], den[1]);
                den[1] = mad_wide(wsn, h1[1], den[1]);
                num[1] = mad_wide(wc, h1[2], num[1]);
                num[1] = mad_wide(wsn, h1[3], num[1]);
              }
            } else {
              int F[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                long long f = mad_wide(h0[c], ax0, FRND);
                if (M == 2) f = mad_wide(h1[c], ax1, f);
                F[c] = fhi(f);
              }
#pragma unroll
              for (int q = 0; q < NPL; ++q) {   // Case 1 (bf_apply_multi): every plan over the same F
                const int wc = __double2loint(fma(gk.c, P.aw[q][t0 + i], MAGIC64));
                const int wsn = __double2loint(fma(gk.s, P.aw[q][t0 + i], MAGIC64));
                den[q] = mad_wide(wc, F[0], den[q]);
                den[q] = mad_wide(wsn, F[1], den[q]);
                num[q] = mad_wide(wc, F[2], num[q]);
                num[q] = mad_wide(wsn, F[3], num[q]);
              }
            }
            if ((i & 7) == 7 || (FULL ? i + 1 == MAXK : i + 1 == nkc))
              bar_arrive(BAR_U_EMPTY + 2 * b + (i >> 3), n_uempty);
          }
        }
      } else {   // warp wholly past the strip: only the barriers
        for (int g = 0; g < ngrp; ++g) {
          bar_sync(BAR_Q_FULL + 2 * b + g, n_qfull);
          bar_arrive(BAR_U_EMPTY + 2 * b + g, n_uempty);
        }
      }
      if constexpr (DUMP) continue;
      if constexpr (CL) {
        const int xb = (y - y0) % XS;                        // exchange slot of this row
        const unsigned ph = (unsigned)((y - y0) / XS) & 1;
        if (rank > 0) {
          // sender: wait until CTA 0 has consumed row y - XS from the slot, then store the partials
          if (wact) {
            if (y - y0 >= XS) mbar_wait(smem_u32(&mbar[XS + xb]), ph ^ 1);
            if (act) {
              const unsigned dst = map_rank(red_l + (unsigned)((xb * P.TW + o) * 32), 0);
              const unsigned fb = map_rank(full_l + 8 * xb, 0);
              red_async_add(dst, num[0], fb);
              red_async_add(dst + 8, den[0], fb);
              red_async_add(dst + 16, num[1], fb);
              red_async_add(dst + 24, den[1], fb);
            }
          }
        } else {
          if (o == 0) mbar_expect(full_l + 8 * xb, (unsigned)((G - 1) * TWv * 32));
          if (wact) {
            mbar_wait(full_l + 8 * xb, ph);
            if (act) {
              // the senders' partials, added exactly in CTA 0's slot (integer adds: any order)
              longlong2* r2 = red + 2 * (xb * P.TW + o);
              const longlong2 v0 = r2[0], v1 = r2[1];
              r2[0] = make_longlong2(0, 0);   // cleared for row y + XS (ordered before the release below)
              r2[1] = make_longlong2(0, 0);
              num[0] += v0.x;
              den[0] += v0.y;
              num[1] += v1.x;
              den[1] += v1.y;
              finish_pixel_pb(P, num, den, ax0, ax1, Ic, prow + (long long)y * P.W, out, hm0, hm1, ws);
            }
          }
          __syncwarp();
          if ((tid & 31) == 0)
            for (int s = 1; s < G; ++s) mbar_arrive_remote(map_rank(smem_u32(&mbar[XS + xb]), s));
        }
      } else if constexpr (PB) {
        if (act) finish_pixel_pb(P, num, den, ax0, ax1, Ic, prow + (long long)y * P.W, out, hm0, hm1, ws);
      } else {
        if (act) {
#pragma unroll
          for (int q = 0; q < NPL; ++q)
            finish_pixel(P, num[q], den[q], Ic, prow + (long long)y * P.W + q * P.plan_stride, out, ws, q == 0,
                         fhi(mad_wide(hm1, ax1, mad_wide(hm0, ax0, FRND))));
        }
      }
    }
  }
  if constexpr (CL) {
    // no CTA may leave while its shared memory can still be the target of a remote operation
    __syncwarp();
    cluster_sync();
  }
}

template <int MAXK, int FORM, bool U8, bool CONSEC, bool FULL, int NPL, int COLS, bool CL, bool DUMP>
cudaError_t go(const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid, size_t smem, cudaStream_t st) {
  auto kfn = bf_ws2_kernel<MAXK, FORM, U8, CONSEC, FULL, NPL, COLS, CL, DUMP>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if constexpr (CL) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(W2_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P.G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kfn, P, in, out, ws);
    if (e != cudaSuccess) return e;
  } else {
    kfn<<<grid, W2_THREADS, smem, st>>>(P, in, out, ws);
  }
  return cudaGetLastError();
}

}  // namespace ws2
}  // namespace bf
