// Launch parameters shared by the host dispatch (bf_apply.cu) and the kernel translation units.
// Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include "bf_internal.h"

namespace bf {

constexpr int MAXB = 4;              // boxes per axis
constexpr int MAXP = BF_MAX_PLANS;   // range plans of one bf_apply_multi

// Ill-conditioned pixels (reading Q27). out = num / den amplifies the fused kernels'
// integer-format rounding (relative ~1e-8 of the full-window denominator, tools/numerics_pixel.py)
// by 1 / cond, cond = den / sum K~_s (the clipped spatial mass). A pixel with cond < tau (or
// den <= 0, whose fallback decision rides on that rounding) is appended to a device list and
// re-evaluated by bf_repair_kernel in fp64 straight from the approximated kernels (the direct
// double loop of pin P1, equal to the box evaluation up to rounding).
// Per flagged pixel: the repair pass's fixed-point accumulators (zeroed by the flagging kernel)
struct RepAcc {
  long long num, den;   // sum of the chunks' partial sums, each rounded to fixed point (exact adds)
  unsigned arrived;     // chunks done
  unsigned pad;
};

struct RepairSink {
  unsigned* count;            // list length (atomic), NULL = repair off
  unsigned long long* list;   // output indices (frame and plan offsets included)
  RepAcc* acc;                // per list entry
  unsigned cap;
  double tau_w;               // tau * 2^wbits: flag if den < tau_w * mass (mass = the k = 0 cosine channel F)
  double mass_full;           // that channel's value for an unclipped window (used when k = 0 is not selected)
  double mass_bound;          // >= the channel's value for any clipped window (kernel 2b tests den against it
                              // first and forms the clipped mass only below it)
};

// Parameters of one launch of a T = D kernel (band / ws / ws2 / cache), passed by value.
struct KParams {
  int H, W;
  long long frame_elems;
  int TW, TH, rlo_x;
  int yb, ye;                 // output rows [yb, ye) of this launch (row chunks of bf_apply_host / bf_apply_ex)
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
                              // F = round(sum_tb H_tb ax_tb / 2^32) (exact int64 products)
  int nk;                     // terms of this launch (all CTAs of a cluster together)
  int kval[BF_MAX_TERMS];     // their frequencies k (ascending)
  int kstep[BF_MAX_TERMS];    // kval[i] - kval[i-1] (i > 0)
  double aw[MAXP][BF_MAX_TERMS];   // a_k * 2^wbits of each range plan (bf_apply_multi; one plan otherwise)
  int nplans;                 // range plans sharing the box-filtered channels (Case 1)
  long long plan_stride;      // output elements between consecutive plans' images
  float invD_hi, invD_lo;     // 1/D as a float-float pair
  double invD, D;
  int pass;                   // 0 = only pass; 1 = first; 2 = middle; 3 = last (workspace passes)
  int ngrp, nseg, seglen;     // 32-channel groups (per CTA); walker row segments
  int wpar;                   // paired-load walker: parity of box 1's leave stream (0 / 1), -1 = scalar walker
  int wv;                     // kernel 2b: extended columns written and scanned (TW + halo rounded up to 8)
  int f_off, l_off, r_off;    // shared-memory carve-up: U' rows, F rows, LUTs, cluster reduction rows
  unsigned char wmap[24];     // kernel 2b: physical warp -> logical warp (role and index; balanced over the SM sub-partitions)
  unsigned char tmblk[24];    // kernel 2b: physical V warp -> its block of TMEM columns within its lane quarter
  int tmcols;                 // kernel 2b: TMEM columns allocated (power of two >= 32)
  unsigned char vq[4][6];     // kernel 2b: the working V warps (index in the V role) of lane quarter q, in TMEM block order
  unsigned char nvq[4];       // kernel 2b: how many
  int G, tpc;                 // kernel 2b cluster split: G CTAs per cluster, CTA c owns terms [c tpc, c tpc + tpc)
  unsigned long long* fb_count;    // optional: += pixels that took the den <= 0 fallback (Q18)
  unsigned char* fb_mask;          // optional: 1 where the pixel took the fallback, else 0
  int* cache;                 // bf_precompute: box-filtered channel planes F[ch][y][x] (int32)
  long long cache_plane;      // int4 entries per cache plane (H * W)
  RepairSink rep;             // ill-conditioned pixels for the fp64 repair pass
  double uscale;              // absolute value of one unit of F (times 2^wbits): wxmax wymax 2^-(abits-32+q-ush)
  double dunit;               // general plans: uscale * 2^-wbits, num / den accumulated in fp64 (0 = off)
};

// Template choices of one launch (the kernel TUs switch on these).
struct LaunchSpec {
  int kern;      // KERN_BAND, KERN_WS, KERN_WS2
  int NT;        // band kernel threads (256 / 512); ws / ws2: 256 class
  int MAXK;      // terms per CTA (8 / 16)
  int FORM;      // 1, 2, 4 separable; 5 rank 2
  bool U8, CONSEC, FULL;
  int NPL;       // range plans combined per pixel (1..4)
  int COLS;      // ws2: extended columns per V thread (1 / 2)
  bool CL;       // ws2: terms split over a CTA cluster (G = P.G CTAs)
  bool DUMP;     // ws2: write the box-filtered channels to P.cache instead of combining (bf_precompute)
  bool DIRECT;   // band, u8: direct trig evaluation instead of the Case 2 LUT (bf_apply_args.u8_trig)
};

constexpr int KERN_BAND = 0, KERN_WS = 1, KERN_WS2 = 2;

// kernel 2b cluster split: row slots of the DSMEM exchange (the senders may run this many rows
// ahead of CTA 0's consumption)
#ifndef BF_XSLOTS
#define BF_XSLOTS 2
#endif
constexpr int W2_XSLOTS = BF_XSLOTS;

// kernel 2 (bf_ws_kernel) role sizes
constexpr int WS_V = 256, WS_S = 64, WS_F = 192, WS_C = 128, WS_THREADS = WS_V + WS_S + WS_F + WS_C;
constexpr int WS_H = WS_S + WS_F;
// kernel 2b (bf_ws2_kernel): V threads (extended columns / COLS), S threads, FH threads (outputs)
constexpr int W2_V = 384, W2_THREADS = 768;
constexpr int w2_nfh(int cols) { return cols == 1 ? 320 : 352; }
constexpr int w2_ns(int cols) { return cols == 1 ? 64 : 32; }
constexpr int w2_up(int cols) { return W2_V * cols + 4; }   // == 4 mod 32: conflict-free 16-byte accesses

// Launchers (one per kernel translation unit). Return cudaErrorInvalidConfiguration for a spec
// the TU has no instantiation for.
cudaError_t launch_band(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                        size_t smem, cudaStream_t st);
cudaError_t launch_ws(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                      size_t smem, cudaStream_t st);
cudaError_t launch_ws2(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                       size_t smem, cudaStream_t st);
cudaError_t launch_ws2_multi_u8(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws,
                                dim3 grid, size_t smem, cudaStream_t st);
cudaError_t launch_ws2_multi_f32(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws,
                                 dim3 grid, size_t smem, cudaStream_t st);
cudaError_t launch_ws2_cluster(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws,
                               dim3 grid, size_t smem, cudaStream_t st);
int ws2_max_clusters(const LaunchSpec& s, size_t smem, int G);

// The literal-window kernel (NEXT f1).
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
  unsigned long long* fb_count;
  unsigned char* fb_mask;
  int klut[512];      // K_lit(t) * 2^30, t = -255..255 (by value: no device table, graph capturable)
};
cudaError_t launch_literal(const LParams& L, const unsigned char* in, float* out, dim3 grid, size_t smem,
                           cudaStream_t st);

// Case 1 cache (NEXT f2): combine-only pass over precomputed box-filtered channels.
struct CParams {
  int H, W;
  long long plane;            // int4 entries per cache plane (H * W)
  int nk;                     // terms combined
  int ch[BF_MAX_TERMS];       // cache plane of term i (its k)
  int kval[BF_MAX_TERMS];
  int kstep[BF_MAX_TERMS + 8];   // k_i - k_{i-1} (i >= 1); 0 in the padding
  double aw[BF_MAX_TERMS + 8];   // a_k * 2^wbits; 0 in the padding (the kernel runs whole chunks)
  int mass_i;                 // index of the k = 0 term, or -1
  double invD, D;
  int u8;
  unsigned long long* fb_count;
  unsigned char* fb_mask;
  RepairSink rep;
};
cudaError_t launch_cached(const CParams& C, const int4* cache, const void* in, float* out, cudaStream_t st);

// fp64 repair of the flagged pixels (bf_k_repair.cu).
constexpr int REP_DEG = 13, REP_TAB = 2048;
struct RParams {
  int H, W;
  long long frame_elems, plan_stride;
  int nplans, nk;
  int k[MAXP][BF_MAX_TERMS];
  double a[MAXP][BF_MAX_TERMS];
  int nkp[MAXP];
  int kmax;
  double D, T;                // cosine period half-width T (= D on the hot path)
  int u8;
  int ns;                     // spatial box-pair terms K~_s(u, v) = sum_s fx_s(u) fy_s(v)
  int nbx[BF_MAX_SP_PASSES], nby[BF_MAX_SP_PASSES];
  int lox[BF_MAX_SP_PASSES][MAXB], hix[BF_MAX_SP_PASSES][MAXB], loy[BF_MAX_SP_PASSES][MAXB], hiy[BF_MAX_SP_PASSES][MAXB];
  double wx[BF_MAX_SP_PASSES][MAXB], wy[BF_MAX_SP_PASSES][MAXB];
  int rad;                    // window half-width (max box extent)
  int nch, rpc;               // chunks per pixel, window rows per chunk
  // f32, one plan: K~_r(t) for t = |I(x) - I(y)| in [0, D] as piecewise Taylor polynomials of
  // degree REP_DEG on ntab intervals of width 2 tab_h (truncation < 1e-15 of sum |a_k|), else the
  // Chebyshev recurrence per tap (ntab = 0)
  int ntab;
  double tab_h;
  double tab[REP_TAB];
  double qscale;              // fixed-point scale of the partial sums: |den partial| * qscale < 2^61
  unsigned* count;
  const unsigned long long* list;
  RepAcc* acc;
  unsigned cap;
  unsigned long long* fb_count;
  unsigned char* fb_mask;
  unsigned long long* repaired;   // optional: += pixels re-evaluated
};
constexpr unsigned REPAIR_SLOTS = 16, REPAIR_CAP = 1u << 15;
// device addresses of repair slot s's counter, list and accumulators (static device storage)
cudaError_t repair_slot(unsigned s, unsigned** count, unsigned long long** list, RepAcc** acc);
cudaError_t launch_repair(const RParams& R, const void* in, float* out, cudaStream_t st);

}  // namespace bf
