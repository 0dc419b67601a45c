// Kernel 2: warp-specialised with an F row buffer (bf_ws_kernel). Runs the rank-2 box-pair plans
// (N_s = 5, NEXT f3), whose two vertical states need more registers than kernel 2b's V role.
#include "bf_walk.cuh"

namespace bf {
namespace {

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
    v_init<MAXK, NB, NS, U8, CONSEC, FULL>(P, in, lut, fbase, col, colok, y0, 0, P.nk, U);
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
      v_row<MAXK, NB, NS, U8, CONSEC, FULL, UP>(P, lut, colok, y, 0, P.nk, Icur, U, Ubuf + b * ustride + tid, &hook);
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

template <int MAXK, int FORM, bool U8, bool CONSEC, bool FULL>
cudaError_t go(const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid, size_t smem, cudaStream_t st) {
  auto kfn = bf_ws_kernel<MAXK, FORM, U8, CONSEC, FULL, false>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kfn<<<grid, WS_THREADS, smem, st>>>(P, in, out, ws);
  return cudaGetLastError();
}

template <int MAXK, int FORM, bool U8>
cudaError_t by_flags(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                     size_t smem, cudaStream_t st) {
  if (s.CONSEC && s.FULL) return go<MAXK, FORM, U8, true, true>(P, in, out, ws, grid, smem, st);
  if (s.CONSEC) return go<MAXK, FORM, U8, true, false>(P, in, out, ws, grid, smem, st);
  return go<MAXK, FORM, U8, false, false>(P, in, out, ws, grid, smem, st);
}

template <bool U8>
cudaError_t by_shape(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                     size_t smem, cudaStream_t st) {
  if (s.NPL != 1) return cudaErrorInvalidConfiguration;
  if (s.MAXK == 8) {
    switch (s.FORM) {
      case 1: return by_flags<8, 1, U8>(s, P, in, out, ws, grid, smem, st);
      case 2: return by_flags<8, 2, U8>(s, P, in, out, ws, grid, smem, st);
      case 5: return by_flags<8, 5, U8>(s, P, in, out, ws, grid, smem, st);
    }
  }
  if (s.MAXK == 16) {
    switch (s.FORM) {
      case 1: return by_flags<16, 1, U8>(s, P, in, out, ws, grid, smem, st);
      case 2: return by_flags<16, 2, U8>(s, P, in, out, ws, grid, smem, st);
    }
  }
  return cudaErrorInvalidConfiguration;
}

}  // namespace

cudaError_t launch_ws(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                      size_t smem, cudaStream_t st) {
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  return s.U8 ? by_shape<true>(s, P, in, out, ws, grid, smem, st) : by_shape<false>(s, P, in, out, ws, grid, smem, st);
}

}  // namespace bf
