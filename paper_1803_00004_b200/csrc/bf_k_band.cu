// Kernel 1: barrier intervals (bf_band_kernel). One thread per extended column; per row interval
// A = V(y) + C(y-1), interval B = H(y) by walker warps. Used for wide halos with up to four boxes
// per axis (NT = 512), the multi-plan combine of plans kernel 2b cannot take, and as the
// reference structure the warp-specialised kernels are tested against (bitwise).
#include "bf_walk.cuh"

namespace bf {
namespace {

template <int MAXK, int NT>
struct Occ {
  static constexpr int value = NT > 256 ? 1 : 2;
};

// FULL: nk == MAXK (no per-term runtime checks). CONSEC: the selected k are consecutive.
// DIRECT (u8, bf_apply_args.u8_trig): the channels' base angles by direct evaluation instead of the
// Case 2 LUT - the same values, so the output is bitwise that of the LUT path
template <int MAXK, int FORM, bool U8, int NT, bool CONSEC, bool FULL, bool MULTI, bool DIRECT = false>
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
  v_init<MAXK, NB, NS, U8, CONSEC, FULL, false, DIRECT>(P, in, lut, fbase, col, colok, y0, 0, P.nk, U);
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
      v_row<MAXK, NB, NS, U8, CONSEC, FULL, UP, GroupSync, false, DIRECT>(P, lut, colok, y, 0, P.nk, Icur, U,
                                                                          Ubuf + tid);
    }
    if (y > y0 && tid < TWv)
      combine_pixel<MAXK, U8, CONSEC, FULL, MULTI, DIRECT>(P, lut64, reinterpret_cast<const int4*>(Fbuf + tid * FPX),
                                                           Ic, fbase + (long long)(y - 1) * P.W + x0 + tid, out, ws);
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

template <int MAXK, int FORM, bool U8, int NT, bool CONSEC, bool FULL, bool MULTI, bool DIRECT = false>
cudaError_t go(const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid, size_t smem, cudaStream_t st) {
  auto kfn = bf_band_kernel<MAXK, FORM, U8, NT, CONSEC, FULL, MULTI, DIRECT>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kfn<<<grid, NT, smem, st>>>(P, in, out, ws);
  return cudaGetLastError();
}

template <int MAXK, int FORM, bool U8, int NT>
cudaError_t by_flags(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                     size_t smem, cudaStream_t st) {
  if constexpr (U8 && NT == 256 && (FORM == 1 || FORM == 2)) {
    if (s.DIRECT) {
      if (s.NPL > 1) return cudaErrorInvalidConfiguration;
      if (s.CONSEC && s.FULL) return go<MAXK, FORM, U8, NT, true, true, false, true>(P, in, out, ws, grid, smem, st);
      if (s.CONSEC) return go<MAXK, FORM, U8, NT, true, false, false, true>(P, in, out, ws, grid, smem, st);
      return go<MAXK, FORM, U8, NT, false, false, false, true>(P, in, out, ws, grid, smem, st);
    }
  }
  if (s.DIRECT) return cudaErrorInvalidConfiguration;
  if (s.NPL > 1) {
    if constexpr (FORM == 1 || FORM == 2) {
      return s.CONSEC ? go<MAXK, FORM, U8, NT, true, false, true>(P, in, out, ws, grid, smem, st)
                      : go<MAXK, FORM, U8, NT, false, false, true>(P, in, out, ws, grid, smem, st);
    }
    return cudaErrorInvalidConfiguration;
  }
  if constexpr (FORM == 4) {   // (rare wide plans: the generic instantiation only)
    return go<MAXK, FORM, U8, NT, false, false, false>(P, in, out, ws, grid, smem, st);
  } else {
    if (s.CONSEC && s.FULL) return go<MAXK, FORM, U8, NT, true, true, false>(P, in, out, ws, grid, smem, st);
    if (s.CONSEC) return go<MAXK, FORM, U8, NT, true, false, false>(P, in, out, ws, grid, smem, st);
    return go<MAXK, FORM, U8, NT, false, false, false>(P, in, out, ws, grid, smem, st);
  }
}

template <bool U8>
cudaError_t by_shape(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                     size_t smem, cudaStream_t st) {
  if (s.NT == 256 && s.MAXK == 8) {
    switch (s.FORM) {
      case 1: return by_flags<8, 1, U8, 256>(s, P, in, out, ws, grid, smem, st);
      case 2: return by_flags<8, 2, U8, 256>(s, P, in, out, ws, grid, smem, st);
      case 4: return by_flags<8, 4, U8, 256>(s, P, in, out, ws, grid, smem, st);
      case 5: return by_flags<8, 5, U8, 256>(s, P, in, out, ws, grid, smem, st);
    }
  }
  if (s.NT == 256 && s.MAXK == 16) {
    switch (s.FORM) {
      case 1: return by_flags<16, 1, U8, 256>(s, P, in, out, ws, grid, smem, st);
      case 2: return by_flags<16, 2, U8, 256>(s, P, in, out, ws, grid, smem, st);
      case 4: return by_flags<16, 4, U8, 256>(s, P, in, out, ws, grid, smem, st);
    }
  }
  if (s.NT == 512 && s.MAXK == 8) {
    switch (s.FORM) {
      case 1: return by_flags<8, 1, U8, 512>(s, P, in, out, ws, grid, smem, st);
      case 2: return by_flags<8, 2, U8, 512>(s, P, in, out, ws, grid, smem, st);
      case 4: return by_flags<8, 4, U8, 512>(s, P, in, out, ws, grid, smem, st);
    }
  }
  if (s.NT == 512 && s.MAXK == 16 && s.FORM == 2) return by_flags<16, 2, U8, 512>(s, P, in, out, ws, grid, smem, st);
  return cudaErrorInvalidConfiguration;
}

}  // namespace

cudaError_t launch_band(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                        size_t smem, cudaStream_t st) {
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  return s.U8 ? by_shape<true>(s, P, in, out, ws, grid, smem, st) : by_shape<false>(s, P, in, out, ws, grid, smem, st);
}

}  // namespace bf
