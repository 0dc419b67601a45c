// Kernel 2b launcher: one range plan, one CTA per strip x band (the cfg0-cfg3 path).
#include "bf_ws2.cuh"

namespace bf {
namespace {

template <int MAXK, int FORM, bool U8>
cudaError_t by_flags(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                     size_t smem, cudaStream_t st) {
  if (s.CONSEC && s.FULL) return ws2::go<MAXK, FORM, U8, true, true, 1, 1, false, false>(P, in, out, ws, grid, smem, st);
  if (s.CONSEC) return ws2::go<MAXK, FORM, U8, true, false, 1, 1, false, false>(P, in, out, ws, grid, smem, st);
  return ws2::go<MAXK, FORM, U8, false, false, 1, 1, false, false>(P, in, out, ws, grid, smem, st);
}

template <bool U8>
cudaError_t by_shape(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                     size_t smem, cudaStream_t st) {
  if (s.NPL != 1 || s.COLS != 1 || s.CL || s.DUMP) return cudaErrorInvalidConfiguration;
  if (s.MAXK == 8 && s.FORM == 1) return by_flags<8, 1, U8>(s, P, in, out, ws, grid, smem, st);
  if (s.MAXK == 8 && s.FORM == 2) return by_flags<8, 2, U8>(s, P, in, out, ws, grid, smem, st);
  if (s.MAXK == 16 && s.FORM == 1) return by_flags<16, 1, U8>(s, P, in, out, ws, grid, smem, st);
  if (s.MAXK == 16 && s.FORM == 2) return by_flags<16, 2, U8>(s, P, in, out, ws, grid, smem, st);
  return cudaErrorInvalidConfiguration;
}

}  // namespace

cudaError_t launch_ws2(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                       size_t smem, cudaStream_t st) {
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  return s.U8 ? by_shape<true>(s, P, in, out, ws, grid, smem, st) : by_shape<false>(s, P, in, out, ws, grid, smem, st);
}

}  // namespace bf
