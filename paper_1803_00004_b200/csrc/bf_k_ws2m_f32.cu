// Kernel 2b launcher, Case 1 multi-plan combine (bf_apply_multi): NPL = 2..4 range plans over one
// pass of shared box-filtered channels, each plan count its own instantiation (no spills).
// f32 input.
#include "bf_ws2.cuh"

namespace bf {
namespace {

template <int MAXK, int FORM, int NPL>
cudaError_t by_consec(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                      size_t smem, cudaStream_t st) {
  if (s.CONSEC) return ws2::go<MAXK, FORM, false, true, false, NPL, 1, false, false>(P, in, out, ws, grid, smem, st);
  return ws2::go<MAXK, FORM, false, false, false, NPL, 1, false, false>(P, in, out, ws, grid, smem, st);
}

template <int MAXK, int FORM>
cudaError_t by_npl(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                   size_t smem, cudaStream_t st) {
  switch (s.NPL) {
    case 2: return by_consec<MAXK, FORM, 2>(s, P, in, out, ws, grid, smem, st);
    case 3: return by_consec<MAXK, FORM, 3>(s, P, in, out, ws, grid, smem, st);
    case 4: return by_consec<MAXK, FORM, 4>(s, P, in, out, ws, grid, smem, st);
  }
  return cudaErrorInvalidConfiguration;
}

}  // namespace

cudaError_t launch_ws2_multi_f32(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws,
                                  dim3 grid, size_t smem, cudaStream_t st) {
  if (smem > 227 * 1024 || s.COLS != 1 || s.CL || s.DUMP || s.NPL < 2) return cudaErrorInvalidConfiguration;
  if (s.MAXK == 8 && s.FORM == 1) return by_npl<8, 1>(s, P, in, out, ws, grid, smem, st);
  if (s.MAXK == 8 && s.FORM == 2) return by_npl<8, 2>(s, P, in, out, ws, grid, smem, st);
  if (s.MAXK == 16 && s.FORM == 1) return by_npl<16, 1>(s, P, in, out, ws, grid, smem, st);
  if (s.MAXK == 16 && s.FORM == 2) return by_npl<16, 2>(s, P, in, out, ws, grid, smem, st);
  return cudaErrorInvalidConfiguration;
}

}  // namespace bf
