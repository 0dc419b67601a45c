// Kernel 2b launchers: the range terms split over a CTA cluster (CL, DSMEM reduction of num /
// den), two columns per V thread for wide radii (COLS = 2), and the channel dump of
// bf_precompute (Case 1 cache).
#include "bf_ws2.cuh"

namespace bf {
namespace {

template <int MAXK, int FORM, bool U8, int COLS, bool CL>
cudaError_t by_flags(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                     size_t smem, cudaStream_t st) {
  if (s.CONSEC && s.FULL) return ws2::go<MAXK, FORM, U8, true, true, 1, COLS, CL, false>(P, in, out, ws, grid, smem, st);
  if (s.CONSEC) return ws2::go<MAXK, FORM, U8, true, false, 1, COLS, CL, false>(P, in, out, ws, grid, smem, st);
  // non-consecutive k with every CTA's term count known at compile time (cfg4: 24 Tukey terms = 3 x 8)
  if constexpr (COLS == 2 && CL)
    if (s.FULL) return ws2::go<MAXK, FORM, U8, false, true, 1, COLS, CL, false>(P, in, out, ws, grid, smem, st);
  return ws2::go<MAXK, FORM, U8, false, false, 1, COLS, CL, false>(P, in, out, ws, grid, smem, st);
}

template <int FORM, bool U8>
cudaError_t by_kind(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws, dim3 grid,
                    size_t smem, cudaStream_t st) {
  if (s.DUMP) {   // consecutive k, 16 per launch
    if (s.COLS != 1 || s.CL || s.MAXK != 16 || !s.CONSEC) return cudaErrorInvalidConfiguration;
    return s.FULL ? ws2::go<16, FORM, U8, true, true, 1, 1, false, true>(P, in, out, ws, grid, smem, st)
                  : ws2::go<16, FORM, U8, true, false, 1, 1, false, true>(P, in, out, ws, grid, smem, st);
  }
  if (s.COLS == 1 && s.CL && s.MAXK == 16) return by_flags<16, FORM, U8, 1, true>(s, P, in, out, ws, grid, smem, st);
  if (s.COLS == 2 && s.CL && s.MAXK == 8) return by_flags<8, FORM, U8, 2, true>(s, P, in, out, ws, grid, smem, st);
  if (s.COLS == 2 && !s.CL && s.MAXK == 8) return by_flags<8, FORM, U8, 2, false>(s, P, in, out, ws, grid, smem, st);
  return cudaErrorInvalidConfiguration;
}

}  // namespace

cudaError_t launch_ws2_cluster(const LaunchSpec& s, const KParams& P, const void* in, float* out, longlong2* ws,
                               dim3 grid, size_t smem, cudaStream_t st) {
  if (smem > 227 * 1024 || s.NPL != 1) return cudaErrorInvalidConfiguration;
  if (s.FORM == 1) return s.U8 ? by_kind<1, true>(s, P, in, out, ws, grid, smem, st)
                               : by_kind<1, false>(s, P, in, out, ws, grid, smem, st);
  if (s.FORM == 2) return s.U8 ? by_kind<2, true>(s, P, in, out, ws, grid, smem, st)
                               : by_kind<2, false>(s, P, in, out, ws, grid, smem, st);
  return cudaErrorInvalidConfiguration;
}

// Clusters of G kernel-2b CTAs that can be resident at once (cudaOccupancyMaxActiveClusters),
// or 0 when it cannot be asked (no device: dry runs on a host without a GPU).
int ws2_max_clusters(const LaunchSpec& s, size_t smem, int G) {
  if (G <= 1 || s.COLS < 1) return 0;
  const void* fn = nullptr;
  if (s.COLS == 1 && s.FORM == 2) fn = s.U8 ? (const void*)ws2::bf_ws2_kernel<16, 2, true, true, true, 1, 1, true, false>
                                            : (const void*)ws2::bf_ws2_kernel<16, 2, false, true, true, 1, 1, true, false>;
  else if (s.COLS == 2 && s.FORM == 2)
    fn = s.U8 ? (const void*)ws2::bf_ws2_kernel<8, 2, true, true, true, 1, 2, true, false>
              : (const void*)ws2::bf_ws2_kernel<8, 2, false, true, true, 1, 2, true, false>;
  else if (s.COLS == 1) fn = s.U8 ? (const void*)ws2::bf_ws2_kernel<16, 1, true, true, true, 1, 1, true, false>
                                  : (const void*)ws2::bf_ws2_kernel<16, 1, false, true, true, 1, 1, true, false>;
  else fn = s.U8 ? (const void*)ws2::bf_ws2_kernel<8, 1, true, true, true, 1, 2, true, false>
                 : (const void*)ws2::bf_ws2_kernel<8, 1, false, true, true, 1, 2, true, false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(W2_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace bf
