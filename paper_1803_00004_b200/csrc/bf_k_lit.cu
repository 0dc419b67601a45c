// Kernel 3: the paper-literal z-window (bf_literal_kernel, NEXT f1), u8 levels.
#include "bf_device.cuh"

namespace bf {
namespace {

// ------------------------------------------------------------------ kernel 3: the literal window
// NEXT f1: the paper's dimension-promoted 3-D box filter with the window [I(x) - T_r, I(x) + T_r]
// (eq:1D_box_N_terms, eq:numerator_2D_box_N_terms) on u8 images. The auxiliary
// images F_c(y, z) = G^c_k(y) delta_{I(y)}(z) depend on y only through the level z = I(y), so
// their 3-D box sums factor into the spatially weighted level counts
//     C_z(x) = sum_y K~_s(x - y) [I(y) = z]
// and the numerator / denominator become
//     num(x) = sum_{|z - I(x)| <= T_r} C_z(x) z K_lit(I(x) - z),  den likewise without z,
// with K_lit(t) = sum_k a_k cos(pi k t / T_r) (eq:trigonometric_N_terms): the shiftable split of
// P:460-468 recombined per level (an exact identity, pinned by the oracle's bf_promoted).
// One CTA = a strip of LIT_NT extended columns x a band of rows; each thread keeps its column's
// level counts for the two vertical boxes packed in one int32 (lo / hi 16 bits) in shared memory,
// sliding them down one row per step (4 taps); the output threads then sum, for every level of
// their window, the counts over the horizontal boxes and accumulate the integer products with
// K_lit quantised to 2^30 exactly in int64; the box weights are applied once per pixel in fp64.
__global__ void __launch_bounds__(LIT_NT, 1)
    bf_literal_kernel(const LParams P, const unsigned char* __restrict__ in, float* __restrict__ out) {
  constexpr int NTP = LIT_NT + 1;                   // level-row pitch (odd: scattered updates spread)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* cnt = reinterpret_cast<int*>(smem_raw);      // [256][NTP] packed counts (box 0 lo16, box 1 hi16)
  int* K = cnt + 256 * NTP;                         // [511] K_lit(t) * 2^30, t = -255..255
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * P.TW;
  const int y0 = blockIdx.y * P.TH;
  const long long fbase = (long long)blockIdx.z * P.frame_elems;
  const int col = x0 - P.rlo_x + tid;
  const bool colok = (col >= 0) & (col < P.W);
  const int TWv = min(P.TW, P.W - x0);
  const int yend = min(y0 + P.TH, P.H);

  for (int i = tid; i < 256 * NTP; i += LIT_NT) cnt[i] = 0;
  for (int i = tid; i < 511; i += LIT_NT) K[i] = P.klut[i];
  __syncthreads();
  // counts of the vertical boxes at row y0 - 1
  if (colok) {
    for (int v = P.vmin; v <= P.vmax; ++v) {
      const int row = y0 - 1 + v;
      if (row < 0 || row >= P.H) continue;
      const int z = in[fbase + (long long)row * P.W + col];
      int inc = 0;
      for (int b = 0; b < P.nby; ++b)
        if (v >= P.vlo[b] && v <= P.vhi[b]) inc += 1 << (16 * b);
      cnt[z * NTP + tid] += inc;
    }
  }
  for (int y = y0; y < yend; ++y) {
    // ---- slide the column's counts down one row: enter y + vhi_b, leave y + vlo_b - 1
    if (colok) {
      for (int b = 0; b < P.nby; ++b) {
        const int re = y + P.vhi[b], rl = y + P.vlo[b] - 1;
        if (re >= 0 && re < P.H) cnt[in[fbase + (long long)re * P.W + col] * NTP + tid] += 1 << (16 * b);
        if (rl >= 0 && rl < P.H) cnt[in[fbase + (long long)rl * P.W + col] * NTP + tid] -= 1 << (16 * b);
      }
    }
    __syncthreads();
    // ---- windowed level sums for the output pixels of row y
    if (tid < TWv) {
      const long long pix = fbase + (long long)y * P.W + x0 + tid;
      const int I0 = in[pix];
      const int zlo = max(0, I0 - P.Tw), zhi = min(255, I0 + P.Tw);
      long long A[2][2] = {{0, 0}, {0, 0}}, B[2][2] = {{0, 0}, {0, 0}};
      const int* base = cnt + tid + P.rlo_x;
      for (int z = zlo; z <= zhi; ++z) {
        const int* rowz = base + z * NTP;
        const int kz = K[I0 - z + 255];
        // horizontal boxes, the inner (b' = 1, nested) first
        int s1 = 0;
        if (P.nbx > 1)
          for (int u = P.hlo[1]; u <= P.hhi[1]; ++u) s1 += rowz[u];
        int s0 = 0;
        if (P.nbx > 1 && P.hlo[0] <= P.hlo[1] && P.hhi[1] <= P.hhi[0]) {
          s0 = s1;
          for (int u = P.hlo[0]; u < P.hlo[1]; ++u) s0 += rowz[u];
          for (int u = P.hhi[1] + 1; u <= P.hhi[0]; ++u) s0 += rowz[u];
        } else {
          for (int u = P.hlo[0]; u <= P.hhi[0]; ++u) s0 += rowz[u];
        }
        const int sb[2] = {s0, s1};
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
#pragma unroll
          for (int by = 0; by < 2; ++by) {
            const int c = (sb[bx] >> (16 * by)) & 0xFFFF;
            A[by][bx] += (long long)c * kz;
            B[by][bx] += (long long)(c * z) * kz;
          }
        }
      }
      double num = 0.0, den = 0.0;
#pragma unroll
      for (int by = 0; by < 2; ++by)
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
          num += P.wxy[by][bx] * (double)B[by][bx];
          den += P.wxy[by][bx] * (double)A[by][bx];
        }
      const bool fb = !(den > 0.0);
      out[pix] = fb ? (float)I0 : (float)(num / den);
      note_fallback(P.fb_count, P.fb_mask, pix, fb);
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_literal(const LParams& L, const unsigned char* in, float* out, dim3 grid, size_t smem,
                           cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(bf_literal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  bf_literal_kernel<<<grid, LIT_NT, smem, st>>>(L, in, out);
  return cudaGetLastError();
}

}  // namespace bf
