// Case 1 of the paper's pre-computation, second phase: bf_apply_cached combines
// precomputed box-filtered channels with a range plan chosen after the fact. With T_{r_i} = D the
// channels g^c_k, g^s_k, G^c_k, G^s_k and their box sums do not depend on the range kernel
// (P:1205), so bf_precompute stores them once per image (plane k: one 16-byte entry
// per pixel holding F of the four channels, F = round(sum_b ax_b H_b / 2^32) as kernels 1 / 2 form
// it) and this kernel only evaluates
//     num = sum_k W_c F_Ic + W_s F_Is,   den = sum_k W_c F_c + W_s F_s   (eq:numerator_2D_box_N_terms)
// per pixel: an HBM-bound pass, 16 B per selected term per pixel plus the input and output.
//
// Design (a streaming pipeline): a persistent CTA per SM walks tiles of CP consecutive pixels. For
// a tile, the entries of each selected term form ONE contiguous CP x 16 B run of its cache plane,
// so a producer thread moves them with bulk asynchronous copies (cp.async.bulk, the TMA engine:
// no registers, no per-thread address arithmetic) into a ring of CS stages in shared memory,
// completing the stage's mbarrier by transaction bytes. The consumer threads (one pixel each)
// wait on the stage, form the fp64 weights (Chebyshev recurrence) and the exact int64 sums, and
// release the stage. Up to CS - 1 stages (32 KB each: 4 terms of 512 pixels) are in flight per SM
// while one is combined, which covers the HBM latency at the per-SM share of the bandwidth. Plans
// with more than CK terms take several stages per tile (the sums carry over). The input pixel is
// loaded by its consumer thread one tile ahead.
#include <algorithm>

#include "bf_device.cuh"

namespace bf {
namespace {

#ifndef BF_CACHE_CP
#define BF_CACHE_CP 512
#endif
#ifndef BF_CACHE_CK
#define BF_CACHE_CK 4
#endif
#ifndef BF_CACHE_CS
#define BF_CACHE_CS 6
#endif
constexpr int CP = BF_CACHE_CP;         // pixels per tile = consumer threads
constexpr int CK = BF_CACHE_CK;         // terms per stage
constexpr int CS = BF_CACHE_CS;         // stages in the ring
constexpr int CTH = CP + 32;            // + one producer warp
constexpr int STAGE_BYTES = CK * CP * 16;          // the entries of CK terms for one tile

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned a, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned a, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mb_expect(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// global -> shared bulk copy (bytes and both addresses multiples of 16), completing mbar's tx count
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

template <bool U8>
__global__ void __launch_bounds__(CTH, 1) bf_cached_kernel(const CParams C, const int4* __restrict__ cache,
                                                           const void* __restrict__ in, float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);   // [CS]
  unsigned long long* empty = full + CS;                                    // [CS]
  double2* lut64 = reinterpret_cast<double2*>(smem + 128);                  // [256] (u8)
  unsigned char* ring = smem + 128 + 256 * sizeof(double2);                 // [CS][STAGE_BYTES]
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < CS; ++s) {
      mb_init(su32(&full[s]), 1);          // the producer's expect_tx arrival + the copies' bytes
      mb_init(su32(&empty[s]), CP / 32);   // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (U8)
    for (int i = tid; i < 256; i += CTH) {
      double s, c;
      sincospi((double)i * C.invD, &s, &c);
      lut64[i] = make_double2(c, s);
    }
  __syncthreads();
  const long long n = (long long)C.H * C.W;
  const long long ntiles = (n + CP - 1) / CP;
  const int nchunk = (C.nk + CK - 1) / CK;   // C.nk: the real terms

  if (tid >= CP) {
    // ---------------------------------------------------------------- producer (one thread)
    if (tid != CP) return;
    int s = 0;
    unsigned ph = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const long long p0 = t * CP;
      const int np = (int)std::min<long long>(CP, n - p0);
      for (int c = 0; c < nchunk; ++c) {
        mb_wait(su32(&empty[s]), ph ^ 1);   // the consumers are done with this stage's last use
        const int k0 = c * CK, nk = min(CK, C.nk - k0);   // (padded terms are not copied)
        mb_expect(su32(&full[s]), (unsigned)(nk * np * 16));
        unsigned char* st = ring + (size_t)s * STAGE_BYTES;
        for (int j = 0; j < nk; ++j)
          bulk_g2s(su32(st + j * CP * 16), cache + (long long)C.ch[k0 + j] * C.plane + p0, (unsigned)(np * 16),
                   su32(&full[s]));
        if (++s == CS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------------ consumers: one pixel each
  // (the term list is padded on the host to a multiple of CK with zero weights: no per-term
  // branches; a padded term reads stale shared memory and adds 0)
  int s = 0;
  unsigned ph = 0;
  const long long step = (long long)gridDim.x * CP;
  float Inext = (long long)blockIdx.x * CP + tid < n ? load_pixel(in, U8, (long long)blockIdx.x * CP + tid) : 0.f;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long pix = t * CP + tid;
    const float Ic = Inext;   // the input pixel, loaded one tile ahead
    if (pix + step < n) Inext = load_pixel(in, U8, pix + step);
    double c1, s1;
    if (U8) {
      const double2 tt = lut64[(int)Ic];
      c1 = tt.x;
      s1 = tt.y;
    } else {
      base_angle_f64(Ic, C.invD, c1, s1);
    }
    Cheb64 g;
    g.init(c1, s1);
    for (int j = 0; j < C.kval[0]; ++j) g.step();
    int mass = 0;
    // four independent exact accumulators (integer sums: the split does not change the result)
    long long nc = 0, ns = 0, dc = 0, ds = 0;
    for (int c = 0; c < nchunk; ++c) {
      mb_wait(su32(&full[s]), ph);
      const int4* st = reinterpret_cast<const int4*>(ring + (size_t)s * STAGE_BYTES);
#pragma unroll
      for (int j = 0; j < CK; ++j) {
        const int i = c * CK + j;
        if (i > 0) {   // k_i - k_{i-1} >= 1 recurrence steps
          g.step();
          extra_steps(C.kstep[i], [&] { g.step(); });
        }
        const int4 f = st[j * CP + tid];
        if (i == C.mass_i) mass = f.x;
        const int wc = __double2loint(fma(g.c, C.aw[i], MAGIC64));
        const int wsn = __double2loint(fma(g.s, C.aw[i], MAGIC64));
        dc = mad_wide(wc, f.x, dc);
        ds = mad_wide(wsn, f.y, ds);
        nc = mad_wide(wc, f.z, nc);
        ns = mad_wide(wsn, f.w, ns);
      }
      __syncwarp();
      if ((tid & 31) == 0) mb_arrive(su32(&empty[s]));
      if (++s == CS) {
        s = 0;
        ph ^= 1;
      }
    }
    if (pix < n) {
      const long long num = nc + ns, den = dc + ds;
      const bool fb = !(den > 0);
      __stcs(out + pix, fb ? Ic : (float)(C.D * (double)num / (double)den));
      const bool fl = flag_pixel(C.rep, den, mass, pix);
      note_fallback(C.fb_count, C.fb_mask, pix, fb && !fl);
    }
  }
}

int sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 148;
  return n > 0 ? n : 148;
}

}  // namespace

cudaError_t launch_cached(const CParams& C, const int4* cache, const void* in, float* out, cudaStream_t st) {
  const long long n = (long long)C.H * C.W;
  const long long ntiles = (n + CP - 1) / CP;
  const int grid = (int)std::min<long long>(ntiles, sms());   // persistent: one CTA per SM
  const size_t smem = 128 + 256 * sizeof(double2) + (size_t)CS * STAGE_BYTES;
  auto kfn = C.u8 ? bf_cached_kernel<true> : bf_cached_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kfn<<<grid, CTH, smem, st>>>(C, cache, in, out);
  return cudaGetLastError();
}

}  // namespace bf
