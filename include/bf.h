/*
 * bf.h - C ABI of the B200 (sm_100a) joint-acceleration bilateral filter library (libbf.so).
 *
 * Implements the hot path of "Speeding up the Bilateral Filter: A Joint Acceleration Way"
 * (Dai, Yuan, Zhang; arXiv 1803.00004). Citations "P:n" are lines of the paper's LaTeX source
 * (PAPER.md); "Q<n>" are the readings of the paper listed in DESIGN.md / SURVEY.md 8(c).
 *
 * The bilateral filter (eq:BF)
 *     out(x) = sum_y K_s(|x-y|) K_r(I(x)-I(y)) I(y) / sum_y K_s(|x-y|) K_r(I(x)-I(y))
 * is evaluated as the paper's box-filter expansion (eq:numerator_2D_box_N_terms):
 *   - K_r is replaced by its best N-term cosine expansion on [-D, D] (the Case 1
 *     substitution T_{r_i} = D of P:1205/P:1215-1217, Q1, which makes the z-window of the
 *     dimension promotion cover every intensity so the 3-D box filters collapse to 2-D);
 *   - the truncated K_s is replaced by its best N_s-term 2-D Haar expansion on
 *     [-(r+1/2), r+1/2]^2 (Q8/Q9), lowered to box filters (Appendix A);
 *   - every cosine term k contributes the channels cos(w_k I), sin(w_k I), I cos(w_k I),
 *     I sin(w_k I), which are box-filtered and recombined with the per-pixel factors
 *     a_k cos(w_k I(x)), a_k sin(w_k I(x)) (Q17); out = num / den.
 *
 * All functions are thread-safe. A plan is immutable after creation and may be used
 * concurrently by several bf_apply calls on different streams. No device-side entry point
 * allocates device memory or synchronises the host (bf_apply_host excepted, see there), so every
 * bf_apply* call can be captured into a CUDA graph.
 */
#ifndef BF_H_
#define BF_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BF_API __attribute__((visibility("default")))
#else
#define BF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque, library-owned, immutable plan (host memory only). */
typedef struct bf_plan bf_plan;

/* CUDA stream handle as an opaque pointer (a cudaStream_t; NULL = the legacy default stream). */
typedef void* bf_stream;

typedef enum {
  BF_OK = 0,
  BF_ERR_INVALID_ARG = 1,   /* NULL pointer, non-positive size, sigma <= 0, N < 1, ...       */
  BF_ERR_UNSUPPORTED = 2,   /* unknown kernel kind, or a plan shape the GPU path lacks       */
  BF_ERR_NO_MEMORY = 3,     /* host allocation failed                                        */
  BF_ERR_CUDA = 4,          /* a CUDA launch or runtime call failed (no device sync is done)  */
  BF_ERR_NUMERIC = 5,       /* the fitter produced no usable term (e.g. all coefficients 0)  */
  BF_ERR_WORKSPACE = 6      /* the plan runs in several passes and needs a device workspace:
                               pass one through bf_apply_ex (size: bf_workspace_size)         */
} bf_status;

/* Spatial kernel K_s: isotropic Gaussian exp(-(u^2+v^2)/2 sigma_s^2) or a box,
 * truncated to the square |u|,|v| <= radius (Q9). */
typedef enum { BF_SPATIAL_GAUSSIAN = 0, BF_SPATIAL_BOX = 1 } bf_spatial_kind;

/* Range kernel K_r: Gaussian exp(-t^2/2 sigma_r^2) (sigma_r = +INFINITY gives
 * K_r == 1), or the Tukey biweight (1-(t/sigma_r)^2)^2 for |t| <= sigma_r, else 0 (Q22). */
typedef enum { BF_RANGE_GAUSSIAN = 0, BF_RANGE_TUKEY = 1 } bf_range_kind;

/* Input pixel type; the output is always float32. */
typedef enum { BF_IN_U8 = 0, BF_IN_F32 = 1 } bf_input_dtype;

typedef struct {
  double intensity_max;  /* D: inputs must lie in [0, D] (not checked on the device); default 255 */
  int n_spatial_terms;   /* N_s, the best-N_s Haar terms of K_s; default 9 (Q15)        */
  int input_dtype;       /* bf_input_dtype; default BF_IN_F32                                   */
  int m_factor;          /* candidate count M = m_factor * N for the range fit; def 20 */
  int haar_levels;       /* Haar levels j <= J considered for K_s; default 4           */
  int range_window;      /* BF_RANGE_WINDOW_FULL (default): T = D, the z-window covers every
                            intensity (Case 1, Q1) -> 2-D box filters of modulated channels;
                            BF_RANGE_WINDOW_LITERAL: the paper's literal 3-D form (NEXT f1):
                            T = T_r = K_r^{-1}(0.01), cosines of period 2 T_r fitted on
                            [-T_r, T_r] and the dimension-promoted window
                            [I(x) - T_r, I(x) + T_r]; u8 input with D = 255 only.  */
} bf_plan_options;

/* bf_plan_options.range_window */
enum { BF_RANGE_WINDOW_FULL = 0, BF_RANGE_WINDOW_LITERAL = 1 };

/* Maximum N (range terms) and N_s (spatial terms) accepted by bf_plan_create. */
#define BF_MAX_TERMS 32
#define BF_MAX_SPATIAL_TERMS 64
/* Maximum range plans one bf_apply_multi evaluates over shared channels. */
#define BF_MAX_PLANS 4
/* Maximum boxes per axis of the separable spatial factor the GPU path runs. */
#define BF_MAX_AXIS_BOXES 4

/* Fills *opt with the defaults listed above. */
BF_API void bf_plan_options_default(bf_plan_options* opt);

/*
 * Fits the expansion coefficients on the host (a one-off cost; Table I):
 *   range:   a_0 = 1/(2D) int_{-D}^{D} K_r,  a_k = 1/D int K_r(t) cos(pi k t / D) dt
 *            (P:204-208 with T = D), k < M = m_factor * n_terms; the n_terms largest |a_k|
 *            (ties to the smaller k, zeros pruned: Q4/Q6/Q7);
 *   spatial: 2-D Haar coefficients (eq:Haar_2D_coefficients) with levels <= J,
 *            best n_spatial_terms (ties by canonical order), lowered to boxes on integer
 *            offsets with half-open cells (Q11), factored into separable 1-D box filters.
 * Arguments: ks, kr kernel kinds; sigma_s > 0 (ignored for BF_SPATIAL_BOX); sigma_r > 0
 * (may be +INFINITY for the Gaussian); radius >= 0 (spatial truncation r, T_s = r + 1/2);
 * n_terms in [1, BF_MAX_TERMS]; opt may be NULL (defaults).
 * On success *out receives a new plan owned by the caller (free with bf_plan_destroy).
 * On failure *out is set to NULL and an error code is returned; no partial state remains.
 */
BF_API bf_status bf_plan_create(bf_plan** out, int ks, int kr, double sigma_s, double sigma_r, int radius,
                                int n_terms, const bf_plan_options* opt);

/* Releases a plan. NULL is a no-op. Returns BF_OK. */
BF_API bf_status bf_plan_destroy(bf_plan* plan);

/* Plan contents, for inspection and cross-checking against an independent fitter. */
typedef struct {
  int n_terms_eff;                           /* N_eff <= N after pruning zero coefficients     */
  int k[BF_MAX_TERMS];                       /* selected frequencies (ascending)               */
  double a[BF_MAX_TERMS];                    /* their coefficients a_k                         */
  double T_range;                            /* T of the cosine basis (D, or T_r if literal)  */
  int n_spatial_eff;                         /* selected 2-D Haar terms                        */
  int sp_family[BF_MAX_SPATIAL_TERMS];       /* 0 phi.phi, 1 phi(x)psi(y), 2 psi(x)phi(y), 3 psi.psi */
  int sp_j1[BF_MAX_SPATIAL_TERMS], sp_k1[BF_MAX_SPATIAL_TERMS];   /* x factor (j,k); -1,0 = phi */
  int sp_j2[BF_MAX_SPATIAL_TERMS], sp_k2[BF_MAX_SPATIAL_TERMS];   /* y factor (j,k); -1,0 = phi */
  double sp_coef[BF_MAX_SPATIAL_TERMS];      /* c_j of the selected terms                      */
  int separable;                             /* 1 if K~_s = fx(u) fy(v) (GPU path supported)  */
  int nbx, nby;                              /* boxes per axis of the separable factors        */
  int box_lo_x[BF_MAX_AXIS_BOXES], box_hi_x[BF_MAX_AXIS_BOXES];  /* column offsets, inclusive  */
  double box_w_x[BF_MAX_AXIS_BOXES];
  int box_lo_y[BF_MAX_AXIS_BOXES], box_hi_y[BF_MAX_AXIS_BOXES];  /* row offsets, inclusive     */
  double box_w_y[BF_MAX_AXIS_BOXES];
  int radius;                                /* spatial truncation radius r                    */
  double intensity_max;                      /* D                                              */
  int input_dtype;                           /* bf_input_dtype                                 */
  int spatial_rank;                          /* terms fx_s(u) fy_s(v) of the GPU box-pair form:
                                                1 separable, 2 rank-2 (e.g. N_s = 5), R for the
                                                general plans below, 0 none                       */
  int range_window;                          /* bf_plan_options.range_window of the plan        */
  int spatial_passes;                        /* separable passes bf_apply runs: 1, or for general
                                                plans (no separable / rank-2 form, e.g. N_s = 13
                                                or 25 at haar_levels 4) one per product of box
                                                groups of an exact rank-R factorisation (<= 16);
                                                0 = no GPU form (BF_ERR_UNSUPPORTED)              */
} bf_plan_info;

/* Copies the plan contents into *info. */
BF_API bf_status bf_plan_get_info(const bf_plan* plan, bf_plan_info* info);

/*
 * Filters one H x W image on the GPU: d_in is a device pointer to a dense row-major image of
 * the plan's input dtype (pitch W elements), d_out a device pointer to H*W float32 (pitch W).
 * The caller owns both buffers and the stream; they must not alias. The work is enqueued
 * asynchronously on `stream` (no host synchronisation, no device allocation, so the call is
 * CUDA-graph capturable); launch errors are returned as BF_ERR_CUDA, faults appear at the
 * caller's next synchronisation. Pixels outside the image contribute nothing (Q16). Pixels
 * whose approximated denominator is <= 0 or not finite get out = I(x) (Q18). The result is
 * deterministic (fixed reduction order, exact integer box sums, no atomics).
 * Returns BF_ERR_INVALID_ARG for NULL pointers, H or W <= 0, H*W overflow or d_in == d_out;
 * BF_ERR_UNSUPPORTED if the plan's spatial kernel has no box-pair form of rank <= 2 (see
 * bf_plan_info.spatial_rank; rank 2 is K~_s = sum_{s<2} fx_s(u) fy_s(v) with box factors);
 * BF_ERR_WORKSPACE if the plan runs in several passes (rank-2 or >= 3-box plans with more than 8
 * or 16 terms; every separable N_s = 9 / box plan with N <= 32 runs in one pass): use bf_apply_ex.
 */
BF_API bf_status bf_apply(const bf_plan* plan, const void* d_in, float* d_out, int H, int W, bf_stream stream);

/* Kernel choice of bf_apply_ex (bf_apply_args.kernel). AUTO is the library's choice; the others
 * force one kernel where it can run the plan (for A/B timing and the bitwise cross-kernel tests:
 * all of them compute the same integers). */
enum { BF_KERNEL_AUTO = 0, BF_KERNEL_BAND = 1, BF_KERNEL_WS = 2, BF_KERNEL_WS2 = 3, BF_KERNEL_WS2_WIDE = 4 };
/* (BF_KERNEL_WS2_WIDE: kernel 2b with two columns per vertical-pass thread and 8 terms per CTA,
 * the range terms split over a CTA cluster: the automatic choice for radii above 96) */

/* Optional arguments of bf_apply_ex / bf_workspace_size / bf_apply_config. Zero-initialised (or
 * bf_apply_args_default) means: library's kernel and tiling, all rows, no workspace, no counters. */
typedef struct {
  int kernel;                           /* BF_KERNEL_*                                             */
  int band_rows;                        /* output rows per CTA band; 0 = the library's cost model  */
  int row_begin, row_end;               /* compute output rows [row_begin, row_end) only (the input
                                           rows their windows need must be valid); 0, 0 = all     */
  void* d_workspace;                    /* device workspace of multi-pass plans, or NULL           */
  size_t workspace_bytes;               /* its size (>= bf_workspace_size)                         */
  unsigned long long* d_fallback_count; /* device counter, or NULL: incremented by the number of
                                           pixels whose approximated denominator is <= 0 (out =
                                           I(x), Q18; "the pixel is counted")                 */
  unsigned char* d_fallback_mask;       /* device n_frames*H*W bytes, or NULL: 1 where the pixel
                                           took that fallback, else 0                               */
  double repair_threshold;              /* pixels whose den / sum K~_s (the clipped spatial mass) is
                                           below this (or den <= 0) are re-evaluated in fp64 from the
                                           approximated kernels (the direct double loop, reading Q27):
                                           0 = the library default (BF_REPAIR_DEFAULT), < 0 = off     */
  unsigned long long* d_repaired_count; /* device counter, or NULL: incremented by the number of
                                           pixels the fp64 repair pass re-evaluated                  */
  int u8_trig;                          /* u8 plans: 0 = the base angles (cos, sin)(pi I / D) from a
                                           256-entry table (Case 2; default), 1 = evaluated
                                           per tap (kernel 1 only): the same values, bitwise the same
                                           output                                            */
} bf_apply_args;

/* Default bf_apply_args.repair_threshold: out = num / den magnifies the fused kernels' rounding
 * (channel values in fp32, 22-bit tap quantisation) by 1 / cond. Measured over the BASELINE configs
 * at full size, |error| * cond <= 2.3e-7 * kmax on the [0, 255] scale (kmax = the largest selected
 * frequency: the fp32 channels' phase error grows with k), so the 1e-3 parity tolerance is reached
 * near cond = 2.3e-4 kmax; the default (threshold 0) re-evaluates every pixel below
 * max(BF_REPAIR_DEFAULT, 4.6e-4 kmax), twice that. At most 32768 flagged pixels per call are
 * repaired (the rest keep the fused value); up to 16 calls may be in flight per device. */
#define BF_REPAIR_DEFAULT 0.008

BF_API void bf_apply_args_default(bf_apply_args* args);

/*
 * bf_apply / bf_apply_batched with optional arguments (args may be NULL). Same contract as
 * bf_apply: asynchronous on `stream`, no allocation, no host synchronisation, graph capturable.
 * Multi-pass plans accumulate num / den (int64) in args->d_workspace (BF_ERR_WORKSPACE if it is
 * missing or too small); the counter / mask are written by the launch that finishes the pixel.
 */
BF_API bf_status bf_apply_ex(const bf_plan* plan, const void* d_in, float* d_out, int n_frames, int H, int W,
                             bf_stream stream, const bf_apply_args* args);

/* Device workspace bytes bf_apply_ex needs for this plan, shape and kernel choice (0 for one-pass
 * plans). Pure host computation. */
BF_API bf_status bf_workspace_size(const bf_plan* plan, int n_frames, int H, int W, const bf_apply_args* args,
                                   size_t* bytes);

/*
 * Filters n_frames independent H x W frames stored back to back (frame f at d_in + f*H*W
 * elements, likewise d_out) in one launch (NEXT f4 of the survey; used for BASELINE cfg3).
 */
BF_API bf_status bf_apply_batched(const bf_plan* plan, const void* d_in, float* d_out, int n_frames, int H, int W,
                           bf_stream stream);

/*
 * Frame sharding for multi-GPU frame streams (NEXT f4; BASELINE configs[3]): frames are independent
 * problems, so N GPUs (one process per GPU) each filter a contiguous block of them with
 * bf_apply_batched / bf_apply_ex on their own device, with no data-path collective. Part `part`
 * of n_parts gets frames [*first, *first + *count): contiguous blocks, the first
 * n_frames % n_parts parts one frame longer, every frame exactly once. Pure host computation.
 */
BF_API bf_status bf_shard_frames(int n_frames, int n_parts, int part, int* first, int* count);

/*
 * Case 1 of the paper's pre-computation: with T_{r_i} = D for every range kernel,
 * the modulated channels F_c, F_s and their box sums do not depend on sigma_r, so n_plans range
 * plans (e.g. several sigma_r, or Gaussian and Tukey) are evaluated in ONE pass that shares the
 * vertical / horizontal box filtering; only the per-pixel combine runs per plan.
 * plans[0..n_plans) must share the spatial plan (same boxes and weights), D and input dtype
 * (else BF_ERR_INVALID_ARG); the union of their selected k must fit one CTA's pass (<= 16 terms)
 * and the spatial plan must be separable with at most two boxes per axis (the default N_s = 9,
 * or a box), else BF_ERR_UNSUPPORTED. d_out holds n_plans H x W float32 images back to back (plan
 * q at d_out + q*H*W). 1 <= n_plans <= BF_MAX_PLANS. Otherwise as bf_apply. For range plans not
 * known up front use bf_precompute / bf_apply_cached below.
 */
BF_API bf_status bf_apply_multi(const bf_plan* const* plans, int n_plans, const void* d_in, float* d_out, int H, int W,
                                bf_stream stream);

/* Host-to-host convenience for end-to-end timing: copies h_in (host) to the device, filters,
 * copies the result back into h_out (host) and synchronises `stream`. Large images run as up to
 * five row chunks pipelined over library-owned streams (ordered after the work already in
 * `stream`): the copy of the next input piece, the filter of the current chunk and the copy back
 * of the previous chunk overlap. Pinned host buffers make the copies asynchronous. Device
 * buffers (input, output and, for multi-pass plans, the workspace) come from a library-owned
 * cache per device (grown on demand, freed at exit); calls on different devices run
 * concurrently, calls on one device are serialised. This is the one entry point that allocates
 * device memory and synchronises (`stream`, before returning). Results equal bf_apply's bitwise. */
BF_API bf_status bf_apply_host(const bf_plan* plan, const void* h_in, float* h_out, int H, int W, bf_stream stream);

/*
 * Number of kernel launches one bf_apply / bf_apply_batched of an H x W image enqueues with this
 * plan (1, or ceil(N_eff / terms-per-pass) passes for multi-pass plans, which accumulate num /
 * den in the caller's workspace). Pure host computation, no device work. Returns
 * BF_ERR_INVALID_ARG for a NULL plan / pointer or H, W <= 0, BF_ERR_UNSUPPORTED as bf_apply would.
 */
BF_API bf_status bf_apply_launches(const bf_plan* plan, int H, int W, int* n_launches);

/* Launch configuration bf_apply_batched(plan, ., ., n_frames, H, W, .) enqueues (bf_apply is
 * n_frames = 1): kernel name (a static string owned by the library), threads per CTA, grid
 * (strips x bands x frames), output tile (columns per strip, rows per band), dynamic shared
 * memory per CTA, the number of launches (passes) and kernel 2b's warp-role map. Pure host computation, no device work;
 * the kernel choice and band height follow the same rules (bf_apply_args.kernel / band_rows)
 * as the apply call. Errors as bf_apply_launches. */
typedef struct bf_launch_config {
  int n_launches;
  const char* kernel;
  int threads_per_cta;
  int grid_x, grid_y, grid_z;    /* grid_x counts every CTA: strips x cluster_size          */
  int tile_w, tile_h;
  size_t smem_bytes;
  int cluster_size;              /* CTAs per cluster (range terms split over the cluster)    */
  int terms_per_cta;             /* range terms one CTA evaluates per pass                   */
  int cols_per_thread;           /* extended columns per vertical-pass thread (kernel 2b)    */
  size_t workspace_bytes;        /* bf_workspace_size of the same call                       */
  unsigned char warp_map[24];    /* kernel 2b: logical warp (role order: box-difference/combine
                                  * warps, scan warps, vertical-pass warps) run by physical warp
                                  * i; the working warps of each role are spread evenly over the
                                  * four SM sub-partitions (i mod 4). All 0 for other kernels.  */
} bf_launch_config;

/* args may be NULL (as bf_apply); args->kernel / band_rows are honoured as in bf_apply_ex. */
BF_API bf_status bf_apply_config(const bf_plan* plan, int n_frames, int H, int W, const bf_apply_args* args,
                                 bf_launch_config* cfg);

/*
 * Case 1 of the paper's pre-computation (NEXT f2), the paper's two phases:
 * bf_precompute runs once per image and stores the box-filtered channels of the frequencies
 * k = 0 .. k_count-1 (S(g^c_k), S(g^s_k), S(G^c_k), S(G^s_k) of eq:numerator_2D_box_N_terms,
 * P:481-493; with T_{r_i} = D they do not depend on the range kernel) in the
 * caller's device buffer d_cache (bf_cache_size bytes, 16-byte aligned; layout: plane k of H*W
 * row-major 16-byte entries, entry = the four channels as int32 in that order, each the
 * box-weighted sum F = round(sum_b ax_b H_b / 2^32) of the exact box sums H_b). bf_apply_cached
 * then evaluates any range plan whose selected k all lie below k_count and whose spatial plan, D
 * and input dtype equal the precompute plan's, as one combine-only pass that reads the cache and
 * the input (HBM-bound: 16 B per selected term per pixel). Its output equals bf_apply's to the
 * rounding of F (bf_apply's default kernel keeps the per-box sums exact; the kernels that form F,
 * BF_KERNEL_WS / BF_KERNEL_BAND, agree with it bitwise). Both are asynchronous on `stream`,
 * allocate nothing and are graph capturable. desc (host memory, filled by bf_precompute) carries
 * what bf_apply_cached checks.
 * Errors: BF_ERR_INVALID_ARG for NULL pointers, sizes, k_count outside [1, BF_MAX_TERMS], a too
 * small or misaligned cache, or a plan that does not match desc; BF_ERR_UNSUPPORTED for literal
 * plans and spatial plans other than separable with at most two boxes per axis.
 */
typedef struct {
  int k_count, H, W, input_dtype;
  double intensity_max;
  unsigned long long spatial_key;   /* fingerprint of the spatial plan and the channel quantisation */
} bf_cache_desc;

BF_API bf_status bf_cache_size(const bf_plan* plan, int k_count, int H, int W, size_t* bytes);
BF_API bf_status bf_precompute(const bf_plan* plan, int k_count, const void* d_in, int H, int W, void* d_cache,
                               size_t cache_bytes, bf_stream stream, bf_cache_desc* desc);
BF_API bf_status bf_apply_cached(const bf_plan* plan, const bf_cache_desc* desc, const void* d_cache,
                                 const void* d_in, float* d_out, bf_stream stream, const bf_apply_args* args);

/* The lowered spatial kernel K~_s(v, u) (eq:Box_N_terms, Appendix A) exactly as the
 * GPU path applies it (its separable / box-pair / general-pass form), on the integer offsets
 * u, v in [-r, r]: K[(v + r) * (2r + 1) + (u + r)]; n_values >= (2r + 1)^2 (host memory). For
 * cross-checking the plan's factorisation against an independent lowering. BF_ERR_UNSUPPORTED if
 * the plan has no GPU form. */
BF_API bf_status bf_plan_spatial_kernel(const bf_plan* plan, double* K, size_t n_values);

/* Static string for a status code. */
BF_API const char* bf_status_string(bf_status s);

/* Library version string ("bf-b200 <semver>"). */
BF_API const char* bf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BF_H_ */
