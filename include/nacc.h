/*
 * nacc.h — C ABI of the B200-native packed-sample volume-rendering core
 * (the data-parallel hot path of NerfAcc, arXiv 2305.04966).
 *
 * The calls mirror Algorithm 1 of the paper:
 *   t0, t1, r_id = nerfacc.sampling(r_o, r_d, estimator, density_fn)
 *       -> nacc_sampling_occgrid (+ caller evaluates σ) -> nacc_filter_early_stop
 *   color, opacity, depth, aux = nerfacc.rendering(t0, t1, r_id, ...)
 *       -> nacc_render_fwd / nacc_render_bwd (fused), or the granular
 *          nacc_render_weights_fwd/bwd + nacc_accumulate_along_rays(_bwd)
 *   estimator.update_every_n_steps(...)
 *       -> nacc_occgrid_points (+ caller evaluates σ, all-reduces MAX)
 *          -> nacc_occgrid_update
 *   proposal-network estimator -> nacc_importance_sample
 * The library never calls the radiance field: Alg. 1's density_fn /
 * rgb_density_fn are evaluated by the caller between calls.
 *
 * Conventions (apply to every call unless stated):
 *  - Pointers are DEVICE pointers unless named *_host.  The caller owns and
 *    allocates every buffer; the library never allocates, frees, retains
 *    pointers past stream completion, or keeps global state (except the
 *    thread-local error string and a launch counter).
 *  - Every call is asynchronous on `stream` and never synchronises.  Counts
 *    that size later buffers (`total`) are written to device int64s.
 *  - Host-side validation runs before any launch.  On invalid arguments the
 *    call returns NACC_ERR_INVALID_ARGUMENT and writes nothing.  n_rays == 0
 *    returns NACC_OK without launching (totals are set to 0 with a memset).
 *    CUDA launch errors return NACC_ERR_CUDA; nacc_last_error() (thread-local)
 *    holds the message.  Nothing aborts, exits or throws across the ABI.
 *  - Device preconditions are NOT checked: σ >= 0 and finite;
 *    ‖d‖ ≈ 1; per-ray intervals ascending and non-overlapping.
 *  - Layout ("sample as interval", "packed tensor"): samples are SoA
 *    t0[N], t1[N], sigma[N] fp32, rgb[N][3] fp32, ray_id[N] int32, ordered by
 *    ray then ascending t; packed_info[n_rays][2] int64 = (start, count).
 *    Arrays must be 4-byte aligned; packed_info / ctx 8-byte aligned.
 *  - Occupancy bitfield layout (public): cell q = l*R^3 + x + R*(y + R*z) of
 *    level l is bit (q & 31) of uint32 word (q >> 5).  Density arrays use the
 *    same cell order (level-major, x fastest; reading #27).
 */
#ifndef NACC_H
#define NACC_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NACC_ABI_VERSION 1

typedef enum {
  NACC_OK = 0,
  NACC_ERR_INVALID_ARGUMENT = 1,
  NACC_ERR_INSUFFICIENT_CAPACITY = 2, /* reported through *status_out of one-shot calls */
  NACC_ERR_CUDA = 3,
  NACC_ERR_UNSUPPORTED = 4
} nacc_status;

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *nacc_last_error(void);
int nacc_abi_version(void);
/* Number of kernels this library has launched in this process (all threads). */
uint64_t nacc_launch_count(void);

/* ------------------------------------------------------------------------ */
/* Occupancy grid ("Spatial Skipping"; Instant-NGP cascade,         */
/* DESIGN.md reading #4): level l covers centre ± half·2^l of `roi`, l < levels */
/* (1..8), res^3 cells per level, levels*res^3 < 2^31.                          */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t levels;
  int32_t res;
  float roi[6]; /* lo_x, lo_y, lo_z, hi_x, hi_y, hi_z of level 0; lo < hi */
} nacc_grid;

/* Ray-marching parameters ("follow the original paper's implementation";
 * P:158 marching step Δt; P:257 coarser steps with distance). */
typedef struct {
  float near_plane; /* lattice anchor when t_min == NULL (reading #1) */
  float far_plane;  /* interval k is emitted only if its midpoint < far */
  float step;       /* Δt (uniform lattice) or Δt_min (cone lattice); > 0 finite */
  float max_step;   /* Δt_max for the cone lattice; >= step */
  float cone_angle; /* c >= 0; 0 = uniform lattice t_k = near + kΔt (reading #5) */
  int32_t stratified; /* jitter each ray's anchor by ξ_r·Δt, ξ_r = Philox(seed,(r,0,0,0)) */
  uint64_t seed;
} nacc_march;

/* Bytes of the bitfield buffer for `grid` (0 if invalid): the public fine bits
 * (4*ceil(levels*res^3/32) bytes, rounded up to 256) followed by a
 * library-private region: a 256-byte header (the boxes enclosing the occupied
 * cells), a skip mask (1 bit per 4^3 macro cell, when res % 4 == 0) and, with
 * it, the OR / AND window masks of w^3 fine cells (1 bit per fine cell each)
 * for w = 2..9 on cascades (levels > 1) and w = 2..5 on a single level. */
size_t nacc_grid_bits_bytes(const nacc_grid *grid);

/* Rebuild the private region of `bits` (occupied-cell boxes, skip mask) from
 * its fine bits.  Required after the caller writes fine bits directly;
 * nacc_occgrid_update does it itself.  nacc_sampling_occgrid reads the region
 * (its results do not depend on it, only its speed — but a stale region would
 * skip occupied cells). */
nacc_status nacc_grid_prepare(const nacc_grid *grid, uint32_t *bits, cudaStream_t stream);

/* Workspace for nacc_sampling_occgrid / _fill with n_rays rays. */
size_t nacc_sampling_occgrid_workspace_bytes(const nacc_grid *grid, const nacc_march *params,
                                             int64_t n_rays);

/* Alg. 1 nerfacc.sampling with the occupancy-grid estimator.
 * For every ray r, interval k of the lattice (uniform t_k = near_r + kΔt, or
 * the cone recurrence t_{k+1} = t_k + clamp(t_k·c, Δt_min, Δt_max)) is emitted
 * iff its midpoint m_k < far_r lies in an occupied cell of the finest level
 * whose box holds it (readings #1-#3; the fp32 op sequence there is
 * normative).  Emitted intervals are packed: t0 = t_k, t1 = t_{k+1},
 * ray_id = r, in ray then k order.
 *   bits          occupancy bitfield (layout above), nacc_grid_bits_bytes() bytes,
 *                 prepared (nacc_grid_prepare / nacc_occgrid_update)
 *   rays_o/_d     [n_rays][3] fp32 origins / unit directions
 *   t_min, t_max  optional per-ray near/far [n_rays] (NULL = params' planes);
 *                 the cone lattice requires t_min == NULL and stratified == 0
 *                 (shared anchor), else NACC_ERR_UNSUPPORTED
 *   packed_info   [n_rays][2] int64 out, always written
 *   total         device int64 out: Σ counts, always written
 *   t0,t1,ray_id  [capacity] out; complete iff total <= capacity (never written
 *                 past capacity; unspecified otherwise), else the
 *                 device int32 *status_out (NULL allowed) is set to
 *                 NACC_ERR_INSUFFICIENT_CAPACITY (else NACC_OK) and the caller
 *                 re-allocates and calls nacc_sampling_occgrid_fill.
 *   ws            workspace of nacc_sampling_occgrid_workspace_bytes() bytes. */
nacc_status nacc_sampling_occgrid(const nacc_grid *grid, const uint32_t *bits,
                                  const nacc_march *params, const float *rays_o,
                                  const float *rays_d, const float *t_min, const float *t_max,
                                  int64_t n_rays, int64_t *packed_info, float *t0, float *t1,
                                  int32_t *ray_id, int64_t capacity, int64_t *total,
                                  int32_t *status_out, void *ws, size_t ws_bytes,
                                  cudaStream_t stream);

/* Writes the samples described by a packed_info produced by
 * nacc_sampling_occgrid with the same inputs (the capacity-retry path). */
nacc_status nacc_sampling_occgrid_fill(const nacc_grid *grid, const uint32_t *bits,
                                       const nacc_march *params, const float *rays_o,
                                       const float *rays_d, const float *t_min,
                                       const float *t_max, int64_t n_rays,
                                       const int64_t *packed_info, float *t0, float *t1,
                                       int32_t *ray_id, void *ws, size_t ws_bytes,
                                       cudaStream_t stream);

/* ------------------------------------------------------------------------ */
/* §4.2 "No Gradient Filtering": drop samples whose ENTERING            */
/* transmittance T_i = exp(-Σ_{j<i} σ_j δ_j) is below ε, i.e. keep the prefix   */
/* with S_i <= neg_log_eps (reading #9; S_i accumulated in fp64).               */
/*   sigma         [n_samples] σ from the caller's no-grad density query        */
/*   neg_log_eps   -ln ε computed by the caller in fp64 (+inf disables)         */
/*   packed_info_out [n_rays][2], total out (device int64), always written;     */
/*   t0_out, t1_out, ray_id_out [capacity] written iff total <= capacity        */
/*   (capacity >= n_samples always suffices).                                   */
/* ------------------------------------------------------------------------ */
size_t nacc_filter_workspace_bytes(int64_t n_rays);
nacc_status nacc_filter_early_stop(const int64_t *packed_info, int64_t n_rays, const float *t0,
                                   const float *t1, const float *sigma, int64_t n_samples,
                                   double neg_log_eps, int64_t *packed_info_out, float *t0_out,
                                   float *t1_out, int32_t *ray_id_out, int64_t capacity,
                                   int64_t *total, void *ws, size_t ws_bytes,
                                   cudaStream_t stream);

/* ------------------------------------------------------------------------ */
/* Transmittance estimator and compositing (Eq. 2, discretised as   */
/* P:246 with the index typo read as σ(t_j), reading #11):                     */
/*   δ_i = t1_i - t0_i, s_i = σ_i δ_i, S_i = Σ_{j<i} s_j (fp64),               */
/*   T_i = exp(-S_i), α_i = 1 - exp(-s_i), w_i = T_i α_i (0 once S_i > -ln ε). */
/* ------------------------------------------------------------------------ */
/* weights/trans/alphas [n_samples] out; trans and alphas may be NULL. */
nacc_status nacc_render_weights_fwd(const int64_t *packed_info, int64_t n_rays, const float *t0,
                                    const float *t1, const float *sigma, int64_t n_samples,
                                    double neg_log_eps, float *weights, float *trans,
                                    float *alphas, cudaStream_t stream);
/* The same outputs on ray-aligned flat tiles (the fused forward's layout: fp64
 * warp segmented scans, float4 runs), for packed samples from the sampling
 * calls: needs ray_id [n_samples] and the contiguous packing (start_0 = 0,
 * start_{r+1} = start_r + count_r).  Same arithmetic as nacc_render_weights_fwd
 * up to summation order (T by the product T_{j+1} = T_j e^{-s_j}). */
nacc_status nacc_render_weights_fwd_flat(const int64_t *packed_info, const int32_t *ray_id,
                                         int64_t n_rays, const float *t0, const float *t1,
                                         const float *sigma, int64_t n_samples, double neg_log_eps,
                                         float *weights, float *trans, float *alphas,
                                         cudaStream_t stream);
/* g_sigma_i = δ_i (g_w_i T_i (1-α_i)[live] - Σ_{j>i} g_w_j w_j - Σ_{j>i} g_T_j T_j);
 * g_trans may be NULL (= 0). */
nacc_status nacc_render_weights_bwd(const int64_t *packed_info, int64_t n_rays, const float *t0,
                                    const float *t1, const float *sigma, int64_t n_samples,
                                    double neg_log_eps, const float *g_weights,
                                    const float *g_trans, float *g_sigma, cudaStream_t stream);

/* The same gradient on ray-aligned flat tiles for packed samples from the sampling
 * calls (ray_id [n_samples], contiguous packing): pass 1 writes each ray's
 * R = Σ (g_w w + g_T T) to the workspace (8 bytes per ray,
 * nacc_render_weights_bwd_flat_workspace_bytes), pass 2 forms Σ_{j>i} = R - prefix. */
size_t nacc_render_weights_bwd_flat_workspace_bytes(int64_t n_rays);
nacc_status nacc_render_weights_bwd_flat(const int64_t *packed_info, const int32_t *ray_id,
                                         int64_t n_rays, const float *t0, const float *t1,
                                         const float *sigma, int64_t n_samples, double neg_log_eps,
                                         const float *g_weights, const float *g_trans,
                                         float *g_sigma, void *ws, size_t ws_bytes,
                                         cudaStream_t stream);

/* Alpha compositing for fields that supply α per interval (SDF-based fields,
 * P:61; "accumulating them through alpha-composition"; DESIGN.md
 * readings #16-#17):  T_i = Π_{j<i} (1 − α_j),  w_i = T_i α_i, and w_i = 0
 * once T_i < exp(−neg_log_eps) (+inf disables).  alphas [n_samples] f32 in
 * [0, 1]; weights [n_samples] out; trans [n_samples] out (NULL allowed),
 * unmasked.  fp64 products inside. */
nacc_status nacc_render_weights_alpha_fwd(const int64_t *packed_info, int64_t n_rays,
                                          const float *alphas, int64_t n_samples,
                                          double neg_log_eps, float *weights, float *trans,
                                          cudaStream_t stream);
/* The same on ray-aligned flat tiles (an fp64 segmented product scan of 1 - α)
 * for packed samples from the sampling calls: needs ray_id [n_samples] and the
 * contiguous packing. */
nacc_status nacc_render_weights_alpha_fwd_flat(const int64_t *packed_info, const int32_t *ray_id,
                                               int64_t n_rays, const float *alphas,
                                               int64_t n_samples, double neg_log_eps,
                                               float *weights, float *trans, cudaStream_t stream);
/* Workspace for the alpha backward: 8 bytes per sample (fp64 T). */
size_t nacc_render_weights_alpha_bwd_workspace_bytes(int64_t n_samples);
/* g_α_k = [live_k] g_w_k T_k − T_k Λ_k,  Λ_k = Σ_{i>k} ([live_i] g_w_i α_i + g_T_i)
 * Π_{k<j<i} (1 − α_j)  (no division: α = 1 is safe).  g_trans may be NULL. */
nacc_status nacc_render_weights_alpha_bwd(const int64_t *packed_info, int64_t n_rays,
                                          const float *alphas, int64_t n_samples,
                                          double neg_log_eps, const float *g_weights,
                                          const float *g_trans, float *g_alphas, void *ws,
                                          size_t ws_bytes, cudaStream_t stream);
/* The same gradient on ray-aligned flat tiles for packed samples from the
 * sampling calls (ray_id [n_samples], contiguous packing); same workspace. */
nacc_status nacc_render_weights_alpha_bwd_flat(const int64_t *packed_info, const int32_t *ray_id,
                                               int64_t n_rays, const float *alphas,
                                               int64_t n_samples, double neg_log_eps,
                                               const float *g_weights, const float *g_trans,
                                               float *g_alphas, void *ws, size_t ws_bytes,
                                               cudaStream_t stream);

/* accumulate_along_rays: out[r][c] = Σ_i w_i v_i[c]; values == NULL means ones
 * (opacity, C must be 1).  1 <= C <= 64. */
nacc_status nacc_accumulate_along_rays(const int64_t *packed_info, int64_t n_rays,
                                       const float *weights, const float *values, int32_t C,
                                       int64_t n_samples, float *out, cudaStream_t stream);
/* The same sums on ray-aligned flat tiles (fp64 lane sums and warp segmented
 * scans) for packed samples from the sampling calls: needs ray_id [n_samples]
 * and the contiguous packing; C > 4 runs the one-warp-per-ray kernel. */
nacc_status nacc_accumulate_along_rays_flat(const int64_t *packed_info, const int32_t *ray_id,
                                            int64_t n_rays, const float *weights,
                                            const float *values, int32_t C, int64_t n_samples,
                                            float *out, cudaStream_t stream);
/* g_weights_i = Σ_c g_out[r][c] v_i[c]; g_values_i = w_i g_out[r] (NULL = skip). */
nacc_status nacc_accumulate_along_rays_bwd(const int64_t *packed_info, int64_t n_rays,
                                           const float *weights, const float *values, int32_t C,
                                           int64_t n_samples, const float *g_out,
                                           float *g_weights, float *g_values,
                                           cudaStream_t stream);
/* The same gradients, one thread per sample with its ray from ray_id [n_samples]
 * (any packing; ray_id must be the packed tensor's ray of every sample). */
nacc_status nacc_accumulate_along_rays_bwd_flat(const int32_t *ray_id, int64_t n_rays,
                                                const float *weights, const float *values,
                                                int32_t C, int64_t n_samples, const float *g_out,
                                                float *g_weights, float *g_values,
                                                cudaStream_t stream);

/* Fused render (Alg. 1 nerfacc.rendering(t0, t1, r_id, ...)).  On the
 * flat path n_samples is the arrays' length (a capacity); the samples in use
 * are [0, start + count of the last ray), read from packed_info on the device,
 * so the call needs no host-side total (CUDA-graph capturable).  Per ray
 *   color = Σ w rgb, opacity = Σ w, depth = Σ w m / max(opacity, 1e-10),
 *   m = (t0+t1)/2 (reading #12).  ctx [n_rays][5] fp64 out (may be NULL) keeps
 *   (C_r, C_g, C_b, O, N) for the backward.  ray_id [n_samples] (the packed
 *   tensor's r) selects the flat ray-aligned-tile kernel, which needs
 *   the contiguous packing the sampling calls produce (start_0 = 0, start_{r+1}
 *   = start_r + count_r); NULL (or rgb == NULL) falls back to one warp per ray.
 *   16-byte aligned arrays take vectorised loads. */
nacc_status nacc_render_fwd(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays,
                            const float *t0,
                            const float *t1, const float *sigma, const float *rgb,
                            int64_t n_samples, double neg_log_eps, float *color, float *opacity,
                            float *depth, double *ctx, cudaStream_t stream);
/* Backward of nacc_render_fwd (t detached): given upstream
 * g_color [n][3], g_opacity [n], g_depth [n] (each may be NULL = 0), writes
 * g_sigma [N] and g_rgb [N][3].  ctx from the forward (NULL = recompute, one
 * warp per ray); with ray_id and ctx the flat kernel runs and needs a
 * workspace of nacc_render_bwd_workspace_bytes(n_rays) bytes (per-ray
 * gradient constants; unused when g_opacity and g_depth are both NULL, a
 * colour-only loss, whose constants the kernel forms itself). */
size_t nacc_render_bwd_workspace_bytes(int64_t n_rays);
nacc_status nacc_render_bwd(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays,
                            const float *t0,
                            const float *t1, const float *sigma, const float *rgb,
                            int64_t n_samples, double neg_log_eps, const double *ctx,
                            const float *g_color, const float *g_opacity, const float *g_depth,
                            float *g_sigma, float *g_rgb, void *ws, size_t ws_bytes,
                            cudaStream_t stream);

/* Combined estimator, grid stage ("stacking an occupancy grid on
 * top of the proposal network ... reduce the number of rays and shrink the
 * near-far plane"; reading #18).  Same inputs as
 * nacc_sampling_occgrid; per ray t_near = t0 of the first interval it would
 * emit and t_far = t1 of the last (bit-identical to those t0/t1), or
 * t_near = t_far = 0 when it emits none (the ray is culled).
 *   t_near, t_far  [n_rays] f32 out
 *   n_alive        device uint64 out: rays with a span (NULL allowed)
 *   ws             nacc_sampling_occgrid_workspace_bytes() bytes */
nacc_status nacc_occgrid_ray_bounds(const nacc_grid *grid, const uint32_t *bits,
                                   const nacc_march *params, const float *rays_o,
                                   const float *rays_d, const float *t_min, const float *t_max,
                                   int64_t n_rays, float *t_near, float *t_far, uint64_t *n_alive,
                                   void *ws, size_t ws_bytes, cudaStream_t stream);

/* Proposal supervision (the "PDF matching loss" that trains the proposal
 * network; form [ext] Mip-NeRF 360, reading #21).  Dense
 * per-ray histograms, edges ascending per ray:
 *   t [n_rays][nf+1], w [n_rays][nf]      final intervals and weights
 *   th [n_rays][np+1], wh [n_rays][np]    proposal intervals and weights
 *   B_i = Σ wh_j over proposal intervals overlapping (t_i, t_{i+1})
 *   loss[r] = Σ_i max(0, w_i − B_i)² / (w_i + eps)       (f32 out, fp64 inside)
 * The backward treats w as a constant target and writes g_wh [n_rays][np]
 * from g_loss [n_rays].  nf, np >= 1; eps > 0. */
nacc_status nacc_pdf_loss(int64_t n_rays, int32_t nf, const float *t, const float *w, int32_t np,
                          const float *th, const float *wh, double eps, float *loss,
                          cudaStream_t stream);
nacc_status nacc_pdf_loss_bwd(int64_t n_rays, int32_t nf, const float *t, const float *w,
                              int32_t np, const float *th, const float *wh, double eps,
                              const float *g_loss, float *g_wh, cudaStream_t stream);

/* ------------------------------------------------------------------------ */
/* Proposal estimator: inverse-transform resampling (Eq. 1) of the  */
/* CDF F = 1 - T (Eq. 3, "compute the CDF directly using 1 - T(t)", */
/* P:220) in s-space.  Per ray, edges e_0..e_m (ascending, in s) and   */
/* either sigma [m] (F_j = 1 - exp(-Σ_{i<j} σ_i (Φ(e_{i+1}) - Φ(e_i)))) or a    */
/* given cdf [m+1]; F̂ = F normalised to [0,1] (uniform if the mass <= 1e-12,   */
/* reading #16).  Output edges s_i = F̂^{-1}(u_i), u_i = i/n_out (i = 0..n_out) */
/* or stratified u_i = (i + ξ_{r,i})/(n_out+1) with ξ = Philox(seed,(r,i,1)),   */
/* linear within each bin; t_out = Φ(s_out) (may be NULL).                      */
/* ------------------------------------------------------------------------ */
typedef enum { NACC_MAP_IDENTITY = 0, NACC_MAP_LINDISP = 1 } nacc_map;
nacc_status nacc_importance_sample(int64_t n_rays, int32_t n_in, const float *s_edges,
                                   const float *sigma, const float *cdf, nacc_map map,
                                   double t_near, double t_far, int32_t n_out,
                                   int32_t stratified, uint64_t seed, float *s_out, float *t_out,
                                   cudaStream_t stream);
/* The same with each ray's own span [t_near[r], t_far[r]] (f32 device arrays,
 * e.g. from nacc_occgrid_ray_bounds; the combined estimator's proposal stage,
 * reading #19).  A ray with !(t_far > t_near) is culled: s_out = uniform
 * edges over [e_0, e_m], t_out = t_near.  Device precondition (unchecked):
 * t_near > 0 on live rays for the lindisp map. */
nacc_status nacc_importance_sample_ranged(int64_t n_rays, int32_t n_in, const float *s_edges,
                                          const float *sigma, const float *cdf, nacc_map map,
                                          const float *t_near, const float *t_far, int32_t n_out,
                                          int32_t stratified, uint64_t seed, float *s_out,
                                          float *t_out, cudaStream_t stream);

/* ------------------------------------------------------------------------ */
/* Occupancy-grid estimator update (EMA σ^k = γσ^{k-1} + (1-γ)σ_q,  */
/* binarise σ̂ = 1[σ > τ]; readings #20-#23).                                  */
/* ------------------------------------------------------------------------ */
typedef enum { NACC_UPDATE_EMA = 0, NACC_UPDATE_MAX_DECAY = 1 } nacc_update_rule;
typedef enum { NACC_THRESH_FIXED = 0, NACC_THRESH_MIN_MEAN = 1 } nacc_thresh_rule;

/* Query points for cells [cell_begin, cell_begin+cell_count): level l, index
 * (i,j,k): x = lo_l + (i + ξ)(hi_l - lo_l)/R in fp64, rounded once; ξ from
 * Philox(seed, (cell_in_level, step, l, 2)) or 1/2 when jitter == 0.
 * xyz [cell_count][3] out. */
nacc_status nacc_occgrid_points(const nacc_grid *grid, uint64_t seed, int64_t step,
                                int32_t jitter, int64_t cell_begin, int64_t cell_count,
                                float *xyz, cudaStream_t stream);
size_t nacc_occgrid_workspace_bytes(const nacc_grid *grid);
/* density [levels*res^3] in/out (fp32 state, updated with fp64 arithmetic,
 * rounded once); fresh [levels*res^3] = the caller's σ(x)·Δt at the points
 * (after the MAX all-reduce across ranks); bits out; mean (device double,
 * NULL allowed) = mean of the updated density. */
nacc_status nacc_occgrid_update(const nacc_grid *grid, float *density, const float *fresh,
                                nacc_update_rule rule, float decay, float threshold,
                                nacc_thresh_rule thresh_rule, uint32_t *bits, double *mean,
                                void *ws, size_t ws_bytes, cudaStream_t stream);
/* (bits: the full nacc_grid_bits_bytes() buffer; its private region is rebuilt.) */
/* Dynamic scenes (one grid shared across frames holds "the maximum
 * opacity at this area over all the timestamps"; reading #20).
 * times[q] = draw `draw` of cell (cell_begin + q)'s timestamp in [0, 1):
 * u24(Philox4x32-10(seed, (cell index in level, step, level, 16 + draw)).x).
 * The caller evaluates σ(x, t) at (nacc_occgrid_points, times) for each draw
 * and folds the draws into `fresh` with nacc_max_merge before the update. */
nacc_status nacc_occgrid_times(const nacc_grid *grid, uint64_t seed, int64_t step, int32_t draw,
                               int64_t cell_begin, int64_t cell_count, float *times,
                               cudaStream_t stream);
/* dst[i] = max(dst[i], src[i]) for i < n (device f32 arrays). */
nacc_status nacc_max_merge(float *dst, const float *src, int64_t n, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* NACC_H */
